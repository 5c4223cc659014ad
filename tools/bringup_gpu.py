"""GPU bring-up diagnostics (run by hand under gpurun; not a pytest module).

Checks the stages of one CTA of the fused kernel against the oracle: S (step 1),
packed P (steps 5-6), final O and l (steps 7-10), then the int8 output."""
import ctypes
import os
import sys
import traceback

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2604_25306_b200 import _lib  # noqa: E402
from paper_2604_25306_b200.inputs import gen_int8_qkv, gen_workload  # noqa: E402


def run(P, N, d, bkv, variant, kind="uniform", sq=0.05, sk=0.05, seed=0):
    q, k, v = gen_int8_qkv(P, N, d, seed=seed, kind=kind)
    dq, dk, dv = (torch.from_numpy(t).cuda() for t in (q, k, v))
    o = torch.empty_like(dq)
    BC = 128 if variant == 2 else bkv
    ds = torch.full((128 * BC,), -7, dtype=torch.int32, device="cuda")
    dp = torch.full((128 * BC // 4,), -7, dtype=torch.int32, device="cuda")
    do = torch.full((128 * (d + 1),), -7, dtype=torch.int32, device="cuda")
    sh = _lib.AttnShape(P, N, d, bkv)
    st = _lib.lib().qflash_debug_attention(dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), sq, sk,
                                           ctypes.byref(sh), variant, o.data_ptr(), ds.data_ptr(),
                                           dp.data_ptr(), do.data_ptr(), None, None)
    torch.cuda.synchronize()
    print(f"--- P={P} N={N} d={d} bkv={bkv} variant={variant} kind={kind}: status {st} {_lib.last_error()}")
    S_gpu = ds.cpu().numpy().reshape(128, BC)
    q64, k64 = q.astype(np.int64), k.astype(np.int64)
    if variant == 2:
        rows = min(N, 64)
        S_ref0 = q64[0, :rows] @ k64[0, :rows].T
        ok0 = np.array_equal(S_gpu[:rows, :rows], S_ref0)
        msg = f"S window0 match={ok0}"
        if P > 1:
            S_ref1 = q64[1, :rows] @ k64[1, :rows].T
            ok1 = np.array_equal(S_gpu[64:64 + rows, 64:64 + rows], S_ref1)
            msg += f" window1 match={ok1}"
        print(msg)
    else:
        rows = min(N, 128)
        cols = min(N, BC)
        S_ref = q64[0, :rows] @ k64[0, :cols].T
        sub = S_gpu[:rows, :cols]
        print("S match:", np.array_equal(sub, S_ref), "mismatches", int((sub != S_ref).sum()), "of", sub.size)
        if not np.array_equal(sub, S_ref):
            print("S_gpu[0,:8]", sub[0, :8], "\nS_ref[0,:8]", S_ref[0, :8])
            print("S_gpu[1,:8]", sub[1, :8], "\nS_ref[1,:8]", S_ref[1, :8])
        # P of tile 0
        prm = oracle.derive_params(sq, sk, d)
        m = S_ref.max(-1, keepdims=True)
        y = oracle.shift_exp2_array((S_ref - m).ravel(), prm["s_inv"]).reshape(S_ref.shape)
        Pref = np.minimum(127, (y * prm["m_p"]) >> prm["r_p"])
        Pw = dp.cpu().numpy().reshape(128, BC // 4).view(np.uint32)
        Pg = np.zeros((128, BC), np.int64)
        for b in range(4):
            Pg[:, b::4] = ((Pw >> (8 * b)) & 0xFF).astype(np.int64)
        okp = np.array_equal(Pg[:rows, :cols], Pref)
        print("P match:", okp, "mismatch", int((Pg[:rows, :cols] != Pref).sum()))
        if not okp:
            print("Pg[0,:12]", Pg[0, :12], "\nPr[0,:12]", Pref[0, :12])
    # final O/l vs oracle state
    nrow = min(N, 128)
    _, l_ref, o_ref = oracle.attention_rows_state(q, k, v, sq, sk, 0, 0, nrow, block_kv=bkv if variant != 2 else 256)
    og = do.cpu().numpy().reshape(128, d + 1)
    print("l match:", np.array_equal(og[:nrow, d], l_ref), "O match:", np.array_equal(og[:nrow, :d], o_ref))
    if not np.array_equal(og[:nrow, d], l_ref):
        print("l_gpu", og[:6, d], "l_ref", l_ref[:6])
    if not np.array_equal(og[:nrow, :d], o_ref):
        print("O_gpu", og[0, :6], "O_ref", o_ref[0, :6])
    ref = oracle.attention(q, k, v, sq, sk, block_kv=bkv if variant != 2 else 256)
    out = o.cpu().numpy()
    print("OUT match:", np.array_equal(out, ref), "mismatch", int((out != ref).sum()), "of", out.size)
    return np.array_equal(out, ref)


if __name__ == "__main__":
    import paper_2604_25306_b200 as q
    print("device", torch.cuda.get_device_name(), torch.cuda.get_device_capability())
    cases = [(1, 128, 64, 128, 1), (1, 197, 64, 128, 1), (3, 197, 64, 64, 1), (2, 49, 32, 128, 2),
             (3, 49, 32, 128, 1), (2, 300, 128, 256, 1), (2, 100, 32, 64, 1)]
    for c in cases:
        try:
            run(*c)
        except Exception:
            traceback.print_exc()
    # quantizer
    try:
        x = torch.randn(1000003, device="cuda") * 3
        xq, s = q.qflash_quantize_per_tensor(x)
        rq, rs = oracle.quantize(x.cpu().numpy())
        print("quant scale", s.item(), rs, "bytes match", np.array_equal(xq.cpu().numpy(), rq))
    except Exception:
        traceback.print_exc()
