"""Diagnose parity failures on the GPU (run by hand under gpurun)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2604_25306_b200 as qf  # noqa: E402
from paper_2604_25306_b200 import _lib  # noqa: E402
from paper_2604_25306_b200.inputs import gen_int8_qkv  # noqa: E402

VAR = {"generic": 1, "packed": 2}
bad = []
for d in (32, 64, 128):
    for N in [1, 2, 31, 32, 33, 48, 49, 50, 63, 64, 65, 127, 128, 129, 196, 197, 255, 256, 257]:
        q, k, v = gen_int8_qkv(3, N, d, seed=N + d)
        dq, dk, dv = (torch.from_numpy(t).cuda() for t in (q, k, v))
        for bkv in (64, 128, 256):
            ref = oracle.attention(q, k, v, 0.05, 0.05, block_kv=bkv)
            for var in (["generic", "packed"] if N <= 64 else ["generic"]):
                out, _ = qf.qflash_attention_int8(dq, dk, dv, 0.05, 0.05, 0.03, block_kv=bkv, variant=var)
                got = out.cpu().numpy()
                nbad = int((got != ref).sum())
                if nbad:
                    rows = np.unique(np.nonzero(got != ref)[1])
                    probs = np.unique(np.nonzero(got != ref)[0])
                    cols = np.unique(np.nonzero(got != ref)[2])
                    bad.append((d, N, bkv, var))
                    print(f"FAIL d={d} N={N} bkv={bkv} {var}: {nbad} bad; problems {probs[:5]} rows {rows[:10]}..{rows[-3:]} cols {cols[:8]}..{cols[-3:]}")
print("failures:", len(bad))
# stage dump for the first failure
if bad:
    d, N, bkv, var = bad[0]
    q, k, v = gen_int8_qkv(3, N, d, seed=N + d)
    dq, dk, dv = (torch.from_numpy(t).cuda() for t in (q, k, v))
    BC = 128 if var == "packed" else bkv
    ds = torch.full((128 * BC,), -7, dtype=torch.int32, device="cuda")
    dp = torch.full((128 * BC // 4,), -7, dtype=torch.int32, device="cuda")
    do = torch.full((128 * (d + 1),), -7, dtype=torch.int32, device="cuda")
    o = torch.empty_like(dq)
    sh = _lib.AttnShape(3, N, d, bkv)
    st = _lib.lib().qflash_debug_attention(dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), 0.05, 0.05,
                                           ctypes.byref(sh), VAR[var], o.data_ptr(), ds.data_ptr(),
                                           dp.data_ptr(), do.data_ptr(), None, None)
    torch.cuda.synchronize()
    rows = min(N, 128 if var == "generic" else 64)
    cols = min(N, BC) if var == "generic" else min(N, 64)
    S = ds.cpu().numpy().reshape(128, BC)
    Sref = q[0, :rows].astype(np.int64) @ k[0, :cols].astype(np.int64).T
    print("S ok:", np.array_equal(S[:rows, :cols], Sref))
    _, l_ref, o_ref = oracle.attention_rows_state(q, k, v, 0.05, 0.05, 0, 0, rows, block_kv=bkv)
    og = do.cpu().numpy().reshape(128, d + 1)
    print("l ok:", np.array_equal(og[:rows, d], l_ref), "O ok:", np.array_equal(og[:rows, :d], o_ref))
    if not np.array_equal(og[:rows, :d], o_ref):
        bc = np.unique(np.nonzero(og[:rows, :d] != o_ref)[1])
        br = np.unique(np.nonzero(og[:rows, :d] != o_ref)[0])
        print("O bad cols", bc[:20], "rows", br[:20])
        print("O gpu", og[br[0], bc[:6]], "ref", o_ref[br[0], bc[:6]])
    if not np.array_equal(og[:rows, d], l_ref):
        print("l gpu", og[:6, d], "ref", l_ref[:6])
    Pw = dp.cpu().numpy().reshape(128, BC // 4).view(np.uint32)
    Pg = np.zeros((128, BC), np.int64)
    for b in range(4):
        Pg[:, b::4] = ((Pw >> (8 * b)) & 0xFF).astype(np.int64)
    prm = oracle.derive_params(0.05, 0.05, d)
    m = Sref.max(-1, keepdims=True)
    y = oracle.shift_exp2_array((Sref - m).ravel(), prm["s_inv"]).reshape(Sref.shape)
    Pref = np.minimum(127, (y * prm["m_p"]) >> prm["r_p"])
    print("P ok (tile0):", np.array_equal(Pg[:rows, :cols], Pref), "P beyond valid zero:", not Pg[:rows, cols:].any())
