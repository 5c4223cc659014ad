"""fig:tile_sqnr on B200 (App. B.1): SQNR against the number
of KV tiles (inner-loop iterations T_c) for Scale Release (Eq. 14, the method) and Scale
Accumulation (Eq. 13), both computed by the CUDA kernels and, for the shorter prefixes,
checked bit-exactly against the CPU oracle's mode 0 / mode 1.

Workload: N = 4096 tokens, d = 64, 4 problems, the SURVEY 8(d) ViT recipe (seed 0);
block_kv = 64, prefix N_t = 64 T_c (Q rows and K/V keys of the first N_t tokens).  The
reference is FP64 softmax attention on the real inputs (oracle/fp_reference.py).
Writes profiles/r2_tile_sqnr.md.  Run on the GPU box: python tools/tile_sqnr_sweep.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (test infrastructure: the reference and the bit-exact check)
import paper_2604_25306_b200 as qf  # noqa: E402
from oracle.fp_reference import attention_fp64, sqnr_db  # noqa: E402
from paper_2604_25306_b200.inputs import gen_real_qkv  # noqa: E402

N, D, P, BKV = 4096, 64, 4, 64
q, k, v = gen_real_qkv(P, N, D, seed=0, family="vit")
rows = []
for tc in (1, 2, 3, 4, 5, 6, 8, 12, 16, 24, 32, 48, 64):
    n = BKV * tc
    qs, ks, vs = (np.ascontiguousarray(x[:, :n]) for x in (q, k, v))
    dq, dk, dv = (torch.from_numpy(x).cuda() for x in (qs, ks, vs))
    (cq, sq), (ck, sk), (cv, sv) = (qf.qflash_quantize_per_tensor(x) for x in (dq, dk, dv))
    sq, sk, sv = (float(s.item()) for s in (sq, sk, sv))
    rel, _ = qf.qflash_attention_int8(cq, ck, cv, sq, sk, sv, block_kv=BKV)
    acc, flags = qf.qflash_attention_int8_accum(cq, ck, cv, sq, sk, block_kv=BKV)
    torch.cuda.synchronize()
    ref = attention_fp64(qs, ks, vs)
    y_rel = rel.cpu().numpy().astype(np.float64) * sv
    y_acc = acc.cpu().numpy().astype(np.float64) * sv
    f = int(flags.item())
    exact = "-"
    if tc <= 8:  # the oracle finishes these in seconds
        oq, ok_, ov = cq.cpu().numpy(), ck.cpu().numpy(), cv.cpu().numpy()
        o0 = oracle.attention(oq, ok_, ov, sq, sk, block_kv=BKV, mode=0, nthreads=os.cpu_count() or 1)
        o1, ovf = oracle.attention(oq, ok_, ov, sq, sk, block_kv=BKV, mode=1, return_overflow=True,
                                   nthreads=os.cpu_count() or 1)
        same = np.array_equal(o0, rel.cpu().numpy()) and np.array_equal(o1, acc.cpu().numpy()) and \
            bool(f & 1) == ovf
        exact = "yes" if same else "NO"
    rows.append((tc, n, sqnr_db(ref, y_rel), sqnr_db(ref, y_acc), bool(f & 2), bool(f & 1), exact))
    print(rows[-1], flush=True)

out = os.path.join(ROOT, "profiles", "r2_tile_sqnr.md")
with open(out, "w") as fh:
    fh.write("# fig:tile_sqnr on B200 -- Scale Release (Eq. 14) vs Scale Accumulation (Eq. 13)\n\n")
    fh.write("`python tools/tile_sqnr_sweep.py` (GPU kernels; oracle bit-exact check for T_c <= 8). "
             "N = 4096 ViT-recipe tokens, d = 64, 4 problems, block_kv = 64, prefix N_t = 64 T_c; SQNR in dB "
             "against FP64 attention on the real inputs (P:L691-697).  Accumulation overflow flags: int32 = "
             "an int32-accumulator kernel would have overflowed, int64 = the int64 accumulators wrapped.\n\n")
    fh.write("| T_c | N_t | SQNR release | SQNR accumulation | int32 ovf | int64 ovf | GPU == oracle |\n")
    fh.write("|---|---|---|---|---|---|---|\n")
    for r in rows:
        fh.write("| %d | %d | %.2f | %.2f | %s | %s | %s |\n" % r)
print("wrote", out)
