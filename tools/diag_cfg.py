"""Localise attention mismatches vs the oracle per kernel configuration (GPU)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2604_25306_b200 as qf  # noqa: E402
from paper_2604_25306_b200.inputs import gen_int8_qkv  # noqa: E402

oracle.build()
cases = [(197, 64, 151, 64, "packed"), (197, 64, 151, 128, "packed"), (197, 64, 151, 128, "generic"), (127, 32, 3, 64, "generic"),
         (127, 32, 3, 64, "packed"), (64, 32, 300, 64, "generic"), (197, 64, 400, 128, "generic"),
         (49, 32, 1536, 64, "packed"), (1025, 64, 6, 128, "generic")]
for (N, d, P, bkv, var) in cases:
    q, k, v = gen_int8_qkv(P, N, d, seed=N * 7 + P)
    ref = oracle.attention(q, k, v, 0.05, 0.05, block_kv=bkv)
    dq, dk, dv = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (q, k, v))
    out, _ = qf.qflash_attention_int8(dq, dk, dv, 0.05, 0.05, 0.03, block_kv=bkv, variant=var)
    got = out.cpu().numpy()
    bad = (got != ref).any(axis=2)
    rows = np.argwhere(bad)
    flat = rows[:, 0] * N + rows[:, 1] if rows.size else np.array([], dtype=np.int64)
    tiles = np.unique(flat // 128) if var == "packed" else np.unique(rows[:, 0] * ((N + 127) // 128) + rows[:, 1] // 128) if rows.size else []
    print(f"N={N} d={d} P={P} bkv={bkv} {var}: bad rows {int(bad.sum())}/{P*N}; tiles {list(tiles)[:12]} "
          f"(n={len(tiles)}); first {rows[:4].tolist()}; maxdiff {int(np.abs(got.astype(int)-ref).max())}")
    sys.stdout.flush()
