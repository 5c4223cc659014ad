"""CTA-0 timeline of the fused step kernel (experiment build with -DQF_FQ_TIMING,
QFLASH_LIB=libqflash_fqt.so): globaltimer stamps written into the workspace."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_25306_b200 as qf  # noqa: E402
from paper_2604_25306_b200.inputs import CATALOG, gen_real_qkv  # noqa: E402

names = {8: "kernel entry", 0: "prologue start", 1: "amax done", 2: "grid sync 1", 3: "constants derived",
         4: "quantized", 5: "grid sync 2", 9: "teardown"}
for wl, b in [("A1", 1), ("A3", 8), ("A4", 8)]:
    w = CATALOG[wl]
    P, N, d = w.problems(b), w.seq_len, w.head_dim
    q, k, v = (torch.from_numpy(x).cuda() for x in gen_real_qkv(P, N, d, seed=0, family=w.family))
    pipe = qf.QFlashPipeline(P, N, d, mode="fused")
    for _ in range(5):
        pipe(q, k, v)
    torch.cuda.synchronize()
    ts = pipe.workspace.view(torch.int64)[768:778].cpu().numpy()
    t0 = ts[8]
    print(f"== {wl} b{b}")
    for kk in [8, 0, 1, 2, 3, 4, 5, 9]:
        print(f"   {names[kk]:20s} {(ts[kk] - t0) / 1e3:8.2f} us")
