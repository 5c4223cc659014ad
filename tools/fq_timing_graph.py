"""Fused-step kernel timeline under the bench's conditions (CUDA graph replay, rotating
cold inputs): globaltimer stamps of CTA 0 (experiment build -DQF_FQ_TIMING,
QFLASH_LIB=libqflash_fqt.so), for the last two steps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_25306_b200 as qf  # noqa: E402
from paper_2604_25306_b200.inputs import CATALOG, gen_real_qkv  # noqa: E402

names = {8: "entry", 0: "prologue", 1: "amax", 2: "sync1", 3: "constants", 4: "quantized",
         5: "sync2", 9: "teardown", 13: "w1:scales", 6: "w1:quantized", 7: "w1:fenced",
         10: "w1:sync2", 12: "lastCTA:teardown", 14: "w1:dq", 15: "w1:rcp", 16: "w1:qfast"}
for wl, b in [("A3", 8), ("A4", 8), ("A1", 1)]:
    w = CATALOG[wl]
    P, N, d = w.problems(b), w.seq_len, w.head_dim
    base = [torch.from_numpy(x).cuda() for x in gen_real_qkv(P, N, d, seed=0, family=w.family)]
    n_sets = int(os.environ.get("FQ_SETS", "12"))
    sets = [[(t * (-1.0 if i % 2 else 1.0)).roll(shifts=i, dims=1).contiguous() for t in base]
            for i in range(n_sets)]
    pipes = [qf.QFlashPipeline(P, N, d) for _ in range(n_sets)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for p, x in zip(pipes, sets):
            p(*x)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for p, x in zip(pipes, sets):
            p(*x)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"== {wl} b{b}: {e0.elapsed_time(e1) * 1e3 / (20 * n_sets):.2f} us per step (graph)")
    stamps = [p.workspace.view(torch.int64)[768:785].cpu().numpy() for p in pipes]
    t0 = stamps[0][8]
    for i in (n_sets - 2, n_sets - 1):
        st = stamps[i]
        print(f"  step {i}: " + "  ".join(f"{names[k]} {(st[k] - st[8]) / 1e3:.2f}" for k in [0, 1, 2, 13, 14, 15, 16, 3, 6, 7, 4, 5, 10, 9, 12])
              + f"  | entry after prev teardown: {(st[8] - stamps[i - 1][9]) / 1e3:.2f} us")
