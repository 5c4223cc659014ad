"""Does the second grid barrier wait on L2 write-allocation?  Fused step, chained graphs over
12 rotating cold input sets, with (a) separate codes / workspace / y per set (bench.py), (b) one
shared codes + workspace (scratch reused across calls, as a model forward would) and a
distinct y per set, (c) everything shared."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_25306_b200 as qf  # noqa: E402
from paper_2604_25306_b200.inputs import CATALOG, gen_real_qkv  # noqa: E402


def chain_ms(fns, reps=200):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for f in fns:
            f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for f in fns:
            f()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(2_000_000)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / len(fns) * 1e3


for wl, b in [("A3", 8), ("A1", 1), ("A4", 8), ("A2", 8)]:
    w = CATALOG[wl]
    P, N, d = w.problems(b), w.seq_len, w.head_dim
    base = [torch.from_numpy(x).cuda() for x in gen_real_qkv(P, N, d, seed=0, family=w.family)]
    n = 12
    sets = [[(t * (-1.0 if i % 2 else 1.0)).roll(shifts=i, dims=1).contiguous() for t in base] for i in range(n)]
    pipes = [qf.QFlashPipeline(P, N, d) for _ in range(n)]
    p0 = pipes[0]
    fa = [lambda p=p, x=x: p(*x) for p, x in zip(pipes, sets)]
    fb = [lambda p=p, x=x: qf.qflash_forward_fused(*x, 128, "auto", out=p.out, codes=p0.qkv_q, scales=p0.scales,
                                                   workspace=p0.workspace) for p, x in zip(pipes, sets)]
    fc = [lambda x=x: p0(*x) for x in sets]
    r = [chain_ms(f) for f in (fa, fb, fc)]
    print(f"{wl} b{b}: separate {r[0]:.2f} us | shared codes+workspace, own y {r[1]:.2f} us | all shared {r[2]:.2f} us")
