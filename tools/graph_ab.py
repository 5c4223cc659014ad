"""Marginal cost of each step stage inside CUDA graphs (rotating cold inputs).

Graphs: Q (quantize_qkv_prepare), QA (+ attention), QAD (whole step), A, D.
python tools/graph_ab.py [--workload A3 --batch 8]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_25306_b200 as qfl  # noqa: E402
from paper_2604_25306_b200.inputs import CATALOG, gen_real_qkv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="A3")
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--steps", type=int, default=3000)
a = ap.parse_args()
w = CATALOG[a.workload]
P, N, d = w.problems(a.batch), w.seq_len, w.head_dim
dev = torch.device("cuda", 0)
set_bytes = 3 * 4 * P * N * d + 4 * P * N * d
n_sets = int(min(64, max(2, np.ceil(2.0 * 126 * 2**20 / set_bytes) + 1)))
q0, k0, v0 = gen_real_qkv(P, N, d, seed=0, family=w.family)
base = [torch.from_numpy(x).to(dev) for x in (q0, k0, v0)]
sets = [[(t * (-1.0 if i % 2 else 1.0)).roll(shifts=i, dims=1).contiguous() for t in base]
        for i in range(n_sets)]
pipes = [qfl.QFlashPipeline(P, N, d, device=dev) for _ in range(n_sets)]
stream = torch.cuda.Stream(device=dev)


def stages(p, s, which):
    if "Q" in which:
        qfl.qflash_quantize_qkv_prepare(*s, outs=p.qkv_q, scales=p.scales, workspace=p.workspace,
                                        stream=stream)
    if "A" in which:
        qfl.qflash_attention_int8_prepared(p.qkv_q[0], p.qkv_q[1], p.qkv_q[2], p.workspace,
                                           out=p.o_q, stream=stream)
    if "D" in which:
        qfl.qflash_dequantize(p.o_q, p.scales[2:3], out=p.out, stream=stream)


with torch.cuda.stream(stream):
    for p, s in zip(pipes, sets):
        p(*s)
torch.cuda.synchronize()
for which in ["QAD", "Q", "A", "D", "QA", "AD", "QAD"]:
    # one graph = n_sets consecutive steps (host replay cost amortised)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(g, stream=stream):
            for p, s in zip(pipes, sets):
                stages(p, s, which)
    torch.cuda.synchronize()
    reps = max(1, a.steps // n_sets)
    with torch.cuda.stream(stream):
        for i in range(3):
            g.replay()
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(reps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    print(f"{a.workload} b{a.batch} graph {which:4s}: {e0.elapsed_time(e1) / (reps * n_sets) * 1e3:8.2f} us/step")
