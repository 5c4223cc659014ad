"""Small parity cases for compute-sanitizer runs (tools/gpu_sanitize.sh)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2604_25306_b200 as qf  # noqa: E402
from paper_2604_25306_b200.inputs import gen_int8_qkv, gen_workload  # noqa: E402

oracle.build()
ok = True
for (N, d, P, var) in [(197, 64, 4, "packed"), (300, 64, 3, "generic"), (49, 32, 40, "packed")]:
    q, k, v = gen_int8_qkv(P, N, d, seed=1)
    dq, dk, dv = (torch.from_numpy(x).cuda() for x in (q, k, v))
    out, _ = qf.qflash_attention_int8(dq, dk, dv, 0.05, 0.05, 0.03, variant=var)
    ref = oracle.attention(q, k, v, 0.05, 0.05)
    ok &= np.array_equal(out.cpu().numpy(), ref)
q, k, v = gen_workload("A1", 1, seed=0)
y = qf.qflash_forward(*(torch.from_numpy(x) for x in (q, k, v)))
print("parity", ok)
# per-head path and the two-launch pipeline
q, k, v = gen_workload("A4", 1, seed=2)
dq, dk, dv = (torch.from_numpy(x).cuda() for x in (q, k, v))
y, o, sc, ws = qf.qflash_forward_per_head(dq, dk, dv, 3)
y2 = qf.QFlashPipeline(*q.shape, mode="two")(dq, dk, dv)
torch.cuda.synchronize()
print("per-head status", int(ws[0].item()))
# fused one-launch step on the cooperative (grid.sync) path: A3 b8 (148 CTAs) vs the
# multi-launch pipeline's output, and the A4 b2 streamed-quantize case
for wl, b in (("A3", 8), ("A4", 2)):
    q, k, v = gen_workload(wl, b, seed=3)
    dq, dk, dv = (torch.from_numpy(x).cuda() for x in (q, k, v))
    yf = qf.QFlashPipeline(*q.shape, mode="fused")(dq, dk, dv).clone()
    yt = qf.QFlashPipeline(*q.shape, mode="three")(dq, dk, dv)
    torch.cuda.synchronize()
    print("fused", wl, b, bool(torch.equal(yf.view(torch.int32), yt.view(torch.int32))))
