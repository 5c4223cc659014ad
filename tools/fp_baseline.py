"""Context for SURVEY 8(f) N4 (the paper's V0 = floating-point FlashAttention): torch SDPA
in bf16 / fp16 on the same [P, N, d] problems, CUDA-event timed, next to this library's
integer attention (int8 in, fused fp32 dequantized out) and its whole fused step."""
import json
import os
import statistics
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_25306_b200 as qf  # noqa: E402
from paper_2604_25306_b200.inputs import CATALOG, gen_real_qkv  # noqa: E402


def timed(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    return statistics.median(ts)


rows = []
for wl, b in [("A3", 8), ("A4", 8), ("L14", 64)]:
    w = CATALOG[wl]
    P, N, d = w.problems(b), w.seq_len, w.head_dim
    q, k, v = (torch.from_numpy(x).cuda() for x in gen_real_qkv(P, N, d, seed=0, family=w.family))
    r = {"workload": f"{wl} b{b}", "P": P, "N": N, "d": d}
    for dt in (torch.bfloat16, torch.float16):
        qq, kk, vv = (t.to(dt).unsqueeze(0) for t in (q, k, v))
        r[f"sdpa_{str(dt).split('.')[-1]}_us"] = timed(lambda: F.scaled_dot_product_attention(qq, kk, vv))
    pipe = qf.QFlashPipeline(P, N, d, mode="two")
    pipe(q, k, v)
    r["qflash_attention_int8_us"] = timed(lambda: qf.qflash_attention_dequant_prepared(
        pipe.qkv_q[0], pipe.qkv_q[1], pipe.qkv_q[2], pipe.workspace, out=pipe.out))
    fused = qf.QFlashPipeline(P, N, d, mode="fused")
    r["qflash_fused_step_us"] = timed(lambda: fused(q, k, v))
    rows.append(r)
    print(json.dumps(r))
