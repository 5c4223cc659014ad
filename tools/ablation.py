"""Ablation analog on B200 (the paper's V0-V4 ladder P:L737-752 and the
energy context P:L523-562): per workload, graph-timed µs per call on cold rotating sets of
  V0  torch SDPA (bf16, flash backend) on the real inputs    -- floating-point reference
  V2  int8 Q K^T + FP exp2 softmax + int8 P V + FP accumulation (qflash_attention_ablation)
  V3  int8 Q K^T + integer ShiftExp2 + int8 P V + FP accumulation
  V4  QFlash: all integer (qflash_attention_int8, int8 out)
with SQNR against FP64 attention, and the energy per call of V4 / V0 from the NVML total
energy counter over >= 2 s of back-to-back calls.  V1 (int8 Q K^T only, FP16 P V) needs an
fp16 V operand path and is not built.  Writes profiles/r2_ablation.md (run on the GPU box)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_25306_b200 as qf  # noqa: E402
from oracle.fp_reference import attention_fp64, sqnr_db  # noqa: E402  (test infrastructure)
from paper_2604_25306_b200.inputs import CATALOG, gen_workload  # noqa: E402

L2 = 126 * 2 ** 20


def gtime(fns, reps=400):
    s = torch.cuda.Stream()
    gs = []
    with torch.cuda.stream(s):
        for f in fns:
            f()
        torch.cuda.synchronize()
        for f in fns:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                f()
            gs.append(g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        for i in range(10):
            gs[i % len(gs)].replay()
        torch.cuda._sleep(2_000_000)
        e0.record(s)
        for i in range(reps):
            gs[i % len(gs)].replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps, gs, s


def energy_uj(gs, s, seconds=2.0):
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    except Exception:
        return None
    n = 0
    torch.cuda.synchronize()
    e_a = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)  # mJ
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        while time.perf_counter() - t0 < seconds:
            for i in range(200):
                gs[(n + i) % len(gs)].replay()
            n += 200
            torch.cuda.synchronize()
    e_b = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
    return (e_b - e_a) * 1e3 / n


rows = []
for name, batch in (("A2", 8), ("A3", 8), ("A7", 8), ("L14", 8)):
    w = CATALOG[name]
    q, k, v = gen_workload(name, batch, seed=0)
    P, N, d = q.shape
    ref = attention_fp64(q, k, v)
    nsets = int(max(2, min(16, np.ceil(2 * L2 / (P * N * d * 8)))))
    sets = []
    for i in range(nsets):
        sg = -1.0 if i % 2 else 1.0
        x = [torch.from_numpy(np.roll(a * sg, i, axis=1)).cuda() for a in (q, k, v)]
        codes = [qf.qflash_quantize_per_tensor(t) for t in x]
        sets.append((x, [c for c, _ in codes], [float(s.item()) for _, s in codes]))
    outs8 = [torch.empty((P, N, d), dtype=torch.int8, device="cuda") for _ in sets]
    outsf = [torch.empty((P, N, d), dtype=torch.float32, device="cuda") for _ in sets]
    x0 = sets[0]
    t4, g4, s4 = gtime([lambda c=c, o=o: qf.qflash_attention_int8(*c[1], *c[2], out=o) for c, o in zip(sets, outs8)])
    t3, _, _ = gtime([lambda c=c, o=o: qf.qflash_attention_ablation(*c[1], *c[2], "V3", out=o)
                      for c, o in zip(sets, outsf)])
    t2, _, _ = gtime([lambda c=c, o=o: qf.qflash_attention_ablation(*c[1], *c[2], "V2", out=o)
                      for c, o in zip(sets, outsf)])
    bf = [[t.to(torch.bfloat16).view(P, 1, N, d) for t in c[0]] for c in sets]
    t0, g0, s0 = gtime([lambda b=b: torch.nn.functional.scaled_dot_product_attention(*b) for b in bf])
    sv = x0[2][2]
    y4 = qf.qflash_attention_int8(*x0[1], *x0[2])[0].cpu().numpy().astype(np.float64) * sv
    y3 = qf.qflash_attention_ablation(*x0[1], *x0[2], "V3").cpu().numpy()
    y2 = qf.qflash_attention_ablation(*x0[1], *x0[2], "V2").cpu().numpy()
    y0 = torch.nn.functional.scaled_dot_product_attention(*bf[0]).float().view(P, N, d).cpu().numpy()
    e4 = energy_uj(g4, s4) if name == "A2" else None
    e0 = energy_uj(g0, s0) if name == "A2" else None
    rows.append((f"{name} b{batch}", t0, t2, t3, t4, sqnr_db(ref, y0), sqnr_db(ref, y2), sqnr_db(ref, y3),
                 sqnr_db(ref, y4), e0, e4))
    print(rows[-1], flush=True)

with open(os.path.join(ROOT, "profiles", "r2_ablation.md"), "w") as fh:
    fh.write("# Ablation analog on B200 (SURVEY 8(f) N4; paper ladder P:L737-752)\n\n")
    fh.write("`python tools/ablation.py` on one B200: graph-timed µs per call over rotating cold input "
             "sets (int8 codes from qflash_quantize_per_tensor; the quantizer is not timed), SQNR "
             "against FP64 attention on the real inputs.  V0 = torch SDPA bf16 (library flash kernel, "
             "context), V2 = int8 QK + FP exp2 softmax + int8 PV + FP accumulation, V3 = int8 QK + "
             "integer ShiftExp2 + int8 PV + FP accumulation, V4 = QFlash (all integer).  Energy: NVML "
             "total-energy counter over >= 2 s of back-to-back calls (A2 b8 only; paper context "
             "754.6 µJ QFlash vs 929.6 µJ I-ViT on the RTX 5090, P:L523-562).\n\n")
    fh.write("| workload | V0 µs | V2 µs | V3 µs | V4 µs | SQNR V0 | V2 | V3 | V4 | µJ/call V0 | V4 |\n")
    fh.write("|---|---|---|---|---|---|---|---|---|---|---|\n")
    for r in rows:
        fmt = lambda x: "-" if x is None else ("%.2f" % x)  # noqa: E731
        fh.write("| %s | %s |\n" % (r[0], " | ".join(fmt(x) for x in r[1:])))
print("wrote profiles/r2_ablation.md")
