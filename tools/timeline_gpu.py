"""Per-CTA timeline of the fused kernel (clock64 stamps of CTA (0,0)); run under gpurun."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_25306_b200 import _lib  # noqa: E402
from paper_2604_25306_b200.inputs import gen_int8_qkv  # noqa: E402

NAMES = {0: "entry", 1: "setup done", 2: "mma: Q landed", 100: "softmax: final PV done",
         101: "softmax: row stored", 102: "teardown", 103: "softmax: tables ready",
         104: "softmax: O, l loaded"}
for j in range(7):
    NAMES[3 + 4 * j] = f"mma: KV{j} landed"
    NAMES[4 + 4 * j] = f"mma: P{j} ready"
    NAMES[5 + 4 * j] = f"prod: KV{j} load issued"
    NAMES[6 + 4 * j] = f"mma: QK{j} issued"
    NAMES[40 + 8 * j] = f"softmax: S{j} ready"
    NAMES[41 + 8 * j] = f"softmax: max{j} exchanged"
    NAMES[42 + 8 * j] = f"softmax: P{j} start"
    NAMES[44 + 8 * j] = f"softmax: P{j} stored (release next)"
    NAMES[45 + 8 * j] = f"softmax: PV{j-1} done (o_full)"
    NAMES[46 + 8 * j] = f"softmax: release{j} loaded"
    NAMES[47 + 8 * j] = f"softmax: release{j} stored"
    NAMES[110 + j] = f"softmax: wait_st{j} done"
    NAMES[43 + 8 * j] = f"softmax: P{j} arrived"
    NAMES[60 + j] = f"softmax: S{j} loaded (tcgen05.ld done)"
    NAMES[70 + j] = f"softmax: S{j} row max done"

for (P, N, d, variant, label) in [(96, 197, 64, 0, "A3 b8"), (1536, 49, 32, 0, "A4 b8"),
                                  (1024, 1025, 64, 0, "L14 b64")]:
    q, k, v = gen_int8_qkv(P, N, d, seed=1)
    dq, dk, dv = (torch.from_numpy(t).cuda() for t in (q, k, v))
    o = torch.empty_like(dq)
    ts = torch.zeros(512, dtype=torch.int64, device="cuda")
    sh = _lib.AttnShape(P, N, d, 128)
    for it in range(3):  # warm, then keep the last
        ts.zero_()
        st = _lib.lib().qflash_debug_attention(dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), 0.05, 0.05,
                                               ctypes.byref(sh), variant, o.data_ptr(), None, None,
                                               None, ts.data_ptr(), None)
        torch.cuda.synchronize()
    t = ts.cpu().numpy()
    t0 = t[0]
    print(f"=== {label}: status {st}")
    for slot in sorted(NAMES):
        if t[slot]:
            print(f"  {slot:4d} {t[slot] - t0:8d} cyc  {NAMES[slot]}")
    g = t[128:].reshape(-1, 2)
    g = g[g[:, 0] > 0]
    if len(g):
        g0 = g[:, 0].min()
        st, en = (g[:, 0] - g0) / 1e3, (g[:, 1] - g0) / 1e3
        print(f"  CTAs {len(g)}: start spread {st.max():.2f} us, end min/median/max "
              f"{en.min():.2f}/{np.median(en):.2f}/{en.max():.2f} us, lifetime median "
              f"{np.median(en - st):.2f} us")
