"""Per-CTA fused-step timeline (timing build -DQF_FQ_TIMING, QFLASH_LIB=libqflash_fqt.so):
prologue start, barrier-1 arrival, barrier-2 arrival and exit of every CTA, for the last
step of a chained graph over rotating cold sets."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_25306_b200 as qf  # noqa: E402
from paper_2604_25306_b200.inputs import CATALOG, gen_real_qkv  # noqa: E402

for wl, b in [("A3", 8), ("A1", 1), ("A4", 8)]:
    w = CATALOG[wl]
    P, N, d = w.problems(b), w.seq_len, w.head_dim
    base = [torch.from_numpy(x).cuda() for x in gen_real_qkv(P, N, d, seed=0, family=w.family)]
    n_sets = int(os.environ.get('FQ_SETS', '12'))
    sets = [[(t * (-1.0 if i % 2 else 1.0)).roll(shifts=i, dims=1).contiguous() for t in base] for i in range(n_sets)]
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
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    for idx in (n_sets - 1,):
        st = pipes[idx].workspace.view(torch.int32)[1600:1600 + 3 * 148].cpu().numpy().astype(np.int64).reshape(148, 3)
        st = st[st[:, 0] != 0]
        st = (st - st[:, 0].min()) & 0xFFFFFFFF
        st = st.astype(np.float64) / 1e3
        G = st.shape[0]
        print(f"== {wl} b{b}: {G} CTAs (us from the first barrier-2 arrival)")
        for k, name in enumerate(os.environ.get("CTA_EVENTS", "barrier-2 arrive,barrier-2 exit,proxy fence done").split(",")):
            c = st[:, k]
            print(f"  {name:18s} min {c.min():6.2f}  median {np.median(c):6.2f}  p90 {np.percentile(c, 90):6.2f}  max {c.max():6.2f}  argmax CTA {int(c.argmax())}")
        q = st[:, 1] - st[:, 0]
        print(f"  barrier1-arrive -> barrier2-arrive (scales+quantize per CTA): min {q.min():.2f} median {np.median(q):.2f} max {q.max():.2f}")
        late = np.argsort(-st[:, 1])[:8]
        print("  latest barrier-2 arrivals (CTA: b1 arrive, b2 arrive):", ", ".join(f"{i}: {st[i,0]:.2f}/{st[i,1]:.2f}" for i in late))
        late1 = np.argsort(-st[:, 0])[:8]
        print("  latest barrier-1 arrivals:", ", ".join(f"{i}: {st[i,0]:.2f}" for i in late1))
