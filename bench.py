#!/usr/bin/env python
"""bench.py -- QFlash hot path on B200: one JSON line per run (rank 0).

A "step" is one pass of the whole hot path over one batch of synthetic input
(SURVEY 8(a)): fused per-tensor quantization of fp32 Q, K, V (Eq. 2) -> the
integer-only fused attention kernel (Algorithm 1, device-derived constants) ->
dequantization of O (s_O = s_V): ONE cooperative launch of libqflash.so's fused
step kernel.  The rotating input sets' steps are captured back to back into one
CUDA graph (a graph-captured model forward's launch pattern); --graph-steps 1
replays one graph per step, and the line also reports that per-step figure.

Default workload: BASELINE.json configs[1], ViT-Base attention at batch 8
(P = 96 problems, N = 197, d = 64).  Inputs are fp32 resident in HBM; the
timed region cycles through enough input sets (> 2x the 126 MB L2) that every
step reads cold inputs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload A3 --batch 8]
  python bench.py --impl reference ...   # the CPU oracle on the host cores

Multi-GPU (torchrun): one process per GPU, weak scaling by default (every rank
runs its own full batch, no collective on the data path); --scaling strong
splits one batch's problems with qflash_partition.  Time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2604_25306_b200.inputs import BASELINE_CONFIGS, CATALOG, gen_real_qkv  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
L2_BYTES = 126 * 1024 * 1024


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0, "source": "fallback"}


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while work runs."""

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples = []  # (t, sm_mhz, reasons_bitmask)
        self._stop = threading.Event()
        self._th = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.perf_counter(), mhz, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()

    def stop(self):
        if self._th:
            self._stop.set()
            self._th.join()

    def summary(self, t0: float, t1: float):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        win = [s for s in self.samples if t0 <= s[0] <= t1]
        where = "timed region"
        if not win:  # timed region shorter than the sampling period: use the loaded surroundings
            win = self.samples
            where = "around timed region"
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksEventReasonGpuIdle", 0x1): "gpu_idle",
            getattr(nv, "nvmlClocksEventReasonApplicationsClocksSetting", 0x2): "applications_clocks",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonSyncBoost", 0x10): "sync_boost",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake_slowdown",
        }
        bits = 0
        for s in win:
            bits |= s[2]
        reasons = sorted(n for b, n in names.items() if bits & b and n != "gpu_idle")
        return {"sm_mhz": float(statistics.median(s[1] for s in win)) if win else None,
                "sm_max_mhz": float(self.max_mhz), "reasons": reasons, "samples": len(win),
                "window": where}


# --------------------------------------------------------------------- helpers
def workload_from_args(args):
    if args.workload is None:
        name, batch = BASELINE_CONFIGS[1]
    else:
        name, batch = args.workload, args.batch
    w = CATALOG[name]
    return name, batch, w


def algorithmic(P, N, d):
    return {
        "int8_ops": 4.0 * N * N * d * P,       # QK^T + PV, 2 ops per MAC
        "score_elems": float(N) * N * P,       # units of the integer softmax
        "attn_bytes": 4.0 * N * d * P,         # read Q, K, V once, write O once (int8)
        "attn_dq_bytes": 7.0 * N * d * P,      # int8 Q, K, V in, fp32 O out (fused dequantize)
        "fused_step_bytes": 16.0 * N * d * P,  # fp32 Q, K, V in, fp32 O out (codes stay in L2)
        "step_bytes": 3 * 4.0 * N * d * P + 3 * N * d * P + 2 * N * d * P + 4.0 * N * d * P,
    }


# ALU roofline of the integer softmax: 10 int32 ops per
# score element against 148 SMs x 128 int32 lanes x clock.
ALU_OPS_PER_ELEM = 10.0

SMS, INT32_LANES = 148, 128


def run_reference(args):
    """--impl reference: the CPU oracle (as it stands) on the host cores, rank 0 only.

    Each step is a bounded sample of the workload (its first `sample_p` problems,
    whole quantize + attention + dequantize) sized so that W + K steps end within
    about two minutes; exactly K steps are timed."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    name, batch, w = workload_from_args(args)
    P, N, d = w.problems(batch), w.seq_len, w.head_dim
    cores = os.cpu_count() or 1

    def one(qs, ks, vs):
        qq, sq = oracle.quantize(qs)
        kq, sk = oracle.quantize(ks)
        vq, sv = oracle.quantize(vs)
        o = oracle.attention(qq, kq, vq, sq, sk, block_kv=args.block_kv, nthreads=cores)
        return oracle.dequantize(o, sv)

    # calibrate on one problem, then size the per-step sample
    q, k, v = gen_real_qkv(P, N, d, seed=0, family=w.family)
    t0 = time.perf_counter()
    one(q[:cores], k[:cores], v[:cores])
    t_per_problem = (time.perf_counter() - t0) / min(P, cores)
    budget = 120.0 / max(1, args.steps + args.warmup)
    sample_p = int(max(1, min(P, budget / max(t_per_problem, 1e-9))))
    if args.ref_problems:
        sample_p = max(1, min(P, args.ref_problems))
    qs, ks, vs = q[:sample_p], k[:sample_p], v[:sample_p]
    for _ in range(args.warmup):
        one(qs, ks, vs)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one(qs, ks, vs)
    dt = (time.perf_counter() - t0) / args.steps
    alg = algorithmic(sample_p, N, d)
    value = alg["int8_ops"] / dt / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TOPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "s8/s32",
        "data": "synthetic (SURVEY 8(d) recipe, seed 0)",
        "config": {"workload": f"{name} b{batch} ({w.source})", "problems": P, "seq_len": N,
                   "head_dim": d, "block_kv": args.block_kv},
        "cpu_baseline": {"value": value, "unit": "TOPS", "cores": cores, "kind": "oracle",
                         "sample": f"{sample_p} of {P} problems per step (quantize + attention + "
                                   f"dequantize), {cores} host threads"},
        "e2e": {"value": value, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(name, batch, w, block_kv, budget_s=10.0):
    """The oracle (as it stands) timed on the host cores on a bounded sample (rank 0,
    N=1): all hardware threads, then a single thread on a smaller sample."""
    import oracle
    P, N, d = w.problems(batch), w.seq_len, w.head_dim
    cores = os.cpu_count() or 1

    def timed(sample_p, nthreads, budget):
        q, k, v = gen_real_qkv(sample_p, N, d, seed=0, family=w.family)
        reps, t_total = 0, 0.0
        while t_total < budget:
            t0 = time.perf_counter()
            qq, sq = oracle.quantize(q)
            kq, sk = oracle.quantize(k)
            vq, sv = oracle.quantize(v)
            o = oracle.attention(qq, kq, vq, sq, sk, block_kv=block_kv, nthreads=nthreads)
            oracle.dequantize(o, sv)
            t_total += time.perf_counter() - t0
            reps += 1
        dt = t_total / reps
        return algorithmic(sample_p, N, d)["int8_ops"] / dt / 1e12, reps, t_total

    sample_p = min(P, max(1, {"L14": 4}.get(name, P)))
    v_all, reps, tt = timed(sample_p, cores, budget_s)
    sample_1 = min(P, max(1, {"L14": 1}.get(name, min(P, 8))))
    v_one, reps1, tt1 = timed(sample_1, 1, budget_s / 2)
    return {"value": v_all, "unit": "TOPS", "cores": cores, "kind": "oracle",
            "sample": f"{sample_p} of {P} problems x {reps} reps ({tt:.1f} s), "
                      "quantize+attention+dequantize, all host threads",
            "single_thread": {"value": v_one, "unit": "TOPS", "cores": 1,
                              "sample": f"{sample_1} of {P} problems x {reps1} reps ({tt1:.1f} s)"},
            "cpu_model": cpu_model()}


def spawn_ranks(args):
    """--gpus N without a torchrun environment: re-launch this script under
    torch.distributed.run with one process per GPU (127.0.0.1 rendezvous)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    os.execvp(cmd[0], cmd)


def measured_peaks(pk):
    """Roofline denominators: the committed microbenchmarks (profiles/r2_peaks.json:
    tcgen05 kind::i8 GEMM, ShiftExp2 integer mix), else nominal figures (stated)."""
    out = {}
    try:
        out = json.load(open(os.path.join(ROOT, "profiles", "r2_peaks.json")))
    except Exception:
        pass
    sm_clk_ghz = (pk.get("sm_max_mhz") or 1965.0) / 1e3
    if "int8_tops" not in out:
        out["int8_tops"] = 2.0 * pk.get("bf16_tflops", 1652.8)
        out["int8_source"] = "nominal: measured bf16 burst x 2 (int8/bf16 ratio)"
    if "alu_elems_per_s" not in out:
        out["alu_elems_per_s"] = SMS * INT32_LANES * sm_clk_ghz * 1e9 / ALU_OPS_PER_ELEM
        out["alu_source"] = "nominal: 148 SM x 128 int32 lanes x %.3f GHz / 10 ops per element" % sm_clk_ghz
    return out


def graph_time(graphs, stream, reps, warm=3):
    """ms per replay of `graphs` (cycled), device events on `stream`, GPU kept busy."""
    import torch
    with torch.cuda.stream(stream):
        for i in range(warm):
            graphs[i % len(graphs)].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        torch.cuda._sleep(2_000_000)
        e0.record(stream)
        for i in range(reps):
            graphs[i % len(graphs)].replay()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def chain_time(fns, stream, steps):
    """ms per step of the callables `fns` captured back to back into ONE CUDA graph
    (one replay = len(fns) steps), replayed for about `steps` steps."""
    g = capture(lambda: [f() for f in fns], stream)
    return graph_time([g], stream, max(1, steps // len(fns))) / len(fns)


def capture(fn, stream):
    import torch
    with torch.cuda.stream(stream):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    return g


def table1_sweep(qfl, dev, stream, reps=400):
    """SURVEY 8(d) metric set in the driver's run: every Table 1 workload (A1-A7)
    at batch 1 and 8 -- the fused one-launch step and the integer attention alone on the
    int8 codes, each CUDA-graph-replayed over rotating input sets that exceed 2x L2 (cold)."""
    import torch
    from paper_2604_25306_b200.inputs import gen_real_qkv_slab
    out = {}
    for name in ("A1", "A2", "A3", "A4", "A5", "A6", "A7"):
        w = CATALOG[name]
        for batch in (1, 8):
            P, N, d = w.problems(batch), w.seq_len, w.head_dim
            alg = algorithmic(P, N, d)
            n_sets = int(min(64, max(2, np.ceil(2.0 * L2_BYTES / alg["step_bytes"]) + 1)))
            q0, k0, v0 = gen_real_qkv_slab(P, N, d, 0, P, seed=0, family=w.family)
            base = [torch.from_numpy(a).to(dev) for a in (q0, k0, v0)]
            sets = [[(t * (-1.0 if i % 2 else 1.0)).roll(shifts=i, dims=1).contiguous() for t in base]
                    for i in range(n_sets)]
            pipes = [qfl.QFlashPipeline(P, N, d, device=dev) for _ in range(n_sets)]
            # one graph per n_sets consecutive steps (each on its own cold set), as the main line
            L = n_sets * max(1, -(-48 // n_sets))  # >= 48 steps per graph, as the main line
            g_step = capture(lambda: [pipes[i % n_sets](*sets[i % n_sets], stream=stream) for i in range(L)], stream)
            t_step = graph_time([g_step], stream, max(1, reps // L)) / L
            g_att = capture(lambda: [qfl.qflash_attention_int8_prepared(
                pipes[i % n_sets].qkv_q[0], pipes[i % n_sets].qkv_q[1], pipes[i % n_sets].qkv_q[2],
                pipes[i % n_sets].workspace, out=pipes[i % n_sets].o_q, stream=stream) for i in range(L)], stream)
            t_att = graph_time([g_att], stream, max(1, reps // L)) / L
            out[f"{name} b{batch}"] = {
                "problems": P, "seq_len": N, "head_dim": d,
                "step_us": t_step * 1e3, "step_tops": alg["int8_ops"] / (t_step * 1e-3) / 1e12,
                "attention_int8_us": t_att * 1e3,
                "attention_int8_tops": alg["int8_ops"] / (t_att * 1e-3) / 1e12}
            del g_step, g_att, pipes, sets, base
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, help="catalog name (default: BASELINE configs[1])")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--block-kv", type=int, default=128)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: each rank a batch-sized slab of a world x batch global batch, per-slab "
                         "scales, no collective; strong: ONE batch partitioned over the ranks, global "
                         "per-tensor scales via a MAX all-reduce of the amax every step")
    ap.add_argument("--ref-problems", type=int, default=0)
    ap.add_argument("--graph-steps", default="sets", choices=["sets", "1"],
                    help="steps per CUDA graph replay: all rotating input sets (default) or 1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the per-stage timing set")
    ap.add_argument("--no-table1", action="store_true",
                    help="skip the A1-A7 batch 1/8 table (default run only: world 1, default workload)")
    ap.add_argument("--mode", default="fused", choices=["fused", "two", "three"],
                    help="step form: one cooperative launch (default), or 2 / 3 launches")
    ap.add_argument("--variant", default="auto", choices=["auto", "generic", "packed"],
                    help="attention tiling (auto: row-packed when it saves a wave)")
    ap.add_argument("--scales", default="per-tensor", choices=["per-tensor", "per-head"],
                    help="granularity (per-head = SURVEY 8(f) N1; 5 launches per step)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: collectives through host copies, ranks may "
                         "share a GPU -- a functional test of the multi-rank path on one device)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d (launch one process per GPU)"
                         % (args.gpus, world))

    import torch
    import torch.distributed as dist

    import paper_2604_25306_b200 as qfl
    from paper_2604_25306_b200 import _lib
    from paper_2604_25306_b200.inputs import gen_real_qkv_slab

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    gloo = args.dist_backend == "gloo"
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def all_reduce(t, op):
        if gloo:  # gloo collectives on host copies
            h = t.cpu()
            dist.all_reduce(h, op=op)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op)

    def all_gather(outs, t):
        if gloo:
            hs = [torch.empty_like(t, device="cpu") for _ in outs]
            dist.all_gather(hs, t.cpu())
            for o, h in zip(outs, hs):
                o.copy_(h)
        else:
            dist.all_gather(outs, t)

    name, batch, w = workload_from_args(args)
    P_batch, N, d = w.problems(batch), w.seq_len, w.head_dim
    strong = args.scaling == "strong" and world > 1
    P_total = P_batch if args.scaling == "strong" else world * P_batch
    p_begin, P_local = qfl.qflash_partition(P_total, world, rank)
    alg = algorithmic(P_local, N, d)
    if args.scales == "per-head" and strong:
        raise SystemExit("bench.py: --scales per-head supports weak scaling only")

    # ---- input sets: fp32 Q, K, V of this rank's slab resident in HBM; enough sets
    # (sign flips / rolls of the slab) that every step reads cold inputs (> 2x L2)
    set_bytes = alg["step_bytes"]
    n_sets = int(min(64, max(2, np.ceil(2.0 * L2_BYTES / max(set_bytes, 1)) + 1)))
    q0, k0, v0 = gen_real_qkv_slab(P_total, N, d, p_begin, P_local, seed=0, family=w.family)
    base = [torch.from_numpy(a).to(dev) for a in (q0, k0, v0)]
    sets = []
    for i in range(n_sets):
        sgn = -1.0 if (i % 2) else 1.0
        sets.append([(t * sgn).roll(shifts=i, dims=1).contiguous() for t in base])
    if args.scales == "per-head":
        pipes = [qfl.QFlashPerHeadPipeline(P_local, N, d, w.heads, block_kv=args.block_kv, device=dev)
                 for _ in range(n_sets)]
        args.no_e2e = True
    else:
        pipes = [qfl.QFlashPipeline(P_local, N, d, block_kv=args.block_kv, device=dev, mode=args.mode,
                                    variant=args.variant)
                 for _ in range(n_sets)]
    stream = torch.cuda.Stream(device=dev)
    amax_bufs = [torch.zeros(3, dtype=torch.float32, device=dev) for _ in range(n_sets)]

    chain = None
    if strong:
        # per step: local amax (graph) -> NCCL MAX all-reduce of 3 floats (eager, on the
        # stream) -> fused step with the global amax (graph)
        g_amax = [capture(lambda s=s, a=a: qfl.qflash_amax_qkv(*s, out=a, stream=stream), stream)
                  for s, a in zip(sets, amax_bufs)]
        g_step = [capture(lambda p=p, s=s, a=a: qfl.qflash_forward_fused(
            *s, args.block_kv, args.variant, out=p.out, codes=p.qkv_q, scales=p.scales,
            workspace=p.workspace, stream=stream, amax=a), stream)
            for p, s, a in zip(pipes, sets, amax_bufs)]

        def run_step(i):
            g_amax[i % n_sets].replay()
            all_reduce(amax_bufs[i % n_sets], dist.ReduceOp.MAX)
            g_step[i % n_sets].replay()
        launches_per_step = 2
    else:
        graphs = [capture(lambda p=p, s=s: p(*s, stream=stream), stream) for p, s in zip(pipes, sets)]
        # one CUDA graph holding the n_sets consecutive steps (every step its own cold
        # input set), as a graph-captured model forward launches them: the per-graph
        # launch cost (~2.5 us) is paid once per n_sets steps; --graph-steps 1 times one
        # graph launch per step
        chain = None
        # the chain cycles the input sets until it holds >= 48 steps (the sets already
        # exceed 2x L2, so every step still reads cold inputs)
        chain_len = n_sets * (max(1, -(-48 // n_sets)) if set_bytes < (64 << 20) else 1)
        chain_len = max(1, min(chain_len, args.steps))  # a short run (K < 48) is one chain of K steps
        if args.graph_steps != "1":
            chain = capture(lambda: [pipes[i % n_sets](*sets[i % n_sets], stream=stream)
                                     for i in range(chain_len)], stream)
            with torch.cuda.stream(stream):
                chain.replay()  # the graph's first launch uploads it: keep that out of the timing
            torch.cuda.synchronize()

        def run_step(i):
            graphs[i % n_sets].replay()

        def run_steps(k):  # k consecutive steps starting at set 0
            done = 0
            if chain is not None:
                while k - done >= chain_len:
                    chain.replay()
                    done += chain_len
            for i in range(done, k):
                run_step(i)
        launches_per_step = pipes[0].launches()
    torch.cuda.synchronize()
    status = int(pipes[0].workspace[0].item())
    if status != 0:
        raise RuntimeError("device-derived scales out of range: %s" % _lib.status_string(status))

    sampler = ClockSampler(local)
    sampler.start()
    if strong:
        def run_steps(k):
            for i in range(k):
                run_step(i)
    with torch.cuda.stream(stream):
        run_steps(args.warmup)
    torch.cuda.synchronize()

    # ---- timed region: K steps, barrier + sync on both sides, device events
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_host0 = time.perf_counter()
    with torch.cuda.stream(stream):
        # host head start so graph replays queue back to back; ~20 ms of device spin also
        # brings the SM clock to its boost level before the first timed step
        torch.cuda._sleep(40_000_000)
        ev0.record(stream)
        run_steps(args.steps)
        ev1.record(stream)
    torch.cuda.synchronize()
    t_host1 = time.perf_counter()
    if world > 1:
        dist.barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    t_all = torch.zeros(world, device=dev, dtype=torch.float64)
    t_all[rank] = elapsed_ms
    if world > 1:
        all_reduce(t_all, dist.ReduceOp.SUM)
    rank_ms = [float(x) / args.steps for x in t_all.cpu().tolist()]
    elapsed_ms = max(float(x) for x in t_all.cpu().tolist())
    ms_per_step = elapsed_ms / args.steps
    # every rank processed its slab each step: the whole job's ops / max-over-ranks time
    value = algorithmic(P_total, N, d)["int8_ops"] * args.steps / (elapsed_ms * 1e-3) / 1e12
    clocks = sampler.summary(t_host0, t_host1)

    # ---- dominant kernel, graph-timed like the step: the fused step kernel (the step
    # itself when the step is one launch), else the attention launches alone
    one_launch = (not strong) and launches_per_step == 1
    per_head = args.scales == "per-head"
    k_launch = min(args.steps, 2000)
    graphs_per_replay = 1
    if one_launch:
        kgraphs = graphs if chain is None else [chain]
        graphs_per_replay = 1 if chain is None else chain_len
        kname = "qflash_attn_kernel<FQ> (fused step: quantize prologue + attention + dequantize)"
    elif strong:
        kgraphs = g_step
        kname = "qflash_attn_kernel<FQ> (fused step with the all-reduced amax)"
    elif per_head:
        kgraphs = [capture(lambda p=p: p.attention(stream=stream), stream) for p in pipes]
        kname = "derive_per_head + qflash_attn_kernel<PH> (int8 out)"
    else:
        kgraphs = [capture(lambda p=p: qfl.qflash_attention_dequant_prepared(
            p.qkv_q[0], p.qkv_q[1], p.qkv_q[2], p.workspace, args.block_kv, args.variant,
            out=p.out, stream=stream), stream) for p in pipes]
        kname = "qflash_attn_kernel (fused dequantize epilogue)"
    attn_ms = graph_time(kgraphs, stream, max(1, k_launch // graphs_per_replay)) / graphs_per_replay
    attn_share = attn_ms / ms_per_step
    # the same step with one graph launch per step (the launch cost included)
    step_graph1_ms = graph_time(graphs, stream, k_launch) if (not strong and chain is not None) else None

    # ---- the per-stage timing set: attention alone on int8 inputs,
    # the quantizer and the dequantizer alone (graphs, cold sets), single-call latency
    extra = None
    if not args.no_extra and not per_head:
        p0 = pipes[0]
        q_prep = [lambda p=p, s=s: qfl.qflash_quantize_qkv_prepare(
            *s, outs=p.qkv_q, scales=p.scales, workspace=p.workspace, stream=stream)
            for p, s in zip(pipes, sets)]
        a_int8 = [lambda p=p: qfl.qflash_attention_int8_prepared(
            p.qkv_q[0], p.qkv_q[1], p.qkv_q[2], p.workspace, args.block_kv, args.variant,
            out=p.o_q, stream=stream) for p in pipes]
        dq = [lambda p=p: qfl.qflash_dequantize(p.o_q, p.scales[2:3], out=p.out, stream=stream)
              for p in pipes]
        t_q = chain_time(q_prep, stream, k_launch)
        t_a = chain_time(a_int8, stream, k_launch)
        t_d = chain_time(dq, stream, k_launch)
        # single call, host wall clock around one synchronized eager step (launch included)
        lat = []
        for i in range(20):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            p0(*sets[i % n_sets], stream=stream)
            torch.cuda.synchronize()
            lat.append(time.perf_counter() - t0)
        E = P_local * N * d
        extra = {
            "attention_int8_us": t_a * 1e3,
            "attention_int8_tops": alg["int8_ops"] / (t_a * 1e-3) / 1e12,
            "quantize_qkv_us": t_q * 1e3,
            "quantize_qkv_gbs": 3 * E * 5 / (t_q * 1e-3) / 1e9,
            "dequantize_us": t_d * 1e3,
            "dequantize_gbs": E * 5 / (t_d * 1e-3) / 1e9,
            "single_call_wall_us": statistics.median(lat) * 1e6,
            "note": "CUDA graphs of the n_sets consecutive calls over the rotating cold sets; attention on the int8 codes "
                    "(qflash_attention_int8_prepared), quantizer = qflash_quantize_qkv_prepare "
                    "(bytes 3 E (4 + 1)), dequantizer bytes E (1 + 4); single call = host wall "
                    "clock of one synchronized eager fused step",
        }

    kbytes = (alg["fused_step_bytes"] if (one_launch or strong) else alg["attn_bytes"] if per_head
              else alg["attn_dq_bytes"])
    pk = peaks()
    mp = measured_peaks(pk)
    alu_peak = ALU_OPS_PER_ELEM * mp["alu_elems_per_s"] / 1e12
    alu_achieved = ALU_OPS_PER_ELEM * alg["score_elems"] / (attn_ms * 1e-3) / 1e12
    roofline = {
        "kernel": kname,
        "bound": "alu", "achieved": alu_achieved,
        "peak": alu_peak, "unit": "T int32-op/s", "frac": alu_achieved / alu_peak,
        "traffic": None,
        "per_unit": "10 int32 ops per score element (SURVEY 8(d)); units = N^2 P per launch",
        "peak_source": mp.get("alu_source"),
        "attn_us": attn_ms * 1e3, "attn_share_of_step": attn_share,
        "attn_timing": "CUDA graph of the kernel's launches alone over the rotating sets",
        "tensor": {"achieved_tops": alg["int8_ops"] / (attn_ms * 1e-3) / 1e12,
                   "peak_tops": mp["int8_tops"],
                   "frac": alg["int8_ops"] / (attn_ms * 1e-3) / 1e12 / mp["int8_tops"],
                   "peak_source": mp.get("int8_source")},
        "hbm": {"achieved_gbs": kbytes / (attn_ms * 1e-3) / 1e9,
                "peak_gbs": pk.get("hbm_gbs"),
                "frac": kbytes / (attn_ms * 1e-3) / 1e9 / pk.get("hbm_gbs", 6452.5),
                "bytes_per_launch": kbytes,
                "per_unit": "16 N d B per problem (fp32 Q, K, V in + fp32 O out)" if (one_launch or strong)
                            else "4 N d B per problem (int8 Q, K, V in + int8 O out)" if per_head
                            else "7 N d B per problem (int8 Q, K, V in + fp32 O out)"},
    }
    traffic_file = os.path.join(ROOT, "profiles", "attn_traffic.json")
    if os.path.exists(traffic_file):
        try:
            tj = json.load(open(traffic_file)).get(
                f"{name}_b{batch}" + ("_fused" if one_launch else "_ph" if per_head else ""))
            if tj:
                roofline["traffic"] = tj
        except Exception:
            pass

    # ---- end to end through the public serving API with host buffers (weak: each
    # rank serves its own slab; strong: the slab's scales would need the collective,
    # so e2e is reported for weak scaling only)
    e2e = None
    if not args.no_e2e and not strong:
        host_sets = []
        for i in range(2):
            sgn = -1.0 if i else 1.0
            host_sets.append([(torch.from_numpy(a) * sgn).pin_memory() for a in (q0, k0, v0)])
        houts = [torch.empty((P_local, N, d), dtype=torch.float32).pin_memory() for _ in range(2)]
        hp = qfl.QFlashHostPipeline(P_local, N, d, block_kv=args.block_kv, device=dev, mode=args.mode)
        k_e2e = max(3, min(args.steps, 200))
        for t in range(4):
            hp(*host_sets[t % 2], houts[t % 2])
        hp.synchronize()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.current_stream())
        for s_ in hp.streams:
            s_.wait_event(e0)
        for t in range(k_e2e):
            hp(*host_sets[t % 2], houts[t % 2])
        for s_ in hp.streams:
            torch.cuda.current_stream().wait_stream(s_)
        e1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1)
        ref_out = pipes[0](*[t_.to(dev) for t_ in host_sets[(k_e2e - 1) % 2]], stream=stream)
        torch.cuda.synchronize()
        assert torch.equal(ref_out.cpu(), houts[(k_e2e - 1) % 2]), "e2e output mismatch"
        e_t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
        if world > 1:
            all_reduce(e_t, dist.ReduceOp.MAX)
        e_ms = float(e_t.item())
        e2e = {"value": algorithmic(P_total, N, d)["int8_ops"] * k_e2e / (e_ms * 1e-3) / 1e12,
               "unit": "TOPS", "h2d_bytes_per_step": 3 * 4 * P_local * N * d,
               "d2h_bytes_per_step": 4 * P_local * N * d, "ms_per_step": e_ms / k_e2e,
               "steps": k_e2e,
               "api": "QFlashHostPipeline (pinned host fp32 in/out, 2 buffer sets overlapping copies and compute)"}
    sampler.stop()

    # ---- verification (outside the timed region): every rank's output of input set
    # 0 is gathered with NCCL (sampled problems byte for byte + a checksum of the slab)
    # and rank 0 compares it with its own 1-GPU run of the same rows
    verify = None
    if world > 1 and not per_head:
        with torch.cuda.stream(stream):
            run_step(0)
        torch.cuda.synchronize()
        y = pipes[0].out
        samp = 2
        loc = torch.zeros((samp, N, d), dtype=torch.float32, device=dev)
        loc[:min(samp, P_local)] = y[:samp]
        csum = y.view(torch.int32).to(torch.int64).sum().reshape(1)
        g_s = [torch.empty_like(loc) for _ in range(world)]
        g_c = [torch.empty_like(csum) for _ in range(world)]
        all_gather(g_s, loc)
        all_gather(g_c, csum)
        ok = True
        if rank == 0:
            ref_q = [torch.from_numpy(a).to(dev) for a in
                     gen_real_qkv_slab(P_total, N, d, 0, P_total, seed=0, family=w.family)]
            for r in range(world):
                b_r, c_r = qfl.qflash_partition(P_total, world, r)
                if strong:  # the whole batch on this GPU, kernel-computed amax
                    if r == 0:
                        full = qfl.qflash_forward_fused(*ref_q, args.block_kv, args.variant)
                    ref = full[b_r:b_r + c_r]
                else:       # the slab alone on this GPU (its own per-tensor scales)
                    ref = qfl.QFlashPipeline(c_r, N, d, block_kv=args.block_kv, device=dev, mode=args.mode,
                                             variant=args.variant)(*[t[b_r:b_r + c_r].contiguous()
                                                                     for t in ref_q])
                ok = ok and torch.equal(ref[:samp].view(torch.int32), g_s[r][:min(samp, c_r)].view(torch.int32))
                ok = ok and int(ref.view(torch.int32).to(torch.int64).sum()) == int(g_c[r].item())
        verify = {"ok": bool(ok), "method": args.dist_backend.upper() + " all_gather of each rank's first %d problems + int64 "
                  "checksum of its fp32 output, compared on rank 0 with a 1-GPU run of the same rows "
                  "(%s)" % (samp, "whole batch" if strong else "each slab")}
        if rank == 0 and not ok:
            print("bench.py: multi-GPU verification FAILED", file=sys.stderr)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(name, batch, w, args.block_kv)
    table1 = None
    if world == 1 and args.workload is None and not args.no_table1 and args.scales == "per-tensor":
        table1 = table1_sweep(qfl, dev, stream)

    if rank == 0:
        step_desc = ("qflash_amax_qkv + NCCL all_reduce(MAX, 3 floats) + qflash_forward_fused_amax"
                     if strong else
                     "qflash_forward_fused_per_head (CUDA graph, 1 cooperative launch)"
                     if (launches_per_step == 1 and per_head) else
                     "qflash_forward_fused (CUDA graph, 1 cooperative launch)" if launches_per_step == 1
                     else "per-head quantize + derive + attention + dequantize (CUDA graph)"
                     if per_head else "quantize_qkv_prepare + attention_dequant_prepared (CUDA graph)")
        line = {
            "metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "us_per_call": ms_per_step * 1e3, "higher_is_better": True,
            "scaling": "strong" if args.scaling == "strong" else "weak", "vs_baseline": None,
            "dtype": "s8/s32",
            "data": "synthetic (SURVEY 8(d) recipe: channel-mean Gaussians, chunk-seeded global batch)",
            "config": {"workload": f"{name} b{batch} ({w.source})", "problems": P_total,
                       "problems_per_rank": P_local, "seq_len": N, "head_dim": d,
                       "block_kv": args.block_kv,
                       "parallelism": (f"{world} ranks x contiguous problem slabs (qflash_partition)"
                                       + (", global scales via all_reduce" if strong else
                                          ", per-slab scales, no collective" if world > 1 else "")),
                       "step": step_desc, "scales": args.scales,
                       "l2": f"rotating {n_sets} input sets ({n_sets * set_bytes / 2**20:.0f} MiB > 2x L2)",
                       "graph": (f"{chain_len} consecutive steps (cycling the {n_sets} input sets) per CUDA graph replay"
                                 if (not strong and chain is not None) else "one CUDA graph replay per step")},
            "us_per_call_graph_per_step": (step_graph1_ms * 1e3 if step_graph1_ms is not None else None),
            "rank_ms_per_step": rank_ms,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks, "roofline": roofline, "stages": extra, "cpu_baseline": cpu, "e2e": e2e,
            "table1": table1,
            "verify": verify,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
