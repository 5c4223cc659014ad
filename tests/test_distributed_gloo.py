"""World-size-2 gloo tests of the multi-GPU partition driver on CPU.

The hot path shards independent problems with no collective; the
per-rank compute here is the CPU oracle standing in for the GPU call, and the
checks are: slabs tile [0, P) exactly, the verification all_gather reassembles
the single-process result byte for byte, and the amax all-reduce reproduces the
single-process per-tensor scale.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, P, N, d, result_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2604_25306_b200.distributed import (allreduce_amax, problem_range,
                                                       run_sharded)
        from paper_2604_25306_b200.inputs import gen_int8_qkv, gen_real_qkv

        q, k, v = (torch.from_numpy(a) for a in gen_int8_qkv(P, N, d, seed=3))

        def attn(qs, ks, vs):
            return torch.from_numpy(oracle.attention(qs.numpy(), ks.numpy(), vs.numpy(),
                                                     0.05, 0.05, block_kv=64))

        local, full = run_sharded(q, k, v, attn)
        b, c = problem_range(P, world, rank)
        assert local.shape[0] == c
        # sharded quantization: the MAX all-reduce gives the 1-process amax
        xr, _, _ = gen_real_qkv(P, N, d, seed=4)
        xs = torch.from_numpy(xr[b:b + c])
        amax = torch.tensor([float(xs.abs().max()) if c else 0.0], dtype=torch.float32)
        allreduce_amax(amax)
        result_q.put((rank, full.numpy() if full is not None else None, float(amax.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P", [6, 5])
def test_gloo_world2_sharded_matches_single(orc, P):
    N, d = 77, 32
    world = 2
    ctx = mp.get_context("spawn")
    q_res = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, P, N, d, q_res)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q_res.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2604_25306_b200.inputs import gen_int8_qkv, gen_real_qkv
    q, k, v = gen_int8_qkv(P, N, d, seed=3)
    ref = orc.attention(q, k, v, 0.05, 0.05, block_kv=64)
    xr, _, _ = gen_real_qkv(P, N, d, seed=4)
    for rank, full, amax in results:
        assert np.array_equal(full, ref)
        assert amax == np.float32(np.abs(xr).max())
