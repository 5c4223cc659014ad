"""Build libqflash.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_objs")
LIB = os.path.join(PKG, "libqflash.so")
SOURCES = ["qflash_attn_d32.cu", "qflash_attn_d64.cu", "qflash_attn_d128.cu", "qflash_attn_dbg.cu",
           "qflash_fused_d32.cu", "qflash_fused_d64.cu", "qflash_fused_d128.cu", "qflash_attn_ph.cu",
           "qflash_attn_acc.cu", "qflash_quant.cu", "qflash_host.cu"]
HEADERS = ["ptx.cuh", "qflash_common.cuh", "qflash_params.cuh", "qflash_attn_kernel.cuh", "qflash_quant_elem.cuh",
           "qflash_attn_inst.cuh"]
PUBLIC_HEADERS = ["qflash.h", "qflash_debug.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17",
                "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden",
                "-Xptxas", "-v", "-diag-suppress", "177"]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, extra_flags=(), lib: str = LIB, objdir: str = BUILD) -> str:
    """Compile and link libqflash.so.  extra_flags / lib / objdir build an
    experiment variant of the same library side by side (tools/, QFLASH_LIB)."""
    os.makedirs(objdir, exist_ok=True)
    inc = os.path.join(os.path.dirname(PKG), "include")
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(inc, h) for h in PUBLIC_HEADERS]
    jobs, objs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        if _stale(o, [s] + hdrs + [__file__]):
            jobs.append([NVCC, *FLAGS, *extra_flags, "-I", inc, "-c", s, "-o", o])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=len(jobs)) as ex:
            results = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs))
        for cmd, res in zip(jobs, results):
            if res.returncode != 0:
                raise RuntimeError("nvcc failed: %s\n%s%s" % (" ".join(cmd), res.stdout, res.stderr))
            if verbose:
                print(res.stderr)
    if _stale(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-Xcompiler", "-fvisibility=hidden"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("link failed: %s\n%s" % (res.stdout, res.stderr))
    return lib


if __name__ == "__main__":
    print(build(verbose=True))
