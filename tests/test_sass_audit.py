"""SASS audit of libqflash.so (CPU only, cuobjdump): every production instantiation
of the fused attention kernel is integer-only -- no floating-point instruction
(the north star's "integer softmax epilogue ... that never touches floating
point") -- and uses the tcgen05 tensor-core / TMEM / TMA path."""
from __future__ import annotations

import os
import re
import shutil
import subprocess

import pytest

from paper_2604_25306_b200 import _build

FP_OPCODES = {
    "FADD", "FADD32I", "FMUL", "FMUL32I", "FFMA", "FFMA32I", "FMNMX", "FSETP", "FSET", "FSEL",
    "FCHK", "FRND", "FCMP", "FSWZADD", "F2I", "F2F", "F2FP", "I2F", "I2FP", "MUFU", "DADD",
    "DMUL", "DFMA", "DSETP", "DMNMX", "HADD2", "HMUL2", "HFMA2", "HSETP2", "HMNMX2",
}


def _functions():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    lib = _build.build()
    out = subprocess.run([exe, "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and cur:
            funcs[cur].append(m.group(2))
    return funcs


def test_attention_kernels_integer_only_and_tensor_core():
    funcs = _functions()
    # template <D, B_c, NSEG, CS, QT, DBG, FQ, PH, VAR>: DBG = false, FQ = 0 are the
    # integer-only attention kernels (VAR 1: the Eq. 13 ablation, integer too); FQ = 1 adds
    # the Eq. 2 quantizer prologue (fp32 by definition) in front of the same integer code;
    # VAR 2 / 3 are the floating-point ablation steps V3 / V2 of SURVEY 8(f) N4 (excluded)
    pat = re.compile(r"qflash_attn_kernelILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELb([01])ELi(\d)"
                     r"ELb([01])ELi(\d)EEEv")
    tpl = {n: pat.search(n) for n in funcs if "qflash_attn_kernel" in n}
    assert all(tpl.values()), [n for n, m in tpl.items() if not m][:3]
    prod = {n: funcs[n] for n, m in tpl.items() if m.group(6) == "0" and m.group(7) == "0" and m.group(9) in "01"}
    fused = [n for n, m in tpl.items() if m.group(6) == "0" and m.group(7) == "1"]
    abl = [n for n, m in tpl.items() if m.group(9) in "23"]
    assert len(abl) >= 4, "ablation instantiations"
    assert len(fused) >= 20
    assert len(prod) >= 20, sorted(funcs)[:10]
    for name, ops in prod.items():
        fp = sorted({o for o in ops if o.split(".")[0] in FP_OPCODES})
        assert not fp, f"{name}: floating-point SASS {fp}"
        base = {o.split(".")[0] for o in ops}
        assert "UTCIMMA" in base or any(o.startswith("UTC") and "MMA" in o for o in ops), name
        assert "LDTM" in base and "STTM" in base, name
        assert "UTMALDG" in base, name
