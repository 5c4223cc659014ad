"""Build an experiment variant of libqflash.so side by side (e.g. the fused-step
timing build: python tools/build_variant.py fqt -DQF_FQ_TIMING); load it with
QFLASH_LIB=libqflash_<name>.so."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_25306_b200 import _build  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
lib = os.path.join(_build.PKG, "libqflash_%s.so" % name)
print(_build.build(extra_flags=flags, lib=lib, objdir=os.path.join(_build.PKG, "_objs_%s" % name)))
