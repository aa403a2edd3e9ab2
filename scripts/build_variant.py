#!/usr/bin/env python
"""Build a variant of libnlse_b200.so with extra -D defines, for A/B measurements.

    python scripts/build_variant.py NAME -DNLSE_TMA_PP64=3 [-D...]
    -> paper_1203_1263_b200/variants/libnlse_NAME.so ; load it with NLSE_LIB=<path>
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1203_1263_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
outdir = os.path.join(B.HERE, "variants")
os.makedirs(outdir, exist_ok=True)
out = os.path.join(outdir, f"libnlse_{name}.so")
B.build_to(out, defines=defs, log=out + ".log")
print(out)
