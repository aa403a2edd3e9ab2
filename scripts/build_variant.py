#!/usr/bin/env python
"""Build a variant of libnlse_b200.so with extra -D defines, for A/B measurements.

    python scripts/build_variant.py NAME -DNLSE_TMA_PP64=3 [-D...]
    -> paper_1203_1263_b200/variants/libnlse_NAME.so ; load it with NLSE_LIB=<path>
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1203_1263_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
outdir = os.path.join(B.HERE, "variants")
os.makedirs(outdir, exist_ok=True)
out = os.path.join(outdir, f"libnlse_{name}.so")
cmd = [B.NVCC, *B.NVCC_FLAGS, *defs, "-I", os.path.join(ROOT, "include"), "-o", out, *B.sources(), "-lcudart"]
res = subprocess.run(cmd, capture_output=True, text=True)
open(out + ".log", "w").write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
if res.returncode:
    sys.stderr.write(res.stderr[-5000:])
    sys.exit(1)
print(out)
