#!/usr/bin/env python
"""Write tests/golden/oracle_sha256.json: SHA-256 digests of the ORACLE's output after the
stated number of steps of the BASELINE configurations that the GPU parity tests cannot afford
to re-run through the oracle inside the test budget (north_star: "match the oracle ... after
the stated number of steps").  Calls only oracle/ (and the closed-form inputs); nothing here
comes from the CUDA path.

    python scripts/make_goldens.py [name ...]      # default: every entry of CASES

Digest = sha256 of the oracle's result array in the run's precision (complex128 for fp64,
complex64 for fp32), C order, shape reversed(dims).  The GPU test hashes its own output
(widened values narrowed back to complex64 for fp32 runs: exact) and compares digests, so a
match is bit-identity of the whole field.
"""
from __future__ import annotations

import fcntl
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1203_1263_b200 import inputs  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_sha256.json")

# name -> (BASELINE config, precision, steps, citation)
CASES = {
    "trap2d_fp64_1000": ("trap2d", "fp64", 1000, "BASELINE configs[2]; 1000 steps = t 5 at k 0.005 (SURVEY §8(d))"),
    "ring3d_fp64_3360": ("ring3d", "fp64", 3360, "BASELINE configs[3]; 3360 steps P:69 (reading R-STEPS)"),
    "ring3d_fp32_3360": ("ring3d", "fp32", 3360, "BASELINE configs[3]; 3360 steps P:69 (reading R-STEPS)"),
}


def digest(arr, precision):
    dt = np.complex128 if precision == "fp64" else np.complex64
    return hashlib.sha256(np.ascontiguousarray(np.asarray(arr).astype(dt)).tobytes()).hexdigest()


def run(name):
    cname, prec, steps, cite = CASES[name]
    cfg = inputs.config(cname)
    p = oracle.Problem(tuple(cfg["dims"]), cfg["h"], a=cfg["a"], s=cfg["s"], bc=cfg["bc"], scheme=cfg["scheme"],
                       precision=prec)
    t0 = time.time()
    out = oracle.step(p, cfg["psi0"], cfg["k"], steps, cfg["V"])
    el = time.time() - t0
    return {"config": cname, "precision": prec, "steps": steps, "k": cfg["k"], "dims": list(cfg["dims"]),
            "sha256": digest(out, prec), "oracle_seconds": round(el, 1), "citation": cite,
            "max_abs": float(np.abs(out).max()), "finite": bool(np.all(np.isfinite(out)))}


def main():
    names = sys.argv[1:] or list(CASES)
    oracle.build()
    for name in names:
        res = run(name)
        with open(OUT + ".lock", "w") as lk:          # several generators may run at once
            fcntl.flock(lk, fcntl.LOCK_EX)
            d = json.load(open(OUT)) if os.path.exists(OUT) else {}
            d[name] = res
            with open(OUT, "w") as fh:
                json.dump(d, fh, indent=1, sort_keys=True)
        print(name, res["sha256"], res["oracle_seconds"], "s", flush=True)


if __name__ == "__main__":
    main()
