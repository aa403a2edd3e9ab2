#!/usr/bin/env python
"""Size sweeps of SURVEY §8(d) ("extra sweeps") and the paper's Table 1-3 sizes: bench.py's
device-timed measurement (CUDA events around one nlse_step call on the library stream, after
warm-up) for a list of configurations, one JSON line each with updates/s, us/step and the
fraction of the HBM roofline (B_min = 16c + 4 r_V bytes per point-step).

    python scripts/bench_sizes.py [--set 1d|big|all] [--generic]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SETS = {
    "1d": ["dark1d_n1000", "dark1d_n10000", "dark1d_n100000", "dark1d_n1000000", "dark1d_n3000000",
           "dark1d_n134217729"],
    "big": ["trap2d_16384", "gpe3d_512", "gpe3d_768"],
}


def run(name, generic=False, precision=None, scheme=None, min_ms=200.0):
    import torch
    from paper_1203_1263_b200 import inputs
    from paper_1203_1263_b200.nlse import Solver
    cfg = inputs.config(name)
    if cfg["psi0"] is None:
        cfg["psi0"], cfg["V"] = inputs.gpe3d_fill(cfg["dims"][0])
    prec = precision or cfg["precision"]
    sch = scheme or cfg["scheme"]
    with Solver(cfg["dims"], cfg["h"], a=cfg["a"], s=cfg["s"], V=cfg["V"], bc=cfg["bc"], scheme=sch,
                precision=prec, generic=generic, force_dt=True) as sv:
        sv.nlse_set_psi(cfg["psi0"])
        info = sv.nlse_get_info()
        stream = torch.cuda.ExternalStream(sv.nlse_get_stream())
        sv.nlse_step(cfg["k"], 16)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sv.nlse_step(cfg["k"], 16)
        e1.record(stream)
        torch.cuda.synchronize()
        per = e0.elapsed_time(e1) / 16
        nst = int(max(16, min(20000, min_ms / max(per, 1e-4))))
        e0.record(stream)
        sv.nlse_step(cfg["k"], nst)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / nst
    pts = int(np.prod(cfg["dims"]))
    c = 16 if prec == "fp64" else 8
    B = 16 * c + (4 * c // 2 if cfg["V"] is not None else 0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    return {"config": name, "grid": list(cfg["dims"]), "precision": prec, "scheme": sch, "bc": cfg["bc"],
            "V": cfg["V"] is not None, "kernel": info["variant"], "steps_timed": nst, "us_per_step": ms * 1e3,
            "updates_per_s": pts / (ms / 1e3), "hbm_roofline_frac": pts * B / (ms / 1e3) / 1e9 / peak,
            "bytes_per_point_step": B}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", default="1d")
    ap.add_argument("--generic", action="store_true")
    ap.add_argument("--configs", default=None)
    args = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    from paper_1203_1263_b200 import build
    build.build()
    names = args.configs.split(",") if args.configs else (SETS["1d"] + SETS["big"] if args.set == "all" else SETS[args.set])
    for n in names:
        print(json.dumps(run(n, generic=args.generic)), flush=True)


if __name__ == "__main__":
    main()
