"""Time every BASELINE.json configuration through the C ABI (one GPU) and print a table.

    python scripts/bench_configs.py [--json out.json]

configs[0] 1D bright soliton (1000 steps), configs[1] 1D dark soliton (h = 0.1, t = 5),
configs[2] 2D trap 1024^2 (1000 steps), configs[3] 3D ring 87x87x203 (3360 steps, the
paper's benchmark: "about one and a half minutes" on a GTX 580) in fp64 and fp32,
configs[4] 3D GPE 1024^3 (20 steps).  Whole runs are timed with CUDA events on the library
stream after one warm-up call; updates/s = points x steps / time.
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--skip-1024", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch
    torch.cuda.set_device(0)
    from paper_1203_1263_b200 import inputs
    from paper_1203_1263_b200.nlse import Solver
    runs = []
    c = inputs.config("bright1d")
    runs.append(("configs[0] 1D bright soliton N=1025 2SHOC fp64 Dirichlet", c, c["steps"], "fp64"))
    c = inputs.config("dark1d_h0.1")
    kb = c["h"] ** 2 / math.sqrt(2) * 0.75
    nst = math.ceil(5.0 / (0.8 * kb))
    c["k"] = 5.0 / nst
    runs.append(("configs[1] 1D dark soliton N=1001 2SHOC MSD fp64 (t=5)", c, nst, "fp64"))
    runs.append(("configs[1] 1D dark soliton N=1001 2SHOC MSD fp32 (t=5)", c, nst, "fp32"))
    c = inputs.config("trap2d")
    runs.append(("configs[2] 2D trap 1024^2 2SHOC MSD fp64 + V", c, c["steps"], "fp64"))
    c = inputs.config("ring3d")
    runs.append(("configs[3] 3D ring 87x87x203 2SHOC MSD fp64 (paper benchmark)", c, c["steps"], "fp64"))
    runs.append(("configs[3] 3D ring 87x87x203 2SHOC MSD fp32", c, c["steps"], "fp32"))
    if not args.skip_1024:
        c = inputs.config("gpe3d")
        psi, V = inputs.gpe3d_fill(1024)
        c["psi0"], c["V"] = psi, V
        runs.append(("configs[4] 3D GPE 1024^3 2SHOC MSD fp64 + V", c, 20, "fp64"))
    out = []
    for name, c, nsteps, prec in runs:
        with Solver(c["dims"], c["h"], a=c["a"], s=c["s"], V=c["V"], bc=c["bc"], scheme=c["scheme"],
                    precision=prec, force_dt=False) as sv:
            sv.nlse_set_psi(c["psi0"])
            st = torch.cuda.ExternalStream(sv.nlse_get_stream())
            sv.nlse_step(c["k"], min(nsteps, 20))          # warm-up (and graph capture)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            sv.nlse_step(c["k"], nsteps)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            info = sv.nlse_get_info()
            pts = int(np.prod(c["dims"]))
            r = {"config": name, "points": pts, "steps": nsteps, "seconds": ms / 1e3,
                 "updates_per_s": pts * nsteps / (ms / 1e3), "us_per_step": 1e3 * ms / nsteps,
                 "variant": info["variant"],
                 "effective_GBps_Bmin": pts * nsteps * (16 * (16 if prec == "fp64" else 8) +
                                                       (4 * (8 if prec == "fp64" else 4) if c["V"] is not None else 0))
                                        / (ms / 1e3) / 1e9}
            out.append(r)
            print(f"{name:62s} {r['seconds']:9.4f} s  {r['us_per_step']:9.2f} us/step  "
                  f"{r['updates_per_s']:.3e} upd/s  {r['effective_GBps_Bmin']:8.1f} GB/s(B_min)  [{r['variant']}]",
                  flush=True)
    if args.json:
        json.dump(out, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
