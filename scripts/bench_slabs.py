#!/usr/bin/env python
"""Slab-mode overhead on one GPU: the same grid stepped as one context and
as P virtual ranks (nlse_dist_connect_local + nlse_step_group: P slab contexts on one device, the
same kernels, fused remote stores into the neighbours' ghost planes and device barriers as one
process per GPU).  The virtual ranks run one after another on one stream, so

    overhead(P) = t(P virtual ranks) / t(one context) - 1

is what slab mode adds per step when nothing overlaps: per-rank launch tails, the barrier kernels
(2 per rank per stage) and the remote stores of the w edge planes.  Prints one JSON line.

    python scripts/bench_slabs.py [--config gpe3d_512] [--steps 10] [--ranks 1,2,4,8]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gpe3d_512")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--ranks", default="1,2,4,8")
    args = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    from paper_1203_1263_b200 import build, inputs, nlse
    build.build()
    cfg = inputs.config(args.config)
    if cfg["psi0"] is None:
        cfg["psi0"], cfg["V"] = inputs.gpe3d_fill(cfg["dims"][0])
    dims, psi0, V = cfg["dims"], cfg["psi0"], cfg["V"]
    kw = dict(a=cfg["a"], s=cfg["s"], bc=cfg["bc"], scheme=cfg["scheme"], precision=cfg["precision"])
    out = {"config": args.config, "grid": list(dims), "steps": args.steps, "runs": []}
    ref = None
    for P in [int(x) for x in args.ranks.split(",")]:
        svs = []
        if P == 1:
            svs = [nlse.Solver(dims, cfg["h"], V=V, **kw)]
            svs[0].nlse_set_psi(psi0)
            step = lambda n: svs[0].nlse_step(cfg["k"], n)
        else:
            for r in range(P):
                z0, nl = nlse.nlse_slab_range(dims[-1], P, r)
                svs.append(nlse.Solver(dims, cfg["h"], V=None if V is None else np.ascontiguousarray(V[z0:z0 + nl]),
                                       dist=(r, P), **kw))
            nlse.nlse_dist_connect_local(svs)
            for sv in svs:
                sv.nlse_set_psi(np.ascontiguousarray(psi0[sv.z0:sv.z0 + sv.shape[0]]))
            step = lambda n: nlse.nlse_step_group(svs, cfg["k"], n)
        step(2)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step(args.steps)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / args.steps
        got = np.concatenate([sv.nlse_get_psi() for sv in svs], axis=0)
        if ref is None:
            ref = got
        same = bool(np.array_equal(got.view(np.uint64), ref.view(np.uint64)))
        for sv in svs:
            sv.close()
        out["runs"].append({"virtual_ranks": P, "ms_per_step": round(ms, 3), "bitwise_equal_to_P1": same})
        print(f"P={P}: {ms:.3f} ms/step, bitwise equal {same}", file=sys.stderr, flush=True)
    t1 = out["runs"][0]["ms_per_step"]
    for r in out["runs"]:
        r["overhead_vs_P1"] = round(r["ms_per_step"] / t1 - 1.0, 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
