"""The paper's chunk-size experiment (Fig. chunk-size) on a B200: wall-clock cost of
returning Psi to the host every `chunk` steps, relative to running all steps on the device.

    python scripts/bench_frames.py [--config ring3d] [--steps 1000]

For each chunk size c: (a) nlse_run_frames(k, c, steps/c) -- downloads of frame f overlap the
compute of chunk f+1; (b) the naive loop nlse_step(k, c); nlse_get_psi() (no overlap); both
against (c) one nlse_step(k, steps).  Host frames are pinned (torch).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="ring3d")
    ap.add_argument("--steps", type=int, default=960)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    import numpy as np
    import torch
    torch.cuda.set_device(0)
    from paper_1203_1263_b200 import inputs
    from paper_1203_1263_b200.nlse import Solver
    c = inputs.config(args.config)
    out = []
    with Solver(c["dims"], c["h"], a=c["a"], s=c["s"], V=c["V"], bc=c["bc"], scheme=c["scheme"],
                precision=c["precision"]) as sv:
        sv.nlse_set_psi(c["psi0"])
        sv.nlse_step(c["k"], 16)
        t0 = time.perf_counter(); sv.nlse_step(c["k"], args.steps); base = time.perf_counter() - t0
        for chunk in (10, 20, 40, 80, 160, 320):
            nf = args.steps // chunk
            n2 = 2 * int(np.prod(c["dims"]))
            pinned = torch.empty(nf * n2, dtype=torch.float64, pin_memory=True)
            frames = pinned.numpy().view(np.complex128).reshape((nf,) + sv.shape)
            t0 = time.perf_counter(); sv.nlse_run_frames(c["k"], chunk, nf, frames); ovl = time.perf_counter() - t0
            one = torch.empty(n2, dtype=torch.float64, pin_memory=True).numpy().view(np.complex128).reshape(sv.shape)
            t0 = time.perf_counter()
            for _ in range(nf):
                sv.nlse_step(c["k"], chunk)
                sv.nlse_get_psi(one)
            naive = time.perf_counter() - t0
            r = {"chunk": chunk, "frames": nf, "steps": nf * chunk, "device_only_s": base * nf * chunk / args.steps,
                 "frames_overlapped_s": ovl, "frames_naive_s": naive}
            r["slowdown_overlapped"] = ovl / r["device_only_s"]
            r["slowdown_naive"] = naive / r["device_only_s"]
            out.append(r)
            print(f"chunk {chunk:4d}: device-only {r['device_only_s']:.4f} s, frames overlapped {ovl:.4f} s "
                  f"(x{r['slowdown_overlapped']:.2f}), step+get {naive:.4f} s (x{r['slowdown_naive']:.2f})", flush=True)
            del pinned, frames
    if args.json:
        json.dump({"config": args.config, "rows": out}, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
