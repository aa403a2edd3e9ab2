#!/usr/bin/env python
"""bench.py -- grid-point RK4 updates/s of the NLSE/GPE hot path (BASELINE.json metric).

Workload (N = 1): BASELINE configs[4], the 3D 1024^3 GPE, RK4 + 2SHOC, fp64, MSD,
harmonic-trap V array (the 3D fp64 2SHOC configuration the metric is quoted on at
1/2/4/8 GPUs; 77.3 GB of device state, far larger than L2).  A "step" is one RK4
step of the whole grid (all §8(a) rows: 4 fused stage kernels + boundary kernels).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config gpe3d|gpe3d_512|ring3d|...]
    python bench.py --impl reference ...     # the CPU oracle arm

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid-point RK4 updates/sec (3D 2SHOC fp64/fp32) and % HBM roofline at 1/2/4/8 GPU"
UNIT = "grid-point RK4 updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="gpe3d")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--generic", action="store_true", help="use the one-thread-per-point kernels")
    ap.add_argument("--scheme", default=None, help="override the workload's scheme (cd | 2shoc), for experiments")
    ap.add_argument("--precision", default=None, help="override the workload's precision (fp32 | fp64)")
    ap.add_argument("--bc", default=None, help="override the workload's boundary condition (dirichlet | msd | l0)")
    return ap.parse_args()


def workload(name, rank=0, world=1):
    """The workload's initial condition (and V): the whole grid at N = 1, this rank's z slab
    (planes [z0, z0 + nloc) of nlse_slab_range) in slab mode."""
    from paper_1203_1263_b200 import inputs
    cfg = inputs.config(name)
    cfg["z0"], cfg["nloc"] = 0, (cfg["dims"][2] if len(cfg["dims"]) == 3 else 1)
    if world > 1:
        from paper_1203_1263_b200.nlse import nlse_slab_range
        z0, nl = nlse_slab_range(cfg["dims"][-1], world, rank)
        cfg["z0"], cfg["nloc"] = z0, nl
        if name.startswith("gpe3d"):
            n = cfg["dims"][0]
            psi = np.empty((nl, n, n), np.complex128)
            V = np.empty((nl, n, n), np.float64)
            step = 8
            for a in range(0, nl, step):
                b = min(nl, a + step)
                psi[a:b], V[a:b] = inputs.gpe3d_slab(n, z0 + a, z0 + b, cfg["h"])
            cfg["psi0"], cfg["V"] = psi, V
        else:
            cfg["psi0"] = np.ascontiguousarray(cfg["psi0"][z0:z0 + nl])
            if cfg["V"] is not None:
                cfg["V"] = np.ascontiguousarray(cfg["V"][z0:z0 + nl])
    elif name.startswith("gpe3d"):
        n = cfg["dims"][0]
        psi, V = inputs.gpe3d_fill(n)
        cfg["psi0"], cfg["V"] = psi, V
    return cfg


def bytes_min_per_point(cfg):
    """B_min = 16c + 4 r_V bytes per point per RK4 step."""
    r = 8 if cfg["precision"] == "fp64" else 4
    return 16 * 2 * r + (4 * r if cfg["V"] is not None else 0)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and s[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def ncu_traffic(variant, pts_per_launch):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from the
    committed `ncu --set full` summary (profiles/ncu_traffic.json: bytes per interior point,
    averaged over the four stage launches of one RK4 step), scaled to this launch's points."""
    f = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(f)).get(variant)
    except Exception:
        return None, None
    if not d:
        return None, None
    return float(d["dram_bytes_per_point_stage"]) * pts_per_launch, f"profiles/ncu_traffic.json ({d['capture']})"


def oracle_cores():
    """Threads the OpenMP oracle build uses (OMP_NUM_THREADS, else every host core)."""
    env = os.environ.get("OMP_NUM_THREADS")
    return int(env) if env and env.isdigit() else (os.cpu_count() or 1)


def oracle_sample(cfg, planes=32):
    """A bounded, representative sample of the workload for the CPU oracle: a z-slab of `planes`
    planes from the middle of a 3D grid (interior-dominated like the full grid; its own MSD
    boundary), or the whole grid in 1D/2D.  Returns (dims, psi, V, description)."""
    from paper_1203_1263_b200 import inputs
    nx, ny, nz = (list(cfg["dims"]) + [1, 1])[:3]
    if len(cfg["dims"]) == 3:
        planes = min(nz, planes)
        z0 = max(0, nz // 2 - planes // 2)
        if cfg.get("psi0") is not None:
            psi = np.ascontiguousarray(cfg["psi0"][z0:z0 + planes])
            V = None if cfg["V"] is None else np.ascontiguousarray(cfg["V"][z0:z0 + planes])
        else:
            psi, V = inputs.gpe3d_slab(nx, z0, z0 + planes, cfg["h"])
        return (nx, ny, planes), psi, V, f"{nx}x{ny}x{planes} z-slab (planes {z0}..{z0 + planes - 1}) of the workload IC"
    return tuple(cfg["dims"]), cfg["psi0"], cfg["V"], "full workload grid"


def cpu_baseline_sample(cfg):
    """The oracle as it stands on the host cores, on a bounded sample of the same workload:
    the OpenMP build (outer loop of each sweep over all cores; same bits as the serial oracle)
    for `value`, plus the serial build on the same sample (`serial_value`, the paper-equivalent
    one-core baseline)."""
    import oracle
    oracle.build()
    dims, psi, V, desc = oracle_sample(cfg)
    p = oracle.Problem(dims, cfg["h"], a=cfg["a"], s=cfg["s"], bc=cfg["bc"], scheme=cfg["scheme"],
                       precision=cfg["precision"])
    pts = int(np.prod(dims))
    out = {}
    for omp, budget in ((True, 6.0), (False, 4.0)):
        sub = psi
        t0 = time.perf_counter()
        nst = 0
        while True:
            sub = oracle.step(p, sub, cfg["k"], 1, V, omp=omp)
            nst += 1
            el = time.perf_counter() - t0
            if el > budget or nst >= 50:
                break
        out[omp] = (pts * nst / el, nst, el)
    v, nst, el = out[True]
    sv, sn, se = out[False]
    return {"value": v, "unit": UNIT, "cores": oracle_cores(), "kind": "oracle",
            "sample": f"{desc}, {nst} RK4 step(s) in {el:.1f} s, OpenMP build of the C oracle "
                      f"(-O2 -ffp-contract=off) on {oracle_cores()} threads",
            "serial_value": sv, "serial_sample": f"same sample, {sn} RK4 step(s) in {se:.1f} s on 1 core"}


def run_reference(args):
    """--impl reference: the CPU oracle arm (OpenMP build, all host cores), on this arm's
    config/metric, each bench step one RK4 step of a bounded sample of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    from paper_1203_1263_b200 import inputs
    cfg = inputs.config(args.config)
    dims, psi, V, desc = oracle_sample(cfg)
    desc += ", 1 RK4 step per bench step"
    p = oracle.Problem(dims, cfg["h"], a=cfg["a"], s=cfg["s"], bc=cfg["bc"], scheme=cfg["scheme"],
                       precision=cfg["precision"])
    for _ in range(args.warmup):
        psi = oracle.step(p, psi, cfg["k"], 1, V, omp=True)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        psi = oracle.step(p, psi, cfg["k"], 1, V, omp=True)
    el = time.perf_counter() - t0
    pts = int(np.prod(dims))
    val = pts * args.steps / el
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if cfg["precision"] == "fp64" else "f32", "data": "synthetic",
            "config": config_block(cfg, args),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": oracle_cores(), "kind": "oracle",
                             "sample": desc + f", OpenMP build of the C oracle on {oracle_cores()} threads"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def inputs_dims(name):
    from paper_1203_1263_b200 import inputs
    return inputs.config_dims(name)


def config_block(cfg, args, replicas=False):
    return {"workload": f"{cfg['name']}: {'x'.join(map(str, cfg['dims']))} {cfg['scheme'].upper()} RK4, "
                        f"{cfg['bc'].upper()} BC, {cfg['precision']}, "
                        f"{'harmonic-trap V array' if cfg.get('has_V', cfg['V'] is not None) else 'V=0'} (BASELINE.json configs)",
            "grid": list(cfg["dims"]), "h": cfg["h"], "k": cfg["k"], "scheme": cfg["scheme"], "bc": cfg["bc"],
            "precision": cfg["precision"], "a": cfg["a"], "s": cfg["s"],
            "parallelism": (f"{args.gpus} independent replicas (1D and small 2D grids are not partitioned)" if replicas
                            else ((f"{'z' if len(cfg['dims']) == 3 else 'y'}-slab x{args.gpus}") if args.gpus > 1
                                  else "single GPU")),
            "l2": "inputs larger than L2 (no flush needed)" if int(np.prod(cfg["dims"])) * 64 > 2e9
                  else "working set L2-resident (L2-scale config, no flush)"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        ndev = torch.cuda.device_count()
        torch.cuda.set_device(local % ndev)
        # torch.distributed is plumbing only here (handle all-gather, max-over-ranks timing;
        # the halo exchange runs over peer memory).  NCCL with one GPU per rank; gloo when
        # several ranks share a GPU (functional test of the N>1 path on a 1-GPU box).
        backend = "nccl" if ndev >= world else "gloo"
        dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    from paper_1203_1263_b200 import build
    build.build()
    from paper_1203_1263_b200.nlse import Solver

    # 3D grids are z-slab partitioned and 2D grids of >= 4096^2 points y-slab partitioned (strong
    # scaling); 1D grids and smaller 2D grids, whose per-GPU stage is shorter than a neighbour
    # barrier, run one independent replica per rank (weak scaling)
    dims_ = inputs_dims(args.config)
    replicas = world > 1 and (len(dims_) == 1 or (len(dims_) == 2 and int(np.prod(dims_)) < 4096 * 4096))
    slab = world > 1 and not replicas
    cfg = workload(args.config, rank, world if slab else 1)
    if args.scheme:
        cfg["scheme"] = args.scheme
    if args.precision:
        cfg["precision"] = args.precision
    if args.bc:
        cfg["bc"] = args.bc
    B = bytes_min_per_point(cfg)
    peak, peak_src = measured_peaks()
    npts = int(np.prod(cfg["dims"])) * (world if replicas else 1)   # whole job
    sv = Solver(cfg["dims"], cfg["h"], a=cfg["a"], s=cfg["s"], V=cfg["V"], bc=cfg["bc"], scheme=cfg["scheme"],
                precision=cfg["precision"], generic=args.generic, dist=(rank, world) if slab else None)
    if slab:
        from paper_1203_1263_b200 import dist as pdist
        pdist.connect(sv)
    info = sv.nlse_get_info()
    nloc_pts = info["points"]
    sv.nlse_set_psi(cfg["psi0"])
    stream = torch.cuda.ExternalStream(sv.nlse_get_stream())
    k = cfg["k"]
    # warm-up: W steps, at least 2 x 8 so that the CUDA graph of 8 steps nlse_step replays for
    # long calls is captured and instantiated before the timed region (reported as "warmup")
    warmup = max(args.warmup, 16)
    sv.nlse_step(k, warmup)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local % max(1, torch.cuda.device_count())) as clk:
        # (1) the bench value: K steps, CUDA events on the library's stream around one nlse_step call
        e0.record(stream)
        sv.nlse_step(k, args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        # (2) the roofline: the same K steps again with per-launch events (kernel shares, launch times)
        sv.nlse_set_timing(True)
        sv.nlse_reset_timing()
        sv.nlse_step(k, args.steps)
        sv.nlse_set_timing(False)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda" if backend == "nccl" else "cpu")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    timing = sv.nlse_get_timing()
    value = npts * args.steps / (ms / 1e3)

    # dominant kernel: the interior stage kernel family
    # persistent kernels (one launch per nlse_step call) are timed under their tile kind
    dom = {"rk4_2d_persistent": "stage2d_tile", "rk4_1d_persistent": "stage1d_tile", "rk4_1d_cluster": "stage1d_tile"}.get(info["variant"], info["variant"])
    td = timing[dom]
    avg_launch_ms = td["ms"] / max(td["launches"], 1)
    pts_per_launch = td["points"] / max(td["launches"], 1)
    if dom == "fused3d_cd":
        # temporal blocking (§8(f) rank 2): each launch is two stages; its compulsory bytes are
        # (3c + r_V) for S1+S2 and (4c + r_V) for S3+S4, i.e. (7c + 2 r_V)/2 per point on average
        c_ = 16 if cfg["precision"] == "fp64" else 8
        r_ = (c_ // 2) if cfg["V"] is not None else 0
        B_fused = 7 * c_ + 2 * r_
        alg_bytes_launch = pts_per_launch * B_fused / 2.0
    else:
        B_fused = None
        alg_bytes_launch = pts_per_launch * B / 4.0      # B_min per point per step spread over 4 stages
    achieved = alg_bytes_launch / (avg_launch_ms / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(dom, pts_per_launch)
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "kernel": dom, "alg_bytes_per_launch": alg_bytes_launch, "avg_launch_ms": avg_launch_ms,
            "peak_source": peak_src, "traffic_source": traffic_src,
            "kernel_share_of_step": round(td["ms"] / sum(v["ms"] for v in timing.values() if v["launches"]), 4),
            "step_frac_of_roofline": round(value * B / 1e9 / peak, 4),
            "bytes_per_point_step": B}
    if B_fused:
        roof["fused_bytes_per_point_step"] = B_fused
        roof["step_frac_of_fused_roofline"] = round(value * B_fused / 1e9 / peak, 4)

    # e2e: the paper's chunk model through the public API with host buffers: per chunk of
    # `steps` RK4 steps, H2D of Psi from pinned memory, the steps, D2H of Psi to pinned memory.
    e2e = None
    if not args.no_e2e:
        pinned = torch.empty(nloc_pts * 2, dtype=torch.float64, pin_memory=True)
        host = pinned.numpy().view(np.complex128).reshape(sv.shape)
        host[...] = cfg["psi0"]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sv.nlse_set_psi(host)
        sv.nlse_step(k, args.steps)
        sv.nlse_get_psi(host)
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], device="cuda" if backend == "nccl" else "cpu")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": npts * args.steps / el, "unit": UNIT, "h2d_bytes_per_step": npts * 16 // args.steps,
               "d2h_bytes_per_step": npts * 16 // args.steps, "chunk_steps": args.steps,
               "what": "nlse_set_psi(pinned host) + nlse_step(k, steps) + nlse_get_psi(pinned host), wall clock, "
                       "max over ranks; bytes summed over ranks (complex128 host I/O)"}
        del pinned, host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(cfg)
    sv.close()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak" if replicas else "strong", "vs_baseline": None,
                "dtype": "f64" if cfg["precision"] == "fp64" else "f32", "data": "synthetic",
                "config": config_block(cfg, args, replicas), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(args.steps * info["launches_per_step"]), "clocks": clk.summary(),
                "kernel_timing": {k2: v for k2, v in timing.items() if v["launches"]},
                "pct_hbm_roofline": round(100 * value * B / 1e9 / peak, 2)}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
