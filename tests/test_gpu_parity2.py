"""GPU parity, round 2: the configurations the round-1 review found without a GPU-vs-oracle
check -- the MSD division guard taken on every kernel path, 1D grids above the persistent-CTA
limit, the frames model against oracle frames, and the BASELINE configurations after their full
stated step counts (against oracle digests in tests/golden/oracle_sha256.json).
Bar: bit-identical, as test_gpu_parity.py."""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from helpers import assert_parity, case_input, guard_field, run_gpu, run_oracle
from paper_1203_1263_b200 import inputs

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "oracle_sha256.json")


def _k(ndim, h, scheme):
    kb = h * h / (ndim * math.sqrt(2)) * (0.75 if scheme == "2shoc" else 1.0)
    return 0.5 * kb


VARIANT_ENV = {
    "fast": {}, "generic": {},
    "edge_lean": {"NLSE_FORCE_EDGE": "1"}, "edge_pp": {"NLSE_FORCE_EDGE": "2"},
    "msd_recompute": {"NLSE_MSD_FB": "0"}, "xfuse_off": {"NLSE_XFUSE": "0"}, "xfuse_on": {"NLSE_XFUSE": "1"},
    "v1": {"NLSE_3D_KERNEL": "v1"},
}


@pytest.mark.parametrize("kernel", list(VARIANT_ENV))
@pytest.mark.parametrize("withV", [False, True], ids=["V0", "V"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("dims", [(1029,), (3001,), (8001,), (133, 70), (70, 37, 29)],
                         ids=["1d", "1d_3pts_per_thread", "1d_tiled", "2d", "3d"])
def test_msd_eps_guard_bitwise(dims, precision, withV, kernel, monkeypatch):
    """R-MSD-GUARD on the GPU: Psi_b' = 0 and eps/2 (guard taken) at face, edge and corner
    neighbours (tests/helpers.guard_points); every kernel path that forms an MSD
    boundary value (the TMA stage kernel's face D and x-face F, the light pass, the recompute
    kernel, the 2D tile kernel, the 1D persistent and tiled kernels, the generic kernel) matches
    the oracle bit for bit.  The guard fires in stage 1 of step 1; later stages see the evolved
    field."""
    if kernel not in ("fast", "generic") and len(dims) != 3:
        pytest.skip("3D kernel variant")
    for k_, v_ in VARIANT_ENV[kernel].items():
        monkeypatch.setenv(k_, v_)
    ndim = len(dims)
    h = {1: 0.05, 2: 0.2, 3: 0.5}[ndim]
    psi0 = guard_field(dims, precision, above=False)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=300 + ndim)) if withV else None
    kw = dict(a=0.9, s=-1.1, V=V, bc="msd", scheme="2shoc", precision=precision)
    k = _k(ndim, h, "2shoc")
    ref = run_oracle(dims, h, psi0, k, 3, **kw)
    assert np.all(np.isfinite(ref))
    got = run_gpu(dims, h, psi0, k, 3, generic=kernel == "generic", **kw)
    assert_parity(got, ref, precision, what=f"guard {dims} {precision} V={withV} {kernel}")


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("bc", ["dirichlet", "msd", "l0"])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
@pytest.mark.parametrize("n", [8001, 100001])
def test_1d_large_grids_bitwise(n, scheme, bc, precision, monkeypatch):
    """1D grids above the persistent single-CTA limit (the paper's Table 1 runs 1D to 3e6 points,
    P:664-686) take the tiled 1D stage kernels (NLSE_1D_CLUSTER=0: not the cluster kernel, which
    holds up to ~25K points): bit for bit against the oracle, with a V array."""
    monkeypatch.setenv("NLSE_1D_CLUSTER", "0")
    dims = (n,)
    h = 0.05
    psi0 = case_input(dims, seed=n % 997)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=11))
    kw = dict(a=0.9, s=-1.1, V=V, bc=bc, scheme=scheme, precision=precision)
    k = _k(1, h, scheme)
    ref = run_oracle(dims, h, psi0, k, 9, **kw)
    got, info = run_gpu(dims, h, psi0, k, 9, with_info=True, **kw)
    assert info["variant"] != "rk4_1d_persistent", info
    assert_parity(got, ref, precision, what=f"1D n={n} {scheme} {bc} {precision} {info['variant']}")


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("bc", ["dirichlet", "msd", "l0"])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
@pytest.mark.parametrize("kernel", ["single", "auto", "c2", "c3", "c8"])
@pytest.mark.parametrize("n", [3, 4, 5, 1023, 1024, 1025, 2049, 3001, 10001])
def test_1d_persistent_sizes_bitwise(n, scheme, bc, precision, kernel, monkeypatch):
    """The persistent 1D kernels: one CTA (one block phase per stage since round 2: D at a point's
    neighbours and F at b' recomputed by the thread), from 3 points to 3 points per thread; and the
    thread-block-cluster variant (segments of the grid in 2-8 CTAs, neighbours' points through
    distributed shared memory, a cluster barrier per stage)."""
    env = {"single": "0", "auto": None, "c2": "2", "c3": "3", "c8": "8"}[kernel]
    if env is not None:
        monkeypatch.setenv("NLSE_1D_CLUSTER", env)
    if kernel == "single" and n > 3001:
        pytest.skip("beyond one CTA's shared memory")
    dims = (n,)
    h = 0.05
    psi0 = case_input(dims, seed=n % 991)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=12))
    kw = dict(a=0.9, s=-1.1, V=V, bc=bc, scheme=scheme, precision=precision)
    k = _k(1, h, scheme)
    ref = run_oracle(dims, h, psi0, k, 23, **kw)
    got, info = run_gpu(dims, h, psi0, k, 23, with_info=True, **kw)
    if kernel == "single":
        assert info["variant"] == "rk4_1d_persistent", info
    elif kernel != "auto" and 4 * int(env) <= n <= 3001:   # (a forced cluster whose segments fit)
        assert info["variant"] == "rk4_1d_cluster", info
    assert_parity(got, ref, precision, what=f"1D n={n} {scheme} {bc} {precision} {info['variant']}")


@pytest.mark.parametrize("ndim,precision,chunk", [(3, "fp64", 20), (3, "fp32", 3), (1, "fp64", 7), (2, "fp32", 5),
                                                  (2, "fp64", 17)])
def test_run_frames_match_oracle(ndim, precision, chunk):
    """nlse_run_frames (the paper's frames model): frame f equals the oracle's
    field after (f + 1) x chunk steps, bit for bit."""
    from paper_1203_1263_b200.nlse import Solver
    dims = {1: (301,), 2: (70, 41), 3: (40, 26, 22)}[ndim]
    h = {1: 0.1, 2: 0.2, 3: 0.5}[ndim]
    psi0 = case_input(dims, seed=91)
    V = 0.2 * np.abs(inputs.random_smooth(dims, seed=92))
    k = _k(ndim, h, "2shoc")
    kw = dict(s=-1.0, V=V, bc="msd", scheme="2shoc", precision=precision)
    with Solver(dims, h, force_dt=True, **kw) as sv:
        sv.nlse_set_psi(psi0)
        frames = sv.nlse_run_frames(k, chunk, 3)
    ref = psi0
    for f in range(3):
        ref = run_oracle(dims, h, ref, k, chunk, **kw)
        assert_parity(frames[f], ref, precision, what=f"frame {f}")


def _golden(name):
    with open(GOLDEN) as fh:
        return json.load(fh)[name]


@pytest.mark.parametrize("name", ["trap2d_fp64_1000", "ring3d_fp64_3360", "ring3d_fp32_3360"])
def test_full_step_counts_match_oracle_digest(name):
    """BASELINE configs[2] (1024^2 trap, 1000 steps) and configs[3] (87x87x203 ring, 3360 steps,
    P:69) after their stated step counts: the SHA-256 of the whole GPU field equals the digest of
    the oracle's field (scripts/make_goldens.py, which calls only oracle/)."""
    g = _golden(name)
    cfg = inputs.config(g["config"])
    assert list(cfg["dims"]) == g["dims"] and cfg["k"] == g["k"]
    got = run_gpu(cfg["dims"], cfg["h"], cfg["psi0"], cfg["k"], g["steps"], a=cfg["a"], s=cfg["s"], V=cfg["V"],
                  bc=cfg["bc"], scheme=cfg["scheme"], precision=g["precision"], force_dt=False)
    dt = np.complex128 if g["precision"] == "fp64" else np.complex64
    h = hashlib.sha256(np.ascontiguousarray(got.astype(dt)).tobytes()).hexdigest()
    assert np.all(np.isfinite(got)) and g["finite"]
    assert h == g["sha256"], (name, float(np.abs(got).max()), g["max_abs"])


@pytest.mark.parametrize("persist", ["1", "0"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("bc", ["dirichlet", "msd", "l0"])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
def test_2d_persistent_and_per_stage_bitwise(scheme, bc, precision, persist, monkeypatch):
    """2D grids up to 2^21 points run every stage of an nlse_step call in one cooperative launch
    (rk4_2d_persistent: grid-wide barriers between stages); NLSE_PERSIST2D=0 forces the per-stage
    kernels (the default warp-strip kernel).  Both bit for bit against the oracle, chunked calls included."""
    monkeypatch.setenv("NLSE_PERSIST2D", persist)
    dims, h = (133, 70), 0.2
    psi0 = case_input(dims, seed=61)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=62))
    kw = dict(a=0.9, s=-1.1, V=V, bc=bc, scheme=scheme, precision=precision)
    k = _k(2, h, scheme)
    ref = run_oracle(dims, h, psi0, k, 19, **kw)
    got, info = run_gpu(dims, h, psi0, k, 19, chunks=[1, 17, 1], with_info=True, **kw)
    assert info["variant"] == ("rk4_2d_persistent" if persist == "1" else "stage2d_strip"), info
    assert_parity(got, ref, precision, what=f"2D persist={persist} {scheme} {bc} {precision}")


def test_c_client_matches_oracle(tmp_path):
    """A plain C client of include/nlse.h (tests/c/abi_demo.c: create, set_psi, step, get_psi,
    diagnostics, destroy) returns the oracle's field bit for bit: the C ABI is the product
    boundary, the ctypes binding only marshals arguments."""
    import subprocess
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from test_abi import build_c_demo
    exe = build_c_demo(tmp_path)
    dims, nsteps = (37, 21, 19), 7
    psi0 = case_input(dims, seed=71)
    fin, fout = str(tmp_path / "in.bin"), str(tmp_path / "out.bin")
    np.ascontiguousarray(psi0, np.complex128).tofile(fin)
    res = subprocess.run([exe, *map(str, dims), str(nsteps), fin, fout], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    got = np.fromfile(fout, dtype=np.complex128).reshape(tuple(reversed(dims)))
    k = float(res.stdout.split()[1])
    ref = run_oracle(dims, 0.5, psi0, k, nsteps, a=1.0, s=-1.0, bc="msd", scheme="2shoc")
    assert_parity(got, ref, "fp64", what="C client")
