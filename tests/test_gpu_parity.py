"""GPU parity: the CUDA path through the C ABI against the CPU oracle, element by
element, on the same seeded inputs.  Bar: bit-identical (max ulp 0), which implies
the north-star tolerances (rel-L2 1e-12 fp64, 1e-5 fp32)."""
import math

import numpy as np
import pytest

from helpers import assert_parity, case_input, rel_l2, run_gpu, run_oracle, ulp_diff
from paper_1203_1263_b200 import inputs

pytestmark = pytest.mark.gpu

# Sizes span several tiles of every kernel family plus ragged tails, yet the oracle
# finishes each case in well under a second.
DIMS = {1: (1029,), 2: (133, 70), 3: (70, 37, 29)}
H = {1: 0.05, 2: 0.2, 3: 0.5}


def _k(ndim, h, scheme):
    kb = h * h / (ndim * math.sqrt(2)) * (0.75 if scheme == "2shoc" else 1.0)
    return 0.5 * kb


@pytest.mark.parametrize("kernel", ["fast", "edge_off", "edge_lean", "edge_pp", "msd_recompute", "xfuse_off", "xfuse_on",
                                    "v1", "tile2d", "generic"])
@pytest.mark.parametrize("withV", [False, True], ids=["V0", "V"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("bc", ["dirichlet", "msd", "l0"])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_matrix_bitwise(ndim, scheme, bc, precision, withV, kernel, monkeypatch):
    """Every kernel family against the oracle: "fast" = the default (3D: TMA z-streaming, 2D: warp
    strips), "v1" = the cp.async z-streaming kernel (3D), "tile2d" = the shared-tile 2D kernel +
    boundary kernel, "generic" = one thread per point."""
    if kernel == "tile2d":
        if ndim != 2:
            pytest.skip("tile2d is a 2D kernel variant")
        monkeypatch.setenv("NLSE_2D_KERNEL", "tile")
    elif kernel != "fast" and kernel != "generic" and ndim != 3:
        pytest.skip(f"{kernel} is a 3D kernel variant")
    if kernel == "v1":
        monkeypatch.setenv("NLSE_3D_KERNEL", "v1")
    if kernel == "msd_recompute":       # 3D MSD: boundary kernel recomputes F(b'), concurrent on the side stream
        if bc != "msd":
            pytest.skip("MSD only")
        monkeypatch.setenv("NLSE_MSD_FB", "0")
    if kernel in ("xfuse_off", "xfuse_on"):   # 3D MSD: x-face points by the light pass / the stage kernel
        if bc != "msd":
            pytest.skip("MSD only")
        monkeypatch.setenv("NLSE_XFUSE", "0" if kernel == "xfuse_off" else "1")
    if kernel.startswith("edge"):       # interior tiles on the branch-free loop (0) / every TMA tile on the lean
        # face-aware loop (1) / on the per-point face path (2); default: 1 where most tiles touch a face
        monkeypatch.setenv("NLSE_FORCE_EDGE", {"edge_off": "0", "edge_lean": "1", "edge_pp": "2"}[kernel])
    generic = kernel == "generic"
    dims = DIMS[ndim]
    h = H[ndim]
    psi0 = case_input(dims, seed=100 + ndim)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=200 + ndim)) if withV else None
    k = _k(ndim, h, scheme)
    n = 12
    kw = dict(a=0.9, s=-1.1, V=V, bc=bc, scheme=scheme, precision=precision)
    ref = run_oracle(dims, h, psi0, k, n, **kw)
    got, info = run_gpu(dims, h, psi0, k, n, generic=generic, with_info=True, **kw)
    want = {"fast": {1: "rk4_1d_cluster" if precision == "fp64" else "rk4_1d_persistent", 2: "stage2d_strip",
                     3: "stage3d_tma"}[ndim], "v1": "stage3d_stream",
            "tile2d": "stage2d_tile", "edge_off": "stage3d_tma",
            "edge_lean": "stage3d_tma", "edge_pp": "stage3d_tma", "msd_recompute": "stage3d_tma", "xfuse_off": "stage3d_tma", "xfuse_on": "stage3d_tma",
            "generic": "stage_generic"}[kernel]
    if not (kernel in ("fast", "edge_off", "edge_lean", "edge_pp", "msd_recompute", "xfuse_off", "xfuse_on") and ndim == 3 and precision == "fp32" and withV):   # fp32 V rows: 4*70 B
        assert info["variant"] == want, info
    assert_parity(got, ref, precision, what=f"{ndim}D {scheme} {bc} {precision} V={withV} {info['variant']}")


@pytest.mark.parametrize("force_edge", ["auto", "0"])
@pytest.mark.parametrize("dims", [(65, 33, 9), (33, 17, 7), (64, 31, 8), (97, 49, 6), (63, 47, 7), (35, 20, 6)])
@pytest.mark.parametrize("bc", ["dirichlet", "msd", "l0"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_tile_alignment_cases(dims, bc, precision, force_edge, monkeypatch):
    """3D grids whose faces fall on every tile position the TMA kernel distinguishes: a face one
    past a tile (nx = 32k + 1, ny = 16k + 1: the face is on the neighbour tile's ring), a face on
    lane 0 of a tile (x-face b' on the previous tile), faces on the last lane / row, ragged."""
    psi0 = case_input(dims, seed=77)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=78))
    h = 0.5
    k = _k(3, h, "2shoc")
    kw = dict(a=0.9, s=-1.1, V=V, bc=bc, scheme="2shoc", precision=precision)
    ref = run_oracle(dims, h, psi0, k, 6, **kw)
    got = run_gpu(dims, h, psi0, k, 6, **kw)
    assert_parity(got, ref, precision, what=f"{dims} {bc} {precision}")


@pytest.mark.parametrize("band", ["0", "1", "3", "4", "16"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_tile_band_orders(band, precision, monkeypatch):
    """The 3D TMA kernel's tile order within a z chunk (row-major, or bands of B tile rows walked
    column by column, the last band partial): every tile exactly once, bit for bit."""
    monkeypatch.setenv("NLSE_TILE_BAND", band)
    dims = (70, 146, 6)              # 3 x 10 tiles of 32 x 16 (fp64) / 3 x 19 of 32 x 8 (fp32)
    psi0 = case_input(dims, seed=44)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=45))
    h = 0.5
    kw = dict(a=0.9, s=-1.1, V=V, bc="msd", scheme="2shoc", precision=precision)
    ref = run_oracle(dims, h, psi0, _k(3, h, "2shoc"), 4, **kw)
    got = run_gpu(dims, h, psi0, _k(3, h, "2shoc"), 4, **kw)
    assert_parity(got, ref, precision, what=f"band {band} {precision}")


@pytest.mark.parametrize("dims", [(3,), (4,), (3, 3), (3, 5), (5, 3), (3, 3, 3), (4, 3, 5), (3, 7, 3), (9, 3, 4)])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
@pytest.mark.parametrize("bc", ["dirichlet", "msd", "l0"])
def test_degenerate_small_grids(dims, scheme, bc):
    """The smallest legal grids (3 points per axis: one interior layer) and thin slabs."""
    psi0 = case_input(dims, seed=5)
    h = 0.5
    k = _k(len(dims), h, scheme)
    ref = run_oracle(dims, h, psi0, k, 7, s=-1.0, bc=bc, scheme=scheme)
    got = run_gpu(dims, h, psi0, k, 7, s=-1.0, bc=bc, scheme=scheme)
    assert_parity(got, ref, "fp64", what=f"{dims}")


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_chunk_invariance(precision):
    dims = (40, 33, 21)
    psi0 = case_input(dims, seed=9)
    k = _k(3, 0.5, "2shoc")
    a = run_gpu(dims, 0.5, psi0, k, 24, s=-1.0, bc="msd", precision=precision)
    b = run_gpu(dims, 0.5, psi0, k, 24, s=-1.0, bc="msd", precision=precision, chunks=[1, 5, 7, 11])
    assert ulp_diff(a, b, precision) == 0


def test_config1_bright_soliton_full():
    """configs[0]: 1D bright soliton, N=1025, h=0.05, 2SHOC fp64 Dirichlet, 1000 steps: bitwise vs the
    oracle and within the exact-solution error."""
    cfg = inputs.config("bright1d")
    kw = dict(a=1.0, s=1.0, bc="dirichlet", scheme="2shoc", precision="fp64")
    ref = run_oracle(cfg["dims"], cfg["h"], cfg["psi0"], cfg["k"], cfg["steps"], **kw)
    got = run_gpu(cfg["dims"], cfg["h"], cfg["psi0"], cfg["k"], cfg["steps"], force_dt=False, **kw)
    assert_parity(got, ref, "fp64", what="config 1")
    ex = inputs.bright_soliton(inputs.axis(1025, cfg["h"]), t=1.0)
    assert np.abs(got - ex).max() < 2e-6


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
def test_config2_dark_soliton_orders(scheme, precision):
    """configs[1]: dark soliton, MSD, t=5 on [-50, 50]: GPU orders 2 / 4 and bitwise = oracle at h = 0.1."""
    errs = []
    for h in (0.2, 0.1, 0.05):
        n = int(round(100 / h)) + 1
        x = inputs.axis(n, h)
        kb = h * h / math.sqrt(2) * (0.75 if scheme == "2shoc" else 1.0)
        nst = math.ceil(5.0 / (0.8 * kb))
        kw = dict(a=1.0, s=-1.0, bc="msd", scheme=scheme, precision=precision)
        got = run_gpu((n,), h, inputs.dark_soliton(x), 5.0 / nst, nst, force_dt=False, **kw)
        if h == 0.1:
            ref = run_oracle((n,), h, inputs.dark_soliton(x), 5.0 / nst, nst, **kw)
            assert_parity(got, ref, precision, what=f"dark soliton {scheme} {precision}")
        errs.append(np.abs(got - inputs.dark_soliton(x, t=5.0)).max())
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    want = 2.0 if scheme == "cd" else 4.0
    if precision == "fp64" or scheme == "cd":
        assert all(abs(o - want) < 0.3 for o in orders), (errs, orders)


def test_config3_trap2d_full_size():
    """configs[2]: 2D vortex in a harmonic trap, 1024^2, 2SHOC fp64 MSD: 10 steps bitwise vs the oracle."""
    cfg = inputs.config("trap2d")
    kw = dict(a=1.0, s=-1.0, V=cfg["V"], bc="msd", scheme="2shoc", precision="fp64")
    ref = run_oracle(cfg["dims"], cfg["h"], cfg["psi0"], cfg["k"], 10, **kw)
    got = run_gpu(cfg["dims"], cfg["h"], cfg["psi0"], cfg["k"], 10, force_dt=False, **kw)
    assert_parity(got, ref, "fp64", what="config 3")


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_config4_ring_full_size(precision):
    """configs[3]: 3D vortex ring 87x87x203, 2SHOC MSD: 20 steps bitwise vs the oracle."""
    cfg = inputs.config("ring3d")
    kw = dict(a=1.0, s=-1.0, bc="msd", scheme="2shoc", precision=precision)
    ref = run_oracle(cfg["dims"], cfg["h"], cfg["psi0"], cfg["k"], 20, **kw)
    got = run_gpu(cfg["dims"], cfg["h"], cfg["psi0"], cfg["k"], 20, force_dt=False, **kw)
    assert_parity(got, ref, precision, what=f"config 4 {precision}")


def test_config4_ring_3360_steps_properties():
    """The paper's benchmark run (3360 steps): finite, MSD keeps the boundary density, and the fp32 run
    tracks the fp64 run (the oracle would need ~15 min; properties that hold at any length instead)."""
    cfg = inputs.config("ring3d")
    kw = dict(a=1.0, s=-1.0, bc="msd", scheme="2shoc", force_dt=False)
    d = run_gpu(cfg["dims"], cfg["h"], cfg["psi0"], cfg["k"], 3360, precision="fp64", **kw)
    f = run_gpu(cfg["dims"], cfg["h"], cfg["psi0"], cfg["k"], 3360, precision="fp32", **kw)
    assert np.all(np.isfinite(d)) and np.all(np.isfinite(f))
    rho0 = np.abs(cfg["psi0"]) ** 2
    for sl in [(0, slice(None), slice(None)), (slice(None), 0, slice(None)), (slice(None), slice(None), -1)]:
        assert np.abs(np.abs(d[sl]) ** 2 - rho0[sl]).max() < 1e-6
    assert rel_l2(f, d) < 1e-4


def test_diagnostics_match_oracle():
    import oracle
    from paper_1203_1263_b200.nlse import Solver
    for dims, V in [((1025,), None), ((130, 77), None), ((40, 30, 20), "V")]:
        psi = case_input(dims, seed=31)
        Vv = np.abs(inputs.random_smooth(dims, seed=32)) if V else None
        for prec in ("fp64", "fp32"):
            with Solver(dims, 0.2, a=0.8, s=-1.2, V=Vv, bc="msd", precision=prec) as sv:
                sv.nlse_set_psi(psi)
                m, h = sv.nlse_diagnostics()
                p = oracle.Problem(dims, 0.2, a=0.8, s=-1.2, bc="msd", precision=prec)
                src = psi if prec == "fp64" else psi.astype(np.complex64)
                mo, ho = oracle.diagnostics(p, src, Vv)
                assert abs(m - mo) <= 1e-12 * abs(mo) and abs(h - ho) <= 1e-12 * abs(ho), (dims, prec, m, mo, h, ho)


def test_errors_and_edge_cases():
    from paper_1203_1263_b200.nlse import NLSE_ERR_ARG, NLSE_ERR_DIVERGED, NLSE_ERR_UNSTABLE, NLSEError, Solver
    dims = (31, 17)
    psi = case_input(dims, seed=3)
    with Solver(dims, 0.1, s=-1.0, bc="msd") as sv:
        sv.nlse_set_psi(psi)
        sv.nlse_step(0.001, 0)                      # no-op
        assert np.array_equal(sv.nlse_get_psi(), psi)
        with pytest.raises(NLSEError) as e:
            sv.nlse_step(0.01, 1)                   # above the 2D 2SHOC bound 0.00265
        assert e.value.status == NLSE_ERR_UNSTABLE
        with pytest.raises(NLSEError) as e:
            sv.nlse_step(-0.001, 1)
        assert e.value.status == NLSE_ERR_ARG
        with pytest.raises(NLSEError) as e:
            sv.nlse_step(float("nan"), 1)
        assert e.value.status == NLSE_ERR_ARG
    with Solver(dims, 0.1, s=-1.0, bc="dirichlet", force_dt=True) as sv:
        sv.nlse_set_psi(psi)
        with pytest.raises(NLSEError) as e:
            sv.nlse_step(0.05, 400)                 # far above the bound: blows up
        assert e.value.status == NLSE_ERR_DIVERGED
        assert "step" in str(e.value)


def test_device_io_roundtrip():
    import torch
    from paper_1203_1263_b200.nlse import Solver
    dims = (20, 10, 6)
    psi = case_input(dims, seed=4)
    for prec, dt in (("fp64", torch.complex128), ("fp32", torch.complex64)):
        with Solver(dims, 0.3, precision=prec) as sv:
            t = torch.from_numpy(psi.astype(np.complex128 if prec == "fp64" else np.complex64)).cuda()
            sv.nlse_set_psi_device(t.data_ptr())
            u = torch.empty_like(t)
            sv.nlse_get_psi_device(u.data_ptr())
            torch.cuda.synchronize()
            assert torch.equal(t, u)
            assert np.array_equal(sv.nlse_get_psi(), t.cpu().numpy().astype(np.complex128))


def test_cuda_graph_replay_matches_direct_launches(monkeypatch):
    """nlse_step with many steps replays a captured CUDA graph of 8 steps (device-side step
    counter and barrier epochs); the result and the divergence step index equal the
    direct-launch path bit for bit."""
    dims = (40, 21, 19)
    psi0 = case_input(dims, seed=61)
    k = _k(3, 0.5, "2shoc")
    a = run_gpu(dims, 0.5, psi0, k, 37, s=-1.0, bc="msd")                     # 4 graph replays + 5
    monkeypatch.setenv("NLSE_GRAPHS", "0")
    b = run_gpu(dims, 0.5, psi0, k, 37, s=-1.0, bc="msd", chunks=[5, 32])
    assert ulp_diff(a, b, "fp64") == 0
    ref = run_oracle(dims, 0.5, psi0, k, 37, s=-1.0, bc="msd")
    assert ulp_diff(a, ref, "fp64") == 0


def test_divergence_step_index_with_graphs():
    from paper_1203_1263_b200.nlse import NLSE_ERR_DIVERGED, NLSEError, Solver
    dims = (31, 17)
    psi = case_input(dims, seed=3)
    msgs = []
    for chunks in ([400], [3, 397]):
        with Solver(dims, 0.1, s=-1.0, bc="dirichlet", force_dt=True) as sv:
            sv.nlse_set_psi(psi)
            with pytest.raises(NLSEError) as e:
                for n in chunks:
                    sv.nlse_step(0.05, n)
            assert e.value.status == NLSE_ERR_DIVERGED
            msgs.append(str(e.value))
    assert msgs[0] == msgs[1], msgs


def test_divergence_flag_cleared_by_set_psi():
    """The divergence report stays until Psi is replaced: after NLSE_ERR_DIVERGED, a fresh
    nlse_set_psi + a stable k steps cleanly and matches the oracle."""
    from paper_1203_1263_b200.nlse import NLSE_ERR_DIVERGED, NLSEError, Solver
    dims = (31, 17)
    psi = case_input(dims, seed=3)
    k = _k(2, 0.1, "2shoc")
    with Solver(dims, 0.1, s=-1.0, bc="dirichlet", force_dt=True) as sv:
        sv.nlse_set_psi(psi)
        with pytest.raises(NLSEError) as e:
            sv.nlse_step(0.05, 400)
        assert e.value.status == NLSE_ERR_DIVERGED
        with pytest.raises(NLSEError):          # still non-finite: reported again
            sv.nlse_step(k, 1)
        sv.nlse_set_psi(psi)
        sv.nlse_step(k, 5)
        got = sv.nlse_get_psi()
    ref = run_oracle(dims, 0.1, psi, k, 5, s=-1.0, bc="dirichlet")
    assert ulp_diff(got, ref, "fp64") == 0


def test_config5_gpe3d_full_size_sampled():
    """configs[4] at full size (1024^3 fp64 + V, 2SHOC, MSD) in the launch configuration bench.py
    times, the stated 10 RK4 steps: sampled outputs vs the oracle, bit for bit, and
    the diagnostics of the whole field vs the oracle's Kahan sums (<= 1e-12 relative, §8(c)).
    A point's value after n steps depends only on Psi within 4 stages x 2 points x n of it, so the
    oracle runs on a sub-block around each sample (sub-blocks that touch the domain boundary keep
    the true boundary) and is compared on the part at least 8n points from its artificial edges."""
    import oracle
    from paper_1203_1263_b200.nlse import Solver
    n, nsteps = 1024, 10
    m = 8 * nsteps
    cfg = inputs.config("gpe3d")
    psi, V = inputs.gpe3d_fill(n)
    half = 6
    # (z, y, x) sample centres: interior, the corner, an x face, the top z face, a y edge
    centres = [(511, 300, 700), (0, 0, 0), (600, 400, 0), (1023, 512, 511), (200, 1023, 900)]
    subs = []
    for cz, cy, cx in centres:
        lo = [max(0, c - half - m) for c in (cz, cy, cx)]
        hi = [min(n, c + half + m + 1) for c in (cz, cy, cx)]
        sl = tuple(slice(a, b) for a, b in zip(lo, hi))
        subs.append((lo, hi, sl, np.ascontiguousarray(psi[sl]), np.ascontiguousarray(V[sl])))
    with Solver(cfg["dims"], cfg["h"], a=1.0, s=-1.0, V=V, bc="msd", scheme="2shoc", precision="fp64") as sv:
        assert sv.nlse_get_info()["variant"] == "stage3d_tma"
        sv.nlse_set_psi(psi)
        del psi
        sv.nlse_step(cfg["k"], nsteps)
        mass, ham = sv.nlse_diagnostics()
        got = sv.nlse_get_psi()
    p_or = lambda d: oracle.Problem(d, cfg["h"], a=1.0, s=-1.0, bc="msd", scheme="2shoc")
    for lo, hi, sl, sub, Vs in subs:
        ref = oracle.step(p_or(tuple(reversed(sub.shape))), sub, cfg["k"], nsteps, Vs)
        # compare where the sub-block edge is a true domain boundary or at least m away
        keep = []
        for ax in range(3):
            a0 = 0 if lo[ax] == 0 else m
            a1 = sub.shape[ax] if hi[ax] == n else sub.shape[ax] - m
            keep.append(slice(a0, a1))
        keep = tuple(keep)
        g = np.ascontiguousarray(got[sl][keep])
        r = np.ascontiguousarray(ref[keep].astype(np.complex128))
        assert g.size > 0
        assert np.array_equal(g.view(np.uint64), r.view(np.uint64)), (lo, rel_l2(g, r))
    mo, ho = oracle.diagnostics(p_or(cfg["dims"]), got, V)
    assert abs(mass - mo) <= 1e-12 * abs(mo) and abs(ham - ho) <= 1e-12 * abs(ho), (mass, mo, ham, ho)


@pytest.mark.parametrize("ndim,precision,chunk", [(3, "fp64", 20), (3, "fp32", 3), (1, "fp64", 7), (2, "fp64", 5)])
def test_run_frames_equal_step_then_get(ndim, precision, chunk):
    """nlse_run_frames (the paper's frames model, downloads overlapped with compute) returns
    exactly what nlse_step(k, chunk) + nlse_get_psi give, frame by frame."""
    from paper_1203_1263_b200.nlse import Solver
    dims = {1: (301,), 2: (70, 41), 3: (40, 26, 22)}[ndim]
    h = {1: 0.1, 2: 0.2, 3: 0.5}[ndim]
    psi0 = case_input(dims, seed=81)
    k = _k(ndim, h, "2shoc")
    kw = dict(s=-1.0, bc="msd", scheme="2shoc", precision=precision, force_dt=True)
    with Solver(dims, h, **kw) as sv:
        sv.nlse_set_psi(psi0)
        frames = sv.nlse_run_frames(k, chunk, 3)
    with Solver(dims, h, **kw) as sv:
        sv.nlse_set_psi(psi0)
        for f in range(3):
            sv.nlse_step(k, chunk)
            assert np.array_equal(frames[f].view(np.uint64), sv.nlse_get_psi().view(np.uint64)), f
