"""GPU parity of the temporally blocked path (csrc/fused3d.cuh): two RK4
stages per HBM pass (S1+S2, S3+S4) for the 3D CD scheme, selected with NLSE_FUSED=1 at context
creation.  Bar: bit-identical to the oracle's four separate stages ((RK4) P:164-180)."""
import math

import numpy as np
import pytest

from helpers import assert_parity, case_input, guard_field, run_gpu, run_oracle
from paper_1203_1263_b200 import inputs

pytestmark = pytest.mark.gpu


def _k(h):
    return 0.5 * h * h / (3 * math.sqrt(2))


@pytest.fixture
def fused(monkeypatch):
    monkeypatch.setenv("NLSE_FUSED", "1")


@pytest.mark.parametrize("ty", ["16", "8"])
@pytest.mark.parametrize("withV", [False, True], ids=["V0", "V"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("bc", ["dirichlet", "msd", "l0"])
@pytest.mark.parametrize("dims", [(70, 37, 29), (33, 17, 9), (64, 32, 6), (97, 49, 40), (5, 5, 5), (3, 4, 3)])
def test_fused_matrix_bitwise(dims, bc, precision, withV, ty, fused, monkeypatch):
    """Ragged grids, faces one past / on a tile edge, z chunks of every length, the smallest
    grids; odd step counts (the Psi buffers end swapped)."""
    monkeypatch.setenv("NLSE_FUSED_TY", ty)
    if bc == "msd" and min(dims[:2]) < 5:
        pytest.skip("MSD fused mode needs the stored-F(b') boundary pass (nx, ny >= 5)")
    h = 0.5
    psi0 = case_input(dims, seed=41)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=42)) if withV else None
    kw = dict(a=0.9, s=-1.1, V=V, bc=bc, scheme="cd", precision=precision)
    ref = run_oracle(dims, h, psi0, _k(h), 5, **kw)
    got, info = run_gpu(dims, h, psi0, _k(h), 5, with_info=True, **kw)
    assert info["variant"] == "fused3d_cd", info
    assert_parity(got, ref, precision, what=f"fused {dims} {bc} {precision} V={withV} TY={ty}")


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_fused_chunks_graphs_and_diagnostics(precision, fused):
    """Chunked calls mixing CUDA-graph replays (8 steps, even) and direct steps (each swaps the
    Psi buffers): bitwise equal to one call and to the oracle; diagnostics read the current Psi."""
    import oracle
    from paper_1203_1263_b200.nlse import Solver
    dims, h = (48, 40, 36), 0.5
    psi0 = case_input(dims, seed=43)
    V = 0.2 * np.abs(inputs.random_smooth(dims, seed=44))
    kw = dict(a=1.0, s=-1.0, V=V, bc="msd", scheme="cd", precision=precision)
    ref = run_oracle(dims, h, psi0, _k(h), 37, **kw)
    a = run_gpu(dims, h, psi0, _k(h), 37, **kw)
    b = run_gpu(dims, h, psi0, _k(h), 37, chunks=[3, 16, 1, 17], **kw)
    assert_parity(a, ref, precision, what="one call")
    assert_parity(b, ref, precision, what="chunks")
    with Solver(dims, h, force_dt=True, **kw) as sv:
        sv.nlse_set_psi(psi0)
        sv.nlse_step(_k(h), 3)
        m, e = sv.nlse_diagnostics()
        got = sv.nlse_get_psi()
    p = oracle.Problem(dims, h, a=1.0, s=-1.0, bc="msd", scheme="cd", precision=precision)
    mo, eo = oracle.diagnostics(p, got if precision == "fp64" else got.astype(np.complex64), V)
    assert abs(m - mo) <= 1e-12 * abs(mo) and abs(e - eo) <= 1e-12 * abs(eo)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_fused_msd_eps_guard(precision, fused):
    """R-MSD-GUARD in the fused kernel's stage-A face values (Psi_b' = 0 / eps/2)."""
    dims, h = (70, 37, 29), 0.5
    psi0 = guard_field(dims, precision, above=False)
    kw = dict(a=0.9, s=-1.1, bc="msd", scheme="cd", precision=precision)
    ref = run_oracle(dims, h, psi0, _k(h), 3, **kw)
    got = run_gpu(dims, h, psi0, _k(h), 3, **kw)
    assert_parity(got, ref, precision, what="fused guard")


def test_fused_full_size_sampled(fused):
    """1024^3 fp64 CD + V, MSD, in the bench launch configuration, 4 steps: sampled outputs
    against the oracle on sub-blocks (a CD stage reaches 1 point, so 4 steps reach 16)."""
    import oracle
    from paper_1203_1263_b200.nlse import Solver
    n, nsteps = 1024, 4
    m = 4 * nsteps
    cfg = inputs.config("gpe3d")
    psi, V = inputs.gpe3d_fill(n)
    half = 8
    subs = []
    for cz, cy, cx in [(511, 300, 700), (0, 0, 0), (1023, 512, 511), (200, 1023, 900)]:
        lo = [max(0, c - half - m) for c in (cz, cy, cx)]
        hi = [min(n, c + half + m + 1) for c in (cz, cy, cx)]
        sl = tuple(slice(a, b) for a, b in zip(lo, hi))
        subs.append((lo, hi, sl, np.ascontiguousarray(psi[sl]), np.ascontiguousarray(V[sl])))
    with Solver(cfg["dims"], cfg["h"], a=1.0, s=-1.0, V=V, bc="msd", scheme="cd", precision="fp64") as sv:
        assert sv.nlse_get_info()["variant"] == "fused3d_cd"
        sv.nlse_set_psi(psi)
        del psi
        sv.nlse_step(cfg["k"], nsteps)
        got = sv.nlse_get_psi()
    for lo, hi, sl, sub, Vs in subs:
        p = oracle.Problem(tuple(reversed(sub.shape)), cfg["h"], a=1.0, s=-1.0, bc="msd", scheme="cd")
        ref = oracle.step(p, sub, cfg["k"], nsteps, Vs)
        keep = tuple(slice(0 if lo[ax] == 0 else m, sub.shape[ax] if hi[ax] == n else sub.shape[ax] - m)
                     for ax in range(3))
        g = np.ascontiguousarray(got[sl][keep])
        r = np.ascontiguousarray(ref[keep].astype(np.complex128))
        assert np.array_equal(g.view(np.uint64), r.view(np.uint64)), lo
