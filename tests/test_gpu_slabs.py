"""Slab mode on one GPU with virtual ranks: the grid split into
P z slabs, each its own context with ghost planes, remote stores into the
neighbours' ghosts from the stage kernels and device-side neighbour barriers between
stages (the same code path as one process per GPU, with peer pointers that happen to
live on the same device).  The bar: bitwise identical to the single-context run, which
is itself bitwise identical to the oracle (test_gpu_parity.py)."""
import math

import numpy as np
import pytest

from helpers import case_input, run_gpu, run_gpu_slabs, run_oracle, ulp_diff
from paper_1203_1263_b200 import inputs

pytestmark = pytest.mark.gpu


def _k(h, scheme):
    return 0.5 * h * h / (3 * math.sqrt(2)) * (0.75 if scheme == "2shoc" else 1.0)


@pytest.mark.parametrize("nranks", [2, 3, 5])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("bc", ["dirichlet", "msd", "l0"])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
def test_slabs_bitwise_equal_single(scheme, bc, precision, nranks):
    dims = (70, 37, 29)
    psi0 = case_input(dims, seed=41)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=42))
    kw = dict(a=0.9, s=-1.1, V=V, bc=bc, scheme=scheme, precision=precision)
    k = _k(0.5, scheme)
    one = run_gpu(dims, 0.5, psi0, k, 9, **kw)
    many = run_gpu_slabs(dims, 0.5, psi0, k, 9, nranks, **kw)
    assert ulp_diff(many, one, precision) == 0


@pytest.mark.parametrize("kernel", ["v1", "generic", "msd_recompute", "xfuse_on", "edge_lean", "edge_pp"])
def test_slabs_other_kernel_families(kernel, monkeypatch):
    dims = (40, 35, 24)          # (nx-1) % 32 != 0 and (ny-1) % 16 != 0: xfuse can apply
    psi0 = case_input(dims, seed=43)
    if kernel == "v1":
        monkeypatch.setenv("NLSE_3D_KERNEL", "v1")
    if kernel == "msd_recompute":        # boundary kernel recomputes F(b') (no light pass)
        monkeypatch.setenv("NLSE_MSD_FB", "0")
    if kernel == "xfuse_on":
        monkeypatch.setenv("NLSE_XFUSE", "1")
    if kernel.startswith("edge"):
        monkeypatch.setenv("NLSE_FORCE_EDGE", "1" if kernel == "edge_lean" else "2")
    kw = dict(s=-1.0, bc="msd", scheme="2shoc", generic=kernel == "generic")
    k = _k(0.5, "2shoc")
    one = run_gpu(dims, 0.5, psi0, k, 7, **kw)
    many = run_gpu_slabs(dims, 0.5, psi0, k, 7, 4, **kw)
    assert ulp_diff(many, one, "fp64") == 0


def test_slabs_match_oracle_and_chunking():
    dims = (33, 30, 26)
    psi0 = case_input(dims, seed=44)
    kw = dict(s=-1.0, bc="msd", scheme="2shoc")
    k = _k(0.5, "2shoc")
    ref = run_oracle(dims, 0.5, psi0, k, 10, **kw)
    a = run_gpu_slabs(dims, 0.5, psi0, k, 10, 3, **kw)
    b = run_gpu_slabs(dims, 0.5, psi0, k, 10, 3, chunks=[3, 1, 6], **kw)
    assert ulp_diff(a, ref, "fp64") == 0
    assert ulp_diff(b, ref, "fp64") == 0


def test_slabs_thinnest_legal():
    """Slabs of exactly 2w planes (the minimum), and uneven splits."""
    for dims, P, scheme in [((20, 18, 8), 2, "2shoc"), ((20, 18, 13), 3, "2shoc"), ((20, 18, 6), 3, "cd")]:
        psi0 = case_input(dims, seed=45)
        kw = dict(s=-1.0, bc="msd", scheme=scheme)
        k = _k(0.5, scheme)
        one = run_gpu(dims, 0.5, psi0, k, 5, **kw)
        many = run_gpu_slabs(dims, 0.5, psi0, k, 5, P, **kw)
        assert ulp_diff(many, one, "fp64") == 0, (dims, P, scheme)


def test_slab_diagnostics_are_global():
    import oracle
    dims = (36, 28, 31)
    psi0 = case_input(dims, seed=46)
    V = np.abs(inputs.random_smooth(dims, seed=47))
    out, (m, h) = run_gpu_slabs(dims, 0.25, psi0, 0.001, 3, 4, s=-1.0, V=V, bc="msd", diag=True)
    p = oracle.Problem(dims, 0.25, a=1.0, s=-1.0, bc="msd")
    mo, ho = oracle.diagnostics(p, out, V)
    assert len(set(m)) == 1 and len(set(h)) == 1        # every rank holds the same global sums
    assert abs(m[0] - mo) <= 1e-12 * abs(mo) and abs(h[0] - ho) <= 1e-12 * abs(ho)


def test_slab_errors():
    from paper_1203_1263_b200.nlse import NLSE_ERR_ARG, NLSE_ERR_COMM, NLSEError, Solver
    with pytest.raises(NLSEError) as e:
        Solver((20, 20, 7), 0.5, scheme="2shoc", dist=(1, 2))       # 4 + 3 planes: 3 < 2w
    assert e.value.status == NLSE_ERR_ARG
    with pytest.raises(NLSEError) as e:
        Solver((7,), 0.5, scheme="2shoc", dist=(1, 2))              # 1D: 4 + 3 points: 3 < 2w
    assert e.value.status == NLSE_ERR_ARG
    with pytest.raises(NLSEError) as e:
        Solver((20, 7), 0.5, scheme="2shoc", dist=(1, 2))           # 2D: 4 + 3 rows: 3 < 2w
    assert e.value.status == NLSE_ERR_ARG
    sv = Solver((20, 20, 16), 0.5, dist=(1, 2))
    with pytest.raises(NLSEError) as e:
        sv.nlse_step(0.001, 1)                                       # not connected yet
    assert e.value.status == NLSE_ERR_COMM
    sv.close()


def test_virtual_group_requires_group_calls():
    from paper_1203_1263_b200 import nlse
    svs = [nlse.Solver((16, 16, 12), 0.5, s=-1.0, bc="msd", dist=(r, 2)) for r in range(2)]
    try:
        nlse.nlse_dist_connect_local(svs)
        with pytest.raises(nlse.NLSEError) as e:
            svs[0].nlse_step(0.001, 1)
        assert e.value.status == nlse.NLSE_ERR_ARG
        with pytest.raises(nlse.NLSEError):
            svs[1].nlse_diagnostics()
    finally:
        for sv in svs:
            sv.close()


# ---------------------------------------------------------------------------------------------
# 2D y-row slabs (§8(f) rank 4): rows are the slowest axis of a 2D grid, so a slab is a
# contiguous block of rows with w ghost rows on each side, exactly as 3D z planes
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("nranks", [2, 3, 5])
@pytest.mark.parametrize("withV", [False, True], ids=["V0", "V"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("bc", ["dirichlet", "msd", "l0"])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
@pytest.mark.parametrize("kernel", ["strip", "tile"])
def test_2d_slabs_bitwise_equal_single(scheme, bc, precision, withV, nranks, kernel, monkeypatch):
    if kernel == "tile":
        monkeypatch.setenv("NLSE_2D_KERNEL", "tile")
    dims = (133, 70)             # tiles of 32 x 16 with ragged tails; slabs cut tiles anywhere
    h = 0.2
    psi0 = case_input(dims, seed=51)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=52)) if withV else None
    kw = dict(a=0.9, s=-1.1, V=V, bc=bc, scheme=scheme, precision=precision)
    k = 0.5 * h * h / (2 * math.sqrt(2)) * (0.75 if scheme == "2shoc" else 1.0)
    one = run_gpu(dims, h, psi0, k, 9, **kw)
    many = run_gpu_slabs(dims, h, psi0, k, 9, nranks, **kw)
    assert ulp_diff(many, one, precision) == 0


@pytest.mark.parametrize("kernel", ["strip", "strip_rows3", "tile", "generic"])
def test_2d_slabs_match_oracle_chunks_thin_and_diagnostics(kernel, monkeypatch):
    """2D slabs against the oracle (chunked calls, CUDA graphs not used by virtual groups),
    slabs of exactly 2w rows and uneven splits, the warp-strip kernel (also with 3-row chunks),
    the shared-tile kernel, the generic kernels, global diagnostics."""
    import oracle
    generic = kernel == "generic"
    if kernel == "tile":
        monkeypatch.setenv("NLSE_2D_KERNEL", "tile")
    if kernel == "strip_rows3":
        monkeypatch.setenv("NLSE_STRIP_ROWS", "3")
    h = 0.25
    for dims, P, scheme in [((64, 48), 3, "2shoc"), ((40, 8), 2, "2shoc"), ((40, 13), 3, "2shoc"), ((37, 6), 3, "cd")]:
        psi0 = case_input(dims, seed=53)
        V = np.abs(inputs.random_smooth(dims, seed=54))
        kw = dict(s=-1.0, V=V, bc="msd", scheme=scheme, generic=generic)
        k = 0.5 * h * h / (2 * math.sqrt(2)) * (0.75 if scheme == "2shoc" else 1.0)
        ref = run_oracle(dims, h, psi0, k, 10, s=-1.0, V=V, bc="msd", scheme=scheme)
        out, (m, e) = run_gpu_slabs(dims, h, psi0, k, 10, P, chunks=[3, 1, 6], diag=True, **kw)
        assert ulp_diff(out, ref, "fp64") == 0, (dims, P)
        mo, eo = oracle.diagnostics(oracle.Problem(dims, h, a=1.0, s=-1.0, bc="msd"), out, V)
        assert len(set(m)) == 1 and abs(m[0] - mo) <= 1e-12 * abs(mo) and abs(e[0] - eo) <= 1e-12 * abs(eo)


# ---------------------------------------------------------------------------------------------
# 1D x slabs (§8(f) rank 4, "large-1D split"): the slab axis is x; w ghost points on each side
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("nranks", [2, 3, 5])
@pytest.mark.parametrize("withV", [False, True], ids=["V0", "V"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("bc", ["dirichlet", "msd", "l0"])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
@pytest.mark.parametrize("generic", [False, True], ids=["tile", "generic"])
def test_1d_slabs_bitwise_equal_single(scheme, bc, precision, withV, nranks, generic):
    dims, h = (4099,), 0.05          # slabs cut the 1024-point tiles anywhere
    psi0 = case_input(dims, seed=55)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=56)) if withV else None
    kw = dict(a=0.9, s=-1.1, V=V, bc=bc, scheme=scheme, precision=precision, generic=generic)
    k = 0.5 * h * h / math.sqrt(2) * (0.75 if scheme == "2shoc" else 1.0)
    one = run_gpu(dims, h, psi0, k, 9, **kw)
    many = run_gpu_slabs(dims, h, psi0, k, 9, nranks, **kw)
    assert ulp_diff(many, one, precision) == 0


def test_1d_slabs_oracle_thin_and_diagnostics():
    import oracle
    h = 0.1
    for n, P, scheme in [(1001, 4, "2shoc"), (8, 2, "2shoc"), (13, 3, "2shoc"), (6, 3, "cd")]:
        dims = (n,)
        psi0 = case_input(dims, seed=57)
        V = np.abs(inputs.random_smooth(dims, seed=58))
        k = 0.5 * h * h / math.sqrt(2) * (0.75 if scheme == "2shoc" else 1.0)
        ref = run_oracle(dims, h, psi0, k, 10, s=-1.0, V=V, bc="msd", scheme=scheme)
        out, (m, e) = run_gpu_slabs(dims, h, psi0, k, 10, P, s=-1.0, V=V, bc="msd", scheme=scheme, chunks=[3, 7],
                                    diag=True)
        assert ulp_diff(out, ref, "fp64") == 0, (n, P)
        mo, eo = oracle.diagnostics(oracle.Problem(dims, h, a=1.0, s=-1.0, bc="msd"), out, V)
        assert len(set(m)) == 1 and abs(m[0] - mo) <= 1e-12 * abs(mo) and abs(e[0] - eo) <= 1e-12 * abs(eo)
