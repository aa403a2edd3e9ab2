"""Pins for the CPU oracle: each test checks the oracle against something other
than itself -- closed forms, identities, special cases reducing to textbook
routines, exact solutions, measured convergence orders, brute force.
(no GPU; `-m "not gpu"`)."""
import math
import os

import numpy as np
import pytest

import oracle
from oracle import Problem
from paper_1203_1263_b200 import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def interior(ndim, margin=1):
    s = slice(margin, -margin)
    return (s,) * ndim


def case_field(dims, seed):
    """Seeded smooth complex field with a background of modulus ~1."""
    return inputs.random_smooth(tuple(dims), seed=seed, modes=5, amp=0.4, offset=1.0)


# ---------------------------------------------------------------------------------------------
# Stencils (2SHOC step 1 / CD, 2SHOC step 2) -- closed forms
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_cd_exact_on_quadratics(oracle_lib, ndim):
    """CD is exact on quadratics: D(x^2 + y^2 + z^2) = 2*ndim at interior points.
    h = 0.5 and x = i*h make every value exactly representable, so the result is exact."""
    dims = (9, 8, 7)[:ndim]
    h = 0.5
    coords = list(reversed(np.meshgrid(*[np.arange(n) * h for n in reversed(dims)], indexing="ij")))
    psi = sum(c * c for c in coords) + 0j
    D, L = oracle.laplacian(Problem(dims, h, scheme="cd"), psi)
    assert np.all(D[interior(ndim)] == 2.0 * ndim)
    assert np.all(L[interior(ndim)] == 2.0 * ndim)


def test_2shoc_exact_on_quartic(oracle_lib):
    """1D 2SHOC on x^4 gives exactly 12 x^2 at points two cells from the edge."""
    h = 0.5
    x = np.arange(21) * h
    D, L = oracle.laplacian(Problem((21,), h, scheme="2shoc"), x ** 4 + 0j)
    np.testing.assert_allclose(L.real[2:-2], 12 * x[2:-2] ** 2, rtol=1e-13, atol=0)


def _plane_wave(dims, h, kvec):
    coords = inputs.mesh(dims, h)
    return np.cos(sum(k * c for k, c in zip(kvec, coords))) + 0j


@pytest.mark.parametrize("ndim", [1, 2, 3])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
def test_stencil_symbol_on_plane_waves(oracle_lib, ndim, scheme):
    """A plane wave cos(k.x) is an eigenfunction: CD symbol sum_a 2(cos k_a h - 1)/h^2
     and 2SHOC symbol sum_a 2(cos k_a h - 1)/h^2 * (7/6 - cos(k_a h)/6) (the
    2D/3D cross terms must cancel the mixed derivatives for this to hold)."""
    dims = (24, 20, 18)[:ndim]
    h = 0.1
    kvec = (1.3, -0.7, 2.1)[:ndim]
    psi = _plane_wave(dims, h, kvec)
    D, L = oracle.laplacian(Problem(dims, h, scheme=scheme), psi)
    sym = 0.0
    for k in kvec:
        cd = 2.0 * (math.cos(k * h) - 1.0) / h ** 2
        sym += cd if scheme == "cd" else cd * (7.0 / 6.0 - math.cos(k * h) / 6.0)
    m = 1 if scheme == "cd" else 2   # 2SHOC's first interior layer uses boundary D (BC form)
    got = L.real[interior(ndim, m)]
    want = sym * psi.real[interior(ndim, m)]
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-11 * abs(sym) + 1e-11)


def _wide_star(psi, h, ndim):
    """Standard wide fourth-order star stencil, sum over axes of (-1/12, 4/3, -5/2, 4/3, -1/12)/h^2."""
    out = np.zeros_like(psi)
    for ax in range(ndim):
        a = psi.ndim - 1 - ax   # x is the last numpy axis
        out += (-np.roll(psi, 2, a) + 16 * np.roll(psi, 1, a) - 30 * psi + 16 * np.roll(psi, -1, a)
                - np.roll(psi, -2, a)) / (12 * h * h)
    return out


@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_2shoc_interior_equals_wide_stencil(oracle_lib, ndim):
    """In exact arithmetic, 2SHOC equals the wide 4th-order star stencil at points >= 2 from the
    boundary. A wrong cross-term weight or sign breaks this on random fields."""
    dims = (17, 15, 13)[:ndim]
    h = 0.3
    psi = inputs.random_smooth(dims, seed=7, modes=6)
    D, L = oracle.laplacian(Problem(dims, h, scheme="2shoc"), psi)
    W = _wide_star(psi, h, ndim)
    sl = interior(ndim, 2)
    scale = np.abs(psi).max() / h ** 2
    np.testing.assert_allclose(L[sl], W[sl], rtol=0, atol=64 * np.finfo(float).eps * scale)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("ndim", [1, 2, 3])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
def test_constant_field(oracle_lib, precision, ndim, scheme):
    """Difference-form stencils annihilate constants exactly: D = L = 0 at every interior point,
    and F = i(s|Y|^2 - V)Y there."""
    dims = (7, 6, 5)[:ndim]
    c0 = 0.6 - 0.3j
    psi = np.full(tuple(reversed(dims)), c0)
    V = np.full(psi.shape, 0.25)
    p = Problem(dims, 0.37, a=1.3, s=-0.8, bc="msd", scheme=scheme, precision=precision)
    D, L = oracle.laplacian(p, psi, V)
    assert np.all(D[interior(ndim)] == 0) and np.all(L[interior(ndim)] == 0)
    F = oracle.rhs(p, psi, V)
    cc = complex(np.complex64(c0)) if precision == "fp32" else c0
    want = 1j * (p.s * abs(cc) ** 2 - 0.25) * cc
    tol = 1e-6 if precision == "fp32" else 1e-15
    np.testing.assert_allclose(F, np.full(psi.shape, want), rtol=0, atol=tol)


# ---------------------------------------------------------------------------------------------
# Boundary conditions
# ---------------------------------------------------------------------------------------------

def _face_mask(dims):
    """Boundary points with exactly one boundary axis, and their inward-normal offsets."""
    shape = tuple(reversed(dims))
    idx = np.indices(shape)
    nb = np.zeros(shape, int)
    for a, n in enumerate(shape):
        nb += (idx[a] == 0) | (idx[a] == n - 1)
    return nb == 1


def _inward(arr, dims):
    """Value at the inward neighbour of every point (one step in along each boundary axis)."""
    shape = tuple(reversed(dims))
    idx = list(np.indices(shape))
    for a, n in enumerate(shape):
        idx[a] = np.where(idx[a] == 0, 1, np.where(idx[a] == n - 1, n - 2, idx[a]))
    return arr[tuple(idx)]


def _complex_plane_wave(dims, h, kvec, amp):
    coords = inputs.mesh(dims, h)
    return amp * np.exp(1j * sum(k * c for k, c in zip(kvec, coords)))


@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_msd_exact_for_complex_plane_waves(oracle_lib, ndim, scheme):
    """A complex plane wave A exp(i k.x) has |Psi| = A at every point, the state the MSD condition
    ((msd) P:331-335) is built to preserve: with a constant V every boundary point -- faces, edges
    and corners, b' the diagonal inward neighbour -- must evolve like the interior, so the whole
    right-hand side is F = i (a mu + s A^2 - V0) Psi with mu the scheme's plane-wave symbol (CD:
    sum_a 2(cos k_a h - 1)/h^2; 2SHOC: times (7/6 - cos(k_a h)/6)).  Closed form,
    independent of how the oracle writes (msd) / (BCMSDlap): a wrong real/imaginary part, sign,
    neighbour or a dropped N term breaks it at the boundary."""
    dims = (11, 9, 8)[:ndim]
    h = 0.3
    kvec = (0.7, -1.1, 0.4)[:ndim]
    amp, a, s, v0 = 1.3, 0.8, -1.2, 0.37
    psi = _complex_plane_wave(dims, h, kvec, amp)
    V = np.full(psi.shape, v0)
    mu = 0.0
    for k in kvec:
        cd = 2.0 * (math.cos(k * h) - 1.0) / h ** 2
        mu += cd if scheme == "cd" else cd * (7.0 / 6.0 - math.cos(k * h) / 6.0)
    F = oracle.rhs(Problem(dims, h, a=a, s=s, bc="msd", scheme=scheme), psi, V)
    want = 1j * (a * mu + s * amp ** 2 - v0) * psi
    np.testing.assert_allclose(F, want, rtol=0, atol=1e-11 * np.abs(want).max())


@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_msd_face_laplacian_on_plane_wave_with_varying_v(oracle_lib, ndim):
    """(BCMSDlap) P:336-344 on a complex plane wave with a non-constant V: D_b' / Psi_b' is the CD
    symbol lambda = sum_a 2(cos k_a h - 1)/h^2 at every interior b', so the face value must be
    D_b = [lambda + (N_b' - N_b)/a] Psi_b with N = s|Psi|^2 - V = s A^2 - V (closed form; pins the
    sign and the 1/a of the potential term, which a constant V cannot see)."""
    dims = (11, 9, 8)[:ndim]
    h = 0.3
    kvec = (0.7, -1.1, 0.4)[:ndim]
    amp, a, s = 1.3, 0.8, -1.2
    psi = _complex_plane_wave(dims, h, kvec, amp)
    V = 0.3 + 0.2 * np.abs(inputs.random_smooth(dims, seed=41))
    lam = sum(2.0 * (math.cos(k * h) - 1.0) / h ** 2 for k in kvec)
    D, _ = oracle.laplacian(Problem(dims, h, a=a, s=s, bc="msd", scheme="2shoc"), psi, V)
    f = _face_mask(dims)
    N = s * amp ** 2 - V
    want = (lam + (_inward(N, dims) - N) / a) * psi
    np.testing.assert_allclose(D[f], want[f], rtol=0, atol=1e-11 * np.abs(want[f]).max())


@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_dirichlet_laplacian_form_is_consistent(oracle_lib, ndim):
    """(BCDlap) P:320-323 substituted into F = i[a Lap + N]Psi gives dPsi_b/dt = 0 (BCDdt), to a few ulp."""
    dims = (9, 8, 7)[:ndim]
    psi = inputs.random_smooth(dims, seed=3, offset=1.0)
    V = np.abs(inputs.random_smooth(dims, seed=4))
    p = Problem(dims, 0.2, a=0.7, s=-1.4, bc="dirichlet", scheme="2shoc")
    D, _ = oracle.laplacian(p, psi, V)
    f = _face_mask(dims)
    N = p.s * np.abs(psi) ** 2 - V
    resid = 1j * (p.a * D + N * psi)
    assert np.all(np.isfinite(D[f]))
    assert np.abs(resid[f]).max() <= 8 * np.finfo(float).eps * np.abs(N * psi)[f].max()
    assert np.all(oracle.rhs(p, psi, V)[f] == 0)


@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_msd_laplacian_form_matches_time_derivative_form(oracle_lib, ndim):
    """(BCMSDlap) P:336-344 is the Laplacian form of (msd) P:331-335: with D_b from it,
    a D_b + N_b Psi_b == (a Re(D_b'/Psi_b') + N_b') Psi_b (the b' growth rate carried to b)."""
    dims = (9, 8, 7)[:ndim]
    psi = inputs.random_smooth(dims, seed=5, offset=1.5)
    V = np.abs(inputs.random_smooth(dims, seed=6))
    p = Problem(dims, 0.2, a=0.7, s=-1.4, bc="msd", scheme="2shoc")
    D, _ = oracle.laplacian(p, psi, V)
    f = _face_mask(dims)
    N = p.s * np.abs(psi) ** 2 - V
    Di, Yi, Ni = _inward(D, dims), _inward(psi, dims), _inward(N, dims)
    lhs = p.a * D + N * psi
    rhs_ = (p.a * (Di / Yi).real + Ni) * psi
    np.testing.assert_allclose(lhs[f], rhs_[f], rtol=0, atol=32 * np.finfo(float).eps * np.abs(rhs_[f]).max())


@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_msd_time_derivative_form(oracle_lib, ndim):
    """(msd) P:331-335: F_b = i Im[F_b'/Psi_b'] Psi_b with b' the (diagonal) inward neighbour, so
    d|Psi_b|^2/dt = 2 Re(conj(Psi_b) F_b) = 0 exactly in exact arithmetic."""
    dims = (9, 8, 7)[:ndim]
    psi = inputs.random_smooth(dims, seed=8, offset=1.5)
    p = Problem(dims, 0.25, a=1.0, s=-1.0, bc="msd", scheme="cd")
    F = oracle.rhs(p, psi)
    shape = psi.shape
    idx = np.indices(shape)
    bnd = np.zeros(shape, bool)
    for a, n in enumerate(shape):
        bnd |= (idx[a] == 0) | (idx[a] == n - 1)
    want = 1j * (_inward(F, dims) / _inward(psi, dims)).imag * psi
    np.testing.assert_allclose(F[bnd], want[bnd], rtol=0, atol=1e-14 * np.abs(want).max())
    assert np.abs((np.conj(psi) * F).real[bnd]).max() < 1e-13 * np.abs(F).max()


# ---------------------------------------------------------------------------------------------
# RK4 -- special cases that reduce to textbook results
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_rk4_taylor_uniform_linear(oracle_lib, ndim):
    """s = 0, uniform V0, uniform Psi0, MSD: one step = Psi0 * sum_{j<=4} (-i V0 k)^j / j!."""
    dims = (6, 5, 5)[:ndim]
    V0, k, c0 = 2.0, 0.05, 0.8 + 0.1j
    psi = np.full(tuple(reversed(dims)), c0)
    V = np.full(psi.shape, V0)
    p = Problem(dims, 0.4, a=1.0, s=0.0, bc="msd", scheme="2shoc")
    out = oracle.step(p, psi, k, 1, V)
    z = -1j * V0 * k
    want = c0 * (1 + z + z ** 2 / 2 + z ** 3 / 6 + z ** 4 / 24)
    np.testing.assert_allclose(out, np.full(psi.shape, want), rtol=2e-16 * 8, atol=0)
    assert abs(want / c0 - np.exp(z)) <= abs(z) ** 5 / 120 * 1.01


def test_rk4_uniform_nonlinear_reduces_to_scalar_ode(oracle_lib):
    """Uniform Psi with s != 0 under MSD stays uniform and follows the scalar RK4 of
    z' = i(s|z|^2 - V0) z (the textbook RK4 on one complex ODE)."""
    dims = (5, 6, 4)
    s, V0, k, n = -1.3, 0.4, 0.02, 25
    z = 0.9 - 0.2j
    psi = np.full(tuple(reversed(dims)), z)
    p = Problem(dims, 0.5, a=1.0, s=s, bc="msd", scheme="2shoc")
    out = oracle.step(p, psi, k, n, np.full(psi.shape, V0))

    def f(w):
        return 1j * (s * abs(w) ** 2 - V0) * w
    for _ in range(n):
        k1 = f(z); k2 = f(z + k / 2 * k1); k3 = f(z + k / 2 * k2); k4 = f(z + k * k3)
        z = z + k / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
    assert np.ptp(out.real) == 0 and np.ptp(out.imag) == 0
    assert abs(out.flat[0] - z) < 1e-14


def _assemble_linear(p, dims, V):
    """Matrix of the (linear, s = 0) F restricted to the interior, column by column."""
    shape = tuple(reversed(dims))
    n = int(np.prod(shape))
    inner = np.zeros(shape, bool)
    inner[interior(len(dims))] = True
    cols = np.flatnonzero(inner.ravel())
    A = np.zeros((len(cols), len(cols)), complex)
    for c, q in enumerate(cols):
        e = np.zeros(n, complex)
        e[q] = 1.0
        A[:, c] = oracle.rhs(p, e.reshape(shape), V).ravel()[cols]
    return A, cols


def test_rk4_is_the_degree4_taylor_polynomial_of_the_linear_operator(oracle_lib):
    """Linear problem (s = 0), Dirichlet-zero boundary: n RK4 steps = P(kA)^n Psi0 with
    P(z) = 1 + z + z^2/2 + z^3/6 + z^4/24 (A assembled from F column by column)."""
    dims = (7, 6)
    V = np.abs(inputs.random_smooth(dims, seed=11))
    p = Problem(dims, 0.3, a=1.0, s=0.0, bc="dirichlet", scheme="2shoc")
    A, cols = _assemble_linear(p, dims, V)
    psi = inputs.random_smooth(dims, seed=12)
    psi[0, :] = psi[-1, :] = 0
    psi[:, 0] = psi[:, -1] = 0
    k, nst = 0.004, 30
    out = oracle.step(p, psi, k, nst, V)
    Z = k * A
    P = np.eye(len(cols)) + Z + Z @ Z / 2 + Z @ Z @ Z / 6 + Z @ Z @ Z @ Z / 24
    want = np.linalg.matrix_power(P, nst) @ psi.ravel()[cols]
    np.testing.assert_allclose(out.ravel()[cols], want, rtol=0, atol=1e-13)
    assert np.all(out.ravel()[np.setdiff1d(np.arange(psi.size), cols)] == 0)


def _golden_bounds():
    rows = []
    with open(os.path.join(GOLDEN, "stability_bounds.txt")) as fh:
        for line in fh:
            if line.strip() and not line.startswith("#"):
                nd, a, h, sch, kmax, tol, cite = line.split()
                rows.append((int(nd), float(a), float(h), sch, float(kmax), float(tol), cite))
    return rows


@pytest.mark.parametrize("row", _golden_bounds())
def test_brute_force_stability_matches_paper_bounds(oracle_lib, row):
    """Brute force: the largest dense eigenvalue of the oracle's linear operator with the RK4
    imaginary-axis limit 2*sqrt(2) reproduces the paper's printed linear bounds from above as
    the grid grows ((stblincd) P:363-367, (stblin2shoc) P:368-372, values P:384 / P:393)."""
    nd, a, h, sch, kpaper, tol, cite = row
    n = 65 if nd == 1 else 17
    dims = (n,) * nd
    p = Problem(dims, h, a=a, s=0.0, bc="dirichlet", scheme=sch)
    A, _ = _assemble_linear(p, dims, None)
    kmax = 2 * math.sqrt(2) / np.abs(np.linalg.eigvals(A)).max()
    assert kmax >= kpaper - tol, (kmax, kpaper, cite)
    assert kmax <= kpaper * (1.03 if nd == 1 else 1.15) + tol, (kmax, kpaper, cite)


# ---------------------------------------------------------------------------------------------
# Exact solutions, convergence orders, conservation
# ---------------------------------------------------------------------------------------------

def test_bright_soliton_config1(oracle_lib):
    """BASELINE configs[0]: 1D bright soliton, N=1025, h=0.05, k=0.001, 1000 steps, 2SHOC, Dirichlet:
    error vs the exact sech solution at t=1, and mass M = 4 sqrt(a Omega)/s = 4, H = c^2 - 4/3."""
    cfg = inputs.config("bright1d")
    p = Problem(cfg["dims"], cfg["h"], a=1.0, s=1.0, bc="dirichlet", scheme="2shoc")
    x = inputs.axis(cfg["dims"][0], cfg["h"])
    out = oracle.step(p, cfg["psi0"], cfg["k"], cfg["steps"])
    ex = inputs.bright_soliton(x, t=1.0)
    assert np.abs(out - ex).max() < 2.0e-6
    assert np.linalg.norm(out - ex) / np.linalg.norm(ex) < 1.0e-6
    m0, h0 = oracle.diagnostics(p, cfg["psi0"])
    m1, h1 = oracle.diagnostics(p, out)
    assert abs(m0 - 4.0) < 1e-12
    assert abs(h0 - (0.25 - 4.0 / 3.0)) < 1e-3       # O(h^2) forward-difference kinetic term
    assert abs(m1 - m0) < 1e-10 and abs(h1 - h0) < 1e-7


def _order(errs):
    return [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]


@pytest.mark.parametrize("scheme,lo,hi", [("cd", 1.85, 2.15), ("2shoc", 3.7, 4.3)])
def test_dark_soliton_msd_convergence_orders(oracle_lib, scheme, lo, hi):
    """BASELINE configs[1]: 1D dark soliton (soliton) P:379-384, MSD, t = 5 on [-50, 50],
    k = 0.8 x the linear bound: spatial orders 2 (CD) and 4 (2SHOC)."""
    errs = []
    for h in (0.2, 0.1, 0.05):
        n = int(round(100 / h)) + 1
        x = inputs.axis(n, h)
        kb = h * h / math.sqrt(2) * (1.0 if scheme == "cd" else 0.75)
        nst = math.ceil(5.0 / (0.8 * kb))
        p = Problem((n,), h, a=1.0, s=-1.0, bc="msd", scheme=scheme)
        out = oracle.step(p, inputs.dark_soliton(x), 5.0 / nst, nst)
        errs.append(np.abs(out - inputs.dark_soliton(x, t=5.0)).max())
        assert abs(abs(out[0]) ** 2 - 1) < 1e-8 and abs(abs(out[-1]) ** 2 - 1) < 1e-8
    for o in _order(errs):
        assert lo <= o <= hi, (errs, _order(errs))


@pytest.mark.parametrize("scheme,lo,hi", [("cd", 1.9, 2.1), ("2shoc", 3.8, 4.2)])
def test_bright_soliton_convergence_orders(oracle_lib, scheme, lo, hi):
    errs = []
    for h in (0.1, 0.05, 0.025):
        n = int(round(51.2 / h)) + 1
        x = inputs.axis(n, h)
        p = Problem((n,), h, a=1.0, s=1.0, bc="dirichlet", scheme=scheme)
        out = oracle.step(p, inputs.bright_soliton(x), 2.5e-4, 4000)
        errs.append(np.abs(out - inputs.bright_soliton(x, t=1.0)).max())
    for o in _order(errs):
        assert lo <= o <= hi, (errs, _order(errs))


def test_temporal_order_four(oracle_lib):
    """RK4 is fourth order in k: self-convergence on the bright soliton at fixed h."""
    h = 0.1
    n = 513
    x = inputs.axis(n, h)
    p = Problem((n,), h, a=1.0, s=1.0, bc="dirichlet", scheme="2shoc")
    ref = oracle.step(p, inputs.bright_soliton(x), 1.0 / 16000, 16000)
    errs = []
    for nst in (250, 500, 1000):
        out = oracle.step(p, inputs.bright_soliton(x), 1.0 / nst, nst)
        errs.append(np.linalg.norm(out - ref) / np.linalg.norm(ref))
    for o in _order(errs):
        assert 3.7 <= o <= 4.3, (errs, _order(errs))


def test_fp32_tracks_fp64(oracle_lib):
    """The single-precision oracle stays within fp32 rounding of the double one (1000 steps)."""
    cfg = inputs.config("bright1d")
    p64 = Problem(cfg["dims"], cfg["h"], a=1.0, s=1.0, bc="dirichlet", scheme="2shoc")
    p32 = Problem(cfg["dims"], cfg["h"], a=1.0, s=1.0, bc="dirichlet", scheme="2shoc", precision="fp32")
    a = oracle.step(p64, cfg["psi0"], cfg["k"], 1000)
    b = oracle.step(p32, cfg["psi0"], cfg["k"], 1000)
    assert b.dtype == np.complex64
    rel = np.linalg.norm(b - a) / np.linalg.norm(a)
    assert 1e-9 < rel < 2e-5


def test_chunk_invariance(oracle_lib):
    """Chunking is observationally invisible: 1 x 60 steps == 4 x 15 steps, bit for bit."""
    dims = (12, 11)
    psi = inputs.random_smooth(dims, seed=21, offset=1.0)
    p = Problem(dims, 0.3, a=1.0, s=-1.0, bc="msd", scheme="2shoc")
    a = oracle.step(p, psi, 0.005, 60)
    b = psi
    for _ in range(4):
        b = oracle.step(p, b, 0.005, 15)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_vortex2d_phase_rotates_at_omega(oracle_lib):
    """(exmp2Dvort) P:386-393: the approximate vortex's phase advances at ~Omega (within 5%)."""
    dims = (70, 70)
    h, k, nst = 0.25, 0.005, 1000
    psi0 = inputs.vortex2d(dims, h)
    p = Problem(dims, h, a=1.0, s=-1.0, bc="msd", scheme="2shoc")
    x, y = inputs.mesh(dims, h)
    r = np.hypot(x - inputs.core_shift(70, h), y - inputs.core_shift(70, h))
    j, i = np.unravel_index(np.argmin(np.abs(r - 5.0)), r.shape)
    out, phases = psi0, [np.angle(psi0[j, i])]
    for _ in range(10):                      # sample the phase 10 times and unwrap
        out = oracle.step(p, out, k, nst // 10)
        phases.append(np.angle(out[j, i]))
    rate = (np.unwrap(phases)[-1] - phases[0]) / (k * nst)
    assert abs(rate - (-1.0)) < 0.05, rate


def test_msd_preserves_background(oracle_lib):
    """MSD keeps the boundary density of the dark soliton at |Omega/s| = 1."""
    h = 0.1
    n = 1001
    x = inputs.axis(n, h)
    p = Problem((n,), h, a=1.0, s=-1.0, bc="msd", scheme="2shoc")
    out = oracle.step(p, inputs.dark_soliton(x), 0.004, 2500)
    assert abs(abs(out[0]) ** 2 - 1) < 1e-3 and abs(abs(out[-1]) ** 2 - 1) < 1e-3


def test_ring3d_smoke(oracle_lib):
    """3D ring (3dvr1) P:395-400 on 29x29x67, h = 1.5, k = 0.03, MSD: stays finite, boundary |Psi|^2 ~ 1."""
    dims = (29, 29, 67)
    psi0 = inputs.vortex_ring(dims, 1.5, d=5.0)
    p = Problem(dims, 1.5, a=1.0, s=-1.0, bc="msd", scheme="2shoc")
    out = oracle.step(p, psi0, 0.03, 200)
    assert np.all(np.isfinite(out))
    assert abs(abs(out[0, 0, 0]) ** 2 - abs(psi0[0, 0, 0]) ** 2) < 1e-6


# ---------------------------------------------------------------------------------------------
# Diagnostics (reading R-DIAG): closed forms for a Gaussian, term by term
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("a,s,w", [(1.0, 0.0, 0.0), (0.5, 0.0, 0.0), (1.0, -2.0, 0.0), (1.0, 0.0, 0.3), (0.7, 1.5, 0.2)])
def test_diagnostics_gaussian_closed_forms(oracle_lib, a, s, w):
    """Psi = exp(-r^2/(2 sig^2)) e^{i kap x} in 2D: M = pi sig^2; H = a(pi + kap^2 pi sig^2)
    + w^2 pi sig^4 - (s/2) pi sig^2 / 2 (forward differences are O(h^2) accurate)."""
    sig, kap, h = 2.0, 0.7, 0.05
    dims = (641, 641)
    x, y = inputs.mesh(dims, h)
    psi = np.exp(-(x * x + y * y) / (2 * sig * sig)) * np.exp(1j * kap * x)
    V = w * w * (x * x + y * y)
    p = Problem(dims, h, a=a, s=s)
    M, H = oracle.diagnostics(p, psi, V)
    assert abs(M - math.pi * sig ** 2) < 1e-10
    Hx = a * (math.pi + kap ** 2 * math.pi * sig ** 2) + w * w * math.pi * sig ** 4 - 0.5 * s * math.pi * sig ** 2 / 2
    assert abs(H - Hx) < 2e-3 * max(1.0, abs(Hx)), (H, Hx)


# ---------------------------------------------------------------- L0 boundary condition (§8(f) rank 1)

@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_l0_uniform_field_is_the_scalar_ode(oracle_lib, ndim):
    """L0 ((BCL0dt) P:347-350, (BCL0lap) P:352-355): a uniform field has Lap = 0 inside and,
    by definition, on the boundary, so every point -- boundary included -- follows the scalar
    RK4 of z' = i(s|z|^2 - V0) z bit for bit."""
    dims = (7, 5, 6)[:ndim]
    s, V0, k, n = 1.7, 0.3, 0.01, 30
    z = 0.6 + 0.7j
    psi = np.full(tuple(reversed(dims)), z)
    p = Problem(dims, 0.5, a=1.0, s=s, bc="l0", scheme="2shoc")
    out = oracle.step(p, psi, k, n, np.full(psi.shape, V0))

    def f(w):
        return 1j * (s * abs(w) ** 2 - V0) * w
    for _ in range(n):
        k1 = f(z); k2 = f(z + k / 2 * k1); k3 = f(z + k / 2 * k2); k4 = f(z + k * k3)
        z = z + k / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
    assert np.ptp(out.real) == 0 and np.ptp(out.imag) == 0
    assert abs(out.flat[0] - z) < 1e-14


@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_l0_boundary_points_decouple(oracle_lib, ndim, scheme):
    """Under L0 the boundary F depends on Psi_b only: with s = 0 and V = V0 every boundary
    point is multiplied per step by the RK4 polynomial of -i V0 k, whatever the interior does."""
    dims = (9, 8, 7)[:ndim]
    psi = case_field(dims, 71)
    V0, k, n = 1.3, 0.004, 12
    p = Problem(dims, 0.3, a=0.8, s=0.0, bc="l0", scheme=scheme)
    out = oracle.step(p, psi, k, n, np.full(psi.shape, V0))
    zz = -1j * V0 * k
    g = (1 + zz + zz ** 2 / 2 + zz ** 3 / 6 + zz ** 4 / 24) ** n
    bnd = ~np.pad(np.ones(tuple(d - 2 for d in reversed(dims)), bool), 1)
    np.testing.assert_allclose(out[bnd], psi[bnd] * g, rtol=1e-14, atol=0)
    assert not np.allclose(out[~bnd], psi[~bnd] * g)        # the interior does feel the Laplacian


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_l0_bc_forms_consistent(oracle_lib, precision):
    """F_b from the Laplacian form (fsplit with Lap = 0) equals the time-derivative form
    i(s|Psi_b|^2 - V_b)Psi_b (evaluated here in numpy complex arithmetic) to a few ulps; D_b = 0
    exactly on faces (2SHOC step 1 boundary values), NaN on edges / corners (R-DFACE)."""
    dims = (8, 7, 6)
    psi = case_field(dims, 72)
    V = np.abs(case_field(dims, 73))
    p = Problem(dims, 0.3, a=0.9, s=-1.2, bc="l0", scheme="2shoc", precision=precision)
    F = oracle.rhs(p, psi, V)
    T = np.float64 if precision == "fp64" else np.float32
    ps = psi.astype(np.complex128 if precision == "fp64" else np.complex64)
    Vt = V.astype(T)
    want = 1j * (T(-1.2) * np.abs(ps) ** 2 - Vt) * ps
    bnd = ~np.pad(np.ones(tuple(d - 2 for d in reversed(dims)), bool), 1)
    eps = np.finfo(T).eps
    assert np.all(np.abs(F[bnd] - want[bnd]) <= 8 * eps * (np.abs(want[bnd]) + np.abs(ps[bnd])))
    D, _ = oracle.laplacian(p, psi, V)
    nb = sum(((np.arange(n) == 0) | (np.arange(n) == n - 1)).astype(int).reshape(
        [-1 if a == ax else 1 for a in range(3)]) for ax, n in enumerate(reversed(dims)))
    assert np.all(D[nb == 1] == 0)
    assert np.all(np.isnan(D[nb >= 2]))


# ---------------------------------------------------------------------------------------------
# MSD division guard, reading R-MSD-GUARD (the paper is silent on 1/Psi_b' at a zero)
# ---------------------------------------------------------------------------------------------

def _boundary_points(dims):
    """All boundary points (x, y, z order) with their diagonal inward neighbour b' (R-MSD-NBR)
    and, for face points, the normal inward neighbour (R-DFACE)."""
    out = []
    for q in np.ndindex(*dims):
        bnd = [i == 0 or i == n - 1 for i, n in zip(q, dims)]
        if not any(bnd):
            continue
        diag = tuple(min(max(i, 1), n - 2) for i, n in zip(q, dims))
        normal = diag if sum(bnd) == 1 else None
        out.append((q, diag, normal))
    return out


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_msd_eps_guard(oracle_lib, ndim, precision):
    """Where |Y_b'|^2 < eps^2 (eps^2 = 1e-24 fp64, 1e-12 fp32) the MSD quotient is taken as 0:
    F_b = 0 exactly ((msd) P:331-335) and D_b = ((N_b' - N_b)/a) Y_b ((BCMSDlap) P:336-344 without
    the Re(D_b'/Y_b') term).  Inputs put Psi_b' = 0, eps/2 (guarded) and 2 eps (not guarded) at
    face, edge and corner neighbours; every other boundary point must keep its quotient (F_b != 0,
    D_b != the guarded form), and unguarded points near the threshold follow (msd) exactly."""
    from helpers import EPS, guard_field, guard_points
    dims = {1: (41,), 2: (30, 23), 3: (44, 21, 17)}[ndim]
    T = np.float64 if precision == "fp64" else np.float32
    psi = guard_field(dims, precision)
    p = Problem(dims, 0.5, a=0.75, s=-1.3, bc="msd", scheme="2shoc", precision=precision)
    F = oracle.rhs(p, psi)
    D, _ = oracle.laplacian(p, psi)
    Y = psi.astype(np.complex128 if precision == "fp64" else np.complex64)
    yr, yi = Y.real.astype(T), Y.imag.astype(T)
    rho = yr * yr + yi * yi
    eps2 = T(EPS[precision] ** 2)
    a, s = T(0.75), T(-1.3)
    inv_a = T(1.0 / 0.75)
    at = lambda arr, q: arr[tuple(reversed(q))]
    zero, below, above = guard_points(dims)
    n_guard = n_quot = 0
    for b, bd, bn in _boundary_points(dims):
        fb = at(F, b)
        if at(rho, bd) < eps2:
            n_guard += 1
            assert fb.real == 0 and fb.imag == 0, (b, bd, fb)
        else:
            n_quot += 1
            f1 = at(F, bd)
            m = (T(f1.imag) * at(yr, bd) - T(f1.real) * at(yi, bd)) / at(rho, bd)
            assert fb.real == -(m * at(yi, b)) and fb.imag == m * at(yr, b), (b, fb)
            assert fb != 0, b
        if bn is not None:
            nb, n1 = s * at(rho, b), s * at(rho, bn)
            g = (n1 - nb) * inv_a
            guarded = (g * at(yr, b), g * at(yi, b))
            db = at(D, b)
            if at(rho, bn) < eps2:
                assert (db.real, db.imag) == guarded, (b, db, guarded)
            else:
                assert (db.real, db.imag) != guarded, b
    # every planted point is an inward neighbour of some boundary point and fired (or not) as set
    assert all(at(rho, q) == 0 for q in zero) and all(at(rho, q) < eps2 for q in below)
    assert all(at(rho, q) > eps2 for q in above)
    assert n_guard >= len(zero) + len(below) and (n_quot > 0 or ndim == 1)


@pytest.mark.parametrize("bc", ["dirichlet", "msd", "l0"])
def test_openmp_build_gives_the_same_bits(oracle_lib, bc):
    """The all-cores build (liboracle_omp.so, bench.py's cpu_baseline) splits only the outer loop
    of each sweep over threads: its result equals the serial oracle bit for bit."""
    dims = (23, 19, 17)
    psi = case_field(dims, seed=7)
    V = np.abs(case_field(dims, seed=8)) * 0.2
    for prec in ("fp64", "fp32"):
        p = Problem(dims, 0.5, a=0.9, s=-1.1, bc=bc, scheme="2shoc", precision=prec)
        a = oracle.step(p, psi, 0.01, 4, V)
        b = oracle.step(p, psi, 0.01, 4, V, omp=True)
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (bc, prec)
