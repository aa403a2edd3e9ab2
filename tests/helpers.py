"""Shared helpers for the parity tests: run the same seeded input through the CUDA
path (C ABI) and through the oracle, compare element by element."""
from __future__ import annotations

import numpy as np

import oracle
from paper_1203_1263_b200 import inputs


def run_oracle(dims, h, psi0, k, nsteps, a=1.0, s=1.0, V=None, bc="dirichlet", scheme="2shoc", precision="fp64"):
    p = oracle.Problem(tuple(dims), h, a=a, s=s, bc=bc, scheme=scheme, precision=precision)
    out = oracle.step(p, psi0, k, nsteps, V)
    return out.astype(np.complex128)


def run_gpu(dims, h, psi0, k, nsteps, a=1.0, s=1.0, V=None, bc="dirichlet", scheme="2shoc", precision="fp64",
            generic=False, chunks=None, force_dt=True, with_info=False):
    from paper_1203_1263_b200.nlse import Solver
    with Solver(dims, h, a=a, s=s, V=V, bc=bc, scheme=scheme, precision=precision, force_dt=force_dt,
                generic=generic) as sv:
        sv.nlse_set_psi(psi0)
        for n in (chunks or [nsteps]):
            sv.nlse_step(k, n)
        out = sv.nlse_get_psi()
        return (out, sv.nlse_get_info()) if with_info else out


def run_gpu_slabs(dims, h, psi0, k, nsteps, nranks, a=1.0, s=1.0, V=None, bc="dirichlet", scheme="2shoc",
                  precision="fp64", generic=False, chunks=None, force_dt=True, diag=False):
    """The same run as run_gpu, partitioned into `nranks` z slabs (3D) or y-row slabs (2D) (virtual ranks on one GPU,
    nlse_dist_connect_local + nlse_step_group).  Returns the gathered global Psi (and the
    per-rank diagnostics after the run when diag=True)."""
    from paper_1203_1263_b200 import nlse
    svs = []
    try:
        for r in range(nranks):
            z0, nl = nlse.nlse_slab_range(dims[-1], nranks, r)
            Vl = None if V is None else np.ascontiguousarray(V[z0:z0 + nl])
            svs.append(nlse.Solver(dims, h, a=a, s=s, V=Vl, bc=bc, scheme=scheme, precision=precision,
                                   force_dt=force_dt, generic=generic, dist=(r, nranks)))
        nlse.nlse_dist_connect_local(svs)
        for sv in svs:
            sv.nlse_set_psi(np.ascontiguousarray(psi0[sv.z0:sv.z0 + sv.shape[0]]))
        for n in (chunks or [nsteps]):
            nlse.nlse_step_group(svs, k, n)
        out = np.concatenate([sv.nlse_get_psi() for sv in svs], axis=0)
        if diag:
            return out, nlse.nlse_diagnostics_group(svs)
        return out
    finally:
        for sv in svs:
            sv.close()


def ulp_diff(a, b, precision):
    """Max distance in units in the last place between two complex arrays (per component),
    compared in the run's precision (fp32 values are widened exactly by the ABI)."""
    if precision == "fp64":
        x = np.ascontiguousarray(a, np.complex128).view(np.int64)
        y = np.ascontiguousarray(b, np.complex128).view(np.int64)
        mask = np.int64(0x7FFFFFFFFFFFFFFF)
    else:
        x = np.ascontiguousarray(np.asarray(a).astype(np.complex64)).view(np.int32).astype(np.int64)
        y = np.ascontiguousarray(np.asarray(b).astype(np.complex64)).view(np.int32).astype(np.int64)
        mask = np.int64(0x7FFFFFFF)
        x = np.where(x >= 2 ** 31, x - 2 ** 32, x) if x.size and x.max() >= 2 ** 31 else x
        y = np.where(y >= 2 ** 31, y - 2 ** 32, y) if y.size and y.max() >= 2 ** 31 else y
    kx = np.where(x < 0, -(x & mask), x)
    ky = np.where(y < 0, -(y & mask), y)
    same = (kx >= 0) == (ky >= 0)
    d = np.where(same, np.abs(kx - np.where(same, ky, 0)), np.int64(2 ** 62))
    return int(d.max()) if d.size else 0


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


TOL = {"fp64": 1e-12, "fp32": 1e-5}   # north_star parity tolerances (relative L2)


def assert_parity(gpu, ref, precision, bitwise=True, what=""):
    assert gpu.shape == ref.shape
    assert np.all(np.isfinite(gpu)), what
    r = rel_l2(gpu, ref)
    assert r <= TOL[precision], f"{what}: rel-L2 {r:.3e} > {TOL[precision]}"
    if bitwise:
        u = ulp_diff(gpu, ref, precision)
        assert u == 0, f"{what}: max ulp {u} (rel-L2 {r:.3e}); the kernels should reproduce the oracle's DAG exactly"


def case_input(dims, seed, kind="smooth"):
    """Seeded input with a background of modulus ~1 (MSD needs |Psi_b| away from 0)."""
    return inputs.random_smooth(tuple(dims), seed=seed, modes=5, amp=0.4, offset=1.0)


# ---------------------------------------------------------------------------------------------
# MSD division guard (reading R-MSD-GUARD): inputs whose inward neighbours b' are zero
# or sit just below / above the threshold |Y_b'|^2 = eps^2, so the guarded branch is taken
# ---------------------------------------------------------------------------------------------

EPS = {"fp64": 1e-12, "fp32": 1e-6}


def guard_points(dims):
    """(zero, below, above): lists of grid indices (x, y, z order, as many as ndim) of points
    one step in from the boundary: `zero` get Psi = 0, `below` |Psi| = eps/2 (guarded),
    `above` |Psi| = 2 eps (not guarded).  They cover face, edge and corner neighbours b'."""
    n = list(dims)
    d = len(n)
    if d == 1:
        return [(1,)], [(n[0] - 2,)], []
    if d == 2:
        return ([(1, 5), (1, 1), (10, 1), (n[0] - 2, n[1] - 2), (n[0] - 2, 9)],
                [(1, 12)], [(1, 14), (7, n[1] - 2)])
    return ([(1, 5, 7), (1, 1, 9), (1, 1, 1), (10, 1, 4), (12, 8, 1), (n[0] - 2, n[1] - 2, n[2] - 2),
             (20, n[1] - 2, 11), (n[0] - 2, 10, 13), (33, 9, n[2] - 2)],
            [(1, 16, 6), (40, 1, 6)], [(1, 14, 6), (n[0] - 2, 6, 8)])


def guard_field(dims, precision, seed=1203, above=True):
    """A smooth field of modulus ~1 with the guard_points set (phase kept).  above=False leaves
    out the unguarded near-threshold points: there F_b = i Im(F_b'/Y_b') Y_b is ~1e12 times the
    field, which a time integration cannot survive (single-evaluation pins only)."""
    psi = case_input(dims, seed=seed)
    zero, below, above_pts = guard_points(dims)
    above = above_pts if above else []
    eps = EPS[precision]
    for pts, mag in ((zero, 0.0), (below, 0.5 * eps), (above, 2.0 * eps)):
        for p in pts:
            idx = tuple(reversed(p))
            v = psi[idx]
            psi[idx] = 0.0 if mag == 0.0 else mag * v / abs(v)
    return psi
