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
    """The same run as run_gpu, partitioned into `nranks` z slabs (virtual ranks on one GPU,
    nlse_dist_connect_local + nlse_step_group).  Returns the gathered global Psi (and the
    per-rank diagnostics after the run when diag=True)."""
    from paper_1203_1263_b200 import nlse
    svs = []
    try:
        for r in range(nranks):
            z0, nl = nlse.nlse_slab_range(dims[2], nranks, r)
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
