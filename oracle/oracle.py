"""TEST INFRASTRUCTURE ONLY: ctypes binding of oracle/liboracle.so.

Arrays are numpy, C order, shape ``(nz, ny, nx)`` for 3D, ``(ny, nx)`` for 2D and
``(nx,)`` for 1D (x fastest, offset ``(k*ny + j)*nx + i``).  Psi is complex
(complex128 for fp64 runs; for fp32 runs the real and imaginary parts are
rounded once to float32, as the paper's single-precision integrators cast their
inputs).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nlse_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c99"]


def _cflags():
    """-mfma when the host has FMA3 (C99 fma() is then one instruction; it is correctly
    rounded either way, so results do not depend on the host).  -ffp-contract=off keeps the
    compiler from fusing anything the source does not fuse explicitly."""
    try:
        if " fma " in open("/proc/cpuinfo").read().replace("\n", " "):
            return CFLAGS + ["-mfma"]
    except OSError:
        pass
    return CFLAGS


def library_path() -> str:
    return _LIB


_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc, no FMA contraction, no fast-math): the serial library and
    its OpenMP twin (same source, outer loops of each sweep split over threads)."""
    deps = [_SRC, os.path.join(_HERE, "nlse_oracle_impl.h"), os.path.join(_HERE, "nlse_oracle.h")]
    for lib, extra in ((_LIB, []), (_LIB_OMP, ["-fopenmp"])):
        if force or not os.path.exists(lib) or any(os.path.getmtime(d) > os.path.getmtime(lib) for d in deps):
            tmp = lib + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", *_cflags(), *extra, "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, lib)
    return _LIB


class _Problem(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int), ("n", ctypes.c_long * 3), ("h", ctypes.c_double),
                ("a", ctypes.c_double), ("s", ctypes.c_double), ("bc", ctypes.c_int),
                ("order", ctypes.c_int)]


BC = {"dirichlet": 0, "msd": 1, "l0": 2}
ORDER = {"cd": 2, "2shoc": 4}


@dataclass(frozen=True)
class Problem:
    dims: tuple            # (nx,) / (nx, ny) / (nx, ny, nz)
    h: float
    a: float = 1.0
    s: float = 1.0
    bc: str = "dirichlet"  # "dirichlet" | "msd" | "l0"
    scheme: str = "2shoc"  # "cd" | "2shoc"
    precision: str = "fp64"  # "fp64" | "fp32"

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def shape(self) -> tuple:
        return tuple(reversed(self.dims))

    def c_struct(self) -> _Problem:
        n = list(self.dims) + [1] * (3 - len(self.dims))
        return _Problem(self.ndim, (ctypes.c_long * 3)(*n), self.h, self.a, self.s,
                        BC[self.bc], ORDER[self.scheme])


_libs = {}


def _load(omp: bool = False):
    if omp not in _libs:
        build()
        lib = ctypes.CDLL(_LIB_OMP if omp else _LIB)
        for prec, T in (("f64", ctypes.c_double), ("f32", ctypes.c_float)):
            P = ctypes.POINTER(T)
            getattr(lib, f"oracle_step_{prec}").argtypes = [ctypes.POINTER(_Problem), P, P, P, ctypes.c_double, ctypes.c_long]
            getattr(lib, f"oracle_rhs_{prec}").argtypes = [ctypes.POINTER(_Problem), P, P, P, P, P]
            getattr(lib, f"oracle_lap_{prec}").argtypes = [ctypes.POINTER(_Problem), P, P, P, P, P, P, P]
        D = ctypes.POINTER(ctypes.c_double)
        lib.oracle_diag_f64.argtypes = [ctypes.POINTER(_Problem), D, D, D, D, D]
        _libs[omp] = lib
    return _libs[omp]


def _real_dtype(p: Problem):
    return np.float64 if p.precision == "fp64" else np.float32


def _ptr(a):
    if a is None:
        return None
    ct = ctypes.c_double if a.dtype == np.float64 else ctypes.c_float
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _split(p: Problem, psi):
    T = _real_dtype(p)
    psi = np.asarray(psi)
    assert psi.shape == p.shape, (psi.shape, p.shape)
    return np.ascontiguousarray(psi.real, dtype=T), np.ascontiguousarray(psi.imag, dtype=T)


def _v(p: Problem, V):
    if V is None:
        return None
    V = np.ascontiguousarray(V, dtype=_real_dtype(p))
    assert V.shape == p.shape
    return V


def _join(re, im):
    out = np.empty(re.shape, dtype=np.complex128 if re.dtype == np.float64 else np.complex64)
    out.real, out.imag = re, im
    return out


def _suffix(p):
    return "f64" if p.precision == "fp64" else "f32"


def step(p: Problem, psi, k: float, nsteps: int, V=None, omp: bool = False):
    """nsteps RK4 steps. Returns a new complex array (complex64 for fp32).
    omp=True runs the OpenMP build (all host cores, OMP_NUM_THREADS; same result bits)."""
    re, im = _split(p, psi)
    Vc = _v(p, V)
    rc = getattr(_load(omp), f"oracle_step_{_suffix(p)}")(ctypes.byref(p.c_struct()), _ptr(Vc), _ptr(re), _ptr(im), float(k), int(nsteps))
    if rc != 0:
        raise ValueError(f"oracle_step rejected its arguments (rc={rc})")
    return _join(re, im)


def rhs(p: Problem, psi, V=None):
    """F(Psi) on the whole grid (interior (fsplit) P:424, boundary BC time-derivative form)."""
    re, im = _split(p, psi)
    fr, fi = np.empty_like(re), np.empty_like(im)
    rc = getattr(_load(), f"oracle_rhs_{_suffix(p)}")(ctypes.byref(p.c_struct()), _ptr(_v(p, V)), _ptr(re), _ptr(im), _ptr(fr), _ptr(fi))
    if rc != 0:
        raise ValueError(f"oracle_rhs rejected its arguments (rc={rc})")
    return _join(fr, fi)


def laplacian(p: Problem, psi, V=None):
    """(D, L): step-1 D (boundary faces from the Laplacian-form BC for 2SHOC) and L (interior)."""
    re, im = _split(p, psi)
    dr, di, lr, li = (np.empty_like(re) for _ in range(4))
    rc = getattr(_load(), f"oracle_lap_{_suffix(p)}")(ctypes.byref(p.c_struct()), _ptr(_v(p, V)), _ptr(re), _ptr(im), _ptr(dr), _ptr(di), _ptr(lr), _ptr(li))
    if rc != 0:
        raise ValueError(f"oracle_lap rejected its arguments (rc={rc})")
    return _join(dr, di), _join(lr, li)


def diagnostics(p: Problem, psi, V=None):
    """(mass, hamiltonian) in fp64 with Kahan sums; fp32 inputs are widened exactly."""
    psi = np.asarray(psi).astype(np.complex128)
    re, im = np.ascontiguousarray(psi.real), np.ascontiguousarray(psi.imag)
    Vd = None if V is None else np.ascontiguousarray(np.asarray(V).astype(_real_dtype(p)).astype(np.float64))
    m, h = ctypes.c_double(), ctypes.c_double()
    q = Problem(p.dims, p.h, p.a, p.s, p.bc, p.scheme, "fp64")
    rc = _load().oracle_diag_f64(ctypes.byref(q.c_struct()), _ptr(Vd), _ptr(re), _ptr(im), ctypes.byref(m), ctypes.byref(h))
    if rc != 0:
        raise ValueError("oracle_diag rejected its arguments")
    return m.value, h.value
