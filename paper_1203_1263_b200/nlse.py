"""Thin ctypes binding of libnlse_b200.so (include/nlse.h): argument marshalling only.

Same names as the C ABI.  Every step of the path runs in the library's CUDA
kernels; importing this module loads the library and raises if it is missing
(there is no CPU fallback).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# NLSE_LIB selects a variant build of the same library (scripts/build_variant.py, A/B
# measurements only); the default is the in-tree libnlse_b200.so
LIB_PATH = os.environ.get("NLSE_LIB") or os.path.join(_HERE, "libnlse_b200.so")

NLSE_OK, NLSE_ERR_ARG, NLSE_ERR_UNSTABLE, NLSE_ERR_OOM, NLSE_ERR_CUDA, NLSE_ERR_COMM, NLSE_ERR_DIVERGED = range(7)
NLSE_BC_DIRICHLET, NLSE_BC_MSD, NLSE_BC_L0 = 0, 1, 2
NLSE_CD2, NLSE_2SHOC4 = 2, 4
NLSE_FP32, NLSE_FP64 = 4, 8
NLSE_FLAG_FORCE_DT, NLSE_FLAG_GENERIC_KERNELS = 1, 2
NLSE_MAX_KINDS = 12

BC = {"dirichlet": NLSE_BC_DIRICHLET, "msd": NLSE_BC_MSD, "l0": NLSE_BC_L0}
ORDER = {"cd": NLSE_CD2, "2shoc": NLSE_2SHOC4}
PREC = {"fp32": NLSE_FP32, "fp64": NLSE_FP64}


class NLSEError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


_STATUS = {0: "NLSE_OK", 1: "NLSE_ERR_ARG", 2: "NLSE_ERR_UNSTABLE", 3: "NLSE_ERR_OOM", 4: "NLSE_ERR_CUDA",
           5: "NLSE_ERR_COMM", 6: "NLSE_ERR_DIVERGED"}


class nlse_timing(ctypes.Structure):
    _fields_ = [("n_kinds", ctypes.c_int), ("name", (ctypes.c_char * 48) * NLSE_MAX_KINDS),
                ("ms", ctypes.c_double * NLSE_MAX_KINDS), ("launches", ctypes.c_int64 * NLSE_MAX_KINDS),
                ("points", ctypes.c_int64 * NLSE_MAX_KINDS)]


class nlse_info(ctypes.Structure):
    _fields_ = [("points", ctypes.c_int64), ("launches_per_step", ctypes.c_int64),
                ("min_bytes_per_step", ctypes.c_int64), ("device_bytes", ctypes.c_int64),
                ("elem_bytes", ctypes.c_int), ("variant", ctypes.c_char * 64),
                ("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("z0", ctypes.c_int64),
                ("nz_local", ctypes.c_int64)]


NLSE_MAX_RANKS = 16
NLSE_DIST_HANDLE_BYTES = 512


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    D = ctypes.POINTER(ctypes.c_double)
    lib.nlse_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_double, ctypes.c_double,
                                ctypes.c_double, D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint32,
                                ctypes.POINTER(P)]
    lib.nlse_set_psi.argtypes = [P, D]
    lib.nlse_get_psi.argtypes = [P, D]
    lib.nlse_set_psi_device.argtypes = [P, P]
    lib.nlse_get_psi_device.argtypes = [P, P]
    lib.nlse_step.argtypes = [P, ctypes.c_double, ctypes.c_int64]
    lib.nlse_diagnostics.argtypes = [P, D, D]
    lib.nlse_stability_bound.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int, D, D]
    lib.nlse_last_error.argtypes = [P]
    lib.nlse_last_error.restype = ctypes.c_char_p
    lib.nlse_status_string.argtypes = [ctypes.c_int]
    lib.nlse_status_string.restype = ctypes.c_char_p
    lib.nlse_destroy.argtypes = [P]
    lib.nlse_destroy.restype = None
    lib.nlse_get_stream.argtypes = [P, ctypes.POINTER(P)]
    lib.nlse_set_timing.argtypes = [P, ctypes.c_int]
    lib.nlse_get_timing.argtypes = [P, ctypes.POINTER(nlse_timing)]
    lib.nlse_reset_timing.argtypes = [P]
    lib.nlse_get_info.argtypes = [P, ctypes.POINTER(nlse_info)]
    I64P = ctypes.POINTER(ctypes.c_int64)
    lib.nlse_slab_range.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, I64P, I64P]
    lib.nlse_create_dist.argtypes = [ctypes.c_int, I64P, ctypes.c_double, ctypes.c_double, ctypes.c_double, D,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint32, ctypes.c_int,
                                     ctypes.c_int, ctypes.POINTER(P)]
    lib.nlse_dist_export.argtypes = [P, ctypes.c_char_p]
    lib.nlse_dist_connect.argtypes = [P, ctypes.c_char_p]
    lib.nlse_dist_connect_local.argtypes = [ctypes.POINTER(P), ctypes.c_int]
    lib.nlse_dist_abort.argtypes = [P]
    lib.nlse_step_group.argtypes = [ctypes.POINTER(P), ctypes.c_int, ctypes.c_double, ctypes.c_int64]
    lib.nlse_run_frames.argtypes = [P, ctypes.c_double, ctypes.c_int64, ctypes.c_int, D]
    lib.nlse_diagnostics_group.argtypes = [ctypes.POINTER(P), ctypes.c_int, D, D]
    for f in ("nlse_create", "nlse_set_psi", "nlse_get_psi", "nlse_set_psi_device", "nlse_get_psi_device",
              "nlse_step", "nlse_diagnostics", "nlse_stability_bound", "nlse_get_stream", "nlse_set_timing",
              "nlse_get_timing", "nlse_reset_timing", "nlse_get_info", "nlse_slab_range", "nlse_create_dist",
              "nlse_dist_export", "nlse_dist_connect", "nlse_dist_connect_local", "nlse_step_group",
              "nlse_diagnostics_group", "nlse_run_frames", "nlse_dist_abort"):
        getattr(lib, f).restype = ctypes.c_int
    return lib


lib = _load()

#: every symbol include/nlse.h declares
EXPORTS = ("nlse_create", "nlse_set_psi", "nlse_get_psi", "nlse_set_psi_device", "nlse_get_psi_device",
           "nlse_step", "nlse_diagnostics", "nlse_stability_bound", "nlse_last_error", "nlse_status_string",
           "nlse_destroy", "nlse_get_stream", "nlse_set_timing", "nlse_get_timing", "nlse_reset_timing",
           "nlse_get_info", "nlse_slab_range", "nlse_create_dist", "nlse_dist_export", "nlse_dist_connect",
           "nlse_dist_connect_local", "nlse_step_group", "nlse_diagnostics_group", "nlse_run_frames",
           "nlse_dist_abort")


def _check(st, ctx=None):
    if st != NLSE_OK:
        msg = lib.nlse_last_error(ctx).decode()
        raise NLSEError(st, msg)


def nlse_stability_bound(ndim: int, a: float, h: float, scheme: str = "2shoc"):
    """(k_max, k_rec): linear bounds (stblincd) P:363-367 / (stblin2shoc) P:368-372, k_rec = 0.8 k_max."""
    km, kr = ctypes.c_double(), ctypes.c_double()
    _check(lib.nlse_stability_bound(ndim, a, h, ORDER[scheme], ctypes.byref(km), ctypes.byref(kr)))
    return km.value, kr.value


def nlse_slab_range(nz: int, nranks: int, rank: int):
    """(z0, nloc): the global planes [z0, z0 + nloc) rank `rank` owns in slab mode."""
    z0, nl = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.nlse_slab_range(int(nz), int(nranks), int(rank), ctypes.byref(z0), ctypes.byref(nl)))
    return z0.value, nl.value


class Solver:
    """Owns one nlse_ctx.  dims = (nx,), (nx, ny) or (nx, ny, nz) (the GLOBAL grid); numpy arrays
    have shape reversed(dims) (x fastest).  dist=(rank, nranks) creates a slab-mode context
    (nlse_create_dist): Psi / V arrays then hold the local slab, shape (nloc, ny, nx) in 3D
    (z planes), (nloc, nx) in 2D (y rows) or (nloc,) in 1D (x points)."""

    def __init__(self, dims, h, a=1.0, s=1.0, V=None, bc="dirichlet", scheme="2shoc", precision="fp64",
                 force_dt=False, generic=False, dist=None):
        self.dims = tuple(int(d) for d in dims)
        self.dist = dist
        if dist is not None:
            # slab axis: z (3D), y (2D) or x (1D), the slowest axis of the (.., y, x) arrays
            rank, nranks = dist
            self.z0, nloc = nlse_slab_range(self.dims[-1], nranks, rank)
            self.shape = (nloc,) + tuple(reversed(self.dims[:-1]))
        else:
            self.shape = tuple(reversed(self.dims))
        self.precision = precision
        d3 = (ctypes.c_int64 * 3)(*(list(self.dims) + [1] * (3 - len(self.dims))))
        Vp = None
        if V is not None:
            self._V = np.ascontiguousarray(V, dtype=np.float64)
            assert self._V.shape == self.shape
            Vp = self._V.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        flags = (NLSE_FLAG_FORCE_DT if force_dt else 0) | (NLSE_FLAG_GENERIC_KERNELS if generic else 0)
        ctx = ctypes.c_void_p()
        if dist is None:
            st = lib.nlse_create(len(self.dims), d3, h, a, s, Vp, BC[bc], ORDER[scheme], PREC[precision], flags,
                                 ctypes.byref(ctx))
        else:
            st = lib.nlse_create_dist(len(self.dims), d3, h, a, s, Vp, BC[bc], ORDER[scheme], PREC[precision],
                                      flags, int(dist[0]), int(dist[1]), ctypes.byref(ctx))
        self._V = None
        _check(st, None)
        self.ctx = ctx

    def close(self):
        if getattr(self, "ctx", None):
            lib.nlse_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # --- C-ABI calls, same names ---------------------------------------------------------------
    def nlse_set_psi(self, psi):
        buf = np.ascontiguousarray(psi, dtype=np.complex128)
        assert buf.shape == self.shape, (buf.shape, self.shape)
        _check(lib.nlse_set_psi(self.ctx, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), self.ctx)

    def nlse_get_psi(self, out=None):
        if out is None:
            out = np.empty(self.shape, dtype=np.complex128)
        assert out.dtype == np.complex128 and out.flags.c_contiguous and out.shape == self.shape
        _check(lib.nlse_get_psi(self.ctx, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), self.ctx)
        return out

    def nlse_set_psi_device(self, ptr: int):
        _check(lib.nlse_set_psi_device(self.ctx, ctypes.c_void_p(ptr)), self.ctx)

    def nlse_get_psi_device(self, ptr: int):
        _check(lib.nlse_get_psi_device(self.ctx, ctypes.c_void_p(ptr)), self.ctx)

    def nlse_step(self, k: float, nsteps: int):
        _check(lib.nlse_step(self.ctx, float(k), int(nsteps)), self.ctx)

    def nlse_run_frames(self, k: float, chunk: int, nframes: int, out=None):
        """nframes x (chunk RK4 steps, then Psi to frame f); returns complex128 (nframes, *shape)."""
        if out is None:
            out = np.empty((int(nframes),) + self.shape, dtype=np.complex128)
        assert out.dtype == np.complex128 and out.flags.c_contiguous and out.shape == (int(nframes),) + self.shape
        _check(lib.nlse_run_frames(self.ctx, float(k), int(chunk), int(nframes),
                                   out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), self.ctx)
        return out

    def nlse_diagnostics(self):
        m, h = ctypes.c_double(), ctypes.c_double()
        _check(lib.nlse_diagnostics(self.ctx, ctypes.byref(m), ctypes.byref(h)), self.ctx)
        return m.value, h.value

    def nlse_get_stream(self) -> int:
        p = ctypes.c_void_p()
        _check(lib.nlse_get_stream(self.ctx, ctypes.byref(p)), self.ctx)
        return p.value or 0

    def nlse_set_timing(self, enable: bool):
        _check(lib.nlse_set_timing(self.ctx, int(bool(enable))), self.ctx)

    def nlse_reset_timing(self):
        _check(lib.nlse_reset_timing(self.ctx), self.ctx)

    def nlse_get_timing(self):
        t = nlse_timing()
        _check(lib.nlse_get_timing(self.ctx, ctypes.byref(t)), self.ctx)
        return {t.name[i].value.decode(): dict(ms=t.ms[i], launches=t.launches[i], points=t.points[i])
                for i in range(t.n_kinds)}

    def nlse_get_info(self):
        t = nlse_info()
        _check(lib.nlse_get_info(self.ctx, ctypes.byref(t)), self.ctx)
        return dict(points=t.points, launches_per_step=t.launches_per_step,
                    min_bytes_per_step=t.min_bytes_per_step, device_bytes=t.device_bytes,
                    elem_bytes=t.elem_bytes, variant=t.variant.decode(), rank=t.rank, nranks=t.nranks,
                    z0=t.z0, nz_local=t.nz_local)

    def nlse_dist_export(self) -> bytes:
        buf = ctypes.create_string_buffer(NLSE_DIST_HANDLE_BYTES)
        _check(lib.nlse_dist_export(self.ctx, buf), self.ctx)
        return buf.raw

    def nlse_dist_connect(self, handles):
        """handles: the nranks exported handles in rank order (list of bytes or one bytes object)."""
        blob = b"".join(handles) if not isinstance(handles, (bytes, bytearray)) else bytes(handles)
        _check(lib.nlse_dist_connect(self.ctx, blob), self.ctx)

    def nlse_dist_abort(self):
        _check(lib.nlse_dist_abort(self.ctx), self.ctx)

    # --- conveniences ----------------------------------------------------------------------------
    set_psi = nlse_set_psi
    get_psi = nlse_get_psi
    step = nlse_step
    diagnostics = nlse_diagnostics


# --- virtual ranks / groups of contexts in one process ----------------------------------------------

def _ctx_array(solvers):
    arr = (ctypes.c_void_p * len(solvers))(*[sv.ctx for sv in solvers])
    return arr


def nlse_dist_connect_local(solvers):
    """Connect the slab contexts of ranks 0..n-1 of one process (virtual ranks)."""
    _check(lib.nlse_dist_connect_local(_ctx_array(solvers), len(solvers)))


def nlse_step_group(solvers, k: float, nsteps: int):
    st = lib.nlse_step_group(_ctx_array(solvers), len(solvers), float(k), int(nsteps))
    if st != NLSE_OK:
        msgs = "; ".join(lib.nlse_last_error(sv.ctx).decode() for sv in solvers)
        raise NLSEError(st, msgs or lib.nlse_last_error(None).decode())


def nlse_diagnostics_group(solvers):
    n = len(solvers)
    m, h = (ctypes.c_double * n)(), (ctypes.c_double * n)()
    st = lib.nlse_diagnostics_group(_ctx_array(solvers), n, m, h)
    if st != NLSE_OK:
        raise NLSEError(st, lib.nlse_last_error(None).decode())
    return list(m), list(h)
