"""Seeded, synthetic input generators shared by the oracle tests, the GPU parity
tests and ``bench.py``.

This module holds NONE of the method's arithmetic (no stencil, no RK4, no
boundary condition): it only evaluates closed-form initial conditions and
potentials on the grid, in float64 on the host, exactly once per run, so that
both the oracle and the CUDA path start from the same bits (SURVEY §8(c)
"Parity bar": CPU and GPU tanh/exp/atan2 differ in the last ulp, so the IC is
generated once on the host).

Arrays are numpy, C order, shape (nz, ny, nx) / (ny, nx) / (nx,), x fastest.
Grid origin: centred, x0 = -(n-1)h/2 (reading R-ORIGIN; the paper
gives only x = x0 + ih).
"""
from __future__ import annotations

import numpy as np

SEED = 1203


def axis(n: int, h: float) -> np.ndarray:
    """Grid coordinates x_i = x0 + i h with x0 = -(n-1) h / 2."""
    return (np.arange(n, dtype=np.float64) - (n - 1) / 2.0) * h


def core_shift(n: int, h: float) -> float:
    """Offset of a vortex core from the domain centre: h/2 along axes with an
    odd point count, so that the core never sits on a grid point (R-ORIGIN)."""
    return 0.5 * h if n % 2 == 1 else 0.0


def mesh(dims, h):
    """Coordinate arrays (x, y, z as needed) broadcast to the grid shape."""
    axes = [axis(n, h) for n in dims]
    grids = np.meshgrid(*reversed(axes), indexing="ij")  # (z, y, x) order
    return list(reversed(grids))  # x, y[, z]


# ---------------------------------------------------------------- closed forms

def bright_soliton(x, t=0.0, a=1.0, s=1.0, omega=1.0, c=0.5):
    """Psi = sqrt(2 Omega/s) sech(sqrt(Omega/a)(x - c t)) exp(i[(c/2a) x + (Omega - c^2/4a) t]).
    Exact for s > 0 (reading R-BRIGHT: same Galilean form as (soliton) P:382)."""
    amp = np.sqrt(2.0 * omega / s)
    env = amp / np.cosh(np.sqrt(omega / a) * (x - c * t))
    ph = (c / (2.0 * a)) * x + (omega - c * c / (4.0 * a)) * t
    return env * np.exp(1j * ph)


def dark_soliton(x, t=0.0, a=1.0, s=-1.0, omega=-1.0, c=0.5):
    """(soliton) P:379-384: sqrt|Omega/s| tanh[sqrt(|Omega|/2a)(x - c t)] exp(i[(c/2a)x + (Omega - c^2/4a) t])."""
    amp = np.sqrt(abs(omega / s))
    env = amp * np.tanh(np.sqrt(abs(omega) / (2.0 * a)) * (x - c * t))
    ph = (c / (2.0 * a)) * x + (omega - c * c / (4.0 * a)) * t
    return env * np.exp(1j * ph)


def tanh_profile(r, a=1.0, s=-1.0, omega=-1.0):
    """f(r) = sqrt|Omega/s| tanh(sqrt(|Omega|/2a) r): the 1D dark-soliton profile for x > 0, c = 0,
    used as the approximate vortex profile."""
    return np.sqrt(abs(omega / s)) * np.tanh(np.sqrt(abs(omega) / (2.0 * a)) * r)


def vortex2d(dims, h, m=1, a=1.0, s=-1.0, omega=-1.0):
    """(exmp2Dvort) P:386-393 at t = 0: f(r) e^{i m theta}, core at the domain centre (R-ORIGIN)."""
    nx, ny = dims
    x, y = mesh(dims, h)
    X = x - core_shift(nx, h)
    Y = y - core_shift(ny, h)
    r = np.hypot(X, Y)
    th = np.arctan2(Y, X)
    return tanh_profile(r, a, s, omega) * np.exp(1j * m * th)


def vortex_ring(dims, h, d=5.0, c=0.5, a=1.0, s=-1.0, omega=-1.0):
    """(3dvr1) P:395-400: g(r, z) exp(i c z / 2a), ring of radius d in the xy plane at the centre.
    g = f(rho+) f(rho-) exp(i(phi+ - phi-)): an m = 1 vortex at r = d in the r-z half plane times its
    mirror image (reading R-RING; the paper's numerically exact g needs nsoli, out of scope)."""
    nx, ny, nz = dims
    x, y, z = mesh(dims, h)
    X = x - core_shift(nx, h)
    Y = y - core_shift(ny, h)
    Z = z - core_shift(nz, h)
    r = np.hypot(X, Y)
    rp, rm = r - d, r + d
    rho_p, rho_m = np.hypot(rp, Z), np.hypot(rm, Z)
    phi_p, phi_m = np.arctan2(Z, rp), np.arctan2(Z, rm)
    g = tanh_profile(rho_p, a, s, omega) * tanh_profile(rho_m, a, s, omega) / np.sqrt(abs(omega / s))
    return g * np.exp(1j * (phi_p - phi_m)) * np.exp(1j * (c / (2.0 * a)) * z)


def harmonic_trap(dims, h, w):
    """V = w^2 r^2 about the domain centre (reading R-TRAP)."""
    coords = mesh(dims, h)
    r2 = sum(cc * cc for cc in coords)
    return (w * w) * r2


def thomas_fermi(psi, V):
    """Multiply by the Thomas-Fermi envelope sqrt(1 - V) (R-TRAP)."""
    return psi * np.sqrt(np.clip(1.0 - V, 0.0, None))


def random_smooth(dims, seed=SEED, modes=4, amp=1.0, offset=0.0):
    """Seeded low-pass random complex field (PCG64; a few Fourier modes per axis), for unit tests."""
    rng = np.random.Generator(np.random.PCG64(seed))
    coords = [np.linspace(0.0, 2.0 * np.pi, n, endpoint=False) for n in dims]
    grids = list(reversed(np.meshgrid(*reversed(coords), indexing="ij")))
    out = np.zeros(tuple(reversed(dims)), dtype=np.complex128)
    for _ in range(modes):
        kvec = rng.integers(-2, 3, size=len(dims))
        ph = rng.uniform(0, 2 * np.pi)
        c = rng.normal() + 1j * rng.normal()
        arg = sum(kv * g for kv, g in zip(kvec, grids)) + ph
        out += c * np.exp(1j * arg)
    return offset + amp * out / modes


# ---------------------------------------------------------------- named workloads (BASELINE.json configs)

def config_dims(name: str):
    """The grid of a BASELINE configuration (as config(name)["dims"], without building its IC)."""
    if name == "bright1d":
        return (1025,)
    if name.startswith("dark1d_n"):
        return (int(name.split("_n")[1]),)
    if name.startswith("dark1d"):
        h = float(name.split("_h")[1]) if "_h" in name else 0.1
        return (int(round(100.0 / h)) + 1,)
    if name.startswith("trap2d"):
        n = int(name.split("_")[1]) if "_" in name else 1024
        return (n, n)
    if name in ("ring3d", "ring3d_fp32"):
        return (87, 87, 203)
    if name.startswith("gpe3d"):
        n = int(name.split("_")[1]) if "_" in name else 1024
        return (n, n, n)
    raise KeyError(name)


def config(name: str):
    """Return a dict describing one BASELINE.json configuration:
    dims, h, k, steps, a, s, bc, scheme, precision, psi0 (complex128), V (float64 or None)."""
    if name == "bright1d":        # configs[0]
        dims = (1025,)
        h = 0.05
        x = axis(1025, h)
        return dict(name=name, dims=dims, h=h, k=0.001, steps=1000, a=1.0, s=1.0, bc="dirichlet",
                    scheme="2shoc", precision="fp64", psi0=bright_soliton(x), V=None)
    if name.startswith("dark1d_n"):  # configs[1] shape at N points on [-50, 50] (Table 1 sizes)
        n = int(name.split("_n")[1])
        h = 100.0 / (n - 1)
        x = axis(n, h)
        kb = 0.75 * h * h / 2 ** 0.5          # (stblin2shoc) P:368-372, 1D
        return dict(name=name, dims=(n,), h=h, k=0.8 * kb, steps=None, a=1.0, s=-1.0, bc="msd",
                    scheme="2shoc", precision="fp64", psi0=dark_soliton(x), V=None)
    if name.startswith("dark1d"):  # configs[1], e.g. dark1d_h0.1
        h = float(name.split("_h")[1]) if "_h" in name else 0.1
        n = int(round(100.0 / h)) + 1
        x = axis(n, h)
        return dict(name=name, dims=(n,), h=h, k=None, steps=None, a=1.0, s=-1.0, bc="msd",
                    scheme="2shoc", precision="fp64", psi0=dark_soliton(x), V=None)
    if name.startswith("trap2d"):  # configs[2]: trap2d (1024^2) or trap2d_<n> (n^2, same physical box / n)
        n = int(name.split("_")[1]) if "_" in name else 1024
        dims = (n, n)
        h = 0.25
        V = harmonic_trap(dims, h, 1.0 / 256.0 * (1024.0 / n))
        return dict(name=name, dims=dims, h=h, k=0.005, steps=1000, a=1.0, s=-1.0, bc="msd",
                    scheme="2shoc", precision="fp64", psi0=thomas_fermi(vortex2d(dims, h), V), V=V)
    if name in ("ring3d", "ring3d_fp32"):  # configs[3]
        dims = (87, 87, 203)
        h = 1.5
        return dict(name=name, dims=dims, h=h, k=0.03, steps=3360, a=1.0, s=-1.0, bc="msd",
                    scheme="2shoc", precision="fp32" if name.endswith("fp32") else "fp64",
                    psi0=vortex_ring(dims, h, d=5.0), V=None)
    if name.startswith("gpe3d"):   # configs[4]: gpe3d (1024^3) or gpe3d_<n> for smaller cubes
        n = int(name.split("_")[1]) if "_" in name else 1024
        return dict(name=name, dims=(n, n, n), h=0.25, k=0.005, steps=100, a=1.0, s=-1.0, bc="msd",
                    scheme="2shoc", precision="fp64", psi0=None, V=None, has_V=True,
                    w=1.0 / 320.0 * (1024.0 / n), ring_d=32.0 * n / 1024.0)
    raise KeyError(name)


def gpe3d_slab(n: int, z0: int, z1: int, h: float = 0.25):
    """Planes [z0, z1) of the n^3 GPE workload (configs[4], reading R-TRAP): a vortex ring of radius
    d = 32 n/1024 (R-RING, c = 0.5) times the Thomas-Fermi envelope sqrt(1 - V), V = w^2 r^2 with
    w = (1/320)(1024/n).  Returns (psi complex128, V float64), shape (z1 - z0, n, n)."""
    w = 1.0 / 320.0 * (1024.0 / n)
    d = 32.0 * n / 1024.0
    ax = axis(n, h)
    zs = ax[z0:z1]
    Z, Yy, X = np.meshgrid(zs, ax, ax, indexing="ij")
    V = (w * w) * (X * X + Yy * Yy + Z * Z)
    sh = core_shift(n, h)
    Xc, Yc, Zc = X - sh, Yy - sh, Z - sh
    r = np.hypot(Xc, Yc)
    rp, rm = r - d, r + d
    g = tanh_profile(np.hypot(rp, Zc)) * tanh_profile(np.hypot(rm, Zc))
    psi = g * np.exp(1j * (np.arctan2(Zc, rp) - np.arctan2(Zc, rm))) * np.exp(1j * 0.25 * Z)
    psi *= np.sqrt(np.clip(1.0 - V, 0.0, None))
    return psi, V


def gpe3d_fill(n: int, psi_out=None, V_out=None, threads: int = 0, h: float = 0.25):
    """The full n^3 GPE workload, generated slab by slab on all host cores (numpy releases the GIL)
    into caller-provided (or new) arrays of shape (n, n, n).  Identical values to gpe3d_slab."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    if psi_out is None:
        psi_out = np.empty((n, n, n), np.complex128)
    if V_out is None:
        V_out = np.empty((n, n, n), np.float64)
    slab = max(1, min(8, n // 8))

    def work(z0):
        z1 = min(n, z0 + slab)
        p, v = gpe3d_slab(n, z0, z1, h)
        psi_out[z0:z1] = p
        V_out[z0:z1] = v
    with ThreadPoolExecutor(threads or os.cpu_count() or 1) as ex:
        list(ex.map(work, range(0, n, slab)))
    return psi_out, V_out
