"""Pin: the oracle's whole discrete map against a second, independent implementation in
50-digit arithmetic (mpmath) on tiny grids.

The second implementation is written here directly from the paper's printed formulas, in
complex arithmetic and in the paper's own stencil form -- not from the oracle's split real /
imaginary, grouped, fused DAG:
  * RK4 as the literal 10-step schedule (RK4) P:164-180, F(Psi) = i[a lap + (s|Psi|^2 - V)Psi]
    (P:182);
  * CD / 2SHOC step 1 as the printed 7-point stencil (3d2shocs) P:232-253, (2shoc1d) P:197;
  * 2SHOC step 2 as the printed weight tables (3d2shocs2): -(1/12)(sum of the 6 face
    D - 10 D) + (1/(6h^2))(sum of the 12 edge Psi - 12 Psi); (2d2shocs2) P:214-228 likewise with
    -12 D and the 4 corners; (2shoc1d2) P:198;
  * boundary D on faces from (BCDlap) P:320-323 / (BCMSDlap) P:336-344 written as printed,
    Im(i lap_b'/Psi_b') with complex division, b' the inward normal neighbour (R-DFACE);
    edge / corner D set to NaN (never used: R-DFACE);
  * boundary F from (BCDdt) P:315-318 / (msd) P:331-335 written as printed,
    i Im[F_b'/Psi_b'] Psi_b with b' one step inward along every boundary axis (R-MSD-NBR).
Agreement to ~1e-13 (fp64) after a few steps means the oracle evaluates the paper's map and
no term, sign, weight or index is off; fp32 must agree to its own precision.
"""
import mpmath as mp
import numpy as np
import pytest

from helpers import case_input, run_oracle
from paper_1203_1263_b200 import inputs

mp.mp.dps = 50


def _mp_grid(a):
    return np.vectorize(lambda z: mp.mpc(complex(z)), otypes=[object])(a)


class MPMap:
    """The paper's RK4 + CD/2SHOC map on an array indexed [k][j][i] (x fastest)."""

    def __init__(self, shape, h, a, s, V, bc, scheme):
        self.shape, self.bc, self.scheme = shape, bc, scheme
        self.h2 = mp.mpf(h) ** 2
        self.a, self.s = mp.mpf(a), mp.mpf(s)
        self.V = None if V is None else np.vectorize(lambda v: mp.mpf(float(v)), otypes=[object])(V)
        self.nd = sum(1 for n in shape if n > 1)

    def axes(self):
        return [ax for ax in range(3) if self.shape[ax] > 1]

    def is_b(self, p, ax):
        return p[ax] == 0 or p[ax] == self.shape[ax] - 1

    def nbd(self, p):
        return [ax for ax in self.axes() if self.is_b(p, ax)]

    def v(self, p):
        return mp.mpf(0) if self.V is None else self.V[p]

    def N(self, Y, p):
        return self.s * abs(Y[p]) ** 2 - self.v(p)

    def step1(self, Y, p):
        """D = Delta_2 Y / h^2, the printed 7-point stencil (3 / 5 / 7 points by dimension)."""
        acc = -2 * len(self.axes()) * Y[p]
        for ax in self.axes():
            for d in (-1, 1):
                q = list(p); q[ax] += d
                acc += Y[tuple(q)]
        return acc / self.h2

    def inward(self, p, axes):
        q = list(p)
        for ax in axes:
            q[ax] += 1 if p[ax] == 0 else -1
        return tuple(q)

    def laplacian(self, Y):
        shp = self.shape
        D = np.empty(shp, dtype=object)
        for p in np.ndindex(*shp):
            b = self.nbd(p)
            if not b:
                D[p] = self.step1(Y, p)
            elif len(b) == 1:
                if self.bc == "dirichlet":          # (BCDlap)
                    D[p] = -(1 / self.a) * self.N(Y, p) * Y[p]
                elif self.bc == "l0":               # (BCL0lap)
                    D[p] = mp.mpc(0)
                else:                               # (BCMSDlap), printed form
                    q = self.inward(p, b)
                    Dq = self.step1(Y, q)
                    D[p] = (mp.im(1j * Dq / Y[q]) + (1 / self.a) * (self.N(Y, q) - self.N(Y, p))) * Y[p]
            else:
                D[p] = mp.mpc(mp.nan, mp.nan)       # edges / corners: never used (R-DFACE)
        if self.scheme == "cd":
            return D
        L = np.empty(shp, dtype=object)
        ax = self.axes()
        for p in np.ndindex(*shp):
            if self.nbd(p):
                continue
            face = sum(D[tuple(p[i] + (d if i == a_ else 0) for i in range(3))] for a_ in ax for d in (-1, 1))
            if self.nd == 1:                        # (2shoc1d2)
                L[p] = mp.mpf(7) / 6 * D[p] - mp.mpf(1) / 12 * face
                continue
            corners = 0
            for i1 in range(len(ax)):
                for i2 in range(i1 + 1, len(ax)):
                    for d1 in (-1, 1):
                        for d2 in (-1, 1):
                            q = list(p); q[ax[i1]] += d1; q[ax[i2]] += d2
                            corners += Y[tuple(q)]
            ncorner = 4 if self.nd == 2 else 12
            wD = -12 if self.nd == 2 else -10       # (2d2shocs2) / (3d2shocs2) centre weights
            L[p] = -(mp.mpf(1) / 12) * (face + wD * D[p]) + (corners - ncorner * Y[p]) / (6 * self.h2)
        return L

    def F(self, Y):
        L = self.laplacian(Y)
        F = np.empty(self.shape, dtype=object)
        for p in np.ndindex(*self.shape):
            if not self.nbd(p):
                F[p] = 1j * (self.a * L[p] + self.N(Y, p) * Y[p])
        for p in np.ndindex(*self.shape):
            b = self.nbd(p)
            if not b:
                continue
            if self.bc == "dirichlet":              # (BCDdt)
                F[p] = mp.mpc(0)
            elif self.bc == "l0":                   # (BCL0dt)
                F[p] = 1j * self.N(Y, p) * Y[p]
            else:                                   # (msd), b' one step in along every boundary axis
                q = self.inward(p, b)
                F[p] = 1j * mp.im(F[q] / Y[q]) * Y[p]
        return F

    def rk4(self, Psi, k, n):
        k = mp.mpf(k)
        for _ in range(n):                          # (RK4) P:164-180, steps 1-10
            Ktot = self.F(Psi)
            Ptmp = Psi + k / 2 * Ktot
            Ktmp = self.F(Ptmp)
            Ktot = Ktot + 2 * Ktmp
            Ptmp = Psi + k / 2 * Ktmp
            Ktmp = self.F(Ptmp)
            Ktot = Ktot + 2 * Ktmp
            Ptmp = Psi + k * Ktmp
            Ktmp = self.F(Ptmp)
            Psi = Psi + k / 6 * (Ktot + Ktmp)
        return Psi


CASES = [
    ((6, 5, 5), "2shoc", "msd", True),
    ((6, 5, 5), "2shoc", "dirichlet", True),
    ((6, 5, 5), "2shoc", "l0", False),
    ((6, 5, 5), "cd", "msd", False),
    ((9, 7), "2shoc", "msd", True),
    ((9, 7), "cd", "dirichlet", True),
    ((11,), "2shoc", "msd", False),
    ((11,), "2shoc", "l0", True),
]


@pytest.mark.parametrize("dims,scheme,bc,withV", CASES)
def test_oracle_equals_50_digit_map(dims, scheme, bc, withV):
    h, a, s, nsteps = 0.5, 0.9, -1.1, 3
    k = 0.3 * h * h / (len(dims) * np.sqrt(2))
    psi0 = case_input(dims, seed=311)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=312)) if withV else None
    shape3 = psi0.shape[::-1] + (1,) * (3 - psi0.ndim)            # (nx, ny, nz) index order
    Y = _mp_grid(psi0.T.reshape(shape3))
    Vm = None if V is None else V.T.reshape(shape3)
    mpmap = MPMap(shape3, h, a, s, Vm, bc, scheme)
    want = np.vectorize(lambda z: complex(z), otypes=[np.complex128])(mpmap.rk4(Y, k, nsteps))
    want = want.reshape(psi0.T.shape).T
    for precision, tol in (("fp64", 2e-13), ("fp32", 2e-5)):
        got = run_oracle(dims, h, psi0, k, nsteps, a=a, s=s, V=V, bc=bc, scheme=scheme, precision=precision)
        err = np.max(np.abs(got - want)) / np.max(np.abs(want))
        assert err < tol, (precision, err)
