"""GPU parity of the 2D warp-strip kernel (csrc/strip2d.cuh, the 2D default since round 2)
against the oracle, bit for bit, on the grid shapes its decomposition distinguishes:

* strips of W = 32 - 2w interior columns (28 for 2SHOC, 30 for CD): nx - 2 a multiple of W, one
  more / one less, the x = nx - 1 face on the lane right after the last output lane of a full
  strip, a single interior column (nx = 3);
* chunks of rows per warp (NLSE_STRIP_ROWS): 1, 2, 3 rows (the face rows 0 / ny - 1 ride along in
  the iterations of rows 1 / ny - 2, a chunk may hold only one of them, or both when ny = 3), and
  the launch heuristic;
* both schemes, the three BCs, fp32 / fp64, with and without V, the MSD division guard.
The oracle is the plain C program of oracle/ (tests/helpers.py)."""
import math

import numpy as np
import pytest

from helpers import assert_parity, case_input, run_gpu, run_oracle
from paper_1203_1263_b200 import inputs

pytestmark = pytest.mark.gpu


def _k(h, scheme):
    return 0.5 * h * h / (2 * math.sqrt(2)) * (0.75 if scheme == "2shoc" else 1.0)


NX = [3, 4, 5, 29, 30, 31, 32, 33, 58, 59, 60, 61, 62, 87, 90]


@pytest.mark.parametrize("nx", NX)
@pytest.mark.parametrize("bc", ["dirichlet", "msd", "l0"])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
def test_strip_widths(nx, bc, scheme):
    dims = (nx, 11)
    h = 0.3
    psi0 = case_input(dims, seed=300 + nx)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=400 + nx))
    kw = dict(a=0.9, s=-1.1, V=V, bc=bc, scheme=scheme)
    ref = run_oracle(dims, h, psi0, _k(h, scheme), 9, **kw)
    got, info = run_gpu(dims, h, psi0, _k(h, scheme), 9, with_info=True, **kw)
    assert info["variant"] == "stage2d_strip", info
    assert_parity(got, ref, "fp64", what=f"nx={nx} {scheme} {bc}")


@pytest.mark.parametrize("div", ["1", "2", "3"])
@pytest.mark.parametrize("rows", ["1", "2", "3", "0"])
@pytest.mark.parametrize("ny", [3, 4, 5, 8, 37])
@pytest.mark.parametrize("bc", ["dirichlet", "msd", "l0"])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
def test_strip_row_chunks(rows, ny, bc, scheme, div, monkeypatch):
    """Row chunks of the interior strips (NLSE_STRIP_ROWS) and of the two edge strips (rows / div)."""
    if rows != "0":
        monkeypatch.setenv("NLSE_STRIP_ROWS", rows)
    monkeypatch.setenv("NLSE_STRIP_EDGE_DIV", div)
    dims = (61, ny)
    h = 0.3
    psi0 = case_input(dims, seed=500 + ny)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=600 + ny))
    kw = dict(a=0.9, s=-1.1, V=V, bc=bc, scheme=scheme)
    ref = run_oracle(dims, h, psi0, _k(h, scheme), 7, **kw)
    got = run_gpu(dims, h, psi0, _k(h, scheme), 7, **kw)
    assert_parity(got, ref, "fp64", what=f"ny={ny} rows={rows} {scheme} {bc}")


@pytest.mark.parametrize("withV", [False, True], ids=["V0", "V"])
@pytest.mark.parametrize("bc", ["dirichlet", "msd", "l0"])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
def test_strip_fp32(withV, bc, scheme):
    dims = (87, 45)
    h = 0.3
    psi0 = case_input(dims, seed=700)
    V = 0.3 * np.abs(inputs.random_smooth(dims, seed=701)) if withV else None
    kw = dict(a=0.9, s=-1.1, V=V, bc=bc, scheme=scheme, precision="fp32")
    ref = run_oracle(dims, h, psi0, _k(h, scheme), 11, **kw)
    got = run_gpu(dims, h, psi0, _k(h, scheme), 11, **kw)
    assert_parity(got, ref, "fp32", what=f"fp32 {scheme} {bc} V={withV}")


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("scheme", ["cd", "2shoc"])
def test_strip_msd_guard(scheme, precision):
    """Psi = 0 on whole rows / columns next to the faces: the MSD quotient at b' is guarded
    (reading R-MSD-GUARD), in the x-face lanes, the y-face rows and the corners."""
    dims = (45, 23)
    h = 0.3
    psi0 = case_input(dims, seed=801)
    psi0[1, :] = 0
    psi0[:, 1] = 0
    psi0[-2, 5:9] = 0
    psi0[3:7, -2] = 0
    kw = dict(a=0.9, s=-1.1, V=None, bc="msd", scheme=scheme, precision=precision)
    ref = run_oracle(dims, h, psi0, _k(h, scheme), 3, **kw)
    got = run_gpu(dims, h, psi0, _k(h, scheme), 3, **kw)
    assert_parity(got, ref, precision, what=f"guard {scheme} {precision}")
