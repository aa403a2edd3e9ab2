"""The C-ABI library loads, exports every symbol include/nlse.h declares, and its
host-side logic (validation, stability bounds) behaves -- no GPU needed."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nlse.h")
GOLDEN = os.path.join(ROOT, "tests", "golden", "stability_bounds.txt")


@pytest.fixture(scope="module")
def nlse():
    from paper_1203_1263_b200 import build
    build.build()
    from paper_1203_1263_b200 import nlse as m
    return m


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nlse_[a-z_]+)\s*\(", src)))


def test_header_declares_the_survey_entry_points():
    fns = declared_functions()
    for f in ("nlse_create", "nlse_step", "nlse_diagnostics", "nlse_set_psi", "nlse_get_psi",
              "nlse_stability_bound", "nlse_last_error", "nlse_destroy"):
        assert f in fns


def test_library_exports_every_declared_symbol(nlse):
    lib = ctypes.CDLL(nlse.LIB_PATH)
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    assert set(nlse.EXPORTS) == set(declared_functions())


def test_library_is_sm100a(nlse):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", nlse.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _golden():
    rows = []
    for line in open(GOLDEN):
        if line.strip() and not line.startswith("#"):
            nd, a, h, sch, kmax, tol, cite = line.split()
            rows.append((int(nd), float(a), float(h), sch, float(kmax), float(tol), cite))
    return rows


@pytest.mark.parametrize("row", _golden())
def test_stability_bound_matches_paper(nlse, row):
    """nlse_stability_bound reproduces the bounds the paper prints."""
    nd, a, h, sch, k, tol, cite = row
    kmax, krec = nlse.nlse_stability_bound(nd, a, h, sch)
    assert abs(kmax - k) <= tol, (kmax, k, cite)
    assert krec == pytest.approx(0.8 * kmax, rel=1e-15)


def test_stability_bound_properties(nlse):
    """2SHOC bound = 3/4 CD bound; decreasing in d and a; the d=3, h=1 value 1/(3 sqrt 2)."""
    cd, _ = nlse.nlse_stability_bound(3, 1.0, 1.0, "cd")
    assert cd == pytest.approx(1 / (3 * 2 ** 0.5), rel=1e-15)
    for d in (1, 2, 3):
        c, _ = nlse.nlse_stability_bound(d, 1.3, 0.2, "cd")
        s, _ = nlse.nlse_stability_bound(d, 1.3, 0.2, "2shoc")
        assert s == pytest.approx(0.75 * c, rel=1e-15)
    assert nlse.nlse_stability_bound(2, 1.0, 0.1)[0] < nlse.nlse_stability_bound(1, 1.0, 0.1)[0]
    assert nlse.nlse_stability_bound(1, 2.0, 0.1)[0] < nlse.nlse_stability_bound(1, 1.0, 0.1)[0]


@pytest.mark.parametrize("bad", [
    dict(ndim=4), dict(ndim=0), dict(dims=(2, 5, 1)), dict(dims=(5, 5, 2)), dict(h=0.0), dict(h=-1.0),
    dict(a=0.0), dict(s=float("nan")), dict(bc=7), dict(order=3), dict(prec=2), dict(V=float("inf")),
])
def test_create_rejects_bad_arguments_before_touching_the_device(nlse, bad):
    args = dict(ndim=2, dims=(5, 5, 1), h=0.1, a=1.0, s=1.0, V=None, bc=0, order=4, prec=8)
    args.update(bad)
    d3 = (ctypes.c_int64 * 3)(*args["dims"])
    Vp = None
    if args["V"] is not None:
        import numpy as np
        arr = np.full(25, args["V"])
        Vp = arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    ctx = ctypes.c_void_p()
    st = nlse.lib.nlse_create(args["ndim"], d3, args["h"], args["a"], args["s"], Vp, args["bc"], args["order"],
                              args["prec"], 0, ctypes.byref(ctx))
    assert st == nlse.NLSE_ERR_ARG
    assert not ctx.value
    assert nlse.lib.nlse_last_error(None)


def test_no_cpu_fallback(nlse):
    """Without a CUDA device nlse_create fails loudly (there is no CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(nlse.NLSEError) as e:
        nlse.Solver((9,), 0.1)
    assert e.value.status == nlse.NLSE_ERR_CUDA


def test_status_strings(nlse):
    assert nlse.lib.nlse_status_string(6) == b"NLSE_ERR_DIVERGED"
    assert nlse.lib.nlse_stability_bound(1, 1.0, 0.1, 3, None, None) == nlse.NLSE_ERR_ARG


def build_c_demo(tmp_path):
    """Compile tests/c/abi_demo.c as plain C against include/nlse.h and link libnlse_b200.so."""
    import subprocess
    from paper_1203_1263_b200 import build
    build.build()
    exe = str(tmp_path / "abi_demo")
    libdir = os.path.dirname(build.LIB)
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-O2", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "c", "abi_demo.c"), "-o", exe, "-L", libdir, "-lnlse_b200",
                           "-Wl,-rpath," + libdir, "-lm"])
    return exe


def test_c_client_compiles_and_links(tmp_path):
    """The header is plain C (no torch / CUDA types) and a C program links every call it makes."""
    assert os.path.exists(build_c_demo(tmp_path))
