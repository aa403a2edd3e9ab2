"""TEST INFRASTRUCTURE ONLY: the plain CPU oracle for the NLSEmagic hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1203_1263_b200`` never imports it and shares no code with it.
"""
from .oracle import (  # noqa: F401
    Problem, build, step, rhs, laplacian, diagnostics, library_path,
)
