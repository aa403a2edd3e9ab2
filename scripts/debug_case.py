"""Run one parity case through the C ABI and compare with the oracle (debug helper)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

from helpers import case_input, run_gpu, run_gpu_slabs, run_oracle, ulp_diff  # noqa: E402
from paper_1203_1263_b200 import inputs  # noqa: E402

dims = tuple(int(x) for x in sys.argv[1].split("x"))
scheme, bc, prec = sys.argv[2], sys.argv[3], sys.argv[4]
withV = len(sys.argv) > 5 and sys.argv[5] == "V"
n = int(os.environ.get("NSTEPS", "4"))
h = 0.5
psi0 = case_input(dims, seed=103)
V = 0.3 * np.abs(inputs.random_smooth(dims, seed=203)) if withV else None
k = 0.5 * h * h / (len(dims) * 2 ** 0.5) * (0.75 if scheme == "2shoc" else 1.0)
kw = dict(a=0.9, s=-1.1, V=V, bc=bc, scheme=scheme, precision=prec)
t0 = time.time()
ranks = int(os.environ.get("SLABS", "0"))          # > 1: that many virtual slab ranks
if ranks > 1:
    got, info = run_gpu_slabs(dims, h, psi0, k, n, ranks, **kw), {"variant": f"{ranks} virtual slab ranks"}
else:
    got, info = run_gpu(dims, h, psi0, k, n, with_info=True, **kw)
t1 = time.time()
ref = run_oracle(dims, h, psi0, k, n, **kw)
u = ulp_diff(got, ref, prec)
bad = np.argwhere(got != ref)
print(f"{dims} {scheme} {bc} {prec} V={withV} variant={info['variant']} gpu {t1-t0:.2f}s maxulp={u} nbad={len(bad)}",
      "first bad (z,y,x):", bad[:5].tolist() if len(bad) else "-")
