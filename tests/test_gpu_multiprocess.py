"""The real slab-mode path (one process per rank, CUDA IPC peer mappings, handle
all-gather over torch.distributed, cross-process device barriers) on the one GPU this
run has: two or three processes all on cuda:0.  Processes on one GPU time-slice, so the
per-stage barriers are slow here, but every code path the 8-GPU run uses is exercised:
nlse_create_dist / nlse_dist_export / dist.connect / nlse_dist_connect, remote stores into
IPC-mapped ghost planes, st.release.sys / ld.acquire.sys flags, diagnostics exchange.
The bar: bitwise equal to the single-context run (itself bitwise equal to the oracle)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from helpers import case_input, run_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, h, k, nsteps, scheme, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)   # bootstrap only
    try:
        from helpers import case_input as ci
        from paper_1203_1263_b200 import dist as pdist
        from paper_1203_1263_b200.nlse import Solver
        psi0 = ci(dims, seed=77)
        with Solver(dims, h, s=-1.0, bc="msd", scheme=scheme, force_dt=True, dist=(rank, world)) as sv:
            pdist.connect(sv)
            sv.nlse_set_psi(np.ascontiguousarray(psi0[sv.z0:sv.z0 + sv.shape[0]]))
            sv.nlse_step(k, nsteps)
            out = sv.nlse_get_psi()
            m, e = sv.nlse_diagnostics()
            q.put((rank, sv.z0, out, m, e))
        dist.barrier()
    except Exception as ex:  # report instead of hanging the parent
        q.put((rank, -1, repr(ex), 0.0, 0.0))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,scheme,dims", [(2, "2shoc", (40, 24, 21)), (3, "cd", (40, 24, 21)),
                                               (2, "2shoc", (70, 45)), (3, "cd", (50, 31))])
def test_multiprocess_slabs_bitwise(world, scheme, dims):
    h, nsteps = 0.5, 5
    k = 0.5 * h * h / (len(dims) * 2 ** 0.5) * (0.75 if scheme == "2shoc" else 1.0)
    psi0 = case_input(dims, seed=77)
    one = run_gpu(dims, h, psi0, k, nsteps, s=-1.0, bc="msd", scheme=scheme)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, h, k, nsteps, scheme, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=500) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] >= 0, f"rank {r[0]} failed: {r[2]}"
    got = np.concatenate([r[2] for r in res], axis=0)
    assert got.shape == one.shape
    assert np.array_equal(got.view(np.uint64), one.view(np.uint64))
    ms = {r[3] for r in res}
    es = {r[4] for r in res}
    assert len(ms) == 1 and len(es) == 1          # every rank holds the same global sums


def _stall_worker(rank, world, port, mode, q):
    """Rank 0 steps; rank 1 never steps (mode "late": it only waits, so rank 0's neighbour
    barrier must time out) or calls nlse_dist_abort while rank 0 waits (mode "abort")."""
    import sys
    import time
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), NLSE_BARRIER_TIMEOUT_S="3")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from helpers import case_input as ci
        from paper_1203_1263_b200 import dist as pdist
        from paper_1203_1263_b200.nlse import NLSEError, Solver
        dims, h = (24, 20, 16), 0.5
        psi0 = ci(dims, seed=5)
        with Solver(dims, h, s=-1.0, bc="msd", force_dt=True, dist=(rank, world)) as sv:
            pdist.connect(sv)
            dist.barrier()
            if rank == 0:
                t0 = time.time()
                try:
                    sv.nlse_set_psi(np.ascontiguousarray(psi0[sv.z0:sv.z0 + sv.shape[0]]))
                    sv.nlse_step(0.01, 3)
                    q.put((rank, "no error", time.time() - t0))
                except NLSEError as e:
                    q.put((rank, f"status {e.status}: {e}", time.time() - t0))
            else:
                time.sleep(1.0)
                if mode == "abort":
                    sv.nlse_dist_abort()
                q.put((rank, "idle", 0.0))
            dist.barrier()      # keep every rank's memory mapped until rank 0 has returned
    except Exception as ex:
        q.put((rank, repr(ex), -1.0))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("mode", ["late", "abort"])
def test_barrier_timeout_and_abort_report_comm_error(mode):
    """A rank whose neighbour never arrives does not hang: its device barrier gives up after
    NLSE_BARRIER_TIMEOUT_S (or as soon as the neighbour calls nlse_dist_abort) and nlse_step
    returns NLSE_ERR_COMM (5)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stall_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (msg, t)) for r, msg, t in (q.get(timeout=240) for _ in procs))
    for p in procs:
        p.join(timeout=60)
    msg, t = res[0]
    assert msg.startswith("status 5"), res
    if mode == "late":
        assert "timed out" in msg and 2.5 < t < 60, res
    else:
        assert "abort" in msg and t < 30, res
