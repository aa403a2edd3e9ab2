"""Host side of slab mode, multi-process on CPU (gloo, world size 2 and 3): the balanced
slab split, the handle all-gather of dist.py, and per-rank input generation that
tiles the global initial condition exactly.  The device side (remote stores, barriers)
is covered on the GPU by tests/test_gpu_slabs.py (virtual ranks)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1203_1263_b200 import dist as pdist, inputs
        res = {}
        # 1. slab split agrees across ranks and tiles [0, nz)
        for nz in (1024, 203, 29, 8):
            z0, nl = pdist.slab_planes(nz, world, rank)
            allr = [None] * world
            dist.all_gather_object(allr, (z0, nl))
            res[f"split{nz}"] = allr
        # 2. handle exchange: fixed-size blobs, rank order
        mine = bytes([rank + 1]) * pdist.HANDLE_BYTES
        hs = pdist.gather_handles(mine)
        res["handles_ok"] = all(h == bytes([j + 1]) * pdist.HANDLE_BYTES for j, h in enumerate(hs))
        try:
            pdist.gather_handles(b"short")
            res["short_rejected"] = False
        except ValueError:
            res["short_rejected"] = True
        # 3. per-rank slab of the GPE workload IC
        n = 16
        z0, nl = pdist.slab_planes(n, world, rank)
        psi, V = inputs.gpe3d_slab(n, z0, z0 + nl, h=0.25 * 1024 / n / 8)
        res["slab"] = (z0, psi, V)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_bootstrap_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for nz in (1024, 203, 29, 8):
        splits = out[0][f"split{nz}"]
        assert all(out[r][f"split{nz}"] == splits for r in range(world))
        assert splits[0][0] == 0
        for r in range(world - 1):
            assert splits[r][0] + splits[r][1] == splits[r + 1][0]
        assert splits[-1][0] + splits[-1][1] == nz
        assert max(s[1] for s in splits) - min(s[1] for s in splits) <= 1
    assert all(out[r]["handles_ok"] and out[r]["short_rejected"] for r in range(world))
    from paper_1203_1263_b200 import inputs
    n = 16
    full_psi, full_V = inputs.gpe3d_slab(n, 0, n, h=0.25 * 1024 / n / 8)
    got_psi = np.concatenate([out[r]["slab"][1] for r in range(world)])
    got_V = np.concatenate([out[r]["slab"][2] for r in range(world)])
    assert np.array_equal(got_psi, full_psi) and np.array_equal(got_V, full_V)
