"""Slab-mode bootstrap over torch.distributed (plumbing only).

One process per GPU: every rank creates its slab context (``Solver(..., dist=(rank,
nranks))``), exports its handle (CUDA IPC handles of its halo'd buffers and comm
block, ``nlse_dist_export``), the handles are all-gathered over the process group,
and each rank maps its peers (``nlse_dist_connect``).  The halo exchange and the
per-stage barriers then run entirely on the devices (comm.cuh): torch.distributed
is used once, here, and never on the step path.
"""
from __future__ import annotations

HANDLE_BYTES = 512   # NLSE_DIST_HANDLE_BYTES


def gather_handles(local: bytes, group=None) -> list:
    """All-gather one fixed-size handle per rank, returned in rank order."""
    import torch.distributed as dist
    if len(local) != HANDLE_BYTES:
        raise ValueError(f"handle must be {HANDLE_BYTES} bytes, got {len(local)}")
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(local), group=group)
    for j, h in enumerate(out):
        if not isinstance(h, (bytes, bytearray)) or len(h) != HANDLE_BYTES:
            raise RuntimeError(f"rank {j} sent a malformed handle")
    return out


def connect(solver, group=None) -> None:
    """Map this rank's slab context to its peers (collective over `group`)."""
    solver.nlse_dist_connect(gather_handles(solver.nlse_dist_export(), group))


def slab_planes(nz: int, nranks: int, rank: int):
    """(z0, nloc) of nlse_slab_range, as a python range helper for input generation."""
    from .nlse import nlse_slab_range
    return nlse_slab_range(nz, nranks, rank)
