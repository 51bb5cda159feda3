"""Row-block partitioning across GPUs.

Each rank assembles a contiguous block of test-function rows of
X = IK1 + X2 with replicated O(N) inputs -- no communication in the hot
loop.  One all-gather returns the full X to every rank, after which a local
epilogue forms A = -(X + X^T)/(4 pi).  The collective only returns the
matrix (north_star: "NCCL allgather over NVLink is used only to return the
assembled matrix").
"""

from __future__ import annotations

import numpy as np


def row_blocks(n: int, world: int, align: int = 32):
    """Contiguous [r0, r1) per rank, sizes multiples of ``align`` except the
    last, covering 0..n exactly (equal-size blocks -> all_gather needs
    equal shards, so shards are padded to the max block)."""
    per = -(-n // world)
    per = -(-per // align) * align
    bounds = []
    for r in range(world):
        r0 = min(r * per, n)
        r1 = min(r0 + per, n)
        bounds.append((r0, r1))
    return bounds, per


def gather_rows(local_block, full, per, group=None):
    """All-gather equal-height row shards into ``full`` (rows >= n dropped).

    ``local_block`` is (per, n); ``full`` is (n, n).  Works for NCCL (CUDA
    tensors) and gloo (CPU tensors)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n = full.shape[0]
    if per * world == n:
        dist.all_gather_into_tensor(full, local_block, group=group)
        return full
    buf = torch.empty((per * world, full.shape[1]), dtype=full.dtype, device=full.device)
    dist.all_gather_into_tensor(buf, local_block, group=group)
    full.copy_(buf[:n])
    return full


def assemble_rows_device(disc, X_block, row0: int, row1: int):
    """Rows [row0, row1) of X = IK1 + X2 into X_block (shape (row1-row0, N)),
    circulant path (closed uniform simple-knot meshes)."""
    from . import assembly as AS
    from . import _lib

    lp, d = AS._logpart_dev(disc)
    if lp.path != "circulant":
        raise NotImplementedError("row-block sharding needs the circulant log-part path")
    AS._ik1_into(disc, X_block, accumulate=False, row0=row0, row1=row1)
    AS._ik2_x2_rows(disc, X_block, row0, row1, accumulate=True)
    return X_block
