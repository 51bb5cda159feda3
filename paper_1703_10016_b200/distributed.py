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


def row_blocks(n: int, world: int, align: int = 64):
    """Contiguous [r0, r1) per rank covering 0..n, block starts aligned to
    ``align`` rows (the kernels' tile height) and equal padded height ``per``
    (all_gather needs equal shards)."""
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


def assemble_rows_device(disc, X_block, row0: int, row1: int, zext=None):
    """Rows [row0, row1) of the unsymmetrised X = IK1 + X2 into X_block
    (leading dimension N), circulant path (closed uniform simple-knot meshes).
    row0 must be a multiple of the 64-row tile; no communication."""
    from . import assembly as AS
    from . import _lib

    if not AS._use_v2(disc):
        raise NotImplementedError("row-block sharding needs the circulant (closed uniform) path")
    T = _lib.WQ_FTILE
    if row0 % T:
        raise ValueError("row blocks must start on a 64-row tile boundary")
    t0, t1 = row0 // T, -(-row1 // T)
    lp, d = AS._logpart_dev(disc)
    sm = AS._smooth(disc)
    st = _lib.stream_handle()
    Zext = AS._zext_table(disc) if zext is None else zext
    N = disc.space.dim
    _lib.call("wq_ik1_rows", AS.ctypes_ref(sm["struct"]), t0, t1, _lib.ptr(X_block),
              X_block.stride(0), _lib.ptr(sm["flag"]), st)
    _lib.call("wq_x2_rows", N, disc.space.degree, lp.da + 1, lp.nApad, lp.s_w.shape[1],
              lp.uext.shape[1], lp.zstride, _lib.ptr(d["uext"]), _lib.ptr(Zext), _lib.ptr(d["s_w"]),
              1.0, 1.0, t0, t1, _lib.ptr(X_block), X_block.stride(0), st)
    return X_block


def assemble_distributed(disc, X, group=None):
    """A = -(X + X^T)/(4 pi) on every rank: local row block, one all-gather,
    local symmetrise epilogue.  X: (N, N) CUDA tensor on this rank."""
    import torch
    import torch.distributed as dist
    from . import _lib

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    N = disc.space.dim
    bounds, per = row_blocks(N, world)
    r0, r1 = bounds[rank]
    Xb = torch.zeros((per, N), dtype=torch.float64, device=X.device)
    if r1 > r0:
        assemble_rows_device(disc, Xb, r0, r1)
    gather_rows(Xb, X, per, group)
    _lib.call("wq_symmetrize", _lib.ptr(X), N, -1.0 / (4.0 * np.pi), _lib.stream_handle())
    return X
