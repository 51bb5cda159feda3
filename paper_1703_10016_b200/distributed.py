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


def assemble_rows_device(disc, X_block, row0: int, row1: int, zext=None, F=None):
    """Rows [row0, row1) of the unsymmetrised X = IK1 + X2 into X_block
    (leading dimension N): the circulant fast path's row kernels, or the
    general path's (assembly.general_rows_into).  row0 must be a multiple of
    the 64-row tile; no communication."""
    from . import assembly as AS
    from . import _lib

    if not AS._use_v2(disc):   # general path (open / repeated knots / graded meshes)
        return AS.general_rows_into(disc, X_block, row0, row1, F=F)
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


def cyclic_blocks(n: int, world: int, chunks: int, align: int = 64):
    """Row blocks of ``sub`` rows dealt cyclically: block b = c*world + r is
    computed by rank r as its c-th chunk, so chunk c of every rank fills the
    contiguous rows [c*world*sub, (c+1)*world*sub) -- an in-place all-gather
    target.  Returns (sub, n_pad) with n_pad = chunks*world*sub >= n."""
    sub = -(-n // (world * chunks))
    sub = -(-sub // align) * align
    return sub, chunks * world * sub


def pipeline_rows(n, world, rank, chunks, compute, Xpad, group=None):
    """Compute and all-gather overlapped: for c = 0..chunks-1, ``compute(r0,
    r1, view)`` writes rows [r0, r1) of X (clipped to n) into ``view`` (rows of
    Xpad), then an asynchronous in-place all_gather of chunk c runs on the
    communicator's stream while chunk c+1 computes.  ``Xpad`` is
    (n_pad, ncols) from ``cyclic_blocks``.  Returns after every gather has been
    waited for on the current stream."""
    import torch.distributed as dist

    sub, n_pad = cyclic_blocks(n, world, chunks)
    assert Xpad.shape[0] == n_pad
    works = []
    for c in range(chunks):
        b = c * world + rank
        r0, r1 = b * sub, min((b + 1) * sub, n)
        if r1 > r0:
            compute(r0, r1, Xpad[b * sub: b * sub + (r1 - r0)])
        seg = Xpad[c * world * sub: (c + 1) * world * sub]
        works.append(dist.all_gather_into_tensor(seg, Xpad[b * sub: (b + 1) * sub], group=group,
                                                 async_op=True))
    for w in works:
        w.wait()
    return Xpad


def upper_rows_device(disc, Xfull, row0: int, row1: int, zext=None):
    """Closed uniform meshes: the upper-triangle tile pairs (I, J >= I) of the tile
    rows covering [row0, row1), assembled straight into A (scaled and, inside each
    pair, symmetric) in the full (>= N, N) buffer ``Xfull``: A(I, J) into rows I,
    the mirror A(J, I) into rows J.  Half the arithmetic of the unsymmetrised row
    block; rows J of other ranks are overwritten by their owners' data in the
    all-gather, and ``wq_mirror_upper`` completes the lower triangle afterwards.
    row0 must be a multiple of the 64-row tile; no communication."""
    from . import assembly as AS
    from . import _lib

    T = _lib.WQ_FTILE
    if row0 % T:
        raise ValueError("row blocks must start on a 64-row tile boundary")
    N = disc.space.dim
    nb = -(-N // T)
    start = lambda t: t * nb - t * (t - 1) // 2     # first upper-triangle pair of tile row t
    a, b = start(row0 // T), start(-(-row1 // T))
    lp, d = AS._logpart_dev(disc)
    sm = AS._smooth(disc)
    st = _lib.stream_handle()
    Zext = AS._zext_table(disc) if zext is None else zext
    _lib.call("wq_ik1_pairs", AS.ctypes_ref(sm["struct"]), a, b, _lib.ptr(Xfull), Xfull.stride(0),
              _lib.ptr(sm["flag"]), st)
    _lib.call("wq_x2_pairs_range", N, disc.space.degree, lp.da + 1, lp.nApad, lp.s_w.shape[1],
              lp.uext.shape[1], lp.zstride, _lib.ptr(d["uext"]), _lib.ptr(Zext), _lib.ptr(d["s_w"]),
              -1.0 / (4.0 * np.pi), 2.0, a, b, _lib.ptr(Xfull), Xfull.stride(0), st)
    return Xfull


def assemble_distributed_pipelined(disc, Xpad, chunks: int = 8, group=None, zext=None):
    """A = -(X + X^T)/(4 pi) on every rank with the row-block compute of chunk
    c+1 overlapping the all-gather of chunk c (cyclic 64-aligned row blocks,
    in-place NCCL all-gather, no copies).  Xpad: (n_pad, N) CUDA tensor with
    n_pad from ``cyclic_blocks(N, world, chunks)``; A is Xpad[:N].

    Closed uniform meshes exploit the symmetry: each rank assembles the upper
    tile pairs of its blocks (``upper_rows_device``; cyclic dealing balances
    the triangle), the all-gather returns every rank's rows, and a local
    upper -> lower mirror completes A.  The mirrored tiles a rank writes into
    other ranks' rows never overlap a gather in flight: they land in rows of
    the current or later rounds, whose gathers are ordered after the compute
    that wrote them.  Other meshes assemble unsymmetrised rows of X and
    finish with A = -(X + X^T)/(4 pi)."""
    import torch.distributed as dist
    from . import assembly as AS
    from . import _lib

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    N = disc.space.dim
    v2 = AS._use_v2(disc)
    Z = (AS._zext_table(disc) if zext is None else zext) if v2 else None
    F = None if v2 else AS.general_prepare(disc)   # replicated D / F, once per assembly

    def compute(r0, r1, view):
        if v2:
            upper_rows_device(disc, Xpad, r0, r1, zext=Z)
        else:
            assemble_rows_device(disc, view, r0, r1, zext=Z, F=F)

    pipeline_rows(N, world, rank, chunks, compute, Xpad, group)
    if v2:
        _lib.call("wq_mirror_upper", _lib.ptr(Xpad), N, Xpad.stride(0), _lib.stream_handle())
    else:
        _lib.call("wq_symmetrize", _lib.ptr(Xpad), N, -1.0 / (4.0 * np.pi), _lib.stream_handle())
    return Xpad[:N]


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
