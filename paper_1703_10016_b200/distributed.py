"""Row-block partitioning across GPUs.

Each rank assembles a block of test-function rows with replicated O(N)
inputs -- no communication in the hot loop -- and the collective only
returns the matrix (north_star: "NCCL allgather over NVLink is used only to
return the assembled matrix").

* Closed uniform meshes (configs 2-4): the symmetric assembly computes the
  upper-triangle 64 x 64 tile pairs (I, J >= I); only the upper tile of a
  pair is new data (A is symmetric).  Equal contiguous pair ranges
  (``pair_blocks``: equal work AND equal buffers) are dealt cyclically over
  ranks and chunks; after chunk c each rank packs its upper tiles
  (``wq_pack_pairs``: half the bytes of full rows) and an asynchronous NCCL
  all-gather of chunk c runs while chunk c+1 computes; received tiles are
  written into their rows and, transposed, into their columns
  (``wq_unpack_pairs``) on a side stream, also overlapped (``PackedGather``,
  ``assemble_distributed_pipelined``).
* Other meshes (general path, config 5): cyclic 64-aligned blocks of full
  rows of the unsymmetrised X, in-place all-gather per chunk, then the local
  epilogue A = -(X + X^T)/(4 pi) (``pipeline_rows``).
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


def pair_blocks(n: int, nblocks: int, tile: int = 64):
    """``nblocks`` contiguous ranges [(p0, p1)] of the upper-triangle tile pairs
    (I, J >= I) of an n x n matrix, numbered row by row, as equal as integers
    allow: equal compute for the symmetric assembly and equal packed buffers
    for the all-gather (no padding)."""
    nb = -(-n // tile)
    total = nb * (nb + 1) // 2
    edges = [total * b // nblocks for b in range(nblocks + 1)]
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])]


TILE2 = 64 * 64


class PackedGather:
    """Buffers and schedule of the packed upper-triangle all-gather: block
    b = c * world + r (pair range ``blocks[b]``) is rank r's work in chunk c;
    chunk c's per-rank buffer holds ``sizes[c]`` tiles (its largest block)."""

    def __init__(self, n: int, world: int, chunks: int, new_buffer):
        self.n, self.world, self.chunks = n, world, chunks
        self.blocks = pair_blocks(n, world * chunks)
        self.sizes = [max(1, max(b - a for a, b in self.blocks[c * world:(c + 1) * world]))
                      for c in range(chunks)]
        self.send = [new_buffer(s * TILE2) for s in self.sizes]
        self.recv = [new_buffer(world * s * TILE2) for s in self.sizes]

    def block(self, c: int, r: int):
        return self.blocks[c * self.world + r]

    def recv_bytes(self, itemsize: int = 8) -> int:
        """Bytes one rank receives per assembly (its own blocks excluded)."""
        return sum((self.world - 1) * s * TILE2 for s in self.sizes) * itemsize

    def run(self, rank, compute, pack, unpack, group=None, unpack_ctx=None, marks=None):
        """compute(p0, p1) assembles the pair range into the local matrix (upper
        tiles and their mirrors), pack(p0, p1, buf) packs its upper tiles,
        unpack(p0, p1, buf) writes a received range (tiles and transposes).
        Chunk c's all-gather is asynchronous (overlaps chunk c+1's compute);
        the unpacks run under ``unpack_ctx`` (a side CUDA stream) as each chunk
        lands.  ``marks``: optional callable(name) recording the progress points
        "computed" and "gathered"."""
        import contextlib

        import torch.distributed as dist

        works = []
        for c in range(self.chunks):
            p0, p1 = self.block(c, rank)
            if p1 > p0:
                compute(p0, p1)
                pack(p0, p1, self.send[c])
            works.append(dist.all_gather_into_tensor(self.recv[c], self.send[c], group=group,
                                                     async_op=True))
        if marks:
            marks("computed")
        with (unpack_ctx() if unpack_ctx else contextlib.nullcontext()):
            for c, w in enumerate(works):
                w.wait()
                if marks and c == self.chunks - 1:
                    marks("gathered")
                s = self.sizes[c] * TILE2
                for r in range(self.world):
                    p0, p1 = self.block(c, r)
                    if r != rank and p1 > p0:
                        unpack(p0, p1, self.recv[c][r * s: r * s + (p1 - p0) * TILE2])


def compute_pairs(disc, A, p0: int, p1: int, zext=None):
    """Upper-triangle tile pairs [p0, p1) straight into the full (N, N) device
    buffer A: A(I, J) into rows I, the mirror A(J, I) into rows J."""
    from . import assembly as AS
    from . import _lib
    N = disc.space.dim
    lp, d = AS._logpart_dev(disc)
    sm = AS._smooth(disc)
    st = _lib.stream_handle()
    Zext = AS._zext_table(disc) if zext is None else zext
    _lib.call("wq_ik1_pairs", AS.ctypes_ref(sm["struct"]), p0, p1, _lib.ptr(A), A.stride(0),
              _lib.ptr(sm["flag"]), st)
    _lib.call("wq_x2_pairs_range", N, disc.space.degree, lp.da + 1, lp.nApad, lp.s_w.shape[1],
              lp.uext.shape[1], lp.zstride, _lib.ptr(d["uext"]), _lib.ptr(Zext), _lib.ptr(d["s_w"]),
              -1.0 / (4.0 * np.pi), 2.0, p0, p1, _lib.ptr(A), A.stride(0), st)
    return A


def pack_pairs(A, N: int, p0: int, p1: int, buf):
    from . import _lib
    _lib.call("wq_pack_pairs", _lib.ptr(A), N, A.stride(0), p0, p1, _lib.ptr(buf),
              _lib.stream_handle())


def unpack_pairs(buf, N: int, p0: int, p1: int, A):
    from . import _lib
    _lib.call("wq_unpack_pairs", _lib.ptr(buf), N, p0, p1, _lib.ptr(A), A.stride(0),
              _lib.stream_handle())


_GATHERS = {}


def packed_gather(N: int, world: int, chunks: int):
    """Cached PackedGather with CUDA buffers on the current device."""
    import torch
    key = (torch.cuda.current_device(), N, world, chunks)
    if key not in _GATHERS:
        _GATHERS[key] = PackedGather(N, world, chunks, lambda s: torch.empty(
            s, dtype=torch.float64, device="cuda"))
    return _GATHERS[key]


def assemble_distributed_pipelined(disc, Xpad, chunks: int = 8, group=None, zext=None,
                                   marks=None):
    """A = -(X + X^T)/(4 pi) on every rank.

    Closed uniform meshes: ``Xpad`` is (N, N); packed upper-triangle all-gather
    of equal tile-pair ranges, compute / gather / unpack overlapped
    (``PackedGather``).  Other meshes: ``Xpad`` is (n_pad, N) from
    ``cyclic_blocks(N, world, chunks)``; cyclic row blocks of the unsymmetrised
    X, in-place all-gather per chunk, local symmetrise (A is Xpad[:N]).
    ``marks(name)``: optional progress hook ("computed", "gathered", "done")."""
    import torch
    import torch.distributed as dist
    from . import assembly as AS
    from . import _lib

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    N = disc.space.dim
    if AS._use_v2(disc):
        Z = AS._zext_table(disc) if zext is None else zext
        pg = packed_gather(N, world, chunks)
        main = torch.cuda.current_stream()
        side = AS._aux_stream(torch)
        side.wait_stream(main)
        pg.run(rank, lambda p0, p1: compute_pairs(disc, Xpad, p0, p1, Z),
               lambda p0, p1, buf: pack_pairs(Xpad, N, p0, p1, buf),
               lambda p0, p1, buf: unpack_pairs(buf, N, p0, p1, Xpad),
               group=group, unpack_ctx=lambda: torch.cuda.stream(side), marks=marks)
        main.wait_stream(side)
        if marks:
            marks("done")
        return Xpad[:N]
    F = AS.general_prepare(disc)   # replicated D / F, once per assembly

    def compute(r0, r1, view):
        assemble_rows_device(disc, view, r0, r1, F=F)

    pipeline_rows(N, world, rank, chunks, compute, Xpad, group)
    if marks:
        marks("computed")
        marks("gathered")
    _lib.call("wq_symmetrize", _lib.ptr(Xpad), N, -1.0 / (4.0 * np.pi), _lib.stream_handle())
    if marks:
        marks("done")
    return Xpad[:N]
