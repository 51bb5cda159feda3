"""CPU (gloo, world_size 2): the multi-GPU plumbing -- row-block partition,
equal-shard all-gather, and the local symmetrise epilogue -- on CPU tensors.
The row-block kernels themselves are checked on one GPU in
test_gpu_parity.py::test_row_blocks_match_full (same code path, ranks
emulated sequentially)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1703_10016_b200.distributed import cyclic_blocks, gather_rows, pipeline_rows, row_blocks


def free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


@pytest.mark.parametrize("n,world", [(1, 1), (64, 2), (130, 2), (32768, 8), (4096, 3), (65, 8)])
def test_row_blocks_cover_exactly(n, world):
    bounds, per = row_blocks(n, world)
    assert per % 64 == 0
    covered = np.zeros(n, int)
    for r0, r1 in bounds:
        assert r0 % 64 == 0 or r0 == n
        assert r1 - r0 <= per
        covered[r0:r1] += 1
    assert np.all(covered == 1)


def _worker(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bounds, per = row_blocks(n, world)
    r0, r1 = bounds[rank]
    i = torch.arange(n, dtype=torch.float64)
    Xfull = torch.sin(i[:, None] * 0.37 + i[None, :] ** 1.3 * 0.011)  # deterministic, asymmetric
    block = torch.zeros((per, n), dtype=torch.float64)
    block[: r1 - r0] = Xfull[r0:r1]
    X = torch.empty((n, n), dtype=torch.float64)
    gather_rows(block, X, per)
    A = -(X + X.T) / (4 * np.pi)
    ok = torch.equal(X, Xfull) and torch.allclose(A, -(Xfull + Xfull.T) / (4 * np.pi), rtol=0, atol=0)
    out[rank] = int(ok)
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [130, 256])
def test_gloo_allgather_assembles_full_matrix(n):
    world = 2
    port = free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, n, out), nprocs=world, join=True)
    assert dict(out) == {0: 1, 1: 1}


@pytest.mark.parametrize("n,world,chunks", [(130, 2, 3), (4096, 8, 8), (32768, 8, 8), (65, 3, 2)])
def test_cyclic_blocks_cover_exactly(n, world, chunks):
    sub, n_pad = cyclic_blocks(n, world, chunks)
    assert sub % 64 == 0 and n_pad >= n and n_pad == chunks * world * sub
    owner = np.full(n_pad, -1)
    for r in range(world):
        for c in range(chunks):
            b = c * world + r
            owner[b * sub:(b + 1) * sub] = r
    assert np.all(owner >= 0)


def _pipe_worker(rank, world, port, n, chunks, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sub, n_pad = cyclic_blocks(n, world, chunks)
    i = torch.arange(n, dtype=torch.float64)
    Xfull = torch.sin(i[:, None] * 0.37 + i[None, :] ** 1.3 * 0.011)
    Xpad = torch.full((n_pad, n), float("nan"), dtype=torch.float64)
    seen = []

    def compute(r0, r1, view):
        seen.append((r0, r1))
        view.copy_(Xfull[r0:r1])

    pipeline_rows(n, world, rank, chunks, compute, Xpad)
    ok = torch.equal(Xpad[:n], Xfull) and all((r0 // sub) % world == rank for r0, _ in seen)
    out[rank] = int(ok)
    dist.destroy_process_group()


@pytest.mark.parametrize("n,chunks", [(130, 3), (300, 2)])
def test_gloo_pipelined_allgather(n, chunks):
    world = 2
    port = free_port()
    out = mp.Manager().dict()
    mp.spawn(_pipe_worker, args=(world, port, n, chunks, out), nprocs=world, join=True)
    assert dict(out) == {0: 1, 1: 1}


def test_bench_spawns_one_rank_per_gpu():
    """bench.py --gpus 2 without a launcher re-runs itself under torchrun with
    two ranks (127.0.0.1 rendezvous) and checks WORLD_SIZE == --gpus (CPU:
    --launcher-check joins a gloo group and all-reduces the rank ids)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                          "--launcher-check"], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line == {"launcher": "ok", "world": 2, "rank_sum": 3.0}
    # a mismatched launch fails loudly
    env["WORLD_SIZE"] = "1"
    bad = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                          "--launcher-check"], capture_output=True, text=True, timeout=120, env=env)
    assert bad.returncode != 0


@pytest.mark.parametrize("n,world,chunks", [(1, 1, 1), (130, 2, 3), (32768, 8, 4), (4096, 3, 5),
                                            (65, 8, 2)])
def test_pair_blocks_equal_and_cover(n, world, chunks):
    from paper_1703_10016_b200.distributed import pair_blocks
    nb = -(-n // 64)
    blocks = pair_blocks(n, world * chunks)
    sizes = [b - a for a, b in blocks]
    assert blocks[0][0] == 0 and blocks[-1][1] == nb * (nb + 1) // 2
    assert all(blocks[k][1] == blocks[k + 1][0] for k in range(len(blocks) - 1))
    assert max(sizes) - min(sizes) <= 1


def _packed_worker(rank, world, port, n, chunks, out):
    """PackedGather with CPU stand-ins for the kernels: compute writes the upper
    tiles of its pair ranges and their mirrors, pack / unpack move upper tiles
    tile-major (the layout of wq_pack_pairs / wq_unpack_pairs)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1703_10016_b200.distributed import PackedGather
    i = torch.arange(n, dtype=torch.float64)
    S = torch.sin(i[:, None] * 0.37 + i[None, :] ** 1.3 * 0.011)
    S = S + S.T                                    # the symmetric result
    nb = -(-n // 64)
    pairs = [(a, b) for a in range(nb) for b in range(a, nb)]
    A = torch.full((n, n), float("nan"), dtype=torch.float64)
    computed = []

    def tile(a, b):
        return slice(64 * a, min(n, 64 * a + 64)), slice(64 * b, min(n, 64 * b + 64))

    def compute(p0, p1):
        computed.append((p0, p1))
        for p in range(p0, p1):
            a, b = pairs[p]
            A[tile(a, b)] = S[tile(a, b)]
            A[tile(b, a)] = S[tile(b, a)]

    def pack(p0, p1, buf):
        for k, p in enumerate(range(p0, p1)):
            a, b = pairs[p]
            t = A[tile(a, b)]
            v = buf[k * 4096:(k + 1) * 4096].view(64, 64)
            v[: t.shape[0], : t.shape[1]] = t

    def unpack(p0, p1, buf):
        for k, p in enumerate(range(p0, p1)):
            a, b = pairs[p]
            v = buf[k * 4096:(k + 1) * 4096].view(64, 64)
            ra, cb = tile(a, b)
            t = v[: ra.stop - ra.start, : cb.stop - cb.start]
            A[ra, cb] = t
            A[cb, ra] = t.T

    pg = PackedGather(n, world, chunks, lambda s: torch.zeros(s, dtype=torch.float64))
    pg.run(rank, compute, pack, unpack)
    ok = torch.equal(A, S) and all(pg.block(c, rank) == computed[k]
                                   for k, c in enumerate(c for c in range(chunks)
                                                         if pg.block(c, rank)[1] > pg.block(c, rank)[0]))
    full = (world - 1) * n * n * 8 // world
    out[rank] = (int(ok), pg.recv_bytes(), full)
    dist.destroy_process_group()


@pytest.mark.parametrize("n,chunks", [(130, 2), (300, 3), (256, 1)])
def test_gloo_packed_upper_allgather(n, chunks):
    world = 2
    port = free_port()
    out = mp.Manager().dict()
    mp.spawn(_packed_worker, args=(world, port, n, chunks, out), nprocs=world, join=True)
    res = dict(out)
    assert all(res[r][0] == 1 for r in range(world)), res


def test_packed_gather_halves_nvlink_bytes_at_config4():
    """Received bytes per rank at C4 (N = 32768), P = 8: the packed upper tiles
    (<= 3.8 GB) against 7.5 GB for full rows."""
    from paper_1703_10016_b200.distributed import PackedGather
    pg = PackedGather(32768, 8, 4, lambda s: None)
    assert pg.recv_bytes() <= 3.8e9
    assert pg.recv_bytes() < 0.52 * 7 * 32768 ** 2 * 8 / 8
