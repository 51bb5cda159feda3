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
    port = 29500 + (os.getpid() % 2000)
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
    port = 31500 + (os.getpid() % 2000)
    out = mp.Manager().dict()
    mp.spawn(_pipe_worker, args=(world, port, n, chunks, out), nprocs=world, join=True)
    assert dict(out) == {0: 1, 1: 1}
