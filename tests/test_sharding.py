"""Multi-GPU host logic on CPU (gloo, world_size 2): row sharding plan and the
exact integer all-reduce of packed partial accumulators."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2204_05496_b200.sharding import combine_partials, packed_count, reduce_packed_mod_q, shard_rows


@pytest.mark.parametrize("R,world", [(1, 1), (256, 2), (256, 8), (7, 3), (4096, 8), (3, 8)])
def test_shard_rows_cover_exactly_once(R, world):
    seen = np.zeros(R, dtype=int)
    for r in range(world):
        lo, cnt = shard_rows(R, world, r)
        seen[lo:lo + cnt] += 1
    assert (seen == 1).all()


def test_packed_count_matches_reference_layout():
    assert packed_count(256, 11, 8192) == 1  # C4: 2816 results in 1 ciphertext
    assert packed_count(4096, 33, 16384) == 9  # C5
    assert packed_count(9, 3, 8) == 4  # test_matmul.cpp:108-126


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(100 + rank)
    # a rank's partial: sums of up to 2816 residues < 2^31 per slot
    part = rng.integers(0, 2 ** 43, size=(1, len(q), 64), dtype=np.int64)
    t = torch.from_numpy(part.copy())
    combine_partials(t)
    if rank == 0:
        np.save(result_path, t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_all_reduce_of_partials_is_exact(tmp_path):
    world = 2
    q = np.array([2147352577, 2147205121, 114689 * 0 + 2147074049], dtype=np.uint64)
    path = str(tmp_path / "sum.npy")
    mp.spawn(_worker, args=(world, _free_port(), q, path), nprocs=world, join=True)
    got = np.load(path).astype(np.uint64)
    want = sum(np.random.default_rng(100 + r).integers(0, 2 ** 43, size=(1, len(q), 64), dtype=np.int64).astype(np.uint64)
               for r in range(world))
    assert np.array_equal(got, want)
    # reduction order is irrelevant mod q: (sum of partials) mod q == sum of (partial mod q) mod q
    parts = [np.random.default_rng(100 + r).integers(0, 2 ** 43, size=(1, len(q), 64), dtype=np.int64).astype(np.uint64)
             for r in range(world)]
    a = reduce_packed_mod_q(got, q)
    b = reduce_packed_mod_q(sum(reduce_packed_mod_q(p, q) for p in parts), q)
    assert np.array_equal(a, b)


def _fb_worker(rank, world, port, total_rows, result_path):
    import torch
    import torch.distributed as dist

    from paper_2204_05496_b200.sharding import reduce_scatter_dots

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cols, ct = 3, 8
    rng = np.random.default_rng(200 + rank)
    part = rng.integers(0, 2 ** 31, size=(total_rows * cols, ct), dtype=np.int64)  # one rank's chunk products
    got = reduce_scatter_dots(torch.from_numpy(part), total_rows)
    np.save(result_path % rank, got.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total_rows", [5, 8])
def test_gloo_feature_block_reduce_scatter_is_exact(tmp_path, total_rows):
    """Feature-block sharding's exchange: every rank receives exactly the sum
    of all ranks' dot partials for its own row block (shard_rows), ragged
    row counts included."""
    from paper_2204_05496_b200.sharding import shard_chunks, shard_rows

    world, cols, ct = 2, 3, 8
    path = str(tmp_path / "rs_%d.npy")
    mp.spawn(_fb_worker, args=(world, _free_port(), total_rows, path), nprocs=world, join=True)
    total = sum(np.random.default_rng(200 + r).integers(0, 2 ** 31, size=(total_rows * cols, ct), dtype=np.int64)
                for r in range(world))
    for r in range(world):
        lo, cnt = shard_rows(total_rows, world, r)
        assert np.array_equal(np.load(path % r), total[lo * cols:(lo + cnt) * cols])
    # chunk blocks partition the chunks exactly once
    for kc in (1, 3, 5):
        seen = []
        for r in range(world):
            lo, cnt = shard_chunks(kc, world, r)
            seen += list(range(lo, lo + cnt))
        assert seen == list(range(kc))


def _ex_worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    from paper_2204_05496_b200.sharding import exchange_partials

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(300 + rank)
    part = rng.integers(0, 2 ** 31 - 1, size=(2, 5, 16), dtype=np.int64).astype(np.int32)  # u32 residues < 2^31
    got = exchange_partials(torch.from_numpy(part))
    np.save(result_path % rank, got.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_exchange_of_reduced_partials(tmp_path, world):
    """Row sharding's exchange: each rank's packed partial is
    reduced mod q to u32 and all-gathered; every rank receives every partial in
    rank order, and summing them mod q equals reducing the sum of the
    unreduced u64 partials (mod-q addition is order-free)."""
    path = str(tmp_path / "ex_%d.npy")
    mp.spawn(_ex_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    parts = [np.random.default_rng(300 + r).integers(0, 2 ** 31 - 1, size=(2, 5, 16), dtype=np.int64) for r in range(world)]
    for r in range(world):
        got = np.load(path % r).astype(np.int64)
        assert got.shape == (world, 2, 5, 16)
        for k in range(world):
            assert np.array_equal(got[k], parts[k])
    q = np.array([2147352577, 2147205121, 2147074049, 2146959361, 2146713601], dtype=np.uint64)
    total = sum(p.astype(np.uint64) for p in parts)
    via_parts = sum(reduce_packed_mod_q(p.astype(np.uint64), q) for p in parts)
    assert np.array_equal(reduce_packed_mod_q(total, q), reduce_packed_mod_q(via_parts, q))
