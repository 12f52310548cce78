"""Multi-rank exchange over peer memory (CUDA IPC), two processes on one GPU.

Each rank encrypts and processes its own rows into its own packed
accumulator, writes it into its slot of rank 0's receive buffer through the
IPC mapping (on a multi-GPU box: an NVLink peer write), and rank 0 sums the
slots, finishes and decrypts. The kernels of the two ranks never wait on each other — only host
barriers order the phases — so this checks the plumbing and the exactness of
the exchange, not multi-GPU performance.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, rows_per_rank, result_path):
    import torch
    import torch.distributed as dist

    from oracle.oracle import production_params
    from paper_2204_05496_b200 import (GpuTwinServer, Prng, ScalingConfig, default_q_primes, encode_inputs_device,
                                       encode_weights)
    from paper_2204_05496_b200.sharding import PeerGather, finish_packed_device, matmul_partial_device, packed_count
    from tests.helpers import synthetic

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    p = production_params(8192)
    q = default_q_primes(8192, p.t0) + default_q_primes(8192, p.t1)
    srv = GpuTwinServer(8192, (p.t0, p.t1), (6, 4), np.array(q, np.uint64), [], None, ScalingConfig())
    srv.keygen(Prng(1))  # deterministic: the same keys on every rank
    total = world * rows_per_rank
    x_all, w, b = synthetic(total, 2000, 11, 0.05, 0.1, seed=5)
    x = x_all[rank * rows_per_rank:(rank + 1) * rows_per_rank]
    ctw = srv.ct_words
    d_in = torch.empty((rows_per_rank, ctw), dtype=torch.int32, device="cuda")
    encode_inputs_device(srv, x, Prng(2 + 2 * rank), Prng(3 + 2 * rank), d_in.data_ptr(), 0)
    ew = encode_weights(srv, w)
    Ct = packed_count(total, 11, 8192)
    gather = PeerGather(Ct * ctw * 8, 0)
    acc = torch.zeros((Ct, ctw), dtype=torch.int64, device="cuda")
    matmul_partial_device(srv, ew, d_in.data_ptr(), rows_per_rank, rank * rows_per_rank, total, acc.data_ptr())
    gather.push(acc.data_ptr())
    torch.cuda.synchronize()
    dist.barrier()  # every rank's slot is written
    if rank == 0:
        gather.reduce()
        out = torch.empty((Ct, ctw), dtype=torch.int32, device="cuda")
        finish_packed_device(srv, ew, gather.total_ptr, b, total, out.data_ptr())
        packed = out.cpu().numpy().view(np.uint32).astype(np.uint64)
        np.save(result_path, srv.unpack_results(packed, total, 11))
    dist.barrier()
    gather.close()
    dist.destroy_process_group()


def test_peer_memory_exchange_two_ranks(tmp_path):
    from tests.helpers import oracle_matmul, synthetic

    world, rows = 2, 3
    path = str(tmp_path / "p2p.npy")
    mp.spawn(_worker, args=(world, _free_port(), rows, path), nprocs=world, join=True)
    x_all, w, b = synthetic(world * rows, 2000, 11, 0.05, 0.1, seed=5)
    assert np.array_equal(np.load(path), oracle_matmul(x_all, w, b))


def _fb_gpu_worker(rank, world, port, result_path):
    """Feature-block sharding through torch.distributed (gloo: host-side
    exchange; the two ranks share one GPU, and no kernel waits on the other
    rank): chunk-product partials reduce-scattered by rows, fold + mask of
    the rank's row block, u32 partials all-gathered, rank 0 finishes."""
    import torch
    import torch.distributed as dist

    from oracle.oracle import production_params
    from paper_2204_05496_b200 import (GpuTwinServer, Prng, ScalingConfig, default_q_primes, encode_inputs_device,
                                       encode_weights, matmul_device)
    from paper_2204_05496_b200.sharding import (chunk_dot_partial_device, exchange_partials, finish_parts_device,
                                                fold_pack_device, packed_count, reduce_packed_device,
                                                reduce_scatter_dots, shard_chunks, shard_rows)
    from paper_2204_05496_b200.workload import workload

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    p = production_params(8192)
    q = default_q_primes(8192, p.t0) + default_q_primes(8192, p.t1)
    srv = GpuTwinServer(8192, (p.t0, p.t1), (6, 4), np.array(q, np.uint64), [], None, ScalingConfig())
    srv.keygen(Prng(1))
    R, f, cols = 5, 20000, 4  # 3 chunks per row
    x, w, b = workload(R, f, cols, 0.03, 0.05, seed=9)
    kc, ctw = srv.chunks(f), srv.ct_words
    d_all = torch.empty((R * kc, ctw), dtype=torch.int32, device="cuda")
    encode_inputs_device(srv, x, Prng(2), Prng(3), d_all.data_ptr(), 0)
    torch.cuda.synchronize()
    klo, kn = shard_chunks(kc, world, rank)
    d_in = d_all.view(R, kc, ctw)[:, klo:klo + kn].contiguous()  # this rank holds only its feature block
    ew = encode_weights(srv, w)
    dot = torch.zeros((R * cols, ctw), dtype=torch.int64, device="cuda")
    chunk_dot_partial_device(srv, ew, d_in.data_ptr(), R, klo, kn, dot.data_ptr())
    mine = reduce_scatter_dots(dot, R)
    Ct = packed_count(R, cols, 8192)
    acc = torch.zeros((Ct, ctw), dtype=torch.int64, device="cuda")
    lo, cnt = shard_rows(R, world, rank)
    fold_pack_device(srv, ew, mine.data_ptr(), lo, cnt, R, acc.data_ptr())
    part = torch.empty((Ct, ctw), dtype=torch.int32, device="cuda")
    reduce_packed_device(srv, acc.data_ptr(), Ct, part.data_ptr())
    gathered = exchange_partials(part)
    if rank == 0:
        out = torch.empty((Ct, ctw), dtype=torch.int32, device="cuda")
        finish_parts_device(srv, ew, gathered.data_ptr(), world, b, R, out.data_ptr())
        one = torch.empty((Ct, ctw), dtype=torch.int32, device="cuda")
        matmul_device(srv, d_all.data_ptr(), R, ew, b, one.data_ptr())  # the single-GPU result
        torch.cuda.synchronize()
        packed = out.cpu().numpy().view(np.uint32).astype(np.uint64)
        np.save(result_path, np.stack([packed, one.cpu().numpy().view(np.uint32).astype(np.uint64)]))
        np.save(result_path + ".dec.npy", srv.unpack_results(packed, R, cols))
    dist.barrier()
    dist.destroy_process_group()


def test_feature_block_exchange_two_ranks(tmp_path):
    from paper_2204_05496_b200.workload import workload

    path = str(tmp_path / "fb.npy")
    mp.spawn(_fb_gpu_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    both = np.load(path)
    assert np.array_equal(both[0], both[1]), "feature-sharded result differs from the single-GPU bytes"
    x, w, b = workload(5, 20000, 4, 0.03, 0.05, seed=9)
    assert np.array_equal(np.load(path + ".dec.npy"), x @ w + b)


def _rows_worker(rank, world, port, result_path):
    """Row sharding with the stream-ordered exchange: each
    rank's packed partial reduced mod q to u32 (reduce_packed_device),
    all-gathered (gloo here: host-side; NCCL on a multi-GPU box), and rank 0
    sums the partials mod q and adds the bias (finish_parts_device)."""
    import torch
    import torch.distributed as dist

    from oracle.oracle import production_params
    from paper_2204_05496_b200 import (GpuTwinServer, Prng, ScalingConfig, default_q_primes, encode_inputs_device,
                                       encode_weights, matmul_device)
    from paper_2204_05496_b200.sharding import (exchange_partials, finish_parts_device, matmul_partial_device,
                                                packed_count, reduce_packed_device, shard_rows)
    from paper_2204_05496_b200.workload import workload

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    p = production_params(8192)
    q = default_q_primes(8192, p.t0) + default_q_primes(8192, p.t1)
    srv = GpuTwinServer(8192, (p.t0, p.t1), (6, 4), np.array(q, np.uint64), [], None, ScalingConfig())
    srv.keygen(Prng(1))
    R, f, cols = 7, 9000, 11
    x, w, b = workload(R, f, cols, 0.05, 0.1, seed=8)
    kc, ctw = srv.chunks(f), srv.ct_words
    d_all = torch.empty((R * kc, ctw), dtype=torch.int32, device="cuda")
    encode_inputs_device(srv, x, Prng(2), Prng(3), d_all.data_ptr(), 0)
    torch.cuda.synchronize()
    lo, cnt = shard_rows(R, world, rank)
    ew = encode_weights(srv, w)
    Ct = packed_count(R, cols, 8192)
    acc = torch.zeros((Ct, ctw), dtype=torch.int64, device="cuda")
    matmul_partial_device(srv, ew, d_all[lo * kc:(lo + cnt) * kc].data_ptr(), cnt, lo, R, acc.data_ptr())
    part = torch.empty((Ct, ctw), dtype=torch.int32, device="cuda")
    reduce_packed_device(srv, acc.data_ptr(), Ct, part.data_ptr())
    gathered = exchange_partials(part)
    if rank == 0:
        out = torch.empty((Ct, ctw), dtype=torch.int32, device="cuda")
        finish_parts_device(srv, ew, gathered.data_ptr(), world, b, R, out.data_ptr())
        one = torch.empty((Ct, ctw), dtype=torch.int32, device="cuda")
        matmul_device(srv, d_all.data_ptr(), R, ew, b, one.data_ptr())
        torch.cuda.synchronize()
        np.save(result_path, np.stack([out.cpu().numpy(), one.cpu().numpy()]))
    dist.barrier()
    dist.destroy_process_group()


def test_row_sharding_reduced_exchange_two_ranks(tmp_path):
    path = str(tmp_path / "rows.npy")
    mp.spawn(_rows_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    both = np.load(path)
    assert np.array_equal(both[0], both[1]), "row-sharded result differs from the single-GPU bytes"
