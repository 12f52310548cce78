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
