"""Individual (row) sharding across GPUs — one process per GPU.

Every (individual, class) pipeline is independent; rank r takes a
contiguous row block and accumulates the masked class results of its rows into
an unreduced u64 packed accumulator. Accumulators of all ranks add exactly
(each rank contributes < rows * 2^31 per slot), so the only exchange is one
integer all-reduce of C * 2 * (L0 + L1) * N words (0.65 M words, 5.2 MB at
C4), followed by the mod-q reduction and a single bias add_plain
(MatmulStream::finish, matmul.cpp:342-374). Order-free, hence bit-exact for
any rank count.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import native
from .native import check, i64p


def shard_rows(total_rows: int, world: int, rank: int):
    """Contiguous block of rows for `rank` (parallel_for's split,
    util/parallel.cpp:34-53): returns (offset, count)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    block = (total_rows + world - 1) // world
    lo = min(total_rows, rank * block)
    hi = min(total_rows, lo + block)
    return lo, hi - lo


def packed_count(total_rows: int, cols: int, n: int) -> int:
    return (total_rows * cols + n - 1) // n


def matmul_partial_device(server, w, d_inputs_ptr: int, rows: int, row_offset: int, total_rows: int, d_acc_ptr: int,
                          stream_ptr: int = 0) -> None:
    check(native.lib().hei_gpu_matmul_partial_device(server.handle, w._h, C.c_void_p(d_inputs_ptr), C.c_uint64(rows),
                                                     C.c_uint64(row_offset), C.c_uint64(total_rows), C.c_void_p(d_acc_ptr),
                                                     C.c_void_p(stream_ptr)))


def finish_packed_device(server, w, d_acc_ptr: int, bias, total_rows: int, d_out_ptr: int, stream_ptr: int = 0) -> None:
    bias = np.ascontiguousarray(bias, dtype=np.int64)
    check(native.lib().hei_gpu_finish_packed_device(server.handle, w._h, C.c_void_p(d_acc_ptr), i64p(bias),
                                                    C.c_uint64(total_rows), C.c_void_p(d_out_ptr), C.c_void_p(stream_ptr)))


def combine_partials(acc, group=None):
    """Sum the ranks' packed accumulators in place (torch int64 tensor; the
    u64 partials never exceed 2^63). NCCL over NVLink on GPUs, gloo on CPU."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return acc


def reduce_packed_mod_q(acc: np.ndarray, q_per_poly: np.ndarray) -> np.ndarray:
    """Host-side reference of the mod-q reduction k_finish applies (used by
    the CPU multi-rank tests): acc [C][polys][N] u64 -> residues."""
    return (acc % q_per_poly[None, :, None].astype(np.uint64)).astype(np.uint64)
