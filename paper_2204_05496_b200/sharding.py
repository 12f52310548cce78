"""Sharding across GPUs — one process per GPU.

Individual (row) sharding is the default:

Every (individual, class) pipeline is independent; rank r takes a
contiguous row block and accumulates the masked class results of its rows into
an unreduced u64 packed accumulator, reduces it mod q to u32 residues (its
partial: C * 2 * (L0 + L1) * N words, 0.65 MB at C4), and the ranks exchange
the partials with one NCCL all-gather on the compute stream (no host
barrier); rank 0 sums them mod q and adds the bias once (MatmulStream::finish,
matmul.cpp:200-232). Mod-q addition is order-free, hence bit-exact for any
rank count.

Feature-block sharding (C5's second mode): rank r holds only chunks
shard_chunks(kc, world, r) of every row, computes the chunk products of those
chunks into an unreduced u64 dot accumulator, the ranks reduce-scatter the
dot partials by rows (each rank receives the summed dots of its row block),
and every rank folds and masks its rows as in individual sharding. The dot
exchange is rows * cols * 2 (L0 + L1) N words, so it is an option for
feature-partitioned inputs, not the default.
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


def reduce_packed_device(server, d_acc_ptr: int, count: int, d_out_ptr: int, stream_ptr: int = 0) -> None:
    """A rank's u64 packed accumulator -> u32 residues mod q (its partial for
    the exchange; stream-ordered, no host wait)."""
    check(native.lib().hei_gpu_reduce_packed_device(server.handle, C.c_void_p(d_acc_ptr), C.c_uint64(count),
                                                    C.c_void_p(d_out_ptr), C.c_void_p(stream_ptr)))


def finish_parts_device(server, w, d_parts_ptr: int, parts: int, bias, total_rows: int, d_out_ptr: int,
                        stream_ptr: int = 0) -> None:
    """Sum `parts` gathered u32 partials mod q and add the bias once
    (MatmulStream::finish, matmul.cpp:200-232); stream-ordered."""
    bias = np.ascontiguousarray(bias, dtype=np.int64)
    check(native.lib().hei_gpu_finish_parts_device(server.handle, w._h, C.c_void_p(d_parts_ptr), C.c_uint32(parts),
                                                   i64p(bias), C.c_uint64(total_rows), C.c_void_p(d_out_ptr),
                                                   C.c_void_p(stream_ptr)))


def exchange_partials(part, group=None):
    """All-gather the ranks' u32 partials (torch int32 [count][twin ct] on the
    device) into [world][count][twin ct] on every rank: one NCCL all-gather
    on the current stream (gloo on CPU). World 1 returns the input with a
    leading axis."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return part.unsqueeze(0)
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "gloo":  # host-side exchange (CPU tests, single-GPU plumbing checks)
        host = part.cpu()
        outs = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(outs, host, group=group)
        return torch.stack(outs).to(part.device)
    out = torch.empty((world,) + tuple(part.shape), dtype=part.dtype, device=part.device)
    dist.all_gather_into_tensor(out, part, group=group)
    return out


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


def shard_chunks(kc: int, world: int, rank: int):
    """Contiguous feature block (chunk range) of `rank`: (chunk_lo, count)."""
    return shard_rows(kc, world, rank)


def chunk_dot_partial_device(server, w, d_inputs_ptr: int, rows: int, chunk_lo: int, chunk_count: int, d_dot_ptr: int,
                             stream_ptr: int = 0) -> None:
    check(native.lib().hei_gpu_chunk_dot_partial_device(server.handle, w._h, C.c_void_p(d_inputs_ptr), C.c_uint64(rows),
                                                        C.c_uint64(chunk_lo), C.c_uint64(chunk_count),
                                                        C.c_void_p(d_dot_ptr), C.c_void_p(stream_ptr)))


def fold_pack_device(server, w, d_dot_ptr: int, row_lo: int, row_count: int, total_rows: int, d_acc_ptr: int,
                     stream_ptr: int = 0) -> None:
    check(native.lib().hei_gpu_fold_pack_device(server.handle, w._h, C.c_void_p(d_dot_ptr), C.c_uint64(row_lo),
                                                C.c_uint64(row_count), C.c_uint64(total_rows), C.c_void_p(d_acc_ptr),
                                                C.c_void_p(stream_ptr)))


def reduce_scatter_dots(dot, total_rows: int, group=None):
    """Sum the ranks' dot partials (torch int64 [total_rows * cols][ct]) and
    return this rank's row block (shard_rows) of the sum. Uses
    reduce_scatter_tensor over equal padded blocks (NCCL on GPUs, gloo on
    CPU); world 1 returns the input."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return dot
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    per_row = dot.shape[0] // total_rows
    block = (total_rows + world - 1) // world
    padded = torch.zeros((block * world * per_row,) + tuple(dot.shape[1:]), dtype=dot.dtype, device=dot.device)
    padded[: dot.shape[0]] = dot
    out = torch.empty((block * per_row,) + tuple(dot.shape[1:]), dtype=dot.dtype, device=dot.device)
    if dist.get_backend(group) == "gloo":
        # gloo has no reduce_scatter: all-reduce on the host and slice
        host = padded.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
        out.copy_(host[rank * block * per_row:(rank + 1) * block * per_row])
    else:
        dist.reduce_scatter_tensor(out, padded, op=dist.ReduceOp.SUM, group=group)
    lo, cnt = shard_rows(total_rows, world, rank)
    return out[: cnt * per_row]


class PeerGather:
    """Exchange of the ranks' packed u64 accumulators over peer memory:
    `owner` allocates a receive buffer with one slot per rank and exports it
    with CUDA IPC; every rank maps it (an NVLink peer mapping between GPUs)
    and `push` writes its accumulator into its slot with one device-to-device
    copy. After a barrier the owner's `reduce` sums the slots (exact u64) into
    slot 0, whose pointer is `total_ptr`. No collective library involved."""

    def __init__(self, nbytes: int, device: int, owner: int = 0, group=None):
        import torch.distributed as dist

        self.owner, self.nbytes = owner, int(nbytes)
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self._own = None
        self._mapped = None
        handle = [None]
        err = None
        if self.rank == owner:
            try:
                p = C.c_void_p()
                check(native.lib().hei_gpu_buffer_alloc(C.c_int(device), C.c_uint64(self.nbytes * self.world),
                                                        C.byref(p)))
                self._own = p
                h = (C.c_uint8 * 64)()
                check(native.lib().hei_gpu_ipc_handle(p, h))
                handle[0] = bytes(h)
                self.base = p.value
            except Exception as e:  # still take part in the broadcast, then fail
                err = e
        dist.broadcast_object_list(handle, src=owner, group=group)
        if err is not None:
            raise err
        if handle[0] is None:
            raise RuntimeError("peer gather: the owner could not export its buffer")
        if self.rank != owner:
            p = C.c_void_p()
            hb = (C.c_uint8 * 64).from_buffer_copy(handle[0])
            check(native.lib().hei_gpu_ipc_open(C.c_int(device), hb, C.byref(p)))
            self._mapped = p
            self.base = p.value
        self.total_ptr = self.base

    def push(self, local_ptr: int, stream_ptr: int = 0) -> None:
        dst = self.base + self.rank * self.nbytes
        check(native.lib().hei_gpu_copy_async(C.c_void_p(dst), C.c_void_p(local_ptr), C.c_uint64(self.nbytes),
                                              C.c_void_p(stream_ptr)))

    def reduce(self, stream_ptr: int = 0) -> None:
        """Owner only, after every rank's push has completed (barrier)."""
        if self._own is not None:
            check(native.lib().hei_gpu_sum_slots(self._own, C.c_uint64(self.nbytes // 8), C.c_uint32(self.world),
                                                 C.c_void_p(stream_ptr)))

    def close(self) -> None:
        if self._mapped is not None:
            check(native.lib().hei_gpu_ipc_close(self._mapped))
            self._mapped = None
        if self._own is not None:
            native.lib().hei_gpu_buffer_free(self._own)
            self._own = None
