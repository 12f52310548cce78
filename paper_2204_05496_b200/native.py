"""ctypes binding of the C ABI in include/heinfer_b200.h.

The product path is libheinfer_b200.so (hand-written sm_100a CUDA). There is
no CPU fallback: if the library is missing or cannot be loaded, every entry
point raises ``NativeLibraryError``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# HEI_LIB_PATH: an alternative in-tree build of the same library (A/B timing of
# two builds on one box); the default is the package's own lib/.
LIB_PATH = os.environ.get("HEI_LIB_PATH") or os.path.join(HERE, "lib", "libheinfer_b200.so")

HEI_OK = 0
HEI_PARAM_ERROR = 1
HEI_KEY_ERROR = 2
HEI_RANGE_ERROR = 3
HEI_NOISE_ERROR = 4
HEI_CODEC_ERROR = 5
HEI_CUDA_ERROR = 6
HEI_INTERNAL = 9
FORM_COEFF = 0
FORM_EVAL = 1


class NativeLibraryError(RuntimeError):
    """libheinfer_b200.so is missing or unusable (no fallback exists)."""


# Exception types mirror hei/util/errors.hpp:13-53.
class HeiError(Exception):
    code = HEI_INTERNAL


class ParamError(HeiError, ValueError):
    code = HEI_PARAM_ERROR


class KeyError_(HeiError, LookupError):
    code = HEI_KEY_ERROR


class RangeError(HeiError, ValueError):
    code = HEI_RANGE_ERROR


class NoiseError(HeiError):
    code = HEI_NOISE_ERROR


class CodecError(HeiError):
    code = HEI_CODEC_ERROR


class CudaError(HeiError):
    code = HEI_CUDA_ERROR


_CODES = {c.code: c for c in (ParamError, KeyError_, RangeError, NoiseError, CodecError, CudaError)}


class OpCounters(C.Structure):
    """matmul::OpCounters (matmul.hpp:21-27)."""

    _fields_ = [
        ("mul_plain_count", C.c_uint64),
        ("rotation_count", C.c_uint64),
        ("add_count", C.c_uint64),
        ("ciphertexts_in", C.c_uint64),
        ("ciphertexts_out", C.c_uint64),
    ]

    def as_tuple(self):
        return (self.mul_plain_count, self.rotation_count, self.add_count, self.ciphertexts_in, self.ciphertexts_out)


class TwinDesc(C.Structure):
    _fields_ = [
        ("n", C.c_uint32),
        ("t", C.c_uint64 * 2),
        ("L", C.c_uint32 * 2),
        ("q", C.POINTER(C.c_uint64)),
        ("s_x", C.c_uint32),
        ("s_w", C.c_uint32),
        ("input_int_bits", C.c_uint32),
        ("device", C.c_int),
    ]


EXPORTED = [
    "hei_gpu_last_error", "hei_gpu_version", "hei_gpu_ctx_create", "hei_gpu_ctx_destroy",
    "hei_gpu_upload_galois_keys", "hei_gpu_upload_public_key", "hei_gpu_weights_create",
    "hei_gpu_weights_encode", "hei_gpu_weights_destroy", "hei_gpu_matmul", "hei_gpu_matmul_device",
    "hei_gpu_stream_create", "hei_gpu_stream_push_row", "hei_gpu_stream_finish", "hei_gpu_stream_destroy",
    "hei_gpu_prng_create", "hei_gpu_prng_destroy", "hei_gpu_prng_draw", "hei_gpu_baseline_matmul", "hei_proposed_counts",
    "hei_baseline_counts", "hei_gpu_ntt", "hei_gpu_apply_galois", "hei_gpu_sum_all_slots",
    "hei_gpu_launch_count", "hei_gpu_reset_launch_count", "hei_gpu_set_batch_pairs",
    "hei_gpu_kernel_timing", "hei_gpu_apply_galois_form", "hei_gpu_kernel_stats", "hei_gpu_measure_butterfly_peak",
    "hei_gpu_matmul_partial_device", "hei_gpu_finish_packed_device",
    "hei_gpu_encode_inputs", "hei_gpu_encode_inputs_device",
    "hei_hect_ciphertext_bytes", "hei_params_hash", "hei_gpu_matmul_wire",
    "hei_gpu_upload_secret_key", "hei_gpu_decrypt_signed", "hei_gpu_noise_budget",
    "hei_gpu_unpack_results", "hei_gpu_unpack_baseline", "hei_gpu_keygen",
    "hei_gpu_debug_rejection_plan", "hei_gpu_chunk_dot_partial_device", "hei_gpu_fold_pack_device",
    "hei_default_q_primes", "hei_gpu_ipc_handle", "hei_gpu_ipc_open", "hei_gpu_ipc_close",
    "hei_gpu_buffer_alloc", "hei_gpu_buffer_zero", "hei_gpu_buffer_free", "hei_gpu_copy_async", "hei_gpu_sum_slots",
    "hei_gpu_reduce_packed_device", "hei_gpu_finish_parts_device",
]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback exists)")
        try:
            l = C.CDLL(LIB_PATH)
        except OSError as e:  # pragma: no cover - depends on the box
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
        l.hei_gpu_last_error.restype = C.c_char_p
        l.hei_gpu_version.restype = C.c_char_p
        l.hei_gpu_launch_count.restype = C.c_uint64
        l.hei_gpu_ctx_destroy.restype = None
        l.hei_gpu_weights_destroy.restype = None
        l.hei_gpu_stream_destroy.restype = None
        l.hei_gpu_prng_destroy.restype = None
        l.hei_gpu_reset_launch_count.restype = None
        l.hei_gpu_set_batch_pairs.restype = None
        l.hei_gpu_set_batch_pairs.argtypes = [C.c_void_p, C.c_uint64]
        l.hei_gpu_buffer_free.restype = None
        l.hei_gpu_buffer_free.argtypes = [C.c_void_p]
        l.hei_hect_ciphertext_bytes.restype = C.c_uint64
        l.hei_hect_ciphertext_bytes.argtypes = [C.c_uint32, C.c_uint32]
        l.hei_params_hash.restype = C.c_uint64
        l.hei_params_hash.argtypes = [C.c_uint32, C.c_uint64, C.c_int, C.POINTER(C.c_uint64), C.c_uint32]
        _lib = l
    return _lib


def check(rc: int) -> None:
    if rc != HEI_OK:
        msg = lib().hei_gpu_last_error().decode(errors="replace")
        raise _CODES.get(rc, HeiError)(msg)


def u64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64)) if a is not None else None


def i64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64)) if a is not None else None


def kernel_timing(server_handle, enable: bool) -> None:
    check(lib().hei_gpu_kernel_timing(server_handle, C.c_int(int(enable))))


def kernel_stats(server_handle, which: int):
    """(launches, total_ms) of the fold kernels timed with CUDA events:
    which = 0 key switch, 1 digit INTT."""
    n = C.c_uint64()
    ms = C.c_double()
    check(lib().hei_gpu_kernel_stats(server_handle, C.c_int(which), C.byref(n), C.byref(ms)))
    return int(n.value), float(ms.value)


def butterfly_peak(device: int = 0) -> float:
    v = C.c_double()
    check(lib().hei_gpu_measure_butterfly_peak(C.c_int(device), C.byref(v)))
    return float(v.value)


def launch_count() -> int:
    return int(lib().hei_gpu_launch_count())


def reset_launch_count() -> None:
    lib().hei_gpu_reset_launch_count()
