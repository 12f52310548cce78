"""Host-side mirror of hei::matmul (proj/include/hei/matmul/matmul.hpp:16-142)
over the C ABI. Same names, argument meaning and error types as the reference:

    proposed_counts / baseline_counts      (matmul.cpp:30-57)
    GpuTwinServer                          (TwinContext::server_backend, twin.cpp:66-75)
    encode_weights                         (matmul.cpp:83-104, on the device)
    EncodedWeights.from_prepared           (upload of reference EncodedWeights)
    encode_bias                            (matmul.cpp:106-112)
    MatmulStream(push_row, finish, counters) (matmul.cpp:114-237)
    matmul                                 (matmul.cpp:239-255)

All residues use the reference's flat u64 layouts (include/heinfer_b200.h).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import native
from .native import FORM_COEFF, FORM_EVAL, OpCounters, ParamError, RangeError, check, i64p, u64p


def proposed_counts(rows: int, cols: int, f: int, n: int) -> OpCounters:
    c = OpCounters()
    check(native.lib().hei_proposed_counts(C.c_uint64(rows), C.c_uint64(cols), C.c_uint64(f), C.c_uint32(n), C.byref(c)))
    return c


def baseline_counts(rows: int, cols: int, f: int, n: int) -> OpCounters:
    c = OpCounters()
    check(native.lib().hei_baseline_counts(C.c_uint64(rows), C.c_uint64(cols), C.c_uint64(f), C.c_uint32(n), C.byref(c)))
    return c


@dataclass
class ScalingConfig:  # fixed_point.hpp:13-20
    s_x: int = 6
    s_w: int = 14
    input_int_bits: int = 8

    def output_scale(self) -> int:
        return self.s_x + self.s_w


def scale_value(x: float, exponent: int) -> int:
    """fixed_point.cpp:37-48: x * 2^e rounded half away from zero."""
    if not math.isfinite(x):
        raise RangeError("scale_value: non-finite input")
    if exponent > 62:
        raise ParamError("scale_value: exponent too large")
    scaled = math.ldexp(x, exponent)
    limit = float((1073872897 * 114689 - 1) // 2)
    if not abs(scaled) <= limit:
        raise RangeError(f"scale_value: {x} * 2^{exponent} exceeds the plaintext capacity")
    # std::llround: half away from zero, without the double rounding of
    # floor(|s| + 0.5) (which gives 1 at 0.49999999999999994); a - floor(a)
    # is exact for every |s| < 2^53 and the |s| >= 2^53 values are integers.
    a = abs(scaled)
    r = math.floor(a)
    if a - r >= 0.5:
        r += 1
    return int(r if scaled >= 0 else -r)


def encode_bias(bias, cfg: ScalingConfig = ScalingConfig()) -> np.ndarray:
    return np.array([scale_value(float(b), cfg.output_scale()) for b in bias], dtype=np.int64)


class GpuTwinServer:
    """Evaluate-only twin backend resident on one GPU: context, tables and the
    Galois keys of both branches (no secret material)."""

    def __init__(self, n: int, t, L, q, galois_elts, galois_keys, scaling: ScalingConfig = ScalingConfig(),
                 device: int = 0, public_keys=None, security_level: int = 128):
        self.n = int(n)
        self.security_level = int(security_level)
        self.t = [int(t[0]), int(t[1])]
        self.L = [int(L[0]), int(L[1])]
        self.q = np.ascontiguousarray(q, dtype=np.uint64)
        self.scaling = scaling
        self.ct_words = 2 * (self.L[0] + self.L[1]) * self.n
        self.pt_words = (self.L[0] + self.L[1]) * self.n
        d = native.TwinDesc()
        d.n = self.n
        d.t[0], d.t[1] = self.t
        d.L[0], d.L[1] = self.L
        d.q = u64p(self.q)
        d.s_x, d.s_w, d.input_int_bits = scaling.s_x, scaling.s_w, scaling.input_int_bits
        d.device = device
        self._h = C.c_void_p()
        check(native.lib().hei_gpu_ctx_create(C.byref(d), C.byref(self._h)))
        elts = np.ascontiguousarray(galois_elts, dtype=np.uint64)
        for b in range(2):
            if galois_keys is None or galois_keys[b] is None:
                continue
            rows = np.ascontiguousarray(galois_keys[b], dtype=np.uint64)
            check(native.lib().hei_gpu_upload_galois_keys(self._h, C.c_uint32(b), C.c_uint32(len(elts)), u64p(elts), u64p(rows)))
        if public_keys is not None:
            for b in range(2):
                pk = np.ascontiguousarray(public_keys[b], dtype=np.uint64)
                check(native.lib().hei_gpu_upload_public_key(self._h, C.c_uint32(b), u64p(pk)))

    @property
    def handle(self):
        return self._h

    def params_hash(self, branch: int) -> int:
        """BfvContext::hash() of a branch (EncryptionParams::hash, params.cpp:68-82)."""
        q0 = self.q[: self.L[0]] if branch == 0 else self.q[self.L[0]:]
        q0 = np.ascontiguousarray(q0, dtype=np.uint64)
        return int(native.lib().hei_params_hash(self.n, self.t[branch], self.security_level, u64p(q0), len(q0)))

    # ---- key generation, SURVEY §8(f) row 4 ----
    def keygen(self, rng: "Prng", install: bool = True):
        """TwinContext::keygen (twin.cpp:41-48) on the device from the replayed
        util::Prng `rng` (advanced exactly as the reference's). Returns
        (elts ascending, [gk0, gk1] [elt][l][part][i][N], sk [2][N] int8,
        pk [branch][part][prime][N] coeff) — the layouts of the oracle's
        galois_keys(). install=True also installs them in this context."""
        ne = self.n.bit_length() - 1  # log2(N) - 1 power-of-two steps + the swap
        elts = np.zeros(ne, np.uint64)
        gk = [np.zeros((ne, self.L[b], 2, self.L[b], self.n), np.uint64) for b in range(2)]
        sk = np.zeros((2, self.n), np.int8)
        pk = np.zeros(self.ct_words, np.uint64)
        check(native.lib().hei_gpu_keygen(self._h, rng._h, C.c_int(int(install)), sk.ctypes.data_as(C.POINTER(C.c_int8)),
                                          u64p(pk), u64p(elts), u64p(gk[0]), u64p(gk[1])))
        return elts, gk, sk, pk

    # ---- client role (decryption), SURVEY §8(f) row 3 ----
    def upload_secret_keys(self, sk) -> None:
        """SecretKey::s of both branches, ternary int8 [2][N]."""
        sk = np.ascontiguousarray(sk, dtype=np.int8).reshape(2, self.n)
        for b in range(2):
            check(native.lib().hei_gpu_upload_secret_key(self._h, C.c_uint32(b), sk[b].ctypes.data_as(C.POINTER(C.c_int8))))

    def decrypt_signed(self, cts: np.ndarray, form: int = FORM_EVAL) -> np.ndarray:
        """TwinBackend::decrypt_signed per twin ciphertext: [count][N] int64."""
        cts = np.ascontiguousarray(cts, dtype=np.uint64).reshape(-1, self.ct_words)
        out = np.zeros((cts.shape[0], self.n), np.int64)
        check(native.lib().hei_gpu_decrypt_signed(self._h, u64p(cts), C.c_int(form), C.c_uint64(cts.shape[0]), i64p(out)))
        return out

    def noise_budget(self, cts: np.ndarray, form: int = FORM_EVAL) -> np.ndarray:
        """TwinBackend::noise_budget per twin ciphertext."""
        cts = np.ascontiguousarray(cts, dtype=np.uint64).reshape(-1, self.ct_words)
        out = np.zeros(cts.shape[0], np.int32)
        check(native.lib().hei_gpu_noise_budget(self._h, u64p(cts), C.c_int(form), C.c_uint64(cts.shape[0]),
                                                out.ctypes.data_as(C.POINTER(C.c_int))))
        return out

    def unpack_results(self, packed: np.ndarray, rows: int, cols: int) -> np.ndarray:
        """matmul::unpack_results (matmul.cpp:257-271)."""
        packed = np.ascontiguousarray(packed, dtype=np.uint64).reshape(-1, self.ct_words)
        out = np.zeros((rows, cols), np.int64)
        check(native.lib().hei_gpu_unpack_results(self._h, u64p(packed), C.c_uint64(packed.shape[0]), C.c_uint64(rows),
                                                  C.c_uint64(cols), i64p(out)))
        return out

    def unpack_baseline(self, blocks: np.ndarray, rows: int, cols: int) -> np.ndarray:
        """matmul::unpack_baseline (matmul.cpp:346-358)."""
        blocks = np.ascontiguousarray(blocks, dtype=np.uint64)
        out = np.zeros((rows, cols), np.int64)
        check(native.lib().hei_gpu_unpack_baseline(self._h, u64p(blocks), C.c_uint64(rows), C.c_uint64(cols), i64p(out)))
        return out

    def hect_bytes(self, branch: int) -> int:
        """Size of one branch ciphertext blob (serialize.cpp:63-78)."""
        return int(native.lib().hei_hect_ciphertext_bytes(self.n, self.L[branch]))

    def chunks(self, f: int) -> int:
        return (f + self.n - 1) // self.n

    def set_batch_pairs(self, pairs: int) -> None:
        native.lib().hei_gpu_set_batch_pairs(self._h, C.c_uint64(pairs))

    # kernel-level seam (kernels::Kernels table, modops.hpp:29-51)
    def ntt(self, branch: int, prime: int, polys: np.ndarray, inverse: bool = False) -> np.ndarray:
        a = np.array(polys, dtype=np.uint64, copy=True, order="C")
        count = a.size // self.n
        check(native.lib().hei_gpu_ntt(self._h, C.c_uint32(branch), C.c_uint32(prime), u64p(a), C.c_uint64(count), C.c_int(int(inverse))))
        return a

    def apply_galois(self, branch: int, elt: int, ct: np.ndarray, form: int = FORM_EVAL) -> np.ndarray:
        """BfvContext::apply_galois (context.cpp:428-507) on a single-branch
        ciphertext [2][L][N] in `form`; the result keeps the input's form."""
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        out = np.zeros_like(ct)
        check(native.lib().hei_gpu_apply_galois_form(self._h, C.c_uint32(branch), C.c_uint64(elt), C.c_int(form), u64p(ct),
                                                     u64p(out)))
        return out

    def sum_all_slots(self, cts: np.ndarray) -> np.ndarray:
        cts = np.ascontiguousarray(cts, dtype=np.uint64)
        out = np.zeros_like(cts)
        count = cts.size // self.ct_words
        check(native.lib().hei_gpu_sum_all_slots(self._h, u64p(cts), u64p(out), C.c_uint64(count)))
        return out

    def close(self):
        if self._h:
            native.lib().hei_gpu_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class EncodedWeights:
    """Device-resident EncodedWeights (matmul.hpp:51-55)."""

    def __init__(self, server: GpuTwinServer, handle, f: int, cols: int):
        self.server, self._h, self.f, self.cols = server, handle, f, cols
        self.n = server.n

    @classmethod
    def from_prepared(cls, server: GpuTwinServer, prepared: np.ndarray, f: int) -> "EncodedWeights":
        prepared = np.ascontiguousarray(prepared, dtype=np.uint64)
        cols = prepared.shape[0]
        h = C.c_void_p()
        check(native.lib().hei_gpu_weights_create(server.handle, u64p(prepared), C.c_uint64(f), C.c_uint64(cols), C.byref(h)))
        return cls(server, h, f, cols)

    def close(self):
        if self._h:
            native.lib().hei_gpu_weights_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def encode_weights(server: GpuTwinServer, w: np.ndarray) -> EncodedWeights:
    """w is f x cols scaled integers; transposition + encoding on the device."""
    w = np.ascontiguousarray(w, dtype=np.int64)
    if w.ndim != 2 or w.size == 0:
        raise ParamError("encode_weights: empty matrix")
    f, cols = w.shape
    h = C.c_void_p()
    check(native.lib().hei_gpu_weights_encode(server.handle, i64p(w), C.c_uint64(f), C.c_uint64(cols), C.byref(h)))
    return EncodedWeights(server, h, f, cols)


class MatmulStream:
    """MatmulStream (matmul.hpp:83-114): push rows in any order, then finish."""

    def __init__(self, server: GpuTwinServer, w: EncodedWeights, bias, total_rows: int):
        self.server, self.w = server, w
        self.bias = np.ascontiguousarray(bias, dtype=np.int64)
        if self.bias.size != w.cols:
            raise ParamError("matmul: bias length does not match output count")
        self.rows = int(total_rows)
        self._h = C.c_void_p()
        self._counters = None
        check(native.lib().hei_gpu_stream_create(server.handle, w._h, i64p(self.bias), C.c_uint64(self.rows), C.byref(self._h)))

    def push_row(self, row_index: int, chunks: np.ndarray, form: int = FORM_EVAL) -> None:
        chunks = np.ascontiguousarray(chunks, dtype=np.uint64)
        if chunks.size != self.server.chunks(self.w.f) * self.server.ct_words:
            raise ParamError("push_row: row has the wrong chunk count")
        check(native.lib().hei_gpu_stream_push_row(self._h, C.c_uint64(row_index), u64p(chunks), C.c_int(form)))

    def finish(self) -> np.ndarray:
        C_ = (self.rows * self.w.cols + self.server.n - 1) // self.server.n
        out = np.zeros((C_, self.server.ct_words), dtype=np.uint64)
        cnt = OpCounters()
        check(native.lib().hei_gpu_stream_finish(self._h, u64p(out), C.byref(cnt)))
        self._counters = cnt
        return out

    def counters(self) -> OpCounters:
        if self._counters is None:
            raise ParamError("counters: stream not finished")
        return self._counters

    def __del__(self):
        try:
            if self._h:
                native.lib().hei_gpu_stream_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass


def matmul(server: GpuTwinServer, inputs: np.ndarray, w: EncodedWeights, bias, form: int = FORM_EVAL):
    """matmul::matmul (matmul.cpp:239-255): inputs [R][k][twin ct] u64 on the
    host. Returns (packed [C][twin ct] eval form, OpCounters)."""
    inputs = np.ascontiguousarray(inputs, dtype=np.uint64)
    if inputs.ndim != 3 or inputs.shape[0] == 0:
        raise ParamError("matmul: empty input")
    R = inputs.shape[0]
    if inputs.shape[1] != server.chunks(w.f):
        raise ParamError("matmul: input and weight shapes do not match")
    bias = np.ascontiguousarray(bias, dtype=np.int64)
    if bias.size != w.cols:
        raise ParamError("matmul: bias length does not match output count")
    C_ = (R * w.cols + server.n - 1) // server.n
    out = np.empty((C_, server.ct_words), dtype=np.uint64)  # every word is written
    cnt = OpCounters()
    check(native.lib().hei_gpu_matmul(server.handle, w._h, u64p(inputs), C.c_int(form), C.c_uint64(R), i64p(bias), u64p(out), C.byref(cnt)))
    return out, cnt


def matmul_device(server: GpuTwinServer, d_inputs_ptr: int, rows: int, w: EncodedWeights, bias, d_out_ptr: int,
                  stream_ptr: int = 0) -> OpCounters:
    """Device-resident variant: u32 residues already in HBM (bench `value`)."""
    bias = np.ascontiguousarray(bias, dtype=np.int64)
    cnt = OpCounters()
    check(native.lib().hei_gpu_matmul_device(server.handle, w._h, C.c_void_p(d_inputs_ptr), C.c_int(FORM_EVAL), C.c_uint64(rows),
                                             i64p(bias), C.c_void_p(d_out_ptr), C.byref(cnt), C.c_void_p(stream_ptr)))
    return cnt


class Prng:
    """util::Prng replay state (rng.hpp:19-68) for the standard algorithm's
    encryption randomness; advances exactly like BfvBackend's rng_."""

    def __init__(self, seed: int):
        self._h = C.c_void_p()
        check(native.lib().hei_gpu_prng_create(C.c_uint64(seed), C.byref(self._h)))

    def draw(self, count: int) -> np.ndarray:
        out = np.zeros(count, dtype=np.uint64)
        check(native.lib().hei_gpu_prng_draw(self._h, C.c_uint64(count), u64p(out)))
        return out

    def __del__(self):
        try:
            if self._h:
                native.lib().hei_gpu_prng_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass


def baseline_matmul(server: GpuTwinServer, x: np.ndarray, w: np.ndarray, bias, rng0: Prng, rng1: Prng):
    """matmul::baseline_matmul (matmul.cpp:273-344): x is R x f, w is f x cols
    (scaled integers). Encrypts each feature column on the device with the
    replayed randomness. Returns (blocks [ceil(R/N)][cols][twin ct], counters)."""
    x = np.ascontiguousarray(x, dtype=np.int64)
    w = np.ascontiguousarray(w, dtype=np.int64)
    if x.ndim != 2 or w.ndim != 2 or x.size == 0 or w.shape[1] == 0:
        raise ParamError("baseline: empty input")
    R, f = x.shape
    if w.shape[0] != f:
        raise ParamError("baseline: input and weight shapes do not match")
    cols = w.shape[1]
    bias = np.ascontiguousarray(bias, dtype=np.int64)
    if bias.size != cols:
        raise ParamError("baseline: bias length does not match output count")
    B = (R + server.n - 1) // server.n
    out = np.zeros((B, cols, server.ct_words), dtype=np.uint64)
    cnt = OpCounters()
    check(native.lib().hei_gpu_baseline_matmul(server.handle, i64p(x), C.c_uint64(R), C.c_uint64(f), i64p(w), C.c_uint64(cols),
                                               i64p(bias), rng0._h, rng1._h, u64p(out), C.byref(cnt)))
    return out, cnt


def encode_inputs(server: GpuTwinServer, x: np.ndarray, rng0: Prng, rng1: Prng) -> np.ndarray:
    """matmul::encode_inputs (matmul.cpp:59-81) on the device: x is R x f
    scaled integers; returns [R][ceil(f/N)][twin ct] u64 eval-form ciphertexts
    drawn from the two branch Prng streams (needs the public keys)."""
    x = np.ascontiguousarray(x, dtype=np.int64)
    if x.ndim != 2 or x.size == 0:
        raise ParamError("encode_inputs: empty matrix")
    R, f = x.shape
    out = np.zeros((R, server.chunks(f), server.ct_words), dtype=np.uint64)
    check(native.lib().hei_gpu_encode_inputs(server.handle, i64p(x), C.c_uint64(R), C.c_uint64(f), rng0._h, rng1._h, u64p(out)))
    return out


def encode_inputs_device(server: GpuTwinServer, x: np.ndarray, rng0: Prng, rng1: Prng, d_out_ptr: int, stream_ptr: int = 0):
    x = np.ascontiguousarray(x, dtype=np.int64)
    R, f = x.shape
    check(native.lib().hei_gpu_encode_inputs_device(server.handle, i64p(x), C.c_uint64(R), C.c_uint64(f), rng0._h, rng1._h,
                                                    C.c_void_p(d_out_ptr), C.c_void_p(stream_ptr)))



def save_ciphertexts(server: GpuTwinServer, cts: np.ndarray, form: int = FORM_EVAL) -> bytes:
    """bfv::save_ciphertext (serialize.cpp:63-78) of every branch of every
    twin ciphertext in `cts` ([..][twin ct] u64), concatenated in order
    [ct][branch] -- the client's request blob list (client.cpp /
    server.cpp:145-147). Eval-form input is brought to coefficient form by
    device inverse NTTs (to_coeff), then written as header (magic, version,
    params hash, parts = 2, kind = ciphertext) + 2L polys of (form byte, N u64)."""
    cts = np.ascontiguousarray(cts, dtype=np.uint64).reshape(-1, server.ct_words)
    M, n = cts.shape[0], server.n
    sizes = [server.hect_bytes(0), server.hect_bytes(1)]
    out = np.zeros((M, sizes[0] + sizes[1]), np.uint8)
    off_w, off_b = 0, 0
    for b in range(2):
        L = server.L[b]
        hdr = np.frombuffer(b"HECT" + (1).to_bytes(2, "little") + server.params_hash(b).to_bytes(8, "little")
                            + (2).to_bytes(4, "little") + bytes([5]), np.uint8)
        blob = out[:, off_b: off_b + sizes[b]]
        blob[:, :19] = hdr
        polys = blob[:, 19:].reshape(M, 2 * L, 1 + 8 * n)
        polys[:, :, 0] = FORM_COEFF
        br = cts[:, off_w: off_w + 2 * L * n].reshape(M, 2, L, n)
        for i in range(L):
            v = np.ascontiguousarray(br[:, :, i, :]).reshape(2 * M, n)
            if form == FORM_EVAL:
                v = server.ntt(b, i, v, inverse=True)
            v = v.reshape(M, 2, n)
            for p in range(2):
                polys[:, p * L + i, 1:] = v[:, p, :].view(np.uint8).reshape(M, 8 * n)
        off_w += 2 * L * n
        off_b += sizes[b]
    return out.tobytes()


def matmul_wire(server: GpuTwinServer, w: EncodedWeights, blobs, rows: int, bias):
    """The server's computation on wire objects (InferenceServer::do_infer,
    server.cpp:112-172): ``blobs`` is the request's HECT ciphertext list
    concatenated in order [row][chunk][branch]. Returns (response blobs
    [packed ct][branch] as a list of bytes — save_ciphertext, coeff form —,
    OpCounters). Parsing, to_eval, the matmul, to_coeff and serialization run
    on the GPU."""
    buf = np.frombuffer(blobs, dtype=np.uint8) if isinstance(blobs, (bytes, bytearray)) else np.ascontiguousarray(blobs, np.uint8)
    bias = np.ascontiguousarray(bias, dtype=np.int64)
    if bias.size != w.cols:
        raise ParamError("matmul: bias length does not match output count")
    hashes = (C.c_uint64 * 2)(server.params_hash(0), server.params_hash(1))
    b0, b1 = server.hect_bytes(0), server.hect_bytes(1)
    C_ = (rows * w.cols + server.n - 1) // server.n
    out = np.zeros(max(C_, 1) * (b0 + b1), np.uint8)
    out_len = C.c_uint64(0)
    cnt = OpCounters()
    u8p = C.POINTER(C.c_uint8)
    check(native.lib().hei_gpu_matmul_wire(server.handle, w._h, hashes, buf.ctypes.data_as(u8p), C.c_uint64(buf.size),
                                           C.c_uint64(rows), i64p(bias), out.ctypes.data_as(u8p), C.c_uint64(out.size),
                                           C.byref(out_len), C.byref(cnt)))
    res = []
    for c in range(C_):
        base = c * (b0 + b1)
        res.append(bytes(out[base: base + b0]))
        res.append(bytes(out[base + b0: base + b0 + b1]))
    return res, cnt


def default_q_primes(n: int, t: int) -> list:
    """bfv::default_q_primes (params.cpp:84-104): the q chain of one branch."""
    out = np.zeros(16, np.uint64)
    cnt = C.c_uint32(0)
    check(native.lib().hei_default_q_primes(C.c_uint32(n), C.c_uint64(t), u64p(out), C.c_uint32(16), C.byref(cnt)))
    return [int(v) for v in out[: cnt.value]]
