"""TEST INFRASTRUCTURE ONLY — ctypes front-ends for the CPU checkers.

* ``Oracle``    — the C restatement (oracle/heoracle.c -> liboracle.so).
* ``Reference`` — the unmodified reference compiled in place
                  (oracle/ref_driver.cpp + /root/reference/proj/src ->
                  oracle/_ref/libheiref.so).

Both expose the same twin-session interface so tests can run one against the
other. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
reference legs import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libheiref.so")

T0, T1 = 1073872897, 114689  # fixed_point.hpp:25-27
T1_16K = 163841  # batching-compatible t1' for N = 16384


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _u64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64)) if a is not None else None


def _i64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64)) if a is not None else None


def _vp(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


@dataclass
class TwinParams:
    n: int = 8192
    t0: int = T0
    t1: int = T1
    sec: int = 128
    s_x: int = 6
    s_w: int = 14
    in_bits: int = 8


def production_params(n: int = 8192) -> TwinParams:
    return TwinParams(n=n, t0=T0, t1=T1 if n < 16384 else T1_16K, sec=128)


class _Twin:
    """Common logic over either library."""

    prefix = ""
    lib: C.CDLL

    def __init__(self, p: TwinParams, key_seed: int = 1, enc_seed: int = 2):
        self.p = p
        self.n = p.n
        self._h = C.c_void_p()
        self._create(p, key_seed, enc_seed)
        L = np.zeros(2, np.uint32)
        q = np.zeros(64, np.uint64)
        h = np.zeros(2, np.uint64)
        self._info(L, q, h)
        self.L = [int(L[0]), int(L[1])]
        self.q = [int(v) for v in q[: self.L[0] + self.L[1]]]
        self.hash = [int(h[0]), int(h[1])]
        self.ct_words = 2 * (self.L[0] + self.L[1]) * self.n
        self.pt_words = (self.L[0] + self.L[1]) * self.n

    def _check(self, rc):
        if rc != 0:
            err = getattr(self.lib, self.prefix + "last_error")
            err.restype = C.c_char_p
            raise OracleError(rc, err().decode())

    def chunks(self, f: int) -> int:
        return (f + self.n - 1) // self.n

    # --- shared API ---
    def galois_keys(self):
        elts = np.zeros(32, np.uint64)
        m = self.num_elts()
        gk = [np.zeros((m, self.L[b], 2, self.L[b], self.n), np.uint64) for b in range(2)]
        sk = np.zeros((2, self.n), np.int8)
        pk = np.zeros(2 * (self.L[0] + self.L[1]) * self.n, np.uint64)
        self._export(elts, gk[0], gk[1], sk, pk)
        return elts[:m].copy(), gk, sk, pk

    def encode_inputs(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.int64)
        R, f = x.shape
        out = np.zeros((R, self.chunks(f), self.ct_words), np.uint64)
        self._check(getattr(self.lib, self.prefix + "encode_inputs")(self._h, _i64p(x), C.c_uint64(R), C.c_uint64(f), _u64p(out)))
        return out

    def encode_weights(self, w: np.ndarray) -> np.ndarray:
        w = np.ascontiguousarray(w, np.int64)
        f, cols = w.shape
        out = np.zeros((cols, self.chunks(f), self.pt_words), np.uint64)
        self._check(getattr(self.lib, self.prefix + "encode_weights")(self._h, _i64p(w), C.c_uint64(f), C.c_uint64(cols), _u64p(out)))
        return out

    def unpack(self, packed: np.ndarray, R: int, cols: int) -> np.ndarray:
        out = np.zeros((R, cols), np.int64)
        packed = np.ascontiguousarray(packed, np.uint64)
        self._check(getattr(self.lib, self.prefix + "unpack")(self._h, _u64p(packed), C.c_uint64(R), C.c_uint64(cols), _i64p(out)))
        return out

    def decrypt_signed(self, ct: np.ndarray, form: int = 1):
        out = np.zeros(self.n, np.int64)
        bud = C.c_int(0)
        ct = np.ascontiguousarray(ct, np.uint64)
        self._check(getattr(self.lib, self.prefix + "decrypt_signed")(self._h, _u64p(ct), C.c_int(form), _i64p(out), C.byref(bud)))
        return out, bud.value

    def apply_galois(self, b: int, elt: int, ct: np.ndarray) -> np.ndarray:
        out = np.zeros_like(ct)
        self._apply_galois(b, elt, np.ascontiguousarray(ct, np.uint64), out)
        return out

    def sum_all_slots(self, ct: np.ndarray) -> np.ndarray:
        out = np.zeros_like(ct)
        self._check(getattr(self.lib, self.prefix + "sum_all_slots")(self._h, _u64p(np.ascontiguousarray(ct)), _u64p(out)))
        return out

    def close(self):
        if self._h:
            getattr(self.lib, self.prefix + "destroy")(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_oracle_lib = None
_ref_lib = None


def oracle_lib() -> C.CDLL:
    global _oracle_lib
    if _oracle_lib is None:
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} not built (make -C oracle)")
        _oracle_lib = C.CDLL(ORACLE_SO)
        _oracle_lib.ho_last_error.restype = C.c_char_p
        _oracle_lib.ho_shoup_precompute.restype = C.c_uint64
        _oracle_lib.ho_shoup_precompute.argtypes = [C.c_uint64, C.c_uint64]
        _oracle_lib.ho_primitive_root_2n.restype = C.c_uint64
        _oracle_lib.ho_primitive_root_2n.argtypes = [C.c_uint32, C.c_uint64]
        _oracle_lib.ho_is_prime.argtypes = [C.c_uint64]
    return _oracle_lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib() -> C.CDLL:
    global _ref_lib
    if _ref_lib is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")
        _ref_lib = C.CDLL(REF_SO)
        _ref_lib.ref_last_error.restype = C.c_char_p
    return _ref_lib


class Oracle(_Twin):
    prefix = "ho_"

    def __init__(self, p: TwinParams, key_seed: int = 1, enc_seed: int = 2):
        self.lib = oracle_lib()
        super().__init__(p, key_seed, enc_seed)

    def _create(self, p, ks, es):
        self._check(self.lib.ho_twin_create(C.byref(self._h), C.c_uint32(p.n), C.c_uint64(p.t0), C.c_uint64(p.t1), C.c_int(p.sec),
                                            C.c_uint32(p.s_x), C.c_uint32(p.s_w), C.c_uint32(p.in_bits), C.c_uint64(ks), C.c_uint64(es)))

    def _info(self, L, q, h):
        self._m = self.lib.ho_twin_info(self._h, L.ctypes.data_as(C.POINTER(C.c_uint32)), _u64p(q), _u64p(h), None)

    def num_elts(self):
        return self._m

    def elts(self):
        e = np.zeros(32, np.uint64)
        m = self.lib.ho_twin_info(self._h, None, None, None, _u64p(e))
        return e[:m].copy()

    def _export(self, elts, g0, g1, sk, pk):
        self.lib.ho_twin_info(self._h, None, None, None, _u64p(elts))
        self._check(self.lib.ho_twin_export_keys(self._h, _u64p(g0), _u64p(g1), _vp(sk), _u64p(pk)))

    def _apply_galois(self, b, elt, ct, out):
        self._check(self.lib.ho_apply_galois(self._h, C.c_int(b), C.c_uint64(elt), _u64p(ct), _u64p(out)))

    def fast_matmul(self, inputs: np.ndarray, f: int, weights: np.ndarray, bias, form: int = 1, threads: int = 0):
        inputs = np.ascontiguousarray(inputs, np.uint64)
        weights = np.ascontiguousarray(weights, np.uint64)
        R = inputs.shape[0]
        cols = weights.shape[0]
        bias = np.ascontiguousarray(bias, np.int64)
        C_ = (R * cols + self.n - 1) // self.n
        out = np.zeros((C_, self.ct_words), np.uint64)
        cnt = np.zeros(5, np.uint64)
        self._check(self.lib.ho_fast_matmul(self._h, _u64p(inputs), C.c_int(form), C.c_uint64(R), C.c_uint64(f), _u64p(weights),
                                            C.c_uint64(cols), _i64p(bias), _u64p(out), _u64p(cnt), C.c_uint(threads)))
        return out, cnt

    def baseline_matmul(self, x, w, bias):
        x = np.ascontiguousarray(x, np.int64)
        w = np.ascontiguousarray(w, np.int64)
        R, f = x.shape
        cols = w.shape[1]
        B = (R + self.n - 1) // self.n
        out = np.zeros((B, cols, self.ct_words), np.uint64)
        cnt = np.zeros(5, np.uint64)
        bias = np.ascontiguousarray(bias, np.int64)
        self._check(self.lib.ho_baseline_matmul(self._h, _i64p(x), C.c_uint64(R), C.c_uint64(f), _i64p(w), C.c_uint64(cols),
                                                _i64p(bias), _u64p(out), _u64p(cnt)))
        return out, cnt

    def baseline_noise(self, encryptions: int) -> np.ndarray:
        out = np.zeros((encryptions, 2, 3, self.n), np.int8)
        self._check(self.lib.ho_baseline_noise(self._h, C.c_uint64(encryptions), _vp(out)))
        return out

    def unpack_baseline(self, blocks, R, cols):
        out = np.zeros((R, cols), np.int64)
        self._check(self.lib.ho_unpack_baseline(self._h, _u64p(np.ascontiguousarray(blocks)), C.c_uint64(R), C.c_uint64(cols), _i64p(out)))
        return out

    def mask(self, slot: int) -> np.ndarray:
        out = np.zeros(self.pt_words, np.uint64)
        self._check(self.lib.ho_mask(self._h, C.c_uint32(slot), _u64p(out)))
        return out


class Reference(_Twin):
    prefix = "ref_"

    def __init__(self, p: TwinParams, key_seed: int = 1, enc_seed: int = 2):
        self.lib = ref_lib()
        super().__init__(p, key_seed, enc_seed)

    def _create(self, p, ks, es):
        self._check(self.lib.ref_create(C.byref(self._h), C.c_uint32(p.n), C.c_uint64(p.t0), C.c_uint64(p.t1), C.c_int(p.sec),
                                        C.c_uint32(p.s_x), C.c_uint32(p.s_w), C.c_uint32(p.in_bits), C.c_uint64(ks), C.c_uint64(es)))

    def _info(self, L, q, h):
        self._check(self.lib.ref_params(self._h, L.ctypes.data_as(C.POINTER(C.c_uint32)), _u64p(q), _u64p(h)))

    def num_elts(self):
        return self.lib.ref_num_galois(self._h)

    def elts(self):
        e = np.zeros(32, np.uint64)
        self._check(self.lib.ref_export_keys(self._h, _u64p(e), None, None, None, None))
        return e[: self.num_elts()].copy()

    def _export(self, elts, g0, g1, sk, pk):
        self._check(self.lib.ref_export_keys(self._h, _u64p(elts), _u64p(g0), _u64p(g1), _vp(sk), _u64p(pk)))

    def _apply_galois(self, b, elt, ct, out):
        self._check(self.lib.ref_apply_galois(self._h, C.c_int(b), C.c_uint64(elt), _u64p(ct), C.c_int(1), _u64p(out)))

    def apply_galois_coeff(self, b: int, elt: int, ct: np.ndarray) -> np.ndarray:
        """The reference's coefficient-form apply_galois (context.cpp:460-465, 499-503)."""
        ct = np.ascontiguousarray(ct, np.uint64)
        out = np.zeros_like(ct)
        self._check(self.lib.ref_apply_galois(self._h, C.c_int(b), C.c_uint64(elt), _u64p(ct), C.c_int(0), _u64p(out)))
        return out

    def load_inputs(self, inputs: np.ndarray, f: int, form: int = 1):
        inputs = np.ascontiguousarray(inputs, np.uint64)
        self._check(self.lib.ref_load_inputs(self._h, _u64p(inputs), C.c_uint64(inputs.shape[0]), C.c_uint64(f), C.c_int(form)))

    def set_weights(self, w):
        w = np.ascontiguousarray(w, np.int64)
        f, cols = w.shape
        self._wcols = cols
        self._check(self.lib.ref_encode_weights(self._h, _i64p(w), C.c_uint64(f), C.c_uint64(cols), None))

    def set_bias(self, bias):
        bias = np.ascontiguousarray(bias, np.int64)
        self._check(self.lib.ref_set_bias(self._h, _i64p(bias), C.c_uint64(len(bias))))

    def encode_weights(self, w: np.ndarray) -> np.ndarray:
        self._wcols = np.asarray(w).shape[1]
        return super().encode_weights(w)

    def keygen_next(self, seed: int, count: int) -> np.ndarray:
        """Raw draws following TwinContext::keygen(Prng(seed))."""
        out = np.zeros(count, np.uint64)
        self._check(self.lib.ref_keygen_next(self._h, C.c_uint64(seed), C.c_uint64(count), _u64p(out)))
        return out

    def inputs_wire(self) -> bytes:
        """The loaded/encoded inputs as the client's HECT blob list."""
        n = C.c_uint64(0)
        self._check(self.lib.ref_inputs_wire(self._h, None, C.c_uint64(0), C.byref(n)))
        out = np.zeros(n.value, np.uint8)
        self._check(self.lib.ref_inputs_wire(self._h, out.ctypes.data_as(C.POINTER(C.c_uint8)), C.c_uint64(out.size), C.byref(n)))
        return out.tobytes()

    def server_wire(self, blobs: bytes, rows: int, threads: int = 0):
        """InferenceServer::do_infer's computation on a blob list; returns
        (response bytes, seconds)."""
        buf = np.frombuffer(blobs, np.uint8)
        n = C.c_uint64(0)
        secs = C.c_double(0)
        C_ = (rows * self._wcols + self.n - 1) // self.n
        cap = C_ * (8 * self.ct_words + 2 * (self.L[0] + self.L[1]) + 38)
        out = np.zeros(cap, np.uint8)
        self._check(self.lib.ref_server_wire(self._h, buf.ctypes.data_as(C.POINTER(C.c_uint8)), C.c_uint64(buf.size),
                                             C.c_uint64(rows), C.c_uint(threads), out.ctypes.data_as(C.POINTER(C.c_uint8)),
                                             C.c_uint64(cap), C.byref(n), C.byref(secs)))
        return out[: n.value].tobytes(), secs.value

    def matmul(self, R: int, cols: int, threads: int = 0, export: bool = True):
        C_ = (R * cols + self.n - 1) // self.n
        out = np.zeros((C_, self.ct_words), np.uint64) if export else None
        cnt = np.zeros(5, np.uint64)
        secs = C.c_double(0)
        self._check(self.lib.ref_matmul(self._h, C.c_uint(threads), _u64p(out), _u64p(cnt), C.byref(secs)))
        return out, cnt, secs.value

    def baseline_matmul(self, x, w, bias, export: bool = True):
        x = np.ascontiguousarray(x, np.int64)
        w = np.ascontiguousarray(w, np.int64)
        R, f = x.shape
        cols = w.shape[1]
        self.set_bias(bias)
        B = (R + self.n - 1) // self.n
        out = np.zeros((B, cols, self.ct_words), np.uint64) if export else None
        cnt = np.zeros(5, np.uint64)
        secs = C.c_double(0)
        self._check(self.lib.ref_baseline(self._h, _i64p(x), C.c_uint64(R), C.c_uint64(f), _i64p(w), C.c_uint64(cols),
                                          _u64p(out), _u64p(cnt), C.byref(secs)))
        return out, cnt, secs.value


# ---------------------------------------------------------------------------
# Seeded synthetic workload: data Prng(7); X row-major
# Bernoulli(p) scaled 2^6, W row-major N(0, sigma) scaled 2^14, bias N(0,0.1)
# scaled 2^20. Restated in numpy from the reference's Prng stream via heoracle.
# ---------------------------------------------------------------------------
def prng_stream(seed: int, count: int):
    lib = oracle_lib()
    raw = np.zeros(count, np.uint64)
    g = np.zeros(count, np.float64)
    u3 = np.zeros(count, np.uint64)
    lib.ho_prng(C.c_uint64(seed), C.c_uint64(count), _u64p(raw), g.ctypes.data_as(C.POINTER(C.c_double)), _u64p(u3))
    return raw, g, u3


def ref_prng_stream(seed: int, count: int):
    lib = ref_lib()
    raw = np.zeros(count, np.uint64)
    g = np.zeros(count, np.float64)
    u3 = np.zeros(count, np.uint64)
    lib.ref_prng(C.c_uint64(seed), C.c_uint64(count), _u64p(raw), g.ctypes.data_as(C.POINTER(C.c_double)), _u64p(u3))
    return raw, g, u3
