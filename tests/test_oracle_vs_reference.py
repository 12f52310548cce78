"""CPU: the C restatement against the reference itself (oracle/_ref), on
seeded random cases beyond the committed fixtures. Skipped where the
reference build is absent (the GPU box carries it only if built here)."""
import numpy as np
import pytest

from oracle.oracle import Oracle, Reference, TwinParams, ref_available

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("n,t0,t1", [(8, 97, 17), (32, 7681, 12289), (8, 1073872897, 114689)])
def test_random_shapes_bit_exact(n, t0, t1):
    p = TwinParams(n, t0, t1, 0, 1, 1, 2)
    rng = np.random.default_rng(n + t1)
    for trial in range(6):
        seed = 100 + trial
        o, r = Oracle(p, seed, seed + 1), Reference(p, seed, seed + 1)
        R = 1 + int(rng.integers(6))
        f = 1 + int(rng.integers(3 * n))
        cols = 1 + int(rng.integers(4))
        x = rng.integers(-5, 6, size=(R, f))
        w = rng.integers(-3, 4, size=(f, cols))
        b = rng.integers(-50, 51, size=cols)
        io, ir = o.encode_inputs(x), r.encode_inputs(x)
        assert np.array_equal(io, ir)
        wo = o.encode_weights(w)
        assert np.array_equal(wo, r.encode_weights(w))
        out, cnt = o.fast_matmul(io, f, wo, b)
        r.load_inputs(io, f)
        r.set_weights(w)
        r.set_bias(b)
        rout, rcnt, _ = r.matmul(R, cols)
        assert np.array_equal(out, rout)
        assert np.array_equal(cnt, rcnt)
        assert np.array_equal(o.unpack(out, R, cols), x @ w + b)


def test_baseline_bit_exact():
    p = TwinParams(32, 7681, 12289, 0, 2, 3, 3)
    rng = np.random.default_rng(3)
    R, f, cols = 40, 9, 3  # two sample blocks
    x = rng.integers(-20, 21, size=(R, f))
    w = rng.integers(-7, 8, size=(f, cols))
    b = rng.integers(-100, 101, size=cols)
    o, r = Oracle(p, 5, 6), Reference(p, 5, 6)
    out, cnt = o.baseline_matmul(x, w, b)
    rout, rcnt, _ = r.baseline_matmul(x, w, b)
    assert np.array_equal(out, rout)
    assert np.array_equal(cnt, rcnt)
    assert np.array_equal(o.unpack_baseline(out, R, cols), x @ w + b)


def test_coeff_form_inputs_bit_exact():
    p = TwinParams(32, 7681, 12289, 0, 2, 3, 3)
    o, r = Oracle(p, 9, 10), Reference(p, 9, 10)
    rng = np.random.default_rng(4)
    x = rng.integers(-9, 10, size=(2, 20))
    w = rng.integers(-3, 4, size=(20, 2))
    b = np.array([1, -1])
    # a coefficient-form copy of the inputs, made by the reference's own INTT
    import ctypes as C
    from oracle.oracle import ref_lib, _u64p

    io = o.encode_inputs(x)
    coeff = io.copy()
    lib = ref_lib()
    n = p.n
    for rr in range(coeff.shape[0]):
        for poly in range(2 * (o.L[0] + o.L[1])):
            bb = 0 if poly < 2 * o.L[0] else 1
            i = poly % o.L[0] if bb == 0 else (poly - 2 * o.L[0]) % o.L[1]
            q = o.q[(o.L[0] if bb else 0) + i]
            seg = np.ascontiguousarray(coeff[rr, 0, poly * n:(poly + 1) * n])
            lib.ref_ntt(C.c_uint32(n), C.c_uint64(q), _u64p(seg), 1, 0)
            coeff[rr, 0, poly * n:(poly + 1) * n] = seg
    out, _ = o.fast_matmul(coeff, 20, o.encode_weights(w), b, form=0)
    r.load_inputs(coeff, 20, form=0)
    r.set_weights(w)
    r.set_bias(b)
    rout, _, _ = r.matmul(2, 2)
    assert np.array_equal(out, rout)


@pytest.mark.parametrize("n", [32, 8192, 16384])
def test_wire_constants_match_reference(n):
    """hei_params_hash == BfvContext::hash() (params.cpp:68-82) and the HECT
    ciphertext size == save_ciphertext's output length (serialize.cpp:63-78);
    host-only C-ABI helpers, no device work."""
    import ctypes as C

    from oracle.oracle import production_params
    from paper_2204_05496_b200 import native
    from tests.helpers import tiny_params

    p = production_params(n) if n >= 8192 else tiny_params(n)
    ref = Reference(p, 1, 2)
    lib = native.lib()
    for b, t in enumerate((p.t0, p.t1)):
        q = np.ascontiguousarray(ref.q[: ref.L[0]] if b == 0 else ref.q[ref.L[0]:], np.uint64)
        h = lib.hei_params_hash(n, t, p.sec, q.ctypes.data_as(C.POINTER(C.c_uint64)), len(q))
        assert h == ref.hash[b]
    x = np.zeros((2, 3), np.int64)
    ref.encode_inputs(x)
    blobs = ref.inputs_wire()
    per = lib.hei_hect_ciphertext_bytes(n, ref.L[0]) + lib.hei_hect_ciphertext_bytes(n, ref.L[1])
    assert len(blobs) == 2 * per
    assert blobs[:4] == b"HECT" and blobs[18] == 5


@pytest.mark.parametrize("n,t", [(8, 7681), (32, 12289), (8, 1073872897), (4096, 114689), (8192, 1073872897),
                                 (8192, 114689), (16384, 1073872897), (16384, 163841)])
def test_default_q_primes_match_make_params(n, t):
    """hei_default_q_primes == bfv::make_params(n, t, .).q (params.cpp:84-114)."""
    import ctypes as C

    from paper_2204_05496_b200 import default_q_primes

    lib = ref_lib_handle()
    out = np.zeros(32, np.uint64)
    cnt = C.c_uint32(0)
    assert lib.ref_default_primes(C.c_uint32(n), C.c_uint64(t), C.c_int(0), out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                  C.byref(cnt)) == 0
    assert default_q_primes(n, t) == [int(v) for v in out[: cnt.value]]


def ref_lib_handle():
    from oracle.oracle import ref_lib

    return ref_lib()
