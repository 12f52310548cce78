"""CPU: pin the C restatement (oracle/heoracle.c) against the golden fixtures
written by the reference itself (tests/golden/make_golden.py), and against the
reference's own known-answer tests restated here."""
import ctypes as C
import hashlib
import json
import os

import numpy as np
import pytest

from oracle.oracle import T0, T1, Oracle, OracleError, TwinParams, _u64p, oracle_lib, prng_stream

HERE = os.path.dirname(os.path.abspath(__file__))
G = json.load(open(os.path.join(HERE, "golden", "golden.json")))
A = np.load(os.path.join(HERE, "golden", "golden_arrays.npz"))


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_modulus_chains():
    lib = oracle_lib()
    buf = (C.c_uint64 * 16)()
    cnt = C.c_uint32()
    for key, want in G["chains"].items():
        n, t, sec = (int(v) for v in key.split("/"))
        rc = lib.ho_default_primes(C.c_uint32(n), C.c_uint64(t), C.c_int(sec), buf, C.byref(cnt))
        if isinstance(want, dict):
            assert rc == want["error"], key  # ParamError: t not 1 mod 2n
        else:
            assert rc == 0 and list(buf[: cnt.value]) == want, key


def test_prng_stream_matches_reference():
    raw, g, u3 = prng_stream(5, 64)
    want = G["prng_seed5"]
    assert [int(v) for v in raw[:16]] == want["raw"]
    assert [float(v) for v in g[:16]] == want["gauss"]
    assert [int(v) for v in u3] == want["uniform3"]


def test_ntt_known_answers():
    lib = oracle_lib()
    for key, want in G["ntt"].items():
        n, q = (int(v) for v in key.split("/"))
        rng = np.random.default_rng(want["seed"])
        a = rng.integers(0, q, size=n, dtype=np.uint64)
        f = a.copy()
        assert lib.ho_ntt(C.c_uint32(n), C.c_uint64(q), _u64p(f), 0) == 0
        assert digest(f) == want["fwd_sha256"], key
        assert [int(v) for v in f[:8]] == want["fwd_head"]
        if n == 32:
            assert np.array_equal(f, A[f"ntt_out_{key}"])
        back = f.copy()
        lib.ho_ntt(C.c_uint32(n), C.c_uint64(q), _u64p(back), 1)
        assert np.array_equal(back, a)


@pytest.mark.parametrize("name", ["worked_8", "tiny_32"])
def test_tiny_sessions_bit_exact(name):
    t = G["tiny"][name]
    p = TwinParams(**t["params"])
    o = Oracle(p, t["key_seed"], t["enc_seed"])
    assert o.L == t["L"] and o.q == t["q"]
    elts, gk, sk, pk = o.galois_keys()
    assert [int(e) for e in elts] == t["elts"]
    assert [digest(gk[0]), digest(gk[1])] == t["gk_sha256"]
    assert digest(pk) == t["pk_sha256"]
    assert np.array_equal(sk, A[f"{name}_sk"])
    x, w, b = A[f"{name}_x"], A[f"{name}_w"], A[f"{name}_b"]
    inputs = o.encode_inputs(x)
    assert np.array_equal(inputs, A[f"{name}_inputs"])
    wp = o.encode_weights(w)
    assert np.array_equal(wp, A[f"{name}_weights"])
    packed, cnt = o.fast_matmul(inputs, x.shape[1], wp, b)
    assert np.array_equal(packed, A[f"{name}_packed"])
    assert [int(v) for v in cnt] == t["counters"]
    assert o.unpack(packed, x.shape[0], w.shape[1]).tolist() == t["result"]
    ct = A[f"{name}_galois_in"]
    n0 = 2 * o.L[0] * p.n
    for k, e in enumerate(elts):
        assert np.array_equal(o.apply_galois(0, int(e), ct[:n0]), A[f"{name}_galois_out"][k])
    assert np.array_equal(o.sum_all_slots(ct), A[f"{name}_fold_out"])


def test_worked_example_slots():
    """test_matmul.cpp:69-106: 2x3 . 3x2 lands in slots [4, 5, 10, 11, 0...]."""
    t = G["tiny"]["worked_8"]
    o = Oracle(TwinParams(**t["params"]), t["key_seed"], t["enc_seed"])
    slots, budget = o.decrypt_signed(A["worked_8_packed"][0])
    assert slots.tolist() == [4, 5, 10, 11, 0, 0, 0, 0]
    assert budget > 0


def test_closed_form_counts():
    """test_matmul.cpp:293-324."""
    lib = oracle_lib()
    c = np.zeros(5, np.uint64)
    lib.ho_proposed_counts(C.c_uint64(1), C.c_uint64(1), C.c_uint64(8), C.c_uint32(8), _u64p(c))
    assert c[:3].tolist() == [2, 3, 4]
    lib.ho_proposed_counts(C.c_uint64(1), C.c_uint64(11), C.c_uint64(40960), C.c_uint32(8192), _u64p(c))
    assert c[0] == 66 and c[1] == 143 and c[3] == 5
    lib.ho_proposed_counts(C.c_uint64(543), C.c_uint64(11), C.c_uint64(40960), C.c_uint32(8192), _u64p(c))
    assert c[0] == 35838 and c[4] == 1
    lib.ho_baseline_counts(C.c_uint64(1), C.c_uint64(11), C.c_uint64(40960), C.c_uint32(8192), _u64p(c))
    assert c[0] == 450560 and c[1] == 0
    assert lib.ho_proposed_counts(C.c_uint64(0), C.c_uint64(1), C.c_uint64(1), C.c_uint32(8), _u64p(c)) == 1
    assert lib.ho_proposed_counts(C.c_uint64(1), C.c_uint64(1), C.c_uint64(1), C.c_uint32(12), _u64p(c)) == 1


@pytest.mark.slow
def test_production_c1_fixture():
    """N = 8192 production parameters, 1 x 1000 x 3: keys, inputs, packed
    output and decrypted scores equal the reference's (digests)."""
    t = G["prod_c1_3"]
    o = Oracle(TwinParams(8192, T0, T1, 128), 1, 2)
    assert o.L == t["L"] and o.q == t["q"]
    elts, gk, sk, pk = o.galois_keys()
    assert [digest(gk[0]), digest(gk[1])] == t["gk_sha256"]
    assert digest(sk) == t["sk_sha256"] and digest(pk) == t["pk_sha256"]
    rng = np.random.default_rng(7)
    x = (rng.random((1, 1000)) < 0.05).astype(np.int64) * 64
    w = np.round(rng.normal(0, 0.1, (1000, 3)) * 2 ** 14).astype(np.int64)
    b = np.array(t["b"], dtype=np.int64)
    assert digest(x) == t["x_sha256"] and digest(w) == t["w_sha256"]
    inputs = o.encode_inputs(x)
    assert digest(inputs) == t["inputs_sha256"]
    packed, cnt = o.fast_matmul(inputs, 1000, o.encode_weights(w), b)
    assert digest(packed) == t["packed_sha256"]
    assert [int(v) for v in cnt] == t["counters"]
    assert o.unpack(packed, 1, 3).tolist() == t["result"]
    assert t["result"] == (x @ w + b).tolist()


def test_error_contract():
    """Errors map to the reference's exception types (errors.hpp:13-53)."""
    with pytest.raises(OracleError) as e:
        Oracle(TwinParams(16384, T0, T1, 128))  # t1 not 1 mod 2n
    assert e.value.code == 1
    o = Oracle(TwinParams(8, 7681, 12289, 0, 6, 14, 8), 21, 22)
    x = np.ones((1, 4), np.int64)
    with pytest.raises(OracleError) as e:
        o.fast_matmul(o.encode_inputs(x), 4, o.encode_weights(np.ones((4, 1), np.int64)), [0])
    assert e.value.code == 3  # RangeError: capacity gate
