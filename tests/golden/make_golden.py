"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/libheiref.so, compiled in place from /root/reference
by oracle/Makefile). Run in the build container:

    make -C oracle ref && python tests/golden/make_golden.py

Every array here is the reference's own output on seeded inputs; large
outputs are stored as SHA-256 digests plus a short prefix.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import T0, T1, T1_16K, Reference, TwinParams, ref_lib, ref_prng_stream  # noqa: E402
import ctypes as C  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    lib = ref_lib()
    out = {"generator": "tests/golden/make_golden.py via oracle/_ref/libheiref.so (reference compiled in place)"}
    arrays = {}

    # ---- modulus chains (params.cpp:84-114)
    chains = {}
    buf = (C.c_uint64 * 16)()
    cnt = C.c_uint32()
    for n, t, sec in [(8192, T0, 128), (8192, T1, 128), (16384, T0, 128), (16384, T1_16K, 128), (8, 97, 0), (8, 17, 0),
                      (32, 7681, 0), (32, 12289, 0), (8, T0, 0), (4096, 40961, 0)]:
        rc = lib.ref_default_primes(C.c_uint32(n), C.c_uint64(t), C.c_int(sec), buf, C.byref(cnt))
        chains[f"{n}/{t}/{sec}"] = list(buf[: cnt.value]) if rc == 0 else {"error": rc}
    rc = lib.ref_default_primes(C.c_uint32(16384), C.c_uint64(T1), C.c_int(128), buf, C.byref(cnt))
    chains["16384/114689/128"] = {"error": rc, "message": lib.ref_last_error().decode()}
    out["chains"] = chains

    # ---- Prng stream (rng.hpp:19-68)
    raw, g, u3 = ref_prng_stream(5, 64)
    out["prng_seed5"] = {"raw": [int(v) for v in raw[:16]], "gauss": [float(v) for v in g[:16]], "uniform3": [int(v) for v in u3]}

    # ---- NTT known answers (modops_scalar.cpp:45-81)
    ntt = {}
    for n in (32, 8192, 16384):
        for q in chains[f"{n}/{T0}/128"] if n >= 8192 else chains["32/7681/0"]:
            rng = np.random.default_rng(n + q % 1000)
            a = rng.integers(0, q, size=n, dtype=np.uint64)
            f = a.copy()
            assert lib.ref_ntt(C.c_uint32(n), C.c_uint64(q), f.ctypes.data_as(C.POINTER(C.c_uint64)), 0, 1) == 0
            key = f"{n}/{q}"
            ntt[key] = {"seed": int(n + q % 1000), "fwd_sha256": digest(f), "fwd_head": [int(v) for v in f[:8]]}
            if n == 32:
                arrays[f"ntt_in_{key}"] = a
                arrays[f"ntt_out_{key}"] = f
    out["ntt"] = ntt

    # ---- tiny twin sessions: keys, encryption, fast matmul (full arrays)
    tiny = {}
    for name, p, ks, es, shape in [
        ("worked_8", TwinParams(8, 97, 17, 0, 1, 1, 2), 7, 8, None),
        ("tiny_32", TwinParams(32, 7681, 12289, 0, 2, 3, 3), 72, 73, (5, 70, 3)),
    ]:
        r = Reference(p, ks, es)
        elts, gk, sk, pk = r.galois_keys()
        if shape is None:
            x = np.array([[1, 2, 3], [4, 5, 6]], dtype=np.int64)  # test_matmul.cpp:69-106
            w = np.array([[1, 0], [0, 1], [1, 1]], dtype=np.int64)
            b = np.zeros(2, dtype=np.int64)
        else:
            R, f, cols = shape
            rng = np.random.default_rng(11)
            x = rng.integers(-20, 21, size=(R, f), dtype=np.int64)
            w = rng.integers(-7, 8, size=(f, cols), dtype=np.int64)
            b = rng.integers(-500, 501, size=cols, dtype=np.int64)
        inputs = r.encode_inputs(x)
        wp = r.encode_weights(w)
        r.set_weights(w)
        r.set_bias(b)
        packed, cnt, _ = r.matmul(x.shape[0], w.shape[1], threads=1)
        res = r.unpack(packed, x.shape[0], w.shape[1])
        tiny[name] = {"params": p.__dict__, "key_seed": ks, "enc_seed": es, "L": r.L, "q": r.q, "elts": [int(e) for e in elts],
                      "counters": [int(v) for v in cnt], "result": res.tolist(),
                      "gk_sha256": [digest(gk[0]), digest(gk[1])], "pk_sha256": digest(pk)}
        for k, v in {"x": x, "w": w, "b": b, "inputs": inputs, "weights": wp, "packed": packed, "sk": sk}.items():
            arrays[f"{name}_{k}"] = v
        # one rotation + fold on a fresh ciphertext (context.cpp:428-507, backend.cpp:63-73)
        ct = inputs[0, 0]
        n0 = 2 * r.L[0] * p.n
        arrays[f"{name}_galois_in"] = ct
        arrays[f"{name}_galois_out"] = np.stack([r.apply_galois(0, int(e), ct[:n0]) for e in elts])
        arrays[f"{name}_fold_out"] = r.sum_all_slots(ct)
        r.close()
    out["tiny"] = tiny

    # ---- production N = 8192 session, C1 restricted to 3 classes
    p = TwinParams(8192, T0, T1, 128)
    r = Reference(p, 1, 2)
    elts, gk, sk, pk = r.galois_keys()
    rng = np.random.default_rng(7)
    x = (rng.random((1, 1000)) < 0.05).astype(np.int64) * 64
    w = np.round(rng.normal(0, 0.1, (1000, 3)) * 2 ** 14).astype(np.int64)
    b = np.round(rng.normal(0, 0.1, 3) * 2 ** 20).astype(np.int64)
    inputs = r.encode_inputs(x)
    r.set_weights(w)
    r.set_bias(b)
    packed, cnt, _ = r.matmul(1, 3, threads=1)
    res = r.unpack(packed, 1, 3)
    out["prod_c1_3"] = {"L": r.L, "q": r.q, "elts": [int(e) for e in elts], "gk_sha256": [digest(gk[0]), digest(gk[1])],
                        "pk_sha256": digest(pk), "sk_sha256": digest(sk), "inputs_sha256": digest(inputs),
                        "packed_sha256": digest(packed), "packed_head": [int(v) for v in packed[0, :8]],
                        "counters": [int(v) for v in cnt], "result": res.tolist(), "x_sha256": digest(x), "w_sha256": digest(w),
                        "b": b.tolist()}
    r.close()

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "golden_arrays.npz"), **arrays)
    print("wrote", os.path.join(HERE, "golden.json"), "and golden_arrays.npz")


if __name__ == "__main__":
    main()
