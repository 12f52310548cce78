"""Golden digests of the UNMODIFIED reference on BASELINE.json's five configs.

Runs oracle/_ref/libheiref.so (the reference compiled in place from
/root/reference by oracle/Makefile) on the seeded workloads of
paper_2204_05496_b200/workload.py with the SURVEY §8(d) seeds -- keys
TwinContext::keygen(util::Prng(1)), client encryption client_backend(keys, 2)
(branch streams Prng(2), Prng(3)), data util::Prng(7) -- and writes one
fixture per case to tests/golden/configs/<case>.json:

  fast_<c>      hei::matmul::matmul (matmul.cpp:239-255): SHA-256 of the
                encrypted inputs [R][k][twin ct] u64 (eval form), of the packed
                output [C][twin ct] u64 (eval form), of the server wire response
                (InferenceServer::do_infer on the client's HECT blobs,
                server.cpp:112-172 / serialize.cpp:63-78), the decrypted scores
                and the op counters.
  stream_c5     the full C5 batch through MatmulStream in 64-row blocks (the
                reference bench's streaming shape), packed-output digest.
  base_<c>      hei::matmul::baseline_matmul (matmul.cpp:273-344) on a fresh
                client (Prng(2), Prng(3) untouched): block digests, counters,
                decrypted scores.

Run in the build container (CPU only; the slow cases take minutes to an hour):

    make -C oracle ref
    python tests/golden/make_golden_configs.py fast_c1 fast_c2 fast_c3 fast_c4 fast_c5s
    python tests/golden/make_golden_configs.py base_c2 base_c3
    python tests/golden/make_golden_configs.py stream_c5
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference, production_params  # noqa: E402
from paper_2204_05496_b200.workload import CONFIGS, config_workload  # noqa: E402

OUT = os.path.join(HERE, "configs")
C5_SLICE_ROWS = 128  # 128 x 33 = 4224 (individual, class) pairs: the C5 full-batch kernels


def sha(a) -> str:
    if isinstance(a, (bytes, bytearray)):
        return hashlib.sha256(a).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _session(n: int) -> Reference:
    return Reference(production_params(n), key_seed=1, enc_seed=2)


def fast(cfg: str, rows: int | None = None, wire: bool = True) -> dict:
    R, f, cols, n, pf, ws = CONFIGS[cfg]
    R = rows or R
    x, w, b = config_workload(cfg, rows=R)
    r = _session(n)
    t0 = time.time()
    inputs = r.encode_inputs(x)
    r.set_weights(w)
    r.set_bias(b)
    packed, cnt, secs = r.matmul(R, cols, threads=0)
    res = r.unpack(packed, R, cols)
    out = {"config": cfg, "rows": R, "f": f, "cols": cols, "n": n, "q": r.q, "L": r.L,
           "x_sha256": sha(x), "w_sha256": sha(w), "b": b.tolist(),
           "inputs_sha256": sha(inputs), "packed_sha256": sha(packed), "packed_words": int(packed.size),
           "packed_head": [int(v) for v in packed.reshape(-1)[:8]],
           "counters": [int(v) for v in cnt], "result_sha256": sha(res),
           "result_equals_integer_product": bool(np.array_equal(res, x @ w + b)),
           "reference_matmul_s": secs}
    if R * cols <= 64:
        out["result"] = res.tolist()
    if wire:
        blobs = r.inputs_wire()
        resp, wsecs = r.server_wire(blobs, R, threads=0)
        out.update({"wire_request_sha256": sha(blobs), "wire_request_bytes": len(blobs),
                    "wire_response_sha256": sha(resp), "wire_response_bytes": len(resp), "reference_wire_s": wsecs})
    out["generator_s"] = time.time() - t0
    r.close()
    return out


def stream_c5() -> dict:
    import ctypes as C

    R, f, cols, n, pf, ws = CONFIGS["c5"]
    x, w, b = config_workload("c5")
    r = _session(n)
    t0 = time.time()
    r.set_weights(w)
    r.set_bias(b)
    Cn = (R * cols + n - 1) // n
    packed = np.zeros((Cn, r.ct_words), np.uint64)
    cnt = np.zeros(5, np.uint64)
    secs = C.c_double(0)
    x = np.ascontiguousarray(x)
    r._check(r.lib.ref_stream_matmul(r._h, x.ctypes.data_as(C.POINTER(C.c_int64)), C.c_uint64(R), C.c_uint64(f),
                                     C.c_uint64(64), C.c_uint(0), packed.ctypes.data_as(C.POINTER(C.c_uint64)),
                                     cnt.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(secs)))
    res = r.unpack(packed, R, cols)
    out = {"config": "c5", "rows": R, "f": f, "cols": cols, "n": n, "q": r.q, "L": r.L,
           "x_sha256": sha(x), "w_sha256": sha(w), "b": b.tolist(),
           "packed_sha256": sha(packed), "packed_words": int(packed.size),
           "packed_head": [int(v) for v in packed.reshape(-1)[:8]],
           "counters": [int(v) for v in cnt], "result_sha256": sha(res),
           "result_equals_integer_product": bool(np.array_equal(res, x @ w + b)),
           "reference_compute_s": secs.value, "generator_s": time.time() - t0,
           "threads": os.cpu_count()}
    r.close()
    return out


def base(cfg: str) -> dict:
    R, f, cols, n, pf, ws = CONFIGS[cfg]
    x, w, b = config_workload(cfg)
    r = _session(n)
    blocks, cnt, secs = r.baseline_matmul(x, w, b)
    out = {"config": cfg, "algorithm": "baseline_matmul", "rows": R, "f": f, "cols": cols, "n": n,
           "x_sha256": sha(x), "w_sha256": sha(w), "b": b.tolist(),
           "blocks_sha256": sha(blocks), "blocks_words": int(blocks.size),
           "blocks_head": [int(v) for v in blocks.reshape(-1)[:8]],
           "counters": [int(v) for v in cnt], "reference_baseline_s": secs, "threads": 1}
    # decrypt each block with the same client (unpack_baseline, matmul.cpp:346-358)
    dec = np.stack([r.decrypt_signed(blocks[0, j])[0][:R] for j in range(cols)], axis=1)
    out["result"] = dec.tolist()
    out["result_equals_integer_product"] = bool(np.array_equal(dec, x @ w + b))
    r.close()
    return out


CASES = {
    "fast_c1": lambda: fast("c1"),
    "fast_c2": lambda: fast("c2"),
    "fast_c3": lambda: fast("c3"),
    "fast_c4": lambda: fast("c4"),
    "fast_c5s": lambda: fast("c5", rows=C5_SLICE_ROWS, wire=False),
    "stream_c5": stream_c5,
    "base_c2": lambda: base("c2"),
    "base_c3": lambda: base("c3"),
}


def main(names):
    os.makedirs(OUT, exist_ok=True)
    for nm in names or list(CASES):
        t0 = time.time()
        d = CASES[nm]()
        d["case"] = nm
        d["generator"] = "tests/golden/make_golden_configs.py via oracle/_ref/libheiref.so (reference compiled in place)"
        with open(os.path.join(OUT, nm + ".json"), "w") as fh:
            json.dump(d, fh, indent=1)
        print(f"{nm}: {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
