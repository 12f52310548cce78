"""Golden fixtures for the coefficient-form apply_galois
(BfvContext::apply_galois, context.cpp:460-465, 499-503; automorphism_coeff,
poly.cpp:107-122), written by the UNMODIFIED reference (oracle/_ref, compiled
in place). Run in the build container:

    make -C oracle ref && python tests/golden/make_golden_galois.py

Inputs are seeded residues in [0, q_i) per prime (any such array is a
coefficient-form ciphertext to apply_galois). N = 32: full arrays; N = 8192:
SHA-256 digests of the outputs (the test regenerates the same inputs).
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

from oracle.oracle import T0, T1, Reference, TwinParams  # noqa: E402

CASES = [  # name, params, key seed, enc seed, input seed
    ("tiny_32", TwinParams(32, 7681, 12289, 0, 2, 3, 3), 72, 73, 5),
    ("prod_8192", TwinParams(8192, T0, T1, 128), 1, 2, 6),
]


def coeff_input(q, L: int, n: int, seed: int) -> np.ndarray:
    """[2][L][n] u64, part p prime i uniform in [0, q_i)."""
    rng = np.random.default_rng(seed)
    ct = np.zeros((2, L, n), dtype=np.uint64)
    for i in range(L):
        ct[:, i, :] = rng.integers(0, int(q[i]), size=(2, n), dtype=np.uint64)
    return ct


def main():
    out, arrays = {"generator": "tests/golden/make_golden_galois.py via oracle/_ref/libheiref.so"}, {}
    for name, p, ks, es, seed in CASES:
        r = Reference(p, ks, es)
        elts = [int(e) for e in r.elts()]
        case = {"params": p.__dict__, "key_seed": ks, "enc_seed": es, "input_seed": seed, "elts": elts, "branches": {}}
        for b in (0, 1):
            L = int(r.L[b])
            q = [int(v) for v in r.q[(0 if b == 0 else int(r.L[0])):][:L]]
            ct = coeff_input(q, L, p.n, seed + b)
            outs = [r.apply_galois_coeff(b, e, ct.reshape(-1)) for e in elts]
            case["branches"][str(b)] = {"q": q, "out_sha256": [hashlib.sha256(o.tobytes()).hexdigest() for o in outs]}
            if p.n == 32:
                arrays[f"{name}_b{b}_in"] = ct
                arrays[f"{name}_b{b}_out"] = np.stack(outs)
        out[name] = case
        r.close()
    with open(os.path.join(HERE, "galois_coeff.json"), "w") as f:
        json.dump(out, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "galois_coeff.npz"), **arrays)


if __name__ == "__main__":
    main()
