"""Shared helpers for the parity tests: build a GPU server from an oracle
session (same keys), seeded synthetic data."""
from __future__ import annotations

import numpy as np

from oracle.oracle import T0, T1, Oracle, TwinParams, production_params  # noqa: F401


def gpu_server_from(o, device: int = 0, with_pk: bool = False, with_sk: bool = False):
    from paper_2204_05496_b200 import GpuTwinServer, ScalingConfig

    elts, gk, sk, pk = o.galois_keys()
    pks = None
    if with_pk:
        n0 = 2 * o.L[0] * o.n
        pks = [pk[:n0], pk[n0:]]
    srv = GpuTwinServer(o.n, (o.p.t0, o.p.t1), o.L, o.q, elts, gk,
                         ScalingConfig(o.p.s_x, o.p.s_w, o.p.in_bits), device=device, public_keys=pks,
                         security_level=o.p.sec)
    if with_sk:
        srv.upload_secret_keys(sk)
    return srv


def tiny_params(n: int) -> TwinParams:
    """test_matmul.cpp:40-42"""
    return TwinParams(n=n, t0=7681, t1=12289, sec=0, s_x=2, s_w=3, in_bits=3)


def random_mat(rng: np.random.Generator, r: int, c: int, mag: int) -> np.ndarray:
    return rng.integers(-mag, mag + 1, size=(r, c), dtype=np.int64)


def oracle_matmul(x, w, bias):
    """Exact integer product (test_matmul.cpp:44-55)."""
    return (x.astype(object) @ w.astype(object) + np.asarray(bias, dtype=object)).astype(np.int64)


def synthetic(R: int, f: int, cols: int, p_feat: float, w_sigma: float, seed: int = 7, b_sigma: float = 0.1):
    """Seeded stand-in for the BASELINE.json configs: Bernoulli(p) 0/1 features
    scaled 2^6, N(0, sigma) weights scaled 2^14, bias N(0, 0.1) scaled 2^20."""
    rng = np.random.default_rng(seed)
    x = (rng.random((R, f)) < p_feat).astype(np.int64) * 64
    w = np.round(rng.normal(0.0, w_sigma, (f, cols)) * 2 ** 14).astype(np.int64)
    b = np.round(rng.normal(0.0, b_sigma, cols) * 2 ** 20).astype(np.int64)
    return x, w, b
