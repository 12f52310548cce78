"""Seeded synthetic workloads for BASELINE.json's five configs.

The reference uses no public dataset on this path,
so seeded synthetic inputs with the paper's shapes stand in for it. All draws
come from the reference's own generator, ``util::Prng`` (mt19937_64 +
hand-rolled distributions, proj/include/hei/util/rng.hpp:19-68), replayed by
the product's host ``Prng`` (hei_gpu_prng_draw):

* X  (R x f, row-major): ``uniform_double() < p``   -> 0/1, scale_value(., 6)
* W  (f x cols, row-major): ``gaussian() * sigma_w`` -> scale_value(., 14)
* bias (cols): ``gaussian() * sigma_b``              -> scale_value(., 20)

in that order from one stream, ``Prng(7)``. ``uniform_double`` is
``(v >> 11) * 2^-53`` (rng.hpp:41-43), exact in numpy. ``gaussian`` is
Box-Muller with one cached spare (rng.hpp:46-62); it is evaluated with
Python's ``math`` module, i.e. glibc's log/sqrt/sin/cos -- the same libm the
reference's std:: calls resolve to -- never numpy's SIMD transcendental
kernels, so the doubles are the reference's to the bit.
"""
from __future__ import annotations

import math

import numpy as np

from .matmul import Prng, scale_value

CONFIGS = {
    # name: (R, f, cols, N, p_feat, w_sigma)   BASELINE.json configs[0..4]
    "c1": (1, 1000, 11, 8192, 0.05, 0.1),
    "c2": (1, 10000, 11, 8192, 0.05, 0.1),
    "c3": (1, 40000, 11, 8192, 0.03, 0.05),
    "c4": (256, 40000, 11, 8192, 0.03, 0.05),
    "c5": (4096, 40000, 33, 16384, 0.03, 0.05),
}
B_SIGMA = 0.1  # bias N(0, 0.1) (stated for C3; used for every config)
DATA_SEED = 7
_TWO_PI = 6.283185307179586476925286766559  # rng.hpp:58 (same double as 2*math.pi)
_CHUNK = 1 << 24
_INV53 = 2.0 ** -53


class _Stream:
    """util::Prng consumer: buffered raw draws plus the reference's
    gaussian() with its cached spare (rng.hpp:46-62)."""

    def __init__(self, seed: int):
        self.rng = Prng(seed)
        self.buf = np.zeros(0, np.uint64)
        self.pos = 0
        self.have_spare = False
        self.spare = 0.0

    def raw(self, count: int) -> np.ndarray:
        assert self.pos == len(self.buf), "raw() after buffered gaussian draws"
        return self.rng.draw(count)

    def _uniform(self) -> float:  # uniform_double (rng.hpp:41-43)
        if self.pos == len(self.buf):
            self.buf = self.rng.draw(1 << 16)
            self.pos = 0
        v = int(self.buf[self.pos])
        self.pos += 1
        return float(v >> 11) * _INV53

    def gaussian(self) -> float:
        if self.have_spare:
            self.have_spare = False
            return self.spare
        u1 = self._uniform()
        while u1 <= 0.0:
            u1 = self._uniform()
        u2 = self._uniform()
        mag = math.sqrt(-2.0 * math.log(u1))
        self.spare = mag * math.sin(_TWO_PI * u2)
        self.have_spare = True
        return mag * math.cos(_TWO_PI * u2)

    def gaussians(self, count: int) -> np.ndarray:
        return np.array([self.gaussian() for _ in range(count)], np.float64)


def workload(R: int, f: int, cols: int, p_feat: float, w_sigma: float, b_sigma: float = B_SIGMA,
             seed: int = DATA_SEED, row_lo: int = 0, row_hi: int | None = None):
    """(x [row_hi-row_lo][f], w [f][cols], b [cols]) as scaled int64, drawn
    from util::Prng(seed) in the order above. Rows outside [row_lo, row_hi)
    are drawn and discarded (the stream is sequential), so every rank of a
    sharded run sees the same model and its own slice of one X."""
    row_hi = R if row_hi is None else row_hi
    if not (0 <= row_lo <= row_hi <= R):
        raise ValueError("workload: bad row range")
    st = _Stream(seed)
    x = np.zeros((row_hi - row_lo, f), np.int64)
    # X: R*f uniform draws, row-major; uniform_double() < p  <=>  (v >> 11) < p * 2^53
    # (both sides exact: v >> 11 < 2^53 converts exactly, the product by 2^53 is exact)
    total = R * f
    done = 0
    thr = p_feat
    while done < total:
        n = min(_CHUNK, total - done)
        v = st.raw(n)
        hit = (v >> np.uint64(11)).astype(np.float64) * _INV53 < thr
        lo = done
        hi = done + n
        a = max(lo, row_lo * f)
        b = min(hi, row_hi * f)
        if a < b:
            x.reshape(-1)[a - row_lo * f: b - row_lo * f] = hit[a - lo: b - lo].astype(np.int64)
        done += n
    xs = scale_value(1.0, 6)
    x *= xs  # scale_value(0, 6) = 0, scale_value(1, 6) = 64
    g = st.gaussians(f * cols + cols)
    w = np.array([scale_value(float(v) * w_sigma, 14) for v in g[: f * cols]], np.int64).reshape(f, cols)
    b = np.array([scale_value(float(v) * b_sigma, 20) for v in g[f * cols:]], np.int64)
    return x, w, b


def config_workload(name: str, row_lo: int = 0, row_hi: int | None = None, rows: int | None = None):
    """The seeded workload of BASELINE.json config `name` (c1..c5). `rows`
    overrides R (the model is then drawn after that many rows)."""
    R, f, cols, _, pf, ws = CONFIGS[name]
    R = rows or R
    return workload(R, f, cols, pf, ws, row_lo=row_lo, row_hi=row_hi)
