"""Probe: time the standard algorithm on the device for a C3 feature prefix
(used for ncu launch lists; not part of the test suite)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2204_05496_b200 import Prng, baseline_matmul, native  # noqa: E402
from tests.helpers import synthetic  # noqa: E402
import ctypes as C  # noqa: E402

f = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
srv, q0, q1 = bench.make_server(8192, 0)
rng = np.random.default_rng(5)
for b, qb in enumerate((q0, q1)):
    a = np.empty((2, len(qb), 8192), dtype=np.uint64)
    for i, qi in enumerate(qb):
        a[:, i, :] = rng.integers(0, qi, size=(2, 8192), dtype=np.uint64)
    native.check(native.lib().hei_gpu_upload_public_key(srv.handle, C.c_uint32(b), native.u64p(a.reshape(-1))))
x, w, bb = synthetic(1, f, 11, 0.03, 0.05)
baseline_matmul(srv, x, w, bb, Prng(2), Prng(3))
t0 = time.perf_counter()
baseline_matmul(srv, x, w, bb, Prng(2), Prng(3))
print(f"baseline f={f}: {1000 * (time.perf_counter() - t0):.1f} ms")
