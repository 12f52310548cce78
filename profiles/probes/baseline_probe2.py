"""Probe: standard algorithm (baseline_matmul) timing at C3, repeated (not a test)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2204_05496_b200 import Prng, baseline_matmul  # noqa: E402
from tests.helpers import synthetic  # noqa: E402

n = 8192
srv, q0, q1, _ = bench.make_server(n, 0)
x3, w3, b3 = synthetic(1, 40000, 11, 0.03, 0.05)
for it in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    baseline_matmul(srv, x3, w3, b3, Prng(2), Prng(3))
    print("baseline ms %.1f" % ((time.perf_counter() - t0) * 1000), flush=True)
