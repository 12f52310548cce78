"""Probe: one standard-algorithm call after warm-up (for launch lists; not a test)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2204_05496_b200 import Prng, baseline_matmul  # noqa: E402
from tests.helpers import synthetic  # noqa: E402

srv, q0, q1, _ = bench.make_server(8192, 0)
x3, w3, b3 = synthetic(1, 40000, 11, 0.03, 0.05)
baseline_matmul(srv, x3, w3, b3, Prng(2), Prng(3))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
baseline_matmul(srv, x3, w3, b3, Prng(2), Prng(3))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
