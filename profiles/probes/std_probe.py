"""Probe: the standard algorithm at C3 (warm call, then one call inside a
cudaProfilerStart/Stop range for `ncu --profile-from-start off`). Not a test."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2204_05496_b200 import Prng, baseline_matmul  # noqa: E402
from paper_2204_05496_b200.workload import config_workload  # noqa: E402

srv, q0, q1, _ = bench.make_server(8192, 0)
x, w, b = config_workload("c3")
baseline_matmul(srv, x, w, b, Prng(2), Prng(3))
torch.cuda.synchronize()
t0 = time.perf_counter()
baseline_matmul(srv, x, w, b, Prng(2), Prng(3))
print("standard algorithm C3: %.1f ms" % (1000 * (time.perf_counter() - t0)))
torch.cuda.cudart().cudaProfilerStart()
baseline_matmul(srv, x, w, b, Prng(2), Prng(3))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
