"""Probe: host-side timeline of one single-individual C-ABI call (HEI_HOST_TRACE)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2204_05496_b200 import Prng, encode_inputs_device, encode_weights, matmul  # noqa: E402
from paper_2204_05496_b200.workload import config_workload  # noqa: E402

srv, q0, q1, _ = bench.make_server(8192, 0)
ctw = 2 * (len(q0) + len(q1)) * 8192
x, w, b = config_workload("c3")
ew = encode_weights(srv, w)
d_in = torch.empty((5, ctw), dtype=torch.int32, device="cuda")
encode_inputs_device(srv, x, Prng(2), Prng(3), d_in.data_ptr(), 0)
torch.cuda.synchronize()
h_in = torch.empty((1, 5, ctw), dtype=torch.int64, pin_memory=True)
h_in.copy_(d_in.view(1, 5, ctw).to(torch.int64).cpu())
h_np = h_in.numpy().view(np.uint64)
for k in range(6):
    print("call", k, file=sys.stderr)
    matmul(srv, h_np, ew, b)
import time  # noqa: E402
dd = torch.empty((1, 5, ctw), dtype=torch.int64, device="cuda")
for _ in range(3):
    dd.copy_(h_in, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    dd.copy_(h_in, non_blocking=True)
torch.cuda.synchronize()
print("torch H2D of the same pinned buffer: %.1f us" % ((time.perf_counter() - t0) / 20 * 1e6), file=sys.stderr)
