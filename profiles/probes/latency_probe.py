"""Probe: single-individual latency (C3 shape) with more iterations (not a test)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2204_05496_b200 import Prng, encode_inputs_device, encode_weights, matmul_device  # noqa: E402
from tests.helpers import synthetic  # noqa: E402

n, f, cols = 8192, 40000, 11
srv, q0, q1, _ = bench.make_server(n, 0)
kc = (f + n - 1) // n
ctw = 2 * (len(q0) + len(q1)) * n
x, w, b = synthetic(1, f, cols, 0.03, 0.05)
ew = encode_weights(srv, w)
d_in = torch.empty((kc, ctw), dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()
encode_inputs_device(srv, x, Prng(2), Prng(3), d_in.data_ptr(), st.cuda_stream)
o1 = torch.empty((1, ctw), dtype=torch.int32, device="cuda")
for _ in range(20):
    matmul_device(srv, d_in.data_ptr(), 1, ew, b, o1.data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
res = []
for rep in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(50):
        matmul_device(srv, d_in.data_ptr(), 1, ew, b, o1.data_ptr(), st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / 50)
print("latency_ms", [round(r, 4) for r in res])
