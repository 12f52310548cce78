"""Probe: single-individual call (C3) — device time per call (events around
each call on its stream) vs back-to-back calls (the bench's number), i.e.
the host gap between synchronous calls."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2204_05496_b200 import Prng, encode_inputs_device, encode_weights, matmul_device  # noqa: E402
from paper_2204_05496_b200.workload import config_workload  # noqa: E402

srv, q0, q1, _ = bench.make_server(8192, 0)
ctw = 2 * (len(q0) + len(q1)) * 8192
x, w, b = config_workload("c3")
ew = encode_weights(srv, w)
st = torch.cuda.Stream()
d_in = torch.empty((5, ctw), dtype=torch.int32, device="cuda")
encode_inputs_device(srv, x, Prng(2), Prng(3), d_in.data_ptr(), st.cuda_stream)
o1 = torch.empty((1, ctw), dtype=torch.int32, device="cuda")
b = np.ascontiguousarray(b, dtype=np.int64)
for _ in range(5):
    matmul_device(srv, d_in.data_ptr(), 1, ew, b, o1.data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
per = []
for _ in range(50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    matmul_device(srv, d_in.data_ptr(), 1, ew, b, o1.data_ptr(), st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    per.append(e0.elapsed_time(e1))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(50):
    matmul_device(srv, d_in.data_ptr(), 1, ew, b, o1.data_ptr(), st.cuda_stream)
e1.record(st)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    matmul_device(srv, d_in.data_ptr(), 1, ew, b, o1.data_ptr(), st.cuda_stream)
wall = (time.perf_counter() - t0) / 50
print("per-call events: median %.3f ms  min %.3f" % (np.median(per), min(per)))
print("back-to-back events: %.3f ms per call" % (e0.elapsed_time(e1) / 50))
print("host wall: %.3f ms per call" % (wall * 1000))
