"""Probe: single-individual (C3) and small-batch latency of matmul_device,
CUDA-event timed (not a test)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2204_05496_b200 import Prng, encode_inputs_device, encode_weights, matmul_device  # noqa: E402
from paper_2204_05496_b200.workload import config_workload, workload  # noqa: E402

srv, q0, q1, _ = bench.make_server(8192, 0)
ctw = 2 * (len(q0) + len(q1)) * 8192
st = torch.cuda.Stream()
for R in (1, 2):
    x, w, b = config_workload("c3") if R == 1 else workload(R, 40000, 11, 0.03, 0.05)
    ew = encode_weights(srv, w)
    d_in = torch.empty((R * 5, ctw), dtype=torch.int32, device="cuda")
    encode_inputs_device(srv, x, Prng(2), Prng(3), d_in.data_ptr(), st.cuda_stream)
    o1 = torch.empty((1, ctw), dtype=torch.int32, device="cuda")
    for _ in range(5):
        matmul_device(srv, d_in.data_ptr(), R, ew, b, o1.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(50):
        matmul_device(srv, d_in.data_ptr(), R, ew, b, o1.data_ptr(), st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    print("dataflow=%s R=%d: %.3f ms per call" % (os.environ.get("HEI_DATAFLOW", "1"), R, e0.elapsed_time(e1) / 50))
