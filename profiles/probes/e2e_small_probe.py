"""Probe: where a single-individual host-buffer call spends its time (not a test)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2204_05496_b200 import Prng, encode_inputs_device, encode_weights, matmul, matmul_device, native  # noqa: E402
from tests.helpers import synthetic  # noqa: E402

n, f, cols = 8192, int(sys.argv[1]) if len(sys.argv) > 1 else 40000, 11
srv, q0, q1, _ = bench.make_server(n, 0)
kc = (f + n - 1) // n
ctw = 2 * (len(q0) + len(q1)) * n
x, w, b = synthetic(1, f, cols, 0.03, 0.05)
ew = encode_weights(srv, w)
d_in = torch.empty((kc, ctw), dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()
encode_inputs_device(srv, x, Prng(2), Prng(3), d_in.data_ptr(), st.cuda_stream)
o1 = torch.empty((1, ctw), dtype=torch.int32, device="cuda")
h_in = torch.empty((1, kc, ctw), dtype=torch.int64, pin_memory=True)
h_in.copy_(d_in.view(1, kc, ctw).to(torch.int64).cpu())
h_np = h_in.numpy().view(np.uint64)
torch.cuda.synchronize()


def wall(fn, it=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(it):
        fn()
    torch.cuda.synchronize()
    return 1000 * (time.perf_counter() - t0) / it


def dev_sync():
    matmul_device(srv, d_in.data_ptr(), 1, ew, b, o1.data_ptr(), st.cuda_stream)
    st.synchronize()


print("device call + sync  %.3f ms" % wall(dev_sync))
print("host-buffer matmul  %.3f ms" % wall(lambda: matmul(srv, h_np, ew, b)))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(100):
    matmul_device(srv, d_in.data_ptr(), 1, ew, b, o1.data_ptr(), st.cuda_stream)
e1.record(st)
torch.cuda.synchronize()
print("device events       %.3f ms" % (e0.elapsed_time(e1) / 100))
