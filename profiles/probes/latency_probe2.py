"""Probe: a few single-individual calls (for ncu launch lists; not a test)."""
import sys

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
for _ in range(3):
    matmul_device(srv, d_in.data_ptr(), 1, ew, b, o1.data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
print("ok")
from paper_2204_05496_b200 import native  # noqa: E402

native.kernel_timing(srv.handle, True)
for _ in range(5):
    matmul_device(srv, d_in.data_ptr(), 1, ew, b, o1.data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
ks = native.kernel_stats(srv.handle, 0)
dg = native.kernel_stats(srv.handle, 1)
native.kernel_timing(srv.handle, False)
print("keyswitch launches %d mean %.1f us; digits launches %d mean %.1f us" % (ks[0], 1000 * ks[1] / max(ks[0], 1), dg[0], 1000 * dg[1] / max(dg[0], 1)))
