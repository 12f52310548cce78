"""Probe (debug build abl/lib_t.so, -DHEI_W2_TRACE): phase timestamps of the
latency key switch k_rot_keyswitch_w2 for one C3 call (graphs off), per
(pair, prime) block and group: 0 start, 1 after the l == i products,
2..4 after each digit, 5 before the CTA barrier, 6 after the finish, 7 after
the next digit's INTT."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ["HEI_NO_GRAPHS"] = "1"
import bench  # noqa: E402
from paper_2204_05496_b200 import Prng, encode_inputs_device, encode_weights, matmul_device, native  # noqa: E402
from paper_2204_05496_b200.workload import config_workload  # noqa: E402

srv, q0, q1, _ = bench.make_server(8192, 0)
ctw = 2 * (len(q0) + len(q1)) * 8192
x, w, b = config_workload("c3")
ew = encode_weights(srv, w)
d_in = torch.empty((5, ctw), dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()
encode_inputs_device(srv, x, Prng(2), Prng(3), d_in.data_ptr(), st.cuda_stream)
o1 = torch.empty((1, ctw), dtype=torch.int32, device="cuda")
for _ in range(3):
    matmul_device(srv, d_in.data_ptr(), 1, ew, b, o1.data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
tr = np.zeros((256, 2, 8), dtype=np.uint64)
assert native.lib().hei_gpu_debug_w2_trace(tr.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
tr = tr[:110].astype(np.float64)
t0 = tr[:, :, 0].min()
rel = (tr - t0) / 1000.0
print("last rotation's launch (the NEXT=false kernel has no INTT, stamp 7 stays 0)")
for name, rows in (("branch0", slice(0, 110)),):
    pass
P = 10
b0 = np.array([k for k in range(110) if k % P < 6])
b1 = np.array([k for k in range(110) if k % P >= 6])
for nm, idx in (("b0", b0), ("b1", b1)):
    for g in (0, 1):
        r = rel[idx, g, :]
        print(nm, "grp", g, "mean us:", " ".join("%5.1f" % v for v in r.mean(axis=0)), " max end", "%5.1f" % r[:, 6].max())
