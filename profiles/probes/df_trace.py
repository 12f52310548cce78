"""Probe: dataflow-fold task timeline (HEI_DF_TRACE) for one C3 call."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2204_05496_b200 import Prng, encode_inputs_device, encode_weights, matmul_device  # noqa: E402
from paper_2204_05496_b200.workload import config_workload  # noqa: E402

path = "gpurun_out/df_trace.bin"
srv, q0, q1, _ = bench.make_server(8192, 0)
ctw = 2 * (len(q0) + len(q1)) * 8192
st = torch.cuda.Stream()
x, w, b = config_workload("c3")
ew = encode_weights(srv, w)
d_in = torch.empty((5, ctw), dtype=torch.int32, device="cuda")
encode_inputs_device(srv, x, Prng(2), Prng(3), d_in.data_ptr(), st.cuda_stream)
o1 = torch.empty((1, ctw), dtype=torch.int32, device="cuda")
for _ in range(3):
    matmul_device(srv, d_in.data_ptr(), 1, ew, b, o1.data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
os.environ["HEI_DF_TRACE"] = path
if os.path.exists(path):
    os.remove(path)
matmul_device(srv, d_in.data_ptr(), 1, ew, b, o1.data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
del os.environ["HEI_DF_TRACE"]
tr = np.fromfile(path, np.uint64).reshape(-1, 4)
tr = tr[tr[:, 2] > 0]
t0 = tr[:, 0].min()
ids = (tr[:, 3] >> np.uint64(32)).astype(np.uint64)
isk = (ids >> np.uint64(30)) & np.uint64(3)
s_ = (ids >> np.uint64(26)) & np.uint64(15)
wait = (tr[:, 1] - tr[:, 0]) / 1000.0
run = (tr[:, 2] - tr[:, 1]) / 1000.0
print("tasks %d, span %.1f us" % (len(tr), (tr[:, 2].max() - t0) / 1000.0))
for k, nm in ((0, "D"), (1, "R"), (2, "K")):
    m = isk == k
    print("%s: n=%d run mean %.2f us p50 %.2f p90 %.2f; wait mean %.2f" % (nm, m.sum(), run[m].mean(), np.median(run[m]),
                                                                         np.percentile(run[m], 90), wait[m].mean()))
for s in range(15):
    m = s_ == s
    if m.any():
        print("rotation %2d: start %.1f us end %.1f us" % (s, (tr[m, 1].min() - t0) / 1000.0, (tr[m, 2].max() - t0) / 1000.0))
sms = (tr[:, 3] & np.uint64(0xffffffff))
print("distinct SMs", len(np.unique(sms)), "busy fraction %.2f" % (run.sum() / (len(np.unique(sms)) * 2 * (tr[:, 2].max() - t0) / 1000.0)))
