"""Probe: where the single-individual end-to-end call (C ABI, host u64
buffers) spends its time beyond the device fold (C3 shape)."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2204_05496_b200 import Prng, encode_inputs_device, encode_weights, matmul, matmul_device, native  # noqa: E402
from paper_2204_05496_b200.native import u64p, i64p  # noqa: E402
from paper_2204_05496_b200.workload import config_workload  # noqa: E402

srv, q0, q1, _ = bench.make_server(8192, 0)
ctw = 2 * (len(q0) + len(q1)) * 8192
x, w, b = config_workload("c3")
ew = encode_weights(srv, w)
d_in = torch.empty((5, ctw), dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()
encode_inputs_device(srv, x, Prng(2), Prng(3), d_in.data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
h_in = torch.empty((1, 5, ctw), dtype=torch.int64, pin_memory=True)
h_in.copy_(d_in.view(1, 5, ctw).to(torch.int64).cpu())
h_np = h_in.numpy().view(np.uint64)
o1 = torch.empty((1, ctw), dtype=torch.int32, device="cuda")
out_pinned = torch.empty((1, ctw), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
b = np.ascontiguousarray(b, dtype=np.int64)


def t_(f, n=50):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1000


print("device matmul_device (host clock)      %.3f ms" % t_(lambda: matmul_device(srv, d_in.data_ptr(), 1, ew, b, o1.data_ptr(), st.cuda_stream)))
print("host matmul() python, pageable out      %.3f ms" % t_(lambda: matmul(srv, h_np, ew, b)))
cnt = native.OpCounters()
print("host C call, pinned out                 %.3f ms" % t_(lambda: native.lib().hei_gpu_matmul(srv.handle, ew._h, u64p(h_np), C.c_int(0), C.c_uint64(1), i64p(b), u64p(out_pinned), C.byref(cnt))))
print("host C call, pinned out, no counters    %.3f ms" % t_(lambda: native.lib().hei_gpu_matmul(srv.handle, ew._h, u64p(h_np), C.c_int(0), C.c_uint64(1), i64p(b), u64p(out_pinned), None)))
