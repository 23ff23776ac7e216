"""A/B of the single explicit apply at C3: the Morton plan with plan-numbered
columns (u gather, ELL kernel, y scatter) against node-numbered columns
(mf_plan_apply_direct, one launch).  Prints stage times and checks bitwise."""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1912_13282_b200 as mf  # noqa: E402
from paper_1912_13282_b200 import _lib, workloads  # noqa: E402

w = workloads.c3()
nodes = mf.find_closest_stencils(mf.NodeSet(w.positions, w.types), w.n)
store = mf.compute_weights(nodes, mf.RbfFd(mf.Polyharmonic(3), 2, "support", "lu"), ["laplacian"])
mat = store.matrix("laplacian")
lib = _lib.load()
u = torch.from_numpy(w.field).cuda()
N = w.N
p = mat.plan(True)
s = mat._s
order, inv = s._order(True)
total = ((N + 31) // 32) * 32 * s.n
idx2 = torch.empty(total, dtype=torch.int32, device="cuda")
val2 = torch.empty(total, dtype=torch.float64, device="cuda")
len2 = torch.empty(N, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def build2():
    _lib.check(lib.mf_plan_build(s.indptr.data_ptr(), s.indices.data_ptr(), mat.data_device.data_ptr(), N, s.n,
                                 order.data_ptr(), None, idx2.data_ptr(), val2.data_ptr(), len2.data_ptr(),
                                 _lib.stream_ptr()), "plan2")


build2()
y1 = mat.apply_device(u)
y2 = torch.empty(N, dtype=torch.float64, device="cuda")
_lib.check(lib.mf_plan_apply_direct(idx2.data_ptr(), val2.data_ptr(), len2.data_ptr(), N, s.n, order.data_ptr(),
                                    u.data_ptr(), y2.data_ptr(), _lib.stream_ptr()), "direct")
torch.cuda.synchronize()
assert torch.equal(y1, y2), "direct apply differs"
res = {"plan_apply_stage": [], "direct": [], "plan_build_inv": [], "plan_build_noinv": []}
for it in range(6):
    for name, fn in [("plan_apply_stage", lambda: mat.apply_device(u)),
                     ("direct", lambda: lib.mf_plan_apply_direct(idx2.data_ptr(), val2.data_ptr(), len2.data_ptr(),
                                                                 N, s.n, order.data_ptr(), u.data_ptr(),
                                                                 y2.data_ptr(), _lib.stream_ptr())),
                     ("plan_build_inv", lambda: s.plan_values(mat.data_device, True)),
                     ("plan_build_noinv", build2)]:
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        res[name].append(a.elapsed_time(b))
for k, v in res.items():
    print(k, " ".join(f"{x * 1e3:.1f}" for x in v), "us")
