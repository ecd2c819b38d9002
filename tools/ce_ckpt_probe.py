"""Copy-engine D2D snapshot next to a running SIMT GEMM: does
cudaMemcpyAsync(DeviceToDevice) of 2 x 64 MiB on a side stream overlap the
FP32 GEMM without slowing it (the GEMM barely touches DRAM), and how fast is
it alone?  cuda-python drives the memcpy so no torch copy kernel is involved.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from cuda.bindings import runtime as cudart  # noqa: E402

from paper_1405_2912_b200 import kernels  # noqa: E402

n = 4096
nb = n * n * 4
a = torch.rand(n, n, device="cuda") + 1
b = torch.rand(n, n, device="cuda") + 1
c = torch.empty(n, n, device="cuda")
srcs = [torch.rand(n * n, device="cuda") for _ in range(2)]
dsts = [torch.empty(n * n, device="cuda") for _ in range(2)]
s_main = torch.cuda.Stream()
s_ce = torch.cuda.Stream(priority=0)


def ce_copy(st):
    for d, s in zip(dsts, srcs):
        err, = cudart.cudaMemcpyAsync(d.data_ptr(), s.data_ptr(), nb, cudart.cudaMemcpyKind.cudaMemcpyDeviceToDevice,
                                      st.cuda_stream)
        assert err == cudart.cudaError_t.cudaSuccess, err


def kern_copy(st):
    for d, s in zip(dsts, srcs):
        kernels.checkpoint(d, s, stream=st)


def timed(fn, st):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    fn()
    e1.record(st)
    return e0, e1


out = {}
for it in range(6):
    torch.cuda.synchronize()
    g0, g1 = timed(lambda: kernels.gemm_simt(a, b, c, stream=s_main), s_main)
    torch.cuda.synchronize()
    c0, c1 = timed(lambda: ce_copy(s_ce), s_ce)
    torch.cuda.synchronize()
    k0, k1 = timed(lambda: kern_copy(s_ce), s_ce)
    torch.cuda.synchronize()
    # overlapped: GEMM on main, CE copies on the side stream right after its launch
    o0, o1 = timed(lambda: kernels.gemm_simt(a, b, c, stream=s_main), s_main)
    x0, x1 = timed(lambda: ce_copy(s_ce), s_ce)
    torch.cuda.synchronize()
    if it >= 2:
        out.setdefault("gemm_alone_ms", []).append(g0.elapsed_time(g1))
        out.setdefault("ce_copy_2x64MiB_alone_us", []).append(1e3 * c0.elapsed_time(c1))
        out.setdefault("kernel_copy_2x64MiB_alone_us", []).append(1e3 * k0.elapsed_time(k1))
        out.setdefault("gemm_with_ce_ms", []).append(o0.elapsed_time(o1))
        out.setdefault("ce_copy_during_gemm_us", []).append(1e3 * x0.elapsed_time(x1))
print(json.dumps({k: sorted(v)[len(v) // 2] for k, v in out.items()}))
