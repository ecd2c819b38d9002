"""SIMT + TC replicas on separate streams: does the TC kernel fill the SIMT tail?"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels  # noqa: E402
from paper_1405_2912_b200._lib import HF_GEMM_COSCHEDULE  # noqa: E402

n = 4096
d = "cuda:0"
a = torch.rand(n, n, device=d) + 1
b = torch.rand(n, n, device=d) + 1
c1, c2 = torch.empty(n, n, device=d), torch.empty(n, n, device=d)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()


def timed(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(iters):
        fn()
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def pair(tc_mode, simt_first=True):
    def f():
        s1.wait_stream(main)
        s2.wait_stream(main)
        if simt_first:
            kernels.gemm_simt(a, b, c1, stream=s1)
            kernels.gemm_tc(a, b, c2, mode=tc_mode, stream=s2)
        else:
            kernels.gemm_tc(a, b, c2, mode=tc_mode, stream=s2)
            kernels.gemm_simt(a, b, c1, stream=s1)
        main.wait_stream(s1)
        main.wait_stream(s2)
    return f


print("simt alone", timed(lambda: kernels.gemm_simt(a, b, c1)))
print("tc alone persistent", timed(lambda: kernels.gemm_tc(a, b, c2)))
print("tc alone cosched", timed(lambda: kernels.gemm_tc(a, b, c2, mode=HF_GEMM_COSCHEDULE)))
print("serial simt+tc", timed(lambda: (kernels.gemm_simt(a, b, c1), kernels.gemm_tc(a, b, c2))))
print("pair simt-first persistent-tc", timed(pair(0)))
print("pair simt-first cosched-tc", timed(pair(HF_GEMM_COSCHEDULE)))
print("pair tc-first cosched-tc", timed(pair(HF_GEMM_COSCHEDULE, simt_first=False)))
