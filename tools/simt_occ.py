"""SIMT GEMM at one vs two CTAs per SM (HF_SGEMM_COSCHED_SMEM in the
environment sets the co-scheduling smem reservation), alone and with the TC
and 3xBF16 replicas on concurrent streams (the HetTMR round on one GPU)."""
import json, os, sys, statistics
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels
from paper_1405_2912_b200._lib import HF_GEMM_COSCHEDULE as CS

n = 4096
a = torch.rand(n, n, device="cuda") + 1
b = torch.rand(n, n, device="cuda") + 1
cs = [torch.empty(n, n, device="cuda") for _ in range(3)]
ss = [torch.cuda.Stream(priority=-1), torch.cuda.Stream(), torch.cuda.Stream()]
main = torch.cuda.current_stream()


def run(which, iters=10):
    ts = []
    for it in range(iters + 3):
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(main)
        for s in ss:
            s.wait_stream(main)
        if "simt" in which:
            kernels.gemm_simt(a, b, cs[0], mode=CS, stream=ss[0])
        if "tc" in which:
            kernels.gemm_tc(a, b, cs[1], mode=CS, stream=ss[1])
        if "tc3" in which:
            kernels.gemm_tc(a, b, cs[2], mode=1 | CS, stream=ss[2])
        if "tc3pair" in which:
            kernels.gemm_tc(a, b, cs[2], mode=1, stream=ss[2])
        if "bf3" in which:
            kernels.gemm_tc(a, b, cs[2], mode=2 | CS, stream=ss[2])
        if "bf3pair" in which:
            kernels.gemm_tc(a, b, cs[2], mode=2, stream=ss[2])
        for s in ss:
            main.wait_stream(s)
        t1.record(main)
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(t0.elapsed_time(t1))
    return round(statistics.median(ts), 4)


out = {"smem": os.environ.get("HF_SGEMM_COSCHED_SMEM", "100000")}
for w in (("simt",), ("tc",), ("tc3",), ("tc3pair",), ("bf3",), ("bf3pair",), ("simt", "tc"),
          ("simt", "tc", "tc3"), ("simt", "tc", "bf3")):
    out["+".join(w)] = run(w)
print(json.dumps(out))
