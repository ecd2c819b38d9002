"""SIMT + TC replicas on separate streams: does the TC kernel fill the SIMT
tail?  Per-launch CUDA events on each stream (medians over iterations), so
the overlap of the two replicas is visible, plus the SM clock seen."""
import statistics
import subprocess
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels  # noqa: E402
from paper_1405_2912_b200._lib import HF_GEMM_COSCHEDULE  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d = "cuda:0"
a = torch.rand(n, n, device=d) + 1
b = torch.rand(n, n, device=d) + 1
c1, c2, c3 = torch.empty(n, n, device=d), torch.empty(n, n, device=d), torch.empty(n, n, device=d)
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=d)


def ev():
    return torch.cuda.Event(enable_timing=True)


def run(order, tc_mode, iters=15, simt_mode=None):
    """order: 'simt', 'tc', 'tc3', 'simt,tc[,tc3]' (concurrent, first listed
    launched first), 'serial'.  simt_mode defaults to tc_mode's cosched flag."""
    if simt_mode is None:
        simt_mode = tc_mode & HF_GEMM_COSCHEDULE
    res = []
    for it in range(iters + 3):
        flush.fill_(it & 0xFF)
        t0 = ev()
        t0.record(main)
        s1.wait_stream(main)
        s2.wait_stream(main)
        s3.wait_stream(main)
        marks = {}
        for what in order.split(","):
            st = {"simt": s1, "tc": s2, "tc3": s3}.get(what, main)
            if order == "serial":
                st = main
            e_a, e_b = ev(), ev()
            if what in ("simt", "serial"):
                e_a.record(st)
                kernels.gemm_simt(a, b, c1, mode=simt_mode, stream=st)
                e_b.record(st)
                marks["simt"] = (e_a, e_b)
            if what in ("tc", "serial"):
                e_c, e_d = ev(), ev()
                e_c.record(st)
                kernels.gemm_tc(a, b, c2, mode=tc_mode, stream=st)
                e_d.record(st)
                marks["tc"] = (e_c, e_d)
            if what == "tc3":
                e_c, e_d = ev(), ev()
                e_c.record(st)
                kernels.gemm_tc(a, b, c3, mode=1 | (tc_mode & HF_GEMM_COSCHEDULE), stream=st)
                e_d.record(st)
                marks["tc3"] = (e_c, e_d)
        main.wait_stream(s1)
        main.wait_stream(s2)
        main.wait_stream(s3)
        t1 = ev()
        t1.record(main)
        torch.cuda.synchronize()
        if it >= 3:
            row = {"total": t0.elapsed_time(t1)}
            for k, (x, y) in marks.items():
                row[k + "_start"] = t0.elapsed_time(x)
                row[k + "_end"] = t0.elapsed_time(y)
            res.append(row)
    keys = res[0].keys()
    return {k: round(statistics.median(r[k] for r in res), 4) for k in keys}


def clocks():
    try:
        return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                               "--format=csv,noheader"], capture_output=True, text=True, timeout=10).stdout.strip()
    except Exception as exc:  # noqa: BLE001
        return str(exc)


print("n", n, "clocks", clocks())
print("simt alone        ", run("simt", 0))
print("tc alone          ", run("tc", 0))
print("tc alone cosched  ", run("tc", HF_GEMM_COSCHEDULE))
print("serial            ", run("serial", 0))
print("simt,tc persistent", run("simt,tc", 0))
print("simt,tc cosched   ", run("simt,tc", HF_GEMM_COSCHEDULE))
print("tc,simt cosched   ", run("tc,simt", HF_GEMM_COSCHEDULE))
print("tc,simt persistent", run("tc,simt", 0))
print("simt,tc cosched-tc only", run("simt,tc", HF_GEMM_COSCHEDULE, simt_mode=0))
print("tmr simt,tc,tc3 plain  ", run("simt,tc,tc3", 0))
print("tmr simt,tc,tc3 cosched", run("simt,tc,tc3", HF_GEMM_COSCHEDULE))
print("clocks", clocks())
