"""BASELINE config C4: voter / checkpoint bandwidth sweep on one B200.

K = 2..5 fp32 replicas of 1 MB .. 4 GB each (bit-identical replicas with a
few injected bit flips, so the common path runs), hf_vote with the voted
output in place over replica 0, and hf_checkpoint of one buffer.  CUDA-event
timing on the launching stream, 3 warm-up + N timed launches; replicas
>= 64 MB exceed half the L2, smaller ones are partly L2-resident (reported
as measured).  Writes one JSON document (default gpurun_out/sweep.json)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels  # noqa: E402


def timed(fn, st, iters):
    """Device time per call over a Python launch loop.  Below ~16 MiB per
    replica a vote_async call (~15 us of host time) outlasts the kernel, so
    those rows are launch-bound, not kernel-bound."""
    torch.cuda.synchronize()     # replicas were generated on the default stream
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(iters):
            fn()
        e1.record(st)
    st.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / iters


def main(out=Path("gpurun_out/sweep.json"), sizes=None, diverse=False):
    peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()) \
        if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else {"hbm_gbs": 6650.0}
    hbm = peaks["hbm_gbs"]
    st = torch.cuda.Stream()
    rows = []
    sizes = sizes or [1 << 20, 16 << 20, 64 << 20, 256 << 20, 1 << 30, 4 << 30]
    for nbytes in sizes:
        n = nbytes // 4
        base = torch.rand(n, device="cuda") + 1
        iters = 20 if nbytes <= (256 << 20) else 5
        for K in (2, 3, 4, 5):
            # identical replicas (exact-equality path) or diverse ones (values
            # 1e-6 apart, like TC vs SIMT outputs: the fp32 screen decides)
            reps = [base] + [base * (1 + 1e-6 * torch.randn_like(base)) if diverse else base.clone()
                             for _ in range(K - 1)]
            for r in range(K):
                kernels.inject_bitflip(reps[r], (r * 7919) % n, 27)
            ws = kernels.VoteWorkspace(0, stream=st)
            voted = reps[0] if K >= 3 else None
            t = timed(lambda: kernels.vote_async(reps, ws, 1e-3, voted=voted, stream=st), st, iters)
            tk = ws.read().kernel_ns * 1e-9          # the last launch's own clock (r2)
            rd = K * nbytes
            rows.append({"kernel": "hf_vote", "K": K, "diverse": diverse, "bytes_per_replica": nbytes, "us": t * 1e6,
                         "read_GBps": rd / t / 1e9, "frac_of_hbm": rd / t / 1e9 / hbm,
                         "kernel_us": tk * 1e6, "frac_of_hbm_kernel_clock": rd / tk / 1e9 / hbm if tk else None,
                         "survey_GBps_(K+1)n": (K + 1) * nbytes / t / 1e9})
            # batched small votes: tools/vote_batch_sweep.py (distinct replica
            # sets per vote; reusing these replicas 32 times would read them
            # from the L2 and overstate the rate)
            print(json.dumps(rows[-1]), flush=True)
            del reps
        dst = torch.empty_like(base)
        t = timed(lambda: kernels.checkpoint(dst, base, stream=st), st, iters)
        rows.append({"kernel": "hf_checkpoint", "bytes": nbytes, "us": t * 1e6, "GBps": 2 * nbytes / t / 1e9,
                     "frac_of_hbm": 2 * nbytes / t / 1e9 / hbm})
        print(json.dumps(rows[-1]), flush=True)
        del base, dst
        torch.cuda.empty_cache()
    out.parent.mkdir(exist_ok=True)
    out.write_text(json.dumps({"peak_hbm_gbs": hbm, "rows": rows}, indent=1))


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("out", nargs="?", default="gpurun_out/sweep.json")
    ap.add_argument("--mib", type=int, nargs="*", help="replica sizes in MiB (default 1 MiB .. 4 GiB)")
    ap.add_argument("--diverse", action="store_true")
    a = ap.parse_args()
    main(Path(a.out), [m << 20 for m in a.mib] if a.mib else None, a.diverse)
