"""Back-to-back hf_vote_async device time (CUDA events over 20 launches) and
the kernel's own time (hf_vote_result.kernel_ns of the last launch), f32,
diverse replicas (1e-6 relative noise), several sizes and K, with and
without in-place voting.  HETFT_LIB selects the library (A/B against an
older build); HF_PDL=0 disables programmatic dependent launch.  One JSON
line per case."""
import json, os, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels

st = torch.cuda.Stream()
cases = [(16, 2), (64, 2), (64, 3), (256, 3)] if os.environ.get("VOTE_AB_SHORT") else [(1, 2), (4, 3), (16, 2), (16, 3), (64, 2), (64, 3), (256, 3), (1024, 3)]
for mib, K in cases:
    for in_place in ((False, True) if K >= 3 else (False,)):
        n = mib * (1 << 18)
        base = torch.rand(n, device="cuda") + 1
        reps = [base * (1 + 1e-6 * torch.randn(n, device="cuda")) for _ in range(K)]
        ws = kernels.VoteWorkspace(0, stream=st)
        iters = 20
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            for _ in range(3):
                kernels.vote_async(reps, ws, 1e-3, voted=reps[0] if in_place else None, stream=st)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(iters):
                kernels.vote_async(reps, ws, 1e-3, voted=reps[0] if in_place else None, stream=st)
            e1.record(st)
        st.synchronize()
        t = e0.elapsed_time(e1) / iters * 1e-3
        r = ws.read()
        assert r.verdict == "match"
        kns = getattr(r, "kernel_ns", 0)
        print(json.dumps({"lib": os.path.basename(os.environ.get("HETFT_LIB", "current")), "mib": mib, "K": K,
                          "in_place": in_place, "us": round(t * 1e6, 2), "kernel_us": round(kns / 1e3, 2),
                          "read_GBps": round(K * n * 4 / t / 1e9, 1)}), flush=True)
        del reps, base
