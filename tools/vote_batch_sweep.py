"""Small votes, one launch each vs hf_vote_batch (BASELINE configs[3]'s lower
half, 1-16 MiB; configs[0]'s 4 MiB TMR shape): B independent votes of S MiB
with K diverse replicas each (distinct buffers, 1e-6 relative noise), voted
back to back with one hf_vote_async per vote or with one hf_vote_batch per 32
votes (kernels.VoteBatch: descriptors built once, one C call per launch).  CUDA events on the stream over the whole set after warm-up; reports
per-vote device time, replica bytes read per second and the fraction of the
HBM copy peak (MEASURED_PEAKS.json).  One JSON line per case.

    python tools/vote_batch_sweep.py [--votes 64]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1405_2912_b200 import kernels  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--votes", type=int, default=64)
args = ap.parse_args()
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() \
    else 6553.9
st = torch.cuda.Stream()
for mib in (1, 4, 16):
    for Kr in (2, 3, 4, 5):
        n = mib * (1 << 18)
        B = args.votes
        sets = []
        for _ in range(B):
            base = torch.rand(n, device="cuda") + 1
            sets.append([base * (1 + 1e-6 * torch.randn(n, device="cuda")) for _ in range(Kr)])
        wss = [kernels.VoteWorkspace(0, stream=st) for _ in range(B)]
        torch.cuda.synchronize()

        def single():
            for reps, ws in zip(sets, wss):
                kernels.vote_async(reps, ws, 1e-3, stream=st)

        batch = kernels.VoteBatch([(reps, None, ws, None) for reps, ws in zip(sets, wss)], 1e-3)

        def batched():
            batch.launch(st)

        out = {"mib": mib, "K": Kr, "votes": B}
        for name, fn in (("single", single), ("batch", batched)):
            with torch.cuda.stream(st):
                fn()
                fn()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(3):
                    fn()
                e1.record(st)
            st.synchronize()
            t = e0.elapsed_time(e1) * 1e-3 / (3 * B)
            assert all(ws.read().verdict == "match" for ws in wss[:4])
            assert all(ws.read().kernel_ns > 0 for ws in wss[:4])
            gbs = Kr * n * 4 / t / 1e9
            out[name] = {"us_per_vote": round(t * 1e6, 3), "read_GBps": round(gbs, 1), "frac_hbm": round(gbs / peak, 3)}
        print(json.dumps(out), flush=True)
        del sets, wss, batch
