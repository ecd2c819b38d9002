"""Why bench.py's K = 2 vote timing (24.6 us) differs from tools/vote_placement.py
(21.5 us) on the same 64 MiB replicas: vary one factor at a time."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1405_2912_b200 import kernels

st = torch.cuda.Stream()
ws = kernels.VoteWorkspace(0, stream=st)


def time_it(fn, iters):
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(iters):
            fn()
        e1.record(st)
    st.synchronize()
    return round(e0.elapsed_time(e1) * 1e3 / iters, 2)


m = 4096 * 4096
base = torch.rand(m, device="cuda") + 1
noisy = [base * (1 + 1e-6 * torch.randn(m, device="cuda")) for _ in range(2)]
exact = base.clone()
cases = {"both_noisy": noisy, "exact_vs_noisy": [exact, noisy[1]], "identical": [exact, base]}
for name, reps in cases.items():
    for iters in (10, 30):
        r = {}
        for key, out in (("verdict_only", None), ):
            r[key] = time_it(lambda: kernels.vote_async(reps, ws, 1e-3, voted=out, stream=st), iters)
        res = ws.read()
        print(json.dumps({"case": name, "iters": iters, "us": r, "verdict": res.verdict,
                          "unequal_frac": float((reps[0] != reps[1]).float().mean())}), flush=True)

# Placement: the same values in (a) two fresh 64 MiB segments, (b) one 128 MiB
# segment, (c) carved by the caching allocator from a freed 1.5 GiB segment.
src = [t.clone() for t in noisy]
del noisy, exact, base, cases, reps
torch.cuda.empty_cache()
a = [torch.empty(m, device="cuda") for _ in range(2)]
big = torch.empty(2 * m, device="cuda")
b = [big[:m], big[m:]]
for name, reps in (("two_segments", a), ("one_segment", b)):
    for r, s in zip(reps, src):
        r.copy_(s)
    print(json.dumps({"case": name, "us": time_it(lambda: kernels.vote_async(reps, ws, 1e-3, stream=st), 30),
                      "ptrs_mib": [round(r.data_ptr() / 2**20, 1) for r in reps]}), flush=True)
del a, big, b
torch.cuda.empty_cache()
pool = torch.empty(24 * m, device="cuda")
del pool
c = [torch.empty(m, device="cuda") for _ in range(2)]
for r, s in zip(c, src):
    r.copy_(s)
print(json.dumps({"case": "carved_from_freed_pool", "us": time_it(lambda: kernels.vote_async(c, ws, 1e-3, stream=st), 30),
                  "ptrs_mib": [round(r.data_ptr() / 2**20, 1) for r in c]}), flush=True)
