"""Back-to-back hf_vote_async device time (CUDA events), f32, several sizes
and K: the launch configuration under test comes from the environment
(HF_PDL).  Prints one JSON line per case."""
import json, os, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels

st = torch.cuda.Stream()
for mib, K in ((16, 2), (64, 2), (64, 3), (256, 3), (1024, 3), (1024, 5)):
    n = mib * (1 << 18)
    base = torch.rand(n, device="cuda") + 1
    reps = [base.clone() for _ in range(K)]
    ws = kernels.VoteWorkspace(0, stream=st)
    iters = 20
    with torch.cuda.stream(st):
        for _ in range(3):
            kernels.vote_async(reps, ws, 1e-3, stream=st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(iters):
            kernels.vote_async(reps, ws, 1e-3, stream=st)
        e1.record(st)
    st.synchronize()
    t = e0.elapsed_time(e1) / iters * 1e-3
    assert ws.read().verdict == "match"
    print(json.dumps({"pdl": os.environ.get("HF_PDL", "1"),
                      "mib": mib, "K": K, "us": round(t * 1e6, 2), "read_GBps": round(K * n * 4 / t / 1e9, 1)}))
    del reps, base
