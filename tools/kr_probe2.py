import json, sys
sys.path.insert(0, ".")
import subprocess
import time
import torch
from paper_1405_2912_b200 import kernels
st = torch.cuda.Stream(); ws = kernels.VoteWorkspace(0, stream=st)
def time_it(reps, iters=30):
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        for _ in range(3): kernels.vote_async(reps, ws, 1e-3, stream=st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        h0 = time.perf_counter()
        for _ in range(iters): kernels.vote_async(reps, ws, 1e-3, stream=st)
        h1 = time.perf_counter()
        e1.record(st)
    st.synchronize()
    # device us per vote, host enqueue us per vote: device >= host means the GPU waited on the host
    return round(e0.elapsed_time(e1) * 1e3 / iters, 2), round((h1 - h0) * 1e6 / iters, 2)
def clocks():
    q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active",
                        "--format=csv,noheader,nounits", "-i", "0"], capture_output=True, text=True).stdout.strip()
    return q


def seg(t):
    p = t.data_ptr()
    for s in torch.cuda.memory_snapshot():
        if s["address"] <= p < s["address"] + s["total_size"]:
            return {"seg_mib": s["total_size"] >> 20, "off_mib": (p - s["address"]) >> 20}
m = 4096 * 4096
base = torch.rand(m, device="cuda") + 1
noisy = [base * (1 + 1e-6 * torch.randn(m, device="cuda")) for _ in range(2)]
print("clocks_start", clocks(), flush=True)
print("noisy", time_it(noisy), [seg(t) for t in noisy], flush=True)
fresh = [torch.empty(m, device="cuda") for _ in range(2)]
for f, x in zip(fresh, noisy): f.copy_(x)
print("fresh_copies", time_it(fresh), [seg(t) for t in fresh], flush=True)
print("clocks_mid", clocks(), flush=True)
print("noisy_again", time_it(noisy), flush=True)
print("clocks_after", clocks(), flush=True)
# keep the GPU busy while timing: a long back-to-back run, clocks sampled inside it
with torch.cuda.stream(st):
    for _ in range(4000): kernels.vote_async(noisy, ws, 1e-3, stream=st)
print("clocks_busy", clocks(), flush=True)
st.synchronize()
print("noisy_after_busy", time_it(noisy, 300), clocks(), flush=True)
print("mixed", time_it([noisy[0], fresh[1]]), time_it([fresh[0], noisy[1]]), flush=True)
print("base_pair", time_it([base, fresh[0]]), seg(base), flush=True)
for s in torch.cuda.memory_snapshot():
    print("segment", s["total_size"] >> 20, [(b["size"] >> 20, b["state"]) for b in s["blocks"]])
