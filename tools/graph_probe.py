"""CUDA-graph capture of libhetft launches: time N captured 64 MiB K=2 votes
+ checkpoints replayed vs the same calls from a Python loop, and check the
last vote's result.  PDL on/off from HF_PDL."""
import json, os, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels

n = 16 << 20
st = torch.cuda.Stream()
a = torch.rand(n, device="cuda") + 1
b = a.clone()
b[12345] += 1.0
dst = torch.empty_like(a)
ws = kernels.VoteWorkspace(0, stream=st)
torch.cuda.synchronize()


def call():
    kernels.vote_async([a, b], ws, 1e-3, stream=st)


def loop_time(fn, iters):
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(iters):
            fn()
        e1.record(st)
    st.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


def graph_time(fn, iters):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(iters):
            fn()
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
    st.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


out = {"pdl": os.environ.get("HF_PDL", "1")}
for it in (10, 20):
    out[f"vote_loop_us_{it}"] = round(loop_time(call, it), 2)
    out[f"vote_graph_us_{it}"] = round(graph_time(call, it), 2)
r = ws.read()
out["result_ok"] = (r.verdict, r.first_div) == ("mismatch", 12345)
out["ckpt_loop_us"] = round(loop_time(lambda: kernels.checkpoint(dst, a, stream=st), 20), 2)
out["ckpt_graph_us"] = round(graph_time(lambda: kernels.checkpoint(dst, a, stream=st), 20), 2)
print(json.dumps(out))
