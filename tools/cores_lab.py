"""Lab (not product code): can the tensor-core replicas run *beside* the SIMT
replica for its whole duration instead of in its last wave?  The SIMT GEMM's
co-scheduling reservation decides how many SIMT CTAs share an SM
(HF_SGEMM_COSCHED_SMEM, read once per process, so one subprocess per
setting).  For each setting: the three 4096^2 replicas of a HetTMR round
alone and launched together (SIMT on a high-priority stream first, then
TF32 and 3xBF16 co-scheduled on normal-priority streams), CUDA-event medians
over 15 iterations with an L2 flush between them.

    python tools/cores_lab.py [n]
"""
import json
import os
import subprocess
import sys

CODE = r'''
import json, statistics, sys, torch
sys.path.insert(0, ".")
from paper_1405_2912_b200 import kernels
from paper_1405_2912_b200._lib import HF_GEMM_COSCHEDULE as CO, HF_GEMM_TF32, HF_GEMM_3XBF16
n = int(sys.argv[1]); d = "cuda:0"
a = torch.rand(n, n, device=d) + 1; b = torch.rand(n, n, device=d) + 1
cs = [torch.empty(n, n, device=d) for _ in range(3)]
hi = torch.cuda.Stream(priority=-1); s2 = torch.cuda.Stream(); s3 = torch.cuda.Stream()
main = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=d)
def ev(): return torch.cuda.Event(enable_timing=True)
def launch(w, st):
    if w == "simt": kernels.gemm_simt(a, b, cs[0], mode=CO, stream=st)
    elif w == "tf32": kernels.gemm_tc(a, b, cs[1], mode=HF_GEMM_TF32 | CO, stream=st)
    elif w == "tc3": kernels.gemm_tc(a, b, cs[2], mode=HF_GEMM_3XBF16 | CO, stream=st)
def run(ws, iters=15):
    out = []
    for it in range(iters + 3):
        flush.fill_(it & 0xFF)
        t0 = ev(); t0.record(main)
        ends = {}
        for w in ws:
            st = {"simt": hi, "tf32": s2, "tc3": s3}[w]
            st.wait_stream(main)
            launch(w, st)
            e = ev(); e.record(st); ends[w] = e
        for st in (hi, s2, s3): main.wait_stream(st)
        t1 = ev(); t1.record(main); torch.cuda.synchronize()
        if it >= 3:
            r = {"total": t0.elapsed_time(t1)}
            r.update({w + "_end": t0.elapsed_time(e) for w, e in ends.items()})
            out.append(r)
    return {k: round(statistics.median(x[k] for x in out), 4) for k in out[0]}
res = {}
import os
orders = [x.split(",") for x in os.environ.get("LAB_ORDERS", "simt;tf32;tc3;simt,tf32,tc3;simt,tc3,tf32").split(";")]
for ws in orders:
    res["+".join(ws)] = run(ws)
print(json.dumps(res))
'''

n = sys.argv[1] if len(sys.argv) > 1 else "4096"
TC_FIRST = "simt;tf32;tc3;tf32,tc3,simt;tc3,tf32,simt;simt,tf32,tc3"
settings = [
    ("default (2 SIMT CTAs/SM, 112 KB each)", {}),
    ("1 SIMT CTA/SM (120 KB reservation)", {"HF_SGEMM_COSCHED_SMEM": "120000"}),
    ("TC persistent 74 + 74 CTAs launched first", {"HF_TC_COSCHED_GRID": "74", "LAB_ORDERS": TC_FIRST}),
    ("TC persistent 148 + 148 launched first", {"HF_TC_COSCHED_GRID": "148", "LAB_ORDERS": TC_FIRST}),
    ("TC persistent 37 + 37 launched first", {"HF_TC_COSCHED_GRID": "37", "LAB_ORDERS": TC_FIRST}),
    ("TC 74 + 74 first, 1 SIMT CTA/SM", {"HF_TC_COSCHED_GRID": "74", "HF_SGEMM_COSCHED_SMEM": "120000",
                                         "LAB_ORDERS": TC_FIRST}),
]
for name, extra in settings:
    env = dict(os.environ, **extra)
    out = subprocess.run([sys.executable, "-c", CODE, n], env=env, capture_output=True, text=True)
    body = json.loads(out.stdout) if out.returncode == 0 else {"error": out.stderr[-400:]}
    print(json.dumps({"setting": name, "env": extra, **body}), flush=True)
