"""A/B the SIMT launch with and without the k-split tail wave
(HF_SIMT_NO_TAIL_SPLIT is read once per process: one subprocess each).

Historical: the k-split tail was measured slower and reverted (DESIGN.md §4,
"Tried and reverted"), so both arms now run the same kernel; kept as the
record of how that A/B was taken."""
import json
import os
import subprocess
import sys

CODE = r'''
import statistics, sys, torch
sys.path.insert(0, ".")
from paper_1405_2912_b200 import kernels
n = int(sys.argv[1])
a = torch.rand(n, n, device="cuda") + 1; b = torch.rand(n, n, device="cuda") + 1
c = torch.empty(n, n, device="cuda")
ts = []
for i in range(40):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); kernels.gemm_simt(a, b, c); e1.record(); torch.cuda.synchronize()
    if i >= 10: ts.append(e0.elapsed_time(e1))
ref = (a.double() @ b.double()).float()
err = ((c - ref).abs() / ref.abs()).max().item()
print(statistics.median(ts), min(ts), err)
'''

for n in [int(x) for x in sys.argv[1:]] or [4096, 2048]:
    for v in (1, 0, 1, 0):
        env = dict(os.environ)
        if v == 1:
            env["HF_SIMT_NO_TAIL_SPLIT"] = "1"
        out = subprocess.run([sys.executable, "-c", CODE, str(n)], env=env, capture_output=True, text=True)
        med, mn, err = out.stdout.split() if out.returncode == 0 else ("nan", "nan", out.stderr[-300:])
        print(json.dumps({"n": n, "variant": {0: "tail-split", 1: "no-split"}[v],
                          "ms_med": med, "ms_min": mn, "max_rel_err": err}), flush=True)
