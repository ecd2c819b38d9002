"""A/B of the SIMT GEMM's accumulation: blocked (default, fp32 chains of
SGEMM_CH k-tiles summed into an smem running total) vs one chain over all
of K (HF_SGEMM_CHAIN=1, read once per process: one subprocess per arm).
Reports the CUDA-event time (median/min of 30 after 10 warm-up calls) and
the max relative error against the binary64 product, with numpy's fp32
matmul error on the same operands for comparison."""
import json
import os
import subprocess
import sys

CODE = r'''
import os, statistics, sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_1405_2912_b200 import kernels
n = int(sys.argv[1])
g = np.random.default_rng(5)
a = g.uniform(1, 2, (n, n)).astype(np.float32); b = g.uniform(1, 2, (n, n)).astype(np.float32)
ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
c = torch.empty(n, n, device="cuda")
ts = []
for i in range(40):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); kernels.gemm_simt(ta, tb, c, mode=int(os.environ.get('AB_MODE', '0'))); e1.record(); torch.cuda.synchronize()
    if i >= 10: ts.append(e0.elapsed_time(e1))
ex = (torch.from_numpy(a).double().cuda() @ torch.from_numpy(b).double().cuda())
err = ((c.double() - ex).abs() / ex.abs()).max().item()
print(statistics.median(ts), min(ts), err)
'''

for n in [int(x) for x in sys.argv[1:]] or [4096, 2048]:
    for v in ("chain", "blocked", "chain", "blocked"):
        env = dict(os.environ)
        if v.startswith("chain"):
            env["HF_SGEMM_CHAIN"] = "1"
            if v == "chain-smem112":      # chain kernel with the blocked kernel's smem footprint
                env["HF_SGEMM_COSCHED_SMEM"] = "114688"
                env["AB_MODE"] = str(0x100)
        out = subprocess.run([sys.executable, "-c", CODE, str(n)], env=env, capture_output=True, text=True)
        med, mn, err = out.stdout.split() if out.returncode == 0 else ("nan", "nan", out.stderr[-300:])
        print(json.dumps({"n": n, "variant": v,
                          "ms_med": med, "ms_min": mn, "max_rel_err": err}), flush=True)
