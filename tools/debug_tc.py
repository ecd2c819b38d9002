"""Structured probes for the tcgen05 GEMM layout (dumps to gpurun_out/)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels  # noqa: E402

out = {}


def run(a, b):
    ta = torch.from_numpy(a).cuda()
    tb = torch.from_numpy(b).cuda()
    c = torch.full((a.shape[0], b.shape[1]), -7.0, device="cuda")
    kernels.gemm_tc(ta, tb, c)
    torch.cuda.synchronize()
    return c.cpu().numpy()


for K in (32, 64):
    M, N = 128, 256
    # probe A: A[i,k] = (k == i % K), B[k,n] = k  -> expect C[i,n] = i % K
    A = np.zeros((M, K), np.float32)
    A[np.arange(M), np.arange(M) % K] = 1
    B = np.repeat(np.arange(K, dtype=np.float32)[:, None], N, axis=1)
    out[f"pA_K{K}"] = run(A, B)
    # probe B: same A, B[k,n] = n -> expect C[i,n] = n
    B2 = np.repeat(np.arange(N, dtype=np.float32)[None, :], K, axis=0)
    out[f"pB_K{K}"] = run(A, B2)
    # probe C: A[i,k] = i (all k), B[k,n] = (k == 0) -> expect C[i,n] = i
    A3 = np.repeat(np.arange(M, dtype=np.float32)[:, None], K, axis=1)
    B3 = np.zeros((K, N), np.float32)
    B3[0] = 1
    out[f"pC_K{K}"] = run(A3, B3)
    # probe D: A[i,k] = (k == 0), B[k,n] = k*256+n... use B[k,n]=n for k==0 else 1000
    A4 = np.zeros((M, K), np.float32)
    A4[:, 0] = 1
    B4 = np.full((K, N), 1000.0, np.float32)
    B4[0] = np.arange(N)
    out[f"pD_K{K}"] = run(A4, B4)
Path("gpurun_out").mkdir(exist_ok=True)
np.savez("gpurun_out/debug_tc.npz", **out)
for k, v in out.items():
    print(k, v[:4, :8].tolist(), v[32:34, :4].tolist())
