"""Host-side cost of one C-ABI call (launch overhead, not GPU time): raw
ctypes calls into libhetft in a loop, microseconds per call, plus the torch
wrapper (kernels.*) cost for comparison."""
import json, sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import _lib, kernels

lib = _lib.load()
_lib.init()
n = 256
a = torch.rand(n, n, device="cuda") + 1
b = torch.rand(n, n, device="cuda") + 1
c = torch.empty(n, n, device="cuda")
st = torch.cuda.Stream()
sp = st.cuda_stream
CS = _lib.HF_GEMM_COSCHEDULE
buf = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
buf2 = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")


def t(name, fn, n_=100):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n_):
        fn()
    dt = (time.perf_counter() - t0) / n_ * 1e6
    torch.cuda.synchronize()
    return name, round(dt, 2)


import ctypes
reps = [torch.rand(1 << 18, device="cuda") for _ in range(3)]
ws = kernels.VoteWorkspace(0, stream=st)
res_host = torch.empty(ctypes.sizeof(_lib.HfVoteResult), dtype=torch.uint8).pin_memory()
rptr = (ctypes.c_void_p * 3)(*[r.data_ptr() for r in reps])
tol = (ctypes.c_double * 3)(1e-3, 1e-3, 1e-3)
rows = [
    t("hf_vote_async raw (K=3, 1 MiB)", lambda: lib.hf_vote_async(rptr, 3, 1 << 18, _lib.HF_F32, tol, None, None,
                                                                   res_host.data_ptr(), ws.ws.data_ptr(), 0, sp)),
    t("kernels.vote_async (K=3, 1 MiB)", lambda: kernels.vote_async(reps, ws, 1e-3, stream=st, result_into=res_host)),
    t("hf_gemm_tc raw (cosched)", lambda: lib.hf_gemm_tc(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, CS, 0, sp)),
    t("hf_gemm_tc raw (plain)", lambda: lib.hf_gemm_tc(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, 0, 0, sp)),
    t("hf_gemm_tc raw 3xtf32 cosched", lambda: lib.hf_gemm_tc(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, CS | 1, 0, sp)),
    t("hf_gemm_simt raw (cosched)", lambda: lib.hf_gemm_simt(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, CS, 0, sp)),
    t("hf_fill raw", lambda: lib.hf_fill(buf.data_ptr(), 0, 1 << 20, 0, sp)),
    t("hf_checkpoint raw", lambda: lib.hf_checkpoint(buf2.data_ptr(), buf.data_ptr(), 1 << 20, None, 0, sp)),
    t("kernels.gemm_tc (cosched)", lambda: kernels.gemm_tc(a, b, c, mode=CS, stream=st)),
    t("kernels.gemm_simt (cosched)", lambda: kernels.gemm_simt(a, b, c, mode=CS, stream=st)),
    t("kernels.fill", lambda: kernels.fill(buf, 0, stream=st)),
    t("kernels.checkpoint", lambda: kernels.checkpoint(buf2, buf, stream=st)),
    t("cudaLaunch via torch (buf.zero_)", lambda: buf.zero_()),
]
for r in rows:
    print(json.dumps({"call": r[0], "us": r[1]}))
