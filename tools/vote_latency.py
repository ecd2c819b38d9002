"""Where does a small vote's time go?  Device time (CUDA events) of
hf_vote_async alone, + the 96-byte result read-back, and the backend's
vote_start/wait path, at 1/16/64 MiB, K = 2 and 3.  Tuning aid."""

import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels  # noqa: E402
from paper_1405_2912_b200.backend import CudaBackend  # noqa: E402
from paper_1405_2912_b200.devices import ValueType  # noqa: E402


def ev_time(fn, st, iters=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    for _ in range(iters):
        fn()
    e.record(st)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def main():
    be = CudaBackend()
    st = be.stream(0)
    for mib in (1, 16, 64):
        n = mib * (1 << 18)
        for K in (2, 3):
            reps = [torch.rand(n, device="cuda") + 1 for _ in range(K)]
            for r in reps[1:]:
                r.copy_(reps[0])
            slot = kernels._SliceSlot(0)
            with torch.cuda.stream(st):
                a = ev_time(lambda: kernels.vote_async(reps, slot.ws, [1e-3] * K, None, stream=st), st)
                b = ev_time(lambda: (kernels.vote_async(reps, slot.ws, [1e-3] * K, None, stream=st),
                                     kernels.copy(slot.host, slot.ws.result, stream=st)), st)
            bufs = [r.view(torch.uint8) for r in reps]
            ns = []
            walls = []
            for i in range(30):
                torch.cuda.synchronize()
                t0 = time.perf_counter_ns()
                h = be.vote_start(bufs, ValueType.FLOAT32, 4, [1e-3] * K)
                res, dn = h.wait()
                walls.append(time.perf_counter_ns() - t0)
                ns.append(dn)
            ns.sort()
            walls.sort()
            print(json.dumps({"mib": mib, "K": K, "vote_async_us": round(a, 2), "vote+d2h_us": round(b, 2),
                              "backend_event_us_med": ns[len(ns) // 2] / 1e3,
                              "backend_wall_us_med": walls[len(walls) // 2] / 1e3,
                              "gbps_kernel": round((K + 1) * n * 4 / (a * 1e3), 1)}), flush=True)


if __name__ == "__main__":
    main()
