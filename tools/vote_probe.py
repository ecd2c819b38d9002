"""Why are diverse-replica votes slower than identical-replica votes at
>= 1 GiB (profiles/r01_vote_sweep_v2.json)?  Answer (later): they are not —
the sweep timed the votes while the default-stream torch ops generating the
diverse replicas were still running; with a device synchronise first both
kinds run at 1.08-1.14 of the HBM copy peak (profiles/r01_sweep_v4_*.json).  Times hf_vote K = 3 / 5 on
1 GiB replicas built several ways and prints their base addresses, so value
effects (which screen path runs) separate from placement effects."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels  # noqa: E402


def timed(fn, st, iters=5):
    with torch.cuda.stream(st):
        for _ in range(2):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(iters):
            fn()
        e1.record(st)
    st.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / iters


def main():
    nbytes = int(sys.argv[1]) << 20 if len(sys.argv) > 1 else 1 << 30
    n = nbytes // 4
    st = torch.cuda.Stream()
    ws = kernels.VoteWorkspace(0, stream=st)
    base = torch.rand(n, device="cuda") + 1
    for K in (3, 5):
        builds = {
            "identical_clone": lambda: [base] + [base.clone() for _ in range(K - 1)],
            "diverse_temporaries": lambda: [base] + [base * (1 + 1e-6 * torch.randn_like(base)) for _ in range(K - 1)],
            "diverse_then_clone": lambda: [base] + [(base * (1 + 1e-6 * torch.randn_like(base))).clone()
                                                    for _ in range(K - 1)],
            "identical_values_diverse_alloc": lambda: [base] + [(base * (1 + 0 * torch.randn_like(base)))
                                                                for _ in range(K - 1)],
        }
        for name, mk in builds.items():
            reps = mk()
            torch.cuda.synchronize()
            t = timed(lambda: kernels.vote_async(reps, ws, 1e-3, voted=None, stream=st), st)
            addrs = [r.data_ptr() for r in reps]
            print(json.dumps({"K": K, "build": name, "us": t * 1e6, "read_GBps": K * nbytes / t / 1e9,
                              "addr_mod_1GiB_MiB": [(a % (1 << 30)) >> 20 for a in addrs],
                              "addr_diff_MiB": [(a - addrs[0]) >> 20 for a in addrs]}), flush=True)
            del reps
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
