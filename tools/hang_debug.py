"""Debug aid for the deferred-path watchdog (tests/test_runtime_gpu.py
hang tests): logs every start/stop query of the watched slots."""
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_1405_2912_b200 as hf
from paper_1405_2912_b200 import executor as ex
import test_runtime_gpu as T
rt, task = T._hang_runtime([0])
T0 = time.perf_counter()
log = []
orig_q = rt.backend.query
def q(ev):
    r = orig_q(ev)
    log.append((round(time.perf_counter() - T0, 4), id(ev) % 10000, r))
    return r
rt.backend.query = q
orig_w = ex.Executor._watch_flight
def w(self, fl):
    for s, a in fl.round_results.items():
        t = a.outcome._timer
        print("slot", s, "deadline", a.prepared.deadline_ns, "start", id(getattr(t, "start_event", None)) % 10000,
              "stop", id(getattr(t, "stop_event", None)) % 10000, flush=True)
    r = orig_w(self, fl)
    print("watch ->", r, flush=True)
    return r
ex.Executor._watch_flight = w
n = 1 << 20
data = np.random.default_rng(2).uniform(1, 2, n).astype(np.float32)
inp = rt.register_data(data.tobytes(), n, hf.ValueType.FLOAT32, "r")
out = rt.register_data(bytes(4 * n), n, hf.ValueType.FLOAT32, "w")
torch.cuda.synchronize()
try:
    with rt.task_stream(depth=1) as ts:
        rep = ts.submit(task, {"input": inp, "output": out, "count": n}, hf.Strategy(hf.StrategyKind.HET_DMR))
    print("no raise", rep.votes, rep.fault_counts)
except Exception as e:
    print("raised", type(e).__name__, e)
print("t", time.perf_counter() - T0)
seen = {}
for t, e, r in log:
    if (e, r) not in seen:
        seen[(e, r)] = t
print(sorted(seen.items(), key=lambda x: x[1]))
