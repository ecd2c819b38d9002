"""Run a script under torch.profiler (CPU + CUDA activities) and write a
gzipped chrome trace plus a per-kernel GPU-time summary.

  python tools/kineto_run.py OUT_PREFIX script.py [args...]
"""
import gzip
import json
import runpy
import shutil
import sys

from torch.profiler import ProfilerActivity, profile

out, script, *rest = sys.argv[1:]
sys.argv = [script, *rest]
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    try:
        runpy.run_path(script, run_name="__main__")
    except SystemExit:
        pass
prof.export_chrome_trace(out + ".json")
with open(out + ".json", "rb") as f, gzip.open(out + ".json.gz", "wb") as g:
    shutil.copyfileobj(f, g)
d = json.load(open(out + ".json"))
ev = [e for e in d["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
if ev:
    t0 = min(e["ts"] for e in ev)
    t1 = max(e["ts"] + e["dur"] for e in ev)
    busy = {}
    for e in ev:
        k = e["name"].split("(")[0][:60]
        busy[k] = busy.get(k, 0) + e["dur"]
    print(json.dumps({"span_ms": (t1 - t0) / 1e3, "kernels": {k: round(v / 1e3, 3) for k, v in
                                                               sorted(busy.items(), key=lambda x: -x[1])}}),
          file=sys.stderr)
