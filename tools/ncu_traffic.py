"""Per-kernel DRAM traffic from an `ncu --set full` capture (run here, on the
.ncu-rep brought back in gpurun_out/): dram__bytes_read.sum +
dram__bytes_write.sum per launch, averaged over the captured launches of each
kernel, plus duration, pipe utilisation and clock.  bench.py reads the
resulting JSON (profiles/) for the roofline's `traffic` field.

    python tools/ncu_traffic.py gpurun_out/prof_full.ncu-rep profiles/r01_ncu_traffic.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

FIELDS = {"dram__bytes_read.sum": "read", "dram__bytes_write.sum": "write",
          "gpu__time_duration.sum": "duration",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
          "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
          "sm__cycles_elapsed.avg.per_second": "sm_clock"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1, "%": 1, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}


def short(name: str) -> str:
    name = name.split("(")[0]
    return name.replace("void ", "").strip()


def main(rep: str, out: str):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    acc = defaultdict(lambda: defaultdict(list))
    for r in rows[2:]:
        k = short(r[hdr.index("Kernel Name")])
        for f, key in FIELDS.items():
            if f in hdr:
                i = hdr.index(f)
                try:
                    acc[k][key].append(float(r[i].replace(",", "")) * SCALE.get(units[i], 1))
                except ValueError:
                    pass
    res = {}
    for k, d in acc.items():
        m = {key: sum(v) / len(v) for key, v in d.items() if v}
        m["launches"] = max(len(v) for v in d.values())
        m["traffic_bytes"] = m.get("read", 0) + m.get("write", 0)
        res[k] = m
    doc = {"source": rep, "note": "per-launch means over the captured launches; ncu replays are cold-cache "
                                  "and serialised (--clock-control none)", "kernels": res}
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    for k, m in res.items():
        print(f"{k:40s} {m['duration'] * 1e6:9.1f} us  traffic {m['traffic_bytes'] / 1e6:8.1f} MB")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
