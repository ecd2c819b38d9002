"""Per-kernel summary of an `ncu --set full` capture (run here on the
.ncu-rep brought back from gpurun): duration, clock, DRAM bytes and %,
pipe utilisation, occupancy, registers, grid, top warp-stall reasons.

    python tools/ncu_full_summary.py [--all] gpurun_out/r02_full.ncu-rep "header line" ... > profiles/r02_ncu_full_summary.txt
(--all: every captured launch, not the first of each kernel name)
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("duration", "gpu__time_duration.sum"),
    ("SM clock", "sm__cycles_elapsed.avg.per_second"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM % of peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor pipe % (avg SM)", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    ("tensor pipe % (max SM)", "sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_active"),
    ("FMA pipe %", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("issue slots busy %", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("L2 hit rate %", "lts__t_sector_hit_rate.pct"),
    ("registers/thread", "launch__registers_per_thread"),
    ("smem/block (dyn)", "launch__shared_mem_per_block_dynamic"),
    ("grid", "launch__grid_size"),
    ("cluster x", "launch__cluster_dim_x"),
]
STALL_PREFIX = "smsp__average_warp_latency_issue_stalled_"

args = sys.argv[1:]
every = "--all" in args
args = [a for a in args if a != "--all"]
rep, *header = args
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
for h in header:
    print(f"# {h}")
seen = set()
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").strip()
    if name in seen and not every:
        continue
    seen.add(name)
    print(f"\n== {name}" + (f"  (launch {r[hdr.index('ID')]})" if every and "ID" in hdr else ""))
    for label, m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            print(f"  {label:28s} {r[i]} {units[i]}")
    stalls = []
    for i, m in enumerate(hdr):
        if m.startswith(STALL_PREFIX) and m.endswith(".ratio") and "not_issued" not in m:
            try:
                stalls.append((float(r[i].replace(",", "")), m[len(STALL_PREFIX):-len(".ratio")]))
            except ValueError:
                pass
    if stalls:
        top = ", ".join(f"{k} {v:.2f}" for v, k in sorted(stalls, reverse=True)[:4])
        print(f"  {'top stalls (cycles/instr)':28s} {top}")
