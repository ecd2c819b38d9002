mkdir -p gpurun_out
HF_LEAN_STREAMS=1 timeout 300 python tools/e2e_probe.py --device --steps 30 --depth 2 --kineto gpurun_out/s2_dmr_trace_lean.json > gpurun_out/s2_probe_dmr_lean.log 2>&1; echo probe rc=$?
tail -1 gpurun_out/s2_probe_dmr_lean.log
