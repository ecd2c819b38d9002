mkdir -p gpurun_out
timeout 300 python tools/e2e_probe.py --device --steps 30 --kineto gpurun_out/s2_dmr_trace.json > gpurun_out/s2_probe_dmr.log 2>&1; echo probe rc=$?
tail -1 gpurun_out/s2_probe_dmr.log
