mkdir -p gpurun_out
timeout 300 python tools/e2e_probe.py --tmr --device --steps 30 --kineto gpurun_out/s2_tmr_trace_8x16.json > gpurun_out/s2_probe_8x16.log 2>&1; echo probe rc=$?
tail -2 gpurun_out/s2_probe_8x16.log
