mkdir -p gpurun_out
timeout 300 python tools/e2e_probe.py --tmr --steps 40 --kineto gpurun_out/s2_e2e_trace.json > gpurun_out/s2_probe_e2e.log 2>&1; echo probe rc=$?
tail -1 gpurun_out/s2_probe_e2e.log | cut -c1-300
