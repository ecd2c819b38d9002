set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2_gputests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/s2_gputests.log
timeout 600 python bench.py > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err; echo bench rc=$?
timeout 300 python tools/e2e_probe.py --tmr --device --steps 30 --kineto gpurun_out/s2_tmr_trace.json > gpurun_out/s2_probe.log 2>&1; echo probe rc=$?
