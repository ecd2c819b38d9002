mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/z_gputests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/z_gputests.log
