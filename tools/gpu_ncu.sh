mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r02c_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --detect-probes 10 --e2e-steps 4 > gpurun_out/r02c_ncu_bench.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sgemm_128|vote_kernel|gemm_tf32|stream_kernel|transpose|round_a|split3" -c 20 -o gpurun_out/r02c_full python tools/ncu_target.py 4096 1 > gpurun_out/r02c_ncu_full.log 2>&1; echo full rc=$?
ls -la gpurun_out/r02c_full.ncu-rep
