mkdir -p gpurun_out
timeout 600 python tools/stream_c5.py --tasks 10000 --out gpurun_out/c5_10k_r2b.json > gpurun_out/c5.log 2>&1; echo c5 rc=$?
tail -2 gpurun_out/c5.log | cut -c1-300
timeout 600 python tools/host_profile.py --tasks 1500 > gpurun_out/host_profile_r2b.txt 2>&1; echo hp rc=$?
head -25 gpurun_out/host_profile_r2b.txt
