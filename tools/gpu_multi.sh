mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --detect-probes 10 --c3-devices 0,0,0 --c4-devices 0,0,0 > gpurun_out/m_c3.json 2> gpurun_out/m_c3.err; echo c3 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/m_c3.json')); print(json.dumps(d.get('c3'))[:600]); print(json.dumps(d.get('c4_cross_gpu'))[:600])"
tail -3 gpurun_out/m_c3.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/m_2rank.json 2> gpurun_out/m_2rank.err; echo 2rank rc=$?
cut -c1-400 gpurun_out/m_2rank.json; tail -3 gpurun_out/m_2rank.err
