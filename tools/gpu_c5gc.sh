mkdir -p gpurun_out
for rep in 1 2; do for g in default freeze off; do for d in 1 2; do
timeout 300 python tools/stream_c5.py --tasks 6000 --gc $g --depth $d 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$g', 'depth', $d, round(d['value'],1), d['verify'][-20:])"
done; done; done
