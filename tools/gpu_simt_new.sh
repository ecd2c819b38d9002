mkdir -p gpurun_out
timeout 300 python tools/simt_ab.py 4096 > gpurun_out/simt_ab_8x16.jsonl 2>&1; echo ab rc=$?
cat gpurun_out/simt_ab_8x16.jsonl
timeout 900 python -m pytest tests -m gpu -x -q -k "simt or gemm or commit or smoke or parity" > gpurun_out/simt_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/simt_tests.log
timeout 600 python bench.py > gpurun_out/s2_bench_8x16.json 2> gpurun_out/s2_bench_8x16.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/s2_bench_8x16.json'))
print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['rooflines']['hf_gemm_simt'], d['dmr']['value'], d['dmr']['e2e']['value'], d['clocks'])"
