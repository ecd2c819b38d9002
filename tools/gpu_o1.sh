mkdir -p gpurun_out
timeout 300 python tools/simt_ab.py 4096 2>&1 | tail -4
python tools/simt_fullwave.py
timeout 900 python -m pytest tests -m gpu -x -q -k "simt or gemm or commit or parity or smoke" > gpurun_out/o1_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/o1_tests.log
timeout 600 python bench.py > gpurun_out/o1_bench.json 2> gpurun_out/o1_bench.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/o1_bench.json'))
print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['rooflines']['hf_gemm_simt']['frac'], d['dmr']['value'], d['dmr']['e2e']['value'])"
