mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/h_bench.json')); print(d['value'], d['e2e']['value'], d['e2e']['pcie_bound'], d['dmr']['value'], d['dmr']['e2e'])"
HETFT_VOTE_STREAM=0 timeout 900 python -m pytest tests -m gpu -x -q -k "runtime or commit or c3 or parity" > gpurun_out/h_tests_vs0.log 2>&1; echo tests_vs0 rc=$?; tail -1 gpurun_out/h_tests_vs0.log
