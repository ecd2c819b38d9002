mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/y_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/y_gputests.log 2>&1; echo tests rc=$?
tail -1 gpurun_out/y_gputests.log
rm -f gpurun_out/y_sanitizer.txt
for t in memcheck racecheck synccheck initcheck; do
  echo "== $t" >> gpurun_out/y_sanitizer.txt
  timeout 600 compute-sanitizer --tool $t python tools/sanitize_target.py 2>&1 | grep -v "^=========     \|^=========$" | tail -4 >> gpurun_out/y_sanitizer.txt
done
grep -E "==|SUMMARY" gpurun_out/y_sanitizer.txt
timeout 600 python bench.py > gpurun_out/y_bench.json 2> gpurun_out/y_bench.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/y_bench.json'))
print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['rooflines']['hf_gemm_simt']['frac'], d['dmr']['value'], d['dmr']['e2e']['value'], d['clocks'])"
