mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_gputests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/f_gputests.log
for t in memcheck racecheck synccheck initcheck; do
  echo "== $t" >> gpurun_out/f_sanitizer.txt
  timeout 600 compute-sanitizer --tool $t python tools/sanitize_target.py 2>&1 | grep -v "^=========     \|^=========$" | tail -6 >> gpurun_out/f_sanitizer.txt
done
cat gpurun_out/f_sanitizer.txt | grep -E "==|ERROR SUMMARY|target"
timeout 600 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/f_reference.json 2> gpurun_out/f_reference.err; echo ref rc=$?
python -c "
import json; d=json.load(open('gpurun_out/f_bench.json'))
print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['dmr']['value'], d['dmr']['e2e']['value'], d['clocks'], d['gpu_launches'])
r=json.load(open('gpurun_out/f_reference.json')); print(r['value'], r.get('cpu_baseline'))"
