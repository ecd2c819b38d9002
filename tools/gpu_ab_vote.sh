mkdir -p gpurun_out
rm -f gpurun_out/lead_probe.jsonl
for i in 1 2 3; do
for v in 0 1; do HETFT_VOTE_STREAM=$v timeout 300 python tools/lead_probe.py 60 >> gpurun_out/lead_probe.jsonl 2>gpurun_out/lead_probe.err; done
done
cat gpurun_out/lead_probe.jsonl; tail -3 gpurun_out/lead_probe.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2_gputests_vs.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/s2_gputests_vs.log
timeout 600 python bench.py > gpurun_out/s2_bench_vs.json 2> gpurun_out/s2_bench_vs.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/s2_bench_vs.json'))
print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['dmr']['value'], d['dmr']['e2e']['value'], d['clocks'])"
