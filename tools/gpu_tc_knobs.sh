mkdir -p gpurun_out
rm -f gpurun_out/tc_knobs.jsonl
for rep in 1 2; do
for knob in "X=0" "HF_TC_COSCHED_BN=128" "HF_TC_COSCHED_GRID=296" "HF_TC_COSCHED_GRID=148"; do
for strat in "" "--dmr"; do
env $knob timeout 300 python tools/lead_probe.py 60 $strat > /tmp/o.json 2>/tmp/o.err
echo "{\"knob\": \"$knob\", \"r\": $(cat /tmp/o.json)}" >> gpurun_out/tc_knobs.jsonl
tail -1 /tmp/o.err
done; done; done
cut -c1-150 gpurun_out/tc_knobs.jsonl
