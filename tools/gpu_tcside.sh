mkdir -p gpurun_out
rm -f gpurun_out/tcside.jsonl
for rep in 1 2; do
for knob in "HF_TC_SIDE=1" "HF_TC_SIDE=0"; do
for strat in "" "--dmr"; do
env $knob timeout 300 python tools/lead_probe.py 60 $strat > /tmp/o.json 2>/tmp/o.err
echo "{\"knob\": \"$knob\", \"r\": $(cat /tmp/o.json)}" >> gpurun_out/tcside.jsonl
tail -1 /tmp/o.err
done; done; done
cut -c1-140 gpurun_out/tcside.jsonl
