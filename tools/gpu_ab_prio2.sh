mkdir -p gpurun_out
rm -f gpurun_out/ab_prio2.jsonl
for rep in 1 2; do
for strat in "--dmr"; do
for cfg in "0 1" "-1 1" "-1 2" "0 2"; do
set -- $cfg
HETFT_COMPUTE_PRIORITY=$1 timeout 300 python tools/lead_probe.py 60 --depth $2 $strat > /tmp/o.json 2>/tmp/o.err
echo "{\"prio\": $1, \"depth\": $2, \"r\": $(cat /tmp/o.json)}" >> gpurun_out/ab_prio2.jsonl
tail -2 /tmp/o.err
done
done
done
cat gpurun_out/ab_prio2.jsonl
