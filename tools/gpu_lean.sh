mkdir -p gpurun_out
rm -f gpurun_out/lean_ab.jsonl
for rep in 1 2; do
for lean in 0 1; do
for cfg in "1 --dmr" "2 --dmr" "1 x" "2 x"; do
set -- $cfg
HF_LEAN_STREAMS=$lean timeout 300 python tools/lead_probe.py 60 --depth $1 $2 > /tmp/o.json 2>/tmp/o.err
echo "{\"lean\": $lean, \"depth\": $1, \"r\": $(cat /tmp/o.json)}" >> gpurun_out/lean_ab.jsonl
tail -2 /tmp/o.err
done
done
done
cut -c1-150 gpurun_out/lean_ab.jsonl
