mkdir -p gpurun_out
rm -f gpurun_out/e2e_ab.txt
for rep in 1 2; do for v in 0 1; do
HETFT_PREFETCH_DIRECT=$v timeout 600 python bench.py --no-cpu-baseline --detect-probes 10 --no-c3 > /tmp/b.json 2>/tmp/b.err
python -c "
import json; d=json.load(open('/tmp/b.json')); print('direct=$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['pcie_bound']['frac'],3), round(d['dmr']['e2e']['value'],1))" >> gpurun_out/e2e_ab.txt
done; done
cat gpurun_out/e2e_ab.txt
