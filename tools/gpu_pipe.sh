mkdir -p gpurun_out
timeout 300 python tools/pipeline_lab.py 60 > gpurun_out/pipeline_lab2.jsonl 2>&1; echo pipe rc=$?
cat gpurun_out/pipeline_lab2.jsonl
