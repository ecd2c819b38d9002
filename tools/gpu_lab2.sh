mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/simt_lab2 tools/simt_lab2.cu
timeout 300 ./tools/simt_lab2 > gpurun_out/lab2d_simt.jsonl 2>&1; echo lab2 rc=$?
cat gpurun_out/lab2d_simt.jsonl
