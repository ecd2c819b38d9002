nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xptxas -O1 -o /tmp/lab tools/simt_lab2.cu > /tmp/cc.log 2>&1 || cat /tmp/cc.log
/tmp/lab 4096 q
