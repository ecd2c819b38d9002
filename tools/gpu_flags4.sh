for o in 1 3; do
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xptxas -O$o -o /tmp/lab tools/simt_lab2.cu > /tmp/cc.log 2>&1 || cat /tmp/cc.log
echo "ptxas -O$o"; /tmp/lab 4096 q | cut -c1-140
done
