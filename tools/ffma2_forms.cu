// FFMA2 operand-order lab (not product code): the SIMT GEMM's per-k-step
// outer product on an 8 x 8 thread tile (8 broadcast a scalars x 4 b pairs =
// 32 FFMA2 into 32 accumulator pairs), issued a-outer (as sgemm_128x128 does)
// or b-outer, to see whether the order changes the sustained FFMA2 rate
// through operand reuse.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
//   -o tools/ffma2_forms tools/ffma2_forms.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 2048

template <bool A_OUTER>
__global__ void __launch_bounds__(256, 2) outer8x8(float* out, float a0, float b0) {
    unsigned long long acc[8][4];
    float a[8];
    unsigned long long b[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = a0 + i * 1e-3f + threadIdx.x * 1e-9f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float2 z = make_float2(threadIdx.x * 1e-7f + i, j * 1e-3f);
            acc[i][j] = *reinterpret_cast<unsigned long long*>(&z);
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float2 s = make_float2(b0 + j * 1e-7f, b0 - j * 1e-7f + threadIdx.x * 1e-11f);
        b[j] = *reinterpret_cast<unsigned long long*>(&s);
    }
    for (int it = 0; it < ITERS; ++it) {
        if (A_OUTER) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                unsigned long long ai;
                asm("mov.b64 %0, {%1, %1};" : "=l"(ai) : "f"(a[i]));
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i][j]) : "l"(ai), "l"(b[j]));
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    unsigned long long ai;
                    asm("mov.b64 %0, {%1, %1};" : "=l"(ai) : "f"(a[i]));
                    asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i][j]) : "l"(ai), "l"(b[j]));
                }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float2 v = *reinterpret_cast<float2*>(&acc[i][j]);
            s += v.x + v.y;
        }
    if (s == 12345.678f) out[threadIdx.x] = s;
}

template <typename K>
static double run(K kern, float* out, int blocks) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) kern<<<blocks, 256>>>(out, 0.999f, 1e-6f);
    double best = 0;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        for (int k = 0; k < 10; ++k) kern<<<blocks, 256>>>(out, 0.999f, 1e-6f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 10.0 * blocks * 256.0 * 64.0 * ITERS * 2.0;   // 32 FFMA2 = 64 FMA per step
        double tf = flops / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
    }
    return best;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 1024 * sizeof(float));
    const int blocks = sms * 2;
    double ao = run(outer8x8<true>, out, blocks);
    double bo = run(outer8x8<false>, out, blocks);
    printf("{\"a_outer_tflops\": %.3f, \"b_outer_tflops\": %.3f, \"error\": \"%s\"}\n", ao, bo,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
