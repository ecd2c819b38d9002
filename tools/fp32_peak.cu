// FP32 SIMT peak probe: the denominator of the SIMT GEMM variant's roofline.
// Every thread runs 16 independent FMA chains (packed fma.rn.f32x2 -> SASS
// FFMA2, and scalar FFMA for comparison) for ITERS iterations; grid = 148 SMs
// x 4 CTAs x 256 threads.  Reports achieved TFLOP/s (2 flop per FMA) from CUDA
// events, best of 5, after warm-up.  Build: make -C tools fp32_peak
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 16
#define ITERS 4096

__global__ void __launch_bounds__(256) ffma2_loop(float* out, float a, float b) {
    unsigned long long acc[CHAINS / 2];
    float2 x = make_float2(a, b);
    unsigned long long av = *reinterpret_cast<unsigned long long*>(&x);
#pragma unroll
    for (int i = 0; i < CHAINS / 2; ++i) {
        float2 s = make_float2(threadIdx.x * 1e-7f + i, i * 1e-3f);
        acc[i] = *reinterpret_cast<unsigned long long*>(&s);
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS / 2; ++i)
            asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(acc[i]) : "l"(av));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < CHAINS / 2; ++i) {
        float2 v = *reinterpret_cast<float2*>(&acc[i]);
        s += v.x + v.y;
    }
    if (s == 12345.678f) out[threadIdx.x] = s;
}

// GEMM operand form: acc pair += broadcast scalar a x pair b (SASS FFMA2 R, Ra.F32, Rb.F32x2, Rc.F32x2),
// 16 accumulator pairs from 4 scalars x 4 pairs, like one k-step of the SIMT GEMM's outer product
__global__ void __launch_bounds__(256) ffma2_bcast_loop(float* out, float a, float b) {
    unsigned long long acc[4][4];
    float av[4];
    unsigned long long bv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        av[i] = a + i * 1e-3f + threadIdx.x * 1e-9f;
        float2 s = make_float2(b + i * 1e-7f + threadIdx.x * 1e-11f, b - i * 1e-7f);
        bv[i] = *reinterpret_cast<unsigned long long*>(&s);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float2 z = make_float2(threadIdx.x * 1e-7f + i, j * 1e-3f);
            acc[i][j] = *reinterpret_cast<unsigned long long*>(&z);
        }
    }
    for (int it = 0; it < ITERS / 2; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            unsigned long long ai;
            asm("mov.b64 %0, {%1, %1};" : "=l"(ai) : "f"(av[i]));
#pragma unroll
            for (int j = 0; j < 4; ++j) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i][j]) : "l"(ai), "l"(bv[j]));
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float2 v = *reinterpret_cast<float2*>(&acc[i][j]);
            s += v.x + v.y;
        }
    if (s == 12345.678f) out[threadIdx.x] = s;
}

// Diagonal pair form (no broadcast operand): acc{(2p,2q),(2p+1,2q+1)} += {a,a'} x {b,b'} and
// acc{(2p,2q+1),(2p+1,2q)} += {a,a'} x {b',b}; the swapped b pairs are rebuilt every step (MOVs)
// as a GEMM would after loading its fragments.  32 FFMA2 + 8 MOV per step, 32 accumulator pairs.
__global__ void __launch_bounds__(256, 2) ffma2_diag_loop(float* out, float a, float b) {
    unsigned long long d1[4][4], d2[4][4], A[4], Bp[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 x = make_float2(a + i * 1e-3f + threadIdx.x * 1e-9f, a - i * 1e-3f);
        float2 y = make_float2(b + i * 1e-7f + threadIdx.x * 1e-11f, b - i * 1e-7f);
        A[i] = *reinterpret_cast<unsigned long long*>(&x);
        Bp[i] = *reinterpret_cast<unsigned long long*>(&y);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float2 z = make_float2(threadIdx.x * 1e-7f + i, j * 1e-3f);
            d1[i][j] = d2[i][j] = *reinterpret_cast<unsigned long long*>(&z);
        }
    }
    for (int it = 0; it < ITERS / 4; ++it) {
        unsigned long long Bs[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float lo, hi;
            asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(Bp[q]));
            asm volatile("mov.b64 %0, {%1, %2};" : "=l"(Bs[q]) : "f"(hi), "f"(lo));
        }
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d1[p][q]) : "l"(A[p]), "l"(Bp[q]));
                asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d2[p][q]) : "l"(A[p]), "l"(Bs[q]));
            }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float2 v = *reinterpret_cast<float2*>(&d1[i][j]);
            float2 w = *reinterpret_cast<float2*>(&d2[i][j]);
            s += v.x + v.y + w.x + w.y;
        }
    if (s == 12345.678f) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) ffma_loop(float* out, float a, float b) {
    float acc[CHAINS];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-7f + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(acc[i]) : "f"(a), "f"(b));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += acc[i];
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
        double flops = 10.0 * blocks * 256.0 * CHAINS * ITERS * 2.0;
        double tf = flops / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
    }
    return best;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out;
    cudaMalloc(&out, 1024 * sizeof(float));
    int blocks = sms * 4;
    double t2 = run(ffma2_loop, out, blocks);
    double t1 = run(ffma_loop, out, blocks);
    double tb = run(ffma2_bcast_loop, out, blocks);
    double td = run(ffma2_diag_loop, out, blocks);
    double nominal = sms * 128.0 * 2.0 * (clk * 1e3) / 1e12;
    cudaError_t err = cudaGetLastError();
    printf("{\"ffma2_tflops\": %.3f, \"ffma_tflops\": %.3f, \"ffma2_bcast_tflops\": %.3f, \"ffma2_diag_tflops\": %.3f, \"nominal_tflops_at_max_clock\": %.3f, "
           "\"sms\": %d, \"max_clock_mhz\": %.0f, \"error\": \"%s\"}\n",
           t2, t1, tb, td, nominal, sms, clk / 1e3, cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
