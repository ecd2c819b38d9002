// hf_gemm_simt: register-tiled FP32 FFMA matmul, C = A·B, row-major (sm_100a).
//
// The SIMT half of the diverse kernel pair that stands in for the paper's
// OpenMP/CUDA variants (§IV-D; attached through the kernel-variant
// slot of /root/reference/pkg/src/hetrt/api.py:131-138).  It never touches the
// tensor cores, accumulates every output in fp32 in ascending k order with
// fused multiply-add, and so fails independently of the tcgen05 variant.
//
// Fast path (M%128 == N%128 == 0, K%8 == 0, 16B-aligned): 128x128x8 CTA
// tile, 256 threads, 8x8 outputs per thread as 2x2 blocks of 4x4, A staged
// transposed in shared memory, two smem stages with a register prefetch of the
// next k-tile, one barrier per k-tile, register double-buffered fragments.  Warps are laid out 4x2 over the
// 16x16 thread grid so each LDS.128 of A and of B is one wavefront.
// Generic path: 16x16 bounds-checked tiles for ragged shapes.
#include "common.cuh"

namespace hf {

constexpr int SB_M = 128, SB_N = 128, SB_K = 8, S_PAD = 4;

// 128x128x8 CTA tile, 256 threads, 8x8 per thread; fragments for k+1 are
// loaded from shared memory while k is multiplied (register double buffer),
// the next k-tile is prefetched from global into registers; <= 128 registers
// so two CTAs (16 warps) share an SM.
__global__ void __launch_bounds__(256, 2)
sgemm_128x128(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C,
              int M, int N, int K) {
    __shared__ __align__(16) float As[2][SB_K][SB_M + S_PAD];
    __shared__ __align__(16) float Bs[2][SB_K][SB_N];

    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int ty = (warp >> 1) * 4 + (lane >> 3);  // 0..15
    const int tx = (warp & 1) * 8 + (lane & 7);    // 0..15

    // grouped tile order: consecutive CTAs share B column panels in L2
    const int tiles_n = N / SB_N;
    const int tiles_m = M / SB_M;
    const int group = 8;
    const int bid = blockIdx.x;
    const int per_group = group * tiles_n;
    const int g = bid / per_group;
    const int first_m = g * group;
    const int gm = min(tiles_m - first_m, group);
    const int tm = first_m + (bid % per_group) % gm;
    const int tn = (bid % per_group) / gm;
    const int m0 = tm * SB_M, n0 = tn * SB_N;

    // global->smem mapping: A 128x8 (one float4 per thread), B 8x128 (one float4)
    const int a_row = t >> 1, a_k = (t & 1) * 4;
    const int b_k = t >> 5, b_n = (t & 31) * 4;
    const float* Ag = A + static_cast<long long>(m0 + a_row) * K + a_k;
    const float* Bg = B + static_cast<long long>(b_k) * N + n0 + b_n;

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    float4 ra = __ldg(reinterpret_cast<const float4*>(Ag));
    float4 rb = __ldg(reinterpret_cast<const float4*>(Bg));
    As[0][a_k + 0][a_row] = ra.x;
    As[0][a_k + 1][a_row] = ra.y;
    As[0][a_k + 2][a_row] = ra.z;
    As[0][a_k + 3][a_row] = ra.w;
    *reinterpret_cast<float4*>(&Bs[0][b_k][b_n]) = rb;
    __syncthreads();

    float4 fa[2][2], fb[2][2];
    fa[0][0] = *reinterpret_cast<const float4*>(&As[0][0][ty * 4]);
    fa[0][1] = *reinterpret_cast<const float4*>(&As[0][0][64 + ty * 4]);
    fb[0][0] = *reinterpret_cast<const float4*>(&Bs[0][0][tx * 4]);
    fb[0][1] = *reinterpret_cast<const float4*>(&Bs[0][0][64 + tx * 4]);

    const int nk = K / SB_K;
    for (int kt = 0; kt < nk; ++kt) {
        const int s = kt & 1;
        const bool more = kt + 1 < nk;
        if (more) {
            ra = __ldg(reinterpret_cast<const float4*>(Ag + (kt + 1) * SB_K));
            rb = __ldg(reinterpret_cast<const float4*>(Bg + static_cast<long long>((kt + 1) * SB_K) * N));
        }
#pragma unroll
        for (int k = 0; k < SB_K; ++k) {
            const int cur = k & 1, nxt = cur ^ 1;
            if (k + 1 < SB_K) {
                fa[nxt][0] = *reinterpret_cast<const float4*>(&As[s][k + 1][ty * 4]);
                fa[nxt][1] = *reinterpret_cast<const float4*>(&As[s][k + 1][64 + ty * 4]);
                fb[nxt][0] = *reinterpret_cast<const float4*>(&Bs[s][k + 1][tx * 4]);
                fb[nxt][1] = *reinterpret_cast<const float4*>(&Bs[s][k + 1][64 + tx * 4]);
            } else if (more) {
                // stage the prefetched tile, then start the next tile's fragments
                As[s ^ 1][a_k + 0][a_row] = ra.x;
                As[s ^ 1][a_k + 1][a_row] = ra.y;
                As[s ^ 1][a_k + 2][a_row] = ra.z;
                As[s ^ 1][a_k + 3][a_row] = ra.w;
                *reinterpret_cast<float4*>(&Bs[s ^ 1][b_k][b_n]) = rb;
                __syncthreads();
                fa[nxt][0] = *reinterpret_cast<const float4*>(&As[s ^ 1][0][ty * 4]);
                fa[nxt][1] = *reinterpret_cast<const float4*>(&As[s ^ 1][0][64 + ty * 4]);
                fb[nxt][0] = *reinterpret_cast<const float4*>(&Bs[s ^ 1][0][tx * 4]);
                fb[nxt][1] = *reinterpret_cast<const float4*>(&Bs[s ^ 1][0][64 + tx * 4]);
            }
            const float a[8] = {fa[cur][0].x, fa[cur][0].y, fa[cur][0].z, fa[cur][0].w,
                                fa[cur][1].x, fa[cur][1].y, fa[cur][1].z, fa[cur][1].w};
            const float b[8] = {fb[cur][0].x, fb[cur][0].y, fb[cur][0].z, fb[cur][0].w,
                                fb[cur][1].x, fb[cur][1].y, fb[cur][1].z, fb[cur][1].w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
    }

#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        float* crow = C + static_cast<long long>(row) * N + n0;
        *reinterpret_cast<float4*>(crow + tx * 4) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        *reinterpret_cast<float4*>(crow + 64 + tx * 4) =
            make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
}

// Generic bounds-checked path.
__global__ void __launch_bounds__(256)
sgemm_generic(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C,
              int M, int N, int K) {
    __shared__ float As[16][17];
    __shared__ float Bs[16][17];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int row = blockIdx.y * 16 + ty, col = blockIdx.x * 16 + tx;
    float acc = 0.f;
    for (int k0 = 0; k0 < K; k0 += 16) {
        As[ty][tx] = (row < M && k0 + tx < K) ? A[static_cast<long long>(row) * K + k0 + tx] : 0.f;
        Bs[ty][tx] = (k0 + ty < K && col < N) ? B[static_cast<long long>(k0 + ty) * N + col] : 0.f;
        __syncthreads();
        const int kmax = min(16, K - k0);
        for (int k = 0; k < kmax; ++k) acc = fmaf(As[ty][k], Bs[k][tx], acc);
        __syncthreads();
    }
    if (row < M && col < N) C[static_cast<long long>(row) * N + col] = acc;
}

}  // namespace hf

extern "C" int hf_gemm_simt(const float* A, const float* B, float* C, int M, int N, int K, int device,
                            void* stream) {
    HF_REQUIRE(A && B && C, "hf_gemm_simt: NULL operand");
    HF_REQUIRE(M > 0 && N > 0 && K > 0, "hf_gemm_simt: bad shape %dx%dx%d", M, N, K);
    hf::DeviceGuard g(device);
    HF_REQUIRE(g.ok, "hf_gemm_simt: cannot select device %d", device);
    cudaStream_t st = hf::as_stream(stream);
    bool aligned = (reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) |
                    reinterpret_cast<uintptr_t>(C)) % 16 == 0;
    if (aligned && M % hf::SB_M == 0 && N % hf::SB_N == 0 && K % hf::SB_K == 0) {
        int tiles = (M / hf::SB_M) * (N / hf::SB_N);
        hf::sgemm_128x128<<<tiles, 256, 0, st>>>(A, B, C, M, N, K);
    } else {
        dim3 grid((N + 15) / 16, (M + 15) / 16);
        hf::sgemm_generic<<<grid, 256, 0, st>>>(A, B, C, M, N, K);
    }
    HF_CHECK_LAUNCH();
    return HF_OK;
}
