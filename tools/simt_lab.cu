// SIMT GEMM tuning lab (not product code): the sgemm_128x128 main loop of
// csrc/gemm_simt.cu as a template over (k-tile depth, pipeline stages), timed
// with CUDA events at 4096^3 and checked bit-for-bit against the product
// shape (same k order => identical results).  Build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a -o tools/simt_lab tools/simt_lab.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void ffma2(unsigned long long& d, unsigned long long a, unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int BK, int ST>
__global__ void __launch_bounds__(256, 2)
sgemm_v(const float* __restrict__ At, const float* __restrict__ B, float* __restrict__ C, int M, int N, int K) {
    constexpr int BM = 128, BN = 128;
    extern __shared__ __align__(16) float sm[];
    float* As = sm;
    float* Bs = sm + ST * BK * BM;
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int ty = (warp >> 1) * 4 + (lane >> 3);
    const int tx = (warp & 1) * 8 + (lane & 7);
    const int tiles_n = N / BN, tiles_m = M / BM;
    const int group = 8, bid = blockIdx.x, per_group = group * tiles_n;
    const int g = bid / per_group, first_m = g * group;
    const int gm = min(tiles_m - first_m, group);
    const int tm = first_m + (bid % per_group) % gm, tn = (bid % per_group) / gm;
    const int m0 = tm * BM, n0 = tn * BN;
    const int c_row = t >> 5, c_col = (t & 31) * 4;
    const float* Ag = At + static_cast<long long>(c_row) * M + m0 + c_col;
    const float* Bg = B + static_cast<long long>(c_row) * N + n0 + c_col;
    auto issue = [&](int kt, int stage) {
        const long long ka = static_cast<long long>(kt) * BK * M;
        const long long kb = static_cast<long long>(kt) * BK * N;
        float* as = As + stage * BK * BM + c_row * BM + c_col;
        float* bs = Bs + stage * BK * BN + c_row * BN + c_col;
#pragma unroll
        for (int r = 0; r < BK; r += 8) {
            cp_async16(as + r * BM, Ag + ka + static_cast<long long>(r) * M);
            cp_async16(bs + r * BN, Bg + kb + static_cast<long long>(r) * N);
        }
    };
    unsigned long long acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0ull;
    const int nk = K / BK;
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < nk) issue(s, s);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<ST - 2>();
        __syncthreads();
        {
            const int nt = kt + ST - 1;
            if (nt < nk) issue(nt, nt % ST);
            cp_async_commit();
        }
        const float* as = As + (kt % ST) * BK * BM;
        const float* bs = Bs + (kt % ST) * BK * BN;
        float4 fa[2][2], fb[2][2];
        fa[0][0] = *reinterpret_cast<const float4*>(as + ty * 4);
        fa[0][1] = *reinterpret_cast<const float4*>(as + 64 + ty * 4);
        fb[0][0] = *reinterpret_cast<const float4*>(bs + tx * 4);
        fb[0][1] = *reinterpret_cast<const float4*>(bs + 64 + tx * 4);
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            const int cur = k & 1, nxt = cur ^ 1;
            if (k + 1 < BK) {
                fa[nxt][0] = *reinterpret_cast<const float4*>(as + (k + 1) * BM + ty * 4);
                fa[nxt][1] = *reinterpret_cast<const float4*>(as + (k + 1) * BM + 64 + ty * 4);
                fb[nxt][0] = *reinterpret_cast<const float4*>(bs + (k + 1) * BN + tx * 4);
                fb[nxt][1] = *reinterpret_cast<const float4*>(bs + (k + 1) * BN + 64 + tx * 4);
            }
            const float a[8] = {fa[cur][0].x, fa[cur][0].y, fa[cur][0].z, fa[cur][0].w,
                                fa[cur][1].x, fa[cur][1].y, fa[cur][1].z, fa[cur][1].w};
            const unsigned long long b[4] = {pack2(fb[cur][0].x, fb[cur][0].y), pack2(fb[cur][0].z, fb[cur][0].w),
                                             pack2(fb[cur][1].x, fb[cur][1].y), pack2(fb[cur][1].z, fb[cur][1].w)};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const unsigned long long ai = pack2(a[i], a[i]);
#pragma unroll
                for (int j = 0; j < 4; ++j) ffma2(acc[i][j], ai, b[j]);
            }
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        float* crow = C + static_cast<long long>(row) * N + n0;
        *reinterpret_cast<ulonglong2*>(crow + tx * 4) = make_ulonglong2(acc[i][0], acc[i][1]);
        *reinterpret_cast<ulonglong2*>(crow + 64 + tx * 4) = make_ulonglong2(acc[i][2], acc[i][3]);
    }
}

// m-pair form: FFMA2 pairs run along m (the A^T float4s), b is the broadcast
// scalar.  Same per-output fma chain as sgemm_v, so bit-identical results.
template <int BK, int ST, bool PAIR_OUTER>
__global__ void __launch_bounds__(256, 2)
sgemm_mpair(const float* __restrict__ At, const float* __restrict__ B, float* __restrict__ C, int M, int N, int K) {
    constexpr int BM = 128, BN = 128;
    extern __shared__ __align__(16) float sm[];
    float* As = sm;
    float* Bs = sm + ST * BK * BM;
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int ty = (warp >> 1) * 4 + (lane >> 3);
    const int tx = (warp & 1) * 8 + (lane & 7);
    const int tiles_n = N / BN, tiles_m = M / BM;
    const int group = 8, bid = blockIdx.x, per_group = group * tiles_n;
    const int g = bid / per_group, first_m = g * group;
    const int gm = min(tiles_m - first_m, group);
    const int tm = first_m + (bid % per_group) % gm, tn = (bid % per_group) / gm;
    const int m0 = tm * BM, n0 = tn * BN;
    const int c_row = t >> 5, c_col = (t & 31) * 4;
    const float* Ag = At + static_cast<long long>(c_row) * M + m0 + c_col;
    const float* Bg = B + static_cast<long long>(c_row) * N + n0 + c_col;
    auto issue = [&](int kt, int stage) {
        const long long ka = static_cast<long long>(kt) * BK * M;
        const long long kb = static_cast<long long>(kt) * BK * N;
        float* as = As + stage * BK * BM + c_row * BM + c_col;
        float* bs = Bs + stage * BK * BN + c_row * BN + c_col;
#pragma unroll
        for (int r = 0; r < BK; r += 8) {
            cp_async16(as + r * BM, Ag + ka + static_cast<long long>(r) * M);
            cp_async16(bs + r * BN, Bg + kb + static_cast<long long>(r) * N);
        }
    };
    // acc[p][j] holds rows (2p, 2p+1) of column j: the pair runs along m
    unsigned long long acc[4][8];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[p][j] = 0ull;
    const int nk = K / BK;
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < nk) issue(s, s);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<ST - 2>();
        __syncthreads();
        {
            const int nt = kt + ST - 1;
            if (nt < nk) issue(nt, nt % ST);
            cp_async_commit();
        }
        const float* as = As + (kt % ST) * BK * BM;
        const float* bs = Bs + (kt % ST) * BK * BN;
        float4 fa[2][2], fb[2][2];
        fa[0][0] = *reinterpret_cast<const float4*>(as + ty * 4);
        fa[0][1] = *reinterpret_cast<const float4*>(as + 64 + ty * 4);
        fb[0][0] = *reinterpret_cast<const float4*>(bs + tx * 4);
        fb[0][1] = *reinterpret_cast<const float4*>(bs + 64 + tx * 4);
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            const int cur = k & 1, nxt = cur ^ 1;
            if (k + 1 < BK) {
                fa[nxt][0] = *reinterpret_cast<const float4*>(as + (k + 1) * BM + ty * 4);
                fa[nxt][1] = *reinterpret_cast<const float4*>(as + (k + 1) * BM + 64 + ty * 4);
                fb[nxt][0] = *reinterpret_cast<const float4*>(bs + (k + 1) * BN + tx * 4);
                fb[nxt][1] = *reinterpret_cast<const float4*>(bs + (k + 1) * BN + 64 + tx * 4);
            }
            const unsigned long long a[4] = {pack2(fa[cur][0].x, fa[cur][0].y), pack2(fa[cur][0].z, fa[cur][0].w),
                                             pack2(fa[cur][1].x, fa[cur][1].y), pack2(fa[cur][1].z, fa[cur][1].w)};
            const float b[8] = {fb[cur][0].x, fb[cur][0].y, fb[cur][0].z, fb[cur][0].w,
                                fb[cur][1].x, fb[cur][1].y, fb[cur][1].z, fb[cur][1].w};
            if (PAIR_OUTER) {
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int j = 0; j < 8; ++j) ffma2(acc[p][j], pack2(b[j], b[j]), a[p]);
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const unsigned long long bj = pack2(b[j], b[j]);
#pragma unroll
                    for (int p = 0; p < 4; ++p) ffma2(acc[p][j], bj, a[p]);
                }
            }
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        float* crow = C + static_cast<long long>(row) * N + n0;
        float r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float lo, hi;
            asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i / 2][j]));
            r[j] = (i & 1) ? hi : lo;
        }
        *reinterpret_cast<float4*>(crow + tx * 4) = make_float4(r[0], r[1], r[2], r[3]);
        *reinterpret_cast<float4*>(crow + 64 + tx * 4) = make_float4(r[4], r[5], r[6], r[7]);
    }
}

template <int BK, int ST>
__global__ void __launch_bounds__(256, 2)
sgemm_diag(const float* __restrict__ At, const float* __restrict__ B, float* __restrict__ C, int M, int N, int K) {
    constexpr int BM = 128, BN = 128;
    extern __shared__ __align__(16) float sm[];
    float* As = sm;
    float* Bs = sm + ST * BK * BM;
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int ty = (warp >> 1) * 4 + (lane >> 3);
    const int tx = (warp & 1) * 8 + (lane & 7);
    const int tiles_n = N / BN, tiles_m = M / BM;
    const int group = 8, bid = blockIdx.x, per_group = group * tiles_n;
    const int g = bid / per_group, first_m = g * group;
    const int gm = min(tiles_m - first_m, group);
    const int tm = first_m + (bid % per_group) % gm, tn = (bid % per_group) / gm;
    const int m0 = tm * BM, n0 = tn * BN;
    const int c_row = t >> 5, c_col = (t & 31) * 4;
    const float* Ag = At + static_cast<long long>(c_row) * M + m0 + c_col;
    const float* Bg = B + static_cast<long long>(c_row) * N + n0 + c_col;
    auto issue = [&](int kt, int stage) {
        const long long ka = static_cast<long long>(kt) * BK * M;
        const long long kb = static_cast<long long>(kt) * BK * N;
        float* as = As + stage * BK * BM + c_row * BM + c_col;
        float* bs = Bs + stage * BK * BN + c_row * BN + c_col;
#pragma unroll
        for (int r = 0; r < BK; r += 8) {
            cp_async16(as + r * BM, Ag + ka + static_cast<long long>(r) * M);
            cp_async16(bs + r * BN, Bg + kb + static_cast<long long>(r) * N);
        }
    };
    // d1[p][q] = {C(r2p, c2q), C(r2p+1, c2q+1)}, d2[p][q] = {C(r2p, c2q+1), C(r2p+1, c2q)}
    unsigned long long d1[4][4], d2[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) d1[i][j] = d2[i][j] = 0ull;
    const int nk = K / BK;
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < nk) issue(s, s);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<ST - 2>();
        __syncthreads();
        {
            const int nt = kt + ST - 1;
            if (nt < nk) issue(nt, nt % ST);
            cp_async_commit();
        }
        const float* as = As + (kt % ST) * BK * BM;
        const float* bs = Bs + (kt % ST) * BK * BN;
        float4 fa[2][2], fb[2][2];
        fa[0][0] = *reinterpret_cast<const float4*>(as + ty * 4);
        fa[0][1] = *reinterpret_cast<const float4*>(as + 64 + ty * 4);
        fb[0][0] = *reinterpret_cast<const float4*>(bs + tx * 4);
        fb[0][1] = *reinterpret_cast<const float4*>(bs + 64 + tx * 4);
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            const int cur = k & 1, nxt = cur ^ 1;
            if (k + 1 < BK) {
                fa[nxt][0] = *reinterpret_cast<const float4*>(as + (k + 1) * BM + ty * 4);
                fa[nxt][1] = *reinterpret_cast<const float4*>(as + (k + 1) * BM + 64 + ty * 4);
                fb[nxt][0] = *reinterpret_cast<const float4*>(bs + (k + 1) * BN + tx * 4);
                fb[nxt][1] = *reinterpret_cast<const float4*>(bs + (k + 1) * BN + 64 + tx * 4);
            }
            const unsigned long long ap[4] = {pack2(fa[cur][0].x, fa[cur][0].y), pack2(fa[cur][0].z, fa[cur][0].w),
                                              pack2(fa[cur][1].x, fa[cur][1].y), pack2(fa[cur][1].z, fa[cur][1].w)};
            const unsigned long long bp[4] = {pack2(fb[cur][0].x, fb[cur][0].y), pack2(fb[cur][0].z, fb[cur][0].w),
                                              pack2(fb[cur][1].x, fb[cur][1].y), pack2(fb[cur][1].z, fb[cur][1].w)};
            const unsigned long long bs[4] = {pack2(fb[cur][0].y, fb[cur][0].x), pack2(fb[cur][0].w, fb[cur][0].z),
                                              pack2(fb[cur][1].y, fb[cur][1].x), pack2(fb[cur][1].w, fb[cur][1].z)};
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    ffma2(d1[p][q], ap[p], bp[q]);
                    ffma2(d2[p][q], ap[p], bs[q]);
                }
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int p = 0; p < 4; ++p) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {       // row 2p + h of the thread's 8
            const int i = 2 * p + h;
            const int row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
            float* crow = C + static_cast<long long>(row) * N + n0;
            float v[8];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float2 x = *reinterpret_cast<float2*>(&d1[p][q]);
                float2 y = *reinterpret_cast<float2*>(&d2[p][q]);
                v[2 * q] = h == 0 ? x.x : y.y;
                v[2 * q + 1] = h == 0 ? y.x : x.y;
            }
            *reinterpret_cast<float4*>(crow + tx * 4) = make_float4(v[0], v[1], v[2], v[3]);
            *reinterpret_cast<float4*>(crow + 64 + tx * 4) = make_float4(v[4], v[5], v[6], v[7]);
        }
    }
}


// 16 (m) x 4 (n) thread tile: per k-step 16 broadcast a scalars x 2 b pairs,
// issued b-pair-outer so each b pair is reused by 16 consecutive FFMA2 (the
// form tools/ffma2_forms.cu measured at the FFMA2 peak).  Warp = 32 lanes
// along n (b fragment 512 contiguous bytes), 8 warps along m (a fragment
// broadcast).  Each output is the same FMA chain in k order as the product
// kernel, so results are bit-identical.
template <int BK, int ST, bool B_OUTER>
__global__ void __launch_bounds__(256, 2)
sgemm_16x4(const float* __restrict__ At, const float* __restrict__ B, float* __restrict__ C, int M, int N, int K) {
    constexpr int BM = 128, BN = 128;
    extern __shared__ __align__(16) float sm[];
    float* As = sm;
    float* Bs = sm + ST * BK * BM;
    const int t = threadIdx.x;
    const int tx = t & 31;          // n: columns 4*tx .. 4*tx+3
    const int ty = t >> 5;          // m: rows 16*ty .. 16*ty+15
    const int tiles_n = N / BN, tiles_m = M / BM;
    const int group = 16, bid = blockIdx.x, per_group = group * tiles_n;
    const int g = bid / per_group, first_m = g * group;
    const int gm = min(tiles_m - first_m, group);
    const int tm = first_m + (bid % per_group) % gm, tn = (bid % per_group) / gm;
    const int m0 = tm * BM, n0 = tn * BN;
    const int c_row = t >> 5, c_col = (t & 31) * 4;
    const float* Ag = At + static_cast<long long>(c_row) * M + m0 + c_col;
    const float* Bg = B + static_cast<long long>(c_row) * N + n0 + c_col;
    auto issue = [&](int kt, int stage) {
        const long long ka = static_cast<long long>(kt) * BK * M;
        const long long kb = static_cast<long long>(kt) * BK * N;
        float* as = As + stage * BK * BM + c_row * BM + c_col;
        float* bs = Bs + stage * BK * BN + c_row * BN + c_col;
#pragma unroll
        for (int r = 0; r < BK; r += 8) {
            cp_async16(as + r * BM, Ag + ka + static_cast<long long>(r) * M);
            cp_async16(bs + r * BN, Bg + kb + static_cast<long long>(r) * N);
        }
    };
    unsigned long long acc[16][2];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0ull;
    const int nk = K / BK;
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < nk) issue(s, s);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<ST - 2>();
        __syncthreads();
        {
            const int nt = kt + ST - 1;
            if (nt < nk) issue(nt, nt % ST);
            cp_async_commit();
        }
        const float* as = As + (kt % ST) * BK * BM + ty * 16;
        const float* bs = Bs + (kt % ST) * BK * BN + tx * 4;
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            const float4 a0 = *reinterpret_cast<const float4*>(as + k * BM);
            const float4 a1 = *reinterpret_cast<const float4*>(as + k * BM + 4);
            const float4 a2 = *reinterpret_cast<const float4*>(as + k * BM + 8);
            const float4 a3 = *reinterpret_cast<const float4*>(as + k * BM + 12);
            const float4 bv = *reinterpret_cast<const float4*>(bs + k * BN);
            const float a[16] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w,
                                 a2.x, a2.y, a2.z, a2.w, a3.x, a3.y, a3.z, a3.w};
            const unsigned long long b[2] = {pack2(bv.x, bv.y), pack2(bv.z, bv.w)};
            if (B_OUTER) {
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int i = 0; i < 16; ++i) ffma2(acc[i][j], pack2(a[i], a[i]), b[j]);
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const unsigned long long ai = pack2(a[i], a[i]);
                    ffma2(acc[i][0], ai, b[0]);
                    ffma2(acc[i][1], ai, b[1]);
                }
            }
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        float* crow = C + static_cast<long long>(m0 + ty * 16 + i) * N + n0 + tx * 4;
        *reinterpret_cast<ulonglong2*>(crow) = make_ulonglong2(acc[i][0], acc[i][1]);
    }
}

template <int BK, int ST, bool B_OUTER>
static void run16(const char* name, const float* At, const float* B, float* C, const float* Cref, int n,
                  size_t bytes) {
    auto k = sgemm_16x4<BK, ST, B_OUTER>;
    const int smem = ST * BK * 256 * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int tiles = (n / 128) * (n / 128);
    for (int i = 0; i < 3; ++i) k<<<tiles, 256, smem>>>(At, B, C, n, n, n);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int i = 0; i < 20; ++i) {
        cudaEventRecord(e0);
        k<<<tiles, 256, smem>>>(At, B, C, n, n, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    std::vector<float> h(bytes / 4), r(bytes / 4);
    cudaMemcpy(h.data(), C, bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(r.data(), Cref, bytes, cudaMemcpyDeviceToHost);
    const bool same = memcmp(h.data(), r.data(), bytes) == 0;
    printf("{\"variant\": \"%s\", \"ms_min\": %.4f, \"tflops\": %.2f, \"bit_identical\": %s, \"err\": \"%s\"}\n", name,
           best, 2.0 * n * n * (double)n / (best * 1e-3) / 1e12, same ? "true" : "false",
           cudaGetErrorString(cudaGetLastError()));
}

template <int BK, int ST, bool DIAG = false, int MPAIR = 0>
static void run(const char* name, const float* At, const float* B, float* C, const float* Cref, int n, size_t bytes) {
    auto k = MPAIR == 1 ? sgemm_mpair<BK, ST, true> : MPAIR == 2 ? sgemm_mpair<BK, ST, false>
           : DIAG ? sgemm_diag<BK, ST> : sgemm_v<BK, ST>;
    const int smem = ST * BK * 256 * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int tiles = (n / 128) * (n / 128);
    for (int i = 0; i < 3; ++i) k<<<tiles, 256, smem>>>(At, B, C, n, n, n);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9, sum = 0;
    for (int i = 0; i < 20; ++i) {
        cudaEventRecord(e0);
        k<<<tiles, 256, smem>>>(At, B, C, n, n, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
        sum += ms;
    }
    bool same = true;
    if (Cref) {
        std::vector<float> h(bytes / 4), r(bytes / 4);
        cudaMemcpy(h.data(), C, bytes, cudaMemcpyDeviceToHost);
        cudaMemcpy(r.data(), Cref, bytes, cudaMemcpyDeviceToHost);
        same = memcmp(h.data(), r.data(), bytes) == 0;
    }
    double fl = 2.0 * n * n * (double)n;
    printf("{\"variant\": \"%s\", \"smem\": %d, \"ms_min\": %.4f, \"ms_mean\": %.4f, \"tflops\": %.2f, "
           "\"bit_identical\": %s, \"err\": \"%s\"}\n",
           name, smem, best, sum / 20, fl / (best * 1e-3) / 1e12, same ? "true" : "false",
           cudaGetErrorString(cudaGetLastError()));
}

__global__ void init(float* p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t x = (uint32_t)i * 2654435761u ^ seed;
        x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
        p[i] = 1.0f + (x >> 8) * (1.0f / 16777216.0f);
    }
}

int main(int argc, char** argv) {
    int n = argc > 1 ? atoi(argv[1]) : 4096;
    size_t bytes = (size_t)n * n * 4;
    float *At, *B, *C, *C0;
    cudaMalloc(&At, bytes); cudaMalloc(&B, bytes); cudaMalloc(&C, bytes); cudaMalloc(&C0, bytes);
    init<<<1184, 256>>>(At, (size_t)n * n, 1);
    init<<<1184, 256>>>(B, (size_t)n * n, 2);
    run<16, 3>("k16s3 (product)", At, B, C0, nullptr, n, bytes);
    run<16, 3, false, 1>("m-pair pair-outer k16s3", At, B, C, C0, n, bytes);
    run<16, 3, false, 2>("m-pair scalar-outer k16s3", At, B, C, C0, n, bytes);
    run<32, 2, false, 1>("m-pair pair-outer k32s2", At, B, C, C0, n, bytes);
    run<16, 3, true>("diag k16s3", At, B, C, C0, n, bytes);
    run<16, 4, true>("diag k16s4", At, B, C, C0, n, bytes);
    run<32, 2, true>("diag k32s2", At, B, C, C0, n, bytes);
    run<16, 3>("k16s3 (again)", At, B, C, C0, n, bytes);
    run16<16, 3, true>("16x4 b-outer k16s3", At, B, C, C0, n, bytes);
    run16<16, 3, false>("16x4 a-outer k16s3", At, B, C, C0, n, bytes);
    run16<32, 2, true>("16x4 b-outer k32s2", At, B, C, C0, n, bytes);
    run16<8, 4, true>("16x4 b-outer k8s4", At, B, C, C0, n, bytes);
    return 0;
}
