// SIMT GEMM lab 2 (not product code): 8 x 16 outputs per thread, 128-thread
// CTAs on the product's 128 x 128 CTA tile (two CTAs per SM, as the product),
// so each thread holds 64 accumulator pairs and reads 6 LDS.128 per 64 FFMA2
// (the product: 4 per 32).  Chain accumulation in ascending k, so results
// are bit-identical to the product's single-chain kernel (sgemm_v here).
// Optional blocked accumulation (CH k-tiles per chain, running totals in
// shared memory) as the product kernel does.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/simt_lab2 tools/simt_lab2.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cstdlib>
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

// product shape (single chain): 256 threads, 8x8 per thread
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

// 8 (m) x 16 (n) per thread, 128 threads.  Warp = 4 (m) x 8 (n) lanes; the 4
// warps stack along m.  Thread rows: ty*4 + {0..3} and 64 + ty*4 + {0..3}
// (ty = warp*4 + lane/8 in 0..15); columns c*32 + tx*4 + {0..3}, c = 0..3
// (tx = lane%8).  Every LDS.128 of a warp touches 4 (A) or 8 (B) distinct
// 16-byte words: one wavefront each.
template <int BK, int ST, int CH, int ORDER>
__global__ void __launch_bounds__(128, 2)
sgemm_8x16(const float* __restrict__ At, const float* __restrict__ B, float* __restrict__ C, int M, int N, int K) {
    constexpr int BM = 128, BN = 128, NT = 128;
    extern __shared__ __align__(16) float sm[];
    float* As = sm;
    float* Bs = sm + ST * BK * BM;
    ulonglong2* Tot = reinterpret_cast<ulonglong2*>(Bs + ST * BK * BN);   // [32][128] x 16 B
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int ty = warp * 4 + (lane >> 3);
    const int tx = lane & 7;
    const int tiles_n = N / BN, tiles_m = M / BM;
    const int group = 16, bid = blockIdx.x, per_group = group * tiles_n;
    const int g = bid / per_group, first_m = g * group;
    const int gm = min(tiles_m - first_m, group);
    const int tm = first_m + (bid % per_group) % gm, tn = (bid % per_group) / gm;
    const int m0 = tm * BM, n0 = tn * BN;
    // copy: each k-row of a tile is 32 chunks of 16 B; thread t moves chunk
    // (t & 31) of rows (t >> 5) + 4r
    const int c_row = t >> 5, c_col = (t & 31) * 4;
    const float* Ag = At + static_cast<long long>(c_row) * M + m0 + c_col;
    const float* Bg = B + static_cast<long long>(c_row) * N + n0 + c_col;
    auto issue = [&](int kt, int stage) {
        const long long ka = static_cast<long long>(kt) * BK * M;
        const long long kb = static_cast<long long>(kt) * BK * N;
        float* as = As + stage * BK * BM + c_row * BM + c_col;
        float* bs = Bs + stage * BK * BN + c_row * BN + c_col;
#pragma unroll
        for (int r = 0; r < BK; r += 4) {
            cp_async16(as + r * BM, Ag + ka + static_cast<long long>(r) * M);
            cp_async16(bs + r * BN, Bg + kb + static_cast<long long>(r) * N);
        }
    };
    unsigned long long acc[8][8];   // [row i][col pair j]: cols (j>>1)*32 + tx*4 + 2*(j&1)
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0ull;
    if constexpr (CH > 0) {
#pragma unroll
        for (int q = 0; q < 32; ++q) Tot[q * NT + t] = make_ulonglong2(0ull, 0ull);
    }
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
        float4 fa[2][2], fb[2][4];
        fa[0][0] = *reinterpret_cast<const float4*>(as + ty * 4);
        fa[0][1] = *reinterpret_cast<const float4*>(as + 64 + ty * 4);
#pragma unroll
        for (int c = 0; c < 4; ++c) fb[0][c] = *reinterpret_cast<const float4*>(bs + c * 32 + tx * 4);
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            const int cur = k & 1, nxt = cur ^ 1;
            if (k + 1 < BK) {
                fa[nxt][0] = *reinterpret_cast<const float4*>(as + (k + 1) * BM + ty * 4);
                fa[nxt][1] = *reinterpret_cast<const float4*>(as + (k + 1) * BM + 64 + ty * 4);
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    fb[nxt][c] = *reinterpret_cast<const float4*>(bs + (k + 1) * BN + c * 32 + tx * 4);
            }
            const float a[8] = {fa[cur][0].x, fa[cur][0].y, fa[cur][0].z, fa[cur][0].w,
                                fa[cur][1].x, fa[cur][1].y, fa[cur][1].z, fa[cur][1].w};
            unsigned long long b[8];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                b[2 * c] = pack2(fb[cur][c].x, fb[cur][c].y);
                b[2 * c + 1] = pack2(fb[cur][c].z, fb[cur][c].w);
            }
            if (ORDER == 0) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const unsigned long long ai = pack2(a[i], a[i]);
#pragma unroll
                    for (int j = 0; j < 8; ++j) ffma2(acc[i][j], ai, b[j]);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j)
#pragma unroll
                    for (int i = 0; i < 8; ++i) ffma2(acc[i][j], pack2(a[i], a[i]), b[j]);
            }
        }
        if constexpr (CH > 0) {
            if ((kt + 1) % CH == 0 || kt + 1 == nk) {
                const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(Tot + t));
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        asm volatile(
                            "{\n\t.reg .b64 t0, t1, t2, t3;\n\t"
                            "ld.shared.v2.b64 {t0, t1}, [%4];\n\t"
                            "ld.shared.v2.b64 {t2, t3}, [%4+2048];\n\t"
                            "add.rn.f32x2 t0, t0, %0;\n\tadd.rn.f32x2 t1, t1, %1;\n\t"
                            "add.rn.f32x2 t2, t2, %2;\n\tadd.rn.f32x2 t3, t3, %3;\n\t"
                            "st.shared.v2.b64 [%4], {t0, t1};\n\t"
                            "st.shared.v2.b64 [%4+2048], {t2, t3};\n\t"
                            "mov.b64 %0, 0;\n\tmov.b64 %1, 0;\n\tmov.b64 %2, 0;\n\tmov.b64 %3, 0;\n\t}"
                            : "+l"(acc[i][4 * h]), "+l"(acc[i][4 * h + 1]), "+l"(acc[i][4 * h + 2]),
                              "+l"(acc[i][4 * h + 3])
                            : "r"(base + static_cast<uint32_t>((4 * i + 2 * h) * NT * 16))
                            : "memory");
            }
        }
    }
    cp_async_wait<0>();
    if constexpr (CH > 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const ulonglong2 v = Tot[(4 * i + q) * NT + t];
                acc[i][2 * q] = v.x;
                acc[i][2 * q + 1] = v.y;
            }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        float* crow = C + static_cast<long long>(row) * N + n0 + tx * 4;
#pragma unroll
        for (int c = 0; c < 4; ++c)
            *reinterpret_cast<ulonglong2*>(crow + c * 32) = make_ulonglong2(acc[i][2 * c], acc[i][2 * c + 1]);
    }
}


// A read row-major (no A^T pre-pass): each k-tile of A (128 rows x 16 k) is
// loaded by LDG.128 into registers one k-tile ahead (lane = row, 4 chunks of
// 4 k per thread) and stored transposed into a 2-stage smem ring after the
// k-tile's math (STS.32, lanes on consecutive rows: conflict-free); B streams
// by cp.async as before.  8 x 16 outputs per thread, 128 threads.
template <int CH, int ORDER>
__global__ void __launch_bounds__(128, 2)
sgemm_rowa(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C, int M, int N, int K) {
    constexpr int BM = 128, BN = 128, BK = 16, NT = 128, SB = 3;
    extern __shared__ __align__(16) float sm[];
    float* As = sm;                         // [2][BK][BM]
    float* Bs = sm + 2 * BK * BM;           // [SB][BK][BN]
    ulonglong2* Tot = reinterpret_cast<ulonglong2*>(Bs + SB * BK * BN);
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int ty = warp * 4 + (lane >> 3);
    const int tx = lane & 7;
    const int tiles_n = N / BN, tiles_m = M / BM;
    const int group = 16, bid = blockIdx.x, per_group = group * tiles_n;
    const int g = bid / per_group, first_m = g * group;
    const int gm = min(tiles_m - first_m, group);
    const int tm = first_m + (bid % per_group) % gm, tn = (bid % per_group) / gm;
    const int m0 = tm * BM, n0 = tn * BN;
    // A: thread t owns row m0 + t (4 x 16 B of each k-tile)
    const float4* Ag = reinterpret_cast<const float4*>(A + static_cast<long long>(m0 + t) * K);
    const int c_row = t >> 5, c_col = (t & 31) * 4;
    const float* Bg = B + static_cast<long long>(c_row) * N + n0 + c_col;
    auto issue_b = [&](int kt, int stage) {
        const long long kb = static_cast<long long>(kt) * BK * N;
        float* bs = Bs + stage * BK * BN + c_row * BN + c_col;
#pragma unroll
        for (int r = 0; r < BK; r += 4) cp_async16(bs + r * BN, Bg + kb + static_cast<long long>(r) * N);
    };
    float4 ra[4];
    auto load_a = [&](int kt) {
#pragma unroll
        for (int c = 0; c < 4; ++c) ra[c] = __ldg(Ag + kt * 4 + c);
    };
    auto store_a = [&](int stage) {
        float* as = As + stage * BK * BM + t;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            as[(4 * c + 0) * BM] = ra[c].x;
            as[(4 * c + 1) * BM] = ra[c].y;
            as[(4 * c + 2) * BM] = ra[c].z;
            as[(4 * c + 3) * BM] = ra[c].w;
        }
    };
    unsigned long long acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0ull;
    if constexpr (CH > 0) {
#pragma unroll
        for (int q = 0; q < 32; ++q) Tot[q * NT + t] = make_ulonglong2(0ull, 0ull);
    }
    const int nk = K / BK;
    load_a(0);
    store_a(0);
#pragma unroll
    for (int s = 0; s < SB - 1; ++s) {
        if (s < nk) issue_b(s, s);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<SB - 2>();
        __syncthreads();
        {
            const int nt = kt + SB - 1;
            if (nt < nk) issue_b(nt, nt % SB);
            cp_async_commit();
        }
        if (kt + 1 < nk) load_a(kt + 1);
        const float* as = As + (kt & 1) * BK * BM;
        const float* bs = Bs + (kt % SB) * BK * BN;
        float4 fa[2][2], fb[2][4];
        fa[0][0] = *reinterpret_cast<const float4*>(as + ty * 4);
        fa[0][1] = *reinterpret_cast<const float4*>(as + 64 + ty * 4);
#pragma unroll
        for (int c = 0; c < 4; ++c) fb[0][c] = *reinterpret_cast<const float4*>(bs + c * 32 + tx * 4);
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            const int cur = k & 1, nxt = cur ^ 1;
            if (k + 1 < BK) {
                fa[nxt][0] = *reinterpret_cast<const float4*>(as + (k + 1) * BM + ty * 4);
                fa[nxt][1] = *reinterpret_cast<const float4*>(as + (k + 1) * BM + 64 + ty * 4);
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    fb[nxt][c] = *reinterpret_cast<const float4*>(bs + (k + 1) * BN + c * 32 + tx * 4);
            }
            const float a[8] = {fa[cur][0].x, fa[cur][0].y, fa[cur][0].z, fa[cur][0].w,
                                fa[cur][1].x, fa[cur][1].y, fa[cur][1].z, fa[cur][1].w};
            unsigned long long b[8];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                b[2 * c] = pack2(fb[cur][c].x, fb[cur][c].y);
                b[2 * c + 1] = pack2(fb[cur][c].z, fb[cur][c].w);
            }
            if (ORDER == 0) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const unsigned long long ai = pack2(a[i], a[i]);
#pragma unroll
                    for (int j = 0; j < 8; ++j) ffma2(acc[i][j], ai, b[j]);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j)
#pragma unroll
                    for (int i = 0; i < 8; ++i) ffma2(acc[i][j], pack2(a[i], a[i]), b[j]);
            }
        }
        if (kt + 1 < nk) store_a((kt + 1) & 1);
        if constexpr (CH > 0) {
            if ((kt + 1) % CH == 0 || kt + 1 == nk) {
                const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(Tot + t));
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        asm volatile(
                            "{\n\t.reg .b64 t0, t1, t2, t3;\n\t"
                            "ld.shared.v2.b64 {t0, t1}, [%4];\n\t"
                            "ld.shared.v2.b64 {t2, t3}, [%4+2048];\n\t"
                            "add.rn.f32x2 t0, t0, %0;\n\tadd.rn.f32x2 t1, t1, %1;\n\t"
                            "add.rn.f32x2 t2, t2, %2;\n\tadd.rn.f32x2 t3, t3, %3;\n\t"
                            "st.shared.v2.b64 [%4], {t0, t1};\n\t"
                            "st.shared.v2.b64 [%4+2048], {t2, t3};\n\t"
                            "mov.b64 %0, 0;\n\tmov.b64 %1, 0;\n\tmov.b64 %2, 0;\n\tmov.b64 %3, 0;\n\t}"
                            : "+l"(acc[i][4 * h]), "+l"(acc[i][4 * h + 1]), "+l"(acc[i][4 * h + 2]),
                              "+l"(acc[i][4 * h + 3])
                            : "r"(base + static_cast<uint32_t>((4 * i + 2 * h) * NT * 16))
                            : "memory");
            }
        }
    }
    cp_async_wait<0>();
    if constexpr (CH > 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const ulonglong2 v = Tot[(4 * i + q) * NT + t];
                acc[i][2 * q] = v.x;
                acc[i][2 * q + 1] = v.y;
            }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        float* crow = C + static_cast<long long>(row) * N + n0 + tx * 4;
#pragma unroll
        for (int c = 0; c < 4; ++c)
            *reinterpret_cast<ulonglong2*>(crow + c * 32) = make_ulonglong2(acc[i][2 * c], acc[i][2 * c + 1]);
    }
}

// A read row-major through cp.async into an m-major smem tile ([128 m][16 k],
// 16-byte chunks XOR-swizzled by (m >> 2) & 3): no A^T pre-pass.  A
// fragments are LDS.128 over 4 consecutive k of each of the thread's 8 rows
// (the same 2 LDS.128 per k-step as the k-major layout), loaded once per
// group of 4 k-steps; B as before.  8 x 16 outputs per thread, j-outer.
template <int CH>
__global__ void __launch_bounds__(128, 2)
sgemm_am(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C, int M, int N, int K) {
    constexpr int BM = 128, BN = 128, BK = 16, NT = 128, ST = 3;
    extern __shared__ __align__(16) float sm[];
    float* As = sm;                         // [ST][BM][BK] swizzled
    float* Bs = sm + ST * BK * BM;          // [ST][BK][BN]
    ulonglong2* Tot = reinterpret_cast<ulonglong2*>(Bs + ST * BK * BN);
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int ty = warp * 4 + (lane >> 3);
    const int tx = lane & 7;
    const int sw = ty & 3;
    const int tiles_n = N / BN, tiles_m = M / BM;
    const int group = 16, bid = blockIdx.x, per_group = group * tiles_n;
    const int g = bid / per_group, first_m = g * group;
    const int gm = min(tiles_m - first_m, group);
    const int tm = first_m + (bid % per_group) % gm, tn = (bid % per_group) / gm;
    const int m0 = tm * BM, n0 = tn * BN;
    // A copy: 4 consecutive threads move the 4 chunks of one row; rows (t >> 2) + 32 r
    const int a_row = t >> 2, a_chk = t & 3;
    const float* Ag = A + static_cast<long long>(m0 + a_row) * K + a_chk * 4;
    const long long a32 = 32LL * K;
    const int c_row = t >> 5, c_col = (t & 31) * 4;
    const float* Bg = B + static_cast<long long>(c_row) * N + n0 + c_col;
    auto issue = [&](int kt, int stage) {
        float* as = As + stage * BK * BM;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int m = a_row + 32 * r;
            cp_async16(as + m * BK + ((a_chk ^ ((m >> 2) & 3)) << 2), Ag + r * a32 + kt * BK);
        }
        const long long kb = static_cast<long long>(kt) * BK * N;
        float* bs = Bs + stage * BK * BN + c_row * BN + c_col;
#pragma unroll
        for (int r = 0; r < BK; r += 4) cp_async16(bs + r * BN, Bg + kb + static_cast<long long>(r) * N);
    };
    unsigned long long acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0ull;
    if constexpr (CH > 0) {
#pragma unroll
        for (int q = 0; q < 32; ++q) Tot[q * NT + t] = make_ulonglong2(0ull, 0ull);
    }
    const int nk = K / BK;
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < nk) issue(s, s);
        cp_async_commit();
    }
    int arow[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) arow[i] = (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4)) * BK;
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
        float4 fb[2][4];
#pragma unroll
        for (int c = 0; c < 4; ++c) fb[0][c] = *reinterpret_cast<const float4*>(bs + c * 32 + tx * 4);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float4 a4[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a4[i] = *reinterpret_cast<const float4*>(as + arow[i] + ((q ^ sw) << 2));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int k = 4 * q + kk;
                const int cur = k & 1, nxt = cur ^ 1;
                if (k + 1 < BK) {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        fb[nxt][c] = *reinterpret_cast<const float4*>(bs + (k + 1) * BN + c * 32 + tx * 4);
                }
                float a[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    a[i] = kk == 0 ? a4[i].x : kk == 1 ? a4[i].y : kk == 2 ? a4[i].z : a4[i].w;
                unsigned long long b[8];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    b[2 * c] = pack2(fb[cur][c].x, fb[cur][c].y);
                    b[2 * c + 1] = pack2(fb[cur][c].z, fb[cur][c].w);
                }
#pragma unroll
                for (int j = 0; j < 8; ++j)
#pragma unroll
                    for (int i = 0; i < 8; ++i) ffma2(acc[i][j], pack2(a[i], a[i]), b[j]);
            }
        }
        if constexpr (CH > 0) {
            if ((kt + 1) % CH == 0 || kt + 1 == nk) {
                const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(Tot + t));
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        asm volatile(
                            "{\n\t.reg .b64 t0, t1, t2, t3;\n\t"
                            "ld.shared.v2.b64 {t0, t1}, [%4];\n\t"
                            "ld.shared.v2.b64 {t2, t3}, [%4+2048];\n\t"
                            "add.rn.f32x2 t0, t0, %0;\n\tadd.rn.f32x2 t1, t1, %1;\n\t"
                            "add.rn.f32x2 t2, t2, %2;\n\tadd.rn.f32x2 t3, t3, %3;\n\t"
                            "st.shared.v2.b64 [%4], {t0, t1};\n\t"
                            "st.shared.v2.b64 [%4+2048], {t2, t3};\n\t"
                            "mov.b64 %0, 0;\n\tmov.b64 %1, 0;\n\tmov.b64 %2, 0;\n\tmov.b64 %3, 0;\n\t}"
                            : "+l"(acc[i][4 * h]), "+l"(acc[i][4 * h + 1]), "+l"(acc[i][4 * h + 2]),
                              "+l"(acc[i][4 * h + 3])
                            : "r"(base + static_cast<uint32_t>((4 * i + 2 * h) * NT * 16))
                            : "memory");
            }
        }
    }
    cp_async_wait<0>();
    if constexpr (CH > 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const ulonglong2 v = Tot[(4 * i + q) * NT + t];
                acc[i][2 * q] = v.x;
                acc[i][2 * q + 1] = v.y;
            }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        float* crow = C + static_cast<long long>(row) * N + n0 + tx * 4;
#pragma unroll
        for (int c = 0; c < 4; ++c)
            *reinterpret_cast<ulonglong2*>(crow + c * 32) = make_ulonglong2(acc[i][2 * c], acc[i][2 * c + 1]);
    }
}

// Early-barrier k-loop: the barrier that publishes tile kt+1 sits before the
// last k-step of tile kt (whose fragments are already in registers), so the
// first LDS.128s of tile kt+1 overlap that k-step's 64 FFMA2 instead of
// following the barrier.  Stage kt is free after that barrier, so tile
// kt+ST is issued into it: ST tiles in flight.  8x16 per thread, j-outer.
template <int CH, int ST>
__global__ void __launch_bounds__(128, 2)
sgemm_early(const float* __restrict__ At, const float* __restrict__ B, float* __restrict__ C, int M, int N, int K) {
    constexpr int BM = 128, BN = 128, BK = 16, NT = 128;
    extern __shared__ __align__(16) float sm[];
    float* As = sm;
    float* Bs = sm + ST * BK * BM;
    ulonglong2* Tot = reinterpret_cast<ulonglong2*>(Bs + ST * BK * BN);
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int ty = warp * 4 + (lane >> 3);
    const int tx = lane & 7;
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
        for (int r = 0; r < BK; r += 4) {
            cp_async16(as + r * BM, Ag + ka + static_cast<long long>(r) * M);
            cp_async16(bs + r * BN, Bg + kb + static_cast<long long>(r) * N);
        }
    };
    unsigned long long acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0ull;
    if constexpr (CH > 0) {
#pragma unroll
        for (int q = 0; q < 32; ++q) Tot[q * NT + t] = make_ulonglong2(0ull, 0ull);
    }
    const int nk = K / BK;
#pragma unroll
    for (int s = 0; s < ST; ++s) {
        if (s < nk) issue(s, s);
        cp_async_commit();
    }
    cp_async_wait<ST - 1>();
    __syncthreads();
    float4 fa[2][2], fb[2][4];
    auto load = [&](int buf, const float* as, const float* bs, int k) {
        fa[buf][0] = *reinterpret_cast<const float4*>(as + k * BM + ty * 4);
        fa[buf][1] = *reinterpret_cast<const float4*>(as + k * BM + 64 + ty * 4);
#pragma unroll
        for (int c = 0; c < 4; ++c) fb[buf][c] = *reinterpret_cast<const float4*>(bs + k * BN + c * 32 + tx * 4);
    };
    auto compute = [&](int cur) {
        const float a[8] = {fa[cur][0].x, fa[cur][0].y, fa[cur][0].z, fa[cur][0].w,
                            fa[cur][1].x, fa[cur][1].y, fa[cur][1].z, fa[cur][1].w};
        unsigned long long b[8];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            b[2 * c] = pack2(fb[cur][c].x, fb[cur][c].y);
            b[2 * c + 1] = pack2(fb[cur][c].z, fb[cur][c].w);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int i = 0; i < 8; ++i) ffma2(acc[i][j], pack2(a[i], a[i]), b[j]);
    };
    load(0, As, Bs, 0);
    for (int kt = 0; kt < nk; ++kt) {
        const int st = kt % ST;
        const float* as = As + st * BK * BM;
        const float* bs = Bs + st * BK * BN;
#pragma unroll
        for (int k = 0; k < BK - 1; ++k) {
            load((k + 1) & 1, as, bs, k + 1);
            compute(k & 1);
        }
        if (kt + 1 < nk) {
            cp_async_wait<ST - 2>();
            __syncthreads();                          // tile kt+1 visible; stage st no longer read
            if (kt + ST < nk) issue(kt + ST, st);
            cp_async_commit();
            const int nst = (kt + 1) % ST;
            load(0, As + nst * BK * BM, Bs + nst * BK * BN, 0);
        }
        compute((BK - 1) & 1);
        if constexpr (CH > 0) {
            if ((kt + 1) % CH == 0 || kt + 1 == nk) {
                const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(Tot + t));
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        asm volatile(
                            "{\n\t.reg .b64 t0, t1, t2, t3;\n\t"
                            "ld.shared.v2.b64 {t0, t1}, [%4];\n\t"
                            "ld.shared.v2.b64 {t2, t3}, [%4+2048];\n\t"
                            "add.rn.f32x2 t0, t0, %0;\n\tadd.rn.f32x2 t1, t1, %1;\n\t"
                            "add.rn.f32x2 t2, t2, %2;\n\tadd.rn.f32x2 t3, t3, %3;\n\t"
                            "st.shared.v2.b64 [%4], {t0, t1};\n\t"
                            "st.shared.v2.b64 [%4+2048], {t2, t3};\n\t"
                            "mov.b64 %0, 0;\n\tmov.b64 %1, 0;\n\tmov.b64 %2, 0;\n\tmov.b64 %3, 0;\n\t}"
                            : "+l"(acc[i][4 * h]), "+l"(acc[i][4 * h + 1]), "+l"(acc[i][4 * h + 2]),
                              "+l"(acc[i][4 * h + 3])
                            : "r"(base + static_cast<uint32_t>((4 * i + 2 * h) * NT * 16))
                            : "memory");
            }
        }
    }
    cp_async_wait<0>();
    if constexpr (CH > 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const ulonglong2 v = Tot[(4 * i + q) * NT + t];
                acc[i][2 * q] = v.x;
                acc[i][2 * q + 1] = v.y;
            }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        float* crow = C + static_cast<long long>(row) * N + n0 + tx * 4;
#pragma unroll
        for (int c = 0; c < 4; ++c)
            *reinterpret_cast<ulonglong2*>(crow + c * 32) = make_ulonglong2(acc[i][2 * c], acc[i][2 * c + 1]);
    }
}

// Rolling B fragments: one buffer of 4 float4 (16 registers instead of 32);
// chunk c of step k+1 is loaded right after its last use in step k, 48
// FFMA2 ahead of its next use.  A stays double-buffered.  8x16, j-outer,
// blocked accumulation as the product.
template <int CH>
__global__ void __launch_bounds__(128, 2)
sgemm_roll(const float* __restrict__ At, const float* __restrict__ B, float* __restrict__ C, int M, int N, int K) {
    constexpr int BM = 128, BN = 128, BK = 16, NT = 128, ST = 3;
    extern __shared__ __align__(16) float sm[];
    float* As = sm;
    float* Bs = sm + ST * BK * BM;
    ulonglong2* Tot = reinterpret_cast<ulonglong2*>(Bs + ST * BK * BN);
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int ty = warp * 4 + (lane >> 3);
    const int tx = lane & 7;
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
        for (int r = 0; r < BK; r += 4) {
            cp_async16(as + r * BM, Ag + ka + static_cast<long long>(r) * M);
            cp_async16(bs + r * BN, Bg + kb + static_cast<long long>(r) * N);
        }
    };
    unsigned long long acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0ull;
    if constexpr (CH > 0) {
#pragma unroll
        for (int q = 0; q < 32; ++q) Tot[q * NT + t] = make_ulonglong2(0ull, 0ull);
    }
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
        float4 fa[2][2], fb[4];
        fa[0][0] = *reinterpret_cast<const float4*>(as + ty * 4);
        fa[0][1] = *reinterpret_cast<const float4*>(as + 64 + ty * 4);
#pragma unroll
        for (int c = 0; c < 4; ++c) fb[c] = *reinterpret_cast<const float4*>(bs + c * 32 + tx * 4);
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            const int cur = k & 1, nxt = cur ^ 1;
            if (k + 1 < BK) {
                fa[nxt][0] = *reinterpret_cast<const float4*>(as + (k + 1) * BM + ty * 4);
                fa[nxt][1] = *reinterpret_cast<const float4*>(as + (k + 1) * BM + 64 + ty * 4);
            }
            const float a[8] = {fa[cur][0].x, fa[cur][0].y, fa[cur][0].z, fa[cur][0].w,
                                fa[cur][1].x, fa[cur][1].y, fa[cur][1].z, fa[cur][1].w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const unsigned long long b0 = pack2(fb[c].x, fb[c].y), b1 = pack2(fb[c].z, fb[c].w);
#pragma unroll
                for (int i = 0; i < 8; ++i) ffma2(acc[i][2 * c], pack2(a[i], a[i]), b0);
#pragma unroll
                for (int i = 0; i < 8; ++i) ffma2(acc[i][2 * c + 1], pack2(a[i], a[i]), b1);
                if (k + 1 < BK) fb[c] = *reinterpret_cast<const float4*>(bs + (k + 1) * BN + c * 32 + tx * 4);
            }
        }
        if constexpr (CH > 0) {
            if ((kt + 1) % CH == 0 || kt + 1 == nk) {
                const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(Tot + t));
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        asm volatile(
                            "{\n\t.reg .b64 t0, t1, t2, t3;\n\t"
                            "ld.shared.v2.b64 {t0, t1}, [%4];\n\t"
                            "ld.shared.v2.b64 {t2, t3}, [%4+2048];\n\t"
                            "add.rn.f32x2 t0, t0, %0;\n\tadd.rn.f32x2 t1, t1, %1;\n\t"
                            "add.rn.f32x2 t2, t2, %2;\n\tadd.rn.f32x2 t3, t3, %3;\n\t"
                            "st.shared.v2.b64 [%4], {t0, t1};\n\t"
                            "st.shared.v2.b64 [%4+2048], {t2, t3};\n\t"
                            "mov.b64 %0, 0;\n\tmov.b64 %1, 0;\n\tmov.b64 %2, 0;\n\tmov.b64 %3, 0;\n\t}"
                            : "+l"(acc[i][4 * h]), "+l"(acc[i][4 * h + 1]), "+l"(acc[i][4 * h + 2]),
                              "+l"(acc[i][4 * h + 3])
                            : "r"(base + static_cast<uint32_t>((4 * i + 2 * h) * NT * 16))
                            : "memory");
            }
        }
    }
    cp_async_wait<0>();
    if constexpr (CH > 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const ulonglong2 v = Tot[(4 * i + q) * NT + t];
                acc[i][2 * q] = v.x;
                acc[i][2 * q + 1] = v.y;
            }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        float* crow = C + static_cast<long long>(row) * N + n0 + tx * 4;
#pragma unroll
        for (int c = 0; c < 4; ++c)
            *reinterpret_cast<ulonglong2*>(crow + c * 32) = make_ulonglong2(acc[i][2 * c], acc[i][2 * c + 1]);
    }
}

__global__ void transpose(const float* __restrict__ A, float* __restrict__ At, int n) {
    __shared__ float tile[32][33];
    const int m0 = blockIdx.y * 32, k0 = blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int r = ty; r < 32; r += 8) tile[r][tx] = A[static_cast<long long>(m0 + r) * n + k0 + tx];
    __syncthreads();
    for (int r = ty; r < 32; r += 8) At[static_cast<long long>(k0 + r) * n + m0 + tx] = tile[tx][r];
}

template <typename Kern>
static void run(const char* name, Kern k, int threads, int smem, const float* At, const float* B, float* C,
                const float* Cref, int n, size_t bytes) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const int tiles = (n / 128) * (n / 128);
    for (int i = 0; i < 3; ++i) k<<<tiles, threads, smem>>>(At, B, C, n, n, n);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9, sum = 0;
    for (int i = 0; i < 20; ++i) {
        cudaEventRecord(e0);
        k<<<tiles, threads, smem>>>(At, B, C, n, n, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
        sum += ms;
    }
    const char* same = "null";
    if (Cref) {
        std::vector<float> h(bytes / 4), r(bytes / 4);
        cudaMemcpy(h.data(), C, bytes, cudaMemcpyDeviceToHost);
        cudaMemcpy(r.data(), Cref, bytes, cudaMemcpyDeviceToHost);
        same = memcmp(h.data(), r.data(), bytes) == 0 ? "true" : "false";
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, smem);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k);
    double fl = 2.0 * n * n * (double)n;
    printf("{\"variant\": \"%s\", \"regs\": %d, \"occ\": %d, \"smem\": %d, \"ms_min\": %.4f, \"ms_mean\": %.4f, "
           "\"tflops\": %.2f, \"bit_identical\": %s, \"err\": \"%s\"}\n",
           name, fa.numRegs, occ, smem, best, sum / 20, fl / (best * 1e-3) / 1e12, same,
           cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
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
    float *A, *At, *B, *C, *C0, *C1, *C2;
    cudaMalloc(&A, bytes); cudaMalloc(&At, bytes); cudaMalloc(&B, bytes); cudaMalloc(&C, bytes);
    cudaMalloc(&C0, bytes); cudaMalloc(&C1, bytes); cudaMalloc(&C2, bytes);
    init<<<1184, 256>>>(A, (size_t)n * n, 1);
    init<<<1184, 256>>>(B, (size_t)n * n, 2);
    transpose<<<dim3(n / 32, n / 32), 256>>>(A, At, n);
    const int ring3 = 3 * 16 * 256 * 4;
    const int tot = 32 * 128 * 16;
    if (argc > 2) {   // quick mode: the product's layout only (A/B of compiler flags)
        run("8x16 blocked32 j-outer", sgemm_8x16<16, 3, 32, 1>, 128, ring3 + tot, At, B, C1, nullptr, n, bytes);
        run("8x16 chain j-outer", sgemm_8x16<16, 3, 0, 1>, 128, ring3, At, B, C, nullptr, n, bytes);
        run("rolling-B blocked32", sgemm_roll<32>, 128, ring3 + tot, At, B, C, C1, n, bytes);
        run("rolling-B chain", sgemm_roll<0>, 128, ring3, At, B, C, nullptr, n, bytes);
        run("8x16 blocked32 j-outer s2", sgemm_8x16<16, 2, 32, 1>, 128, 2 * 16 * 256 * 4 + tot, At, B, C, C1, n,
            bytes);
        run("8x16 blocked16 j-outer", sgemm_8x16<16, 3, 16, 1>, 128, ring3 + tot, At, B, C, nullptr, n, bytes);
        run("8x16 blocked32 j-outer k8s4", sgemm_8x16<8, 4, 64, 1>, 128, 4 * 8 * 256 * 4 + tot, At, B, C, C1, n,
            bytes);
        return 0;
    }
    run("product chain 8x8 k16s3", sgemm_v<16, 3>, 256, ring3, At, B, C0, nullptr, n, bytes);
    run("8x16 chain j-outer", sgemm_8x16<16, 3, 0, 1>, 128, ring3, At, B, C, C0, n, bytes);
    run("early chain s2", sgemm_early<0, 2>, 128, 2 * 16 * 256 * 4, At, B, C, C0, n, bytes);
    run("early chain s3", sgemm_early<0, 3>, 128, ring3, At, B, C, C0, n, bytes);
    run("8x16 blocked32 j-outer", sgemm_8x16<16, 3, 32, 1>, 128, ring3 + tot, At, B, C1, nullptr, n, bytes);
    run("early blocked32 s2", sgemm_early<32, 2>, 128, 2 * 16 * 256 * 4 + tot, At, B, C, C1, n, bytes);
    run("early blocked32 s3", sgemm_early<32, 3>, 128, ring3 + tot, At, B, C, C1, n, bytes);
    run("8x16 blocked32 j-outer (again)", sgemm_8x16<16, 3, 32, 1>, 128, ring3 + tot, At, B, C, C1, n, bytes);
    run("early blocked32 s3 (again)", sgemm_early<32, 3>, 128, ring3 + tot, At, B, C, C1, n, bytes);
    // the product kernel shape with blocked accumulation: 8x8, 256 threads (csrc/gemm_simt.cu)
    {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        float best = 1e9;
        for (int i = 0; i < 23; ++i) {
            cudaEventRecord(e0);
            transpose<<<dim3(n / 32, n / 32), 256>>>(A, At, n);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (i >= 3) best = ms < best ? ms : best;
        }
        printf("{\"variant\": \"A^T pre-pass alone\", \"ms_min\": %.4f}\n", best);
    }
    return 0;
}
