// hf_gemm_simt: register-tiled FP32 FFMA matmul, C = A·B, row-major (sm_100a).
//
// The SIMT half of the diverse kernel pair that stands in for the paper's
// OpenMP/CUDA variants (§IV-D; attached through the kernel-variant
// slot of /root/reference/pkg/src/hetrt/api.py:131-138).  It never touches the
// tensor cores, accumulates every output in fp32 in ascending k order with
// fused multiply-add (in chunks of 512 products summed blockwise, see
// sgemm_128x128), and so fails independently of the tcgen05 variant.
//
// Fast path (M%128 == N%128 == 0, K%32 == 0, 16B-aligned): A is transposed
// once by a tiled pre-pass (~2|A| bytes, ~1% of the GEMM) so both operands
// stream as contiguous k-rows; 128x128x16 CTA tile, 128 threads, 8x16
// outputs per thread, cp.async 3-stage smem ring, one barrier per k-tile,
// register double-buffered fragments, two CTAs per SM; the outer product
// issues packed FFMA2 (fma.rn.f32x2): every output is still an fp32 FMA
// chain in ascending k, so results equal the FFMA formulation bit for bit.
// Generic path: 16x16 bounds-checked tiles for ragged shapes.
#include "common.cuh"

#include <stdlib.h>

namespace hf {

constexpr int SB_M = 128, SB_N = 128, SB_K = 16, S_STAGES = 3;

// Packed fp32x2 FMA (sm_100 FFMA2): two independent IEEE fp32 fused
// multiply-adds with round-to-nearest per instruction — bit-identical to two
// FFMAs, half the issue slots and register-port pressure.
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void ffma2(unsigned long long& d, unsigned long long a, unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 128x128x16 CTA tile, 128 threads, 8 (m) x 16 (n) outputs per thread (r2;
// round 1: 256 threads x 8x8).  Operands are A^T (K x M, from the transpose
// pre-pass) and B (K x N): both k-tiles are 16 rows of 512 contiguous bytes,
// streamed by cp.async into a 3-stage smem ring without staging registers;
// fragments for k+1 are read from smem while k is multiplied.  Per k-step a
// thread reads 2 LDS.128 of A and 4 of B for 64 FFMA2 (8x8/256 threads: 4
// for 32) and issues them column-pair-outer: each b pair is reused by 8
// consecutive FFMA2.  ~254 registers, two CTAs (8 warps) per SM.  Warp =
// 4 (m) x 8 (n) lanes, the 4 warps stacked along m; thread rows ty*4 + {0..3}
// and 64 + ty*4 + {0..3} (ty = warp*4 + lane/8), columns c*32 + tx*4 + {0..3}
// for c = 0..3 (tx = lane%8): every LDS.128 of a warp touches 4 (A) or 8 (B)
// distinct 16-byte words, one wavefront each.  Measured against the 8x8
// layout at 4096^3 (tools/simt_lab2.cu, profiles/r02_simt_lab2b.jsonl):
// blocked accumulation 2.175 ms (the 8x8 kernel's single chain: 2.172, its
// blocked form ~2.30); the a-scalar-outer issue order of the same layout
// 2.285.  Results are bit-identical to the 8x8 kernel (same chains, same
// chunk sums).
//
// Blocked accumulation (CH > 0, the default): the fp32 FMA chain of an
// output runs over CH k-tiles (CH*16 products) only; the chunk's sum is then
// added (one rounding) into a running total that lives in shared memory, 128
// floats per thread laid out [32][128] x 16 B (conflict-free 128-bit
// accesses), and the register accumulators restart at zero — the blocked
// summation an optimised CPU sgemm does.  At 4096^2 the max relative error
// against the binary64 product is 7.1e-7 (numpy/OpenBLAS fp32, the
// reference body's arithmetic: 5.5e-7) instead of 5.4e-6 for one 4096-long
// chain, for 64 KB more smem per CTA (112 KB: still two CTAs per SM).
// CH = 0: one chain in ascending k (A/B only).
constexpr int SGEMM_THREADS = 128;
template <int CH>
__global__ void __launch_bounds__(SGEMM_THREADS, 2)
sgemm_128x128(const float* __restrict__ At, const float* __restrict__ B, float* __restrict__ C,
              int M, int N, int K, int group) {
    constexpr int NT = SGEMM_THREADS;
    extern __shared__ __align__(16) float sm[];
    float* As = sm;                                   // [S][SB_K][SB_M]
    float* Bs = sm + S_STAGES * SB_K * SB_M;          // [S][SB_K][SB_N]
    ulonglong2* Tot = reinterpret_cast<ulonglong2*>(Bs + S_STAGES * SB_K * SB_N);   // [32][NT]

    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int ty = warp * 4 + (lane >> 3);   // 0..15
    const int tx = lane & 7;                 // 0..7

    // grouped tile order: consecutive CTAs share B column panels in L2
    const int tiles_n = N / SB_N;
    const int tiles_m = M / SB_M;
    const int bid = blockIdx.x;
    const int per_group = group * tiles_n;
    const int g = bid / per_group;
    const int first_m = g * group;
    const int gm = min(tiles_m - first_m, group);
    const int tm = first_m + (bid % per_group) % gm;
    const int tn = (bid % per_group) / gm;
    const int m0 = tm * SB_M, n0 = tn * SB_N;

    // copy mapping: each of the 16 k-rows is 32 chunks of 16 B per operand;
    // thread t moves chunk (t & 31) of rows (t >> 5) + {0, 4, 8, 12}
    const int c_row = t >> 5, c_col = (t & 31) * 4;
    const float* Ag = At + static_cast<long long>(c_row) * M + m0 + c_col;
    const float* Bg = B + static_cast<long long>(c_row) * N + n0 + c_col;
    const long long a4 = 4LL * M, b4 = 4LL * N;

    auto issue = [&](int kt, int stage) {
        const long long ka = static_cast<long long>(kt) * SB_K * M;
        const long long kb = static_cast<long long>(kt) * SB_K * N;
        float* as = As + stage * SB_K * SB_M + c_row * SB_M + c_col;
        float* bs = Bs + stage * SB_K * SB_N + c_row * SB_N + c_col;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            cp_async16(as + r * 4 * SB_M, Ag + ka + r * a4);
            cp_async16(bs + r * 4 * SB_N, Bg + kb + r * b4);
        }
    };

    // acc[i][j] holds the output pair of row i, columns (j>>1)*32 + tx*4 + 2*(j&1) + {0, 1}
    unsigned long long acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0ull;

    if constexpr (CH > 0) {
#pragma unroll
        for (int q = 0; q < 32; ++q) Tot[q * NT + t] = make_ulonglong2(0ull, 0ull);
    }
    // running total += chunk sum (acc pairs (i, 4h..4h+3) <-> Tot[q = 4i + 2h,
    // 4i + 2h + 1]), then the chain restarts at zero.  Written in asm that
    // updates the accumulators in place, called behind a uniform branch from
    // the single k-tile loop: a C++ restart at zero (or a nested chunk loop)
    // gave every accumulator a second definition, ptxas assigned them
    // different registers and the loop back-edge grew MOVs (round 2 A/B,
    // tools/simt_ab.py, profiles/r02_simt_ab_fv.jsonl).
    const uint32_t tot_s = static_cast<uint32_t>(__cvta_generic_to_shared(Tot + t));
    auto flush = [&]() {
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
                    : "+l"(acc[i][4 * h]), "+l"(acc[i][4 * h + 1]), "+l"(acc[i][4 * h + 2]), "+l"(acc[i][4 * h + 3])
                    : "r"(tot_s + static_cast<uint32_t>((4 * i + 2 * h) * NT * 16))
                    : "memory");
    };
    const int nk = K / SB_K;
    pdl_wait();     // launched with PDL behind the A^T pre-pass: At is complete from here
#pragma unroll
    for (int s = 0; s < S_STAGES - 1; ++s) {
        if (s < nk) issue(s, s);
        cp_async_commit();
    }

    auto ktile = [&](int kt) {
        cp_async_wait<S_STAGES - 2>();
        __syncthreads();
        {
            const int nt = kt + S_STAGES - 1;
            if (nt < nk) issue(nt, nt % S_STAGES);
            cp_async_commit();
        }
        const float* as = As + (kt % S_STAGES) * SB_K * SB_M;
        const float* bs = Bs + (kt % S_STAGES) * SB_K * SB_N;
        float4 fa[2][2], fb[2][4];
        fa[0][0] = *reinterpret_cast<const float4*>(as + ty * 4);
        fa[0][1] = *reinterpret_cast<const float4*>(as + 64 + ty * 4);
#pragma unroll
        for (int c = 0; c < 4; ++c) fb[0][c] = *reinterpret_cast<const float4*>(bs + c * 32 + tx * 4);
#pragma unroll
        for (int k = 0; k < SB_K; ++k) {
            const int cur = k & 1, nxt = cur ^ 1;
            if (k + 1 < SB_K) {
                fa[nxt][0] = *reinterpret_cast<const float4*>(as + (k + 1) * SB_M + ty * 4);
                fa[nxt][1] = *reinterpret_cast<const float4*>(as + (k + 1) * SB_M + 64 + ty * 4);
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    fb[nxt][c] = *reinterpret_cast<const float4*>(bs + (k + 1) * SB_N + c * 32 + tx * 4);
            }
            const float a[8] = {fa[cur][0].x, fa[cur][0].y, fa[cur][0].z, fa[cur][0].w,
                                fa[cur][1].x, fa[cur][1].y, fa[cur][1].z, fa[cur][1].w};
            // b pairs are the LDS.128 destination registers, already adjacent
            unsigned long long b[8];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                b[2 * c] = pack2(fb[cur][c].x, fb[cur][c].y);
                b[2 * c + 1] = pack2(fb[cur][c].z, fb[cur][c].w);
            }
            // column-pair-outer: the b pair stays in the operand reuse cache
            // across 8 FFMA2 (a scalars folded into FFMA2's broadcast operand)
#pragma unroll
            for (int j = 0; j < 8; ++j)
#pragma unroll
                for (int i = 0; i < 8; ++i) ffma2(acc[i][j], pack2(a[i], a[i]), b[j]);
        }
    };
    for (int kt = 0; kt < nk; ++kt) {
        ktile(kt);
        if constexpr (CH > 0) {
            if ((kt + 1) % CH == 0 || kt + 1 == nk) flush();
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

// k-tiles per FMA chain: 32 (512 products).  At 4096^2 (tools/simt_ab.py,
// profiles/r02_simt_ab6.jsonl): max rel err 7.1e-7 (numpy fp32 5.5e-7; one
// 4096-long chain 5.4e-6), 2.346 ms vs 2.220 ms for the chain kernel.  CH 8:
// 4.5e-7 but the flushes' smem traffic adds another 2%; CH 64: 1.3e-6, 2.336 ms.
constexpr int SGEMM_CH = 32;
constexpr int SGEMM_SMEM_RING = S_STAGES * SB_K * (SB_M + SB_N) * 4;   // 48 KB
constexpr int SGEMM_SMEM = SGEMM_SMEM_RING + 32 * SGEMM_THREADS * 16;   // + 64 KB running totals
// Co-scheduled with the tensor-core replica (HF_GEMM_COSCHEDULE): each CTA
// reserves 100 KB although it uses 48 KB.  Two SIMT CTAs still fit an SM,
// and when one retires the space it frees takes one TC CTA (2-stage shape,
// ~98 KB) beside the remaining SIMT CTA, so the tensor-core replica runs on
// the tensor pipe while the FMA pipe keeps working.  Measured on B200 at
// 4096^2, SIMT + TC replicas on two streams: 2.33 ms vs 2.45 ms with the
// 48 KB reservation (tools/cosched_bench.py); at <= 96 KB the TC CTAs are
// not placed until the SIMT grid drains.
// With the 112 KB of the blocked-accumulation kernel the reservation is its
// own footprint: two CTAs use 226 KB of the SM's 228 KB, and one retiring
// frees room for one TC CTA exactly as the 100 KB reservation did.
constexpr int SGEMM_SMEM_COSCHED = SGEMM_SMEM > 100000 ? SGEMM_SMEM : 100000;
constexpr int SGEMM_SMEM_MAX = 227 * 1024;

// A (M x K) -> At (K x M), 32x32 tiles through padded smem.
__global__ void __launch_bounds__(256) transpose_a(const float* __restrict__ A, float* __restrict__ At, int M, int K) {
    __shared__ float tile[32][33];
    pdl_wait();                 // A may come from the previous kernel of the stream
    pdl_launch_dependents();    // the GEMM may launch (and wait) while this pass drains
    const int m0 = blockIdx.y * 32, k0 = blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
    for (int r = ty; r < 32; r += 8) tile[r][tx] = A[static_cast<long long>(m0 + r) * K + k0 + tx];
    __syncthreads();
#pragma unroll
    for (int r = ty; r < 32; r += 8) At[static_cast<long long>(k0 + r) * M + m0 + tx] = tile[tx][r];
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

static const int kRegistered =
    register_kernels({(const void*)sgemm_128x128<SGEMM_CH>, (const void*)sgemm_128x128<0>,
                      (const void*)transpose_a, (const void*)sgemm_generic});

}  // namespace hf

namespace hf {
// Co-scheduling smem reservation per SIMT CTA (HF_SGEMM_COSCHED_SMEM bytes,
// experiments only; default SGEMM_SMEM_COSCHED).
static bool sgemm_chain() {
    static const int on = getenv("HF_SGEMM_CHAIN") != nullptr && getenv("HF_SGEMM_CHAIN")[0] == '1';
    return on != 0;
}

static int sgemm_cosched_smem() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("HF_SGEMM_COSCHED_SMEM");
        int x = e ? atoi(e) : SGEMM_SMEM_COSCHED;
        v = x >= SGEMM_SMEM_RING && x <= SGEMM_SMEM_MAX ? x : SGEMM_SMEM_COSCHED;
        if (v < SGEMM_SMEM && !sgemm_chain()) v = SGEMM_SMEM;
    }
    return v;
}

// Tile-row group of the grouped CTA order (HF_SGEMM_GROUP, default 16: at
// 4096^3 the resident CTAs then share 16 A panels and ~19 B panels in L2;
// DRAM reads 333 MB with 8, 286 MB with 16, 509 MB with 32, same time).
static bool side_prepass() {
    static const int on = getenv("HF_SIMT_SIDE_PREPASS") == nullptr || getenv("HF_SIMT_SIDE_PREPASS")[0] != '0';
    return on != 0;
}

static bool simt_pdl() {
    static const int on = getenv("HF_SIMT_PDL") != nullptr && getenv("HF_SIMT_PDL")[0] == '1';
    return on != 0 && pdl_enabled();
}

static int sgemm_group() {
    static int g = -1;
    if (g < 0) {
        const char* e = getenv("HF_SGEMM_GROUP");
        int v = e ? atoi(e) : 16;
        g = v >= 1 && v <= 64 ? v : 16;
    }
    return g;
}
}  // namespace hf

extern "C" int hf_gemm_simt(const float* A, const float* B, float* C, int M, int N, int K, int mode,
                            int device, void* stream) {
    HF_REQUIRE(A && B && C, "hf_gemm_simt: NULL operand");
    HF_REQUIRE((mode & ~HF_GEMM_COSCHEDULE) == 0, "hf_gemm_simt: unknown mode 0x%x", mode);
    HF_REQUIRE(M > 0 && N > 0 && K > 0, "hf_gemm_simt: bad shape %dx%dx%d", M, N, K);
    hf::DeviceGuard g(device);
    HF_REQUIRE(g.ok, "hf_gemm_simt: cannot select device %d", device);
    cudaStream_t st = hf::as_stream(stream);
    hf::retain_scratch_pool(device);
    bool aligned = (reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) |
                    reinterpret_cast<uintptr_t>(C)) % 16 == 0;
    if (aligned && M % hf::SB_M == 0 && N % hf::SB_N == 0 && K % 32 == 0) {
        static bool attr[64] = {false};
        if (!attr[device]) {
            HF_CUDA_CHECK(cudaFuncSetAttribute(hf::sgemm_128x128<hf::SGEMM_CH>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, hf::SGEMM_SMEM_MAX));
            HF_CUDA_CHECK(cudaFuncSetAttribute(hf::sgemm_128x128<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               hf::SGEMM_SMEM_MAX));
            // the whole unified L1 as shared memory (the ring is filled by
            // cp.async.cg, which bypasses L1): an SM running one SIMT CTA then
            // still has room for a co-scheduled TC CTA beside it
            HF_CUDA_CHECK(cudaFuncSetAttribute(hf::sgemm_128x128<hf::SGEMM_CH>,
                                               cudaFuncAttributePreferredSharedMemoryCarveout,
                                               cudaSharedmemCarveoutMaxShared));
            HF_CUDA_CHECK(cudaFuncSetAttribute(hf::sgemm_128x128<0>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                               cudaSharedmemCarveoutMaxShared));
            attr[device] = true;
        }
        // HF_SGEMM_CHAIN=1 (A/B only): one fp32 chain over all of K, 48 KB
        const bool chain = hf::sgemm_chain();
        auto kern = chain ? hf::sgemm_128x128<0> : hf::sgemm_128x128<hf::SGEMM_CH>;
        float* At = static_cast<float*>(hf::stream_scratch(device, st, 2, static_cast<size_t>(M) * K * sizeof(float)));
        if (!At) {
            hf::set_error("hf_gemm_simt: cannot allocate the A^T scratch");
            return HF_ECUDA;
        }
        // Co-scheduled: the A^T pre-pass runs on the device's greatest-priority
        // side stream, ahead of the tensor-core replica's pre-pass (level 1),
        // so this GEMM's grid is pending before the TC GEMM's and, launched on
        // the executor's higher-priority lead stream, is dispatched first; the
        // TC CTAs then fill its last wave.
        int tiles = (M / hf::SB_M) * (N / hf::SB_N);
        int smem = (mode & HF_GEMM_COSCHEDULE) ? hf::sgemm_cosched_smem() : hf::SGEMM_SMEM;
        if (chain && !(mode & HF_GEMM_COSCHEDULE)) smem = hf::SGEMM_SMEM_RING;
        if (hf::simt_pdl()) {
            // HF_SIMT_PDL=1: A^T pre-pass and GEMM on the caller's stream, the
            // GEMM launched with PDL (no launch gap after the pre-pass).  Off
            // by default: co-scheduled with a TC replica the TC GEMM then got
            // SMs at the start of the SIMT grid, 2.46 -> 2.49 ms per DMR round
            HF_CUDA_CHECK(hf::launch_pdl(hf::transpose_a, dim3(K / 32, M / 32), dim3(256), 0, st, A, At, M, K));
            HF_CUDA_CHECK(hf::launch_pdl(kern, dim3(tiles), dim3(hf::SGEMM_THREADS), smem, st, At, B, C, M, N, K,
                                         hf::sgemm_group()));
        } else if (hf::side_prepass()) {
            // default: the pre-pass on the device's greatest-priority side
            // stream, joined back by an event (~20 us of launch gap before
            // the GEMM, but the A^T pass reliably finishes before the TC
            // replica's pre-pass, so the SIMT grid is pending first)
            hf::SideStream* side = (mode & HF_GEMM_COSCHEDULE) ? hf::side_stream(device, 0) : nullptr;
            cudaStream_t ps = st;
            // (r2: the GEMM on the side stream right behind the pre-pass, plain
            // or PDL, removes the event gap but lost 1.6% per HetTMR task and
            // 0-1.6% per HetDMR task: 345 vs 350.5 tasks/s, tools/tmr_order_ab.py)
            HF_CUDA_CHECK(hf::begin_side_launch(side, st, &ps));
            hf::transpose_a<<<dim3(K / 32, M / 32), 256, 0, ps>>>(A, At, M, K);
            HF_CUDA_CHECK(hf::end_side_launch(side, st));
            kern<<<tiles, hf::SGEMM_THREADS, smem, st>>>(At, B, C, M, N, K, hf::sgemm_group());
        } else {
            // HF_SIMT_SIDE_PREPASS=0: pre-pass and GEMM in stream order on the
            // caller's stream (no event gap).  Co-scheduled, the TC pre-pass
            // then often finished first and its GEMM took the SMs ahead of
            // the SIMT grid, even with the lead stream at the greatest priority
            // (2.44 -> 2.57 ms per DMR round)
            hf::transpose_a<<<dim3(K / 32, M / 32), 256, 0, st>>>(A, At, M, K);
            kern<<<tiles, hf::SGEMM_THREADS, smem, st>>>(At, B, C, M, N, K, hf::sgemm_group());
        }
    } else {
        dim3 grid((N + 15) / 16, (M + 15) / 16);
        hf::sgemm_generic<<<grid, 256, 0, st>>>(A, B, C, M, N, K);
    }
    HF_CHECK_LAUNCH();
    return HF_OK;
}
