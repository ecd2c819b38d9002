// hf_gemm_tc: tensor-core fp32 matmul via tcgen05.mma kind::tf32 (sm_100a).
//
// The tensor-core half of the diverse kernel pair (§IV-D; attached
// through the kernel-variant slot of /root/reference/pkg/src/hetrt/api.py:131-138).
// C = A·B, row-major fp32.  Both UMMA operands are K-major.  The operands are
// RN-rounded to tf32 first (truncation would bias the sum), and B's rounding
// pass also transposes it to B^T (N x K): ~2·|B| bytes of HBM traffic either
// way, the same as rounding B in place.  (An MN-major tf32 B would need the
// 32-byte-atom 128B swizzle, descriptor layout type 1: tools/tc_probe.cu v12.)
// A gets the same RN rounding in a vectorised pass; 3xTF32 / 3xBF16 modes do
// the hi/lo splits in the same passes.
//
// Structure (persistent, warp-specialised, one CTA per SM):
//   warp 0      TMA producer: A box {32k x 128m} + B^T box {32k x 256n} per
//               k-block into a 4-stage ring of 128B-swizzled smem (48 KB/stage)
//   warp 1      MMA issuer: one thread issues 4 x tcgen05.mma (M=128, N=256,
//               K=8) per k-block into a TMEM accumulator; tcgen05.commit frees
//               the smem stage and, after the last k-block, signals the epilogue
//   warp 2      TMEM allocator (2 x 256 columns: double-buffered accumulators)
//   warps 4..7  epilogue: tcgen05.ld 32x32b.x32 -> registers -> global,
//               overlapping the next tile's main loop
// Ragged M/N/K are handled by TMA out-of-bounds zero fill plus masked stores.
// Mode HF_GEMM_3XTF32 splits each operand into tf32 big + small parts in the
// pre-pass and runs the same kernel over K' = 3K:
//   [A_hi | A_hi | A_lo] x [B_hi ; B_lo ; B_hi]  ~= fp32-accurate product.
#include "common.cuh"

#include <cuda.h>
#include <cuda_bf16.h>
#include <mutex>
#include <stdlib.h>

namespace hf {
namespace tc {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 32;          // one 128-byte swizzle row of fp32
constexpr int A_STAGE = BM * BK * 4;   // 16 KB
constexpr int NUM_THREADS = 256;
template <int S, int BNT = BN>
constexpr int smem_bytes() { return S * (A_STAGE + BNT * BK * 4) + 1024 /*align*/ + 256 /*barriers*/; }

// ---- PTX wrappers ----------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tc_mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Operand kind of a GEMM launch: tf32 (32-bit elements, UMMA K = 8) or bf16
// (16-bit elements, UMMA K = 16, kind::f16 at twice the tf32 rate).  Either
// way one 128-byte swizzle row holds BK_BYTES of K, a stage is the same
// number of bytes, and each UMMA advances the descriptor by 32 bytes.
template <bool BF16>
struct OpKind {
    static constexpr int ELEM = BF16 ? 2 : 4;
    static constexpr int BKE = 128 / ELEM;          // K elements per stage (one swizzle row)
    static constexpr uint32_t FMT = BF16 ? 1u : 2u;  // instruction-descriptor A/B format code
};

template <bool BF16>
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
    if constexpr (BF16)
        tc_mma_bf16(d_tmem, a_desc, b_desc, idesc, accumulate);
    else
        tc_mma_tf32(d_tmem, a_desc, b_desc, idesc, accumulate);
}

// tcgen05.ld 32 lanes x 32 bits, 32 consecutive columns per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor (SM100 "version 1" layout):
//   [0,14) start>>4  [16,30) LBO>>4  [32,46) SBO>>4  [46,48) version=1
//   [49,52) base offset  [52] LBO mode  [61,64) layout (2 = SWIZZLE_128B)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}

// Instruction descriptor, kind::tf32 (fmt 2) or kind::f16 with bf16 (fmt 1),
// fp32 accumulate, A and B K-major.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, uint32_t fmt = 2u) {
    return (1u << 4)            // D format f32
           | (fmt << 7)         // A format
           | (fmt << 10)        // B format
           | (0u << 15)         // A K-major
           | (0u << 16)         // B K-major (B^T staged by the pre-pass)
           | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

template <int STAGES>
struct Barriers {
    uint64_t full[STAGES];
    uint64_t empty[STAGES];
    uint64_t tmem_full[2];
    uint64_t tmem_empty[2];
    uint32_t tmem_base;
};

// STAGES smem ring stages; ACCS TMEM accumulators (2: persistent kernel that
// overlaps a tile's epilogue with the next tile's main loop; 1: one tile per
// CTA, 2 CTAs/SM co-resident, used when the kernel shares the GPU with the
// SIMT replica so its CTAs fill the SIMT kernel's last wave).
template <int STAGES, int ACCS, bool BF16 = false, int BNT = BN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_tf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, float* __restrict__ C,
                 int M, int N, int K) {
    using OK = OpKind<BF16>;
    constexpr int SB = A_STAGE + BNT * BK * 4;      // bytes per stage (B tile BNT rows of 128 B)
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the SWIZZLE_128B atoms
    const uint32_t base_u32 = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (base_u32 & 1023)) & 1023);
    constexpr int TMEM_COLS = ACCS * BNT;
    Barriers<STAGES>* bars = reinterpret_cast<Barriers<STAGES>*>(smem + STAGES * SB);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int tiles_m = (M + BM - 1) / BM;
    const int tiles_n = (N + BNT - 1) / BNT;
    const int num_tiles = tiles_m * tiles_n;
    const int nkb = (K + OK::BKE - 1) / OK::BKE;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int a = 0; a < ACCS; ++a) {
            mbar_init(&bars->tmem_full[a], 1);
            mbar_init(&bars->tmem_empty[a], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&bars->tmem_base)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp == 0) {
        // ===== TMA producer =====
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int tm = tile % tiles_m, tn = tile / tiles_m;
                const int m0 = tm * BM, n0 = tn * BNT;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&bars->empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * SB;
                    uint8_t* sb = sa + A_STAGE;
                    mbar_expect_tx(&bars->full[stage], SB);
                    tma_load_2d(sa, &tmA, &bars->full[stage], kb * OK::BKE, m0);
                    tma_load_2d(sb, &tmB, &bars->full[stage], kb * OK::BKE, n0);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        if (lane == 0) {
            constexpr uint32_t idesc = make_idesc(BM, BNT, OK::FMT);
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
                const int acc = local % ACCS;
                const uint32_t acc_phase = (local / ACCS) & 1;
                mbar_wait(&bars->tmem_empty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem + acc * BNT;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&bars->full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + stage * SB);
                    const uint32_t sb = sa + A_STAGE;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {   // 4 UMMAs of 32 bytes of K per 128-byte row
                        // K-major SW128: advance 32 B along the swizzled 128 B row;
                        // SBO = 1 KB between 8-row groups (LBO unused when swizzled)
                        uint64_t adesc = make_desc(sa + kk * 32, 16, 1024);
                        uint64_t bdesc = make_desc(sb + kk * 32, 16, 1024);
                        tc_mma<BF16>(d_tmem, adesc, bdesc, idesc, (kb | kk) != 0);
                    }
                    tc_commit(&bars->empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc_commit(&bars->tmem_full[acc]);
            }
        }
    } else if (warp >= 4) {
        // ===== epilogue: TMEM -> registers -> global =====
        const int ew = warp - 4;                 // TMEM lane quarter
        const int row_in_tile = ew * 32 + lane;
        int local = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
            const int tm = tile % tiles_m, tn = tile / tiles_m;
            const int m0 = tm * BM, n0 = tn * BNT;
            const int acc = local % ACCS;
            mbar_wait(&bars->tmem_full[acc], (local / ACCS) & 1);
            tc_fence_after();
            const int row = m0 + row_in_tile;
            const uint32_t tbase = tmem + (static_cast<uint32_t>(ew * 32) << 16) + acc * BNT;
            float* crow = C + static_cast<long long>(row) * N;
#pragma unroll 1
            for (int c = 0; c < BNT / 32; ++c) {
                float v[32];
                tmem_ld32(tbase + c * 32, v);
                const int col0 = n0 + c * 32;
                if (row < M) {
                    if (col0 + 32 <= N && (N & 3) == 0) {
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            *reinterpret_cast<float4*>(crow + col0 + 4 * q) =
                                make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    } else {
                        for (int q = 0; q < 32; ++q)
                            if (col0 + q < N) crow[col0 + q] = v[q];
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->tmem_empty[acc]);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// ---- CTA-pair variant (cta_group::2) ---------------------------------------
// A cluster of two CTAs on one TPC computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M = 256): CTA rank r stages rows [128r, 128r+128)
// of the A tile and rows [128r, 128r+128) of the B^T tile, the tensor cores of
// the pair read both halves, and each CTA's TMEM accumulates its 128 rows x
// 256 columns.  Per 256 x 256 x 32 k-block the pair moves 64 KB through L2
// instead of the 96 KB two single-CTA 128 x 256 tiles need, and each SM's
// shared memory takes 32 KB of TMA writes instead of 48 KB.
//   leader (rank 0): warp 0 TMA (its halves; arms the stage's full barrier
//                    with both CTAs' bytes), warp 1 MMA issue, warp 2 TMEM
//   peer   (rank 1): warp 0 TMA (its halves, completing on the leader's
//                    barrier), warp 2 TMEM
//   both: warps 4..7 epilogue of their own 128 rows; commits multicast to
//         both CTAs' barriers; the leader's tmem_empty counts 8 warps.
constexpr int PBM = 256;            // pair tile rows (128 per CTA)
constexpr int PBN = 256;            // pair tile cols (B^T rows, 128 per CTA)
constexpr int P_STAGE = (PBM / 2) * BK * 4 + (PBN / 2) * BK * 4;   // 32 KB per CTA
template <int S>
constexpr int pair_smem_bytes() { return S * P_STAGE + 1024 + 256; }

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                 int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tc_mma_tf32_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

template <bool BF16>
__device__ __forceinline__ void tc_mma_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    if constexpr (BF16)
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
            "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
            : "memory");
    else
        tc_mma_tf32_pair(d_tmem, a_desc, b_desc, idesc, accumulate);
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

// Tail split (stream-K style, deterministic): of T pair tiles over P pairs,
// the last R = T mod P tiles are cut into `splits` k-ranges so the final
// round keeps R*splits <= P pairs busy instead of R.  Split j < splits-1
// stores its 128 x 256 partial per CTA into `partial` and raises its flag;
// the last split waits for the flags and writes C = ((P0 + P1) + ...) + own,
// a fixed summation order, so results are run-to-run identical.
struct PairSplit {
    int full_tiles;      // T - R tiles computed whole
    int splits;          // k-ranges per tail tile (1: no split)
    float* partial;      // R * (splits-1) slots of 256 x 256 floats
    int* flags;          // R * (splits-1) * 2 (per CTA rank), zeroed per launch
};

__device__ __forceinline__ void store_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int load_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int STAGES, bool BF16 = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
gemm_tf32_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      float* __restrict__ C, int M, int N, int K, PairSplit sp) {
    using OK = OpKind<BF16>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base_u32 = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (base_u32 & 1023)) & 1023);
    constexpr int ACCS = 2;
    constexpr int TMEM_COLS = ACCS * PBN;
    constexpr int A_HALF = (PBM / 2) * BK * 4;   // 16 KB
    Barriers<STAGES>* bars = reinterpret_cast<Barriers<STAGES>*>(smem + STAGES * P_STAGE);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int pair = blockIdx.x >> 1;
    const int npairs = gridDim.x >> 1;
    const int tiles_m = (M + PBM - 1) / PBM;
    const int tiles_n = (N + PBN - 1) / PBN;
    const int num_tiles = tiles_m * tiles_n;
    const int nkb = (K + OK::BKE - 1) / OK::BKE;
    const int tail = num_tiles - sp.full_tiles;
    const int num_units = sp.full_tiles + tail * sp.splits;
    // unit -> (tile, k-block range, split index)
    auto unit_of = [&](int u, int& tile, int& kb0, int& kb1, int& split) {
        if (u < sp.full_tiles) {
            tile = u, kb0 = 0, kb1 = nkb, split = -1;
        } else {
            const int v = u - sp.full_tiles;
            tile = sp.full_tiles + v / sp.splits;
            split = v % sp.splits;
            kb0 = static_cast<int>(static_cast<long long>(nkb) * split / sp.splits);
            kb1 = static_cast<int>(static_cast<long long>(nkb) * (split + 1) / sp.splits);
        }
    };

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int a = 0; a < ACCS; ++a) {
            mbar_init(&bars->tmem_full[a], 1);
            mbar_init(&bars->tmem_empty[a], 8);     // 4 epilogue warps x 2 CTAs (leader's copy is used)
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&bars->tmem_base)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();      // both CTAs' barriers initialised and TMEM allocated
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp == 0) {
        // ===== TMA producer (both CTAs): this CTA's A and B^T halves =====
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int u = pair; u < num_units; u += npairs) {
                int tile, kb0, kb1, split;
                unit_of(u, tile, kb0, kb1, split);
                const int tm = tile % tiles_m, tn = tile / tiles_m;
                const int m0 = tm * PBM + static_cast<int>(rank) * (PBM / 2);
                const int n0 = tn * PBN + static_cast<int>(rank) * (PBN / 2);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&bars->empty[stage], phase ^ 1);
                    const uint32_t sa = smem_u32(smem + stage * P_STAGE);
                    const uint32_t sb = sa + A_HALF;
                    const uint32_t full_leader = map_rank(smem_u32(&bars->full[stage]), 0);
                    if (rank == 0) mbar_expect_tx(&bars->full[stage], 2 * P_STAGE);
                    tma_load_2d_pair(sa, &tmA, full_leader, kb * OK::BKE, m0);
                    tma_load_2d_pair(sb, &tmB, full_leader, kb * OK::BKE, n0);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (leader only) =====
        if (rank == 0 && lane == 0) {
            constexpr uint32_t idesc = make_idesc(PBM, PBN, OK::FMT);
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int u = pair; u < num_units; u += npairs, ++local) {
                int tile, kb0, kb1, split;
                unit_of(u, tile, kb0, kb1, split);
                const int acc = local % ACCS;
                const uint32_t acc_phase = (local / ACCS) & 1;
                mbar_wait(&bars->tmem_empty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem + acc * PBN;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&bars->full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + stage * P_STAGE);
                    const uint32_t sb = sa + A_HALF;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        uint64_t adesc = make_desc(sa + kk * 32, 16, 1024);
                        uint64_t bdesc = make_desc(sb + kk * 32, 16, 1024);
                        tc_mma_pair<BF16>(d_tmem, adesc, bdesc, idesc, (kb != kb0) | kk);
                    }
                    tc_commit_pair(&bars->empty[stage]);      // frees the stage in both CTAs
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc_commit_pair(&bars->tmem_full[acc]);        // both CTAs' epilogues
            }
        }
    } else if (warp >= 4) {
        // ===== epilogue (both CTAs): own 128 rows x 256 cols =====
        const int ew = warp - 4;
        const int row_in_tile = static_cast<int>(rank) * (PBM / 2) + ew * 32 + lane;
        const uint32_t empty_leader_base = map_rank(smem_u32(&bars->tmem_empty[0]), 0);
        const int etid = threadIdx.x - 128;          // 0..127 over the 4 epilogue warps
        int local = 0;
        for (int u = pair; u < num_units; u += npairs, ++local) {
            int tile, kb0, kb1, split;
            unit_of(u, tile, kb0, kb1, split);
            const int tm = tile % tiles_m, tn = tile / tiles_m;
            const int m0 = tm * PBM, n0 = tn * PBN;
            const int acc = local % ACCS;
            mbar_wait(&bars->tmem_full[acc], (local / ACCS) & 1);
            tc_fence_after();
            const int row = m0 + row_in_tile;
            const uint32_t tbase = tmem + (static_cast<uint32_t>(ew * 32) << 16) + acc * PBN;
            float* crow = C + static_cast<long long>(row) * N;
            // tail-split bookkeeping: this CTA's 128 x 256 slot of tail tile t
            const int t = tile - sp.full_tiles;
            const bool partial_out = split >= 0 && split < sp.splits - 1;
            const bool fixup = split == sp.splits - 1 && sp.splits > 1;
            auto slot = [&](int j) {
                return sp.partial + ((static_cast<long long>(t) * (sp.splits - 1) + j) * PBM +
                                     static_cast<int>(rank) * (PBM / 2) + ew * 32 + lane) * PBN;
            };
            auto flag = [&](int j) { return sp.flags + (t * (sp.splits - 1) + j) * 2 + static_cast<int>(rank); };
            if (fixup) {      // earlier k-ranges of this tile must have landed
                if (etid == 0)
                    for (int j = 0; j < sp.splits - 1; ++j)
                        while (load_acquire_gpu(flag(j)) == 0) __nanosleep(64);
                asm volatile("bar.sync 1, 128;" ::: "memory");
            }
#pragma unroll 1
            for (int c = 0; c < PBN / 32; ++c) {
                float v[32];
                tmem_ld32(tbase + c * 32, v);
                const int col0 = n0 + c * 32;
                if (partial_out) {
                    float4* dst = reinterpret_cast<float4*>(slot(split) + c * 32);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        __stcg(dst + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
                    continue;
                }
                if (fixup) {
                    float w[32];
                    const float4* src0 = reinterpret_cast<const float4*>(slot(0) + c * 32);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float4 x = __ldcg(src0 + q);
                        w[4 * q] = x.x, w[4 * q + 1] = x.y, w[4 * q + 2] = x.z, w[4 * q + 3] = x.w;
                    }
                    for (int j = 1; j < sp.splits - 1; ++j) {
                        const float4* srcj = reinterpret_cast<const float4*>(slot(j) + c * 32);
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float4 x = __ldcg(srcj + q);
                            w[4 * q] += x.x, w[4 * q + 1] += x.y, w[4 * q + 2] += x.z, w[4 * q + 3] += x.w;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 32; ++q) v[q] = w[q] + v[q];
                }
                if (row < M) {
                    if (col0 + 32 <= N && (N & 3) == 0) {
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            *reinterpret_cast<float4*>(crow + col0 + 4 * q) =
                                make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    } else {
                        for (int q = 0; q < 32; ++q)
                            if (col0 + q < N) crow[col0 + q] = v[q];
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(empty_leader_base + acc * sizeof(uint64_t));
            if (partial_out) {    // publish this CTA's partial slot
                __threadfence();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (etid == 0) store_release_gpu(flag(split), 1);
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync_all();      // the peer may still be signalling the leader's barriers
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// Pre-pass.  transpose: Bt[n][k] = tf32_rn(B[k][n]).  3xTF32: hi = tf32(x)
// (cvt.rna), lo = tf32(x - hi); A3 = [A_hi | A_hi | A_lo] (M x 3K) and
// Bt3 = [B_hi^T | B_lo^T | B_hi^T] (N x 3K), so one tf32 GEMM over 3K sums
// A_hi·B_hi + A_hi·B_lo + A_lo·B_hi.  32x32 tiles through padded smem keep
// both the read and the write coalesced.
__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

template <bool kSplit>
__global__ void __launch_bounds__(256) transpose_b(const float* __restrict__ B, float* __restrict__ Bt, int K, int N) {
    __shared__ float tile[32][33];
    const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
    for (int r = ty; r < 32; r += 8) {
        const int k = k0 + r, n = n0 + tx;
        tile[r][tx] = (k < K && n < N) ? B[static_cast<long long>(k) * N + n] : 0.f;
    }
    __syncthreads();
    const long long ld = kSplit ? 3LL * K : K;
#pragma unroll
    for (int r = ty; r < 32; r += 8) {
        const int n = n0 + r, k = k0 + tx;
        if (n < N && k < K) {
            const float x = tile[tx][r];
            float* row = Bt + static_cast<long long>(n) * ld;
            if (kSplit) {
                const float hi = to_tf32(x);
                const float lo = to_tf32(x - hi);
                row[k] = hi;
                row[K + k] = lo;
                row[2LL * K + k] = hi;
            } else {
                row[k] = to_tf32(x);
            }
        }
    }
}

// Round-to-nearest tf32 copy of A.  The tensor core would otherwise truncate
// the low 13 mantissa bits, a bias that accumulates over K (measured 7e-4
// max relative error at K = 1024 vs 4.5e-5 with RN operands).
__global__ void __launch_bounds__(256) round_a(const float4* __restrict__ A, float4* __restrict__ Ar, long long n4) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float4 v = A[i];
        Ar[i] = make_float4(to_tf32(v.x), to_tf32(v.y), to_tf32(v.z), to_tf32(v.w));
    }
}

// One thread per 4 consecutive k (K % 4 == 0): one 16-byte load, three
// 16-byte stores into the [A_hi | A_hi | A_lo] row.
__global__ void __launch_bounds__(256) split3_a(const float* __restrict__ A, float* __restrict__ A3, int M, int K) {
    const int vpr = K / 4;
    const long long total = static_cast<long long>(M) * vpr;
    for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < total;
         v += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long m = v / vpr;
        const int k = static_cast<int>(v - m * vpr) * 4;
        const float4 x = *reinterpret_cast<const float4*>(A + m * K + k);
        const float4 hi = make_float4(to_tf32(x.x), to_tf32(x.y), to_tf32(x.z), to_tf32(x.w));
        const float4 lo = make_float4(to_tf32(x.x - hi.x), to_tf32(x.y - hi.y), to_tf32(x.z - hi.z),
                                      to_tf32(x.w - hi.w));
        float4* row = reinterpret_cast<float4*>(A3 + m * 3LL * K + k);
        const long long seg = K / 4;
        row[0] = hi;
        row[seg] = hi;
        row[2 * seg] = lo;
    }
}

// 3xBF16 pre-pass: x = hi + lo + O(2^-17 |x|) with hi = bf16_rn(x), lo =
// bf16_rn(x - hi) (x - hi is exact in fp32).  Segments of Kp = K rounded up
// to 8 elements (16-byte TMA row pitch), zero-padded:
//   A3[m]  = [A_hi | A_hi | A_lo]      (M x 3Kp bf16)
//   Bt3[n] = [B_hi^T | B_lo^T | B_hi^T] (N x 3Kp bf16)
// so one bf16 GEMM over 3Kp sums A_hi·B_hi + A_hi·B_lo + A_lo·B_hi, on the
// kind::f16 path at twice the tf32 rate (the dropped A_lo·B_lo is ~2^-16).
__device__ __forceinline__ void bf16_split(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
    hi = __float2bfloat16_rn(x);
    lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

// One thread per 8 consecutive k of a row: two 16-byte loads, three
// 16-byte stores (hi | hi | lo segments).  Kp % 8 == 0 and K % 4 == 0, so a
// vector is either fully inside K, half inside (K % 8 == 4), or padding.
__global__ void __launch_bounds__(256) split3_a_bf16(const float* __restrict__ A, __nv_bfloat16* __restrict__ A3,
                                                     int M, int K, int Kp) {
    const int vpr = Kp / 8;                                   // vectors per row
    const long long total = static_cast<long long>(M) * vpr;
    for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < total;
         v += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long m = v / vpr;
        const int k = static_cast<int>(v - m * vpr) * 8;
        const float* src = A + m * K + k;
        float x[8];
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 x0 = k < K ? *reinterpret_cast<const float4*>(src) : z4;
        const float4 x1 = k + 4 < K ? *reinterpret_cast<const float4*>(src + 4) : z4;
        x[0] = x0.x, x[1] = x0.y, x[2] = x0.z, x[3] = x0.w, x[4] = x1.x, x[5] = x1.y, x[6] = x1.z, x[7] = x1.w;
        __align__(16) __nv_bfloat16 hi[8], lo[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) bf16_split(x[q], hi[q], lo[q]);
        uint4* row = reinterpret_cast<uint4*>(A3 + m * 3LL * Kp + k);
        const uint4 h = *reinterpret_cast<const uint4*>(hi), l = *reinterpret_cast<const uint4*>(lo);
        const long long seg = Kp / 8;                             // uint4 per segment
        row[0] = h;
        row[seg] = h;
        row[2 * seg] = l;
    }
}

// 64(k) x 32(n) tiles: each thread stores bf16 pairs (two consecutive k), so
// a warp writes 128 contiguous bytes of each output row segment.
__global__ void __launch_bounds__(256) transpose_b_split3_bf16(const float* __restrict__ B,
                                                               __nv_bfloat16* __restrict__ Bt3, int K, int N,
                                                               int Kp) {
    __shared__ float tile[64][33];
    const int k0 = blockIdx.y * 64, n0 = blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
    for (int r = ty; r < 64; r += 8) {
        const int k = k0 + r, n = n0 + tx;
        tile[r][tx] = (k < K && n < N) ? B[static_cast<long long>(k) * N + n] : 0.f;
    }
    __syncthreads();
    const int k = k0 + 2 * tx;                   // this thread's k pair
#pragma unroll
    for (int r = ty; r < 32; r += 8) {
        const int n = n0 + r;
        if (n < N && k < Kp) {                   // Kp even: k + 1 < Kp too
            __nv_bfloat16 h0, l0, h1, l1;        // zero (k >= K) splits to zeros
            bf16_split(tile[2 * tx][r], h0, l0);
            bf16_split(tile[2 * tx + 1][r], h1, l1);
            __nv_bfloat162* row = reinterpret_cast<__nv_bfloat162*>(Bt3 + static_cast<long long>(n) * 3 * Kp + k);
            const long long seg = Kp / 2;         // bf16 pairs per segment
            const __nv_bfloat162 hh = __halves2bfloat162(h0, h1), ll = __halves2bfloat162(l0, l1);
            row[0] = hh;
            row[seg] = ll;
            row[2 * seg] = hh;
        }
    }
}

// ---- host side ----------------------------------------------------------------

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

static int make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                    uint32_t box_inner, uint32_t box_outer, bool bf16 = false) {
    EncodeFn enc = get_encode();
    if (!enc) {
        set_error("hf_gemm_tc: cuTensorMapEncodeTiled unavailable");
        return HF_ECUDA;
    }
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                     const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("hf_gemm_tc: cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
        return HF_ECUDA;
    }
    return HF_OK;
}

constexpr int PAIR_STAGES = 6;

static const int kRegistered = register_kernels(
    {(const void*)gemm_tf32_kernel<4, 2>, (const void*)gemm_tf32_kernel<2, 1>,
     (const void*)gemm_tf32_kernel<3, 1, false, 128>, (const void*)gemm_tf32_kernel<3, 1, true, 128>,
     (const void*)gemm_tf32_pair_kernel<PAIR_STAGES>, (const void*)gemm_tf32_kernel<4, 2, true>,
     (const void*)gemm_tf32_kernel<2, 1, true>, (const void*)gemm_tf32_pair_kernel<PAIR_STAGES, true>,
     (const void*)transpose_b<true>, (const void*)transpose_b<false>, (const void*)round_a, (const void*)split3_a,
     (const void*)split3_a_bf16, (const void*)transpose_b_split3_bf16});

// HF_GEMM_TC_PAIR=0 selects the single-CTA persistent kernel for standalone
// calls (A/B comparisons); the default is the CTA-pair kernel.
static bool pair_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("HF_GEMM_TC_PAIR");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

// HF_GEMM_TC_SPLIT=0 disables the deterministic tail split of the pair kernel.
static bool split_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("HF_GEMM_TC_SPLIT");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

// Co-scheduled tile width: HF_TC_COSCHED_BN=128 (3 stages of 128 x 128) or
// 256 (2 stages of 128 x 256, the default).
static int cosched_bn() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("HF_TC_COSCHED_BN");
        v = (e && atoi(e) == 128) ? 128 : 256;
    }
    return v;
}

// Co-scheduled grid cap (HF_TC_COSCHED_GRID, experiments only; default 0 =
// one CTA per tile): the kernel is persistent, so a cap makes it hold that
// many CTA slots for its whole run.
static int cosched_grid() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("HF_TC_COSCHED_GRID");
        v = e ? atoi(e) : 0;
        if (v < 0) v = 0;
    }
    return v;
}

// Launch shape: CTA pairs (6 stages, double-buffered TMEM, 74 persistent
// pairs) by default; single-CTA persistent (4 stages, grid = SMs) with
// HF_GEMM_TC_PAIR=0 or below 256 x 256; co-scheduling (2 stages, 1
// accumulator, grid = tiles) with
// default; co-scheduling (2 stages, 1 accumulator, grid = tiles) with
// HF_GEMM_COSCHEDULE, when the TC replica runs concurrently with the SIMT
// replica on the same GPU.
// A: M x K row-major, Bt: N x K row-major (both K-major; K counts elements
// of the operand kind, row pitch K * ELEM bytes)
template <bool BF16>
static int launch(const void* A, const void* Bt, float* C, int M, int N, int K, int device, cudaStream_t st,
                  bool cosched) {
    using OK = OpKind<BF16>;
    const uint64_t pitch = static_cast<uint64_t>(K) * OK::ELEM;
    CUtensorMap ta, tb;
    if (!cosched && pair_enabled() && M >= PBM && N >= PBN) {
        // CTA pairs: each CTA stages half of the 256 x 256 tile's operands
        int rc = make_map(&ta, A, static_cast<uint64_t>(K), static_cast<uint64_t>(M), pitch, OK::BKE, PBM / 2, BF16);
        if (rc) return rc;
        rc = make_map(&tb, Bt, static_cast<uint64_t>(K), static_cast<uint64_t>(N), pitch, OK::BKE, PBN / 2, BF16);
        if (rc) return rc;
        static bool pair_attr[64] = {false};
        if (!pair_attr[device]) {
            HF_CUDA_CHECK(cudaFuncSetAttribute(gemm_tf32_pair_kernel<PAIR_STAGES, BF16>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               pair_smem_bytes<PAIR_STAGES>()));
            pair_attr[device] = true;
        }
        const int ptiles = ((M + PBM - 1) / PBM) * ((N + PBN - 1) / PBN);
        const int pairs_max = num_sms(device) / 2;
        const int pairs = ptiles < pairs_max ? ptiles : pairs_max;
        PairSplit sp{ptiles, 1, nullptr, nullptr};
        const int R = ptiles % pairs;
        const int nkb = (K + OK::BKE - 1) / OK::BKE;
        if (R > 0 && ptiles > pairs && split_enabled()) {
            int splits = pairs / R;
            if (splits > 4) splits = 4;
            if (splits > nkb) splits = nkb;
            if (splits > 1) {
                sp.full_tiles = ptiles - R;
                sp.splits = splits;
                const size_t slots = static_cast<size_t>(R) * (splits - 1);
                const size_t pbytes = slots * PBM * PBN * sizeof(float);
                const size_t fbytes = slots * 2 * sizeof(int);
                uint8_t* ws = nullptr;
                HF_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&ws), pbytes + fbytes, st));
                sp.partial = reinterpret_cast<float*>(ws);
                sp.flags = reinterpret_cast<int*>(ws + pbytes);
                HF_CUDA_CHECK(cudaMemsetAsync(sp.flags, 0, fbytes, st));
            }
        }
        // With the tail split, a fixup CTA spins on flags that partial CTAs
        // of lower-numbered pairs publish (the split units of a tile are
        // consecutive and the last, the fixup, has the highest pair), so the
        // wait needs those CTAs co-resident.  A cooperative launch guarantees
        // it (the grid is one persistent CTA per SM); if the device refuses
        // one, the kernel runs without the split (whole tiles only, no
        // inter-CTA waits) — same bytes per tile, just a ragged last round.
        cudaError_t le = cudaSuccess;
        if (sp.splits > 1) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(2 * pairs);
            cfg.blockDim = dim3(NUM_THREADS);
            cfg.dynamicSmemBytes = pair_smem_bytes<PAIR_STAGES>();
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeCooperative;
            at[0].val.cooperative = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            le = cudaLaunchKernelEx(&cfg, gemm_tf32_pair_kernel<PAIR_STAGES, BF16>, ta, tb, C, M, N, K, sp);
            static const bool verbose = getenv("HF_GEMM_TC_VERBOSE") != nullptr;
            if (verbose)
                fprintf(stderr, "hf_gemm_tc: pair kernel, %d tail tiles split %d ways, cooperative launch: %s\n",
                        ptiles - sp.full_tiles, sp.splits, cudaGetErrorString(le));
            if (le != cudaSuccess) {
                cudaGetLastError();
                cudaFreeAsync(sp.partial, st);
                sp = PairSplit{ptiles, 1, nullptr, nullptr};
            }
        }
        if (sp.splits == 1)
            gemm_tf32_pair_kernel<PAIR_STAGES, BF16><<<2 * pairs, NUM_THREADS, pair_smem_bytes<PAIR_STAGES>(), st>>>(
                ta, tb, C, M, N, K, sp);
        if (sp.partial) cudaFreeAsync(sp.partial, st);
        HF_CHECK_LAUNCH();
        return HF_OK;
    }
    const bool narrow = cosched && cosched_bn() == 128;
    int rc = make_map(&ta, A, static_cast<uint64_t>(K), static_cast<uint64_t>(M), pitch, OK::BKE, BM, BF16);
    if (rc) return rc;
    rc = make_map(&tb, Bt, static_cast<uint64_t>(K), static_cast<uint64_t>(N), pitch, OK::BKE, narrow ? 128 : BN,
                  BF16);
    if (rc) return rc;
    const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
    static bool attr_set[64] = {false};
    if (!attr_set[device]) {
        HF_CUDA_CHECK(cudaFuncSetAttribute(gemm_tf32_kernel<4, 2, BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           smem_bytes<4>()));
        HF_CUDA_CHECK(cudaFuncSetAttribute(gemm_tf32_kernel<2, 1, BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           smem_bytes<2>()));
        HF_CUDA_CHECK(cudaFuncSetAttribute(gemm_tf32_kernel<3, 1, BF16, 128>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<3, 128>()));
        // co-scheduled shapes share SMs with SIMT CTAs: whichever kernel's CTA
        // reaches an idle SM first, the SM is configured all-shared
        HF_CUDA_CHECK(cudaFuncSetAttribute(gemm_tf32_kernel<2, 1, BF16>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                           cudaSharedmemCarveoutMaxShared));
        HF_CUDA_CHECK(cudaFuncSetAttribute(gemm_tf32_kernel<3, 1, BF16, 128>,
                                           cudaFuncAttributePreferredSharedMemoryCarveout,
                                           cudaSharedmemCarveoutMaxShared));
        attr_set[device] = true;
    }
    if (narrow) {
        // co-scheduled, 128 x 128 tiles and 3 stages in about the smem of
        // 2 stages of 128 x 256: twice the CTAs, each half as long, so they
        // pack the SIMT grid's last wave more tightly
        const int tiles_narrow = ((M + BM - 1) / BM) * ((N + 127) / 128);
        gemm_tf32_kernel<3, 1, BF16, 128><<<tiles_narrow, NUM_THREADS, smem_bytes<3, 128>(), st>>>(ta, tb, C, M, N,
                                                                                                K);
    } else if (cosched) {
        const int cap = cosched_grid();
        gemm_tf32_kernel<2, 1, BF16><<<cap > 0 && cap < tiles ? cap : tiles, NUM_THREADS, smem_bytes<2>(), st>>>(
            ta, tb, C, M, N, K);
    } else {
        const int sms = num_sms(device);
        const int grid = tiles < sms ? tiles : sms;
        gemm_tf32_kernel<4, 2, BF16><<<grid, NUM_THREADS, smem_bytes<4>(), st>>>(ta, tb, C, M, N, K);
    }
    HF_CHECK_LAUNCH();
    return HF_OK;
}

}  // namespace tc
}  // namespace hf

extern "C" int hf_gemm_tc(const float* A, const float* B, float* C, int M, int N, int K, int mode, int device,
                          void* stream) {
    HF_REQUIRE(A && B && C, "hf_gemm_tc: NULL operand");
    HF_REQUIRE(M > 0 && N > 0 && K > 0, "hf_gemm_tc: bad shape %dx%dx%d", M, N, K);
    const bool cosched = (mode & HF_GEMM_COSCHEDULE) != 0;
    mode &= ~HF_GEMM_COSCHEDULE;
    HF_REQUIRE(mode == HF_GEMM_TF32 || mode == HF_GEMM_3XTF32 || mode == HF_GEMM_3XBF16,
               "hf_gemm_tc: unknown mode %d", mode);
    if (K % 4 != 0 || N % 4 != 0 || (reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) % 16 != 0) {
        hf::set_error("hf_gemm_tc: TMA needs 16-byte aligned operands and K %% 4 == N %% 4 == 0 (got K=%d N=%d)", K, N);
        return HF_EUNSUP;
    }
    hf::DeviceGuard g(device);
    HF_REQUIRE(g.ok, "hf_gemm_tc: cannot select device %d", device);
    cudaStream_t st = hf::as_stream(stream);
    hf::retain_scratch_pool(device);
    const bool bf16 = mode == HF_GEMM_3XBF16;
    const bool split = mode != HF_GEMM_TF32;
    const int Kp = bf16 ? (K + 7) / 8 * 8 : K;
    const int Ke = split ? 3 * Kp : K;
    const size_t elem = bf16 ? 2 : 4;
    void* Bt = hf::stream_scratch(device, st, 0, static_cast<size_t>(N) * Ke * elem);
    void* A3 = hf::stream_scratch(device, st, 1, static_cast<size_t>(M) * Ke * elem);
    if (!Bt || !A3) {
        hf::set_error("hf_gemm_tc: cannot allocate %zu bytes of operand scratch", static_cast<size_t>(M + N) * Ke * elem);
        return HF_ECUDA;
    }
    // Co-scheduled with a SIMT replica: the pre-pass runs on a high-priority
    // side stream (level 1: one below the SIMT pre-pass), so its CTAs are
    // dispatched ahead of the SIMT GEMM's pending CTAs, while the GEMM itself
    // stays on the caller's (lower-priority) stream and fills the SIMT grid's
    // last wave.  Without it the pre-pass, and so the GEMM, waited for that
    // last wave whenever the SIMT grid reached the GPU first.
    hf::SideStream* side = cosched ? hf::side_stream(device, 1) : nullptr;
    cudaStream_t ps = st;
    HF_CUDA_CHECK(hf::begin_side_launch(side, st, &ps));
    const int pre_grid = hf::num_sms(device) * 8;
    if (bf16) {
        dim3 tgrid((N + 31) / 32, (Kp + 63) / 64);
        hf::tc::transpose_b_split3_bf16<<<tgrid, 256, 0, ps>>>(B, static_cast<__nv_bfloat16*>(Bt), K, N, Kp);
        hf::tc::split3_a_bf16<<<pre_grid, 256, 0, ps>>>(A, static_cast<__nv_bfloat16*>(A3), M, K, Kp);
    } else if (split) {
        dim3 tgrid((N + 31) / 32, (K + 31) / 32);
        hf::tc::transpose_b<true><<<tgrid, 256, 0, ps>>>(B, static_cast<float*>(Bt), K, N);
        hf::tc::split3_a<<<pre_grid, 256, 0, ps>>>(A, static_cast<float*>(A3), M, K);
    } else {
        dim3 tgrid((N + 31) / 32, (K + 31) / 32);
        hf::tc::transpose_b<false><<<tgrid, 256, 0, ps>>>(B, static_cast<float*>(Bt), K, N);
        const long long n4 = static_cast<long long>(M) * K / 4;  // K % 4 == 0
        hf::tc::round_a<<<pre_grid, 256, 0, ps>>>(reinterpret_cast<const float4*>(A), static_cast<float4*>(A3), n4);
    }
    HF_CUDA_CHECK(hf::end_side_launch(side, st));
    return bf16 ? hf::tc::launch<true>(A3, Bt, C, M, N, Ke, device, st, cosched)
                : hf::tc::launch<false>(A3, Bt, C, M, N, Ke, device, st, cosched);
}
