// Stage-by-stage probe of the tcgen05 GEMM building blocks (debug tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -Ipaper_1405_2912_b200/csrc -Iinclude \
//        -o tools/tc_probe tools/tc_probe.cu -lcuda -Lpaper_1405_2912_b200 -lhetft \
//        -Xlinker -rpath,'$ORIGIN/../paper_1405_2912_b200'
// Prints PASS/FAIL lines per stage.
#include "../paper_1405_2912_b200/csrc/gemm_tc.cu"

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

using namespace hf::tc;
constexpr int B_STAGE = 256 * 32 * 4;  // one 256n x 32k fp32 B tile

// 1. TMEM roundtrip: st 32x32b.x32 then ld
__global__ void tmem_roundtrip(float* out) {
    __shared__ uint32_t base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&base)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t t = base + (static_cast<uint32_t>(warp * 32) << 16);
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(static_cast<float>((warp * 32 + lane) * 1000 + i));
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(t),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    float v[32];
    tmem_ld32(t, v);
    for (int i = 0; i < 32; ++i) out[(warp * 32 + lane) * 32 + i] = v[i];
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(512));
    }
}

// 2. TMA placement: load one A box and one B box, dump smem bytes
__global__ void tma_dump(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, float* outA,
                         float* outB) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + A_STAGE + 4096);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(bar, A_STAGE + 4096);
        tma_load_2d(smem, &tmA, bar, 0, 0);
        tma_load_2d(smem + A_STAGE, &tmB, bar, 0, 0);
    }
    mbar_wait(bar, 0);
    const float* f = reinterpret_cast<const float*>(smem);
    for (int i = threadIdx.x; i < A_STAGE / 4; i += blockDim.x) outA[i] = f[i];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) outB[i] = f[A_STAGE / 4 + i];
}


// 4. One k-block of MMAs on TMA-filled smem with a sentinel-prefilled
// accumulator; variant selects descriptor hypotheses.
__global__ void mma_probe(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmBt, const __grid_constant__ CUtensorMap tmB32,
                          float* out, int variant) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
    uint8_t* sa = smem;
    uint8_t* sb = smem + A_STAGE;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + A_STAGE + B_STAGE);
    uint64_t* bar2 = bar + 1;
    __shared__ uint32_t base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool kmajorB = variant < 12 && (variant & 4) != 0;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(bar2, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&base)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        mbar_expect_tx(bar, A_STAGE + B_STAGE);
        tma_load_2d(sa, &tmA, bar, 0, 0);
        if (kmajorB) {
            tma_load_2d(sb, &tmBt, bar, 0, 0);
            tma_load_2d(sb + B_STAGE / 2, &tmBt, bar, 0, 128);
        } else {
            // variants >= 12: B boxes written with the 32-byte-atom 128B swizzle
            const CUtensorMap* mb = variant >= 12 ? &tmB32 : &tmB;
            for (int j = 0; j < 8; ++j) tma_load_2d(sb + j * 4096, mb, bar, 32 * j, 0);
        }
    }
    mbar_wait(bar, 0);
    const uint32_t t = base + (static_cast<uint32_t>(warp * 32) << 16);
    {
        uint32_t s5 = __float_as_uint(5.0f);
        for (int c = 0; c < 256; c += 32)
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
                "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(t + c), "r"(s5));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        uint32_t idesc = make_idesc(128, 256);
        if (variant & 1) {  // M field at bit 23
            idesc &= ~(0x1Fu << 24);
            idesc |= (128u >> 4) << 23;
        }
        // make_idesc is K-major for both operands; the MN-major variants set the
        // B-transpose bit (bit 16).  (An earlier version of this probe only ever
        // cleared it, so its "MN-major" runs were K-major reads of MN-major data.)
        if (!kmajorB) idesc |= 1u << 16;
        if (variant & 2) idesc &= ~((2u << 7) | (2u << 10));  // format codes 0
        for (int kk = 0; kk < 4; ++kk) {
            uint64_t ad = make_desc(smem_u32(sa) + kk * 32, 16, 1024);
            uint64_t bd = kmajorB ? make_desc(smem_u32(sb) + kk * 32, 16, 1024)
                                  : make_desc(smem_u32(sb) + kk * 1024, 4096, 1024);
            if (variant == 8) bd = make_desc(smem_u32(sb) + kk * 1024, 1024, 4096);       // swapped
            if (variant == 9) bd = make_desc(smem_u32(sb) + kk * 1024, 4096, 1024) | (1ull << 52);  // lbo mode
            if (variant == 10) {  // a_major MN instead of b (sanity on bit position)
                idesc = make_idesc(128, 256) & ~(1u << 16);
                idesc |= 1u << 15;
            }
            if (variant == 11) {  // N = 32: single MN atom, LBO irrelevant
                idesc = (make_idesc(128, 256) & ~(0x3Fu << 17)) | ((32u >> 3) << 17);
            }
            if (variant >= 12) {
                // MN-major tf32: SWIZZLE_128B_BASE32B (layout type 1) is the
                // only layout CUTLASS's SM100 builder allows for it.
                // 12: LBO 4096 (next 32-column MN atom), SBO 512 (next 4-row K group)
                // 13: the two swapped; 14: LBO 4096, SBO 1024 with layout type 2;
                // 15: LBO 4096, SBO 1024 with layout type 1
                const uint32_t lbo = variant == 13 ? 512 : 4096;
                const uint32_t sbo = variant == 13 ? 4096 : (variant == 12 ? 512 : 1024);
                bd = make_desc(smem_u32(sb) + kk * 1024, lbo, sbo);
                bd = (bd & ~(7ull << 61)) | ((variant == 14 ? 2ull : 1ull) << 61);
            }
            tc_mma_tf32(base, ad, bd, idesc, 1);
        }
        tc_commit(bar2);
    }
    mbar_wait(bar2, 0);
    tc_fence_after();
    for (int c = 0; c < 256; c += 32) {
        float v[32];
        tmem_ld32(t + c, v);
        for (int i = 0; i < 32; ++i) out[(warp * 32 + lane) * 256 + c + i] = v[i];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(256));
    }
}

static CUtensorMap mk(const void* base, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo) {
    CUtensorMap m;
    if (make_map(&m, base, inner, outer, inner * 4, bi, bo) != HF_OK) {
        printf("make_map failed: %s\n", hf_last_error());
        exit(1);
    }
    return m;
}

int main(int argc, char** argv) {
    cudaSetDevice(0);
    // --- 1
    float* d;
    cudaMalloc(&d, 128 * 32 * 4);
    tmem_roundtrip<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> h(128 * 32);
    cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int l = 0; l < 128; ++l)
        for (int i = 0; i < 32; ++i)
            if (h[l * 32 + i] != l * 1000 + i) ++bad;
    printf("tmem_roundtrip: %s (err=%s, bad=%d, sample %g %g)\n", bad ? "FAIL" : "PASS", cudaGetErrorString(e), bad,
           h[0], h[33 * 32 + 5]);

    // --- 2
    const int M = 128, K = 32, N = 256;
    std::vector<float> A(M * K), B(K * N);
    for (int i = 0; i < M * K; ++i) A[i] = i;
    for (int i = 0; i < K * N; ++i) B[i] = i;
    float *dA, *dB, *oA, *oB, *dC;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&oA, A_STAGE);
    cudaMalloc(&oB, 4096);
    cudaMalloc(&dC, M * N * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap ta = mk(dA, K, M, BK, BM), tb = mk(dB, N, K, 32, BK);
    cudaFuncSetAttribute(tma_dump, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    tma_dump<<<1, 128, 64 * 1024>>>(ta, tb, oA, oB);
    e = cudaDeviceSynchronize();
    std::vector<float> hA(A_STAGE / 4), hB(1024);
    cudaMemcpy(hA.data(), oA, A_STAGE, cudaMemcpyDeviceToHost);
    cudaMemcpy(hB.data(), oB, 4096, cudaMemcpyDeviceToHost);
    // expected SW128: element (row r, col c) at float index r*32 + (((c/4) ^ (r%8))*4 + c%4)
    int badA = 0, badB = 0;
    for (int r = 0; r < 128; ++r)
        for (int c = 0; c < 32; ++c)
            if (hA[r * 32 + (((c / 4) ^ (r % 8)) * 4 + c % 4)] != A[r * K + c]) ++badA;
    for (int r = 0; r < 32; ++r)
        for (int c = 0; c < 32; ++c)
            if (hB[r * 32 + (((c / 4) ^ (r % 8)) * 4 + c % 4)] != B[r * N + c]) ++badB;
    printf("tma_dump: %s (err=%s badA=%d badB=%d; A[0..7]=%g %g %g %g %g %g %g %g)\n", (badA || badB) ? "FAIL" : "PASS",
           cudaGetErrorString(e), badA, badB, hA[0], hA[1], hA[2], hA[3], hA[4], hA[5], hA[6], hA[7]);

    // --- 3 full kernel on one tile, identity-ish A
    std::vector<float> A1(M * K, 0.f);
    for (int i = 0; i < M; ++i) A1[i * K + (i % K)] = 1.f;
    for (int k = 0; k < K; ++k)
        for (int n = 0; n < N; ++n) B[k * N + n] = k;
    cudaMemcpy(dA, A1.data(), A1.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    int rc = hf_gemm_tc(dA, dB, dC, M, N, K, 0, 0, nullptr);
    e = cudaDeviceSynchronize();
    std::vector<float> hC(M * N);
    cudaMemcpy(hC.data(), dC, hC.size() * 4, cudaMemcpyDeviceToHost);
    int badC = 0;
    for (int i = 0; i < M; ++i)
        for (int n = 0; n < N; ++n)
            if (hC[i * N + n] != i % K) ++badC;
    printf("gemm_identity: %s (rc=%d err=%s badC=%d; C[1,0]=%g C[5,3]=%g C[40,100]=%g)\n", badC ? "FAIL" : "PASS", rc,
           cudaGetErrorString(e), badC, hC[N], hC[5 * N + 3], hC[40 * N + 100]);
    // --- 4 MMA probes
    {
        std::vector<float> Ar(M * K), Br(K * N), Bt(N * K);
        for (int i = 0; i < M * K; ++i) Ar[i] = static_cast<float>((i * 7) % 5);
        for (int i = 0; i < K * N; ++i) Br[i] = static_cast<float>((i * 3) % 7);
        if (getenv("TC_PROBE_EYE")) {  // C - 5 then shows which (k, n % 32) of B each output read
            for (int i = 0; i < M * K; ++i) Ar[i] = (i % K) == ((i / K) % K) ? 1.f : 0.f;
            for (int k = 0; k < K; ++k)
                for (int n = 0; n < N; ++n) Br[k * N + n] = static_cast<float>(k + 32 * (n % 32));
        }
        for (int k = 0; k < K; ++k)
            for (int n = 0; n < N; ++n) Bt[n * K + k] = Br[k * N + n];
        float* dBt;
        cudaMalloc(&dBt, Bt.size() * 4);
        cudaMemcpy(dA, Ar.data(), Ar.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, Br.data(), Br.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dBt, Bt.data(), Bt.size() * 4, cudaMemcpyHostToDevice);
        CUtensorMap tA = mk(dA, K, M, BK, BM), tB = mk(dB, N, K, 32, BK), tBt = mk(dBt, K, N, BK, 128);
        CUtensorMap tB32;
        {
            cuuint64_t dims[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(K)};
            cuuint64_t strides[1] = {static_cast<cuuint64_t>(N) * 4};
            cuuint32_t box[2] = {32, static_cast<cuuint32_t>(BK)};
            cuuint32_t estr[2] = {1, 1};
            CUresult r = get_encode()(&tB32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            printf("tB32 encode: %d\n", static_cast<int>(r));
        }
        cudaFuncSetAttribute(mma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
        std::vector<float> ref(M * N);
        for (int i = 0; i < M; ++i)
            for (int n = 0; n < N; ++n) {
                float acc = 5.f;
                for (int k = 0; k < K; ++k) acc += Ar[i * K + k] * Br[k * N + n];
                ref[i * N + n] = acc;
            }
        if (argc > 1 && std::string(argv[1]) == "dump32") {
            // Where TMA's SWIZZLE_128B_ATOM_32B puts B's 32-byte chunks: row k, chunk c -> chunk
            std::vector<float> iota(K * N);
            for (int i = 0; i < K * N; ++i) iota[i] = static_cast<float>(i);
            cudaMemcpy(dB, iota.data(), iota.size() * 4, cudaMemcpyHostToDevice);
            cudaFuncSetAttribute(tma_dump, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
            tma_dump<<<1, 128, 64 * 1024>>>(ta, tB32, oA, oB);
            cudaDeviceSynchronize();
            cudaMemcpy(hB.data(), oB, 4096, cudaMemcpyDeviceToHost);
            for (int r = 0; r < 12; ++r) {
                printf("dump32 row %2d:", r);
                for (int q = 0; q < 4; ++q) {  // smem chunk q holds source chunk ...
                    const int col = static_cast<int>(hB[r * 32 + q * 8]) - r * N;
                    printf(" %d", col / 8);
                }
                printf("\n");
            }
            return 0;
        }
        std::vector<int> variants = {12, 13, 14, 15, 4, 0, 9, 10, 11, 8};
        if (argc > 1) variants = {atoi(argv[1])};  // one variant per process: a fault poisons the context
        for (int variant : variants) {
            cudaMemset(dC, 0, M * N * 4);
            mma_probe<<<1, 128, 80 * 1024>>>(tA, tB, tBt, tB32, dC, variant);
            e = cudaDeviceSynchronize();
            cudaMemcpy(hC.data(), dC, hC.size() * 4, cudaMemcpyDeviceToHost);
            int nb = 0, n5 = 0, nb32 = 0;
            for (int i = 0; i < M * N; ++i) {
                nb += hC[i] != ref[i];
                n5 += hC[i] == 5.f;
                if (i % N < 32) nb32 += hC[i] != ref[i];
            }
            printf("  (first-32-column mismatches: %d)\n", nb32);
            if (argc > 2) {  // raw C (fp32, 128 x 256) for offline analysis
                FILE* f = fopen(argv[2], "wb");
                fwrite(hC.data(), 4, hC.size(), f);
                fclose(f);
            }
            printf("mma_probe v%d: %s (err=%s bad=%d sentinel_only=%d; C[0,0]=%g ref %g; C[1,2]=%g ref %g)\n", variant,
                   nb ? "FAIL" : "PASS", cudaGetErrorString(e), nb, n5, hC[0], ref[0], hC[N + 2], ref[N + 2]);
            if (e != cudaSuccess) break;
        }
    }
    return 0;
}
