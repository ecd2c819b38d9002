// Copy / checkpoint / restore / checksum (sm_100a).
//
// Replaces the O(n) payload copies of the reference memory manager
// (/root/reference/pkg/src/hetrt/memory.py:146,160,164 — sibling transfers —
// and :176-189 _maybe_checkpoint, the backup of the sole max-version copy)
// with device-memory streams: 128-bit loads/stores, 4 vectors in flight per
// thread, grid sized to a multiple of the SM count.  Cross-device copies
// pull over NVLink P2P (copy kernel on the destination GPU loading the peer
// pointer) when peer access is enabled, else fall back to the copy engine.
//
// Checksum (new; lets a restore verify the snapshot it reads back): for the
// 32-bit little-endian word w_j at word index j (a ragged tail is zero
// padded into one last word)
//     x  = w_j ^ lo32(j * 0x9E3779B9) ^ (hi32(j) * 0x7F4A7C15)
//     x *= 0x85EBCA6B;  x ^= x >> 13;  x *= 0xC2B2AE35;  x ^= x >> 16
//     S  = sum_j x  (mod 2^64)
//     checksum = S ^ (nbytes * 0x9E3779B97F4A7C15)  (mod 2^64)
// It is position sensitive and order independent, so a parallel sum
// reduction computes it exactly; oracle/checksum.py restates it.
#include "common.cuh"

#include <mutex>
#include <vector>

namespace hf {

__device__ __forceinline__ uint32_t mix_word(uint32_t w, unsigned long long j) {
    uint32_t x = w ^ static_cast<uint32_t>(j * 0x9E3779B9ull) ^
                 (static_cast<uint32_t>(j >> 32) * 0x7F4A7C15u);
    x *= 0x85EBCA6Bu;
    x ^= x >> 13;
    x *= 0xC2B2AE35u;
    x ^= x >> 16;
    return x;
}

__device__ __forceinline__ unsigned long long mix_vec(const uint4& v, unsigned long long j0) {
    return static_cast<unsigned long long>(mix_word(v.x, j0)) + mix_word(v.y, j0 + 1) +
           mix_word(v.z, j0 + 2) + mix_word(v.w, j0 + 3);
}

template <bool kStore, bool kSum>
__global__ void __launch_bounds__(256) stream_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                     long long nvec, const uint8_t* __restrict__ src_b,
                                                     uint8_t* __restrict__ dst_b, long long nbytes,
                                                     unsigned long long* sum_out) {
    constexpr int U = 4;
    const long long gtid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long gs = static_cast<long long>(gridDim.x) * blockDim.x;
    unsigned long long acc = 0;
    long long j = gtid;
    pdl_wait();     // launched with PDL: the previous grid's writes are visible from here
    for (; j + (U - 1) * gs < nvec; j += U * gs) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_stream(src + j + u * gs);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if constexpr (kStore) st_stream(dst + j + u * gs, v[u]);
            if constexpr (kSum) acc += mix_vec(v[u], static_cast<unsigned long long>(j + u * gs) * 4);
        }
    }
    for (; j < nvec; j += gs) {
        uint4 v = ld_stream(src + j);
        if constexpr (kStore) st_stream(dst + j, v);
        if constexpr (kSum) acc += mix_vec(v, static_cast<unsigned long long>(j) * 4);
    }
    pdl_launch_dependents();
    // ragged tail (< 16 bytes, or everything when unaligned): per byte copy,
    // per word checksum
    const long long tail0 = nvec * 16;
    if (tail0 < nbytes) {
        for (long long b = tail0 + gtid; b < nbytes; b += gs)
            if constexpr (kStore) dst_b[b] = src_b[b];
        if constexpr (kSum) {
            for (long long w = tail0 / 4 + gtid; w * 4 < nbytes; w += gs) {
                uint32_t word = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    long long b = w * 4 + q;
                    if (b < nbytes) word |= static_cast<uint32_t>(src_b[b]) << (8 * q);
                }
                acc += mix_word(word, static_cast<unsigned long long>(w));
            }
        }
    }
    if constexpr (kSum) {
        __shared__ unsigned long long s_acc;
        if (threadIdx.x == 0) s_acc = 0;
        __syncthreads();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((threadIdx.x & 31) == 0 && acc) atomicAdd(&s_acc, acc);
        __syncthreads();
        if (threadIdx.x == 0 && s_acc) atomicAdd(sum_out, s_acc);
    }
}

static int grid_for(long long work, int device) {
    const int threads = 256;
    long long want = (work + threads * 4 - 1) / (threads * 4);
    if (want < 1) want = 1;
    long long cap = static_cast<long long>(num_sms(device)) * 8;
    return static_cast<int>(want < cap ? want : cap);
}

// Launch the streaming kernel; nvec = 16B vectors when both pointers are 16B
// aligned, else 0 (byte path).
static int launch_stream(void* dst, const void* src, long long nbytes, unsigned long long* sum,
                         int device, cudaStream_t st) {
    // Source loads are ld.global.nc whether `src` is local HBM, a peer GPU's
    // memory or mapped host memory: the source is read-only for the kernel's
    // lifetime (its producers are ordered before this launch by stream
    // events), which is all .nc requires (see ld_stream in common.cuh).
    bool aligned = reinterpret_cast<uintptr_t>(src) % 16 == 0 &&
                   (dst == nullptr || reinterpret_cast<uintptr_t>(dst) % 16 == 0);
    long long nvec = aligned ? nbytes / 16 : 0;
    long long work = nvec > 0 ? nvec : (nbytes + 3) / 4;
    int grid = grid_for(work, device);
    auto d4 = static_cast<uint4*>(dst);
    auto s4 = static_cast<const uint4*>(src);
    auto sb = static_cast<const uint8_t*>(src);
    auto db = static_cast<uint8_t*>(dst);
    if (dst && sum) {
        HF_CUDA_CHECK(launch_pdl(stream_kernel<true, true>, dim3(grid), dim3(256), 0, st, d4, s4, nvec, sb, db, nbytes, sum));
    } else if (dst) {
        HF_CUDA_CHECK(launch_pdl(stream_kernel<true, false>, dim3(grid), dim3(256), 0, st, d4, s4, nvec, sb, db, nbytes, sum));
    } else {
        HF_CUDA_CHECK(launch_pdl(stream_kernel<false, true>, dim3(grid), dim3(256), 0, st, d4, s4, nvec, sb, db, nbytes, sum));
    }
    HF_CHECK_LAUNCH();
    return HF_OK;
}

// Pool of (device accumulator, pinned host mirror) for synchronous checksums.
struct SumSlot {
    unsigned long long* d = nullptr;
    unsigned long long* h = nullptr;
};
static std::mutex g_mu;
static std::vector<SumSlot> g_slots[64];

static int acquire(int device, SumSlot& s) {
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!g_slots[device].empty()) {
            s = g_slots[device].back();
            g_slots[device].pop_back();
            return HF_OK;
        }
    }
    HF_CUDA_CHECK(cudaMalloc(&s.d, sizeof(unsigned long long)));
    HF_CUDA_CHECK(cudaMallocHost(&s.h, sizeof(unsigned long long)));
    return HF_OK;
}

static void release(int device, const SumSlot& s) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_slots[device].push_back(s);
}

static int checksum_impl(void* dst, const void* src, long long nbytes, uint64_t* out,
                         int device, cudaStream_t st) {
    SumSlot s;
    int rc = acquire(device, s);
    if (rc) return rc;
    HF_CUDA_CHECK(cudaMemsetAsync(s.d, 0, sizeof(unsigned long long), st));
    rc = launch_stream(dst, src, nbytes, s.d, device, st);
    if (rc) return rc;
    HF_CUDA_CHECK(cudaMemcpyAsync(s.h, s.d, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    HF_CUDA_CHECK(cudaStreamSynchronize(st));
    *out = static_cast<uint64_t>(*s.h) ^ (static_cast<uint64_t>(nbytes) * 0x9E3779B97F4A7C15ull);
    release(device, s);
    return HF_OK;
}

static const int kRegistered = register_kernels(
    {(const void*)stream_kernel<true, true>, (const void*)stream_kernel<true, false>,
     (const void*)stream_kernel<false, true>});

}  // namespace hf

extern "C" {

int hf_copy(void* dst, int dst_dev, const void* src, int src_dev, int64_t nbytes, void* stream) {
    HF_REQUIRE(nbytes >= 0, "hf_copy: negative size");
    if (nbytes == 0) return HF_OK;
    HF_REQUIRE(dst != nullptr && src != nullptr, "hf_copy: NULL pointer");
    cudaStream_t st = hf::as_stream(stream);
    if (dst_dev >= 0 && src_dev >= 0) {
        if (dst_dev == src_dev || hf_peer_enabled(dst_dev, src_dev)) {
            hf::DeviceGuard g(dst_dev);
            HF_REQUIRE(g.ok, "hf_copy: cannot select device %d", dst_dev);
            return hf::launch_stream(dst, src, nbytes, nullptr, dst_dev, st);
        }
        HF_CUDA_CHECK(cudaMemcpyPeerAsync(dst, dst_dev, src, src_dev, static_cast<size_t>(nbytes), st));
        return HF_OK;
    }
    // a host side: copy engine (pinned memory gives async DMA)
    hf::DeviceGuard g(dst_dev >= 0 ? dst_dev : src_dev);
    HF_CUDA_CHECK(cudaMemcpyAsync(dst, src, static_cast<size_t>(nbytes), cudaMemcpyDefault, st));
    return HF_OK;
}

int hf_fill(void* dst, int value, int64_t nbytes, int device, void* stream) {
    HF_REQUIRE(nbytes >= 0, "hf_fill: negative size");
    if (nbytes == 0) return HF_OK;
    HF_REQUIRE(dst != nullptr, "hf_fill: NULL pointer");
    hf::DeviceGuard g(device >= 0 ? device : -1);
    HF_CUDA_CHECK(cudaMemsetAsync(dst, value & 0xFF, static_cast<size_t>(nbytes), hf::as_stream(stream)));
    return HF_OK;
}

int hf_checkpoint(void* ckpt, const void* buf, int64_t nbytes, uint64_t* checksum, int device,
                  void* stream) {
    HF_REQUIRE(nbytes >= 0, "hf_checkpoint: negative size");
    HF_REQUIRE(device >= 0 && device < 64, "hf_checkpoint: bad device %d", device);
    if (nbytes == 0) {
        if (checksum) *checksum = 0;
        return HF_OK;
    }
    HF_REQUIRE(ckpt != nullptr && buf != nullptr, "hf_checkpoint: NULL pointer");
    hf::DeviceGuard g(device);
    HF_REQUIRE(g.ok, "hf_checkpoint: cannot select device %d", device);
    cudaStream_t st = hf::as_stream(stream);
    // The snapshot may live on a peer GPU: the kernel runs on `device` and
    // stores through the peer pointer (NVLink write).
    if (checksum) return hf::checksum_impl(ckpt, buf, nbytes, checksum, device, st);
    return hf::launch_stream(ckpt, buf, nbytes, nullptr, device, st);
}

int hf_restore(void* buf, const void* ckpt, int64_t nbytes, const uint64_t* expect, int device,
               void* stream) {
    HF_REQUIRE(nbytes >= 0, "hf_restore: negative size");
    HF_REQUIRE(device >= 0 && device < 64, "hf_restore: bad device %d", device);
    if (nbytes == 0) return HF_OK;
    HF_REQUIRE(ckpt != nullptr && buf != nullptr, "hf_restore: NULL pointer");
    hf::DeviceGuard g(device);
    HF_REQUIRE(g.ok, "hf_restore: cannot select device %d", device);
    cudaStream_t st = hf::as_stream(stream);
    if (expect) {
        // verify first, then write: a snapshot that fails its checksum never
        // reaches `buf` (one extra read pass of the snapshot)
        uint64_t got = 0;
        int rc = hf::checksum_impl(nullptr, ckpt, nbytes, &got, device, st);
        if (rc) return rc;
        if (got != *expect) {
            hf::set_error("hf_restore: checksum mismatch (expected %016llx, got %016llx); buffer left untouched",
                          static_cast<unsigned long long>(*expect), static_cast<unsigned long long>(got));
            return HF_ECHECKSUM;
        }
    }
    return hf::launch_stream(buf, ckpt, nbytes, nullptr, device, st);
}

int hf_checksum(const void* buf, int64_t nbytes, uint64_t* out, int device, void* stream) {
    HF_REQUIRE(out != nullptr, "hf_checksum: NULL out");
    HF_REQUIRE(nbytes >= 0, "hf_checksum: negative size");
    HF_REQUIRE(device >= 0 && device < 64, "hf_checksum: bad device %d", device);
    if (nbytes == 0) {
        *out = 0;
        return HF_OK;
    }
    HF_REQUIRE(buf != nullptr, "hf_checksum: NULL buffer");
    hf::DeviceGuard g(device);
    HF_REQUIRE(g.ok, "hf_checksum: cannot select device %d", device);
    return hf::checksum_impl(nullptr, buf, nbytes, out, device, hf::as_stream(stream));
}

}  // extern "C"
