// GPU bodies of the reference's 1-D workloads (/root/reference/pkg/src/hetrt/
// workloads.py:24-58): "inc" (dst = src + 1), "pathfinder-like" (dst[i] =
// a[i] + min(a[i-1], a[i], a[i+1]) with the ends clamped) and the buggy-inc
// variant (inc over the first n-1 elements).  fp32 round-to-nearest adds, and
// numpy's NaN rules (payloads included), so results equal the numpy bodies
// bit for bit.  Grid-stride, one element per thread per step, coalesced.
#include "common.cuh"

namespace hf {

// numpy float32 semantics, payloads included (x86 SSE, numpy 2.x loops):
//   np.minimum(a, b): a if a is NaN, else b if b is NaN (payloads untouched),
//                     else (a < b ? a : b) — so min(+0, -0) = -0, min(-0, +0) = +0
//   np.add(a, b):     quiet(a) if a is NaN, else quiet(b) if b is NaN, else a + b (RN),
//                     an invalid sum (inf + -inf) being 0xFFC00000 as on x86
__device__ __forceinline__ bool is_nan(float x) { return x != x; }
__device__ __forceinline__ float quiet(float x) { return __uint_as_float(__float_as_uint(x) | 0x00400000u); }

__device__ __forceinline__ float np_min(float a, float b) {
    if (is_nan(a)) return a;
    if (is_nan(b)) return b;
    return a < b ? a : b;
}

__device__ __forceinline__ float np_add(float a, float b) {
    if (is_nan(a)) return quiet(a);
    if (is_nan(b)) return quiet(b);
    const float r = __fadd_rn(a, b);
    return is_nan(r) ? __uint_as_float(0xFFC00000u) : r;   // inf + -inf: x86's "real indefinite"
}

__global__ void __launch_bounds__(256) vec_inc_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                                      long long n) {
    pdl_wait();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        dst[i] = np_add(src[i], 1.0f);
}

__global__ void __launch_bounds__(256) vec_path_kernel(const float* __restrict__ a, float* __restrict__ dst,
                                                       long long n) {
    pdl_wait();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const float x = a[i];
        const float l = i > 0 ? a[i - 1] : x;
        const float r = i + 1 < n ? a[i + 1] : x;
        dst[i] = np_add(x, np_min(np_min(l, x), r));
    }
}

static const int kRegistered = register_kernels({(const void*)vec_inc_kernel, (const void*)vec_path_kernel});

static int grid_for(long long n, int device) {
    long long want = (n + 255) / 256;
    long long cap = static_cast<long long>(num_sms(device)) * 8;
    if (want < 1) want = 1;
    return static_cast<int>(want < cap ? want : cap);
}

}  // namespace hf

extern "C" int hf_vec_inc(const float* src, float* dst, int64_t n, int device, void* stream) {
    HF_REQUIRE(n >= 0, "hf_vec_inc: negative n");
    if (n == 0) return HF_OK;
    HF_REQUIRE(src && dst, "hf_vec_inc: NULL buffer");
    hf::DeviceGuard g(device);
    HF_REQUIRE(g.ok, "hf_vec_inc: cannot select device %d", device);
    HF_CUDA_CHECK(hf::launch_pdl(hf::vec_inc_kernel, dim3(hf::grid_for(n, device)), dim3(256), 0,
                                 hf::as_stream(stream), src, dst, static_cast<long long>(n)));
    return HF_OK;
}

extern "C" int hf_vec_path(const float* src, float* dst, int64_t n, int device, void* stream) {
    HF_REQUIRE(n >= 0, "hf_vec_path: negative n");
    if (n == 0) return HF_OK;
    HF_REQUIRE(src && dst, "hf_vec_path: NULL buffer");
    HF_REQUIRE(src != dst, "hf_vec_path: in-place update is not supported");
    hf::DeviceGuard g(device);
    HF_REQUIRE(g.ok, "hf_vec_path: cannot select device %d", device);
    HF_CUDA_CHECK(hf::launch_pdl(hf::vec_path_kernel, dim3(hf::grid_for(n, device)), dim3(256), 0,
                                 hf::as_stream(stream), src, dst, static_cast<long long>(n)));
    return HF_OK;
}
