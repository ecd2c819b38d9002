// Shared helpers for libhetft (sm_100a).  Error plumbing for the C-ABI,
// stream/device guards and small device utilities.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include "../../include/hetft.h"

#include <initializer_list>

namespace hf {

// Thread-local last-error message (hf_last_error).
void set_error(const char* fmt, ...);
void clear_error();

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs (queried at init; this is the default)
int num_sms(int device);
// Keep stream-ordered scratch (cudaMallocAsync) cached in the device's
// default pool between calls instead of returning it at every sync.
void retain_scratch_pool(int device);
// High-priority side streams for the operand pre-passes of co-scheduled
// GEMM replicas (HF_GEMM_COSCHEDULE).  level 0 = the device's greatest
// stream priority, level 1 = the next one down.  fork() makes the side
// stream wait for `st`'s pending work; join() makes `st` wait for what was
// launched on the side stream.  The caller holds `mu` between the two so
// concurrent callers cannot interleave their event record/wait pairs.
struct SideStream {
    cudaStream_t stream = nullptr;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    void* mu = nullptr;   // std::mutex (kept out of this header)
    cudaError_t fork(cudaStream_t st);
    cudaError_t join(cudaStream_t st);
    void lock();
    void unlock();
};
SideStream* side_stream(int device, int level);

// Stream-ordered scratch owned per (device, stream, slot): reused by every
// later call on the same stream (stream order makes reuse safe), grown with
// cudaMallocAsync/cudaFreeAsync on that stream when a call needs more.  Saves
// the per-call allocate/free pair of the GEMM pre-passes.  Never freed (the
// process owns a few per unit stream).  Returns nullptr on failure.  Calls
// that share a stream must come from one host thread at a time (the runtime
// launches each unit stream from its dispatcher thread), since a growth frees
// the old block in stream order.
void* stream_scratch(int device, cudaStream_t st, int slot, size_t bytes);
// begin: lock + fork, *launch_stream = side stream (or `st` when side is
// NULL).  end: check the launches, join back into `st`, unlock.  Both return
// the first CUDA error; end always unlocks.
cudaError_t begin_side_launch(SideStream* side, cudaStream_t st, cudaStream_t* launch_stream);
cudaError_t end_side_launch(SideStream* side, cudaStream_t st);

// Every __global__ of the library registers itself (static initialiser) so
// hf_init can load them all up front: with CUDA's lazy module loading the
// first launch of a kernel may wait for the device to go idle, which would
// stall a replica behind an unrelated long-running one (and defeat the
// executor's watchdog).
int register_kernels(std::initializer_list<const void*> fns);
void preload_kernels(int device);

// RAII device guard: switches the calling thread's current device and
// restores it on scope exit.
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    bool switched = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (dev >= 0 && dev != prev) {
            ok = cudaSetDevice(dev) == cudaSuccess;
            switched = ok;
        }
        if (ok) preload_kernels(dev >= 0 ? dev : (prev >= 0 ? prev : 0));
    }
    ~DeviceGuard() {
        // restore only what was changed: every C-ABI call takes a guard, and
        // the common case (already on the right device) then costs one query
        if (switched && prev >= 0) cudaSetDevice(prev);
    }
};

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int elem_size(int dtype);  // bytes per element or -1

// Launch with programmatic stream serialisation (PDL): the grid may become
// resident while the stream's previous kernel drains; the kernel itself must
// execute griddepcontrol.wait before touching memory that kernel produced.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    if (!pdl_enabled()) {
        kernel<<<grid, block, smem, st>>>(static_cast<KArgs>(args)...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace hf

#define HF_CUDA_CHECK(expr)                                                        \
    do {                                                                           \
        cudaError_t _e = (expr);                                                   \
        if (_e != cudaSuccess) {                                                   \
            hf::set_error("%s:%d: %s -> %s", __FILE__, __LINE__, #expr,            \
                          cudaGetErrorString(_e));                                 \
            return HF_ECUDA;                                                       \
        }                                                                          \
    } while (0)

#define HF_CHECK_LAUNCH()                                                          \
    do {                                                                           \
        cudaError_t _e = cudaGetLastError();                                       \
        if (_e != cudaSuccess) {                                                   \
            hf::set_error("%s:%d: kernel launch failed: %s", __FILE__, __LINE__,   \
                          cudaGetErrorString(_e));                                 \
            return HF_ECUDA;                                                       \
        }                                                                          \
    } while (0)

#define HF_REQUIRE(cond, ...)                                                      \
    do {                                                                           \
        if (!(cond)) {                                                             \
            hf::set_error(__VA_ARGS__);                                            \
            return HF_EINVAL;                                                      \
        }                                                                          \
    } while (0)

// ---- device utilities ----------------------------------------------------
namespace hf {

// Global nanosecond timer (same clock on every SM).
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// PDL: wait for the previous grid of the stream (no-op without PDL launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// PDL: let the stream's next grid start launching.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Load rule for source buffers (replicas, copy sources, snapshots): a
// buffer the kernel only reads is read-only for the kernel's lifetime — its
// producers (another stream, another GPU, the host) are ordered before the
// launch by events — so it is loaded with ld.global.nc whether it is local
// HBM, a peer GPU's memory (NVLink) or mapped pinned host memory (UVA).  A
// buffer the same kernel also stores into (the in-place vote target) is
// loaded coherently with ld_stream_rw.
// 128-bit streaming load that does not allocate in L1 (read-once data).
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// 128-bit coherent streaming load (no .nc, no L1 allocation): for a buffer
// the kernel itself writes (in-place vote target).
__device__ __forceinline__ uint4 ld_stream_rw(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// 128-bit streaming store (evict-first: written once, not re-read soon).
__device__ __forceinline__ void st_stream(uint4* p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

}  // namespace hf
