// Library-level entry points of libhetft: initialisation, peer access,
// error reporting.  The device model of the reference (simulated units and
// memory spaces, src/hetrt/devices.py:54-62, :126-166, fleets.py:17-36) maps
// onto real CUDA devices here: one memory space per device ordinal, peer
// access enabled all-to-all over NVLink/NVSwitch when requested.
#include "common.cuh"

#include <vector>

#include <mutex>
#include <map>
#include <tuple>
#include <string.h>
#include <stdlib.h>

namespace hf {

static thread_local char g_err[1024] = {0};

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

void clear_error() { g_err[0] = 0; }

static std::mutex g_mu;
static int g_sms[64] = {0};
static int g_peer[64][64] = {{0}};

int num_sms(int device) {
    if (device < 0 || device >= 64) return kNumSMs;
    int v = __atomic_load_n(&g_sms[device], __ATOMIC_ACQUIRE);
    if (v > 0) return v;
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
        sms <= 0)
        sms = kNumSMs;
    __atomic_store_n(&g_sms[device], sms, __ATOMIC_RELEASE);
    return sms;
}

static std::vector<const void*>& kernel_registry() {
    static std::vector<const void*> v;
    return v;
}

int register_kernels(std::initializer_list<const void*> fns) {
    for (const void* f : fns) kernel_registry().push_back(f);
    return 0;
}

void preload_kernels(int device) {
    static int done[64] = {0};
    static std::mutex mu;
    if (device < 0 || device >= 64 || __atomic_load_n(&done[device], __ATOMIC_ACQUIRE)) return;
    std::lock_guard<std::mutex> lk(mu);
    if (done[device]) return;
    typedef int (*FuncLoad)(void*);
    static FuncLoad func_load = nullptr;
    static bool looked_up = false;
    if (!looked_up) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuFuncLoad", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            func_load = reinterpret_cast<FuncLoad>(fn);
        cudaGetLastError();
        looked_up = true;
    }
    for (const void* k : kernel_registry()) {
        cudaFuncAttributes a;
        cudaFuncGetAttributes(&a, k);
        if (func_load) {
            cudaFunction_t f = nullptr;
            if (cudaGetFuncBySymbol(&f, k) == cudaSuccess && f) func_load(f);
        }
    }
    cudaGetLastError();
    __atomic_store_n(&done[device], 1, __ATOMIC_RELEASE);
}

cudaError_t SideStream::fork(cudaStream_t st) {
    cudaError_t e = cudaEventRecord(fork_ev, st);
    return e != cudaSuccess ? e : cudaStreamWaitEvent(stream, fork_ev, 0);
}

cudaError_t SideStream::join(cudaStream_t st) {
    cudaError_t e = cudaEventRecord(join_ev, stream);
    return e != cudaSuccess ? e : cudaStreamWaitEvent(st, join_ev, 0);
}

void SideStream::lock() { static_cast<std::mutex*>(mu)->lock(); }
void SideStream::unlock() { static_cast<std::mutex*>(mu)->unlock(); }

SideStream* side_stream(int device, int level) {
    constexpr int kLevels = 2;
    static SideStream sides[64][kLevels];
    static std::mutex mus[64][kLevels];
    static std::once_flag once[64][kLevels];
    if (device < 0 || device >= 64 || level < 0 || level >= kLevels) return nullptr;
    SideStream* s = &sides[device][level];
    std::call_once(once[device][level], [s, device, level] {
        int least = 0, greatest = 0;
        if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) return;
        int prio = greatest + level;     // greatest is the most negative
        if (prio > least) prio = least;
        s->mu = &mus[device][level];
        if (cudaStreamCreateWithPriority(&s->stream, cudaStreamNonBlocking, prio) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->fork_ev, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->join_ev, cudaEventDisableTiming) != cudaSuccess)
            s->stream = nullptr;
    });
    return s->stream ? s : nullptr;
}

void* stream_scratch(int device, cudaStream_t st, int slot, size_t bytes) {
    struct Buf {
        void* ptr = nullptr;
        size_t bytes = 0;
    };
    static std::mutex mu;
    static std::map<std::tuple<int, cudaStream_t, int>, Buf> bufs;
    std::lock_guard<std::mutex> lk(mu);
    Buf& b = bufs[std::make_tuple(device, st, slot)];
    if (b.bytes < bytes) {
        if (b.ptr) cudaFreeAsync(b.ptr, st);
        b.ptr = nullptr;
        b.bytes = 0;
        if (cudaMallocAsync(&b.ptr, bytes, st) != cudaSuccess) {
            b.ptr = nullptr;
            return nullptr;
        }
        b.bytes = bytes;
    }
    return b.ptr;
}

cudaError_t begin_side_launch(SideStream* side, cudaStream_t st, cudaStream_t* launch_stream) {
    *launch_stream = st;
    if (!side) return cudaSuccess;
    side->lock();
    cudaError_t e = side->fork(st);
    if (e != cudaSuccess) {
        side->unlock();
        return e;
    }
    *launch_stream = side->stream;
    return cudaSuccess;
}

cudaError_t end_side_launch(SideStream* side, cudaStream_t st) {
    cudaError_t e = cudaGetLastError();
    if (side) {
        if (e == cudaSuccess) e = side->join(st);
        side->unlock();
    }
    return e;
}

// HF_PDL=0 launches every PDL-capable kernel the classic way (A/B timing).
bool pdl_enabled() {
    static const int on = getenv("HF_PDL") == nullptr || getenv("HF_PDL")[0] != '0';
    return on != 0;
}

void retain_scratch_pool(int device) {
    static int done[64] = {0};
    if (device < 0 || device >= 64 || __atomic_load_n(&done[device], __ATOMIC_ACQUIRE)) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    __atomic_store_n(&done[device], 1, __ATOMIC_RELEASE);
}

int elem_size(int dtype) {
    switch (dtype) {
        case HF_F32: return 4;
        case HF_F64: return 8;
        case HF_U8: return 1;
        case HF_U16: return 2;
        case HF_U32: return 4;
        case HF_U64: return 8;
        default: return -1;
    }
}

}  // namespace hf

extern "C" {

const char* hf_last_error(void) { return hf::g_err; }

int hf_version(void) { return 1; }

int hf_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int hf_init(int ndev, int enable_peer_all) {
    std::lock_guard<std::mutex> lk(hf::g_mu);
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        hf::set_error("hf_init: no CUDA device available (%s)",
                      e == cudaSuccess ? "count=0" : cudaGetErrorString(e));
        return HF_ENOINIT;
    }
    if (ndev <= 0 || ndev > count) ndev = count;
    if (ndev > 64) ndev = 64;
    int cur = 0;
    cudaGetDevice(&cur);
    for (int d = 0; d < ndev; ++d) {
        hf::num_sms(d);
        hf::g_peer[d][d] = 1;
        if (d == cur) hf::preload_kernels(d);   // other devices: on first use (DeviceGuard)
    }
    if (!enable_peer_all) return HF_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    for (int d = 0; d < ndev; ++d) {
        if (cudaSetDevice(d) != cudaSuccess) continue;
        for (int p = 0; p < ndev; ++p) {
            if (p == d || hf::g_peer[d][p]) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, d, p);
            if (!can) continue;
            cudaError_t pe = cudaDeviceEnablePeerAccess(p, 0);
            if (pe == cudaSuccess || pe == cudaErrorPeerAccessAlreadyEnabled) {
                hf::g_peer[d][p] = 1;
            }
            cudaGetLastError();  // clear "already enabled"
        }
    }
    cudaSetDevice(prev);
    return HF_OK;
}

int hf_peer_enabled(int dev, int peer) {
    if (dev < 0 || peer < 0 || dev >= 64 || peer >= 64) return 0;
    return hf::g_peer[dev][peer];
}

}  // extern "C"
