// Fault injection on device buffers (sm_100a).
//
// The host draws the fault schedule with the reference's RNG and draw order
// (/root/reference/pkg/src/hetrt/devices.py:144-160 draw_fault, :207-220
// _corrupt_buffer, :241-247 scribble); the device never
// draws random numbers.  These kernels apply one drawn fault in place on the
// replica's device, ordered on the replica's stream after its kernel body.
#include "common.cuh"

#include <string.h>

namespace hf {

__global__ void bitflip_kernel(uint8_t* buf, long long byte_off, uint8_t mask) {
    buf[byte_off] ^= mask;
}

// devices.py:216-219: float x -> x*(1+rel) in binary64, stored with
// round-to-nearest (numpy float32 assignment); x == 0 -> rel; ints ^ 0x01.
__global__ void scale_kernel(void* buf, int dtype, long long elem, double rel) {
    switch (dtype) {
        case HF_F32: {
            float* p = static_cast<float*>(buf) + elem;
            double x = static_cast<double>(*p);
            double y = x != 0.0 ? x * (1.0 + rel) : rel;
            *p = __double2float_rn(y);
            break;
        }
        case HF_F64: {
            double* p = static_cast<double*>(buf) + elem;
            double x = *p;
            *p = x != 0.0 ? x * (1.0 + rel) : rel;
            break;
        }
        case HF_U8: static_cast<uint8_t*>(buf)[elem] ^= 0x01u; break;
        case HF_U16: static_cast<uint16_t*>(buf)[elem] ^= 0x01u; break;
        case HF_U32: static_cast<uint32_t*>(buf)[elem] ^= 0x01u; break;
        case HF_U64: static_cast<unsigned long long*>(buf)[elem] ^= 0x01ull; break;
    }
}

struct ScribbleBytes {
    uint8_t b[64];
};

__global__ void scribble_kernel(uint8_t* buf, const __grid_constant__ ScribbleBytes bytes, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = bytes.b[i];
}

__global__ void spin_kernel(const volatile int* flag, unsigned long long max_ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        if (flag != nullptr && *flag != 0) return;
        __nanosleep(1000);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < max_ns);
}

static const int kRegistered = register_kernels(
    {(const void*)bitflip_kernel, (const void*)scale_kernel, (const void*)scribble_kernel, (const void*)spin_kernel});

}  // namespace hf

extern "C" {

int hf_debug_spin(const int* flag, int64_t max_ns, int device, void* stream) {
    HF_REQUIRE(max_ns >= 0, "hf_debug_spin: negative duration");
    if (max_ns > 5000000000LL) max_ns = 5000000000LL;
    hf::DeviceGuard g(device);
    HF_REQUIRE(g.ok, "hf_debug_spin: cannot select device %d", device);
    hf::spin_kernel<<<1, 1, 0, hf::as_stream(stream)>>>(flag, static_cast<unsigned long long>(max_ns));
    HF_CHECK_LAUNCH();
    return HF_OK;
}

int hf_inject_bitflip(void* buf, int dtype, int64_t elem, int bit, int device, void* stream) {
    int w = hf::elem_size(dtype);
    HF_REQUIRE(w > 0, "hf_inject_bitflip: unknown dtype %d", dtype);
    HF_REQUIRE(buf != nullptr, "hf_inject_bitflip: NULL buffer");
    HF_REQUIRE(elem >= 0, "hf_inject_bitflip: negative element index");
    HF_REQUIRE(bit >= 0 && bit < 8 * w, "hf_inject_bitflip: bit %d outside [0, %d)", bit, 8 * w);
    hf::DeviceGuard g(device);
    HF_REQUIRE(g.ok, "hf_inject_bitflip: cannot select device %d", device);
    // little-endian: bit b of the element lives in byte b/8
    long long off = static_cast<long long>(elem) * w + bit / 8;
    hf::bitflip_kernel<<<1, 1, 0, hf::as_stream(stream)>>>(static_cast<uint8_t*>(buf), off,
                                                           static_cast<uint8_t>(1u << (bit % 8)));
    HF_CHECK_LAUNCH();
    return HF_OK;
}

int hf_inject_scale(void* buf, int dtype, int64_t elem, double rel, int device, void* stream) {
    HF_REQUIRE(hf::elem_size(dtype) > 0, "hf_inject_scale: unknown dtype %d", dtype);
    HF_REQUIRE(buf != nullptr, "hf_inject_scale: NULL buffer");
    HF_REQUIRE(elem >= 0, "hf_inject_scale: negative element index");
    hf::DeviceGuard g(device);
    HF_REQUIRE(g.ok, "hf_inject_scale: cannot select device %d", device);
    hf::scale_kernel<<<1, 1, 0, hf::as_stream(stream)>>>(buf, dtype, elem, rel);
    HF_CHECK_LAUNCH();
    return HF_OK;
}

int hf_scribble(void* buf, const uint8_t* bytes, int nbytes, int device, void* stream) {
    HF_REQUIRE(nbytes >= 0 && nbytes <= 64, "hf_scribble: size %d outside [0, 64]", nbytes);
    if (nbytes == 0) return HF_OK;
    HF_REQUIRE(buf != nullptr && bytes != nullptr, "hf_scribble: NULL pointer");
    hf::ScribbleBytes sb;
    memset(&sb, 0, sizeof(sb));
    memcpy(sb.b, bytes, static_cast<size_t>(nbytes));
    hf::DeviceGuard g(device);
    HF_REQUIRE(g.ok, "hf_scribble: cannot select device %d", device);
    hf::scribble_kernel<<<1, 64, 0, hf::as_stream(stream)>>>(static_cast<uint8_t*>(buf), sb, nbytes);
    HF_CHECK_LAUNCH();
    return HF_OK;
}

}  // extern "C"
