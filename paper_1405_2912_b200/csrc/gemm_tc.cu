// hf_gemm_tc: tcgen05 kind::tf32 matmul (placeholder until the tcgen05 kernel lands).
#include "common.cuh"
extern "C" int hf_gemm_tc(const float* A, const float* B, float* C, int M, int N, int K, int mode,
                          int device, void* stream) {
    hf::set_error("hf_gemm_tc: not built yet");
    return HF_EUNSUP;
}
