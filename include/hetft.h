/*
 * hetft.h — C-ABI of libhetft.so, the B200 (sm_100a) hot path of the
 * heterogeneity-aware fault-tolerant runtime of arXiv 1405.2912.
 *
 * Every entry point takes plain pointers and sizes; no torch or C++ types
 * cross this boundary.  Device buffers are allocated by the caller (PyTorch
 * in the Python drop-in) and passed as raw device pointers; `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).
 *
 * Return codes: 0 on success, < 0 on error (see HF_E*).  hf_last_error()
 * returns a thread-local message describing the most recent failure.  The
 * Python drop-in maps HF_EINVAL onto DispatchError (reference
 * src/hetrt/errors.py:33-35) and HF_ECUDA onto the `api_error` fault class
 * (reference src/hetrt/devices.py:23-27).
 *
 * Reference interfaces each group replaces (paths relative to
 * /root/reference/pkg):
 *   hf_vote*            src/hetrt/voting.py:68-123 (_compare_floats,
 *                       compare_payloads, compare), generalised to K replicas
 *                       (SURVEY.md Appendix A); called from
 *                       src/hetrt/executor.py:312-336 (Executor._vote)
 *   hf_copy / hf_checkpoint / hf_restore / hf_checksum
 *                       src/hetrt/memory.py:136-189 (payload copies of
 *                       _request_read/_request_write/_maybe_checkpoint)
 *   hf_inject_scale     src/hetrt/devices.py:207-220 (_corrupt_buffer)
 *   hf_inject_bitflip   new: the north-star "seeded single bit-flip" mode
 *   hf_scribble         src/hetrt/devices.py:241-247 (abort/api_error scribble)
 *   hf_gemm_tc / hf_gemm_simt
 *                       the kernel-variant slot of src/hetrt/api.py:131-138
 *                       (attach_kernel) — the paper's diverse CUDA/OpenMP pair
 */
#ifndef HETFT_H
#define HETFT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------- */
#define HF_OK        0
#define HF_EINVAL   -1   /* bad arguments (-> DispatchError)              */
#define HF_ECUDA    -2   /* CUDA runtime/driver error (-> api_error)       */
#define HF_ENOINIT  -3   /* library not initialised / device unavailable   */
#define HF_EUNSUP   -4   /* unsupported shape/alignment for this kernel    */

/* ---- element types (ValueType x element width) ------------------------ */
#define HF_F32    0      /* ValueType.FLOAT32                               */
#define HF_F64    1      /* ValueType.FLOAT64                               */
#define HF_U8     2      /* ValueType.INT, width 1                          */
#define HF_U16    3      /* ValueType.INT, width 2                          */
#define HF_U32    4      /* ValueType.INT, width 4                          */
#define HF_U64    5      /* ValueType.INT, width 8                          */

#define HF_MAX_K  8      /* max replicas per vote                           */

/* vote verdicts (rule 5) */
#define HF_VERDICT_MATCH      0  /* every replica agrees with the voted value */
#define HF_VERDICT_CORRECTED  1  /* a majority exists everywhere; some replica differs */
#define HF_VERDICT_MISMATCH   2  /* >=1 element without a majority: rerun  */

/* GEMM modes (hf_gemm_tc; hf_gemm_simt takes only the COSCHEDULE flag) */
#define HF_GEMM_TF32     0   /* single-pass kind::tf32                       */
#define HF_GEMM_3XTF32   1   /* error-compensated big+small split (3 passes) */
#define HF_GEMM_3XBF16   2   /* the same split on bf16 halves, kind::f16 (2x rate) */
#define HF_GEMM_COSCHEDULE 0x100 /* flag: launch shapes that share SMs with a
                                    concurrent replica of the other variant:
                                    TC 2 stages, 1 tile/CTA, operand pre-pass on
                                    a high-priority side stream; SIMT a 100 KB
                                    smem reservation per CTA */

/* Result of one K-replica vote.  Plain POD; identical layout on host and
 * device (the async entry points write it in device memory). */
typedef struct hf_vote_result {
    int64_t mismatch[HF_MAX_K]; /* per replica: #elements where it disagrees
                                   with the voted value, or unresolved      */
    int64_t unresolved;         /* #elements with no majority               */
    int64_t first_div;          /* lowest element index with any disagreement,
                                   -1 if none                               */
    int32_t winner;             /* argmin mismatch, ties -> lowest index     */
    int32_t verdict;            /* HF_VERDICT_*                              */
    int32_t K;
    int32_t reserved;
    uint64_t first_raw0;        /* K >= 3: replica 0's raw element bits at
                                   first_div as read, before an in-place vote
                                   stored over it; 0 if none, K = 2 or
                                   arbitrary widths                         */
    int64_t  kernel_ns;         /* the vote kernel's own device time: earliest
                                   CTA start (after its stream dependency) to
                                   the last CTA's finalisation, %globaltimer;
                                   0 for arbitrary widths                   */
} hf_vote_result;

/* ---- library -------------------------------------------------------- */
int         hf_init(int ndev, int enable_peer_all);
const char* hf_last_error(void);
int         hf_version(void);
int         hf_device_count(void);
/* 1 if device `dev` can load from device `peer`'s memory (after hf_init
 * with enable_peer_all). */
int         hf_peer_enabled(int dev, int peer);

/* ---- voter ------------------------------------------------------------
 * replicas : host array of K device pointers (may be peer-device pointers
 *            when peer access is enabled; the kernel loads them directly)
 * n        : elements per replica
 * rel_tol  : host array [K], per-replica (per-variant) relative tolerance δ;
 *            a pair (r,s) uses max(δ_r, δ_s).  Ignored for integer dtypes.
 * ulp_tol  : host array [K] or NULL; a float pair also agrees when its
 *            ordered-integer distance is <= max(u_r, u_s) (never across NaN)
 * voted    : device buffer of n elements (may be NULL: no voted output)
 * out      : host result
 * Synchronous: returns after the result is on the host. */
int hf_vote(const void* const* replicas, int K, int64_t n, int dtype,
            const double* rel_tol, const int32_t* ulp_tol,
            void* voted, hf_vote_result* out, int device, void* stream);

/* Asynchronous variant: writes the result to `dev_out` and returns without
 * synchronising.  `dev_out` may be device memory or pinned host memory
 * (device-visible through UVA): then the last CTA stores the 112-byte result
 * straight over the bus and no separate read-back copy is needed.  `workspace` is caller-owned device memory
 * of hf_vote_workspace_bytes() bytes initialised once with
 * hf_vote_workspace_init(); the kernel leaves it re-initialised, so one
 * workspace serves any number of back-to-back votes on one stream.
 * n = 0 is legal here and in hf_vote_batch items (one block writes a match
 * result with first_div = -1, as the reference compares empty payloads). */
int64_t hf_vote_workspace_bytes(void);
int hf_vote_workspace_init(void* workspace, int device, void* stream);
int hf_vote_async(const void* const* replicas, int K, int64_t n, int dtype,
                  const double* rel_tol, const int32_t* ulp_tol,
                  void* voted, hf_vote_result* dev_out, void* workspace,
                  int device, void* stream);

/* Several votes in one launch: `count` items (any number; launched in
 * groups of HF_VOTE_BATCH_MAX) sharing K, dtype and tolerances, each with
 * its own replicas, size, optional voted buffer (== replicas[0]: in place),
 * result (device or pinned host memory) and workspace (as for
 * hf_vote_async; one per item in flight).  Asynchronous.  Small votes are
 * bound by the per-launch host cost and each grid's ramp and tail; one
 * shared grid amortises both (e.g. every output area of a task, or the
 * votes of several tasks). */
#define HF_VOTE_BATCH_MAX 32
typedef struct hf_vote_item {
    const void* replicas[HF_MAX_K];
    int64_t n;
    void* voted;
    hf_vote_result* out;
    void* workspace;
} hf_vote_item;
int hf_vote_batch(const hf_vote_item* items, int count, int K, int dtype,
                  const double* rel_tol, const int32_t* ulp_tol,
                  int device, void* stream);

/* Integer areas of arbitrary element width (ValueType.INT, any width):
 * elements agree iff all `elem_width` bytes are equal. */
int hf_vote_bytes(const void* const* replicas, int K, int64_t n, int elem_width,
                  void* voted, hf_vote_result* out, int device, void* stream);

/* ---- copy / checkpoint -------------------------------------------------- */
/* dst on dst_dev, src on src_dev (either may be -1 = pinned/registered host
 * memory).  Same device: vectorised copy kernel.  Different devices with
 * peer access: copy kernel on dst_dev pulling over NVLink.  Otherwise the
 * copy engine (cudaMemcpyPeerAsync / cudaMemcpyAsync). Asynchronous. */
int hf_copy(void* dst, int dst_dev, const void* src, int src_dev,
            int64_t nbytes, void* stream);

/* Fill nbytes of dst (device `device`, or pinned host when device < 0)
 * with byte `value` (provisional write buffers start zeroed, as the
 * reference's bytearray(n) does, memory.py:168). Asynchronous. */
int hf_fill(void* dst, int value, int64_t nbytes, int device, void* stream);

/* Snapshot `buf` into `ckpt` (same device or a peer pointer). If checksum is
 * non-NULL the copy is fused with the position-sensitive 64-bit checksum of
 * the bytes (see hf_checksum) and the call synchronises to return it. */
int hf_checkpoint(void* ckpt, const void* buf, int64_t nbytes,
                  uint64_t* checksum, int device, void* stream);
/* Restore `buf` from `ckpt`; optional verification against `expect`
 * (NULL = no verification).  Returns HF_EINVAL-class -5 on mismatch. */
#define HF_ECHECKSUM -5
int hf_restore(void* buf, const void* ckpt, int64_t nbytes,
               const uint64_t* expect, int device, void* stream);
/* Checksum only (synchronous). */
int hf_checksum(const void* buf, int64_t nbytes, uint64_t* out,
                int device, void* stream);

/* ---- fault injection ----------------------------------------------------- */
/* XOR bit `bit` (0 = LSB) of element `elem` of a buffer of `dtype`. */
int hf_inject_bitflip(void* buf, int dtype, int64_t elem, int bit,
                      int device, void* stream);
/* Reference corruption semantics (devices.py:207-220): floats become
 * x*(1+rel) computed in binary64 and stored with round-to-nearest (or `rel`
 * when x == 0); integers are XORed with 0x01. */
int hf_inject_scale(void* buf, int dtype, int64_t elem, double rel,
                    int device, void* stream);
/* Overwrite the first nbytes (<= 64) bytes of buf with host `bytes`: the
 * abort/api_error scribble of devices.py:241-247 (8 random bytes for float
 * areas; up to 8 random *elements* for typed INT views, i.e. <= 64 bytes). */
int hf_scribble(void* buf, const uint8_t* bytes, int nbytes,
                int device, void* stream);

/* ---- test support ------------------------------------------------------- */
/* A one-thread kernel that spins until *flag != 0 (device or mapped host
 * memory) or for max_ns nanoseconds of %globaltimer, whichever comes first
 * (max_ns is capped at 5 s).  It stands in for a hung replica kernel when
 * testing the executor's stream watchdog; it can never hang the GPU. */
int hf_debug_spin(const int* flag, int64_t max_ns, int device, void* stream);

/* ---- matmul kernel variants (row-major fp32, C = A·B) -------------------- */
/* tcgen05.mma kind::tf32 with TMA-fed, 128B-swizzled smem and TMEM
 * accumulators (CTA pairs, cta_group::2, when standalone).  Any M, N, K >= 1
 * with N % 4 == 0, K % 4 == 0 and 16-byte aligned operands (TMA); ragged
 * tiles are zero-filled by TMA and stored masked.  mode: HF_GEMM_TF32,
 * HF_GEMM_3XTF32 or HF_GEMM_3XBF16, optionally | HF_GEMM_COSCHEDULE. */
int hf_gemm_tc(const float* A, const float* B, float* C, int M, int N, int K,
               int mode, int device, void* stream);
/* Register-tiled FP32 FFMA (no tensor cores). Any M, N, K >= 1.
 * mode: 0 or HF_GEMM_COSCHEDULE. */
int hf_gemm_simt(const float* A, const float* B, float* C, int M, int N, int K,
                 int mode, int device, void* stream);

/* ---- GPU bodies of the reference's 1-D workloads ------------------------- */
/* src/hetrt/workloads.py:24-28 (inc; buggy-inc = inc over n-1 elements,
 * :53-58): dst[i] = src[i] + 1.0f. */
int hf_vec_inc(const float* src, float* dst, int64_t n, int device, void* stream);
/* src/hetrt/workloads.py:35-42 (pathfinder-like): dst[i] = a[i] +
 * min(a[i-1], a[i], a[i+1]) with the ends clamped, np.minimum NaN rules.
 * src and dst must not alias. */
int hf_vec_path(const float* src, float* dst, int64_t n, int device, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HETFT_H */
