// csk_internal.cuh -- shared internals of libcsk.so (product side).
// Nothing here is shared with oracle/; the Philox round below is written from
// the generator's definition (Salmon et al. SC'11), R1/R3.
#pragma once

#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>

#include <cublas_v2.h>
#include <cuda_runtime.h>

#include "csk.h"

namespace csk {

// ------------------------------------------------------------------ errors
void set_error(const char* fmt, ...);
const char* last_error();

#define CSK_REQUIRE(cond, status, ...)        \
    do {                                       \
        if (!(cond)) {                         \
            ::csk::set_error(__VA_ARGS__);     \
            return (status);                   \
        }                                      \
    } while (0)

#define CSK_CUDA_TRY(call)                                                                  \
    do {                                                                                    \
        cudaError_t err__ = (call);                                                         \
        if (err__ != cudaSuccess) {                                                         \
            ::csk::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(err__),    \
                             __FILE__, __LINE__);                                           \
            return CSK_ECUDA;                                                               \
        }                                                                                   \
    } while (0)

#define CSK_LAUNCH_CHECK()                                                                  \
    do {                                                                                    \
        ::csk::count_launch();                                                              \
        cudaError_t err__ = cudaGetLastError();                                             \
        if (err__ != cudaSuccess) {                                                         \
            ::csk::set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(err__), \
                             __FILE__, __LINE__);                                           \
            return CSK_ECUDA;                                                               \
        }                                                                                   \
    } while (0)

void count_launch();

// --------------------------------------------------------------- device info
struct DeviceInfo {
    int device = -1;
    int num_sms = 0;
    int smem_optin = 0;      // max dynamic smem per block (bytes)
    int l2_bytes = 0;
    cudaMemPool_t pool = nullptr;   // the library's stream-ordered pool (plan.cu)
};
const DeviceInfo& device_info();   // of the current device

// stream-ordered allocation from the library pool of the current device (freed with cudaFreeAsync)
cudaError_t csk_malloc_async(void** p, size_t bytes, cudaStream_t st);
template <typename T>
inline cudaError_t csk_malloc_async(T** p, size_t bytes, cudaStream_t st) {
    return csk_malloc_async(reinterpret_cast<void**>(p), bytes, st);
}

// -------------------------------------------------------------------- plan
}  // namespace csk

struct csk_plan_s {
    int64_t d = 0, k1 = 0, row0 = 0;
    uint64_t seed = 0;
    int device = -1;
    bool from_arrays = false;
    int32_t* code = nullptr;      // d codes: bucket | sign << 31 (NULL for a CSK_PLAN_HASH plan until needed)
    bool hash = false;            // CSK_PLAN_HASH: kernels may hash rows on the fly
    int64_t* offsets = nullptr;   // k1 + 1 (CSK_PLAN_SORT)
    int32_t* perm = nullptr;      // d      (CSK_PLAN_SORT)
    std::mutex mu;                // guards the Gaussian caches
    std::map<int64_t, double*> gauss64;   // G per k2 (ld round_up(k2, 8), tail padded)
};

namespace csk {

// ------------------------------------------------------------- Philox4x32-10
__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    return __umulhi(a, b);
#else
    return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

__host__ __device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k.x += 0x9E3779B9u;
            k.y += 0xBB67AE85u;
        }
        const uint32_t hi0 = mulhi32(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = mulhi32(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

// code of GLOBAL row g (R3): word g & 3 of Philox(ctr = (lo32(g>>2), hi32(g>>2), 0, 0), key = seed),
// bucket = mulhi(w, k1), sign bit = w & 1 -- the same function codes_kernel stores
__device__ __forceinline__ uint4 hash_block(uint64_t g, uint32_t key0, uint32_t key1) {
    const uint64_t q = g >> 2;
    return philox4x32_10(make_uint4((uint32_t)q, (uint32_t)(q >> 32), 0u, 0u), make_uint2(key0, key1));
}
__device__ __forceinline__ uint32_t code_from_word(uint32_t w, uint32_t k1) {
    return __umulhi(w, k1) | ((w & 1u) << 31);
}

// code word: bucket in bits 0..30, sign (1 = negative) in bit 31
__host__ __device__ __forceinline__ uint32_t code_bucket(uint32_t code) { return code & 0x7fffffffu; }
__host__ __device__ __forceinline__ uint64_t code_sign_mask64(uint32_t code) {
    return (uint64_t)(code & 0x80000000u) << 32;
}
__host__ __device__ __forceinline__ uint32_t code_sign_mask32(uint32_t code) { return code & 0x80000000u; }

__device__ __forceinline__ double apply_sign(double v, uint32_t code) {
    return __longlong_as_double(__double_as_longlong(v) ^ (long long)code_sign_mask64(code));
}
__device__ __forceinline__ float apply_sign(float v, uint32_t code) {
    return __int_as_float(__float_as_int(v) ^ (int)code_sign_mask32(code));
}

// ------------------------------------------------------------ launch helpers
// runs f on scope exit (every return path releases streams, events and workspaces)
template <typename F>
struct ScopeExit {
    F f;
    ~ScopeExit() { f(); }
};
template <typename F>
ScopeExit<F> on_exit(F f) {
    return ScopeExit<F>{f};
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// validated column-pointer table for [A b]: column c < n is A + c*lda, column n is b
template <typename T>
struct Cols {
    const T* A;
    const T* b;
    int64_t lda;
    int n;
    __device__ __forceinline__ const T* col(int c) const { return c < n ? A + (int64_t)c * lda : b; }
};

// plan.cu: materialise the codes of a CSK_PLAN_HASH plan (no-op when present)
csk_status ensure_codes(csk_plan_t plan, cudaStream_t st);

// mbarrier + 1-D bulk copy (TMA) helpers, shared by the CountSketch and SRHT kernels
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
        : "memory");
}

// cs_apply implementation entry (countsketch.cu), also used by ms_apply
// RowOut (nullable): when the row-scatter variants ran, hand the caller the row-major SA^T workspace
// instead of transposing it (the caller cudaFreeAsync's rowout->ws): element (m, c) at
// (c / cw) * cs + m * lc + (c % cw).  rowout->ws == NULL means SA was written as usual.
struct RowOut {
    double* ws = nullptr;
    int cw = 0, ncols = 0;
    int64_t lc = 0, cs = 0;
};
// multisketch.cu: column-major fp64 SA (ld) -> a new regular row-major workspace described by *ro
csk_status rows_from_colmajor(const double* SA, int64_t ld, int64_t k1, int ncols, RowOut* ro, cudaStream_t st);
// With rowout != NULL the result is ALWAYS handed over as an fp64 row-major workspace (SA may be NULL);
// the caller cudaFreeAsync's rowout->ws.
csk_status cs_apply_impl(csk_plan_t plan, csk_dtype dtype, int64_t n, const void* A, int64_t lda,
                         const void* b, void* SA, int64_t ldsa, int variant, cudaStream_t st,
                         int64_t row_begin, int64_t row_end, bool accumulate, RowOut* rowout = nullptr);
// the plan's cached G (k2 x k1, fp64, column-major with ld *ldg = round_up(k2, 8), rows past k2 zero,
// followed by kGstageTailPad zero doubles so 128-row tiles may read past the last column)
constexpr int kGstageTailPad = 256;
csk_status gauss_get(csk_plan_t plan, int64_t k2, cudaStream_t st, const double** G, int64_t* ldg);
// gstage.cu: Z (k2 x ro.ncols, column-major ldz, fp64 or fp32) = G Y with Y^T the row-major workspace
// described by ro (chunks of <= kGstageMaxCw columns), hand-written fp64 DMMA (a5)
constexpr int kGstageMaxCw = 72;
csk_status gstage_launch(const double* G, int64_t ldg, int64_t k2, int64_t k1, const RowOut& ro, void* Z,
                         int64_t ldz, bool z_f32, cudaStream_t st);
struct cublasContext;
csk_status blas_handle(cudaStream_t st, struct cublasContext** h);

bool is_device_pointer(const void* p);

// small-solve status written by the solve kernels (multisketch.cu, qr_wy.cu)
struct SolveStatus {
    int status;
    double sk_resid;
};
csk_status qr_wy_launch(const double* Z, int64_t ldz, int m, int nc, double* Rg, int ldr, double* scratch,
                        double* x, SolveStatus* status, cudaStream_t st, bool* launched);
size_t qr_wy_scratch_doubles(int m, int nc);
// multisketch.cu: Z = G S [A b] (ms_apply) and the sketched QR solve (ms_solve).  solve_impl
// optionally exports R (nc x nc upper, ld nc, device) for rand_cholQR's R0.
csk_status ms_apply_impl(csk_plan_t plan, int64_t k2, csk_dtype dtype, int64_t n, const void* A, int64_t lda,
                         const void* b, void* Z, int64_t ldz, cudaStream_t st);
csk_status solve_impl(int64_t k2, int64_t n, const double* Z, int64_t ldz, double* x, double* sk_resid,
                      cudaStream_t st, bool x_host, double* R_out,
                      int32_t* status_dev = nullptr, double* resid_dev = nullptr);
csk_status blas_handle(cudaStream_t st, cublasHandle_t* out);
// multisketch.cu: N(0,1) pairs of Philox stream 1 divided by div, starting at pair t_off
template <typename T>
__global__ void gauss_kernel(T* __restrict__ G, int64_t total, double div, uint32_t key_lo, uint32_t key_hi,
                             int64_t t_off);
// randcholqr.cu: x = R0^-1 u (+ R = R1 R0 when R != NULL), one CTA; skipped if *chol_status != 0
__global__ void __launch_bounds__(1024, 1) rc_finish_kernel(const double* __restrict__ R0, int ldr0,
                                                            const double* __restrict__ S, int nc, int n,
                                                            const double* __restrict__ u, double* __restrict__ x,
                                                            double* __restrict__ R, int ldr,
                                                            const int* __restrict__ chol_status);
// srht.cu
csk_status srht_impl(int64_t d, int64_t dglob, int64_t row0, int64_t k, uint64_t seed, int64_t n, const double* A,
                     int64_t lda, const double* b, double* Y, int64_t ldy, cudaStream_t st);
// normal_eq.cu: upper Cholesky of the augmented Gram C (nc x nc, upper part read) in S (ld nc);
// x = R^-1 R^-T C[:n, n]; *status = CSK_ENOTPD on a non-positive pivot.
__global__ void __launch_bounds__(1024, 1) chol_solve_kernel(const double* __restrict__ Cg, int nc, int use_smem,
                                                             double* __restrict__ Sg,
                                  double* __restrict__ x, int* __restrict__ status);

}  // namespace csk
