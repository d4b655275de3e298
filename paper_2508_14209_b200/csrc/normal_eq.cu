// normal_eq.cu -- ne_lstsq, the normal-equations baseline.
//
// "computing the Gram matrix G = A^T A, and augmenting the right hand side
// y = A^T b using GeMM and GeMV ... Cholesky factorization (POTRF) G = R^T R ...
// two TRSVs: x = R^-1 (R^-T y)".  Exactly that: DGEMM for A^T A, DGEMV for A^T b,
// DDOT for b^T b (the fastest cuBLAS form on B200, R15 / 6.3; CSK_NE_GRAM
// selects the alternatives for measurement).  The augmented Cholesky
// [[C11, c12], [c12^T, beta]] = [[R^T, 0], [y^T, rho]] [[R, y], [0, rho]] yields
// y = R^-T c12 for free; one CTA then back-substitutes R x = y.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <cublas_v2.h>

#include "csk_internal.cuh"

namespace csk {

csk_status blas_handle(cudaStream_t st, cublasHandle_t* out);

__global__ void __launch_bounds__(1024, 1) chol_solve_kernel(const double* __restrict__ Cg, int nc, int use_smem,
                                                             double* __restrict__ Sg, double* __restrict__ x,
                                                             int* __restrict__ status) {
    extern __shared__ double csm[];
    __shared__ int s_fail;
    __shared__ double s_r;
    double* S = use_smem ? csm : Sg;
    const int n = nc - 1;
    // symmetric copy from the upper triangle (cuBLAS SYRK fills only the upper part)
    for (int e = threadIdx.x; e < nc * nc; e += blockDim.x) {
        const int i = e % nc, j = e / nc;
        S[e] = i <= j ? Cg[i + (int64_t)j * nc] : Cg[j + (int64_t)i * nc];
    }
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        if (threadIdx.x == 0) {
            const double piv = S[j + (int64_t)j * nc];
            if (!(piv > 0.0)) s_fail = 1;
            s_r = sqrt(piv);
            S[j + (int64_t)j * nc] = s_r;
        }
        __syncthreads();
        if (s_fail) break;
        const double r = s_r;
        for (int c = j + 1 + threadIdx.x; c < nc; c += blockDim.x) S[j + (int64_t)c * nc] /= r;
        __syncthreads();
        // trailing update of the upper triangle: S[i,c] -= R[j,i] R[j,c], j < i <= c
        const int m = nc - j - 1;
        for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
            const int i = j + 1 + e % m, c = j + 1 + e / m;
            if (i <= c) S[i + (int64_t)c * nc] -= S[j + (int64_t)i * nc] * S[j + (int64_t)c * nc];
        }
        __syncthreads();
    }
    if (s_fail) {
        if (threadIdx.x == 0) *status = CSK_ENOTPD;
        return;
    }
    // back substitution R x = y, y = S[0:n, n]
    double* y = S + (int64_t)n * nc;
    for (int c = n - 1; c >= 0; --c) {
        const double xc = y[c] / S[c + (int64_t)c * nc];
        __syncthreads();
        for (int i = threadIdx.x; i < c; i += blockDim.x) y[i] -= S[i + (int64_t)c * nc] * xc;
        if (threadIdx.x == 0) x[c] = xc;
        __syncthreads();
    }
    if (threadIdx.x == 0) *status = 0;
}

// fixed-order sum of the per-block Gram partials (deterministic for a given d)
__global__ void gram_reduce_kernel(const double* __restrict__ W, int64_t parts, int64_t elems, double* __restrict__ C) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < elems; e += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t p = 0; p < parts; ++p) s += W[p * elems + e];
        C[e] = s;
    }
}

// Gram of [A b] split over P row blocks (split-K): strided-batched DGEMMs write one
// nc x nc partial per block (plus one for the ragged tail), then a fixed-order
// reduction.  A single cuBLAS DSYRK/DGEMM with K = d and a 129 x 129 output runs on a
// handful of CTAs (measured 0.2-0.3 s at d = 2^24); this is the strong baseline.
static csk_status gram_split_k(cublasHandle_t h, int64_t d, int n, const double* A, int64_t lda, const double* b,
                               double* C, int nc, cudaStream_t st) {
    const DeviceInfo& di = device_info();
    const int64_t P = std::max<int64_t>(1, std::min<int64_t>(d / 8192, 2 * (int64_t)di.num_sms));
    const int64_t rb = d / P;
    const int64_t tail = d - P * rb;
    const int64_t elems = (int64_t)nc * nc;
    double* W = nullptr;
    CSK_CUDA_TRY(csk_malloc_async(&W, (size_t)(P + 1) * elems * 8, st));
    CSK_CUDA_TRY(cudaMemsetAsync(W, 0, (size_t)(P + 1) * elems * 8, st));
    const double one = 1.0, zero = 0.0;
    const bool fused = b == A + (int64_t)n * lda;
    cublasStatus_t bs = CUBLAS_STATUS_SUCCESS;
    auto batched = [&](int m_, int n_, const double* X, int64_t ldx, const double* Y, int64_t ldy, double* out) {
        if (bs != CUBLAS_STATUS_SUCCESS) return;
        bs = cublasDgemmStridedBatched(h, CUBLAS_OP_T, CUBLAS_OP_N, m_, n_, (int)rb, &one, X, (int)ldx, rb, Y,
                                       (int)ldy, rb, &zero, out, nc, elems, (int)P);
        if (bs == CUBLAS_STATUS_SUCCESS && tail > 0)
            bs = cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, m_, n_, (int)tail, &one, X + P * rb, (int)ldx, Y + P * rb,
                             (int)ldy, &zero, out + P * elems, nc);
    };
    if (fused) {
        batched(nc, nc, A, lda, A, lda, W);
    } else {
        batched(n, n, A, lda, A, lda, W);                          // A^T A
        batched(n, 1, A, lda, b, d, W + (int64_t)n * nc);          // A^T b
        batched(1, 1, b, d, b, d, W + (int64_t)n * nc + n);        // b^T b
    }
    if (bs != CUBLAS_STATUS_SUCCESS) {
        cudaFreeAsync(W, st);
        set_error("cuBLAS batched Gram failed (%d)", (int)bs);
        return CSK_ECUDA;
    }
    gram_reduce_kernel<<<(unsigned)std::min<int64_t>(ceil_div(elems, 256), 1024), 256, 0, st>>>(W, P + 1, elems, C);
    CSK_LAUNCH_CHECK();
    CSK_CUDA_TRY(cudaFreeAsync(W, st));
    return CSK_OK;
}

}  // namespace csk

using namespace csk;

extern "C" csk_status ne_lstsq(int64_t d, int64_t n, const double* A, int64_t lda, const double* b, double* x,
                               void* stream) {
    CSK_REQUIRE(A != nullptr && b != nullptr && x != nullptr, CSK_EINVAL, "A, b, x must be non-NULL");
    CSK_REQUIRE(n >= 1 && n <= 4096, CSK_EINVAL, "n=%lld must be in [1, 4096]", (long long)n);
    CSK_REQUIRE(d >= n && d <= 2147483647LL, CSK_ESHAPE, "d=%lld must be in [n, 2^31-1]", (long long)d);
    CSK_REQUIRE(lda >= d, CSK_ESHAPE, "lda=%lld < d=%lld", (long long)lda, (long long)d);
    CSK_REQUIRE(is_device_pointer(A) && is_device_pointer(b) && is_device_pointer(x), CSK_EINVAL,
                "ne_lstsq takes device pointers");
    cudaStream_t st = (cudaStream_t)stream;
    const int nc = (int)n + 1;
    cublasHandle_t h;
    csk_status s = blas_handle(st, &h);
    if (s != CSK_OK) return s;
    double* C = nullptr;
    const size_t cbytes = (size_t)nc * nc * 8;
    CSK_CUDA_TRY(csk_malloc_async(&C, 2 * cbytes + 64, st));
    double* Sg = C + (size_t)nc * nc;
    int* sd = reinterpret_cast<int*>(Sg + (size_t)nc * nc);
    const double one = 1.0, zero = 0.0;
    // Gram variants (measured on B200 at C2/C4): default = one DGEMM for A^T A
    // (n x n: cuBLAS runs K = d split internally at 28-33 TF/s when n is a multiple of 64) +
    // DGEMV for A^T b + DDOT for b^T b.  "gemm"/"syrk" = one call on [A b] (n+1 columns: the
    // ragged 65th/129th column costs cuBLAS 2-3x), "splitk" = strided-batched DGEMM over row blocks.
    const char* gram = std::getenv("CSK_NE_GRAM");
    const bool use_gemm = gram && std::strcmp(gram, "gemm") == 0;
    const bool use_syrk = gram && std::strcmp(gram, "syrk") == 0;
    const bool use_splitk = gram && std::strcmp(gram, "splitk") == 0;
    cublasStatus_t bs = CUBLAS_STATUS_SUCCESS;
    if (!use_gemm && !use_syrk && !use_splitk) {
        bs = cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)n, (int)n, (int)d, &one, A, (int)lda, A, (int)lda, &zero, C,
                         nc);
        if (bs == CUBLAS_STATUS_SUCCESS)
            bs = cublasDgemv(h, CUBLAS_OP_T, (int)d, (int)n, &one, A, (int)lda, b, 1, &zero, C + (size_t)n * nc, 1);
        if (bs == CUBLAS_STATUS_SUCCESS) {
            cublasSetPointerMode(h, CUBLAS_POINTER_MODE_DEVICE);
            bs = cublasDdot(h, (int)d, b, 1, b, 1, C + (size_t)n * nc + n);
            cublasSetPointerMode(h, CUBLAS_POINTER_MODE_HOST);
        }
    } else if (use_splitk) {
        csk_status gs = gram_split_k(h, d, (int)n, A, lda, b, C, nc, st);
        if (gs != CSK_OK) {
            cudaFreeAsync(C, st);
            return gs;
        }
    } else if (b == A + n * lda) {
        // [A b] is one d x (n+1) column-major matrix
        if (use_gemm)
            bs = cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, nc, nc, (int)d, &one, A, (int)lda, A, (int)lda, &zero, C, nc);
        else
            bs = cublasDsyrk(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, nc, (int)d, &one, A, (int)lda, &zero, C, nc);
    } else {
        if (use_gemm)
            bs = cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)n, (int)n, (int)d, &one, A, (int)lda, A, (int)lda, &zero,
                             C, nc);
        else
            bs = cublasDsyrk(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, (int)n, (int)d, &one, A, (int)lda, &zero, C, nc);
        if (bs == CUBLAS_STATUS_SUCCESS)
            bs = cublasDgemv(h, CUBLAS_OP_T, (int)d, (int)n, &one, A, (int)lda, b, 1, &zero, C + (size_t)n * nc, 1);
        if (bs == CUBLAS_STATUS_SUCCESS) {
            cublasSetPointerMode(h, CUBLAS_POINTER_MODE_DEVICE);
            bs = cublasDdot(h, (int)d, b, 1, b, 1, C + (size_t)n * nc + n);
            cublasSetPointerMode(h, CUBLAS_POINTER_MODE_HOST);
        }
    }
    if (bs != CUBLAS_STATUS_SUCCESS) {
        cudaFreeAsync(C, st);
        set_error("cuBLAS Gram failed (%d)", (int)bs);
        return CSK_ECUDA;
    }
    const DeviceInfo& di = device_info();
    const int use_smem = cbytes <= (size_t)di.smem_optin ? 1 : 0;
    const size_t smem = use_smem ? cbytes : 0;
    CSK_CUDA_TRY(cudaFuncSetAttribute(chol_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    chol_solve_kernel<<<1, 1024, smem, st>>>(C, nc, use_smem, Sg, x, sd);
    CSK_LAUNCH_CHECK();
    int hs = 0;
    CSK_CUDA_TRY(cudaMemcpyAsync(&hs, sd, sizeof(int), cudaMemcpyDeviceToHost, st));
    CSK_CUDA_TRY(cudaFreeAsync(C, st));
    CSK_CUDA_TRY(cudaStreamSynchronize(st));
    if (hs != 0) {
        set_error("normal equations: Cholesky pivot <= 0 (Gram matrix not numerically positive definite)");
        return (csk_status)hs;
    }
    return CSK_OK;
}
