// normal_eq.cu -- ne_lstsq, the normal-equations baseline.
//
// "computing the Gram matrix G = A^T A, and augmenting the right hand side
// y = A^T b using GeMM and GeMV ... Cholesky factorization (POTRF) G = R^T R ...
// two TRSVs: x = R^-1 (R^-T y)".  Here the Gram of the augmented [A b] is one
// cuBLAS call (DSYRK by default, DGEMM with CSK_NE_GRAM=gemm; R15) when
// b is stored as column n of A, else DSYRK + DGEMV.  The augmented Cholesky
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
    CSK_CUDA_TRY(cudaMallocAsync(&C, 2 * cbytes + 64, st));
    double* Sg = C + (size_t)nc * nc;
    int* sd = reinterpret_cast<int*>(Sg + (size_t)nc * nc);
    const double one = 1.0, zero = 0.0;
    const char* gram = std::getenv("CSK_NE_GRAM");
    const bool use_gemm = gram && std::strcmp(gram, "gemm") == 0;
    cublasStatus_t bs = CUBLAS_STATUS_SUCCESS;
    if (b == A + n * lda) {
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
