// sketch_solve.cu -- the other sketch-and-solve operators of the paper's least-squares study
// (Fig 5 bars; future work P:L389):
//   gs_apply / gs_lstsq    Gaussian sketch S = G (k x d, N(0, 1/k)), applied by row chunks:
//                          each chunk's G slice is generated on the fly (Philox stream 1, element
//                          e = r + row*k, the same stream as the multisketch's G) and multiplied in
//                          with DGEMM, so the k x d matrix that ran the paper's H100 out of memory
//                           is never materialised.
//   cs_lstsq               CountSketch-only sketch-and-solve: QR of the k1 x (n+1) sketch with
//                          cuSOLVER GEQRF (the paper's GeQRF; "it must perform GeQRF on a
//                          larger problem"), back substitution on the GPU.
//   msh_apply / msh_lstsq  Count+SRHT multisketch: Z = SRHT_k2 (S1 [A b]), k1 a power of two.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>

#include <cusolverDn.h>

#include "csk_internal.cuh"

namespace csk {

static csk_status solver_handle(cudaStream_t st, cusolverDnHandle_t* out) {
    static thread_local std::map<int, cusolverDnHandle_t> handles;
    int dev = 0;
    CSK_CUDA_TRY(cudaGetDevice(&dev));
    auto it = handles.find(dev);
    if (it == handles.end()) {
        cusolverDnHandle_t h = nullptr;
        CSK_REQUIRE(cusolverDnCreate(&h) == CUSOLVER_STATUS_SUCCESS, CSK_ECUDA, "cusolverDnCreate failed");
        it = handles.emplace(dev, h).first;
    }
    CSK_REQUIRE(cusolverDnSetStream(it->second, st) == CUSOLVER_STATUS_SUCCESS, CSK_ECUDA, "cusolverDnSetStream failed");
    *out = it->second;
    return CSK_OK;
}

// Z (k x ncols) = G[:, row0 .. row0+d) [A b]
static csk_status gs_apply_impl(int64_t d, int64_t row0, int64_t k, uint64_t seed, int64_t n, const double* A,
                                int64_t lda, const double* b, double* Z, int64_t ldz, cudaStream_t st) {
    const int64_t ncols = n + (b ? 1 : 0);
    CSK_REQUIRE(d >= 1 && k >= 2 && n >= 0 && ncols >= 1 && Z != nullptr, CSK_EINVAL, "bad Gaussian sketch arguments");
    CSK_REQUIRE((k & 1) == 0, CSK_EINVAL, "k=%lld must be even (Box-Muller pairs per row)", (long long)k);
    CSK_REQUIRE(row0 >= 0, CSK_EINVAL, "row0 < 0");
    CSK_REQUIRE(n == 0 || (A != nullptr && lda >= d), CSK_ESHAPE, "A NULL or lda < d");
    CSK_REQUIRE(ldz >= k, CSK_ESHAPE, "ldz=%lld < k=%lld", (long long)ldz, (long long)k);
    CSK_REQUIRE(k <= 1 << 16 && d <= 2147483647LL, CSK_EINVAL, "k or d out of range");
    CSK_REQUIRE((n == 0 || is_device_pointer(A)) && (!b || is_device_pointer(b)) && is_device_pointer(Z), CSK_EINVAL,
                "gs_apply takes device pointers");
    cublasHandle_t h;
    csk_status s = blas_handle(st, &h);
    if (s != CSK_OK) return s;
    // chunk: the G slice (k x mc doubles) is 1/4 of L2, so it is consumed from L2 by the GEMM.
    // Two slices alternate: chunk i+1's Gaussians are generated on a second stream (fp64 ALU:
    // log, sqrt, sincospi) while chunk i's GEMM runs (fp64 DMMA), ordered by events.
    int64_t mc = std::max<int64_t>(256, (int64_t)device_info().l2_bytes / 4 / (8 * k));
    if (const char* e = std::getenv("CSK_GS_CHUNK")) mc = std::max<int64_t>(2, std::atoll(e));
    mc = std::min(mc, d);
    double* G = nullptr;
    cudaStream_t gen = nullptr;
    cudaEvent_t ev[5] = {};
    // every generated slice is waited on by st before its GEMM, so freeing G on st is ordered after
    // the generator's writes; the stream and events are released once their pending work completes
    auto cleanup = on_exit([&] {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (gen) cudaStreamDestroy(gen);
        if (G) cudaFreeAsync(G, st);
    });
    CSK_CUDA_TRY(csk_malloc_async(&G, 2 * (size_t)k * mc * 8, st));
    CSK_CUDA_TRY(cudaStreamCreateWithFlags(&gen, cudaStreamNonBlocking));
    for (auto& e : ev) CSK_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    // ev[0]: G allocated (st); ev[1 + s]: slice s generated (gen); ev[3 + s]: slice s consumed (st)
    CSK_CUDA_TRY(cudaEventRecord(ev[0], st));
    CSK_CUDA_TRY(cudaStreamWaitEvent(gen, ev[0], 0));
    const double one = 1.0, zero = 0.0, div = std::sqrt((double)k);
    cublasStatus_t bs = CUBLAS_STATUS_SUCCESS;
    auto generate = [&](int64_t c0, int slot) -> csk_status {
        const int64_t m = std::min(mc, d - c0);
        const int64_t total = k * m;
        const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(total / 2, 256), 148 * 16);
        gauss_kernel<double><<<grid, 256, 0, gen>>>(G + (size_t)slot * k * mc, total, div, (uint32_t)seed,
                                                    (uint32_t)(seed >> 32), (row0 + c0) * (k / 2));
        CSK_LAUNCH_CHECK();
        CSK_CUDA_TRY(cudaEventRecord(ev[1 + slot], gen));
        return CSK_OK;
    };
    csk_status gs_st = generate(0, 0);
    int64_t it = 0;
    for (int64_t c0 = 0; gs_st == CSK_OK && c0 < d && bs == CUBLAS_STATUS_SUCCESS; c0 += mc, ++it) {
        const int slot = (int)(it & 1);
        const int64_t m = std::min(mc, d - c0);
        if (c0 + mc < d) {   // next slice on the generator stream, once its previous GEMM is done
            if (it >= 1) CSK_CUDA_TRY(cudaStreamWaitEvent(gen, ev[3 + (slot ^ 1)], 0));
            gs_st = generate(c0 + mc, slot ^ 1);
        }
        CSK_CUDA_TRY(cudaStreamWaitEvent(st, ev[1 + slot], 0));
        const double* Gs = G + (size_t)slot * k * mc;
        const double* beta = c0 == 0 ? &zero : &one;
        if (n > 0)
            bs = cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)k, (int)n, (int)m, &one, Gs, (int)k, A + c0, (int)lda,
                             beta, Z, (int)ldz);
        if (b && bs == CUBLAS_STATUS_SUCCESS)
            bs = cublasDgemv(h, CUBLAS_OP_N, (int)k, (int)m, &one, Gs, (int)k, b + c0, 1, beta, Z + (size_t)n * ldz, 1);
        CSK_CUDA_TRY(cudaEventRecord(ev[3 + slot], st));
    }
    if (gs_st != CSK_OK) return gs_st;
    if (bs != CUBLAS_STATUS_SUCCESS) {
        set_error("cuBLAS Gaussian sketch failed (%d)", (int)bs);
        return CSK_ECUDA;
    }
    return CSK_OK;
}

// Z (k2 x ncols) = SRHT_k2 (S1 [A b]) (Count+SRHT multisketch, seed = the plan's)
static csk_status msh_apply_impl(csk_plan_t plan, int64_t k2, int64_t n, const double* A, int64_t lda, const double* b,
                                 double* Z, int64_t ldz, cudaStream_t st) {
    CSK_REQUIRE(plan != nullptr, CSK_EINVAL, "plan is NULL");
    const int64_t k1 = plan->k1, ncols = n + (b ? 1 : 0);
    CSK_REQUIRE((k1 & (k1 - 1)) == 0, CSK_ESHAPE, "Count+SRHT needs k1=%lld a power of two", (long long)k1);
    CSK_REQUIRE(ncols >= 1 && Z != nullptr, CSK_EINVAL, "bad arguments");
    double* SA = nullptr;
    CSK_CUDA_TRY(csk_malloc_async(&SA, (size_t)k1 * ncols * 8, st));
    csk_status s = cs_apply_impl(plan, CSK_F64, n, A, lda, b, SA, k1, CSK_VAR_AUTO, st, 0, plan->d, false);
    if (s == CSK_OK) s = srht_impl(k1, k1, 0, k2, plan->seed, ncols, SA, k1, nullptr, Z, ldz, st);
    cudaFreeAsync(SA, st);
    return s;
}

__global__ void diag_kernel(const double* __restrict__ R, int64_t ldr, int n, double* __restrict__ dg) {
    for (int i = threadIdx.x; i <= n; i += blockDim.x) dg[i] = R[i + (int64_t)i * ldr];
}

// CountSketch-only: SA = S1 [A b] (k1 x nc), GEQRF, x = R11^-1 r12, sk_resid = |R_nn|
static csk_status cs_lstsq_impl(csk_plan_t plan, int64_t n, const double* A, int64_t lda, const double* b, double* x,
                                double* sk_resid, cudaStream_t st) {
    CSK_REQUIRE(plan != nullptr && A != nullptr && b != nullptr && x != nullptr, CSK_EINVAL, "NULL argument");
    const int64_t k1 = plan->k1, nc = n + 1;
    CSK_REQUIRE(n >= 1 && k1 >= nc, CSK_ESHAPE, "k1=%lld must be >= n+1", (long long)k1);
    CSK_REQUIRE(k1 * nc < (1LL << 31), CSK_EUNSUPPORTED, "k1 x (n+1) too large for GEQRF");
    CSK_REQUIRE(is_device_pointer(x), CSK_EINVAL, "x must be a device pointer");
    CSK_REQUIRE(nc <= 1025, CSK_EUNSUPPORTED, "n=%lld > 1024", (long long)n);
    cusolverDnHandle_t sh;
    csk_status s = solver_handle(st, &sh);
    if (s != CSK_OK) return s;
    int lwork = 0;
    CSK_REQUIRE(cusolverDnDgeqrf_bufferSize(sh, (int)k1, (int)nc, nullptr, (int)k1, &lwork) == CUSOLVER_STATUS_SUCCESS,
                CSK_ECUDA, "geqrf_bufferSize failed");
    auto pad = [](size_t c) { return (c + 31) & ~(size_t)31; };
    const size_t total = pad((size_t)k1 * nc) + pad(nc) + pad(nc) + pad((size_t)lwork) + 32;
    double* ws = nullptr;
    CSK_CUDA_TRY(csk_malloc_async(&ws, total * 8, st));
    double* SA = ws;
    double* tau = SA + pad((size_t)k1 * nc);
    double* dg = tau + pad(nc);
    double* work = dg + pad(nc);
    int* info = reinterpret_cast<int*>(work + pad((size_t)lwork));
    s = cs_apply_impl(plan, CSK_F64, n, A, lda, b, SA, k1, CSK_VAR_AUTO, st, 0, plan->d, false);
    if (s == CSK_OK) {
        if (cusolverDnDgeqrf(sh, (int)k1, (int)nc, SA, (int)k1, tau, work, lwork, info) != CUSOLVER_STATUS_SUCCESS) {
            set_error("cusolverDnDgeqrf failed");
            s = CSK_ECUDA;
        }
    }
    double hd[1025];
    if (s == CSK_OK) {
        diag_kernel<<<1, 256, 0, st>>>(SA, k1, (int)n, dg);
        CSK_LAUNCH_CHECK();
        CSK_CUDA_TRY(cudaMemsetAsync(info, 0, sizeof(int), st));
        // x = R11^-1 R[:n, n] (rc_finish_kernel's back substitution; *info == 0 lets it run)
        rc_finish_kernel<<<1, 1024, (size_t)n * 8, st>>>(SA, (int)k1, nullptr, (int)nc, (int)n, SA + (size_t)n * k1, x,
                                                        nullptr, 0, info);
        CSK_LAUNCH_CHECK();
        CSK_CUDA_TRY(cudaMemcpyAsync(hd, dg, (size_t)nc * 8, cudaMemcpyDeviceToHost, st));
    }
    cudaFreeAsync(ws, st);
    CSK_CUDA_TRY(cudaStreamSynchronize(st));
    if (s != CSK_OK) return s;
    double rmax = 0.0;
    for (int64_t i = 0; i < n; ++i) rmax = std::max(rmax, std::fabs(hd[i]));
    for (int64_t i = 0; i < n; ++i)
        if (!(std::fabs(hd[i]) > 1e-14 * rmax)) {
            set_error("CountSketch R is numerically singular");
            return CSK_ESINGULAR;
        }
    if (sk_resid) *sk_resid = std::fabs(hd[n]);
    return CSK_OK;
}

// sketch Z (k x (n+1)) of [A b] by `apply`, then the cluster Householder solve of ms_solve
template <typename F>
static csk_status sketch_then_solve(int64_t k, int64_t n, double* x, double* sk_resid, cudaStream_t st, F apply) {
    CSK_REQUIRE(x != nullptr && n >= 1, CSK_EINVAL, "x NULL or n < 1");
    CSK_REQUIRE(k >= n + 1, CSK_ESHAPE, "k=%lld must be >= n+1", (long long)k);
    double* Z = nullptr;
    CSK_CUDA_TRY(csk_malloc_async(&Z, (size_t)k * (n + 1) * 8, st));
    csk_status s = apply(Z);
    if (s == CSK_OK) s = solve_impl(k, n, Z, k, x, sk_resid, st, !is_device_pointer(x), nullptr);
    cudaFreeAsync(Z, st);
    return s;
}

}  // namespace csk

using namespace csk;

extern "C" {

csk_status gs_apply(int64_t d, int64_t row0, int64_t k, uint64_t seed, int64_t n, const double* A, int64_t lda,
                    const double* b, double* Z, int64_t ldz, void* stream) {
    return gs_apply_impl(d, row0, k, seed, n, A, lda, b, Z, ldz, (cudaStream_t)stream);
}

csk_status gs_lstsq(int64_t d, int64_t k, uint64_t seed, int64_t n, const double* A, int64_t lda, const double* b,
                    double* x, double* sk_resid, void* stream) {
    CSK_REQUIRE(b != nullptr, CSK_EINVAL, "b is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    return sketch_then_solve(k, n, x, sk_resid, st,
                             [&](double* Z) { return gs_apply_impl(d, 0, k, seed, n, A, lda, b, Z, k, st); });
}

csk_status msh_apply(csk_plan_t plan, int64_t k2, int64_t n, const double* A, int64_t lda, const double* b, double* Z,
                     int64_t ldz, void* stream) {
    return msh_apply_impl(plan, k2, n, A, lda, b, Z, ldz, (cudaStream_t)stream);
}

csk_status msh_lstsq(csk_plan_t plan, int64_t k2, int64_t n, const double* A, int64_t lda, const double* b, double* x,
                     double* sk_resid, void* stream) {
    CSK_REQUIRE(b != nullptr, CSK_EINVAL, "b is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    return sketch_then_solve(k2, n, x, sk_resid, st,
                             [&](double* Z) { return msh_apply_impl(plan, k2, n, A, lda, b, Z, k2, st); });
}

csk_status cs_lstsq(csk_plan_t plan, int64_t n, const double* A, int64_t lda, const double* b, double* x,
                    double* sk_resid, void* stream) {
    return cs_lstsq_impl(plan, n, A, lda, b, x, sk_resid, (cudaStream_t)stream);
}

}  // extern "C"
