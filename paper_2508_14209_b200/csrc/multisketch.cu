// multisketch.cu -- ms_apply / ms_solve / ms_lstsq.
//
// a4 G:    k2 x k1 Gaussian, G_ij ~ N(0, 1/k2) ("2n x 2n^2 Gaussian"),
//          Philox stream 1 + Box-Muller (R4), cached in the plan per k2.
// a5 Z:    Z = G (S [A b])  -- the multisketch S2(S1 x), the hand-written fp64 DMMA
//          G-stage of gstage.cu on the CountSketch's row-major workspace (Table 1 P:L99 "n^4" term).
// a7 solve: Householder QR of Z = [GSA | GSb] in one CTA, back substitution
//          (Alg 1 lines 2-3; GeQRF + OrMQR + TRSV of P:L230).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>
#include <cublas_v2.h>

#include "csk_internal.cuh"

namespace csk {

// --------------------------------------------------------------- cuBLAS
csk_status blas_handle(cudaStream_t st, cublasHandle_t* out) {
    // one handle per (thread, device, stream): cuBLAS keeps its split-K workspace in the handle,
    // so GEMMs in flight on two streams of one thread must not share one
    static thread_local std::map<std::pair<int, cudaStream_t>, cublasHandle_t> handles;
    int dev = 0;
    CSK_CUDA_TRY(cudaGetDevice(&dev));
    const auto key = std::make_pair(dev, st);
    auto it = handles.find(key);
    if (it == handles.end()) {
        cublasHandle_t h = nullptr;
        CSK_REQUIRE(cublasCreate(&h) == CUBLAS_STATUS_SUCCESS, CSK_ECUDA, "cublasCreate failed");
        // fp64 stays fp64; no TF32 for fp32 (tolerance 1e-5 needs full fp32 products)
        cublasSetMathMode(h, CUBLAS_PEDANTIC_MATH);
        if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) {
            cublasDestroy(h);
            set_error("cublasSetStream failed");
            return CSK_ECUDA;
        }
        it = handles.emplace(key, h).first;
    }
    *out = it->second;
    return CSK_OK;
}

// ------------------------------------------------------------------ a4: G
template <typename T>
__global__ void gauss_kernel(T* __restrict__ G, int64_t total, double inv_sqrt_scale_div, uint32_t key_lo,
                             uint32_t key_hi, int64_t t_off) {
    // element e of the stream is G[e - 2 t_off] (t_off: first pair, for row-chunked Gaussian sketches)
    const int64_t npairs = total >> 1;
    for (int64_t tl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; tl < npairs; tl += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = tl + t_off;
        const uint4 x = philox4x32_10(make_uint4((uint32_t)t, (uint32_t)(t >> 32), 1u, 0u), make_uint2(key_lo, key_hi));
        const uint64_t w1 = ((uint64_t)x.y << 32) | x.x;
        const uint64_t w2 = ((uint64_t)x.w << 32) | x.z;
        const double u1 = (double)((w1 >> 11) + 1) * 0x1.0p-53;
        const double u2 = (double)(w2 >> 11) * 0x1.0p-53;
        const double rho = sqrt(-2.0 * log(u1));
        double s, c;
        sincospi(2.0 * u2, &s, &c);
        G[2 * tl] = (T)((rho * c) / inv_sqrt_scale_div);
        G[2 * tl + 1] = (T)((rho * s) / inv_sqrt_scale_div);
    }
}

// G stored with a padded leading dimension for the G-stage's 16-B tile loads: element e = r + c k2 of
// the Philox stream (R4) lives at G[r + c ldg]; rows k2..ldg-1 and the tail stay zero
__global__ void gauss_ld_kernel(double* __restrict__ G, int64_t k2, int64_t ldg, int64_t total, double div,
                                uint32_t key_lo, uint32_t key_hi) {
    const int64_t npairs = (total + 1) >> 1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < npairs; t += (int64_t)gridDim.x * blockDim.x) {
        const uint4 x = philox4x32_10(make_uint4((uint32_t)t, (uint32_t)(t >> 32), 1u, 0u), make_uint2(key_lo, key_hi));
        const uint64_t w1 = ((uint64_t)x.y << 32) | x.x;
        const uint64_t w2 = ((uint64_t)x.w << 32) | x.z;
        const double u1 = (double)((w1 >> 11) + 1) * 0x1.0p-53;
        const double u2 = (double)(w2 >> 11) * 0x1.0p-53;
        const double rho = sqrt(-2.0 * log(u1));
        double sn, cs;
        sincospi(2.0 * u2, &sn, &cs);
        const int64_t e0 = 2 * t, e1 = 2 * t + 1;
        G[(e0 % k2) + (e0 / k2) * ldg] = (rho * cs) / div;
        if (e1 < total) G[(e1 % k2) + (e1 / k2) * ldg] = (rho * sn) / div;
    }
}

csk_status gauss_get(csk_plan_t plan, int64_t k2, cudaStream_t st, const double** out, int64_t* ldg_out) {
    std::lock_guard<std::mutex> lk(plan->mu);
    const int64_t ldg = (k2 + 7) & ~(int64_t)7;
    *ldg_out = ldg;
    auto it = plan->gauss64.find(k2);
    if (it != plan->gauss64.end()) {
        *out = it->second;
        return CSK_OK;
    }
    const int64_t total = k2 * plan->k1;
    const size_t bytes = ((size_t)ldg * plan->k1 + kGstageTailPad) * sizeof(double);
    double* G = nullptr;
    if (cudaMalloc(&G, bytes) != cudaSuccess) {
        cudaGetLastError();
        set_error("allocation of G (%lld x %lld) failed", (long long)k2, (long long)plan->k1);
        return CSK_ENOMEM;
    }
    auto fail = [&](const char* what) {
        cudaFree(G);
        set_error("%s", what);
        return CSK_ECUDA;
    };
    if (cudaMemsetAsync(G, 0, bytes, st) != cudaSuccess) return fail("G memset failed");
    const double div = std::sqrt((double)k2);
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(std::max<int64_t>((total + 1) / 2, 1), 256), 148 * 32);
    gauss_ld_kernel<<<grid, 256, 0, st>>>(G, k2, ldg, total, div, (uint32_t)plan->seed, (uint32_t)(plan->seed >> 32));
    count_launch();
    // synchronised before the pointer is published: a consumer on another stream may read it next
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) return fail("gauss kernel failed");
    plan->gauss64[k2] = G;
    *out = G;
    return CSK_OK;
}

template __global__ void gauss_kernel<double>(double*, int64_t, double, uint32_t, uint32_t, int64_t);
template __global__ void gauss_kernel<float>(float*, int64_t, double, uint32_t, uint32_t, int64_t);

// ---------------------------------------------------- a3 over host inputs
// Host A/b: stream row chunks through two device staging buffers; the copy of
// chunk i+1 overlaps the sketch of chunk i (the sketch is linear in row blocks,
// P:L375).  Accumulates into the fp64 column-major buffer SA.
static csk_status sketch_host_rows(csk_plan_t plan, int64_t n, const double* A, int64_t lda, const double* b,
                                   double* SA, int64_t ldsa, cudaStream_t st) {
    const int ncols = (int)(n + (b ? 1 : 0));
    const int64_t d = plan->d;
    const int64_t chunk = std::min<int64_t>(d, std::max<int64_t>(1 << 16, (int64_t)(256ll << 20) / (8 * ncols)));
    double* stage[2] = {nullptr, nullptr};
    cudaEvent_t copied[2] = {}, consumed[2] = {};
    cudaStream_t cs = nullptr;
    auto cleanup = on_exit([&] {
        if (cs) cudaStreamSynchronize(cs);
        for (int i = 0; i < 2; ++i) {
            if (stage[i]) cudaFreeAsync(stage[i], st);
            if (copied[i]) cudaEventDestroy(copied[i]);
            if (consumed[i]) cudaEventDestroy(consumed[i]);
        }
        if (cs) cudaStreamDestroy(cs);
    });
    CSK_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
        CSK_CUDA_TRY(csk_malloc_async(&stage[i], (size_t)chunk * ncols * 8, st));
        CSK_CUDA_TRY(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
        CSK_CUDA_TRY(cudaEventCreateWithFlags(&consumed[i], cudaEventDisableTiming));
        CSK_CUDA_TRY(cudaEventRecord(consumed[i], st));
    }
    csk_status s = CSK_OK;
    int k = 0;
    for (int64_t r0 = 0; r0 < d && s == CSK_OK; r0 += chunk, k ^= 1) {
        const int64_t rows = std::min(chunk, d - r0);
        CSK_CUDA_TRY(cudaStreamWaitEvent(cs, consumed[k], 0));
        if (n > 0)   // one strided copy per chunk (n column segments), not n separate copies
            CSK_CUDA_TRY(cudaMemcpy2DAsync(stage[k], rows * 8, A + r0, lda * 8, rows * 8, n, cudaMemcpyHostToDevice,
                                           cs));
        if (b) CSK_CUDA_TRY(cudaMemcpyAsync(stage[k] + n * rows, b + r0, rows * 8, cudaMemcpyHostToDevice, cs));
        CSK_CUDA_TRY(cudaEventRecord(copied[k], cs));
        CSK_CUDA_TRY(cudaStreamWaitEvent(st, copied[k], 0));
        s = cs_apply_impl(plan, CSK_F64, n, stage[k], rows, b ? stage[k] + n * rows : nullptr, SA, ldsa,
                          CSK_VAR_AUTO, st, r0, r0 + rows, /*accumulate=*/true);
        CSK_CUDA_TRY(cudaEventRecord(consumed[k], st));
    }
    return s;
}

// ------------------------------------------------------------- a7: ms_solve
// One CTA.  W (m x nc, column-major, ld m) is a private copy of Z, held in shared
// memory when it fits (else in global memory, L2-resident: <= 1 MB at BASELINE sizes).
// Householder with the LAPACK sign choice R_jj = -sign(x0) ||x||.  One __syncthreads
// per column: every thread recomputes alpha and beta = 2/(v^T v) = 1/(alpha (alpha - x0))
// from the column's norm^2, which the warp updating column j+1 accumulates during step j
// (look-ahead).  Back substitution by one warp.
constexpr int kQrThreads = 512;

__global__ void __launch_bounds__(kQrThreads, 1) qr_solve_kernel(double* __restrict__ Wg, int m, int nc,
                                                                 int use_smem, double* __restrict__ x,
                                                                 SolveStatus* __restrict__ status) {
    extern __shared__ double qsm[];
    __shared__ double red[kQrThreads / 32];
    __shared__ int s_fail;
    double* norm2 = qsm;               // nc + 1
    double* diag = norm2 + nc + 1;     // nc
    double* y = diag + nc;             // nc
    double* W = use_smem ? y + nc + 1 : Wg;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (use_smem)
        for (int e = threadIdx.x; e < m * nc; e += blockDim.x) W[e] = Wg[e];
    __syncthreads();
    {   // norm^2 of column 0, fixed-order reduction
        double part = 0.0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) part += W[i] * W[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) red[warp] = part;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += red[w];
            norm2[0] = s;
        }
        __syncthreads();
    }
    for (int j = 0; j < nc; ++j) {
        const double* wj = W + (int64_t)j * m;
        const double x0 = wj[j];
        const double nrm = sqrt(norm2[j]);
        const double alpha = nrm == 0.0 ? 0.0 : (x0 >= 0.0 ? -nrm : nrm);
        const double beta = nrm == 0.0 ? 0.0 : 1.0 / (alpha * (alpha - x0));
        const double v0 = x0 - alpha;
        if (threadIdx.x == 0) diag[j] = alpha;
        for (int c = j + 1 + warp; c < nc; c += nw) {
            double* wc = W + (int64_t)c * m;
            double dot = lane == 0 ? v0 * wc[j] : 0.0;
            for (int i = j + 1 + lane; i < m; i += 32) dot += wj[i] * wc[i];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
            const double f = beta * dot;
            if (lane == 0) wc[j] -= f * v0;
            double ss = 0.0;
            for (int i = j + 1 + lane; i < m; i += 32) {
                const double t = wc[i] - f * wj[i];
                wc[i] = t;
                ss += t * t;
            }
            if (c == j + 1) {   // look-ahead: norm^2 of the next pivot column below the diagonal
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
                if (lane == 0) norm2[j + 1] = ss;
            }
        }
        __syncthreads();
    }
    // R: diagonal in diag[], strictly upper part in W.  Singularity check on R[:n,:n].
    const int n = nc - 1;
    if (threadIdx.x == 0) {
        double rmax = 0.0;
        for (int i = 0; i < n; ++i) rmax = fmax(rmax, fabs(diag[i]));
        int st = 0;
        for (int i = 0; i < n; ++i)
            if (!(fabs(diag[i]) > 1e-14 * rmax)) st = CSK_ESINGULAR;
        status->status = st;
        status->sk_resid = fabs(diag[n]);
        s_fail = st;
    }
    __syncthreads();
    if (s_fail || warp != 0) return;
    // back substitution R[:n,:n] x = R[:n, n] (= Q^T z), column-oriented, one warp
    for (int i = lane; i < n; i += 32) y[i] = W[i + (int64_t)n * m];
    __syncwarp();
    for (int c = n - 1; c >= 0; --c) {
        const double xc = y[c] / diag[c];
        for (int i = lane; i < c; i += 32) y[i] -= W[i + (int64_t)c * m] * xc;
        if (lane == 0) x[c] = xc;
        __syncwarp();
    }
}


// Cluster-distributed Householder QR + back substitution.  Columns of Z are dealt
// block-cyclically to the P CTAs of one thread-block cluster (column c lives in CTA c % P,
// in shared memory).  Step j: the owner of column j forms v and beta from the norm its own
// look-ahead produced, writes v (and beta) into every CTA's shared memory through DSMEM,
// one cluster barrier, then every CTA updates its own columns c > j; the warp updating
// column j+1 also accumulates its norm below the diagonal (look-ahead for the next owner).
// R goes to global memory; CTA 0 checks the diagonal and back-substitutes with an 8-deep
// register prefetch of R's columns.
constexpr int kQrcThreads = 512;

__global__ void __launch_bounds__(kQrcThreads, 1) qr_cluster_kernel(const double* __restrict__ Z, int64_t ldz, int m,
                                                                   int nc, int P, double* __restrict__ Rg, int ldr,
                                                                   double* __restrict__ x,
                                                                   SolveStatus* __restrict__ status) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = P > 1 ? (int)cl.block_rank() : 0;
    extern __shared__ double qc[];
    double* vbuf = qc;            // [2][m]  Householder vectors (double-buffered by step parity)
    double* scal = qc + 2 * m;    // [0..1] beta per buffer, [2] norm^2 of this CTA's next pivot
    double* Wl = qc + 2 * m + 4;  // [ncl][ldw] local columns; odd stride so column groups hit distinct banks
    const int ldw = m | 1;
    const int ncl = (nc - rank + P - 1) / P;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int e = threadIdx.x; e < ncl * m; e += blockDim.x) {
        const int t = e / m, i = e - t * m;
        Wl[t * ldw + i] = Z[i + (int64_t)(rank + P * t) * ldz];
    }
    __syncthreads();
    if (rank == 0 && warp == 0) {
        double ss = 0.0;
        for (int i = lane; i < m; i += 32) ss += Wl[i] * Wl[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if (lane == 0) scal[2] = ss;
    }
    __syncthreads();
    for (int j = 0; j < nc; ++j) {
        const int owner = j % P, buf = j & 1;
        if (rank == owner) {
            const double* wj = Wl + (int64_t)(j / P) * ldw;
            const double x0 = wj[j];
            const double nrm = sqrt(scal[2]);
            const double alpha = nrm == 0.0 ? 0.0 : (x0 >= 0.0 ? -nrm : nrm);
            const double beta = nrm == 0.0 ? 0.0 : 1.0 / (alpha * (alpha - x0));
            const double v0 = x0 - alpha;
            if (threadIdx.x == 0) {
                Rg[j + (int64_t)j * ldr] = alpha;
                scal[buf] = beta;
            }
            for (int i = j + threadIdx.x; i < m; i += blockDim.x) vbuf[buf * m + i] = i == j ? v0 : wj[i];
        }
        if (P > 1) {
            // every CTA pulls v and beta out of the owner's shared memory (DSMEM reads run in
            // parallel on all P SMs; a push from the owner serialises on its DSMEM port)
            cl.sync();
            if (rank != owner) {
                const double* src = cl.map_shared_rank(vbuf, owner) + buf * m;
                for (int i = j + threadIdx.x; i < m; i += blockDim.x) vbuf[buf * m + i] = src[i];
                if (threadIdx.x == 0) scal[buf] = cl.map_shared_rank(scal, owner)[buf];
            }
        }
        __syncthreads();
        const double* v = vbuf + buf * m;
        const double beta = scal[buf];
        const int t0 = j + 1 - rank > 0 ? (j + 1 - rank + P - 1) / P : 0;
        const int nact = ncl - t0;   // trailing local columns
        if (nact > 0) {
            // G lanes per column (power of 2, <= 32), as many column groups as the block holds;
            // lane g of a group takes rows j + g, j + g + G, ...  (all values warp-uniform)
            int G = 32;
            while (G > 1 && (int)(blockDim.x / G) < nact) G >>= 1;
            const int ngrp = blockDim.x / G;
            const int g = lane & (G - 1);
            for (int base = 0; base < nact; base += ngrp) {   // block-uniform trip count (shuffles below)
                const int grp = base + (int)(threadIdx.x / G);
                const bool act = grp < nact;
                const int t = t0 + (act ? grp : 0);
                double* wc = Wl + (int64_t)t * ldw;
                double d0 = 0.0, d1 = 0.0;
                int i = j + g;
                if (act) {
                    for (; i + G < m; i += 2 * G) {
                        d0 += v[i] * wc[i];
                        d1 += v[i + G] * wc[i + G];
                    }
                    if (i < m) d0 += v[i] * wc[i];
                }
                double dot = d0 + d1;
                for (int o = G >> 1; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
                const double f = beta * dot;
                double ss = 0.0;
                if (act) {
                    for (int r = j + g; r < m; r += G) {
                        const double tv = wc[r] - f * v[r];
                        wc[r] = tv;
                        if (r > j) ss += tv * tv;
                    }
                }
                if (__any_sync(0xffffffffu, act && rank + P * t == j + 1)) {
                    for (int o = G >> 1; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
                    if (act && rank + P * t == j + 1 && g == 0) scal[2] = ss;
                }
            }
        }
        __syncthreads();
    }
    // strictly upper part of R to global (rows < c of local column c)
    for (int t = 0; t < ncl; ++t) {
        const int c = rank + P * t;
        for (int i = threadIdx.x; i < c; i += blockDim.x) Rg[i + (int64_t)c * ldr] = Wl[(int64_t)t * ldw + i];
    }
    if (P > 1)
        cl.sync();
    else
        __syncthreads();
    if (rank != 0) return;
    const int n = nc - 1;
    double* diag = vbuf;          // reuse: nc
    double* y = vbuf + nc;        // n
    __shared__ int s_fail;
    for (int i = threadIdx.x; i < nc; i += blockDim.x) diag[i] = Rg[i + (int64_t)i * ldr];
    for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = Rg[i + (int64_t)n * ldr];
    __syncthreads();
    if (threadIdx.x == 0) {
        double rmax = 0.0;
        for (int i = 0; i < n; ++i) rmax = fmax(rmax, fabs(diag[i]));
        int stt = 0;
        for (int i = 0; i < n; ++i)
            if (!(fabs(diag[i]) > 1e-14 * rmax)) stt = CSK_ESINGULAR;
        status->status = stt;
        status->sk_resid = fabs(diag[n]);
        s_fail = stt;
    }
    __syncthreads();
    if (s_fail) return;
    const int i = threadIdx.x;
    if (n <= (int)blockDim.x) {
        double ring[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int c = n - 1 - k;
            ring[k] = (c >= 0 && i < c) ? Rg[i + (int64_t)c * ldr] : 0.0;
        }
        for (int cb = n - 1; cb >= 0; cb -= 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int c = cb - k;
                if (c >= 0) {
                    const double xc = y[c] / diag[c];
                    if (i < c) y[i] -= ring[k] * xc;
                    if (i == 0) x[c] = xc;
                    const int cn = c - 8;
                    ring[k] = (cn >= 0 && i < cn) ? Rg[i + (int64_t)cn * ldr] : 0.0;
                    __syncthreads();
                }
            }
        }
    } else {
        for (int c = n - 1; c >= 0; --c) {
            const double xc = y[c] / diag[c];
            for (int r = threadIdx.x; r < c; r += blockDim.x) y[r] -= Rg[r + (int64_t)c * ldr] * xc;
            if (threadIdx.x == 0) x[c] = xc;
            __syncthreads();
        }
    }
}

csk_status solve_impl(int64_t k2, int64_t n, const double* Z, int64_t ldz, double* x, double* sk_resid,
                      cudaStream_t st, bool x_host, double* R_out, int32_t* status_dev, double* resid_dev) {
    CSK_REQUIRE(Z != nullptr && x != nullptr, CSK_EINVAL, "Z and x must be non-NULL");
    CSK_REQUIRE(n >= 1 && n <= 65535, CSK_EINVAL, "n=%lld must be in [1, 65535]", (long long)n);
    CSK_REQUIRE(k2 >= n + 1, CSK_ESHAPE, "k2=%lld must be >= n+1=%lld", (long long)k2, (long long)(n + 1));
    CSK_REQUIRE(ldz >= k2, CSK_ESHAPE, "ldz=%lld < k2=%lld", (long long)ldz, (long long)k2);
    const int m = (int)k2, nc = (int)(n + 1);
    double* W = nullptr;
    double* xd = nullptr;
    SolveStatus* sd = nullptr;
    const size_t wbytes = (size_t)(m + 1) * nc * 8;   // >= the R of the WY path, (nc rounded to even) x nc
    const size_t scratch_bytes = qr_wy_scratch_doubles(m, nc) * 8;
    const size_t scratch_off = (wbytes + 64 + (x_host ? n * 8 : 0) + 255) & ~(size_t)255;   // 16-B vector loads
    CSK_CUDA_TRY(csk_malloc_async(&W, scratch_off + scratch_bytes, st));
    // R's unused (lower) part is read by 16-B block loads and by the R export: keep it defined
    CSK_CUDA_TRY(cudaMemsetAsync(W, 0, wbytes + 64, st));   // + the status struct (its padding is copied out)
    sd = reinterpret_cast<SolveStatus*>(reinterpret_cast<char*>(W) + wbytes);
    xd = x_host ? reinterpret_cast<double*>(reinterpret_cast<char*>(W) + wbytes + 64) : x;
    double* scratch = reinterpret_cast<double*>(reinterpret_cast<char*>(W) + scratch_off);
    const DeviceInfo& di = device_info();
    // register-blocked compact-WY cluster QR (qr_wy.cu) when Z fits <= 16 CTAs
    {
        bool wy = false;
        const csk_status ws = qr_wy_launch(Z, ldz, m, nc, W, (nc + 1) & ~1, scratch, xd, sd, st, &wy);   // even ld: 16-B R reads
        if (ws != CSK_OK) {
            cudaFreeAsync(W, st);
            return ws;
        }
        if (wy) {
            if (R_out)   // R (nc x nc, upper) -> caller's buffer, ld nc
                CSK_CUDA_TRY(cudaMemcpy2DAsync(R_out, nc * 8, W, ((nc + 1) & ~1) * 8, nc * 8, nc,
                                               cudaMemcpyDeviceToDevice, st));
            goto launched;
        }
    }
    {
    // cluster-distributed unblocked QR when a column slice fits shared memory on <= 8 CTAs
    int P = 0;
    for (int p = 1; p <= 8; p *= 2) {
        const size_t need = (size_t)(2 * m + 4 + (size_t)((nc + p - 1) / p) * (m | 1)) * 8;
        if (need <= (size_t)di.smem_optin && p <= nc) {
            P = p;
            break;
        }
    }
    if (P > 0 && !std::getenv("CSK_QR_SINGLE")) {
        const size_t smem = (size_t)(2 * m + 4 + (size_t)((nc + P - 1) / P) * (m | 1)) * 8;
        CSK_CUDA_TRY(cudaFuncSetAttribute(qr_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(P);
        cfg.blockDim = dim3(kQrcThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = P;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        // W doubles as the R output (ld = nc)
        CSK_CUDA_TRY(cudaLaunchKernelEx(&cfg, qr_cluster_kernel, Z, (int64_t)ldz, m, nc, P, W, nc, xd, sd));
        CSK_LAUNCH_CHECK();
        if (R_out) CSK_CUDA_TRY(cudaMemcpyAsync(R_out, W, (size_t)nc * nc * 8, cudaMemcpyDeviceToDevice, st));
    } else {
    if (R_out) {
        cudaFreeAsync(W, st);
        set_error("R export needs the cluster QR paths (k2=%lld, n=%lld too large)", (long long)k2, (long long)n);
        return CSK_EUNSUPPORTED;
    }
    CSK_CUDA_TRY(cudaMemcpy2DAsync(W, m * 8, Z, ldz * 8, m * 8, nc, cudaMemcpyDeviceToDevice, st));
    const size_t small = (size_t)(3 * nc + 2) * 8;
    const size_t smem_need = small + (size_t)m * nc * 8;
    const int use_smem = smem_need <= (size_t)di.smem_optin ? 1 : 0;
    const size_t smem = use_smem ? smem_need : small;
    CSK_CUDA_TRY(cudaFuncSetAttribute(qr_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    qr_solve_kernel<<<1, kQrThreads, smem, st>>>(W, m, nc, use_smem, xd, sd);
    CSK_LAUNCH_CHECK();
    }
    }
launched:
    if (status_dev) {   // asynchronous form (ms_solve_async): the status stays on the device, no sync
        CSK_CUDA_TRY(cudaMemcpyAsync(status_dev, &sd->status, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        if (resid_dev)
            CSK_CUDA_TRY(cudaMemcpyAsync(resid_dev, &sd->sk_resid, sizeof(double), cudaMemcpyDeviceToDevice, st));
        CSK_CUDA_TRY(cudaFreeAsync(W, st));
        return CSK_OK;
    }
    SolveStatus hs;
    CSK_CUDA_TRY(cudaMemcpyAsync(&hs, sd, sizeof(hs), cudaMemcpyDeviceToHost, st));
    if (x_host) CSK_CUDA_TRY(cudaMemcpyAsync(x, xd, n * 8, cudaMemcpyDeviceToHost, st));
    CSK_CUDA_TRY(cudaFreeAsync(W, st));
    CSK_CUDA_TRY(cudaStreamSynchronize(st));
    if (sk_resid) *sk_resid = hs.sk_resid;
    if (hs.status != 0) {
        set_error("sketched R is numerically singular (|R_ii| <= 1e-14 max|R_jj|)");
        return (csk_status)hs.status;
    }
    return CSK_OK;
}

// SA (k1 x ncols column-major fp64, ld) -> the regular row-major workspace (lc = round_up(ncols, 2))
__global__ void colmajor_to_rows_kernel(const double* __restrict__ SA, int64_t ld, int64_t k1, int ncols,
                                        double* __restrict__ Yt, int64_t lc) {
    __shared__ double t[32][33];
    const int64_t m0 = blockIdx.x * 32;
    const int c0 = blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int c = c0 + j;
        const int64_t m = m0 + threadIdx.x;
        t[j][threadIdx.x] = (m < k1 && c < ncols) ? SA[m + (int64_t)c * ld] : 0.0;
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int64_t m = m0 + j;
        const int c = c0 + threadIdx.x;
        if (m < k1 && c < (int)lc) Yt[m * lc + c] = t[threadIdx.x][j];
    }
}

csk_status rows_from_colmajor(const double* SA, int64_t ld, int64_t k1, int ncols, RowOut* ro, cudaStream_t st) {
    const int64_t lc = (ncols + 1) & ~1;
    double* Yt = nullptr;
    CSK_CUDA_TRY(csk_malloc_async(&Yt, (size_t)k1 * lc * sizeof(double), st));
    dim3 grid((unsigned)ceil_div(k1, 32), (unsigned)ceil_div(lc, 32));
    colmajor_to_rows_kernel<<<grid, dim3(32, 8), 0, st>>>(SA, ld, k1, ncols, Yt, lc);
    count_launch();
    if (cudaGetLastError() != cudaSuccess) {
        cudaFreeAsync(Yt, st);
        set_error("row-major conversion launch failed");
        return CSK_ECUDA;
    }
    ro->ws = Yt;
    ro->ncols = ncols;
    ro->lc = lc;
    ro->cw = ncols;
    ro->cs = ncols;
    return CSK_OK;
}

csk_status ms_apply_impl(csk_plan_t plan, int64_t k2, csk_dtype dtype, int64_t n, const void* A, int64_t lda,
                         const void* b, void* Z, int64_t ldz, cudaStream_t st) {
    CSK_REQUIRE(plan != nullptr, CSK_EINVAL, "plan is NULL");
    CSK_REQUIRE(Z != nullptr, CSK_EINVAL, "Z is NULL");
    CSK_REQUIRE(k2 >= 1 && k2 <= 1 << 20, CSK_EINVAL, "k2=%lld out of range", (long long)k2);
    CSK_REQUIRE(ldz >= k2, CSK_ESHAPE, "ldz=%lld < k2=%lld", (long long)ldz, (long long)k2);
    CSK_REQUIRE(dtype == CSK_F64 || dtype == CSK_F32, CSK_EDTYPE, "dtype %d not supported", (int)dtype);
    const int64_t ncols = n + (b ? 1 : 0);
    CSK_REQUIRE(n >= 0 && ncols >= 1, CSK_EINVAL, "n + (b != NULL) must be >= 1");
    CSK_REQUIRE(n == 0 || A != nullptr, CSK_EINVAL, "A is NULL");
    const bool host_in = (n > 0 && !is_device_pointer(A)) || (b && !is_device_pointer(b));
    CSK_REQUIRE(!host_in || dtype == CSK_F64, CSK_EDTYPE, "host-resident inputs are supported for fp64 only");
    const int64_t k1 = plan->k1;
    csk_status s;
    RowOut ro;
    // a3: the CountSketch hands over its fp64 row-major SA^T workspace ("interpreted Y stored in
    // row-major as the transpose ... computed Z^T = Y^T G^T"), so no k1 x ncols transpose is made on the
    // default path
    if (host_in) {
        CSK_REQUIRE(n == 0 || lda >= plan->d, CSK_ESHAPE, "lda < d");
        double* SA = nullptr;
        CSK_CUDA_TRY(csk_malloc_async(&SA, (size_t)k1 * ncols * 8, st));
        s = cudaMemsetAsync(SA, 0, (size_t)k1 * ncols * 8, st) == cudaSuccess ? CSK_OK : CSK_ECUDA;
        if (s == CSK_OK) s = sketch_host_rows(plan, n, (const double*)A, lda, (const double*)b, SA, k1, st);
        if (s == CSK_OK) s = rows_from_colmajor(SA, k1, k1, (int)ncols, &ro, st);
        cudaFreeAsync(SA, st);
    } else {
        s = cs_apply_impl(plan, dtype, n, A, lda, b, nullptr, k1, CSK_VAR_AUTO, st, 0, plan->d, false, &ro);
    }
    if (s != CSK_OK) {
        if (ro.ws) cudaFreeAsync(ro.ws, st);
        return s;
    }
    // a regular (one-row) layout wider than the G-stage's chunk is the same memory cut into 64-column chunks
    if (ro.cw > kGstageMaxCw) {
        ro.cw = 64;
        ro.cs = 64;
    }
    if (ro.ncols <= ro.cw) ro.cs = 0;   // one chunk: the chunk stride is never used
    // a4 + a5: G from the plan (drawn once per k2), Z = G Y on the fp64 tensor pipe (fp32 input: the
    // sketch was accumulated in fp64, R12, and Z is rounded to fp32 once)
    const double* G = nullptr;
    int64_t ldg = 0;
    s = gauss_get(plan, k2, st, &G, &ldg);
    if (s == CSK_OK) s = gstage_launch(G, ldg, k2, k1, ro, Z, ldz, dtype == CSK_F32, st);
    cudaFreeAsync(ro.ws, st);
    return s;
}

}  // namespace csk

using namespace csk;

extern "C" {

csk_status ms_apply(csk_plan_t plan, int64_t k2, csk_dtype dtype, int64_t n, const void* A, int64_t lda,
                    const void* b, void* Z, int64_t ldz, void* stream) {
    return ms_apply_impl(plan, k2, dtype, n, A, lda, b, Z, ldz, (cudaStream_t)stream);
}

csk_status ms_solve(int64_t k2, int64_t n, const double* Z, int64_t ldz, double* x, double* sk_resid, void* stream) {
    CSK_REQUIRE(x == nullptr || is_device_pointer(x), CSK_EINVAL, "x must be a device pointer");
    return solve_impl(k2, n, Z, ldz, x, sk_resid, (cudaStream_t)stream, false, nullptr);
}

csk_status ms_solve_async(int64_t k2, int64_t n, const double* Z, int64_t ldz, double* x, double* sk_resid,
                          int32_t* status, void* stream) {
    CSK_REQUIRE(x == nullptr || is_device_pointer(x), CSK_EINVAL, "x must be a device pointer");
    CSK_REQUIRE(status != nullptr && is_device_pointer(status), CSK_EINVAL, "status must be a device pointer");
    CSK_REQUIRE(sk_resid == nullptr || is_device_pointer(sk_resid), CSK_EINVAL, "sk_resid must be a device pointer");
    return solve_impl(k2, n, Z, ldz, x, nullptr, (cudaStream_t)stream, false, nullptr, status, sk_resid);
}

csk_status ms_lstsq(csk_plan_t plan, int64_t k2, int64_t n, const double* A, int64_t lda, const double* b, double* x,
                    double* sk_resid, void* stream) {
    CSK_REQUIRE(plan != nullptr, CSK_EINVAL, "plan is NULL");
    CSK_REQUIRE(b != nullptr && x != nullptr, CSK_EINVAL, "b and x must be non-NULL");
    CSK_REQUIRE(n >= 1, CSK_EINVAL, "n must be >= 1");
    CSK_REQUIRE(k2 >= n + 1, CSK_ESHAPE, "k2=%lld must be >= n+1", (long long)k2);
    cudaStream_t st = (cudaStream_t)stream;
    double* Z = nullptr;
    CSK_CUDA_TRY(csk_malloc_async(&Z, (size_t)k2 * (n + 1) * 8, st));
    csk_status s = ms_apply_impl(plan, k2, CSK_F64, n, A, lda, b, Z, k2, st);
    if (s == CSK_OK) s = solve_impl(k2, n, Z, k2, x, sk_resid, st, !is_device_pointer(x), nullptr);
    cudaFreeAsync(Z, st);
    return s;
}

}  // extern "C"
