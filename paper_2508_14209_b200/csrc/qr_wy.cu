// qr_wy.cu -- a7 small solve: register-blocked Householder QR of Z = [GSA | GSb] (k2 x (n+1))
// over a thread-block cluster, followed by back substitution (Alg 1 lines 2-3, P:L120-121;
// GeQRF + OrMQR + TRSV of P:L230).
//
// The solve is latency-bound (68 MFLOP at C3 = ~2 us of fp64 DMMA), so the design minimises the
// serial chain per column, not flops:
//  * panels of kB = 4 columns; panel k is owned by CTA k % P (column-block-cyclic); each CTA keeps
//    its columns in shared memory;
//  * a team of 4 warps factors a panel with the panel held in registers (row blocks of 32 dealt to
//    the 4 warps): per column ONE team reduction (warp butterfly + one named barrier) yields
//    ||x_(j+1:)||^2, x_(j+1:)^T c for every other panel column (v = x - alpha e_j gives
//    v^T c = x^T c - alpha c_j) and the pivot-row values;
//  * compact WY: Q_k = H_0..H_3 = I - V T V^T (T from the Gram V^T V, LAPACK larft forward);
//  * look-ahead: while the other warps apply Q_k^T to the trailing columns, the team of the owner of
//    panel k+1 applies Q_k^T to that panel and factors it, then joins the trailing update (columns
//    are handed out by a shared counter), so a step costs ~max(panel path, trailing update) plus
//    ONE barrier (cluster barrier when P > 1; V, T go through L2);
//  * the trailing update keeps V (4 x m) in registers: per column one read + one write of the
//    column in shared memory and one 4-value warp reduction.
// DESIGN.md section 6.2 has the measured per-shape times.
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "csk_internal.cuh"

namespace csk {
namespace {

constexpr int kB = 4;          // panel width
constexpr int kThreads = 256;  // 8 warps
constexpr int kWarps = kThreads / 32;

struct WyArgs {
    const double* Z;
    int64_t ldz;
    int m, nc, P, npan, ldw;
    double* Vg;   // [npan][kB][ldw]   published V (P > 1)
    double* Tg;   // [npan][kB*kB]     published T (P > 1)
    double* Rg;   // [nc][ldr]         R, column-major
    int ldr;
    double* x;
    SolveStatus* status;
#ifdef CSK_QR_PROFILE
    long long* prof;   // [P][npan+1][8] clock64 stamps (scripts/qr_wy_prof.cu)
#endif
};

#ifdef CSK_QR_PROFILE
#define QPROF(kk, slot)                                                                   \
    do {                                                                                  \
        if (a.prof) a.prof[((size_t)rank * (a.npan + 1) + (kk)) * 8 + (slot)] = clock64(); \
    } while (0)
#else
#define QPROF(kk, slot) \
    do {                \
    } while (0)
#endif

template <int N>
__device__ __forceinline__ void warp_sum_n(double (&v)[N]) {
    // butterfly: every lane ends with the bit-identical total (each add pairs the same partials)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    }
}

__device__ __forceinline__ void sync_all(int P) {
    if (P > 1)
        cooperative_groups::this_cluster().sync();   // barrier.cluster arrive.release / wait.acquire
    else
        __syncthreads();
}

// Panel team = warps 0..3 (threads 0..127, named barrier 1).  Row block tb (rows 32 tb .. 32 tb + 31)
// belongs to team warp tb & 3, as its local block tb >> 2, so every lane holds RPLT = RPL/4 row blocks.
constexpr int kTeamWarps = 4;
constexpr int kTeam = 32 * kTeamWarps;

__device__ __forceinline__ void team_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kTeam) : "memory"); }

// Sum N per-thread partials over the team; every team thread gets the bit-identical total
// (warp butterfly, then the four warp totals added in warp order).  buf: [2][kTeamWarps][16]
// shared ring, `ph` alternates per call so one barrier per call suffices.
template <int N>
__device__ __forceinline__ void team_sum(double (&v)[N], double* buf, int& ph) {
    static_assert(N <= 16, "team_sum: N <= 16");
    warp_sum_n<N>(v);
    const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
    double* b = buf + ph * (kTeamWarps * 16);
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < N; ++i) b[q * 16 + i] = v[i];
    }
    team_bar();
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = ((b[i] + b[16 + i]) + b[32 + i]) + b[48 + i];
    ph ^= 1;
}

// The panel team of the owner CTA: load panel kp (local shared-memory columns `cols`) into
// registers, optionally apply the previous panel's Q^T (Vin, Tin in shared memory), factor it,
// write R (rows <= diagonal) to global, V/T to shared memory (and to global when P > 1).
template <int RPL>
__device__ __forceinline__ void factor_panel(const WyArgs& a, const double* cols, int kp, double* Vout, double* Tout,
                                             const double* Vin, const double* Tin, double* rbuf) {
    constexpr int RPLT = (RPL + kTeamWarps - 1) / kTeamWarps;
    const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
    const int m = a.m, ldw = a.ldw, j0 = kp * kB, bw = min(kB, a.nc - j0);
    int ph = 0;
    double p[kB][RPLT];
#pragma unroll
    for (int c = 0; c < kB; ++c)
#pragma unroll
        for (int u = 0; u < RPLT; ++u) {
            const int r = 32 * (q + kTeamWarps * u) + lane;
            p[c][u] = r < m ? cols[c * ldw + r] : 0.0;
        }
    if (Vin != nullptr) {
        // p <- (I - V T^T V^T) p with the previous panel (V is zero above its pivots)
        const int tp = (j0 - kB) >> 5;
        double y[kB * kB];
#pragma unroll
        for (int e = 0; e < kB * kB; ++e) y[e] = 0.0;
#pragma unroll
        for (int u = 0; u < RPLT; ++u) {
            const int tb = q + kTeamWarps * u, r = 32 * tb + lane;
            if (tb < tp || r >= m) continue;
#pragma unroll
            for (int i = 0; i < kB; ++i) {
                const double vi = Vin[i * ldw + r];
#pragma unroll
                for (int c = 0; c < kB; ++c) y[c * kB + i] += vi * p[c][u];
            }
        }
        team_sum<kB * kB>(y, rbuf, ph);
        double w[kB * kB];
#pragma unroll
        for (int c = 0; c < kB; ++c)
#pragma unroll
            for (int i = 0; i < kB; ++i) {
                double s = 0.0;
#pragma unroll
                for (int l = 0; l <= i; ++l) s += Tin[l + i * kB] * y[c * kB + l];
                w[c * kB + i] = s;
            }
#pragma unroll
        for (int u = 0; u < RPLT; ++u) {
            const int tb = q + kTeamWarps * u, r = 32 * tb + lane;
            if (tb < tp || r >= m) continue;
#pragma unroll
            for (int i = 0; i < kB; ++i) {
                const double vi = Vin[i * ldw + r];
#pragma unroll
                for (int c = 0; c < kB; ++c) p[c][u] -= vi * w[c * kB + i];
            }
        }
    }
    double beta[kB];
#pragma unroll
    for (int i = 0; i < kB; ++i) {
        beta[i] = 0.0;
        if (i >= bw) continue;   // padding column of the last panel: H = I, v = 0
        const int j = j0 + i, tj = j >> 5;
        // one team reduction: red[0] = sum_{r>j} x_r^2, red[c] = sum_{r>j} x_r c_r (c > i),
        // red[kB] = x_j, red[kB + c] = c_j (only the pivot row's lane contributes; + 0 is exact)
        double red[2 * kB];
#pragma unroll
        for (int e = 0; e < 2 * kB; ++e) red[e] = 0.0;
#pragma unroll
        for (int u = 0; u < RPLT; ++u) {
            const int tb = q + kTeamWarps * u, r = 32 * tb + lane;
            if (tb < tj) continue;
            const double xr = r > j ? p[i][u] : 0.0;
            red[0] += xr * xr;
#pragma unroll
            for (int c = i + 1; c < kB; ++c) red[c] += xr * p[c][u];
            if (r == j) {
                red[kB] = p[i][u];
#pragma unroll
                for (int c = i + 1; c < kB; ++c) red[kB + c] = p[c][u];
            }
        }
        team_sum<2 * kB>(red, rbuf, ph);
        const double xj = red[kB];
        const double nrm = sqrt(red[0] + xj * xj);
        const double alpha = nrm == 0.0 ? 0.0 : (xj >= 0.0 ? -nrm : nrm);
        const double bt = nrm == 0.0 ? 0.0 : 1.0 / (alpha * (alpha - xj));
        const double v0 = xj - alpha;
        // apply H_i to the panel's later columns: c -= beta (v^T c) v, v^T c = red[c] + v0 c_j
#pragma unroll
        for (int c = i + 1; c < kB; ++c) {
            const double s = bt * (red[c] + v0 * red[kB + c]);
#pragma unroll
            for (int u = 0; u < RPLT; ++u) {
                const int tb = q + kTeamWarps * u, r = 32 * tb + lane;
                if (tb < tj) continue;
                if (r > j)
                    p[c][u] -= s * p[i][u];
                else if (r == j)
                    p[c][u] -= s * v0;
            }
        }
        // R column j: rows < j are final in p[i]; diagonal alpha.  Then p[i] <- v.
        double* Rc = a.Rg + (int64_t)j * a.ldr;
#pragma unroll
        for (int u = 0; u < RPLT; ++u) {
            const int r = 32 * (q + kTeamWarps * u) + lane;
            if (r < j) Rc[r] = p[i][u];
            p[i][u] = r < j ? 0.0 : (r == j ? v0 : p[i][u]);
        }
        if (threadIdx.x == 0) Rc[j] = alpha;
        beta[i] = bt;
    }
    // Gram of V and T (T[i + l kB], upper; T[:, l] = [-beta_l T[0:l,0:l] G[0:l,l]; beta_l])
    double g[kB * (kB - 1) / 2];
#pragma unroll
    for (int e = 0; e < kB * (kB - 1) / 2; ++e) g[e] = 0.0;
#pragma unroll
    for (int u = 0; u < RPLT; ++u) {
        int e = 0;
#pragma unroll
        for (int l = 1; l < kB; ++l)
#pragma unroll
            for (int i = 0; i < l; ++i) g[e++] += p[i][u] * p[l][u];
    }
    team_sum<kB * (kB - 1) / 2>(g, rbuf, ph);
    double T[kB * kB];
#pragma unroll
    for (int e = 0; e < kB * kB; ++e) T[e] = 0.0;
    {
        int e = 0;
#pragma unroll
        for (int l = 0; l < kB; ++l) {
            const int e0 = e;   // g index of G[0, l] (G[i, l] at e0 + i)
#pragma unroll
            for (int i = 0; i < l; ++i) {
                double s = 0.0;
#pragma unroll
                for (int qq = i; qq < l; ++qq) s += T[i + qq * kB] * g[e0 + qq];
                T[i + l * kB] = -beta[l] * s;
            }
            T[l + l * kB] = beta[l];
            e += l;
        }
    }
    // publish V (row blocks >= j0/32; zeros above the pivots) and T
    const int t0 = j0 >> 5;
    const bool pub = a.P > 1;
    double* Vgk = a.Vg + (size_t)kp * kB * ldw;
#pragma unroll
    for (int c = 0; c < kB; ++c)
#pragma unroll
        for (int u = 0; u < RPLT; ++u) {
            const int tb = q + kTeamWarps * u, r = 32 * tb + lane;
            if (tb >= t0 && r < m) {
                Vout[c * ldw + r] = p[c][u];
                if (pub) Vgk[c * ldw + r] = p[c][u];
            }
        }
    if (threadIdx.x < kB * kB) {
        double tv = 0.0;
#pragma unroll
        for (int e = 0; e < kB * kB; ++e)
            if ((int)threadIdx.x == e) tv = T[e];
        Tout[threadIdx.x] = tv;
        if (pub) a.Tg[(size_t)kp * kB * kB + threadIdx.x] = tv;
    }
}

// Trailing update of one shared-memory column C (rows >= 32 t0): C -= V (T^T (V^T C)).
template <int RPL>
__device__ __forceinline__ void apply_wy(double* C, const double (&vr)[kB][RPL], const double (&Tr)[kB * kB], int t0,
                                         int m) {
    const int lane = threadIdx.x & 31;
    double cr[RPL];
    double y[kB];
#pragma unroll
    for (int i = 0; i < kB; ++i) y[i] = 0.0;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
        const int r = lane + 32 * t;
        cr[t] = (t >= t0 && r < m) ? C[r] : 0.0;
#pragma unroll
        for (int i = 0; i < kB; ++i) y[i] += vr[i][t] * cr[t];
    }
    warp_sum_n<kB>(y);
    double w[kB];
#pragma unroll
    for (int i = 0; i < kB; ++i) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l <= i; ++l) s += Tr[l + i * kB] * y[l];
        w[i] = s;
    }
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
        const int r = lane + 32 * t;
        if (t >= t0 && r < m) {
            double v = cr[t];
#pragma unroll
            for (int i = 0; i < kB; ++i) v -= vr[i][t] * w[i];
            C[r] = v;
        }
    }
}

// Back substitution R11 x = r12 by one CTA (R in global memory, column-major, ld ldr), with the
// singularity test |R_ii| <= 1e-14 max |R_jj| and the sketched residual |R_nn|.
// Blocked by 32 from the bottom: warp 0 solves the 32 x 32 diagonal block with the block in
// registers (lane l holds row c0 + l; x_c = y_c * (1/R_cc) broadcast by shuffle), then every
// thread updates one row of y above the block with the block's 32 columns (coalesced L2 reads).
// diag, yv: shared scratch of nc and n doubles.
__device__ void back_substitute(const double* __restrict__ Rg, int ldr, int nc, double* __restrict__ x,
                                SolveStatus* __restrict__ status, double* diag, double* yv) {
    const int n = nc - 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ int s_fail;
    __shared__ double s_wmax[kWarps];
    double mx = 0.0;
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
        const double di = Rg[i + (int64_t)i * ldr];
        diag[i] = di;
        if (i < n) mx = fmax(mx, fabs(di));
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) yv[i] = Rg[i + (int64_t)n * ldr];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) s_wmax[warp] = mx;
    __syncthreads();
    if (warp == 0) {
        double rmax = lane < kWarps ? s_wmax[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
        int bad = 0;
        for (int i = lane; i < n; i += 32) bad |= !(fabs(diag[i]) > 1e-14 * rmax);
        bad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
            status->status = bad ? CSK_ESINGULAR : 0;
            status->sk_resid = fabs(diag[n]);
            s_fail = bad;
        }
    }
    __syncthreads();
    if (s_fail) return;
    for (int c1 = n; c1 > 0; c1 -= 32) {
        const int c0 = max(0, c1 - 32), bs = c1 - c0;
        if (warp == 0) {
            // diagonal block: lane l owns row c0 + l
            double rb[32];
#pragma unroll
            for (int cc = 0; cc < 32; ++cc)
                rb[cc] = (cc < bs && lane < cc) ? Rg[c0 + lane + (int64_t)(c0 + cc) * ldr] : 0.0;
            double yl = lane < bs ? yv[c0 + lane] : 0.0;
            const double rinv = lane < bs ? 1.0 / diag[c0 + lane] : 0.0;
            double xl = 0.0;
#pragma unroll
            for (int cc = 31; cc >= 0; --cc) {
                if (cc < bs) {
                    const double xc = __shfl_sync(0xffffffffu, yl * rinv, cc);
                    if (lane == cc) xl = xc;
                    yl -= rb[cc] * xc;   // rb[cc] = 0 for lane >= cc
                }
            }
            if (lane < bs) {
                yv[c0 + lane] = xl;   // x of the block, read by the update below
                x[c0 + lane] = xl;
            }
        }
        __syncthreads();
        if (c0 > 0) {
            for (int i = threadIdx.x; i < c0; i += blockDim.x) {
                double s = yv[i];
#pragma unroll 8
                for (int cc = 0; cc < bs; ++cc) s -= Rg[i + (int64_t)(c0 + cc) * ldr] * yv[c0 + cc];
                yv[i] = s;
            }
            __syncthreads();
        }
    }
}

__host__ __device__ inline size_t wy_smem_doubles(int m, int nc, int P) {
    const int ldw = (m + 1) & ~1;
    const int npan = (nc + kB - 1) / kB;
    const int nlp = (npan + P - 1) / P;
    return (size_t)nlp * kB * ldw + 2 * (size_t)kB * ldw + 2 * kB * kB;
}

template <int RPL>
__global__ void __launch_bounds__(kThreads, 1) qr_wy_kernel(WyArgs a) {
    const int P = a.P;
    const int rank = P > 1 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
    const int m = a.m, nc = a.nc, npan = a.npan, ldw = a.ldw;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nlp = (npan - rank + P - 1) / P;   // local panels: global panel rank + P*lp
    const int nlp_max = (npan + P - 1) / P;      // identical layout in every CTA
    extern __shared__ __align__(16) double sm[];
    double* Wl = sm;                                     // [nlp_max*kB][ldw] local columns
    double* Vst = Wl + (size_t)nlp_max * kB * ldw;       // [2][kB][ldw] V of the current/next panel
    double* Tst = Vst + 2 * (size_t)kB * ldw;            // [2][kB*kB]
    __shared__ double s_rbuf[2 * kTeamWarps * 16];       // team reduction ring
    __shared__ int s_ctr[2];                             // trailing-column work counters (per step parity)
    if (threadIdx.x == 0) QPROF(npan, 0);
    // local columns (zero padding past nc); one column per warp iteration, RPL loads in flight
    for (int lc = warp; lc < nlp * kB; lc += kWarps) {
        const int gcol = (rank + P * (lc / kB)) * kB + (lc % kB);
        double v[RPL];
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
            const int r = lane + 32 * t;
            v[t] = (gcol < nc && r < m) ? __ldg(a.Z + r + (int64_t)gcol * a.ldz) : 0.0;
        }
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
            const int r = lane + 32 * t;
            if (r < m) Wl[(size_t)lc * ldw + r] = v[t];
        }
    }
    if (threadIdx.x == 0) s_ctr[0] = 0;
    __syncthreads();
    if (threadIdx.x == 0) QPROF(npan, 1);
    if (rank == 0 && warp < kTeamWarps) factor_panel<RPL>(a, Wl, 0, Vst, Tst, nullptr, nullptr, s_rbuf);
    if (threadIdx.x == 0) QPROF(npan, 2);
    for (int k = 0; k < npan; ++k) {
        sync_all(P);   // panel k factored and published
        if (threadIdx.x == 0) QPROF(k, 0);
        if (threadIdx.x == kThreads - 1) QPROF(k, 4);
        if (threadIdx.x == kThreads - 1) s_ctr[(k + 1) & 1] = 0;   // last used in step k-1
        const int owner = k % P, j0 = k * kB, buf = k & 1, t0 = j0 >> 5;
        double* V = Vst + (size_t)buf * kB * ldw;
        double* T = Tst + buf * kB * kB;
        if (rank != owner) {
            const double* Vgk = a.Vg + (size_t)k * kB * ldw;
            const int r0 = t0 * 32;
            const int len = m - r0;
            for (int e = threadIdx.x; e < kB * len; e += kThreads) {
                const int c = e / len, r = r0 + (e - c * len);
                V[c * ldw + r] = __ldcg(Vgk + c * ldw + r);
            }
            if (threadIdx.x < kB * kB) T[threadIdx.x] = __ldcg(a.Tg + (size_t)k * kB * kB + threadIdx.x);
            __syncthreads();
        }
        if (threadIdx.x == 0) QPROF(k, 1);
        const bool la = (k + 1 < npan) && rank == (k + 1) % P;
        const int lp_next = la ? (k + 1) / P : -1;
        if (la && warp < kTeamWarps) {
            const int nb = (k + 1) & 1;
            factor_panel<RPL>(a, Wl + (size_t)lp_next * kB * ldw, k + 1, Vst + (size_t)nb * kB * ldw,
                              Tst + nb * kB * kB, V, T, s_rbuf);
            if (threadIdx.x == 0) QPROF(k, 2);
        }
        // trailing local columns (global panel index > k, panel k+1 excluded when la), handed out
        // one at a time; the panel team joins when it is done
        const int lp0 = k - rank >= 0 ? (k - rank) / P + 1 : 0;
        const int ncols = (nlp - lp0) * kB;
        if (ncols <= 0) {
            if (threadIdx.x == 0) QPROF(k, 3);
            if (threadIdx.x == kThreads - 1) QPROF(k, 5);
            continue;
        }
        bool have_v = false;
        double vr[kB][RPL];
        double Tr[kB * kB];
        for (;;) {
            int q = 0;
            if (lane == 0) q = atomicAdd(&s_ctr[k & 1], 1);
            q = __shfl_sync(0xffffffffu, q, 0);
            if (q >= ncols) break;
            const int lc = lp0 * kB + q;
            const int lp = lc / kB;
            if (lp == lp_next) continue;
            const int gcol = (rank + P * lp) * kB + (lc % kB);
            if (gcol >= nc) continue;
            if (!have_v) {
#pragma unroll
                for (int i = 0; i < kB; ++i)
#pragma unroll
                    for (int t = 0; t < RPL; ++t) {
                        const int r = lane + 32 * t;
                        vr[i][t] = (t >= t0 && r < m) ? V[i * ldw + r] : 0.0;
                    }
#pragma unroll
                for (int e = 0; e < kB * kB; ++e) Tr[e] = T[e];
                have_v = true;
            }
            apply_wy<RPL>(Wl + (size_t)lc * ldw, vr, Tr, t0, m);
        }
        if (threadIdx.x == 0) QPROF(k, 3);
        if (threadIdx.x == kThreads - 1) QPROF(k, 5);
    }
    sync_all(P);   // all of R written
    if (threadIdx.x == 0) QPROF(npan, 3);
    if (rank != 0) return;
    back_substitute(a.Rg, a.ldr, nc, a.x, a.status, Vst, Vst + nc);
    if (threadIdx.x == 0) QPROF(npan, 4);
}

}  // namespace

#ifdef CSK_QR_PROFILE
long long* qr_wy_prof_buffer = nullptr;
#endif

// Launch the register-blocked solve when Z fits the shared memory of <= 16 CTAs and m <= 512.
// *launched = false (and CSK_OK) when the shape is outside that envelope.
csk_status qr_wy_launch(const double* Z, int64_t ldz, int m, int nc, double* Rg, int ldr, double* scratch,
                        double* x, SolveStatus* status, cudaStream_t st, bool* launched) {
    *launched = false;
    if (const char* e = std::getenv("CSK_QR_WY"))
        if (std::atoi(e) == 0) return CSK_OK;
    if (m > 512 || nc < 2) return CSK_OK;
    const DeviceInfo& di = device_info();
    const int npan = (nc + kB - 1) / kB;
    int P = 0;
    for (int p = 1; p <= 16; p *= 2)
        if (wy_smem_doubles(m, nc, p) * 8 <= (size_t)di.smem_optin) {
            P = p;
            break;
        }
    if (P == 0) return CSK_OK;
    if (const char* e = std::getenv("CSK_QR_WY_P")) P = std::max(P, std::min(16, std::atoi(e)));
    P = std::min(P, npan);
    const size_t smem = wy_smem_doubles(m, nc, P) * 8;
    WyArgs a;
    a.Z = Z;
    a.ldz = ldz;
    a.m = m;
    a.nc = nc;
    a.P = P;
    a.npan = npan;
    a.ldw = (m + 1) & ~1;
    a.Vg = scratch;
    a.Tg = scratch + (size_t)npan * kB * a.ldw;
    a.Rg = Rg;
    a.ldr = ldr;
    a.x = x;
    a.status = status;
#ifdef CSK_QR_PROFILE
    a.prof = qr_wy_prof_buffer;
#endif
    void (*kern)(WyArgs) = m <= 128 ? qr_wy_kernel<4> : (m <= 256 ? qr_wy_kernel<8> : qr_wy_kernel<16>);
    CSK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (P > 8) CSK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CSK_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a));
    CSK_LAUNCH_CHECK();
    *launched = true;
    return CSK_OK;
}

size_t qr_wy_scratch_doubles(int m, int nc) {
    const int npan = (nc + kB - 1) / kB;
    return (size_t)npan * kB * ((m + 1) & ~1) + (size_t)npan * kB * kB;
}

}  // namespace csk
