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
    int push;   // DSMEM push of V/T to the next panel owner (CSK_QR_PUSH=0 disables, for A/B)
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

// Warp reduce-scatter of N = 2^K values (B300_MICROARCH / scripts/lat_bench.cu: a 64-bit shuffle
// costs ~5 issue cycles, so a full 5-level butterfly of 8 values takes ~420 cycles; halving the
// vector at each of the first K levels needs N - 1 + (5 - K) shuffles instead of 5 N).
// Returns the warp total of value lane >> (5 - K); lanes sharing those top K bits hold
// bit-identical totals (every add pairs the same two partials).
template <int K>
__device__ __forceinline__ double warp_reduce_scatter(double* v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int lev = 0; lev < K; ++lev) {
        const int o = 16 >> lev, n = (1 << K) >> (lev + 1);
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < n; ++i) {
            const double send = up ? v[i] : v[i + n];
            const double keep = up ? v[i + n] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    double r = v[0];
#pragma unroll
    for (int o = 16 >> K; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    return r;
}

// Sum 2^K per-thread partials over the panel team; every team thread gets the bit-identical
// totals.  Warp reduce-scatter, one lane per value stores its warp total, named barrier, lane i
// adds value i over the four warps (fixed order) into a per-warp slot, every lane reads all.
// buf: [2][kTeamWarps][16] ring (ph alternates per call: one team barrier per call suffices);
// tot: [kTeamWarps][16] per-warp totals.
template <int K>
__device__ __forceinline__ void team_sum(double* v, double* buf, double* tot, int& ph) {
    constexpr int N = 1 << K;
    static_assert(N <= 16, "team_sum: N <= 16");
    const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
    const double r = warp_reduce_scatter<K>(v);
    double* b = buf + ph * (kTeamWarps * 16);
    if ((lane & ((32 >> K) - 1)) == 0) b[q * 16 + (lane >> (5 - K))] = r;
    team_bar();
    double* t = tot + q * 16;
    if (lane < N) t[lane] = ((b[lane] + b[16 + lane]) + b[32 + lane]) + b[48 + lane];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = t[i];
    __syncwarp();   // t is rewritten by this warp's next call
    ph ^= 1;
}

// The panel team of the owner CTA: load panel kp (local shared-memory columns `cols`) into
// registers, optionally apply the previous panel's Q^T (Vin, Tin in shared memory), factor it,
// write R (rows <= diagonal) to global, V/T to shared memory (and to global when P > 1).
template <int RPL>
__device__ __forceinline__ void factor_panel(const WyArgs& a, const double* cols, int kp, double* Vout, double* Tout,
                                             const double* Vin, const double* Tin, double* rbuf, double* rtot) {
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
        team_sum<4>(y, rbuf, rtot, ph);
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
        team_sum<3>(red, rbuf, rtot, ph);
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
    double g[8];   // 6 Gram entries, padded to 2^3 for the reduction
#pragma unroll
    for (int e = 0; e < 8; ++e) g[e] = 0.0;
#pragma unroll
    for (int u = 0; u < RPLT; ++u) {
        int e = 0;
#pragma unroll
        for (int l = 1; l < kB; ++l)
#pragma unroll
            for (int i = 0; i < l; ++i) g[e++] += p[i][u] * p[l][u];
    }
    team_sum<3>(g, rbuf, rtot, ph);
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
    // the owner of panel kp + 1 applies Q_kp to its panel on the critical path of the next step: push
    // V and T straight into its shared memory (same buffer offset, DSMEM) so it skips the L2 staging
    // after the cluster barrier (2.7 K cycles per step at 256 x 129, scripts/qr_wy_prof.cu)
    double* Vrem = nullptr;
    double* Trem = nullptr;
    if (pub && a.push && kp + 1 < a.npan) {
        cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
        const unsigned nxt = (unsigned)((kp + 1) % a.P);
        Vrem = cl.map_shared_rank(Vout, nxt);
        Trem = cl.map_shared_rank(Tout, nxt);
    }
#pragma unroll
    for (int c = 0; c < kB; ++c)
#pragma unroll
        for (int u = 0; u < RPLT; ++u) {
            const int tb = q + kTeamWarps * u, r = 32 * tb + lane;
            if (tb >= t0 && r < m) {
                Vout[c * ldw + r] = p[c][u];
                if (pub) Vgk[c * ldw + r] = p[c][u];
                if (Vrem) Vrem[c * ldw + r] = p[c][u];
            }
        }
    if (threadIdx.x < kB * kB) {
        double tv = 0.0;
#pragma unroll
        for (int e = 0; e < kB * kB; ++e)
            if ((int)threadIdx.x == e) tv = T[e];
        Tout[threadIdx.x] = tv;
        if (pub) a.Tg[(size_t)kp * kB * kB + threadIdx.x] = tv;
        if (Trem) Trem[threadIdx.x] = tv;
    }
}

// Trailing update of up to 4 shared-memory columns by one warp, a quarter-warp (8 lanes) per
// column: C -= V (T^T (V^T C)) over rows >= r0 (V is zero above its pivots).  The V^T C
// reduction is 3 shuffle levels within the quarter, shared by the 4 columns (24 shuffles per 4
// columns instead of 40 per column for a full-warp butterfly); V rows are broadcast LDS.
__device__ __forceinline__ void apply_wy4(double* C, bool active, const double* V, int ldw, const double* Tr, int r0,
                                          int m) {
    const int sub = threadIdx.x & 7;
    double y[kB];
#pragma unroll
    for (int i = 0; i < kB; ++i) y[i] = 0.0;
    if (active) {
#pragma unroll 4
        for (int r = r0 + sub; r < m; r += 8) {
            const double c = C[r];
#pragma unroll
            for (int i = 0; i < kB; ++i) y[i] += V[i * ldw + r] * c;
        }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
#pragma unroll
        for (int i = 0; i < kB; ++i) y[i] += __shfl_xor_sync(0xffffffffu, y[i], o);
    }
    if (!active) return;
    double w[kB];
#pragma unroll
    for (int i = 0; i < kB; ++i) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l <= i; ++l) s += Tr[l + i * kB] * y[l];
        w[i] = s;
    }
#pragma unroll 4
    for (int r = r0 + sub; r < m; r += 8) {
        double c = C[r];
#pragma unroll
        for (int i = 0; i < kB; ++i) c -= V[i * ldw + r] * w[i];
        C[r] = c;
    }
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Back substitution R11 x = r12 by one CTA (R in global memory, column-major, ld ldr), with the
// singularity test |R_ii| <= 1e-14 max |R_jj| and the sketched residual |R_nn|.
// Blocked by 32 columns from the bottom.  Block column R[0:c1, c0:c1] is prefetched into shared
// memory (cp.async, double-buffered) while the previous block is solved; warp 0 solves the
// diagonal block (lane l owns row c0 + l; x_c = y_c * (1/R_cc) broadcast by shuffle), then each
// thread updates one row of y above the block.
// diag, yv: shared scratch of nc and n doubles; rbuf: shared scratch of 2 * 32 * n doubles.
__device__ void back_substitute(const double* __restrict__ Rg, int ldr, int nc, double* __restrict__ x,
                                SolveStatus* __restrict__ status, double* diag, double* yv, double* rbuf) {
    const int n = nc - 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ int s_fail;
    __shared__ double s_wmax[kWarps];
    // block column b covers columns [c0, c1) with c1 = n - 32 b; its rows [0, c1) go to
    // rbuf[(b & 1) * 32 * n + cc * c1 + r]
    auto prefetch = [&](int c1) {
        const int c0 = max(0, c1 - 32), bs = c1 - c0;
        double* dst = rbuf + (size_t)(((n - c1) / 32) & 1) * 32 * n;
        if (((ldr | c1) & 1) == 0) {   // 16-B chunks (ldr, c1 even: Rg columns and rbuf rows 16-B aligned)
            const int h = c1 >> 1;
            for (int cc = warp; cc < bs; cc += kWarps)
                for (int e = lane; e < h; e += 32) cp_async16(dst + cc * c1 + 2 * e, Rg + 2 * e + (int64_t)(c0 + cc) * ldr);
        } else {
            for (int cc = warp; cc < bs; cc += kWarps)
                for (int r = lane; r < c1; r += 32) cp_async8(dst + cc * c1 + r, Rg + r + (int64_t)(c0 + cc) * ldr);
        }
        cp_async_commit();
    };
    prefetch(n);
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
    if (s_fail) {
        cp_async_wait_all();
        return;
    }
    for (int c1 = n; c1 > 0; c1 -= 32) {
        const int c0 = max(0, c1 - 32), bs = c1 - c0;
        const double* Rb = rbuf + (size_t)(((n - c1) / 32) & 1) * 32 * n;   // [bs][c1]
        cp_async_wait_all();
        __syncthreads();
        if (c0 > 0) prefetch(c0);   // next block column streams in while this one is solved
        if (warp == 0) {
            double rb[32];
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) rb[cc] = (cc < bs && lane < cc) ? Rb[cc * c1 + c0 + lane] : 0.0;
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
        for (int i = threadIdx.x; i < c0; i += blockDim.x) {
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int cc = 0;
            for (; cc + 4 <= bs; cc += 4) {
                s0 += Rb[cc * c1 + i] * yv[c0 + cc];
                s1 += Rb[(cc + 1) * c1 + i] * yv[c0 + cc + 1];
                s2 += Rb[(cc + 2) * c1 + i] * yv[c0 + cc + 2];
                s3 += Rb[(cc + 3) * c1 + i] * yv[c0 + cc + 3];
            }
            for (; cc < bs; ++cc) s0 += Rb[cc * c1 + i] * yv[c0 + cc];
            yv[i] -= (s0 + s1) + (s2 + s3);
        }
    }
}

// column stride: even (16-B vectors) and = 8 mod 16 doubles, so the two quarter-warps of a
// half-warp (same rows of adjacent columns) hit disjoint shared-memory banks in apply_wy4
__host__ __device__ inline int wy_ldw(int m) { return ((m + 15) & ~15) + 8; }

// local-column region: the CTA's panels, and (CTA 0, after the factorization) the two
// back-substitution block-column buffers of 32 x n doubles
__host__ __device__ inline size_t wy_local_doubles(int m, int nc, int P) {
    const int ldw = wy_ldw(m);
    const int npan = (nc + kB - 1) / kB;
    const int nlp = (npan + P - 1) / P;
    const size_t cols = (size_t)nlp * kB * ldw, bsub = (size_t)2 * 32 * (nc - 1);
    return cols > bsub ? cols : bsub;
}
__host__ __device__ inline size_t wy_smem_doubles(int m, int nc, int P) {
    const int ldw = wy_ldw(m);
    return wy_local_doubles(m, nc, P) + 2 * (size_t)kB * ldw + 2 * kB * kB;
}

template <int RPL>
__global__ void __launch_bounds__(kThreads, 1) qr_wy_kernel(WyArgs a) {
    const int P = a.P;
    const int rank = P > 1 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
    const int m = a.m, nc = a.nc, npan = a.npan, ldw = a.ldw;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nlp = (npan - rank + P - 1) / P;   // local panels: global panel rank + P*lp
    extern __shared__ __align__(16) double sm[];
    double* Wl = sm;                                             // [nlp_max*kB][ldw] local columns
    double* Vst = Wl + wy_local_doubles(m, nc, P);               // [2][kB][ldw] V of the current/next panel
    double* Tst = Vst + 2 * (size_t)kB * ldw;                    // [2][kB*kB]
    __shared__ __align__(16) double s_rbuf[2 * kTeamWarps * 16];   // team reduction ring
    __shared__ __align__(16) double s_rtot[kTeamWarps * 16];       // team totals (per warp)
    __shared__ int s_ctr[2];                                     // trailing-panel work counters (step parity)
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
    if (rank == 0 && warp < kTeamWarps) factor_panel<RPL>(a, Wl, 0, Vst, Tst, nullptr, nullptr, s_rbuf, s_rtot);
    if (threadIdx.x == 0) QPROF(npan, 2);
    for (int k = 0; k < npan; ++k) {
        sync_all(P);   // panel k factored and published
        if (threadIdx.x == 0) QPROF(k, 0);
        if (threadIdx.x == kThreads - 1) QPROF(k, 4);
        if (threadIdx.x == kThreads - 1) s_ctr[(k + 1) & 1] = 0;   // last used in step k-1
        const int owner = k % P, j0 = k * kB, buf = k & 1;
        double* V = Vst + (size_t)buf * kB * ldw;
        double* T = Tst + buf * kB * kB;
        // the owner of panel k + 1 received V_k and T_k by DSMEM from the owner of panel k (factor_panel)
        const bool pushed = a.push && P > 1 && k + 1 < npan && rank == (k + 1) % P;
        if (rank != owner && !pushed) {
            // V rows >= 32*(j0/32) of the 4 columns (16-B vectors; ldw and the row start are even)
            const double* Vgk = a.Vg + (size_t)k * kB * ldw;
            const int r0 = (j0 >> 5) * 32, h = (m - r0 + 1) >> 1;
#pragma unroll
            for (int c = 0; c < kB; ++c) {
                const double2* src = reinterpret_cast<const double2*>(Vgk + (size_t)c * ldw + r0);
                double2* dst = reinterpret_cast<double2*>(V + (size_t)c * ldw + r0);
                for (int e = threadIdx.x; e < h; e += kThreads) dst[e] = __ldcg(src + e);
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
                              Tst + nb * kB * kB, V, T, s_rbuf, s_rtot);
            if (threadIdx.x == 0) QPROF(k, 2);
        }
        // trailing local panels (global index > k; panel k+1 excluded when la), one panel of 4
        // columns per warp at a time (quarter-warp per column), handed out by a shared counter;
        // the panel team joins when it is done
        const int lp0 = k - rank >= 0 ? (k - rank) / P + 1 : 0;
        const int npl = nlp - lp0;
        if (npl > 0) {
            double Tr[kB * kB];
#pragma unroll
            for (int e = 0; e < kB * kB; ++e) Tr[e] = T[e];
            const int r0 = j0 & ~7;
            for (;;) {
                int q = 0;
                if (lane == 0) q = atomicAdd(&s_ctr[k & 1], 1);
                q = __shfl_sync(0xffffffffu, q, 0);
                if (q >= npl) break;
                const int lp = lp0 + q;
                if (lp == lp_next) continue;
                const int g = lane >> 3;
                const int gcol = (rank + P * lp) * kB + g;
                apply_wy4(Wl + (size_t)(lp * kB + g) * ldw, gcol < nc, V, ldw, Tr, r0, m);
            }
        }
        if (threadIdx.x == 0) QPROF(k, 3);
        if (threadIdx.x == kThreads - 1) QPROF(k, 5);
    }
    sync_all(P);   // all of R written
    if (threadIdx.x == 0) QPROF(npan, 3);
    if (rank != 0) return;
    back_substitute(a.Rg, a.ldr, nc, a.x, a.status, Vst, Vst + nc, Wl);
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
    // wide sketches: a 16-CTA cluster (measured, scripts/solve_timing.py: 256 x 129 280 -> 235 us,
    // 512 x 257 575 -> 502 us; 128 x 65 is fastest on one CTA, 110 vs 132 us)
    if (m >= 256 && nc >= 64) P = 16;
    if (const char* e = std::getenv("CSK_QR_WY_P"))
        if (*e) P = std::max(P, std::min(16, std::atoi(e)));
    P = std::min(P, npan);
    const size_t smem = wy_smem_doubles(m, nc, P) * 8;
    WyArgs a;
    a.Z = Z;
    a.ldz = ldz;
    a.m = m;
    a.nc = nc;
    a.P = P;
    a.npan = npan;
    a.ldw = wy_ldw(m);
    a.Vg = scratch;
    a.Tg = scratch + (size_t)npan * kB * a.ldw;
    a.Rg = Rg;
    a.ldr = ldr;
    a.x = x;
    a.status = status;
    {
        const char* pe = std::getenv("CSK_QR_PUSH");
        a.push = !(pe && std::atoi(pe) == 0);
    }
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
    return (size_t)npan * kB * wy_ldw(m) + (size_t)npan * kB * kB;
}

}  // namespace csk
