// randcholqr.cu -- rc_lstsq: rand_cholQR least squares, Alg 5.
//
//   1  Y = S A                    ms_apply_impl on [A b] (the multisketch G S1 of this path, R23)
//   2  [~, R0] = qr(Y, 0)         the cluster Householder QR of ms_solve (R0 = R[:n,:n] of [Y | Sb])
//   3  Q0 = A R0^-1               row-chunked TRSM (R24: a triangular solve, not an explicit inverse)
//   4  G = Q0^T Q0, z = Q0^T b    accumulated chunk by chunk while the chunk is L2-resident
//   5  R1 = chol(G)               chol_solve_kernel (normal_eq.cu), which also returns u = R1^-1 R1^-T z
//   6  R = R1 R0                  rc_finish_kernel (only when the caller asks for R)
//   7-8 x = R^-1 R1^-T z          = R0^-1 u (R23), rc_finish_kernel
//
// Lines 3-4 are the single pass over A: each chunk of rows is copied into an
// L2-sized workspace, solved in place against R0 (cuBLAS DTRSM), and folded into the Gram with
// DGEMM (Q0^T Q0, n x n: the K = rows split keeps it at the DMMA roofline when n is a multiple of
// 64) and DGEMV (Q0^T b); Q0 never reaches HBM as a whole.
#include <algorithm>
#include <cstdlib>

#include <cublas_v2.h>

#include "csk_internal.cuh"

namespace csk {

// x = R0^-1 u (back substitution, R0 upper n x n, ld ldr0), and optionally R = R1 R0 with R1 the
// upper Cholesky factor left in S (ld nc).  One CTA.
__global__ void __launch_bounds__(1024, 1) rc_finish_kernel(const double* __restrict__ R0, int ldr0,
                                                            const double* __restrict__ S, int nc, int n,
                                                            const double* __restrict__ u, double* __restrict__ x,
                                                            double* __restrict__ R, int ldr,
                                                            const int* __restrict__ chol_status) {
    if (*chol_status != 0) return;
    extern __shared__ double fsm[];
    double* y = fsm;   // n
    for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = u[i];
    __syncthreads();
    for (int c = n - 1; c >= 0; --c) {
        const double xc = y[c] / R0[c + (int64_t)c * ldr0];
        __syncthreads();
        for (int i = threadIdx.x; i < c; i += blockDim.x) y[i] -= R0[i + (int64_t)c * ldr0] * xc;
        if (threadIdx.x == 0) x[c] = xc;
        __syncthreads();
    }
    if (R != nullptr) {
        // R[i,j] = sum_{l=i..j} R1[i,l] R0[l,j]
        for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
            const int i = e % n, j = e / n;
            double acc = 0.0;
            for (int l = i; l <= j; ++l) acc += S[i + (int64_t)l * nc] * R0[l + (int64_t)j * ldr0];
            R[i + (int64_t)j * ldr] = i <= j ? acc : 0.0;
        }
    }
}

// ---------------------------------------------------------------- fused pass (lines 3-4)
// One persistent CTA per SM walks 64-row tiles of A; fp64 tensor cores (DMMA 8x8x4, the native fp64
// MMA of sm_100a: every f64 mma.sync shape lowers to it) do both halves, and Q0 never reaches HBM:
//  * TRSM (line 3, R24): rows are independent, so a TRSM warp solves its own rows with no CTA
//    barrier: for each 8-column block J, T = A[:, J] - Q[:, <J] R0[<J, J] (DMMAs with the warp's Q
//    rows as the A operand and packed R0 from shared memory as B), then Q[:, J] = T W_J with W_J the
//    8x8 inverse of the diagonal block (two DMMAs);
//  * Gram (line 4): Gram warps accumulate Q^T Q of the previous tile into the upper 8x8 blocks
//    (accumulators in registers for the whole kernel) and z = Q^T b with plain FMAs.
// Each CTA writes its partial [C | z] once; rc_reduce_kernel sums the partials in a fixed order.
// Shared memory: packed upper R0 (8-column blocks), Q as [row][col] with ld = NP + 4 (== 4 mod 16
// doubles: the fragment loads of a half-warp touch 16 distinct bank pairs).

__device__ __forceinline__ double ldcs_pred_rc(const double* p, bool pred) {
    double v = 0.0;
    asm("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.global.cs.f64 %0, [%1]; }" : "+d"(v) : "l"(p), "r"((int)pred));
    return v;
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Packed upper R0: 8-column block J holds rows 0 .. 8J+7 of its columns with ld 8J + 12
// (== 4 or 12 mod 16: conflict-free fragment loads), at offset 32 J (J-1) + 96 J.
__host__ __device__ constexpr int rc_r0_off(int J) { return 32 * J * (J - 1) + 96 * J; }

// ------------------------------------------------------------ warp-specialised pipeline
// The two halves overlap: TRSM warps and Gram warps, Q tiles double-buffered in shared memory and
// handed over with named barriers (FULL[q]: TRSM -> Gram, EMPTY[q]: Gram -> TRSM), so the
// latency-bound TRSM chain of tile i+1 runs under the DMMA-bound Gram of tile i.  (Round 1 also
// kept the unpipelined kernel and a 32-row, one-group-per-warp version of this pipeline; both were
// slower than v3 -- 17.65 / 14.15 ms vs 10.38 ms at C4, DESIGN.md 6.4 -- and were removed in round 2.)
constexpr int kWsSolve = 4, kWsGram = 4;

__device__ __forceinline__ void nbar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ----------------------------------------------------- v3: two row groups per TRSM warp
// Each TRSM warp solves 16 rows of a 64-row tile as two independent
// 8-row groups (twice the DMMA chains per warp: the TRSM was the limiter), the R0 B-fragment is
// shared by both groups, and A is not staged in shared memory: every lane keeps a ring of P
// prefetched column blocks in registers (the TRSM warps have the Gram warps' register budget).
// Shared memory: packed R0, 2 x 64-row Q buffers, the 8x8 diagonal inverses, b.
constexpr int kV3Rows = 64;

template <int NB>
__global__ void __launch_bounds__((kWsSolve + kWsGram) * 32, 1)
    rc_pass_v3_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ b, int64_t d, int n,
                      const double* __restrict__ R0g, int ldr0g, double* __restrict__ part, int nc) {
    constexpr int NP = 8 * NB, LD = NP + 4;
    constexpr int P = NB < 8 ? NB : 8;                                   // prefetch distance (column blocks)
    constexpr int NPAIR = NB / 2;
    constexpr int PPW = NPAIR >= kWsGram ? NPAIR / kWsGram : 1;
    constexpr int KS = NPAIR >= kWsGram ? 1 : kWsGram / NPAIR;
    constexpr int GK = kV3Rows / KS;
    constexpr int NSLOT = PPW * (NB + 1);
    extern __shared__ __align__(16) double rsm[];
    double* R0p = rsm;                                   // packed upper R0
    double* Qs = R0p + rc_r0_off(NB);                    // [2][kV3Rows][LD]
    double* bs = Qs + 2 * kV3Rows * LD;                  // [2][kV3Rows]
    double* invd = bs + 2 * kV3Rows;                     // [NP]
    double* Wd = invd + NP;                              // [NB][8][12]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    for (int J = 0; J < NB; ++J)
        for (int e = threadIdx.x; e < 8 * (8 * J + 8); e += blockDim.x) {
            const int k = e % (8 * J + 8), j = 8 * J + e / (8 * J + 8);
            const double v = (k < n && j < n) ? R0g[k + (int64_t)j * ldr0g] : (k == j ? 1.0 : 0.0);
            R0p[rc_r0_off(J) + (j - 8 * J) * (8 * J + 12) + k] = (k <= j) ? v : 0.0;
            if (k == j) invd[j] = 1.0 / v;
        }
    __syncthreads();
    for (int e = threadIdx.x; e < NB * 8; e += blockDim.x) {
        const int J = e >> 3, c = e & 7;
        const double* rd = R0p + rc_r0_off(J) + 8 * J;
        const int ldJ = 8 * J + 12;
        double w[8];
#pragma unroll
        for (int r = 7; r >= 0; --r) {
            double acc = (r == c) ? 1.0 : 0.0;
#pragma unroll
            for (int l = r + 1; l < 8; ++l) acc -= rd[l * ldJ + r] * w[l];
            w[r] = acc * invd[8 * J + r];
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) Wd[J * 96 + c * 12 + r] = w[r];
    }
    __syncthreads();
    const int64_t ntiles = (d + kV3Rows - 1) / kV3Rows;
    const int64_t my = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (warp < kWsSolve) {
        // ================================================================ TRSM warps
        // prefetch ring: slot J % P holds A[rowA/rowB, 8J + 2t + {0,1}] of the step being prefetched
        double pa0[P], pa1[P], pb0[P], pb1[P];
        auto load_step = [&](int64_t i, int J, double& a0, double& a1, double& b0, double& b1) {
            const int64_t r0 = (blockIdx.x + i * gridDim.x) * kV3Rows + 16 * warp + g;
            const int c0 = 8 * J + 2 * t;
            const bool ok = i < my;
            const bool va = ok && r0 < d, vb = ok && r0 + 8 < d;
            const double* p0 = A + (int64_t)min(c0, n - 1) * lda;
            const double* p1 = A + (int64_t)min(c0 + 1, n - 1) * lda;
            const int64_t ra = va ? r0 : 0, rb = vb ? r0 + 8 : 0;
            a0 = ldcs_pred_rc(p0 + ra, va && c0 < n);
            a1 = ldcs_pred_rc(p1 + ra, va && c0 + 1 < n);
            b0 = ldcs_pred_rc(p0 + rb, vb && c0 < n);
            b1 = ldcs_pred_rc(p1 + rb, vb && c0 + 1 < n);
        };
#pragma unroll
        for (int J = 0; J < P; ++J) load_step(0, J, pa0[J], pa1[J], pb0[J], pb1[J]);
        double bnext = 0.0;   // b of this lane's row (lanes 0..15: rows 16w + lane) for tile i
        {
            const int64_t r = (int64_t)blockIdx.x * kV3Rows + 16 * warp + lane;
            bnext = (lane < 16 && my > 0 && r < d) ? __ldcs(b + r) : 0.0;
        }
        for (int64_t i = 0; i < my; ++i) {
            const int q = (int)(i & 1);
            const double bcur = bnext;
            {
                const int64_t r = (blockIdx.x + (i + 1) * gridDim.x) * kV3Rows + 16 * warp + lane;
                bnext = (lane < 16 && i + 1 < my && r < d) ? __ldcs(b + r) : 0.0;
            }
            if (i >= 2) nbar_sync(3 + q, 256);                 // EMPTY[q]
            double* qs = Qs + q * kV3Rows * LD;
            double* qrowA = qs + (16 * warp + g) * LD;
            double* qrowB = qrowA + 8 * LD;
#pragma unroll
            for (int J = 0; J < NB; ++J) {
                constexpr int dummy = 0;
                (void)dummy;
                double tA0 = pa0[J % P], tA1 = pa1[J % P], tB0 = pb0[J % P], tB1 = pb1[J % P];
                if (J + P < NB)
                    load_step(i, J + P, pa0[J % P], pa1[J % P], pb0[J % P], pb1[J % P]);
                else
                    load_step(i + 1, J + P - NB, pa0[J % P], pa1[J % P], pb0[J % P], pb1[J % P]);
                double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0, b00 = 0.0, b01 = 0.0, b10 = 0.0, b11 = 0.0;
                const double* qa = qrowA + t;
                const double* qb = qrowB + t;
                const double* rb = R0p + rc_r0_off(J) + g * (8 * J + 12) + t;
#pragma unroll
                for (int k = 0; k < 8 * J; k += 8) {
                    const double r0v = rb[k], r1v = rb[k + 4];
                    dmma884(a00, a01, qa[k], r0v);
                    dmma884(b00, b01, qb[k], r0v);
                    dmma884(a10, a11, qa[k + 4], r1v);
                    dmma884(b10, b11, qb[k + 4], r1v);
                }
                tA0 -= a00 + a10;
                tA1 -= a01 + a11;
                tB0 -= b00 + b10;
                tB1 -= b01 + b11;
                // Q[:, J] = T W_J (W_J = R_JJ^-1; A operand T[g][t], T[g][t+4] by shuffles)
                const int src0 = (lane & ~3) | (t >> 1), src1 = (lane & ~3) | (2 + (t >> 1));
                const double xa00 = __shfl_sync(0xffffffffu, tA0, src0), xa01 = __shfl_sync(0xffffffffu, tA1, src0);
                const double xa10 = __shfl_sync(0xffffffffu, tA0, src1), xa11 = __shfl_sync(0xffffffffu, tA1, src1);
                const double xb00 = __shfl_sync(0xffffffffu, tB0, src0), xb01 = __shfl_sync(0xffffffffu, tB1, src0);
                const double xb10 = __shfl_sync(0xffffffffu, tB0, src1), xb11 = __shfl_sync(0xffffffffu, tB1, src1);
                const double* wb = Wd + J * 96 + g * 12 + t;
                const double w0 = wb[0], w1 = wb[4];
                double qa0 = 0.0, qa1 = 0.0, qb0 = 0.0, qb1 = 0.0;
                dmma884(qa0, qa1, (t & 1) ? xa01 : xa00, w0);
                dmma884(qb0, qb1, (t & 1) ? xb01 : xb00, w0);
                dmma884(qa0, qa1, (t & 1) ? xa11 : xa10, w1);
                dmma884(qb0, qb1, (t & 1) ? xb11 : xb10, w1);
                *reinterpret_cast<double2*>(qrowA + 8 * J + 2 * t) = make_double2(qa0, qa1);
                *reinterpret_cast<double2*>(qrowB + 8 * J + 2 * t) = make_double2(qb0, qb1);
                __syncwarp();
            }
            if (lane < 16) bs[q * kV3Rows + 16 * warp + lane] = bcur;
            __threadfence_block();
            nbar_arrive(1 + q, 256);                           // FULL[q]
        }
        for (int64_t i = (my >= 2 ? my - 2 : 0); i < my; ++i) nbar_sync(3 + (int)(i & 1), 256);   // drain EMPTY
    } else {
        // ================================================================ Gram warps
        const int gw = warp - kWsSolve;
        const int pair0 = (gw % (kWsGram / KS)) * PPW, gk0 = (gw / (kWsGram / KS)) * GK;
        double acc[NSLOT][2];
#pragma unroll
        for (int p = 0; p < NSLOT; ++p) acc[p][0] = acc[p][1] = 0.0;
        double zacc0 = 0.0;
        const int gtid = threadIdx.x - kWsSolve * 32;
        for (int64_t i = 0; i < my; ++i) {
            const int q = (int)(i & 1);
            nbar_sync(1 + q, 256);                             // FULL[q]
            const double* qs = Qs + q * kV3Rows * LD;
            const double* qk = qs + (gk0 + t) * LD + g;
#pragma unroll 2
            for (int k = 0; k < GK; k += 4, qk += 4 * LD) {
#pragma unroll
                for (int pp = 0; pp < PPW; ++pp) {
                    const int J1 = pair0 + pp, J2 = NB - 1 - J1;
                    const double b1 = qk[8 * J1], b2 = qk[8 * J2];
#pragma unroll
                    for (int s2 = 0; s2 <= NB; ++s2) {
                        const bool first = s2 <= J1;
                        const int I = first ? s2 : s2 - J1 - 1;
                        dmma884(acc[pp * (NB + 1) + s2][0], acc[pp * (NB + 1) + s2][1], qk[8 * I], first ? b1 : b2);
                    }
                }
            }
            if (gtid < NP) {
                const double* bt = bs + q * kV3Rows;
                double sz = 0.0;
#pragma unroll 4
                for (int r = 0; r < kV3Rows; ++r) sz += qs[r * LD + gtid] * bt[r];
                zacc0 += sz;
            }
            nbar_arrive(3 + q, 256);                           // EMPTY[q]
        }
        double* Pp = part + (size_t)blockIdx.x * nc * nc;
#pragma unroll
        for (int pp = 0; pp < PPW; ++pp) {
            const int J1 = pair0 + pp, J2 = NB - 1 - J1;
#pragma unroll
            for (int s2 = 0; s2 <= NB; ++s2) {
                const bool first = s2 <= J1;
                const int I = first ? s2 : s2 - J1 - 1, J = first ? J1 : J2;
                const int ii = 8 * I + g, j0 = 8 * J + 2 * t;
                if (ii < n && j0 < n) atomicAdd(Pp + ii + (int64_t)j0 * nc, acc[pp * (NB + 1) + s2][0]);
                if (ii < n && j0 + 1 < n) atomicAdd(Pp + ii + (int64_t)(j0 + 1) * nc, acc[pp * (NB + 1) + s2][1]);
            }
        }
        if (gtid < n) atomicAdd(Pp + gtid + (int64_t)(nc - 1) * nc, zacc0);
    }
}

// ------------------------------------------------- wide n (128 < n <= 256): TRSM to a workspace
// The fused kernels keep packed R0 in shared memory, which no longer fits next to the Q tiles past
// n = 128.  Here the TRSM warps of rc_pass_v3_kernel run alone (4 warps x 16 rows = 64-row tiles,
// two 8-row groups per warp, A in a register ring), with the packed R0 and the 8x8 diagonal inverses
// read through the read-only cache from global memory (L2-resident: 0.3 MB at n = 256), the warp's
// Q rows in shared memory, and each finished tile written to the Q0 workspace column by column
// (coalesced); cuBLAS DGEMM/DGEMV then form [Q0^T Q0 | Q0^T b] chunk by chunk.
__global__ void rc_pack_r0_kernel(const double* __restrict__ R0g, int ldr0g, int n, int NB, double* __restrict__ R0p,
                                  double* __restrict__ Wd) {
    // packed upper R0 (as rc_pass_*: block J holds rows 0..8J+7 with ld 8J+12) and W_J = R_JJ^-1
    for (int J = blockIdx.x; J < NB; J += gridDim.x) {
        for (int e = threadIdx.x; e < 8 * (8 * J + 8); e += blockDim.x) {
            const int k = e % (8 * J + 8), j = 8 * J + e / (8 * J + 8);
            const double v = (k < n && j < n) ? R0g[k + (int64_t)j * ldr0g] : (k == j ? 1.0 : 0.0);
            R0p[rc_r0_off(J) + (j - 8 * J) * (8 * J + 12) + k] = (k <= j) ? v : 0.0;
        }
        __syncthreads();
        if (threadIdx.x < 8) {
            const int c = threadIdx.x;
            const double* rd = R0p + rc_r0_off(J) + 8 * J;
            const int ldJ = 8 * J + 12;
            double w[8];
            for (int r = 7; r >= 0; --r) {
                double acc = (r == c) ? 1.0 : 0.0;
                for (int l = r + 1; l < 8; ++l) acc -= rd[l * ldJ + r] * w[l];
                w[r] = acc / rd[r * ldJ + r];
            }
            for (int r = 0; r < 8; ++r) Wd[J * 96 + c * 12 + r] = w[r];
        }
        __syncthreads();
    }
}

// R0 block column J (packed, 64 J + 96 doubles) followed by W_J (96 doubles): the per-J shared stage
__host__ __device__ constexpr int rc_blk_doubles(int J) { return 64 * J + 96 + 96; }

__device__ __forceinline__ void rc_cp16(double* dst, const double* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}

template <int NB>
__global__ void __launch_bounds__(kWsSolve * 32, 1)
    rc_trsm_kernel(const double* __restrict__ A, int64_t lda, int64_t d, int n, const double* __restrict__ R0p,
                   const double* __restrict__ Wd, double* __restrict__ Q, int64_t ldq) {
    constexpr int NP = 8 * NB, LD = NP + 4;
    constexpr int P = 8;
    constexpr int SB = rc_blk_doubles(NB - 1);   // stage size (the largest block)
    extern __shared__ __align__(16) double qsm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    double* qw = qsm + (size_t)warp * 16 * LD;                 // this warp's 16 Q rows
    double* stg = qsm + (size_t)kWsSolve * 16 * LD;            // [2][SB] R0 block J | W_J, double-buffered
    // Block J's R0 fragments and diagonal inverse are read by all four warps: one cp.async copy per J
    // into a shared stage (prefetched one J ahead, one 4-warp barrier per J) instead of every warp
    // reading them from L2 (ncu r02 at n = 256, d = 2^22 chunk: 6.57 -> 4.53 ms, DMMA 30% -> 42%;
    // splitting the k loop into eight DMMA chains measured 4.86 ms: the unrolled code then misses in
    // the instruction cache more often)
    auto stage = [&](int J, int buf) {
        double* dst = stg + buf * SB;
        const double* src = R0p + rc_r0_off(J);
        const int nb = (64 * J + 96) / 2;   // 16-B chunks of the packed block
        for (int e = threadIdx.x; e < nb; e += kWsSolve * 32) rc_cp16(dst + 2 * e, src + 2 * e);
        if (threadIdx.x < 48) rc_cp16(dst + 64 * J + 96 + 2 * threadIdx.x, Wd + J * 96 + 2 * threadIdx.x);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int64_t ntiles = (d + kV3Rows - 1) / kV3Rows;
    const int64_t my = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    double pa0[P], pa1[P], pb0[P], pb1[P];
    auto load_step = [&](int64_t i, int J, double& a0, double& a1, double& b0, double& b1) {
        const int64_t r0 = (blockIdx.x + i * gridDim.x) * kV3Rows + 16 * warp + g;
        const int c0 = 8 * J + 2 * t;
        const bool ok = i < my;
        const bool va = ok && r0 < d, vb = ok && r0 + 8 < d;
        const double* p0 = A + (int64_t)min(c0, n - 1) * lda;
        const double* p1 = A + (int64_t)min(c0 + 1, n - 1) * lda;
        const int64_t ra = va ? r0 : 0, rb = vb ? r0 + 8 : 0;
        a0 = ldcs_pred_rc(p0 + ra, va && c0 < n);
        a1 = ldcs_pred_rc(p1 + ra, va && c0 + 1 < n);
        b0 = ldcs_pred_rc(p0 + rb, vb && c0 < n);
        b1 = ldcs_pred_rc(p1 + rb, vb && c0 + 1 < n);
    };
    if (my == 0) return;   // uniform per CTA: no barrier below is skipped by part of it
#pragma unroll
    for (int J = 0; J < P; ++J) load_step(0, J, pa0[J], pa1[J], pb0[J], pb1[J]);
    stage(0, 0);
    double* qrowA = qw + g * LD;
    double* qrowB = qrowA + 8 * LD;
    for (int64_t i = 0; i < my; ++i) {
        // fully unrolled (~140 KB of SASS at NB = 32); grouping J as (runtime jg) x (unrolled j < 8)
        // cut the code to 43 KB but measured slower (9.0 vs 6.6 ms per 2^20-row chunk at n = 256)
#pragma unroll
        for (int J = 0; J < NB; ++J) {
            // block J has landed in stage J & 1, and every warp is done with stage (J + 1) & 1 (block
            // J - 1): prefetch the next block (the next tile's block 0 after the last)
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            asm volatile("bar.sync 1, %0;" ::"n"(kWsSolve * 32) : "memory");
            stage(J + 1 < NB ? J + 1 : 0, (J + 1) & 1);
            const double* sj = stg + (J & 1) * SB;
            double tA0 = pa0[J % P], tA1 = pa1[J % P], tB0 = pb0[J % P], tB1 = pb1[J % P];
            if (J + P < NB)
                load_step(i, J + P, pa0[J % P], pa1[J % P], pb0[J % P], pb1[J % P]);
            else
                load_step(i + 1, J + P - NB, pa0[J % P], pa1[J % P], pb0[J % P], pb1[J % P]);
            double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0, b00 = 0.0, b01 = 0.0, b10 = 0.0, b11 = 0.0;
            const double* qa = qrowA + t;
            const double* qb = qrowB + t;
            const double* rb = sj + g * (8 * J + 12) + t;
#pragma unroll
            for (int k = 0; k < 8 * J; k += 8) {
                const double r0v = rb[k], r1v = rb[k + 4];
                dmma884(a00, a01, qa[k], r0v);
                dmma884(b00, b01, qb[k], r0v);
                dmma884(a10, a11, qa[k + 4], r1v);
                dmma884(b10, b11, qb[k + 4], r1v);
            }
            tA0 -= a00 + a10;
            tA1 -= a01 + a11;
            tB0 -= b00 + b10;
            tB1 -= b01 + b11;
            const int src0 = (lane & ~3) | (t >> 1), src1 = (lane & ~3) | (2 + (t >> 1));
            const double xa00 = __shfl_sync(0xffffffffu, tA0, src0), xa01 = __shfl_sync(0xffffffffu, tA1, src0);
            const double xa10 = __shfl_sync(0xffffffffu, tA0, src1), xa11 = __shfl_sync(0xffffffffu, tA1, src1);
            const double xb00 = __shfl_sync(0xffffffffu, tB0, src0), xb01 = __shfl_sync(0xffffffffu, tB1, src0);
            const double xb10 = __shfl_sync(0xffffffffu, tB0, src1), xb11 = __shfl_sync(0xffffffffu, tB1, src1);
            const double* wb = sj + 64 * J + 96 + g * 12 + t;
            const double w0 = wb[0], w1 = wb[4];
            double qa0 = 0.0, qa1 = 0.0, qb0 = 0.0, qb1 = 0.0;
            dmma884(qa0, qa1, (t & 1) ? xa01 : xa00, w0);
            dmma884(qb0, qb1, (t & 1) ? xb01 : xb00, w0);
            dmma884(qa0, qa1, (t & 1) ? xa11 : xa10, w1);
            dmma884(qb0, qb1, (t & 1) ? xb11 : xb10, w1);
            *reinterpret_cast<double2*>(qrowA + 8 * J + 2 * t) = make_double2(qa0, qa1);
            *reinterpret_cast<double2*>(qrowB + 8 * J + 2 * t) = make_double2(qb0, qb1);
            __syncwarp();
        }
        // the warp's 16 rows -> Q0 (column-major): lanes 0-15 column c, lanes 16-31 column c+1
        const int64_t rbase = (blockIdx.x + i * gridDim.x) * kV3Rows + 16 * warp;
        const int rr = lane & 15;
        for (int c = lane >> 4; c < n; c += 2)
            if (rbase + rr < d) Q[rbase + rr + (int64_t)c * ldq] = qw[rr * LD + c];
        __syncwarp();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// C[e] = sum_p part[p][e], fixed order (deterministic for a given grid)
__global__ void rc_reduce_kernel(const double* __restrict__ part, int parts, int64_t elems, double* __restrict__ C) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < elems; e += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int p = 0; p < parts; ++p) s += part[(size_t)p * elems + e];
        C[e] = s;
    }
}

// Alg 5 lines 3-4 over this block's rows: C (nc x nc, ld ldc) = [Q0^T Q0 (upper) | Q0^T b],
// Q0 = A R0^-1, R0 upper n x n (ld ldr0).  Row-partitioned callers sum the C's.
static csk_status rc_gram_impl(int64_t d, int64_t n, const double* A, int64_t lda, const double* b, const double* R0,
                               int64_t ldr0, double* C, int64_t ldc, cudaStream_t st) {
    CSK_REQUIRE(A != nullptr && b != nullptr && R0 != nullptr && C != nullptr, CSK_EINVAL, "NULL argument");
    CSK_REQUIRE(n >= 1 && n <= 1024 && d >= 1, CSK_EINVAL, "n=%lld must be in [1, 1024], d >= 1", (long long)n);
    CSK_REQUIRE(lda >= d && ldr0 >= n && ldc >= n + 1, CSK_ESHAPE, "bad leading dimension");
    CSK_REQUIRE(is_device_pointer(A) && is_device_pointer(b) && is_device_pointer(R0) && is_device_pointer(C),
                CSK_EINVAL, "rc_gram takes device pointers");
    const int nc = (int)n + 1;
    const char* pe = std::getenv("CSK_RC_PATH");
    const bool fused = n <= 128 && !(pe && std::atoi(pe) == 0);
    // the fused kernels and the reduction write an nc x nc C with ld nc; copy out when ldc differs
    double* Cw = C;
    if (ldc != nc) CSK_CUDA_TRY(csk_malloc_async(&Cw, (size_t)nc * nc * 8, st));
    CSK_CUDA_TRY(cudaMemsetAsync(Cw, 0, (size_t)nc * nc * 8, st));   // the lower part stays defined (0)
    csk_status s = CSK_OK;
    if (fused) {
        const int nb = n <= 16 ? 2 : n <= 32 ? 4 : n <= 64 ? 8 : 16;
        const int NP = 8 * nb, LD = NP + 4;
        const DeviceInfo& di = device_info();
        const int64_t tiles = ceil_div(d, kV3Rows);
        const int grid = (int)std::min<int64_t>(tiles, di.num_sms);
        double* part = nullptr;
        CSK_CUDA_TRY(csk_malloc_async(&part, (size_t)grid * nc * nc * 8, st));
        CSK_CUDA_TRY(cudaMemsetAsync(part, 0, (size_t)grid * nc * nc * 8, st));
        const size_t smem_v3 = ((size_t)rc_r0_off(nb) + 2 * (size_t)kV3Rows * LD + 2 * kV3Rows + NP +
                                (size_t)nb * 96) * 8;
        auto kern = nb == 2 ? rc_pass_v3_kernel<2> : nb == 4 ? rc_pass_v3_kernel<4>
                  : nb == 8 ? rc_pass_v3_kernel<8> : rc_pass_v3_kernel<16>;
        CSK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_v3));
        kern<<<grid, (kWsSolve + kWsGram) * 32, smem_v3, st>>>(A, lda, b, d, (int)n, R0, (int)ldr0, part, nc);
        CSK_LAUNCH_CHECK();
        rc_reduce_kernel<<<(unsigned)std::min<int64_t>(ceil_div((int64_t)nc * nc, 256), 1024), 256, 0, st>>>(
            part, grid, (int64_t)nc * nc, Cw);
        CSK_LAUNCH_CHECK();
        CSK_CUDA_TRY(cudaFreeAsync(part, st));
    } else if (n <= 256 && !(pe && std::atoi(pe) == 0)) {
        // 128 < n <= 256: DMMA TRSM kernel into a row-chunked Q0 workspace + cuBLAS Gram per chunk
        const int nb = 32, NP = 8 * nb, LD = NP + 4;
        int64_t mc = std::min<int64_t>(d, 1 << 20);
        cublasHandle_t h;
        s = blas_handle(st, &h);
        if (s != CSK_OK) {
            if (Cw != C) cudaFreeAsync(Cw, st);
            return s;
        }
        double* ws = nullptr;
        const size_t pk = (size_t)rc_r0_off(nb), wd = (size_t)nb * 96;
        CSK_CUDA_TRY(csk_malloc_async(&ws, (pk + wd + (size_t)mc * n) * 8, st));
        double* R0p = ws;
        double* Wd = ws + pk;
        double* Qw = Wd + wd;
        rc_pack_r0_kernel<<<nb, 256, 0, st>>>(R0, (int)ldr0, (int)n, nb, R0p, Wd);
        CSK_LAUNCH_CHECK();
        const size_t smem = ((size_t)kWsSolve * 16 * LD + 2 * (size_t)rc_blk_doubles(nb - 1)) * 8;
        CSK_CUDA_TRY(cudaFuncSetAttribute(rc_trsm_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const DeviceInfo& di = device_info();
        const double one = 1.0, zero = 0.0;
        cublasStatus_t bs = CUBLAS_STATUS_SUCCESS;
        for (int64_t r0 = 0; r0 < d && bs == CUBLAS_STATUS_SUCCESS; r0 += mc) {
            const int64_t m = std::min(mc, d - r0);
            const int grid = (int)std::min<int64_t>(ceil_div(m, kV3Rows), di.num_sms);
            rc_trsm_kernel<32><<<grid, kWsSolve * 32, smem, st>>>(A + r0, lda, m, (int)n, R0p, Wd, Qw, m);
            CSK_LAUNCH_CHECK();
            const double* beta = r0 == 0 ? &zero : &one;
            bs = cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)n, (int)n, (int)m, &one, Qw, (int)m, Qw, (int)m, beta, Cw,
                             nc);
            if (bs == CUBLAS_STATUS_SUCCESS)
                bs = cublasDgemv(h, CUBLAS_OP_T, (int)m, (int)n, &one, Qw, (int)m, b + r0, 1, beta,
                                 Cw + (size_t)n * nc, 1);
        }
        cudaFreeAsync(ws, st);
        if (bs != CUBLAS_STATUS_SUCCESS) {
            set_error("cuBLAS rand_cholQR Gram failed (%d)", (int)bs);
            s = CSK_ECUDA;
        }
        if (s == CSK_OK) CSK_CUDA_TRY(cudaMemsetAsync(Cw + (size_t)n * nc + n, 0, 8, st));
    } else {
        // row-chunked cuBLAS: chunk copy -> DTRSM in place -> DGEMM (Q0^T Q0) + DGEMV (Q0^T b); the chunk's Q0
        // (rows x n doubles) stays L2-resident between the calls
        int64_t mc = (int64_t)device_info().l2_bytes / 4 / (8 * n);
        if (const char* e = std::getenv("CSK_RC_CHUNK")) mc = std::max<int64_t>(256, std::atoll(e));
        mc = std::min(std::max<int64_t>(1024, mc & ~(int64_t)255), d);
        cublasHandle_t h;
        s = blas_handle(st, &h);
        double* Wk = nullptr;
        if (s == CSK_OK) CSK_CUDA_TRY(csk_malloc_async(&Wk, (size_t)mc * n * 8, st));
        const double one = 1.0, zero = 0.0;
        cublasStatus_t bs = CUBLAS_STATUS_SUCCESS;
        for (int64_t r0 = 0; s == CSK_OK && r0 < d && bs == CUBLAS_STATUS_SUCCESS; r0 += mc) {
            const int64_t m = std::min(mc, d - r0);
            const double* beta = r0 == 0 ? &zero : &one;
            CSK_CUDA_TRY(cudaMemcpy2DAsync(Wk, m * 8, A + r0, lda * 8, m * 8, n, cudaMemcpyDeviceToDevice, st));
            bs = cublasDtrsm(h, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, (int)m,
                             (int)n, &one, R0, (int)ldr0, Wk, (int)m);
            if (bs == CUBLAS_STATUS_SUCCESS)
                bs = cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)n, (int)n, (int)m, &one, Wk, (int)m, Wk, (int)m,
                                 beta, Cw, nc);
            if (bs == CUBLAS_STATUS_SUCCESS)
                bs = cublasDgemv(h, CUBLAS_OP_T, (int)m, (int)n, &one, Wk, (int)m, b + r0, 1, beta,
                                 Cw + (size_t)n * nc, 1);
        }
        if (Wk) cudaFreeAsync(Wk, st);
        if (s == CSK_OK && bs != CUBLAS_STATUS_SUCCESS) {
            set_error("cuBLAS rand_cholQR pass failed (%d)", (int)bs);
            s = CSK_ECUDA;
        }
        if (s == CSK_OK) CSK_CUDA_TRY(cudaMemsetAsync(Cw + (size_t)n * nc + n, 0, 8, st));
    }
    if (Cw != C) {
        if (s == CSK_OK)
            CSK_CUDA_TRY(cudaMemcpy2DAsync(C, ldc * 8, Cw, nc * 8, nc * 8, nc, cudaMemcpyDeviceToDevice, st));
        cudaFreeAsync(Cw, st);
    }
    return s;
}

// Alg 5 lines 5-8 from the (all-reduced) C: R1 = chol(C11), u = R1^-1 R1^-T z, x = R0^-1 u, R = R1 R0
static csk_status rc_finish_impl(int64_t n, const double* C, int64_t ldc, const double* R0, int64_t ldr0, double* x,
                                 double* R, int64_t ldr, cudaStream_t st) {
    CSK_REQUIRE(C != nullptr && R0 != nullptr && x != nullptr, CSK_EINVAL, "NULL argument");
    CSK_REQUIRE(n >= 1 && n <= 1024, CSK_EINVAL, "n out of range");
    CSK_REQUIRE(ldc >= n + 1 && ldr0 >= n && (R == nullptr || ldr >= n), CSK_ESHAPE, "bad leading dimension");
    CSK_REQUIRE(is_device_pointer(C) && is_device_pointer(R0) && is_device_pointer(x) &&
                    (R == nullptr || is_device_pointer(R)),
                CSK_EINVAL, "rc_finish takes device pointers");
    const int nc = (int)n + 1;
    auto pad = [](size_t cnt) { return (cnt + 31) & ~(size_t)31; };
    double* ws = nullptr;
    CSK_CUDA_TRY(csk_malloc_async(&ws, (2 * pad((size_t)nc * nc) + pad(nc) + 32) * 8, st));
    double* Cc = ws;
    double* S = Cc + pad((size_t)nc * nc);
    double* u = S + pad((size_t)nc * nc);
    int* sd = reinterpret_cast<int*>(u + pad(nc));
    CSK_CUDA_TRY(cudaMemcpy2DAsync(Cc, nc * 8, C, ldc * 8, nc * 8, nc, cudaMemcpyDeviceToDevice, st));
    CSK_CUDA_TRY(cudaMemsetAsync(Cc + (size_t)n * nc + n, 0, 8, st));   // b^T b is not needed for x
    CSK_CUDA_TRY(cudaFuncSetAttribute(chol_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 0));
    chol_solve_kernel<<<1, 1024, 0, st>>>(Cc, nc, 0, S, u, sd);
    CSK_LAUNCH_CHECK();
    rc_finish_kernel<<<1, 1024, (size_t)n * 8, st>>>(R0, (int)ldr0, S, nc, (int)n, u, x, R, (int)ldr, sd);
    CSK_LAUNCH_CHECK();
    int hs = 0;
    CSK_CUDA_TRY(cudaMemcpyAsync(&hs, sd, sizeof(int), cudaMemcpyDeviceToHost, st));
    CSK_CUDA_TRY(cudaFreeAsync(ws, st));
    CSK_CUDA_TRY(cudaStreamSynchronize(st));
    if (hs != 0) {
        set_error("rand_cholQR: Cholesky of Q0^T Q0 failed (pivot <= 0)");
        return (csk_status)hs;
    }
    return CSK_OK;
}

// Alg 5 line 2 from the (all-reduced) sketch Z = [G S A | G S b]: R0 = R[:n, :n] of qr(Z) (ld ldr0).
static csk_status rc_r0_impl(int64_t k2, int64_t n, const double* Z, int64_t ldz, double* R0, int64_t ldr0,
                             cudaStream_t st) {
    CSK_REQUIRE(R0 != nullptr && is_device_pointer(R0), CSK_EINVAL, "R0 must be a device pointer");
    CSK_REQUIRE(ldr0 >= n, CSK_ESHAPE, "ldr0 < n");
    const int nc = (int)n + 1;
    double* ws = nullptr;
    CSK_CUDA_TRY(csk_malloc_async(&ws, ((size_t)nc * nc + nc) * 8, st));
    csk_status s = solve_impl(k2, n, Z, ldz, ws + (size_t)nc * nc, nullptr, st, false, ws);
    if (s == CSK_OK)
        CSK_CUDA_TRY(cudaMemcpy2DAsync(R0, ldr0 * 8, ws, nc * 8, n * 8, n, cudaMemcpyDeviceToDevice, st));
    cudaFreeAsync(ws, st);
    return s;
}

static csk_status rc_impl(csk_plan_t plan, int64_t k2, int64_t n, const double* A, int64_t lda, const double* b,
                          double* x, double* R, int64_t ldr, cudaStream_t st) {
    CSK_REQUIRE(plan != nullptr, CSK_EINVAL, "plan is NULL");
    CSK_REQUIRE(A != nullptr && b != nullptr && x != nullptr, CSK_EINVAL, "A, b, x must be non-NULL");
    CSK_REQUIRE(n >= 1 && n <= 1024, CSK_EINVAL, "n=%lld must be in [1, 1024]", (long long)n);
    CSK_REQUIRE(k2 >= n + 1, CSK_ESHAPE, "k2=%lld must be >= n+1=%lld", (long long)k2, (long long)(n + 1));
    const int64_t d = plan->d;
    CSK_REQUIRE(d >= n, CSK_ESHAPE, "d=%lld < n=%lld", (long long)d, (long long)n);
    CSK_REQUIRE(lda >= d, CSK_ESHAPE, "lda=%lld < d=%lld", (long long)lda, (long long)d);
    CSK_REQUIRE(R == nullptr || ldr >= n, CSK_ESHAPE, "ldr=%lld < n", (long long)ldr);
    CSK_REQUIRE(is_device_pointer(A) && is_device_pointer(b) && is_device_pointer(x) &&
                    (R == nullptr || is_device_pointer(R)),
                CSK_EINVAL, "rc_lstsq takes device pointers");
    const int nc = (int)n + 1;
    auto pad = [](size_t cnt) { return (cnt + 31) & ~(size_t)31; };
    double* ws = nullptr;
    CSK_CUDA_TRY(csk_malloc_async(&ws, (pad((size_t)k2 * nc) + 2 * pad((size_t)nc * nc)) * 8, st));
    double* Z = ws;
    double* R0 = Z + pad((size_t)k2 * nc);      // n x n, ld nc
    double* C = R0 + pad((size_t)nc * nc);      // nc x nc
    csk_status s = ms_apply_impl(plan, k2, CSK_F64, n, A, lda, b, Z, k2, st);   // line 1
    if (s == CSK_OK) s = rc_r0_impl(k2, n, Z, k2, R0, nc, st);                   // line 2
    if (s == CSK_OK) s = rc_gram_impl(d, n, A, lda, b, R0, nc, C, nc, st);       // lines 3-4
    if (s == CSK_OK) s = rc_finish_impl(n, C, nc, R0, nc, x, R, ldr, st);        // lines 5-8
    cudaFreeAsync(ws, st);
    return s;
}

}  // namespace csk

extern "C" {

csk_status rc_lstsq(csk_plan_t plan, int64_t k2, int64_t n, const double* A, int64_t lda, const double* b, double* x,
                    double* R, int64_t ldr, void* stream) {
    return csk::rc_impl(plan, k2, n, A, lda, b, x, R, ldr, (cudaStream_t)stream);
}

csk_status rc_r0(int64_t k2, int64_t n, const double* Z, int64_t ldz, double* R0, int64_t ldr0, void* stream) {
    return csk::rc_r0_impl(k2, n, Z, ldz, R0, ldr0, (cudaStream_t)stream);
}

csk_status rc_gram(int64_t d, int64_t n, const double* A, int64_t lda, const double* b, const double* R0, int64_t ldr0,
                   double* C, int64_t ldc, void* stream) {
    return csk::rc_gram_impl(d, n, A, lda, b, R0, ldr0, C, ldc, (cudaStream_t)stream);
}

csk_status rc_finish(int64_t n, const double* C, int64_t ldc, const double* R0, int64_t ldr0, double* x, double* R,
                     int64_t ldr, void* stream) {
    return csk::rc_finish_impl(n, C, ldc, R0, ldr0, x, R, ldr, (cudaStream_t)stream);
}

}  // extern "C"
