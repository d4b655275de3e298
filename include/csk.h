/*
 * csk.h -- C-ABI of the B200 (sm_100a) CountSketch / multisketch / sketch-and-solve
 * library (libcsk.so), the hot path of arXiv 2508.14209.
 *
 * Citations: P:Lx = PAPER.md line x (section / equation / algorithm).
 *
 * Conventions for every entry point
 *  - Plain C linkage, no C++ exception ever crosses this boundary.
 *  - Matrices are COLUMN-MAJOR with an explicit leading dimension (elements).
 *  - "stream" is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Device-side arguments are device pointers (or host pointers where stated);
 *    the CALLER owns every buffer it passes.  A plan owns its codes, sort and
 *    cached Gaussian matrices until cs_plan_destroy.
 *  - Arguments are validated before any launch.  Errors are returned as a
 *    csk_status; csk_last_error() gives a thread-local detail string.
 *      null pointer / non-positive size .................. CSK_EINVAL
 *      bad leading dimension or incompatible shapes ...... CSK_ESHAPE
 *      unsupported dtype for the call .................... CSK_EDTYPE
 *      allocation failure ................................ CSK_ENOMEM
 *      CUDA / cuBLAS failure ............................. CSK_ECUDA
 *      Cholesky pivot <= 0 (normal equations) ............ CSK_ENOTPD
 *      |R_ii| <= 1e-14 max|R_jj| (sketched QR) ............ CSK_ESINGULAR
 *      variant not applicable to this plan/shape ......... CSK_EUNSUPPORTED
 *  - cs_plan*, cs_apply and ms_apply are asynchronous on the stream.
 *    ms_solve, ms_lstsq and ne_lstsq synchronise the stream before returning
 *    (they report a numerical status); ms_solve_async leaves it on the device.
 */
#ifndef CSK_H
#define CSK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CSK_OK = 0,
    CSK_EINVAL = 1,
    CSK_ESHAPE = 2,
    CSK_EDTYPE = 3,
    CSK_ENOMEM = 4,
    CSK_ECUDA = 5,
    CSK_ENOTPD = 6,
    CSK_ESINGULAR = 7,
    CSK_EUNSUPPORTED = 8
} csk_status;

typedef enum { CSK_F64 = 0, CSK_F32 = 1 } csk_dtype;

/* cs_apply kernel variants.  CSK_VAR_AUTO picks from the table
 * measured on B200 over d = 2^20 and 2^23, n = 8..256, fp64 and fp32
 * (profiles/r02_variant_table.json): B won every row at round-2 close
 * (its narrow-row instantiations run 2-3 CTAs per SM), so AUTO = B; the other variants
 * stay selectable (G is the bitwise-reproducible one). */
typedef enum {
    CSK_VAR_AUTO = -1,
    CSK_VAR_ATOMIC_COL = 0,   /* L: one L2 reduction (REDG) per element, column-major target  */
    CSK_VAR_ATOMIC_ROW = 1,   /* T: row tiles transposed in smem, coalesced REDG into SA^T    */
    CSK_VAR_SMEM = 2,         /* S: per-CTA shared-memory privatised buckets, one flush/CTA   */
    CSK_VAR_SORTED = 3,       /* G: deterministic signed segmented gather over the plan sort   */
    CSK_VAR_BULK_ROW = 4,     /* B: row tiles in smem, TMA bulk reduce-add (cp.reduce.async.bulk) */
    CSK_VAR_TMA_ROW = 5       /* X: TMA tensor loads of 2-D [A b] tiles + coalesced REDG per row;
                                 needs a uniform column stride (b == NULL or b == A + n*lda) with
                                 16-B aligned columns, else it falls back to T */
} csk_variant;

/* cs_plan flags */
#define CSK_PLAN_SORT 0x2u    /* also build the stable counting sort (needed by CSK_VAR_SORTED) */
#define CSK_PLAN_HASH 0x4u    /* store no codes: the fp64 row-tile CountSketch recomputes h(i), s(i)
                                 from (seed, global row) on the fly -- the hash-based generation of
                                 P:L389 -- and every other consumer materialises the codes on first
                                 use (ignored together with CSK_PLAN_SORT, which needs them) */

typedef struct csk_plan_s* csk_plan_t;

/* ---------------------------------------------------------------- plans --
 * cs_plan: the CountSketch S (k1 x d) of Def 3, drawn from a
 * counter-based hash of (seed, GLOBAL row) -- the hash-based generation the
 * paper lists as future work.  Local row i of this plan is global row
 * row0 + i, so the plans of a row-partitioned A are slices of one sketch
 * (block-row distribution).  Device memory: 4*d bytes of codes
 * (bucket | sign<<31); with CSK_PLAN_SORT also offsets (8*(k1+1)) and perm (4*d).
 *   d      rows of the (local) block, 1 <= d <= 2^31 - 1
 *   k1     embedding dimension, 1 <= k1 <= 2^31 - 1
 *   seed   sketch seed (Philox key);  row0 >= 0 global index of local row 0
 *   flags  0, CSK_PLAN_SORT and/or CSK_PLAN_HASH
 *   out    receives the plan handle (NULL on failure) */
csk_status cs_plan(int64_t d, int64_t k1, uint64_t seed, int64_t row0, uint32_t flags,
                   void* stream, csk_plan_t* out);

/* cs_plan_from_arrays: a plan with caller-chosen buckets h[i] in [0,k1) and
 * signs s[i] in {-1,+1} (HOST arrays of length d, copied).  Used to force a
 * sketch (identity, permutation, the worked example of S:L231). */
csk_status cs_plan_from_arrays(int64_t d, int64_t k1, const int32_t* h, const int8_t* s,
                               uint32_t flags, void* stream, csk_plan_t* out);

/* cs_plan_export: copy the plan's codes (int32[d], bucket | sign<<31), and if the
 * plan was built with CSK_PLAN_SORT the sort (offsets int64[k1+1], perm int32[d]).
 * Pointers may be host or device (UVA copy); any may be NULL to skip.
 * Synchronises the stream. */
csk_status cs_plan_export(csk_plan_t plan, int32_t* code, int64_t* offsets, int32_t* perm,
                          void* stream);

/* cs_plan_info: d, k1, row0 of a plan (any output may be NULL). */
csk_status cs_plan_info(csk_plan_t plan, int64_t* d, int64_t* k1, int64_t* row0);

void cs_plan_destroy(csk_plan_t plan);

/* ------------------------------------------------------------- sketches --
 * cs_apply: SA = S [A b], Eq 2, Alg 2:
 *   SA[m, c] = sum_{i : h(i) = m} s(i) A[i, c]   (c < n),   SA[m, n] = S b (if b).
 *   dtype   CSK_F64 (A, b, SA double) or CSK_F32 (float)
 *   n       columns of A (n >= 0; n + (b != NULL) >= 1)
 *   A       d x n column-major, lda >= d (device pointer; may be NULL if n == 0)
 *   b       optional extra column of length d (device pointer or NULL)
 *   SA      k1 x (n + (b != NULL)) column-major, ldsa >= k1 (device pointer);
 *           fully overwritten (empty buckets become exactly 0)
 *   variant csk_variant; CSK_VAR_SORTED needs a plan built with CSK_PLAN_SORT
 * Floating-point order is unspecified except for CSK_VAR_SORTED, which is
 * bitwise deterministic; integer-valued inputs give exact sums in every variant. */
csk_status cs_apply(csk_plan_t plan, csk_dtype dtype, int64_t n, const void* A, int64_t lda,
                    const void* b, void* SA, int64_t ldsa, int variant, void* stream);

/* ms_apply: the multisketch ("Count-Gauss"; Table 1)
 *   Z = G S [A b],  G k2 x k1 with G_ij ~ N(0, 1/k2), drawn from Philox
 *   stream 1 of the plan's seed (cached in the plan per k2, R4).
 *   Z       k2 x (n + (b != NULL)) column-major, ldz >= k2 (device pointer).
 *   A, b    device pointers, or HOST pointers (then streamed through the GPU in
 *           row chunks, copies overlapped with the sketch -- P:L375 linearity).
 *   Workspace for SA (k1 x ncols) comes from the stream-ordered allocator.
 *   The G-stage is a hand-written fp64 DMMA kernel on the CountSketch's row-major
 *   SA^T (Z^T = Y^T G^T, no transpose); fp32 input is sketched in fp32
 *   bounded-depth copies combined in fp64 (R12) and Z is fp32.
 * For a row-partitioned A every rank calls ms_apply on its block
 * with its row0-plan and the same seed, and the caller sums the Z's (NCCL
 * all-reduce) before ms_solve. */
csk_status ms_apply(csk_plan_t plan, int64_t k2, csk_dtype dtype, int64_t n, const void* A,
                    int64_t lda, const void* b, void* Z, int64_t ldz, void* stream);

/* ms_solve: the solve phase of sketch-and-solve (Alg 1 lines 2-3)
 * on the augmented sketch Z = [G S A | G S b] (k2 x (n+1), fp64, device,
 * not modified): R = qr(Z) by Householder, x = R[:n,:n]^-1 R[:n,n] (= R^-1 Q^T z).
 *   x         device pointer, n doubles
 *   sk_resid  HOST pointer or NULL: |R[n,n]| = ||G S (b - A x)||_2
 * Requires k2 >= n + 1.  Returns CSK_ESINGULAR if some |R_ii| <= 1e-14 max|R_jj|.
 * Synchronises the stream. */
csk_status ms_solve(int64_t k2, int64_t n, const double* Z, int64_t ldz, double* x,
                    double* sk_resid, void* stream);

/* ms_solve_async: ms_solve without the host synchronisation, for pipelined
 * callers (one solve per batch, status checked later).  Same arithmetic and
 * launches as ms_solve.
 *   x         device pointer, n doubles
 *   sk_resid  DEVICE pointer or NULL: receives |R[n,n]|
 *   status    DEVICE pointer to one int32: receives CSK_OK or CSK_ESINGULAR
 *             (the numerical status ms_solve would return), stream-ordered
 * Returns CSK_OK once the work is enqueued (argument and launch errors are
 * returned immediately); asynchronous on the stream. */
csk_status ms_solve_async(int64_t k2, int64_t n, const double* Z, int64_t ldz, double* x,
                          double* sk_resid, int32_t* status, void* stream);

/* ms_lstsq: multisketched sketch-and-solve least squares min ||G S (A x - b)||
 * (Alg 1 with S := G S1; "multisketch" bars of Fig 5):
 * ms_apply(plan, k2, A, b) followed by ms_solve.  fp64.
 *   A d x n (lda >= d), b length d: device or HOST pointers (host inputs are
 *   streamed, see ms_apply); x: n doubles, device or HOST pointer;
 *   sk_resid: HOST pointer or NULL.  Synchronises the stream. */
csk_status ms_lstsq(csk_plan_t plan, int64_t k2, int64_t n, const double* A, int64_t lda,
                    const double* b, double* x, double* sk_resid, void* stream);

/* ne_lstsq: the normal-equations baseline: C = [A b]^T [A b] with
 * cuBLAS (DGEMM A^T A + DGEMV A^T b + DDOT b^T b, the fastest form measured on
 * B200, R15), Cholesky
 * of C[:n,:n] = R^T R, y = R^-T C[:n,n], x = R^-1 y.
 *   A d x n (lda >= d), b length d, x n doubles: device pointers.
 * Returns CSK_ENOTPD if a Cholesky pivot is <= 0 (the breakdown of Fig 8,
 * P:L369).  Synchronises the stream. */
csk_status ne_lstsq(int64_t d, int64_t n, const double* A, int64_t lda, const double* b,
                    double* x, void* stream);

/* rc_lstsq: rand_cholQR least squares, Alg 5 (Alg 4): the TRUE
 * least-squares solution min ||A x - b|| (no sketch distortion), stable for kappa(A) < u^-1
 * (P:L314-318).  Y = G S [A b] (ms_apply with this plan and k2), R0 = qr(Y)[:n,:n],
 * Q0 = A R0^-1 by a row-chunked triangular solve, G = Q0^T Q0 and z = Q0^T b in the same pass,
 * R1 = chol(G), x = R^-1 R1^-T z with R = R1 R0 (R23-R24).
 *   A d x n (lda >= d), b length d, x n doubles: DEVICE pointers (d = the plan's d)
 *   R  nullable DEVICE pointer: n x n column-major (ldr >= n) receives R = R1 R0, the R factor
 *      of A (A = Q R with Q = A R^-1 orthonormal)
 * Requires k2 >= n + 1 and k2 <= 512 (the cluster QR of ms_solve); n <= 1024.
 * Returns CSK_ESINGULAR if the sketched R0 is numerically singular, CSK_ENOTPD if the Cholesky
 * of Q0^T Q0 breaks down.  Workspace: k2*(n+1) + 3(n+1)^2 + (L2/4 bytes) doubles, stream-ordered.
 * Synchronises the stream. */
csk_status rc_lstsq(csk_plan_t plan, int64_t k2, int64_t n, const double* A, int64_t lda, const double* b,
                    double* x, double* R, int64_t ldr, void* stream);

/* The phases of rc_lstsq, for a row-partitioned A: every rank calls ms_apply on
 * its block (sum the Z's: all-reduce 1), rc_r0 on the summed Z, rc_gram on its block (sum the
 * C's: all-reduce 2), then rc_finish.  rc_lstsq == these four calls on one GPU.
 * rc_r0:     R0 = R[:n,:n] of the Householder QR of Z = [G S A | G S b] (k2 x (n+1), ldz);
 *            R0 n x n upper, ld ldr0 >= n.  k2 <= 512.  ESINGULAR as ms_solve.  Synchronises.
 * rc_gram:   C = [Q0^T Q0 | Q0^T b] over this block's d rows, Q0 = A R0^-1 (R24) computed tile by
 *            tile and never stored; C (n+1) x (n+1), ld ldc >= n+1: the upper triangle of
 *            C[:n,:n] and column n are written (C[n,n] = 0, the rest unspecified).  Asynchronous.
 * rc_finish: R1 = chol(C[:n,:n]) (ENOTPD on breakdown), x = R0^-1 R1^-1 R1^-T C[:n,n];
 *            R (nullable) = R1 R0, n x n, ld ldr.  Synchronises.
 * All pointers are DEVICE pointers. */
csk_status rc_r0(int64_t k2, int64_t n, const double* Z, int64_t ldz, double* R0, int64_t ldr0, void* stream);
csk_status rc_gram(int64_t d, int64_t n, const double* A, int64_t lda, const double* b, const double* R0, int64_t ldr0,
                   double* C, int64_t ldc, void* stream);
csk_status rc_finish(int64_t n, const double* C, int64_t ldc, const double* R0, int64_t ldr0, double* x, double* R,
                     int64_t ldr, void* stream);

/* srht_apply: the SRHT S = k^-1/2 P H_d D (Def) applied to
 * [A b]:  Y[j, c] = k^-1/2 (H_d D [A b][:, c])[p_j],  fp64.
 *   D_ii = +-1 and the k sampled rows p_j (i.i.d. uniform, with replacement) come from Philox
 *   streams 6 and 7 of seed over GLOBAL rows (R20-R21); H_d is the Sylvester
 *   Hadamard matrix, H[p, i] = (-1)^popcount(p & i) (Alg 3 computes it; R22).
 *   dglob  global row count, a power of two, <= 2^32
 *   d, row0  this block's rows [row0, row0 + d) of the global matrix: a row-partitioned A sums
 *          the Y of its blocks (linearity).  For dglob >= 4096, row0 and d must be
 *          multiples of 4096; for dglob < 4096 the block is the whole matrix.
 *   A      d x n column-major (lda >= d), b optional extra column, Y k x (n + (b != NULL))
 *          column-major (ldy >= k): DEVICE pointers; Y is overwritten.  k <= 1024.
 * Asynchronous on the stream.  Workspace: d/8 + 4k bytes, stream-ordered. */
csk_status srht_apply(int64_t d, int64_t dglob, int64_t row0, int64_t k, uint64_t seed, int64_t n,
                      const double* A, int64_t lda, const double* b, double* Y, int64_t ldy, void* stream);

/* ------------------------------------------- other sketch-and-solve operators (Fig 5)
 * gs_apply: Gaussian sketch Z = G[:, row0 .. row0+d) [A b], G k x dglob with G_ij ~ N(0, 1/k)
 *    from Philox stream 1 of seed, element e = r + (global row) * k (R4's
 *   generator over a k x d matrix).  The k x d matrix is never stored: each row chunk's slice
 *   is generated and multiplied in (DGEMM) while L2-resident.  k even.  A (lda >= d), b
 *   (nullable), Z k x (n + (b != NULL)) (ldz >= k): DEVICE pointers.  Asynchronous. */
csk_status gs_apply(int64_t d, int64_t row0, int64_t k, uint64_t seed, int64_t n, const double* A, int64_t lda,
                    const double* b, double* Z, int64_t ldz, void* stream);
/* gs_lstsq: Gaussian sketch-and-solve (Alg 1 with S = G, k = 2n in the paper): gs_apply on
 *   [A b] followed by the ms_solve Householder solve.  x: device or host; sk_resid: host or
 *   NULL.  Requires n + 1 <= k <= 512.  Synchronises the stream. */
csk_status gs_lstsq(int64_t d, int64_t k, uint64_t seed, int64_t n, const double* A, int64_t lda, const double* b,
                    double* x, double* sk_resid, void* stream);
/* cs_lstsq: CountSketch-only sketch-and-solve (Alg 1 with S = S1, k1 = 2n^2): QR of the
 *   k1 x (n+1) sketch [S1 A | S1 b] by cuSOLVER GEQRF (the paper's GeQRF, whose cost
 *   dominates this variant), x = R11^-1 r12 on the GPU, sk_resid = |R_nn|.
 *   A, b, x: DEVICE pointers; sk_resid host or NULL.  ESINGULAR as for ms_solve.  Synchronises. */
csk_status cs_lstsq(csk_plan_t plan, int64_t n, const double* A, int64_t lda, const double* b, double* x,
                    double* sk_resid, void* stream);
/* msh_apply / msh_lstsq: the Count+SRHT multisketch the paper lists as future work:
 *   Z = SRHT_k2(S1 [A b]) with the SRHT of srht_apply over the k1 rows of the CountSketch
 *   output (k1 must be a power of two, seed = the plan's).  msh_lstsq adds the ms_solve solve
 *   (k2 >= n + 1).  DEVICE A, b, Z; x device or host.  msh_apply is asynchronous, msh_lstsq
 *   synchronises. */
csk_status msh_apply(csk_plan_t plan, int64_t k2, int64_t n, const double* A, int64_t lda, const double* b, double* Z,
                     int64_t ldz, void* stream);
csk_status msh_lstsq(csk_plan_t plan, int64_t k2, int64_t n, const double* A, int64_t lda, const double* b, double* x,
                     double* sk_resid, void* stream);

/* ------------------------------------------------------------- utilities */
const char* csk_status_str(csk_status st);
const char* csk_last_error(void);      /* thread-local detail of the last failure */
/* Number of device kernels this library launched on this host thread since
 * the last reset (bench.py counts gpu_launches with it). */
uint64_t csk_launch_count(int reset);
/* Library version string. */
const char* csk_version(void);

/* Kernel timing for the roofline (bench.py): while enabled on this host thread,
 * every launch of the dominant cs_apply kernel is bracketed by CUDA events on
 * its launching stream.  csk_profile_read synchronises those events and returns
 * the summed kernel time (ms) and the number of bracketed launches since the
 * last enable, then clears them.  Off by default (no events recorded). */
void csk_profile_enable(int on);
csk_status csk_profile_read(double* total_ms, uint64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* CSK_H */
