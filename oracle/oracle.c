/*
 * oracle/oracle.c -- CPU ORACLE for the hot path of arXiv 2508.14209
 * ("A High Performance GPU CountSketch Implementation and Its Application to
 * Multisketching and Least Squares Problems", Higgins, Boman, Yamazaki).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2508_14209_b200/, include/csk.h) never links,
 * imports or calls it, and this file shares no code, header, table or
 * constant generator with paper_2508_14209_b200/csrc/.
 *
 * Plain, slow, obviously-correct loops in fp64, written from the paper:
 *   P:Lx  = /root/reference/PAPER.md line x (section / equation / algorithm).
 *   S:Lx  = /root/reference/SPEC.md line x.
 *   DESIGN.md "Readings" R1..R12 = where the paper is silent or garbled.
 * Compile: gcc -O2 -fno-fast-math -ffp-contract=off -fPIC -shared (no OpenMP;
 * the oracle is single-threaded by design, so bench.py reports cores=1).
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"):
 *   or_philox4x32_10  Random123 known-answer vectors (tests/golden/philox4x32_10_kat.txt)
 *   or_codes          chi-square uniformity, sign balance, k1=2^b prefix invariance
 *   or_count_sort     numpy.argsort(kind="stable") + bincount (library)
 *   or_cs_apply       dense densify(S)@A brute force; SPEC worked example;
 *                     k1=1 closed form (column sums / s^T A); integer exactness;
 *                     identity plan; E||Sx||^2 = ||x||^2 with closed-form variance
 *   or_gauss          moments, Kolmogorov-Smirnov vs scipy.stats.norm, E||Gy||^2
 *   or_gemm_comp      numpy matmul (library)
 *   or_householder_qr numpy.linalg.qr (library, |R| agreement), Q^TQ=I, QR=A
 *   or_sketch_solve   numpy.linalg.lstsq on the oracle's Z (library);
 *                     identity sketch == QR least squares
 *   or_normal_eq      scipy.linalg.cho_solve (library); NOT_PD past kappa~1e8
 *   or_rand_cholqr_lstsq  numpy.linalg.lstsq on A itself (library: rand_cholQR has no
 *                     distortion); R^T R = A^T A and |R| = |qr(A).R|; identity sketch;
 *                     stability at kappa = 1e10 where the normal equations fail
 *   or_srht_draws     sign balance, uniform samples (chi-square)
 *   or_fwht_rad4      scipy.linalg.hadamard (Sylvester) brute force; H H = d I; Parseval
 *   or_srht_apply     dense (1/sqrt k) P H D A brute force; E||Sx||^2 = ||x||^2
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* status codes: same numeric meaning as the C-ABI (include/csk.h) but
 * declared independently here -- the oracle includes no product header. */
enum { OR_OK = 0, OR_EINVAL = 1, OR_ENOTPD = 6, OR_ESINGULAR = 7 };

/* ------------------------------------------------------------------------
 * c1. Counter-based hash: Philox4x32-10 (Salmon et al., SC'11; the generator
 * family cuRAND exposes, "The cuRAND library was used").  The paper
 * never names its generator (Reading R1), so we fix Philox4x32-10.
 * One round:  (hi0,lo0) = mulhilo(0xD2511F53, c0); (hi1,lo1) = mulhilo(0xCD9E8D57, c2)
 *             c <- (hi1^c1^k0, lo1, hi0^c3^k1, lo0)
 * Key bump between rounds: k0 += 0x9E3779B9, k1 += 0xBB67AE85.
 * ---------------------------------------------------------------------- */
void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* CountSketch bucket and sign of GLOBAL row i (Def 3):
 * r_i uniform on {0..k1-1} (0-based, Reading R2), sigma_i Rademacher.
 * x = Philox(ctr = (lo32(i>>2), hi32(i>>2), 0, 0), key = (lo32 seed, hi32 seed));
 * w = x[i & 3]; h = floor(w * k1 / 2^32); s = (w & 1) ? -1 : +1   (Reading R3). */
static void code_of_row(uint64_t seed, uint64_t i, uint32_t k1, int32_t* h, int8_t* s) {
    uint64_t q = i >> 2;
    uint32_t ctr[4] = {(uint32_t)q, (uint32_t)(q >> 32), 0u, 0u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t x[4];
    or_philox4x32_10(ctr, key, x);
    uint32_t w = x[i & 3u];
    *h = (int32_t)(((uint64_t)w * (uint64_t)k1) >> 32);
    *s = (w & 1u) ? (int8_t)-1 : (int8_t)1;
}

/* Codes for local rows 0..d-1 whose global index is row0 + local (P:L375:
 * C = [C^(1) ... C^(p)], each block a slice of the one global sketch). */
int or_codes(int64_t d, int64_t k1, uint64_t seed, int64_t row0, int32_t* h, int8_t* s) {
    if (d < 0 || k1 < 1 || k1 > 2147483647LL || row0 < 0 || (d > 0 && (!h || !s))) return OR_EINVAL;
    for (int64_t i = 0; i < d; ++i)
        code_of_row(seed, (uint64_t)(row0 + i), (uint32_t)k1, &h[i], &s[i]);
    return OR_OK;
}

/* ------------------------------------------------------------------------
 * c2. Stable counting sort of rows by bucket (a plan-time step; P:L144 uses
 * atomics instead, BASELINE.json north_star names this deterministic form).
 * offsets[m] = #{i : h(i) < m}, offsets[k1] = d;
 * perm[offsets[h(i)] + #{i' < i : h(i') = h(i)}] = i.
 * ---------------------------------------------------------------------- */
int or_count_sort(int64_t d, int64_t k1, const int32_t* h, int64_t* offsets, int32_t* perm) {
    if (d < 0 || k1 < 1 || !offsets || (d > 0 && (!h || !perm))) return OR_EINVAL;
    for (int64_t m = 0; m <= k1; ++m) offsets[m] = 0;
    for (int64_t i = 0; i < d; ++i) {
        if (h[i] < 0 || h[i] >= k1) return OR_EINVAL;
        offsets[h[i] + 1] += 1;                      /* histogram */
    }
    for (int64_t m = 0; m < k1; ++m) offsets[m + 1] += offsets[m];   /* exclusive scan */
    int64_t* fill = (int64_t*)malloc((size_t)k1 * sizeof(int64_t));
    if (!fill) return OR_EINVAL;
    for (int64_t m = 0; m < k1; ++m) fill[m] = offsets[m];
    for (int64_t i = 0; i < d; ++i) perm[fill[h[i]]++] = (int32_t)i;  /* stable scatter */
    free(fill);
    return OR_OK;
}

/* ------------------------------------------------------------------------
 * c3. CountSketch apply, Eq 2:  Y_{m,:} = sum_{j: r_j = m} sigma_j A_{j,:}
 * written as the plain loop over rows of Alg 2, one column at a
 * time.  Column c < n is A[:, c] (column-major, leading dimension lda); column
 * c == n is the optional right-hand side b, sketched by the same S (Alg 1
 * line 1: "Y = SA, z = Sb").  Accumulation is Neumaier-compensated in
 * fp64 so the oracle's own error (~2u * sum|terms|) is far below the GPU
 * tolerance.  Tabs (nullable) receives T = |S| |A|, the sum of |terms| per
 * output, which every GPU tolerance is scaled by.
 * fp32 input (is_f32) is widened exactly to fp64 and accumulated in fp64.
 * ---------------------------------------------------------------------- */
static void neumaier_add(double* sum, double* comp, double v) {
    double t = *sum + v;
    if (fabs(*sum) >= fabs(v)) *comp += (*sum - t) + v;
    else                       *comp += (v - t) + *sum;
    *sum = t;
}

static double load_elem(const void* base, int is_f32, int64_t idx) {
    return is_f32 ? (double)((const float*)base)[idx] : ((const double*)base)[idx];
}

int or_cs_apply(int64_t d, int64_t n, int64_t k1, const int32_t* h, const int8_t* s,
                const void* A, int64_t lda, const void* b, int is_f32,
                double* SA, int64_t ldsa, double* Tabs) {
    int64_t ncols = n + (b ? 1 : 0);
    if (d < 0 || n < 0 || k1 < 1 || ldsa < k1 || (n > 0 && lda < d) || !SA) return OR_EINVAL;
    if (d > 0 && (!h || !s || (n > 0 && !A))) return OR_EINVAL;
    double* sum = (double*)calloc((size_t)k1, sizeof(double));
    double* comp = (double*)calloc((size_t)k1, sizeof(double));
    double* asum = (double*)calloc((size_t)k1, sizeof(double));
    double* acomp = (double*)calloc((size_t)k1, sizeof(double));
    if (!sum || !comp || !asum || !acomp) { free(sum); free(comp); free(asum); free(acomp); return OR_EINVAL; }
    for (int64_t c = 0; c < ncols; ++c) {
        for (int64_t m = 0; m < k1; ++m) sum[m] = comp[m] = asum[m] = acomp[m] = 0.0;
        for (int64_t j = 0; j < d; ++j) {
            double a = (c < n) ? load_elem(A, is_f32, j + c * lda) : load_elem(b, is_f32, j);
            int32_t m = h[j];
            if (m < 0 || m >= k1) { free(sum); free(comp); free(asum); free(acomp); return OR_EINVAL; }
            /* "multiplying by the random signs ... is equivalent to either adding or
             *  subtracting A_{j,:}" */
            double v = (s[j] > 0) ? a : -a;
            neumaier_add(&sum[m], &comp[m], v);
            neumaier_add(&asum[m], &acomp[m], fabs(a));
        }
        for (int64_t m = 0; m < k1; ++m) {
            SA[m + c * ldsa] = sum[m] + comp[m];
            if (Tabs) Tabs[m + c * ldsa] = asum[m] + acomp[m];
        }
    }
    free(sum); free(comp); free(asum); free(acomp);
    return OR_OK;
}

/* ------------------------------------------------------------------------
 * c4. Gaussian stage G (k2 x k1, column-major), G_ij ~ N(0, 1/k2)
 * ("s_ij ~ N(0, k^-1)"; multisketch second stage P:L88).
 * Element e = r + c*k2, pair t = e >> 1:
 *   x  = Philox(ctr = (lo32 t, hi32 t, 1, 0), key = seed)     (stream 1, Reading R4)
 *   u1 = (((x1<<32 | x0) >> 11) + 1) * 2^-53  in (0,1]
 *   u2 = ( (x3<<32 | x2) >> 11)      * 2^-53  in [0,1)
 *   rho = sqrt(-2 ln u1);  N_2t = rho cos(2 pi u2);  N_2t+1 = rho sin(2 pi u2)  (Box-Muller)
 *   G_e = N_e / sqrt(k2)
 * ---------------------------------------------------------------------- */
int or_gauss(int64_t k2, int64_t k1, uint64_t seed, double* G, int64_t ldg) {
    if (k2 < 1 || k1 < 1 || ldg < k2 || !G) return OR_EINVAL;
    const double two_pi = 6.283185307179586476925286766559;
    const double inv53 = 1.0 / 9007199254740992.0;  /* 2^-53 */
    double scale = sqrt((double)k2);
    int64_t total = k2 * k1;
    for (int64_t e = 0; e < total; ++e) {
        uint64_t t = (uint64_t)e >> 1;
        uint32_t ctr[4] = {(uint32_t)t, (uint32_t)(t >> 32), 1u, 0u};
        uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
        uint32_t x[4];
        or_philox4x32_10(ctr, key, x);
        uint64_t w1 = ((uint64_t)x[1] << 32) | x[0];
        uint64_t w2 = ((uint64_t)x[3] << 32) | x[2];
        double u1 = (double)((w1 >> 11) + 1u) * inv53;
        double u2 = (double)(w2 >> 11) * inv53;
        double rho = sqrt(-2.0 * log(u1));
        double N = (e & 1) ? rho * sin(two_pi * u2) : rho * cos(two_pi * u2);
        int64_t r = e % k2, c = e / k2;
        G[r + c * ldg] = N / scale;
    }
    return OR_OK;
}

/* c5. G-stage, Z = G Y: plain triple loop with Neumaier-compensated dot
 * products (the multisketch S2(S1 x); Z = GY).
 * Zabs (nullable) = |G| |Yabs| if Yabs given, the sum of |terms| bound. */
int or_gemm_comp(int64_t m, int64_t n, int64_t k, const double* G, int64_t ldg,
                 const double* Y, int64_t ldy, double* Z, int64_t ldz,
                 const double* Yabs, double* Zabs) {
    if (m < 0 || n < 0 || k < 0 || ldg < m || ldy < k || ldz < m || !Z) return OR_EINVAL;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) {
            double sum = 0.0, comp = 0.0, asum = 0.0, acomp = 0.0;
            for (int64_t p = 0; p < k; ++p) {
                neumaier_add(&sum, &comp, G[i + p * ldg] * Y[p + j * ldy]);
                if (Yabs && Zabs) neumaier_add(&asum, &acomp, fabs(G[i + p * ldg]) * Yabs[p + j * ldy]);
            }
            Z[i + j * ldz] = sum + comp;
            if (Yabs && Zabs) Zabs[i + j * ldz] = asum + acomp;
        }
    return OR_OK;
}

/* ------------------------------------------------------------------------
 * c6. Unblocked Householder QR (Golub & Van Loan Alg 5.2.1), in place on the
 * m x nc column-major W; writes R (nc x nc upper, column-major, ldr) with the
 * LAPACK sign convention R_jj = -sign(x_0) ||x||.  Used for the economy QR of
 * Alg 1 line 2 on the augmented sketch [SA | Sb].
 * ---------------------------------------------------------------------- */
int or_householder_qr(int64_t m, int64_t nc, double* W, int64_t ldw, double* R, int64_t ldr) {
    if (m < nc || nc < 1 || ldw < m || ldr < nc || !W || !R) return OR_EINVAL;
    double* v = (double*)malloc((size_t)m * sizeof(double));
    if (!v) return OR_EINVAL;
    for (int64_t j = 0; j < nc; ++j) {
        double norm2 = 0.0;
        for (int64_t i = j; i < m; ++i) norm2 += W[i + j * ldw] * W[i + j * ldw];
        double norm = sqrt(norm2);
        double x0 = W[j + j * ldw];
        double alpha = (x0 >= 0.0) ? -norm : norm;       /* R_jj */
        if (norm == 0.0) alpha = 0.0;
        /* v = x - alpha e1, beta = 2 / (v^T v) */
        double vtv = 0.0;
        for (int64_t i = j; i < m; ++i) {
            v[i] = W[i + j * ldw];
            if (i == j) v[i] -= alpha;
            vtv += v[i] * v[i];
        }
        W[j + j * ldw] = alpha;
        for (int64_t i = j + 1; i < m; ++i) W[i + j * ldw] = 0.0;
        if (vtv > 0.0) {
            double beta = 2.0 / vtv;
            for (int64_t c = j + 1; c < nc; ++c) {           /* W[:,c] -= beta v (v^T W[:,c]) */
                double dot = 0.0;
                for (int64_t i = j; i < m; ++i) dot += v[i] * W[i + c * ldw];
                double f = beta * dot;
                for (int64_t i = j; i < m; ++i) W[i + c * ldw] -= f * v[i];
            }
        }
    }
    for (int64_t c = 0; c < nc; ++c)
        for (int64_t r = 0; r < nc; ++r) R[r + c * ldr] = (r <= c) ? W[r + c * ldw] : 0.0;
    free(v);
    return OR_OK;
}

/* Back substitution R x = y for upper-triangular n x n R (column-major). */
static void back_subst(int64_t n, const double* R, int64_t ldr, const double* y, double* x) {
    for (int64_t i = n - 1; i >= 0; --i) {
        double acc = y[i];
        for (int64_t c = i + 1; c < n; ++c) acc -= R[i + c * ldr] * x[c];
        x[i] = acc / R[i + i * ldr];
    }
}

/* Sketch-and-solve solve phase (Alg 1 lines 2-3) on the augmented
 * sketched matrix Zaug = [S A | S b] (m x (n+1)): R = qr([SA | Sb]);
 * then R[:n,:n] x = R[:n, n] (= Q^T z) and the sketched residual
 * ||S(b - Ax)|| = |R[n,n]|.  Status ESINGULAR if some |R_ii| <= 1e-14 max|R_jj|
 * (S:L340).  Zaug is overwritten. */
int or_sketch_solve(int64_t m, int64_t n, double* Zaug, int64_t ldz, double* x, double* sk_resid) {
    if (n < 1 || m < n + 1 || ldz < m || !Zaug || !x) return OR_EINVAL;
    int64_t nc = n + 1;
    double* R = (double*)malloc((size_t)(nc * nc) * sizeof(double));
    if (!R) return OR_EINVAL;
    int st = or_householder_qr(m, nc, Zaug, ldz, R, nc);
    if (st != OR_OK) { free(R); return st; }
    double rmax = 0.0;
    for (int64_t i = 0; i < n; ++i) rmax = fmax(rmax, fabs(R[i + i * nc]));
    for (int64_t i = 0; i < n; ++i)
        if (!(fabs(R[i + i * nc]) > 1e-14 * rmax)) { free(R); return OR_ESINGULAR; }
    back_subst(n, R, nc, &R[n * nc], x);
    if (sk_resid) *sk_resid = fabs(R[n + n * nc]);
    free(R);
    return OR_OK;
}

/* ------------------------------------------------------------------------
 * c7. Normal equations: C = A^T A, y = A^T b (one Gram of [A b]),
 * Cholesky C = R^T R (POTRF, upper), then two triangular solves
 * x = R^-1 (R^-T y).  A non-positive pivot returns ENOTPD (this failure
 * is load-bearing, "fail for kappa(A) > 10^8").
 * ---------------------------------------------------------------------- */
int or_normal_eq(int64_t d, int64_t n, const double* A, int64_t lda, const double* b, double* x) {
    if (d < n || n < 1 || lda < d || !A || !b || !x) return OR_EINVAL;
    double* C = (double*)calloc((size_t)(n * n), sizeof(double));
    double* y = (double*)calloc((size_t)n, sizeof(double));
    double* z = (double*)calloc((size_t)n, sizeof(double));
    if (!C || !y || !z) { free(C); free(y); free(z); return OR_EINVAL; }
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t i = 0; i <= j; ++i) {
            double acc = 0.0;
            for (int64_t r = 0; r < d; ++r) acc += A[r + i * lda] * A[r + j * lda];
            C[i + j * n] = acc;
            C[j + i * n] = acc;
        }
        double acc = 0.0;
        for (int64_t r = 0; r < d; ++r) acc += A[r + j * lda] * b[r];
        y[j] = acc;
    }
    /* Cholesky, upper: for j: R_jj = sqrt(C_jj - sum_k R_kj^2); R_ji = (C_ji - sum R_kj R_ki)/R_jj */
    for (int64_t j = 0; j < n; ++j) {
        double piv = C[j + j * n];
        for (int64_t k = 0; k < j; ++k) piv -= C[k + j * n] * C[k + j * n];
        if (!(piv > 0.0)) { free(C); free(y); free(z); return OR_ENOTPD; }
        double rjj = sqrt(piv);
        C[j + j * n] = rjj;
        for (int64_t i = j + 1; i < n; ++i) {
            double v = C[j + i * n];
            for (int64_t k = 0; k < j; ++k) v -= C[k + j * n] * C[k + i * n];
            C[j + i * n] = v / rjj;
        }
    }
    /* forward: R^T z = y */
    for (int64_t i = 0; i < n; ++i) {
        double acc = y[i];
        for (int64_t k = 0; k < i; ++k) acc -= C[k + i * n] * z[k];
        z[i] = acc / C[i + i * n];
    }
    back_subst(n, C, n, z, x);
    free(C); free(y); free(z);
    return OR_OK;
}

/* ------------------------------------------------------------------------
 * NEXT-1. rand_cholQR least squares, Alg 5 (Alg 4),
 * written in the paper's order and notation:
 *   1  Y = S A                      (given: the k x n sketch, here the multisketch G S1 A)
 *   2  [~, R0] = qr(Y, 0)           (Householder, or_householder_qr)
 *   3  Q0 = A R0^-1                 (row-wise forward substitution: q R0 = a, i.e. TRSM)
 *   4  G = Q0^T Q0,  z = Q0^T b     (plain loops)
 *   5  R1 = chol(G)                 (upper, ENOTPD on a non-positive pivot)
 *   6  R = R1 R0
 *   7  y = R1^-T z
 *   8  x = R^-1 y
 * R (nullable, n x n column-major, ldr) receives line 6's R.  Returns ESINGULAR if
 * some |R0_ii| <= 1e-14 max|R0_jj| (as for sketch-and-solve).
 * ---------------------------------------------------------------------- */
int or_rand_cholqr_lstsq(int64_t d, int64_t n, const double* A, int64_t lda, const double* b,
                         const double* Y, int64_t k, int64_t ldy, double* x, double* R, int64_t ldr) {
    if (n < 1 || d < n || k < n || lda < d || ldy < k || !A || !b || !Y || !x || (R && ldr < n))
        return OR_EINVAL;
    double* W = (double*)malloc((size_t)(k * n) * sizeof(double));
    double* R0 = (double*)malloc((size_t)(n * n) * sizeof(double));
    double* Q0 = (double*)malloc((size_t)(d * n) * sizeof(double));
    double* G = (double*)calloc((size_t)(n * n), sizeof(double));
    double* z = (double*)calloc((size_t)n, sizeof(double));
    double* Rf = (double*)calloc((size_t)(n * n), sizeof(double));
    double* y = (double*)calloc((size_t)n, sizeof(double));
    int st = OR_OK;
    if (!W || !R0 || !Q0 || !G || !z || !Rf || !y) { st = OR_EINVAL; goto done; }
    /* line 2 */
    for (int64_t c = 0; c < n; ++c)
        for (int64_t r = 0; r < k; ++r) W[r + c * k] = Y[r + c * ldy];
    st = or_householder_qr(k, n, W, k, R0, n);
    if (st != OR_OK) goto done;
    {
        double rmax = 0.0;
        for (int64_t i = 0; i < n; ++i) rmax = fmax(rmax, fabs(R0[i + i * n]));
        for (int64_t i = 0; i < n; ++i)
            if (!(fabs(R0[i + i * n]) > 1e-14 * rmax)) { st = OR_ESINGULAR; goto done; }
    }
    /* line 3: for every row r, q R0 = a  =>  q_j = (a_j - sum_{l<j} q_l R0[l,j]) / R0[j,j] */
    for (int64_t r = 0; r < d; ++r)
        for (int64_t j = 0; j < n; ++j) {
            double acc = A[r + j * lda];
            for (int64_t l = 0; l < j; ++l) acc -= Q0[r + l * d] * R0[l + j * n];
            Q0[r + j * d] = acc / R0[j + j * n];
        }
    /* line 4 */
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t i = 0; i <= j; ++i) {
            double acc = 0.0;
            for (int64_t r = 0; r < d; ++r) acc += Q0[r + i * d] * Q0[r + j * d];
            G[i + j * n] = acc;
            G[j + i * n] = acc;
        }
        double acc = 0.0;
        for (int64_t r = 0; r < d; ++r) acc += Q0[r + j * d] * b[r];
        z[j] = acc;
    }
    /* line 5: upper Cholesky G = R1^T R1, R1 stored in the upper triangle of G */
    for (int64_t j = 0; j < n; ++j) {
        double piv = G[j + j * n];
        for (int64_t l = 0; l < j; ++l) piv -= G[l + j * n] * G[l + j * n];
        if (!(piv > 0.0)) { st = OR_ENOTPD; goto done; }
        double rjj = sqrt(piv);
        G[j + j * n] = rjj;
        for (int64_t i = j + 1; i < n; ++i) {
            double v = G[j + i * n];
            for (int64_t l = 0; l < j; ++l) v -= G[l + j * n] * G[l + i * n];
            G[j + i * n] = v / rjj;
        }
    }
    /* line 6: R = R1 R0 (both upper) */
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i <= j; ++i) {
            double acc = 0.0;
            for (int64_t l = i; l <= j; ++l) acc += G[i + l * n] * R0[l + j * n];
            Rf[i + j * n] = acc;
        }
    /* line 7: R1^T y = z (forward) */
    for (int64_t i = 0; i < n; ++i) {
        double acc = z[i];
        for (int64_t l = 0; l < i; ++l) acc -= G[l + i * n] * y[l];
        y[i] = acc / G[i + i * n];
    }
    /* line 8: R x = y (back) */
    back_subst(n, Rf, n, y, x);
    if (R)
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < n; ++i) R[i + j * ldr] = Rf[i + j * n];
done:
    free(W); free(R0); free(Q0); free(G); free(z); free(Rf); free(y);
    return st;
}

/* ------------------------------------------------------------------------
 * NEXT-3. SRHT (Def): S = k^-1/2 P H_d D, d = 2^q.
 *   D = diag(d_i), d_i = +-1: bit 0 of w_i, w_i = word (i & 3) of
 *       Philox(ctr = (lo32(i>>2), hi32(i>>2), 6, 0), key = seed)      (stream 6, Reading R17)
 *   P: k sampled rows p_j = mulhi32(v_j, d) (Lemire), v_j = word (j & 3) of
 *       Philox(ctr = (lo32(j>>2), hi32(j>>2), 7, 0), key = seed)      (stream 7; i.i.d.
 *       uniform row sampling with replacement, Reading R16)
 *   H_d: Sylvester-ordered Hadamard, applied by Alg 3: radix-4 stages
 *       at stride d/4, d/16, ..., with one radix-2 stage at stride 1 when q is odd
 *       (Reading R18); 0-based indices i0 = b + k (the paper's b + k + 1 is 1-based).
 * ---------------------------------------------------------------------- */
static uint32_t stream_word(uint64_t seed, uint64_t i, uint32_t stream) {
    uint32_t ctr[4] = {(uint32_t)(i >> 2), (uint32_t)(i >> 34), stream, 0u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t x[4];
    or_philox4x32_10(ctr, key, x);
    return x[i & 3];
}

int or_srht_draws(int64_t d, int64_t k, uint64_t seed, int8_t* D, int64_t* p) {
    if (d < 1 || k < 1 || (d & (d - 1)) || !D || !p) return OR_EINVAL;
    for (int64_t i = 0; i < d; ++i) D[i] = (stream_word(seed, (uint64_t)i, 6u) & 1u) ? -1 : 1;
    for (int64_t j = 0; j < k; ++j)
        p[j] = (int64_t)(((uint64_t)stream_word(seed, (uint64_t)j, 7u) * (uint64_t)d) >> 32);
    return OR_OK;
}

/* Alg 3, in place on a (length d = 2^q). */
int or_fwht_rad4(int64_t d, double* a) {
    if (d < 1 || (d & (d - 1)) || !a) return OR_EINVAL;
    int64_t stride = d / 4;
    while (stride >= 1) {
        int64_t s4 = stride * 4;
        for (int64_t b = 0; b <= d - s4; b += s4)
            for (int64_t kk = 0; kk < stride; ++kk) {
                int64_t i0 = b + kk, i1 = i0 + stride, i2 = i0 + 2 * stride, i3 = i0 + 3 * stride;
                double x = a[i0], y = a[i1], zz = a[i2], t = a[i3];
                double X = x + zz, Y = y + t, Z = x - zz, T = y - t;
                a[i0] = X + Y; a[i1] = X - Y; a[i2] = Z + T; a[i3] = Z - T;
            }
        stride /= 4;
    }
    /* odd q: the radix-4 sweep ended at stride 2 (it covered bits q-1..1); bit 0 remains */
    int q = 0;
    while (((int64_t)1 << q) < d) ++q;
    if (q & 1)
        for (int64_t i0 = 0; i0 < d; i0 += 2) {
            double x = a[i0], y = a[i0 + 1];
            a[i0] = x + y; a[i0 + 1] = x - y;
        }
    return OR_OK;
}

/* Y = S [A b] (k x ncols, column-major, ldy): per column, v = D a; v = H v (Alg 3);
 * Y[j, c] = v[p_j] / sqrt(k). */
int or_srht_apply(int64_t d, int64_t n, int64_t k, uint64_t seed, const double* A, int64_t lda,
                  const double* b, double* Y, int64_t ldy) {
    int64_t ncols = n + (b ? 1 : 0);
    if (d < 1 || (d & (d - 1)) || k < 1 || ncols < 1 || ldy < k || (n > 0 && (!A || lda < d)) || !Y)
        return OR_EINVAL;
    int8_t* D = (int8_t*)malloc((size_t)d);
    int64_t* p = (int64_t*)malloc((size_t)k * sizeof(int64_t));
    double* v = (double*)malloc((size_t)d * sizeof(double));
    if (!D || !p || !v) { free(D); free(p); free(v); return OR_EINVAL; }
    or_srht_draws(d, k, seed, D, p);
    double scale = 1.0 / sqrt((double)k);
    for (int64_t c = 0; c < ncols; ++c) {
        for (int64_t i = 0; i < d; ++i) {
            double a = (c < n) ? A[i + c * lda] : b[i];
            v[i] = D[i] > 0 ? a : -a;
        }
        or_fwht_rad4(d, v);
        for (int64_t j = 0; j < k; ++j) Y[j + c * ldy] = v[p[j]] * scale;
    }
    free(D); free(p); free(v);
    return OR_OK;
}

/* ||b - A x||_2 with compensated accumulation (P:L338 relative residual
 * numerator; verification only, not part of the timed path). */
double or_residual_norm(int64_t d, int64_t n, const double* A, int64_t lda, const double* b, const double* x) {
    double ss = 0.0, sc = 0.0;
    for (int64_t r = 0; r < d; ++r) {
        double acc = 0.0, comp = 0.0;
        neumaier_add(&acc, &comp, b[r]);
        for (int64_t c = 0; c < n; ++c) neumaier_add(&acc, &comp, -A[r + c * lda] * x[c]);
        double e = acc + comp;
        neumaier_add(&ss, &sc, e * e);
    }
    return sqrt(ss + sc);
}
