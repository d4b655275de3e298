// gstage.cu -- a5, the multisketch's Gaussian stage Z = G (S [A b]) on the fp64 tensor pipe.
//
// P:L88 (S = S2 S1), P:L228 ("computed the product Z = GY ... via Z^T = Y^T G^T": Y = S1 [A b] is
// consumed in its row-major form), Table 1 P:L99 (the dn + n^4 term: 2 k2 k1 (n+1) flops, 8 n^4 at
// k1 = 2n^2, k2 = 2n).  G is k2 x k1 column-major (ld ldg >= k2, rows past k2 zero), Y^T is the
// CountSketch's row-major workspace (RowOut layout: element (m, c) at (c / cw) cs + m lc + (c % cw)).
//
// Design:
//  * the output is tiny (k2 x (n+1)) and K = k1 is long, so the k-blocks of every output tile are
//    flattened into one range that is split evenly over the CTAs (stream-K): CTA c takes
//    [c total / P, (c+1) total / P) and writes one partial tile per tile it touches; a second kernel
//    adds the partials of each tile in increasing k order (fixed order: deterministic, and the
//    accumulation depth of one chain is bounded, see below);
//  * CTA tile BM = 64 MW rows x BN = 8 NT columns (a column chunk of Y^T, <= 72); 8 warps, warp w owns
//    rows [8 MW w, 8 MW (w+1)) x all BN columns: MW x NT independent DMMA m8n8k4 accumulators;
//  * operands staged by cp.async (16 B, zero-filled past k1) into a STAGES-deep ring; shared rows are
//    padded to ld == 4 (mod 16) doubles so the A fragment (row g, k t) and B fragment (k t, col g)
//    loads of a half-warp hit 16 distinct double-banks (conflict-free);
//  * error bound: a DMMA chain accumulates at most kFlushK = 4096 products, then is
//    added into a second register accumulator; with <= ceil(k1 / 4096) + #partials further fp64 adds
//    the error stays <= (4096 + ~50) u |G| T, inside 1e-12 |G| T.
#include <algorithm>
#include <cstdlib>

#include "csk_internal.cuh"

namespace csk {

namespace {

constexpr int kGsWarps = 8;
constexpr int kFlushK = 4096;

__host__ __device__ constexpr int pad16_4(int x) { return ((x + 11) / 16) * 16 + 4; }   // >= x, == 4 mod 16

template <int MW, int NT, int BK, int STAGES>
struct Cfg {
    static constexpr int BM = 8 * kGsWarps * MW;
    static constexpr int BN = 8 * NT;
    static constexpr int LDA = pad16_4(BM);
    static constexpr int LDB = pad16_4(BN);
    static constexpr int A_STAGE = BK * LDA;   // doubles
    static constexpr int B_STAGE = BK * LDB;
    static constexpr int STAGE = A_STAGE + B_STAGE;
    static constexpr size_t SMEM = (size_t)STAGES * STAGE * sizeof(double);
    static constexpr int FLUSH_BLOCKS = kFlushK / BK;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    const int n = valid ? 16 : 0;   // src-size 0: 16 zero bytes (K tail)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// not volatile: a pure function of its operands, so the compiler may interleave it with the
// fragment loads of the next k-step (the DMMA chains' latency is what the issue order must hide)
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

struct GsArgs {
    const double* G;
    int64_t ldg;
    int k2;
    int64_t k1;
    const double* Yt;   // RowOut workspace
    int64_t lc, cs;
    int cw, ncols;
    int MT, NCH;        // M tiles, column chunks
    int64_t KB;         // k-blocks per tile
    int64_t total;      // MT * NCH * KB
    int P;              // CTAs
    int maxseg;         // partial slots per CTA
    double* part;       // P * maxseg partial tiles (BM x BN, column-major)
};

// q0(c) = floor(c * total / P): the first flattened k-block of CTA c
__host__ __device__ __forceinline__ int64_t range_begin(int64_t c, int64_t total, int P) {
    return (int64_t)(((uint64_t)c * (uint64_t)total) / (uint64_t)P);   // c <= P <= 2^16, total < 2^47
}

template <int MW, int NT, int BK, int STAGES>
__global__ void __launch_bounds__(kGsWarps * 32, 1) gstage_kernel(GsArgs a) {
    using C = Cfg<MW, NT, BK, STAGES>;
    extern __shared__ __align__(16) double gs_smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int64_t q0 = range_begin(blockIdx.x, a.total, a.P);
    const int64_t q1 = range_begin(blockIdx.x + 1, a.total, a.P);
    if (q0 >= q1) return;
    const int64_t tile0 = q0 / a.KB;

    // ---- loader: flattened k-block q -> stage slot
    auto load = [&](int64_t q, int slot) {
        const int64_t tile = q / a.KB, kb = q - tile * a.KB;
        const int mt = (int)(tile % a.MT), ch = (int)(tile / a.MT);
        const int64_t k0 = kb * BK;
        double* sA = gs_smem + (size_t)slot * C::STAGE;
        double* sB = sA + C::A_STAGE;
        // G tile: BK columns of BM contiguous doubles (rows m0 .. m0 + BM; ldg >= k2 and the
        // allocation has BM doubles of tail padding, so reads past row k2 stay in bounds)
        const double* Gt = a.G + (int64_t)mt * C::BM;
        constexpr int A_CHUNKS = BK * C::BM / 2;
#pragma unroll
        for (int i = 0; i < (A_CHUNKS + kGsWarps * 32 - 1) / (kGsWarps * 32); ++i) {
            const int id = tid + i * kGsWarps * 32;
            if (A_CHUNKS % (kGsWarps * 32) == 0 || id < A_CHUNKS) {
                const int kk = id / (C::BM / 2), m2 = id - kk * (C::BM / 2);
                const int64_t k = k0 + kk;
                const bool v = k < a.k1;
                cp_async16(sA + kk * C::LDA + 2 * m2, Gt + (v ? k : 0) * a.ldg + 2 * m2, v);
            }
        }
        // Y^T tile: BK rows of the chunk's (<= BN) columns, 16-B pieces up to the even width
        const int c0 = ch * a.cw;
        const int ncw = min(a.cw, a.ncols - c0);
        const int pieces = (ncw + 1) >> 1;
        const double* Yc = a.Yt + (int64_t)ch * a.cs;
        for (int id = tid; id < BK * (C::BN / 2); id += kGsWarps * 32) {
            const int kk = id / (C::BN / 2), p = id - kk * (C::BN / 2);
            if (p < pieces) {
                const int64_t k = k0 + kk;
                const bool v = k < a.k1;
                cp_async16(sB + kk * C::LDB + 2 * p, Yc + (v ? k : 0) * a.lc + 2 * p, v);
            }
        }
    };

    double acc[MW][NT][2], hi[MW][NT][2];
#pragma unroll
    for (int i = 0; i < MW; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = hi[i][j][0] = hi[i][j][1] = 0.0;

    const int64_t nq = q1 - q0;
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nq) load(q0 + s, s);
        cp_async_commit();
    }
    int64_t seg_begin = q0;
    for (int64_t i = 0; i < nq; ++i) {
        const int64_t q = q0 + i;
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        if (i + STAGES - 1 < nq) load(q + STAGES - 1, (int)((i + STAGES - 1) % STAGES));
        cp_async_commit();
        const double* sA = gs_smem + (size_t)(i % STAGES) * C::STAGE + 8 * MW * warp + g;
        const double* sB = gs_smem + (size_t)(i % STAGES) * C::STAGE + C::A_STAGE + g;
        // fragments double-buffered in registers: step k4 + 1's loads issue before step k4's DMMAs
        double fa[2][MW], fb[2][NT];
#pragma unroll
        for (int mi = 0; mi < MW; ++mi) fa[0][mi] = sA[t * C::LDA + 8 * mi];
#pragma unroll
        for (int nj = 0; nj < NT; ++nj) fb[0][nj] = sB[t * C::LDB + 8 * nj];
#pragma unroll
        for (int k4 = 0; k4 < BK / 4; ++k4) {
            const int cur = k4 & 1, nxt = cur ^ 1;
            if (k4 + 1 < BK / 4) {
#pragma unroll
                for (int mi = 0; mi < MW; ++mi) fa[nxt][mi] = sA[(4 * k4 + 4 + t) * C::LDA + 8 * mi];
#pragma unroll
                for (int nj = 0; nj < NT; ++nj) fb[nxt][nj] = sB[(4 * k4 + 4 + t) * C::LDB + 8 * nj];
            }
#pragma unroll
            for (int mi = 0; mi < MW; ++mi)
#pragma unroll
                for (int nj = 0; nj < NT; ++nj) dmma(acc[mi][nj][0], acc[mi][nj][1], fa[cur][mi], fb[cur][nj]);
        }
        const int64_t tile = q / a.KB;
        const bool seg_end = (q + 1 == q1) || ((q + 1) % a.KB == 0);
        if (seg_end || (q - seg_begin + 1) % C::FLUSH_BLOCKS == 0) {
#pragma unroll
            for (int mi = 0; mi < MW; ++mi)
#pragma unroll
                for (int nj = 0; nj < NT; ++nj) {
                    hi[mi][nj][0] += acc[mi][nj][0];
                    hi[mi][nj][1] += acc[mi][nj][1];
                    acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
                }
        }
        if (seg_end) {
            // partial tile (BM x BN column-major) of this segment -> slot (CTA, tile - tile0)
            double* P = a.part + ((int64_t)blockIdx.x * a.maxseg + (tile - tile0)) * (C::BM * C::BN);
#pragma unroll
            for (int mi = 0; mi < MW; ++mi)
#pragma unroll
                for (int nj = 0; nj < NT; ++nj) {
                    const int m = 8 * MW * warp + 8 * mi + g, n = 8 * nj + 2 * t;
                    P[(int64_t)n * C::BM + m] = hi[mi][nj][0];
                    P[(int64_t)(n + 1) * C::BM + m] = hi[mi][nj][1];
                    hi[mi][nj][0] = hi[mi][nj][1] = 0.0;
                }
            seg_begin = q + 1;
        }
    }
    cp_async_wait<0>();
}

// Z[m, c] (valid rows < k2, columns < ncols) = sum over the CTAs that touched the tile, in CTA order
// (= increasing k), of their partials.  One thread per output element.
template <typename TZ>
__global__ void gstage_reduce_kernel(GsArgs a, int BM, int BN, TZ* __restrict__ Z, int64_t ldz) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t per_tile = (int64_t)BM * BN;
    const int64_t tile = e / per_tile;
    if (tile >= (int64_t)a.MT * a.NCH) return;
    const int r = (int)(e - tile * per_tile);
    const int m_loc = r % BM, n_loc = r / BM;
    const int mt = (int)(tile % a.MT), ch = (int)(tile / a.MT);
    const int m = mt * BM + m_loc, c = ch * a.cw + n_loc;
    if (m >= a.k2 || n_loc >= a.cw || c >= a.ncols) return;
    // contributors: CTAs whose range [q0, q1) meets [tile KB, (tile+1) KB)
    const int64_t lo = tile * a.KB, hi = lo + a.KB;
    int c_lo = 0, c_hi = a.P - 1;
    {   // largest c with q0(c) <= lo
        int L = 0, R = a.P - 1;
        while (L < R) {
            const int mid = (L + R + 1) >> 1;
            if (range_begin(mid, a.total, a.P) <= lo) L = mid; else R = mid - 1;
        }
        c_lo = L;
        L = c_lo, R = a.P - 1;   // largest c with q0(c) < hi
        while (L < R) {
            const int mid = (L + R + 1) >> 1;
            if (range_begin(mid, a.total, a.P) < hi) L = mid; else R = mid - 1;
        }
        c_hi = L;
    }
    double z = 0.0;
    for (int cc = c_lo; cc <= c_hi; ++cc) {
        const int64_t q0 = range_begin(cc, a.total, a.P), q1 = range_begin(cc + 1, a.total, a.P);
        if (q1 <= q0) continue;   // empty range (P > total)
        const int64_t slot = (int64_t)cc * a.maxseg + (tile - q0 / a.KB);
        z += a.part[slot * per_tile + r];
    }
    Z[m + (int64_t)c * ldz] = (TZ)z;
}

template <int MW, int NT, int BK, int STAGES>
csk_status launch(GsArgs& a, void* Z, int64_t ldz, bool z_f32, cudaStream_t st) {
    using C = Cfg<MW, NT, BK, STAGES>;
    auto kern = gstage_kernel<MW, NT, BK, STAGES>;
    CSK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    a.MT = (a.k2 + C::BM - 1) / C::BM;
    a.NCH = (a.ncols + a.cw - 1) / a.cw;
    a.KB = ceil_div(a.k1, BK);
    a.total = (int64_t)a.MT * a.NCH * a.KB;
    const int nsm = device_info().num_sms;
    // at least ~2 k-blocks per CTA (the ring needs work to overlap), at most one CTA per SM
    int64_t P = std::min<int64_t>(nsm, std::max<int64_t>(1, a.total / 2));
    if (const char* e = std::getenv("CSK_GS_CTAS")) P = std::max<int64_t>(1, std::min<int64_t>(std::atoll(e), a.total));
    a.P = (int)P;
    CSK_REQUIRE(a.total < (int64_t(1) << 47), CSK_EUNSUPPORTED, "G-stage: k1 too large");
    const int64_t share = ceil_div(a.total, P);
    a.maxseg = (int)(ceil_div(share, a.KB) + 1);
    const size_t part_bytes = (size_t)P * a.maxseg * C::BM * C::BN * sizeof(double);
    double* part = nullptr;
    CSK_CUDA_TRY(csk_malloc_async(&part, part_bytes, st));
    a.part = part;
    kern<<<(unsigned)P, kGsWarps * 32, C::SMEM, st>>>(a);
    count_launch();
    cudaError_t e1 = cudaGetLastError();
    const int64_t outs = (int64_t)a.MT * a.NCH * C::BM * C::BN;
    const unsigned rgrid = (unsigned)ceil_div(outs, 256);
    if (e1 == cudaSuccess) {
        if (z_f32)
            gstage_reduce_kernel<float><<<rgrid, 256, 0, st>>>(a, C::BM, C::BN, (float*)Z, ldz);
        else
            gstage_reduce_kernel<double><<<rgrid, 256, 0, st>>>(a, C::BM, C::BN, (double*)Z, ldz);
        count_launch();
        e1 = cudaGetLastError();
    }
    cudaFreeAsync(part, st);
    if (e1 != cudaSuccess) {
        set_error("G-stage launch failed: %s", cudaGetErrorString(e1));
        return CSK_ECUDA;
    }
    return CSK_OK;
}

template <int MW>
csk_status dispatch_nt(GsArgs& a, int nt, void* Z, int64_t ldz, bool z_f32, cudaStream_t st) {
    constexpr int BK = 32;
    constexpr int ST = 4;
    if (nt <= 1) return launch<MW, 1, BK, ST>(a, Z, ldz, z_f32, st);
    if (nt <= 2) return launch<MW, 2, BK, ST>(a, Z, ldz, z_f32, st);
    if (nt <= 4) return launch<MW, 4, BK, ST>(a, Z, ldz, z_f32, st);
    if (nt <= 7) return launch<MW, 7, BK, ST>(a, Z, ldz, z_f32, st);
    return launch<MW, 9, BK, ST>(a, Z, ldz, z_f32, st);
}

}  // namespace

// Z (k2 x ncols, column-major, ldz; fp64 or fp32) = G (k2 x k1, ldg, >= 256 doubles of tail padding)
// times the row-major workspace described by ro (ro.cw <= 72 columns per chunk).
csk_status gstage_launch(const double* G, int64_t ldg, int64_t k2, int64_t k1, const RowOut& ro, void* Z,
                         int64_t ldz, bool z_f32, cudaStream_t st) {
    CSK_REQUIRE(ro.ws != nullptr && ro.cw >= 1 && ro.cw <= kGstageMaxCw, CSK_EINVAL,
                "G-stage: chunk width %d not in [1, %d]", ro.cw, kGstageMaxCw);
    CSK_REQUIRE((ro.lc & 1) == 0 && (ro.cs & 1) == 0 && (ldg & 1) == 0 && ((uintptr_t)ro.ws & 15) == 0 &&
                    ((uintptr_t)G & 15) == 0,
                CSK_EINVAL, "G-stage: operands must be 16-B aligned");
    GsArgs a{};
    a.G = G;
    a.ldg = ldg;
    a.k2 = (int)k2;
    a.k1 = k1;
    a.Yt = ro.ws;
    a.lc = ro.lc;
    a.cs = ro.cs;
    a.cw = ro.cw;
    a.ncols = ro.ncols;
    const int nt = (ro.cw + 7) / 8;
    // BM = 128 rows per CTA tile (MW = 2): the two register accumulator sets (DMMA chain + flush target)
    // of a 128 x 72 tile take 144 of a thread's registers; 256-row tiles would spill
    return dispatch_nt<2>(a, nt, Z, ldz, z_f32, st);
}

}  // namespace csk
