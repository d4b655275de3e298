// srht.cu -- srht_apply: the SRHT S = k^-1/2 P H_d D (Def)
// applied to [A b], column-major, fp64.
//
// B200 design (not the paper's multi-pass FWHT): only k of the d rows of H D a are
// kept, and H_d = H_{d/L} (x) H_L (Sylvester order: H[p, i] = (-1)^popcount(p & i)), so with
// i = hi*L + lo and p_j = ph_j*L + pl_j
//     y_j = k^-1/2 sum_hi (-1)^popcount(ph_j & hi) * (H_L (D a)[hi-block])[pl_j].
// One pass over A: a warp (or, for k > 512, a 64-thread CTA) takes (column, row block) units, applies
// D while loading the block (coalesced), runs the block's FWHT on chip in registers with one padded
// shared-memory exchange, and adds the k sampled entries, signed by the block's hi index, into
// per-thread accumulators that are flushed to Y once per column.
// HBM traffic = d * ncols * 8 bytes read (+ d/8 bytes of D bits); the paper's implementation
// reads and writes A O(log k) times.  Alg 3's radix-4 butterfly order
// becomes radix-32/64 in registers; every stage is the same Sylvester factor, so the result is
// H_L regardless of stage order (R22).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "csk_internal.cuh"

namespace csk {

void prof_mark(cudaStream_t st, bool begin);

constexpr int kHL = 4096;            // FWHT block length on chip


// D as packed bits: bit (i & 31) of dbits[i >> 5] = 1 iff D_ii = -1, local row i = global row0 + i
// (Reading R21: bit 0 of word (g & 3) of Philox(ctr = (lo32(g>>2), hi32(g>>2), 6, 0), key = seed)).
__global__ void srht_dbits_kernel(uint32_t* __restrict__ dbits, int64_t nwords, int64_t row0, uint32_t key0,
                                  uint32_t key1) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords; w += (int64_t)gridDim.x * blockDim.x) {
        uint32_t bits = 0;
        const uint64_t g0 = (uint64_t)row0 + (uint64_t)w * 32;   // multiple of 4
        for (int q = 0; q < 8; ++q) {
            const uint64_t blk = (g0 >> 2) + q;
            const uint4 x = philox4x32_10(make_uint4((uint32_t)blk, (uint32_t)(blk >> 32), 6u, 0u), make_uint2(key0, key1));
            bits |= ((x.x & 1u) | ((x.y & 1u) << 1) | ((x.z & 1u) << 2) | ((x.w & 1u) << 3)) << (4 * q);
        }
        dbits[w] = bits;
    }
}

// sampled rows p_j = floor(w_j * dglob / 2^32) (dglob <= 2^32), w_j from stream 7
__global__ void srht_samples_kernel(uint32_t* __restrict__ p, int64_t k, uint64_t dglob, uint32_t key0, uint32_t key1) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
        const uint4 x = philox4x32_10(make_uint4((uint32_t)(j >> 2), (uint32_t)(j >> 34), 7u, 0u), make_uint2(key0, key1));
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
        p[j] = (uint32_t)(((uint64_t)w[j & 3] * dglob) >> 32);
    }
}

// (Round 1's 3-phase radix-16 CTA kernels -- register loads, and a 2-stage TMA ring -- measured 2.44 /
// 2.40 ms against the warp kernel's 1.87 ms at d = 2^23 x 129, k = 256; removed in round 2.)

// Radix-64 CTA variant (default for k > 512): 64 threads per block of L = 4096 rows, 64 elements per
// thread, so H_L = two radix-64 register phases with ONE padded shared-memory exchange, and only
// the k sampled positions are written back for the gather (a 4096-bit sample map).  Per 32 KB of
// A this moves ~68 KB through shared memory (the 3-phase kernels move ~200-260 KB: shared-memory
// bandwidth, not HBM, bounded them at ~3.6 TB/s).  Loads go straight to registers, coalesced.
constexpr int kH64Threads = 64;
constexpr int kH64Pad = kHL + kHL / 64;
__device__ __forceinline__ int hpad64(int i) { return i + (i >> 6); }

__device__ __forceinline__ void fwht64(double (&x)[64]) {
#pragma unroll
    for (int h = 1; h < 64; h <<= 1)
#pragma unroll
        for (int i = 0; i < 64; ++i)
            if ((i & h) == 0) {
                const double a = x[i], b = x[i + h];
                x[i] = a + b;
                x[i + h] = a - b;
            }
}

template <int R>   // samples per thread: k <= 64 R
__global__ void __launch_bounds__(kH64Threads) srht_r64_kernel(const double* __restrict__ A, int64_t lda,
                                                               const double* __restrict__ bvec, int n, int ncols,
                                                               int64_t nblk, int64_t hb0,
                                                               const uint32_t* __restrict__ dbits,
                                                               const uint32_t* __restrict__ psamp, int k, double scale,
                                                               double* __restrict__ Y, int64_t ldy) {
    __shared__ double xs[kH64Pad];
    __shared__ uint32_t smap[kHL / 32];   // bit pos set iff some sample has in-block row pos
    const int t = threadIdx.x;
    const int64_t total = nblk * ncols;
    const int64_t per = (total + gridDim.x - 1) / gridDim.x;
    const int64_t u0 = blockIdx.x * per, u1 = min(total, u0 + per);
    if (u0 >= u1) return;
    for (int w = t; w < kHL / 32; w += kH64Threads) smap[w] = 0u;
    __syncthreads();
    int pl[R];
    uint32_t ph[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int j = t + r * kH64Threads;
        const uint32_t pj = j < k ? psamp[j] : 0u;
        pl[r] = (int)(pj & (kHL - 1));
        ph[r] = pj / kHL;
        if (j < k) atomicOr(&smap[pl[r] >> 5], 1u << (pl[r] & 31));
    }
    __syncthreads();
    const uint32_t m0 = smap[2 * t], m1 = smap[2 * t + 1];   // samples among this thread's phase-2 rows t*64 + e
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    int cur = (int)(u0 / nblk);
    for (int64_t u = u0; u < u1; ++u) {
        const int c = (int)(u / nblk);
        const int64_t blk = u - (int64_t)c * nblk;
        if (c != cur) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int j = t + r * kH64Threads;
                if (j < k) atomicAdd(Y + j + (int64_t)cur * ldy, acc[r] * scale);
                acc[r] = 0.0;
            }
            cur = c;
        }
        const double* col = (c < n ? A + (int64_t)c * lda : bvec) + blk * kHL;
        const uint32_t* db = dbits + blk * (kHL / 32);
        // phase 1: rows e*64 + t (coalesced), D as a sign flip; FWHT over bits 6..11
        double x[64];
#pragma unroll
        for (int e = 0; e < 64; ++e) x[e] = __ldcs(col + e * kH64Threads + t);
#pragma unroll
        for (int e = 0; e < 64; ++e) {
            const uint32_t bit = (__ldg(db + 2 * e + (t >> 5)) >> (t & 31)) & 1u;
            x[e] = __longlong_as_double(__double_as_longlong(x[e]) ^ ((long long)bit << 63));
        }
        fwht64(x);
#pragma unroll
        for (int e = 0; e < 64; ++e) xs[hpad64(e * kH64Threads + t)] = x[e];
        __syncthreads();
        // phase 2: rows t*64 + e; FWHT over bits 0..5; write back only the sampled rows
#pragma unroll
        for (int e = 0; e < 64; ++e) x[e] = xs[hpad64(t * 64 + e)];
        fwht64(x);
        __syncthreads();   // every thread has read its rows before the sampled ones are rewritten
#pragma unroll
        for (int e = 0; e < 64; ++e)
            if (((e < 32 ? m0 : m1) >> (e & 31)) & 1u) xs[hpad64(t * 64 + e)] = x[e];
        __syncthreads();
        const uint32_t hi = (uint32_t)(hb0 + blk);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double v = xs[hpad64(pl[r])];
            acc[r] += (__popc(ph[r] & hi) & 1) ? -v : v;
        }
        __syncthreads();   // xs is rewritten by the next unit
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int j = t + r * kH64Threads;
        if (j < k) atomicAdd(Y + j + (int64_t)cur * ldy, acc[r] * scale);
    }
}

// Warp-block variant (default for k <= 512): every WARP owns whole 1024-row blocks, 32 rows per
// lane, so H_1024 = two radix-32 register phases with one warp-private padded exchange and no CTA
// barrier at all; 16 resident warps per SM keep ~130 KB of loads in flight.  Samples: lane l
// takes j = l + 32 r; the block's sampled rows are the only ones written back.
constexpr int kHW = 1024;                       // rows per warp block
constexpr int kHWWarps = 4;                     // warps per CTA (independent)
constexpr int kHWPad = kHW + kHW / 32;
__device__ __forceinline__ int hpadw(int i) { return i + (i >> 5); }

__device__ __forceinline__ void fwht32(double (&x)[32]) {
#pragma unroll
    for (int h = 1; h < 32; h <<= 1)
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if ((i & h) == 0) {
                const double a = x[i], b = x[i + h];
                x[i] = a + b;
                x[i + h] = a - b;
            }
}

template <int R>   // samples per lane: k <= 32 R
__global__ void __launch_bounds__(kHWWarps * 32) srht_warp_kernel(const double* __restrict__ A, int64_t lda,
                                                                  const double* __restrict__ bvec, int n, int ncols,
                                                                  int64_t nblk, int64_t hb0,
                                                                  const uint32_t* __restrict__ dbits,
                                                                  const uint32_t* __restrict__ psamp, int k,
                                                                  double scale, double* __restrict__ Y, int64_t ldy) {
    __shared__ double xsall[kHWWarps][kHWPad];
    __shared__ uint32_t smap[kHW / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* xs = xsall[warp];
    for (int w = threadIdx.x; w < kHW / 32; w += blockDim.x) smap[w] = 0u;
    __syncthreads();
    int pl[R];
    uint32_t ph[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int j = lane + 32 * r;
        const uint32_t pj = j < k ? psamp[j] : 0u;
        pl[r] = (int)(pj & (kHW - 1));
        ph[r] = pj / kHW;
        if (j < k && warp == 0) atomicOr(&smap[pl[r] >> 5], 1u << (pl[r] & 31));
    }
    __syncthreads();
    const uint32_t mymap = smap[lane];   // sampled rows among this lane's phase-2 rows lane*32 + e
    const int64_t total = nblk * ncols;
    const int64_t nw = (int64_t)gridDim.x * kHWWarps, gw = (int64_t)blockIdx.x * kHWWarps + warp;
    const int64_t per = (total + nw - 1) / nw;
    const int64_t u0 = gw * per, u1 = min(total, u0 + per);
    if (u0 >= u1) return;
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    int cur = (int)(u0 / nblk);
    for (int64_t u = u0; u < u1; ++u) {
        const int c = (int)(u / nblk);
        const int64_t blk = u - (int64_t)c * nblk;
        if (c != cur) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int j = lane + 32 * r;
                if (j < k) atomicAdd(Y + j + (int64_t)cur * ldy, acc[r] * scale);
                acc[r] = 0.0;
            }
            cur = c;
        }
        const double* col = (c < n ? A + (int64_t)c * lda : bvec) + blk * kHW;
        const uint32_t* db = dbits + blk * (kHW / 32);
        double x[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = __ldcs(col + e * 32 + lane);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            const uint32_t bit = (__ldg(db + e) >> lane) & 1u;
            x[e] = __longlong_as_double(__double_as_longlong(x[e]) ^ ((long long)bit << 63));
        }
        fwht32(x);   // bits 5..9
#pragma unroll
        for (int e = 0; e < 32; ++e) xs[hpadw(e * 32 + lane)] = x[e];
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = xs[hpadw(lane * 32 + e)];
        fwht32(x);   // bits 0..4
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 32; ++e)
            if ((mymap >> e) & 1u) xs[hpadw(lane * 32 + e)] = x[e];
        __syncwarp();
        const uint32_t hi = (uint32_t)(hb0 + blk);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double v = xs[hpadw(pl[r])];
            acc[r] += (__popc(ph[r] & hi) & 1) ? -v : v;
        }
        __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int j = lane + 32 * r;
        if (j < k) atomicAdd(Y + j + (int64_t)cur * ldy, acc[r] * scale);
    }
}

// TMA-fed warp-block variant: as srht_warp_kernel, but each warp's next 1024-row block arrives by
// one cp.async.bulk (8 KB) into a per-warp stage while the current block is transformed, so the
// HBM stream no longer pauses for the FWHT (the register kernel is latency-bound at 16 warps/SM
// when k = 256).  Needs 16-B aligned columns.
template <int R>
__global__ void __launch_bounds__(kHWWarps * 32) srht_warp_tma_kernel(const double* __restrict__ A, int64_t lda,
                                                                      const double* __restrict__ bvec, int n,
                                                                      int ncols, int64_t nblk, int64_t hb0,
                                                                      const uint32_t* __restrict__ dbits,
                                                                      const uint32_t* __restrict__ psamp, int k,
                                                                      double scale, double* __restrict__ Y,
                                                                      int64_t ldy) {
    extern __shared__ __align__(128) double wsm[];
    __shared__ uint32_t smap[kHW / 32];
    __shared__ __align__(8) uint64_t bar[kHWWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* stage = wsm + (size_t)warp * (kHW + kHWPad);
    double* xs = stage + kHW;
    for (int w = threadIdx.x; w < kHW / 32; w += blockDim.x) smap[w] = 0u;
    __syncthreads();
    int pl[R];
    uint32_t ph[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int j = lane + 32 * r;
        const uint32_t pj = j < k ? psamp[j] : 0u;
        pl[r] = (int)(pj & (kHW - 1));
        ph[r] = pj / kHW;
        if (j < k && warp == 0) atomicOr(&smap[pl[r] >> 5], 1u << (pl[r] & 31));
    }
    __syncthreads();
    const uint32_t mymap = smap[lane];
    const int64_t total = nblk * ncols;
    const int64_t nw = (int64_t)gridDim.x * kHWWarps, gw = (int64_t)blockIdx.x * kHWWarps + warp;
    const int64_t per = (total + nw - 1) / nw;
    const int64_t u0 = gw * per, u1 = min(total, u0 + per);
    if (u0 >= u1) return;
    auto src_of = [&](int64_t u) {
        const int c = (int)(u / nblk);
        const int64_t blk = u - (int64_t)c * nblk;
        return (c < n ? A + (int64_t)c * lda : bvec) + blk * kHW;
    };
    if (lane == 0) {
        mbar_init(&bar[warp], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(&bar[warp], kHW * 8);
        bulk_load_1d(stage, src_of(u0), kHW * 8, &bar[warp]);
    }
    __syncwarp();
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    int cur = (int)(u0 / nblk);
    uint32_t parity = 0;
    for (int64_t u = u0; u < u1; ++u) {
        const int c = (int)(u / nblk);
        const int64_t blk = u - (int64_t)c * nblk;
        if (c != cur) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int j = lane + 32 * r;
                if (j < k) atomicAdd(Y + j + (int64_t)cur * ldy, acc[r] * scale);
                acc[r] = 0.0;
            }
            cur = c;
        }
        const uint32_t* db = dbits + blk * (kHW / 32);
        uint32_t dw[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) dw[e] = __ldg(db + e);
        mbar_wait(&bar[warp], parity);
        parity ^= 1u;
        double x[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            const uint32_t bit = (dw[e] >> lane) & 1u;
            x[e] = __longlong_as_double(__double_as_longlong(stage[e * 32 + lane]) ^ ((long long)bit << 63));
        }
        __syncwarp();   // every lane has read the stage: the next block may overwrite it
        if (lane == 0 && u + 1 < u1) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bar[warp], kHW * 8);
            bulk_load_1d(stage, src_of(u + 1), kHW * 8, &bar[warp]);
        }
        fwht32(x);   // bits 5..9
#pragma unroll
        for (int e = 0; e < 32; ++e) xs[hpadw(e * 32 + lane)] = x[e];
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = xs[hpadw(lane * 32 + e)];
        fwht32(x);   // bits 0..4
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 32; ++e)
            if ((mymap >> e) & 1u) xs[hpadw(lane * 32 + e)] = x[e];
        __syncwarp();
        const uint32_t hi = (uint32_t)(hb0 + blk);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double v = xs[hpadw(pl[r])];
            acc[r] += (__popc(ph[r] & hi) & 1) ? -v : v;
        }
        __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int j = lane + 32 * r;
        if (j < k) atomicAdd(Y + j + (int64_t)cur * ldy, acc[r] * scale);
    }
}

// d < 4096: one CTA per column, the whole vector in shared memory, radix-2 stages (Alg 3's
// butterflies, one barrier per stage).
__global__ void __launch_bounds__(256) srht_small_kernel(const double* __restrict__ A, int64_t lda,
                                                         const double* __restrict__ bvec, int n, int d,
                                                         const uint32_t* __restrict__ dbits,
                                                         const uint32_t* __restrict__ psamp, int k, double scale,
                                                         double* __restrict__ Y, int64_t ldy) {
    __shared__ double v[kHL];
    const int c = blockIdx.x;
    const double* col = c < n ? A + (int64_t)c * lda : bvec;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        const uint32_t bit = (dbits[i >> 5] >> (i & 31)) & 1u;
        v[i] = bit ? -col[i] : col[i];
    }
    __syncthreads();
    for (int h = 1; h < d; h <<= 1) {
        for (int q = threadIdx.x; q < d / 2; q += blockDim.x) {
            const int i = (q / h) * 2 * h + (q % h);
            const double a = v[i], b = v[i + h];
            v[i] = a + b;
            v[i + h] = a - b;
        }
        __syncthreads();
    }
    for (int j = threadIdx.x; j < k; j += blockDim.x) Y[j + (int64_t)c * ldy] = v[psamp[j]] * scale;
}

csk_status srht_impl(int64_t d, int64_t dglob, int64_t row0, int64_t k, uint64_t seed, int64_t n,
                            const double* A, int64_t lda, const double* b, double* Y, int64_t ldy, cudaStream_t st) {
    const int64_t ncols = n + (b ? 1 : 0);
    CSK_REQUIRE(d >= 1 && k >= 1 && n >= 0 && ncols >= 1 && Y != nullptr, CSK_EINVAL, "bad SRHT arguments");
    CSK_REQUIRE(n == 0 || A != nullptr, CSK_EINVAL, "A is NULL");
    CSK_REQUIRE(dglob >= 1 && (dglob & (dglob - 1)) == 0 && dglob <= (1LL << 32), CSK_ESHAPE,
                "dglob=%lld must be a power of two <= 2^32 (P:L165: log2 d integer)", (long long)dglob);
    CSK_REQUIRE(row0 >= 0 && row0 + d <= dglob, CSK_ESHAPE, "rows [row0, row0+d) outside [0, dglob)");
    CSK_REQUIRE(n == 0 || lda >= d, CSK_ESHAPE, "lda=%lld < d=%lld", (long long)lda, (long long)d);
    CSK_REQUIRE(ldy >= k, CSK_ESHAPE, "ldy=%lld < k=%lld", (long long)ldy, (long long)k);
    CSK_REQUIRE(k <= 1024, CSK_EUNSUPPORTED, "k=%lld > 1024 sampled rows", (long long)k);
    CSK_REQUIRE(ncols <= 1 << 20, CSK_EINVAL, "too many columns");
    const bool small = dglob < kHL;
    if (small) CSK_REQUIRE(row0 == 0 && d == dglob, CSK_ESHAPE, "dglob < 4096 cannot be row-partitioned");
    else
        CSK_REQUIRE(row0 % kHL == 0 && d % kHL == 0, CSK_ESHAPE,
                    "row blocks must be multiples of 4096 rows (row0=%lld, d=%lld)", (long long)row0, (long long)d);
    CSK_REQUIRE((n == 0 || is_device_pointer(A)) && (!b || is_device_pointer(b)) && is_device_pointer(Y), CSK_EINVAL,
                "srht_apply takes device pointers");
    const int64_t nwords = (d + 31) / 32;
    uint32_t* ws = nullptr;
    CSK_CUDA_TRY(csk_malloc_async(&ws, (size_t)(nwords + k) * 4, st));
    uint32_t* dbits = ws;
    uint32_t* psamp = ws + nwords;
    const uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);
    srht_dbits_kernel<<<(unsigned)std::min<int64_t>(ceil_div(nwords, 256), 4096), 256, 0, st>>>(dbits, nwords, row0,
                                                                                               key0, key1);
    CSK_LAUNCH_CHECK();
    srht_samples_kernel<<<(unsigned)ceil_div(k, 256), 256, 0, st>>>(psamp, k, (uint64_t)dglob, key0, key1);
    CSK_LAUNCH_CHECK();
    const double scale = 1.0 / std::sqrt((double)k);
    if (small) {
        srht_small_kernel<<<(unsigned)ncols, 256, 0, st>>>(A, lda, b, (int)n, (int)d, dbits, psamp, (int)k, scale, Y,
                                                           ldy);
        CSK_LAUNCH_CHECK();
    } else {
        if (ldy == k) {
            CSK_CUDA_TRY(cudaMemsetAsync(Y, 0, (size_t)k * ncols * 8, st));
        } else {
            CSK_CUDA_TRY(cudaMemset2DAsync(Y, ldy * 8, 0, k * 8, ncols, st));
        }
        const int64_t nblk = d / kHL, total = nblk * ncols;
        const DeviceInfo& di = device_info();
        int per_sm = 0;
        const bool al = (n == 0 || (((uintptr_t)A & 15) == 0 && (lda & 1) == 0)) && (!b || ((uintptr_t)b & 15) == 0);
        const char* v = std::getenv("CSK_SRHT_KERNEL");   // test hook: 2 = radix-64 blocks for any k
        const int kv = v ? std::atoi(v) : 0;
        if (kv == 0 && al && k > 128 && k <= 256) {
            // the TMA-fed warp kernel: k = 2n = 256 1.87 -> 1.61 ms at d = 2^23 x 129 (the register
            // kernel is latency-bound there); for k <= 128 (1.58 vs 1.46 ms) and k = 512 (3.89 vs
            // 3.51 ms) the register kernel is faster
            auto kern = srht_warp_tma_kernel<8>;
            const size_t smem = (size_t)kHWWarps * (kHW + kHWPad) * 8;
            CSK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CSK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kHWWarps * 32, smem));
            const int64_t nblk1 = d / kHW, total1 = nblk1 * ncols;
            const int64_t grid = std::min<int64_t>(ceil_div(total1, kHWWarps), (int64_t)di.num_sms * std::max(per_sm, 1));
            prof_mark(st, true);
            kern<<<(unsigned)grid, kHWWarps * 32, smem, st>>>(A, lda, b, (int)n, (int)ncols, nblk1, row0 / kHW, dbits,
                                                              psamp, (int)k, scale, Y, ldy);
            CSK_LAUNCH_CHECK();
        } else if (kv == 0 && k <= 512) {
            auto kern = k <= 128 ? srht_warp_kernel<4> : k <= 256 ? srht_warp_kernel<8> : srht_warp_kernel<16>;
            // (the driver's default carveout measured best: 1.49 ms at d = 2^24 x 65, k = 128; a larger
            // carveout shrinks the L1 that stages the in-flight loads)
            CSK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kHWWarps * 32, 0));
            const int64_t nblk1 = d / kHW, total1 = nblk1 * ncols;
            const int64_t grid = std::min<int64_t>(ceil_div(total1, kHWWarps), (int64_t)di.num_sms * std::max(per_sm, 1));
            prof_mark(st, true);
            kern<<<(unsigned)grid, kHWWarps * 32, 0, st>>>(A, lda, b, (int)n, (int)ncols, nblk1, row0 / kHW, dbits,
                                                           psamp, (int)k, scale, Y, ldy);
            CSK_LAUNCH_CHECK();
        } else {   // k > 512, or CSK_SRHT_KERNEL=2 (test hook): radix-64 CTA blocks
            auto kern = k <= 256 ? srht_r64_kernel<4> : k <= 512 ? srht_r64_kernel<8> : srht_r64_kernel<16>;
            CSK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kH64Threads, 0));
            const int64_t grid = std::min<int64_t>(total, (int64_t)di.num_sms * std::max(per_sm, 1));
            prof_mark(st, true);
            kern<<<(unsigned)grid, kH64Threads, 0, st>>>(A, lda, b, (int)n, (int)ncols, nblk, row0 / kHL, dbits,
                                                         psamp, (int)k, scale, Y, ldy);
            CSK_LAUNCH_CHECK();
        }
        prof_mark(st, false);
    }
    CSK_CUDA_TRY(cudaFreeAsync(ws, st));
    return CSK_OK;
}

}  // namespace csk

extern "C" csk_status srht_apply(int64_t d, int64_t dglob, int64_t row0, int64_t k, uint64_t seed, int64_t n,
                                 const double* A, int64_t lda, const double* b, double* Y, int64_t ldy, void* stream) {
    return csk::srht_impl(d, dglob, row0, k, seed, n, A, lda, b, Y, ldy, (cudaStream_t)stream);
}
