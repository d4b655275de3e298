// gstage.cu -- a5, the multisketch's Gaussian stage Z = G (S [A b]) on the fp64 tensor pipe.
//
// P:L88 (S = S2 S1), P:L228 ("computed the product Z = GY ... via Z^T = Y^T G^T": Y = S1 [A b] is
// consumed in its row-major form), Table 1 P:L99 (the dn + n^4 term: 2 k2 k1 (n+1) flops, 8 n^4 at
// k1 = 2n^2, k2 = 2n).  G is k2 x k1 column-major (ld ldg >= k2, rows past k2 zero), Y^T is the
// CountSketch's row-major workspace (RowOut layout: element (m, c) at (c / cw) cs + m lc + (c % cw)).
//
// Design:
//  * the output is tiny (k2 x (n+1)) and K = k1 is long.  Every output tile's K range is cut into
//    slabs of kSlabK = 4096 (the accumulation-depth bound below); the (tile, slab) k-blocks are
//    flattened into one range cut into P contiguous segments (stream-K, >= 32 k-blocks each, up to 4
//    per CTA slot) that the persistent CTAs grab from a counter -- a CTA whose SM is busy elsewhere
//    (the pipelined step's solve) just takes fewer.  A segment keeps one running partial per tile it
//    touches (its slabs added in order) in its own slot, and the reduce kernel adds the segments'
//    partials of each tile in segment order (= increasing k; deterministic whatever CTA ran them);
//  * CTA = 4 DMMA warps + 1 TMA producer warp, two CTAs per SM.  CTA tile BM = 32 MW rows x BN = 8 NT
//    columns (a column chunk of Y^T, <= 72); DMMA warp w owns 8 MW rows x all BN columns: MW x NT
//    independent m8n8k4 accumulator chains, MW + NT fragment loads per MW NT DMMAs;
//  * operands staged by the TMA engine (1-D bulk copies, one per G row slice / Y^T row, issued by the
//    producer warp) into a 4-deep ring handed over by full (TMA bytes) and empty (one arrive per DMMA
//    warp) mbarriers -- no CTA barrier per k-block; shared rows are padded to ld == 4 (mod 16) doubles
//    so the A fragment (row g, k t) and B fragment (k t, col g) loads of a half-warp hit 16 distinct
//    double-banks (conflict-free);
//  * error bound: one DMMA chain accumulates at most kSlabK = 4096 products; the
//    ceil(k1 / 4096) slab sums and the segment partials are then added in fp64, so the error stays
//    <= (4096 + k1 / 4096 + #segments per tile) u |G| T, inside 1e-12 |G| T for k1 <= 2^27.
#include <algorithm>
#include <cstdlib>

#include "csk_internal.cuh"

namespace csk {

namespace {

constexpr int kGsWarps = 4;   // consumer (DMMA) warps; warp kGsWarps is the TMA producer
constexpr int kSlabK = 4096;
constexpr int kBK = 16;
constexpr int kStages = 4;

__host__ __device__ constexpr int pad16_4(int x) { return ((x + 11) / 16) * 16 + 4; }   // >= x, == 4 mod 16

// NT n8 tiles (BN = 8 NT columns) x MW m8 tiles per consumer warp (BM = 32 MW rows per CTA): MW = 4
// (128 rows) except for the widest chunk (NT = 9), whose 72 accumulators per thread need MW = 2 to
// stay inside the 168 registers two 5-warp CTAs per SM allow
template <int NT>
struct Cfg {
    static constexpr int MW = NT > 8 ? 2 : 4;
    static constexpr int BM = 8 * kGsWarps * MW;
    static constexpr int BN = 8 * NT;
    static constexpr int LDA = pad16_4(BM);
    static constexpr int LDB = pad16_4(BN);
    static constexpr int A_STAGE = kBK * LDA;   // doubles
    static constexpr int B_STAGE = kBK * LDB;
    static constexpr int STAGE = A_STAGE + B_STAGE;
    static constexpr size_t SMEM = (size_t)kStages * STAGE * sizeof(double);
};

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
    int64_t VKB;        // k-blocks per slab
    int64_t NS;         // slabs per tile
    int64_t total;      // MT * NCH * NS * VKB (flattened, last slab of a tile padded)
    int P;              // segments (stream-K ranges), grabbed dynamically by the CTAs
    int maxseg;         // partial slots per segment
    double* part;       // P * maxseg partial tiles (BM x BN, column-major)
    unsigned long long* work;   // segment counter (zeroed before the launch)
};

// q0(c) = floor(c * total / P): the first flattened k-block of CTA c
__host__ __device__ __forceinline__ int64_t range_begin(int64_t c, int64_t total, int P) {
    return (int64_t)(((uint64_t)c * (uint64_t)total) / (uint64_t)P);   // c <= P <= 2^16, total < 2^47
}
// the CTA whose range holds flattened k-block q
__device__ __forceinline__ int cta_of(int64_t q, int64_t total, int P) {
    int c = (int)(((uint64_t)q * (uint64_t)P) / (uint64_t)total);
    while (c + 1 < P && range_begin(c + 1, total, P) <= q) ++c;
    while (c > 0 && range_begin(c, total, P) > q) --c;
    return c;
}

// position of a flattened k-block: (tile, slab, k-block within the slab), advanced without divisions
struct Cursor {
    int64_t kb;      // k-block within the tile (slab * VKB + kin)
    int64_t kin;     // k-block within the slab
    int64_t slab, tile;
    int mt, ch;
    __device__ void init(int64_t q, const GsArgs& a) {
        const int64_t vt = q / a.VKB;
        kin = q - vt * a.VKB;
        tile = vt / a.NS;
        slab = vt - tile * a.NS;
        kb = slab * a.VKB + kin;
        mt = (int)(tile % a.MT);
        ch = (int)(tile / a.MT);
    }
    __device__ void next(const GsArgs& a) {
        ++kb;
        if (++kin == a.VKB) {
            kin = 0;
            if (++slab == a.NS) {
                slab = 0;
                ++tile;
                if (++mt == a.MT) {
                    mt = 0;
                    ++ch;
                }
            }
            kb = slab * a.VKB;
        }
    }
};

__device__ __forceinline__ void mbar_expect_only(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
        : "memory");
}

template <int NT>
__global__ void __launch_bounds__((kGsWarps + 1) * 32, 2) gstage_kernel(GsArgs a) {
    using C = Cfg<NT>;
    extern __shared__ __align__(16) double gs_smem[];
    __shared__ __align__(8) uint64_t full_bar[kStages];
    __shared__ __align__(8) uint64_t empty_bar[kStages];
    __shared__ int64_t s_seg[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    if (tid < kStages) {
        mbar_init(&full_bar[tid], 1);            // the producer's arrive (+ the stage's TMA bytes)
        mbar_init(&empty_bar[tid], kGsWarps);    // one arrive per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");

    // Segments: the flattened (tile, slab, k-block) range is cut into a.P contiguous stream-K segments
    // (~4 per CTA) that the persistent CTAs grab from a counter, so a CTA whose SM is still held by
    // another kernel (the pipelined step's small solve) just takes fewer segments; each segment owns its
    // partial slots, so the fixed-order reduce (segment order = increasing k) is independent of which
    // CTA ran it.  Stage slots and mbarrier phases follow the CTA's running k-block count `base`.
    int64_t base = 0;
    for (int round = 0;; ++round) {
        if (tid == 0) s_seg[round & 1] = (int64_t)atomicAdd(a.work, 1ull);
        __syncthreads();   // (also orders the barrier inits before first use)
        const int64_t seg = s_seg[round & 1];
        if (seg >= a.P) break;
        const int64_t q0 = range_begin(seg, a.total, a.P);
        const int64_t nq = range_begin(seg + 1, a.total, a.P) - q0;
        if (nq <= 0) continue;

        if (warp == kGsWarps) {
            // ---- producer warp: k-block j (CTA count base + j) goes to stage (base + j) % S once the
            // consumers released that stage's previous k-block (empty barrier).  1-D bulk copies (TMA
            // engine), one row per lane: lanes 0..15 the G rows (BM doubles), lanes 16..31 the Y^T rows
            // (the chunk's columns rounded up to 16 B); rows past k1 are zeroed in shared memory instead.
            // Lane 0 posts the byte count first and arrives after the warp's copies and zero stores are
            // issued; padding k-blocks of a short last slab load nothing (the arrive alone completes the
            // phase).  A dedicated warp: inside a DMMA warp the producer ran late behind its own k-blocks
            // (ncu r02: DMMA 77.5%); with a CTA barrier per k-block the barrier stall was 26% (82.6%).
            Cursor lc;
            lc.init(q0, a);
            for (int64_t j = 0; j < nq; ++j) {
                const int64_t pj = base + j;
                const int slot = (int)(pj % kStages);
                if (pj >= kStages) mbar_wait(&empty_bar[slot], (uint32_t)((pj / kStages - 1) & 1));
                uint64_t* bar = &full_bar[slot];
                if (lc.kb < a.KB) {
                    const int64_t k0 = lc.kb * kBK;
                    const int nrows = (int)(a.k1 - k0 < kBK ? a.k1 - k0 : kBK);
                    const int pieces = (min(a.cw, a.ncols - lc.ch * a.cw) + 1) >> 1;
                    const uint32_t bbytes = (uint32_t)pieces * 16;
                    if (lane == 0) mbar_expect_only(bar, (uint32_t)nrows * (C::BM * 8 + bbytes));
                    __syncwarp();
                    double* sA = gs_smem + (size_t)slot * C::STAGE;
                    double* sB = sA + C::A_STAGE;
                    const int kk = lane & 15;
                    if (lane < 16) {
                        if (kk < nrows)
                            bulk_g2s(sA + kk * C::LDA, a.G + (int64_t)lc.mt * C::BM + (k0 + kk) * a.ldg, C::BM * 8,
                                     bar);
                        else
                            for (int e = 0; e < C::BM; ++e) sA[kk * C::LDA + e] = 0.0;
                    } else {
                        if (kk < nrows)
                            bulk_g2s(sB + kk * C::LDB, a.Yt + (int64_t)lc.ch * a.cs + (k0 + kk) * a.lc, bbytes, bar);
                        else
                            for (int e = 0; e < 2 * pieces; ++e) sB[kk * C::LDB + e] = 0.0;
                    }
                    if (nrows < kBK) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                }
                if (lane == 0) mbar_arrive(bar);
                lc.next(a);
            }
        } else {
            // ---- consumer warps: warp w owns rows [8 MW w, 8 MW (w + 1)) of the tile x all BN columns
            double acc[C::MW][NT][2];
#pragma unroll
            for (int i = 0; i < C::MW; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
            Cursor cc;
            cc.init(q0, a);
            const int64_t tile0 = cc.tile;
            bool first_flush = true;   // the running sum of this tile's slot is not written yet
            for (int64_t i = 0; i < nq; ++i) {
                const int64_t pi = base + i;
                const int slot = (int)(pi % kStages);
                mbar_wait(&full_bar[slot], (uint32_t)((pi / kStages) & 1));
                if (cc.kb < a.KB) {
                    const double* sA = gs_smem + (size_t)slot * C::STAGE + 8 * C::MW * warp + g;
                    const double* sB = gs_smem + (size_t)slot * C::STAGE + C::A_STAGE + g;
#pragma unroll
                    for (int k4 = 0; k4 < kBK / 4; ++k4) {
                        double fa[C::MW], fb[NT];
#pragma unroll
                        for (int mi = 0; mi < C::MW; ++mi) fa[mi] = sA[(4 * k4 + t) * C::LDA + 8 * mi];
#pragma unroll
                        for (int nj = 0; nj < NT; ++nj) fb[nj] = sB[(4 * k4 + t) * C::LDB + 8 * nj];
#pragma unroll
                        for (int nj = 0; nj < NT; ++nj)
#pragma unroll
                            for (int mi = 0; mi < C::MW; ++mi) dmma(acc[mi][nj][0], acc[mi][nj][1], fa[mi], fb[nj]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[slot]);   // the warp's shared reads of this stage are done
                const bool seg_end = i + 1 == nq;
                const bool slab_end = cc.kin + 1 == a.VKB;
                const bool tile_end = slab_end && cc.slab + 1 == a.NS;
                if (seg_end || slab_end) {
                    // fold this slab's DMMA chains (<= 4096 products) into the tile's running sum in the
                    // segment's own partial slot (L2-resident; each thread touches only its own elements)
                    double* P = a.part + (seg * a.maxseg + (cc.tile - tile0)) * (C::BM * C::BN);
#pragma unroll
                    for (int mi = 0; mi < C::MW; ++mi)
#pragma unroll
                        for (int nj = 0; nj < NT; ++nj) {
                            const int m = 8 * C::MW * warp + 8 * mi + g, n = 8 * nj + 2 * t;
                            double* p0 = P + (int64_t)n * C::BM + m;
                            double* p1 = p0 + C::BM;
                            if (first_flush) {
                                *p0 = acc[mi][nj][0];
                                *p1 = acc[mi][nj][1];
                            } else {
                                *p0 += acc[mi][nj][0];
                                *p1 += acc[mi][nj][1];
                            }
                            acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
                        }
                    first_flush = tile_end;
                }
                cc.next(a);
            }
        }
        base += nq;
    }
}

// Z = sum of the partials of each tile, fixed order.  A block owns 32 consecutive elements (lane) of
// one tile; warp w adds the partials of the contributing CTAs c_lo + w, c_lo + w + 8, ... (CTA order =
// increasing k), and the 8 warp sums are added in warp order.
template <typename TZ>
__global__ void __launch_bounds__(256) gstage_reduce_kernel(GsArgs a, int BM, int BN, TZ* __restrict__ Z,
                                                            int64_t ldz) {
    __shared__ double red[8][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t per_tile = (int64_t)BM * BN;
    const int64_t blocks_per_tile = per_tile / 32;
    const int64_t tile = blockIdx.x / blocks_per_tile;
    const int r = (int)((blockIdx.x - tile * blocks_per_tile) * 32 + lane);
    const int64_t tq = a.NS * a.VKB;   // flattened k-blocks per tile
    const int c_lo = cta_of(tile * tq, a.total, a.P), c_hi = cta_of((tile + 1) * tq - 1, a.total, a.P);
    // slot of segment cc for this tile: cc * maxseg + (tile - first tile of cc).  The first tiles come
    // from one 64-bit division per segment, done once per block into shared memory (a division per
    // partial load made the reduce ALU-bound: 21 us at C4)
    constexpr int kMaxSeg = 1024;
    __shared__ int64_t s_slot[kMaxSeg];
    const int nseg = c_hi - c_lo + 1;
    const bool tab = nseg <= kMaxSeg;
    if (tab)
        for (int i = threadIdx.x; i < nseg; i += blockDim.x)
            s_slot[i] = (int64_t)(c_lo + i) * a.maxseg + (tile - range_begin(c_lo + i, a.total, a.P) / tq);
    __syncthreads();
    auto part_of = [&](int cc) {
        const int64_t slot = tab ? s_slot[cc - c_lo]
                                 : (int64_t)cc * a.maxseg + (tile - range_begin(cc, a.total, a.P) / tq);
        return a.part[slot * per_tile + r];
    };
    // segments c_lo + warp, + 8, + 16, ... added in that order; four loads issued before their adds
    // (a dependent load per add made the reduce latency-bound: 49 us at C3, ncu r02)
    double z = 0.0;
    int cc = c_lo + warp;
    for (; cc + 24 <= c_hi; cc += 32) {
        const double v0 = part_of(cc), v1 = part_of(cc + 8), v2 = part_of(cc + 16), v3 = part_of(cc + 24);
        z += v0;
        z += v1;
        z += v2;
        z += v3;
    }
    for (; cc <= c_hi; cc += 8) z += part_of(cc);
    red[warp][lane] = z;
    __syncthreads();
    if (warp == 0) {
        double zz = red[0][lane];
#pragma unroll
        for (int w = 1; w < 8; ++w) zz += red[w][lane];
        const int m_loc = r % BM, n_loc = r / BM;
        const int mt = (int)(tile % a.MT), ch = (int)(tile / a.MT);
        const int m = mt * BM + m_loc, c = ch * a.cw + n_loc;
        if (m < a.k2 && n_loc < a.cw && c < a.ncols) Z[m + (int64_t)c * ldz] = (TZ)zz;
    }
}

template <int NT>
csk_status launch(GsArgs& a, void* Z, int64_t ldz, bool z_f32, cudaStream_t st) {
    using C = Cfg<NT>;
    auto kern = gstage_kernel<NT>;
    CSK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    // two CTAs per SM need the largest shared-memory carveout (ncu r02: the driver's default fit one)
    CSK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    a.MT = (a.k2 + C::BM - 1) / C::BM;
    a.NCH = (a.ncols + a.cw - 1) / a.cw;
    a.KB = ceil_div(a.k1, kBK);
    a.VKB = std::min<int64_t>(kSlabK / kBK, a.KB);
    a.NS = ceil_div(a.KB, a.VKB);
    a.total = (int64_t)a.MT * a.NCH * a.NS * a.VKB;
    CSK_REQUIRE(a.total < (int64_t(1) << 47), CSK_EUNSUPPORTED, "G-stage: k1 too large");
    const int nsm = device_info().num_sms;
    // two CTAs per SM (fewer when there are < 8 k-blocks per CTA); P = 4, 2 or 1 segments per CTA, the
    // most that leaves >= 24 k-blocks per segment (each segment adds a pipeline fill and a partial tile
    // per tile it touches to the fixed-order reduce: C2 with 32-k-block segments on 32 CTAs took 48 us,
    // with 8-k-block segments on 128 CTAs 12 us; C3 takes 4 x 296)
    int64_t grid = std::min<int64_t>(2 * nsm, std::max<int64_t>(1, a.total / 8));
    int64_t P = grid;
    for (int k = 4; k >= 2; k /= 2)
        if (a.total / (k * grid) >= 24) {
            P = k * grid;
            break;
        }
    if (const char* e = std::getenv("CSK_GS_CTAS")) P = std::max<int64_t>(1, std::min<int64_t>(std::atoll(e), a.total));
    a.P = (int)P;
    grid = std::min<int64_t>(grid, P);
    a.maxseg = (int)(ceil_div(ceil_div(a.total, P), a.NS * a.VKB) + 1);   // tiles one segment can touch
    const size_t part_bytes = (size_t)P * a.maxseg * C::BM * C::BN * sizeof(double);
    double* part = nullptr;
    CSK_CUDA_TRY(csk_malloc_async(&part, part_bytes + 16, st));
    a.part = part;
    a.work = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(part) + part_bytes);
    CSK_CUDA_TRY(cudaMemsetAsync(a.work, 0, sizeof(unsigned long long), st));
    kern<<<(unsigned)grid, (kGsWarps + 1) * 32, C::SMEM, st>>>(a);
    count_launch();
    cudaError_t e1 = cudaGetLastError();
    const unsigned rgrid = (unsigned)((int64_t)a.MT * a.NCH * (C::BM * C::BN / 32));
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

}  // namespace

// Z (k2 x ncols, column-major, ldz; fp64 or fp32) = G (k2 x k1, ldg, kGstageTailPad doubles of tail
// padding) times the row-major workspace described by ro (ro.cw <= 72 columns per chunk).
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
    if (nt <= 1) return launch<1>(a, Z, ldz, z_f32, st);
    if (nt <= 2) return launch<2>(a, Z, ldz, z_f32, st);
    if (nt <= 4) return launch<4>(a, Z, ldz, z_f32, st);
    if (nt <= 7) return launch<7>(a, Z, ldz, z_f32, st);
    return launch<9>(a, Z, ldz, z_f32, st);
}

}  // namespace csk
