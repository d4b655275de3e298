// countsketch.cu -- cs_apply: SA = S [A b]  (the hot kernel).
//
// Eq 2: Y_{m,:} = sum_{j: r_j = m} sigma_j A_{j,:}; Alg 2
// scatters whole rows atomically.  A is column-major here (BASELINE.json; R7),
// so a row is ncols strided elements.  Variants:
//   L  cs_col_kernel    : each element -> one REDG.F64 into column-major SA (simplest)
//   T  cs_row_kernel    : a warp loads a 32-row x 32-col tile (coalesced column reads),
//                         transposes it through shared memory, and issues one coalesced
//                         256-B REDG per row into SA^T (row-major, k1 x ldt) -- Alg 2's
//                         "add rows atomically" with rows made contiguous on chip
//   B  cs_row_kernel<BULK> : as T, but each row is reduced by the TMA engine with
//                         cp.reduce.async.bulk .add.f64 (one 256-B bulk op per row)
//   S  cs_smem_kernel   : per-CTA shared-memory privatised buckets for a group of columns;
//                         each warp owns one column's k1 accumulators (no atomics on the
//                         shared path, duplicates inside a warp merged with __match_any_sync),
//                         one flush per CTA and column
//   G  cs_sorted_kernel : deterministic signed segmented gather-sum over the plan's stable
//                         counting sort (north_star form 1); bitwise reproducible
// All variants accumulate in fp64 (fp32 input is widened; R12).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "csk_internal.cuh"

namespace csk {

void prof_mark(cudaStream_t st, bool begin);

// Row-major SA^T workspace layout: element (m, c) lives at (c / cw) * cs + m * lc + (c % cw).
// Regular layout: one chunk of all columns (cw >= ncols), lc = ldt.  Chunk-major layout
// (large k1 * ncols, e.g. C3): each cw-column chunk is its own k1 x lc slice (cs = k1 * lc)
// and the kernels walk chunk by chunk, so only one slice has to stay L2-resident.
struct RowLayout {
    int cw = 1;
    int64_t lc = 0, cs = 0;
    bool chunk_major = false;
    bool tma = false;   // launch marked TMA-eligible by cs_apply_impl (variant X)
    // fp32 accumulation (fp32 input): ncopies row-block copies of a float SA^T (lc, cs in floats),
    // copy p takes rows [p * rows_per_copy, ...) so every bucket sum in a copy has a bounded depth
    int ncopies = 0;
    int64_t rows_per_copy = 0, copy_stride = 0;
    // CSK_PLAN_HASH: global row of local row 0 and the Philox key (codes recomputed in the kernel)
    int64_t g0 = 0;
    uint32_t hkey0 = 0, hkey1 = 0;
    // fp64 B32 with few buckets (k1 (n+1) small, e.g. n = 32 at k1 = 2n^2): CTA c reduces into copy
    // c % nspread of SA^T (stride spread_stride doubles), so the bulk reduce-adds of all SMs are not
    // funnelled into the few L2 lines of a small SA^T; the copies are summed afterwards in fixed order
    int nspread = 1;
    int64_t spread_stride = 0;
    int f32_spread = 1;   // fp32 copies: consecutive tiles interleaved over this many copies
    unsigned long long* work = nullptr;   // dynamic work counter of the B kernels (zeroed with the workspace)
    int grab = 8;                         // units per counter grab (4/8/16/32 measured: 8)
    int grab_tail = 1;                    // fp32 kernel: single-unit grabs in the last 2 * grab * warps units
    __host__ __device__ int64_t base(int ch, uint32_t bucket) const { return (int64_t)ch * cs + (int64_t)bucket * lc; }
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ void red_add_f64(double* p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T ldg_stream(const T* p) {
    return __ldcs(p);   // streaming: A is read exactly once
}

// Predicated streaming loads (branch-free; a lane with pred == false fetches nothing and
// returns 0).  The address must still be legal: callers clamp it.
__device__ __forceinline__ double ldcs_pred(const double* p, bool pred) {
    double v = 0.0;
    asm("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.global.cs.f64 %0, [%1]; }" : "+d"(v) : "l"(p), "r"((int)pred));
    return v;
}
__device__ __forceinline__ double ldcs_pred(const float* p, bool pred) {
    float v = 0.0f;
    asm("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.global.cs.f32 %0, [%1]; }" : "+f"(v) : "l"(p), "r"((int)pred));
    return (double)v;
}
__device__ __forceinline__ double2 ldcs2_pred(const double* p, bool pred) {
    double2 v = make_double2(0.0, 0.0);
    asm("{ .reg .pred q; setp.ne.b32 q, %3, 0; @q ld.global.cs.v2.f64 {%0, %1}, [%2]; }"
        : "+d"(v.x), "+d"(v.y)
        : "l"(p), "r"((int)pred));
    return v;
}

// ------------------------------------------------------------------ variant L
template <typename T>
__global__ void __launch_bounds__(256) cs_col_kernel(const uint32_t* __restrict__ code, int64_t rows, Cols<T> cols,
                                                     int ncols, double* __restrict__ out, int64_t ldo) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += stride) {
        const uint32_t cd = __ldg(code + i);
        double* dst = out + code_bucket(cd);
        for (int c = 0; c < ncols; ++c) {
            const double v = (double)ldg_stream(cols.col(c) + i);
            red_add_f64(dst + (int64_t)c * ldo, apply_sign(v, cd));
        }
    }
}

// ------------------------------------------------------------------ variant T
// A warp owns a 32-row x 32-column unit: lane r loads A[r, c0..c0+31] (32 coalesced
// 256-B column reads; rows and columns past the edge are clamped to legal addresses
// and zeroed with a select, so the unrolled body has no branches), writes the signed
// values into row r of a padded (odd-stride, conflict-free) smem tile, then for each
// row j the warp issues one coalesced red.global.add.f64 of 32 lanes into
// SA^T[h(j), c0:c0+32] -- Alg 2's "add rows atomically" with the row made contiguous on chip.
constexpr int kRowWarps = 8;
constexpr int kTileLd = 33;

template <typename T>
__global__ void __launch_bounds__(kRowWarps * 32) cs_row_kernel(const uint32_t* __restrict__ code, int64_t rows,
                                                                Cols<T> cols, int ncols, double* __restrict__ SAt,
                                                                int64_t ldt) {
    extern __shared__ double row_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* tile = row_smem + (size_t)warp * 32 * kTileLd;
    const int nchunks = (ncols + 31) >> 5;
    const int64_t ngroups = (rows + 31) >> 5;
    const int64_t nunits = ngroups * nchunks;
    const int64_t gwarp = blockIdx.x * (int64_t)kRowWarps + warp;
    const int64_t nwarps = (int64_t)gridDim.x * kRowWarps;
    for (int64_t u = gwarp; u < nunits; u += nwarps) {
        const int64_t g = u / nchunks;
        const int ch = (int)(u - g * nchunks);
        const int c0 = ch * 32;
        const int nc = min(32, ncols - c0);
        const int64_t r = g * 32 + lane;
        const bool valid = r < rows;
        const int64_t rc = valid ? r : rows - 1;
        const uint32_t cd = __ldg(code + rc);
        const long long smask = valid ? (long long)code_sign_mask64(cd) : 0ll;
        double v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (double)ldg_stream(cols.col(min(c0 + j, ncols - 1)) + rc);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const double x = (j < nc && valid) ? v[j] : 0.0;
            tile[lane * kTileLd + j] = __longlong_as_double(__double_as_longlong(x) ^ smask);
        }
        __syncwarp();
        const int nrows = (int)min((int64_t)32, rows - g * 32);
        double* dst = SAt + c0 + lane;
#pragma unroll 8
        for (int j = 0; j < 32; ++j) {
            const uint32_t b = code_bucket(__shfl_sync(0xffffffffu, cd, j));
            const double x = tile[j * kTileLd + lane];
            if (j < nrows && lane < nc) red_add_f64(dst + (int64_t)b * ldt, x);
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ variant X
// TMA-fed row scatter.  [A b] must be one 2-D tensor (uniform column stride).  A warp
// owns a ring of kTmaStages smem tiles; lane 0 issues one cp.async.bulk.tensor.2d per
// tile (RB rows x cw columns, RB*sizeof(T) = 128 B per column, 128B swizzle, rows past d
// zero-filled by the TMA unit) completing on a per-stage mbarrier.  For each row j the
// warp reads SA^T's row slice straight out of the swizzled tile (lane = column) and issues
// ceil(cw/32) coalesced red.global.add.f64 -- no register staging, no transpose, and
// ~7 warp instructions per 32 elements (the LDG variant T needed ~65).
constexpr int kTmaWarps = 8;
constexpr int kTmaStages = 3;
constexpr int kTmaMaxCols = 96;

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(dst)),
        "l"(map), "r"(x), "r"(y), "r"((uint32_t)__cvta_generic_to_shared(bar))
        : "memory");
}

template <typename T>
__device__ __forceinline__ double swz_load(const uint8_t* tile, int c, int j) {
    // 128B swizzle: the 16-B chunk index of each 128-B column row is XORed with (column & 7)
    constexpr int kPerChunk = 16 / sizeof(T);
    const int off = c * 128 + ((((j / kPerChunk) ^ (c & 7))) << 4) + (j % kPerChunk) * (int)sizeof(T);
    return (double)*reinterpret_cast<const T*>(tile + off);
}

__device__ __forceinline__ void unit_coords(int64_t u, int nchunks, int64_t ngroups, bool chunk_major, int64_t& g,
                                            int& ch) {
    if (chunk_major) {
        ch = (int)(u / ngroups);
        g = u - (int64_t)ch * ngroups;
    } else {
        g = u / nchunks;
        ch = (int)(u - g * nchunks);
    }
}

template <typename T>
__global__ void __launch_bounds__(kTmaWarps * 32, 1) cs_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                    const uint32_t* __restrict__ code, int64_t rows,
                                                                    int ncols, int stage_bytes,
                                                                    double* __restrict__ SAt, RowLayout L) {
    constexpr int RB = 128 / sizeof(T);   // rows per tile: 16 (fp64) / 32 (fp32)
    extern __shared__ uint8_t tma_smem_raw[];
    // 1024-B alignment for the 128B swizzle, by pointer arithmetic on the __shared__ array so
    // the compiler keeps the shared state space (LDS/STS, not generic LD/ST)
    uint8_t* smem = tma_smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(tma_smem_raw) & 1023u)) & 1023u);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // layout: [warps][stages] tiles | [warps][stages][RB] codes | [warps][stages] mbarriers
    uint8_t* ring = smem + (size_t)warp * kTmaStages * stage_bytes;
    uint32_t* codes_all = reinterpret_cast<uint32_t*>(smem + (size_t)kTmaWarps * kTmaStages * stage_bytes);
    uint32_t* codes = codes_all + warp * kTmaStages * RB;
    uint64_t* bars = reinterpret_cast<uint64_t*>(codes_all + kTmaWarps * kTmaStages * RB) + warp * kTmaStages;
    const int cw = L.cw;
    const int nchunks = (ncols + cw - 1) / cw;
    const int64_t ngroups = (rows + RB - 1) / RB;
    const int64_t nunits = ngroups * nchunks;
    const int64_t gwarp = blockIdx.x * (int64_t)kTmaWarps + warp;
    const int64_t nwarps = (int64_t)gridDim.x * kTmaWarps;
    const uint32_t tile_bytes = (uint32_t)cw * 128u;
    auto issue = [&](int64_t u, int s) {
        int64_t g;
        int ch;
        unit_coords(u, nchunks, ngroups, L.chunk_major, g, ch);
        mbar_expect_tx(&bars[s], tile_bytes + RB * 4);
        tma_load_2d(ring + s * stage_bytes, &tmap, (int)(g * RB), ch * cw, &bars[s]);
        bulk_load_1d(codes + s * RB, code + g * RB, RB * 4, &bars[s]);
    };
    if (lane == 0) {
        for (int s = 0; s < kTmaStages; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < kTmaStages; ++s)
            if (gwarp + s * nwarps < nunits) issue(gwarp + s * nwarps, s);
    }
    __syncwarp();
    for (int64_t k = 0;; ++k) {
        const int64_t u = gwarp + k * nwarps;
        if (u >= nunits) break;
        const int s = (int)(k % kTmaStages);
        int64_t g;
        int ch;
        unit_coords(u, nchunks, ngroups, L.chunk_major, g, ch);
        const int c0 = ch * cw;
        const int nc = min(cw, ncols - c0);
        const int nr = (int)min((int64_t)RB, rows - g * RB);
        mbar_wait(&bars[s], (uint32_t)((k / kTmaStages) & 1));
        const uint32_t cdl = codes[s * RB + (lane % RB)];
        const uint8_t* tile = ring + s * stage_bytes;
#pragma unroll 4
        for (int j = 0; j < RB; ++j) {
            const uint32_t cd = __shfl_sync(0xffffffffu, cdl, j);
            double* dst = SAt + L.base(ch, code_bucket(cd));
            const long long smask = (long long)code_sign_mask64(cd);
#pragma unroll
            for (int q = 0; q < kTmaMaxCols / 32; ++q) {
                const int c = q * 32 + lane;
                if (q * 32 < nc && c < nc && j < nr) {
                    const double x = swz_load<T>(tile, c, j);
                    red_add_f64(dst + c, __longlong_as_double(__double_as_longlong(x) ^ smask));
                }
            }
        }
        // this warp's generic reads of the stage precede the next async (TMA) write into it
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0 && u + kTmaStages * nwarps < nunits) issue(u + kTmaStages * nwarps, s);
    }
}

static int tma_chunk_width(int ncols) {
    if (ncols <= kTmaMaxCols) return ncols;
    const int nch = (ncols + 63) / 64;
    return (ncols + nch - 1) / nch;
}

// ------------------------------------------------------------------ variant B
// A warp owns 16-row x cw-column tiles (cw <= 66: all of [A b] at C2).  Lanes (r, half)
// load column pairs (two coalesced 128-B half-warp reads per instruction, streaming
// ld.global.cs), write the signed values row-major into a 16-B aligned smem row, and lane r
// hands the whole row to the TMA engine as ONE bulk reduce-add
// (cp.reduce.async.bulk ... .add.f64, cw*8 bytes) into SA^T[h(r), c0:c0+cw].
// BulkCfg<W, NB, PIPE>: W warps per CTA, NB smem tile buffers per warp (recycled with
// cp.async.bulk.wait_group.read NB-1), PIPE = register double-buffering of the loads (the
// next tile's loads are in flight while this tile is transposed and reduced).
constexpr int kBulkRows = 16;
constexpr int kBulkMaxCols = 66;

template <int W, int NB, bool PIPE>
struct BulkCfg {
    static constexpr int kWarps = W, kBufs = NB;
    static constexpr bool kPipe = PIPE;
};

__host__ __device__ inline int bulk_chunk_width(int ncols) {
    if (ncols <= kBulkMaxCols) return ncols;
    const int nch = (ncols + kBulkMaxCols - 1) / kBulkMaxCols;   // fewest chunks: each re-reads the codes
    return (((ncols + nch - 1) / nch) + 1) & ~1;   // even: every chunk start stays 16-B aligned
}

template <typename T>
__device__ __forceinline__ void bulk_load_tile(double (&v)[kBulkMaxCols / 2], const Cols<T>& cols, int ncols, int c0,
                                               int nc, int half, int64_t rc) {
#pragma unroll
    for (int j = 0; j < kBulkMaxCols / 2; ++j) {
        const int c = 2 * j + half;
        const double x = (double)ldg_stream(cols.col(c0 + min(c, nc - 1)) + rc);   // re-read the last column
        v[j] = (c < nc) ? x : 0.0;
    }
}

template <typename T, typename C, int EXP>
__global__ void __launch_bounds__(C::kWarps * 32, 1) cs_bulk_kernel(const uint32_t* __restrict__ code, int64_t rows,
                                                                     Cols<T> cols, int ncols, int ldtile,
                                                                     double* __restrict__ SAt, RowLayout L) {
    // EXP: compile-time experiment switches for roofline attribution (0 in production):
    // bit 0 = skip the bulk reduce, bit 1 = skip the A loads
    constexpr int NB = C::kBufs;
    const int cw = L.cw;
    extern __shared__ __align__(16) double bulk_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int half = lane >> 4, rr = lane & 15;
    double* tiles = bulk_smem + (size_t)warp * NB * kBulkRows * ldtile;
    for (int e = lane; e < NB * kBulkRows * ldtile; e += 32) tiles[e] = 0.0;
    __syncwarp();
    const int nchunks = (ncols + cw - 1) / cw;
    const int64_t ngroups = (rows + kBulkRows - 1) / kBulkRows;
    const int64_t nunits = ngroups * nchunks;
    const int64_t gwarp = blockIdx.x * (int64_t)C::kWarps + warp;
    const int64_t nwarps = (int64_t)gridDim.x * C::kWarps;
    auto coords = [&](int64_t u, int64_t& g, int& c0, int& nc, int64_t& rc, bool& valid) {
        int ch;
        unit_coords(u, nchunks, ngroups, L.chunk_major, g, ch);
        c0 = ch * cw;
        nc = min(cw, ncols - c0);
        const int64_t r = g * kBulkRows + rr;
        valid = r < rows;
        rc = valid ? r : rows - 1;
    };
    double v[kBulkMaxCols / 2];
    double vn[C::kPipe ? kBulkMaxCols / 2 : 1];
    int buf = 0;
    int64_t u = gwarp;
    if (C::kPipe && u < nunits) {
        int64_t g, rc;
        int c0, nc;
        bool valid;
        coords(u, g, c0, nc, rc, valid);
        if (EXP & 2) {
#pragma unroll
            for (int j = 0; j < kBulkMaxCols / 2; ++j) v[j] = (double)(rc + j);
        } else {
            bulk_load_tile(v, cols, ncols, c0, nc, half, rc);
        }
    }
    for (; u < nunits; u += nwarps) {
        int64_t g, rc;
        int c0, nc;
        bool valid;
        coords(u, g, c0, nc, rc, valid);
        const uint32_t cd = __ldg(code + rc);
        if constexpr (C::kPipe) {
            // next tile's loads go out before this tile is transposed and reduced
            const int64_t un = u + nwarps;
            if (un < nunits) {
                int64_t gn, rcn;
                int c0n, ncn;
                bool validn;
                coords(un, gn, c0n, ncn, rcn, validn);
                if (EXP & 2) {
#pragma unroll
                    for (int j = 0; j < kBulkMaxCols / 2; ++j) vn[j] = (double)(rcn + j);
                } else {
                    bulk_load_tile(vn, cols, ncols, c0n, ncn, half, rcn);
                }
            }
        } else {
            if (EXP & 2) {
#pragma unroll
                for (int j = 0; j < kBulkMaxCols / 2; ++j) v[j] = (double)(rc + j);
            } else {
                bulk_load_tile(v, cols, ncols, c0, nc, half, rc);
            }
        }
        double* tile = tiles + buf * kBulkRows * ldtile;
        // the TMA engine must be done reading this buffer (its bulk ops were committed NB units ago)
        if constexpr (NB == 1)
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        else
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kBulkMaxCols / 2; ++j) {
            const int c = 2 * j + half;
            if (c < nc) tile[rr * ldtile + c] = apply_sign(v[j], cd);
        }
        if ((nc & 1) && half == 0) tile[rr * ldtile + nc] = 0.0;   // 16-B padding column
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (half == 0 && valid && !(EXP & 1)) {
            const uint32_t bytes = (uint32_t)(((nc + 1) & ~1) * 8);
            double* dst = SAt + L.base((int)(c0 / cw), code_bucket(cd));
            const uint32_t src = (uint32_t)__cvta_generic_to_shared(tile + rr * ldtile);
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(dst),
                         "r"(src), "r"(bytes)
                         : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if constexpr (C::kPipe) {
#pragma unroll
            for (int j = 0; j < kBulkMaxCols / 2; ++j) v[j] = vn[j];
        }
        buf = (buf + 1) % NB;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------ variant B, 32-row tiles
// Same dataflow as cs_bulk_kernel with 32-row tiles and 16-byte loads: lane (p, half) loads
// rows (2p, 2p+1) of column 2j+half as one double2, so every column segment is 256 B
// contiguous (measured: 32-row tiles stream at 6.4 TB/s where 16-row tiles reach 4.8 TB/s
// at the same occupancy, scripts/tile_read_bench.cu).  One tile buffer per warp; lane r
// bulk-reduces row r.  fp64, 16-B aligned columns (lda even); the ragged last tile falls
// back to clamped scalar loads.
constexpr int kB32Rows = 32;
constexpr int64_t kSpreadBytes = 256ll << 10;   // spread-copy footprint target (measured)
// row r of a warp's tile: 8-row group g = r >> 3 is shifted by 2g doubles (rows never overlap, 16-B aligned)
__device__ __forceinline__ int b32_row(int r, int ld) { return r * ld + 2 * (r >> 3); }
constexpr int kB32Pad = 6;   // doubles per warp tile beyond 32 rows (the shift of the last group)

// KJ = column pairs a lane holds (2 KJ >= the chunk's columns + pad).  Narrow [A b] (n <= 32) take a
// narrow instantiation: its smaller register file lets 2 (KJ = 17) or 3 (KJ = 9) CTAs share an SM, so
// 2-3x the tiles are in flight -- with one 32-row tile per warp, the narrow shapes were bound by the
// per-tile latency (load, store, bulk issue: ~2.5 us per tile at n = 8 ... 32, the same time for any width).
template <int KJ>
constexpr int b32_ctas_per_sm() { return KJ <= 9 ? 3 : KJ <= 17 ? 2 : 1; }
// register width of the B32 instantiation for a chunk of cw columns (CSK_B32_NARROW=0 disables the
// narrow ones, for A/B measurements)
static int b32_kj(int cw) {
    const char* e = std::getenv("CSK_B32_NARROW");
    const bool off = e && std::atoi(e) == 0;
    const int slots = (cw + 1) & ~1;   // columns + the 16-B pad
    return off ? kBulkMaxCols / 2 : slots <= 18 ? 9 : slots <= 34 ? 17 : kBulkMaxCols / 2;
}
template <int W, int EXP = 0, bool PRED = false, bool HASH = false, int KJ = kBulkMaxCols / 2>
__global__ void __launch_bounds__(W * 32, b32_ctas_per_sm<KJ>()) cs_bulk32_kernel(const uint32_t* __restrict__ code, int64_t rows,
                                                               Cols<double> cols, int ncols, int ldtile,
                                                               double* __restrict__ SAt, RowLayout L, int k1) {
    // EXP: compile-time experiment switches for roofline attribution (0 in production):
    // bit 0 = skip the bulk reduce (load path alone), bit 1 = skip the A loads (reduce path alone)
    const int cw = L.cw;
    extern __shared__ __align__(16) double b32_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // lane = 2p + half: each 16-lane phase of an 8-B STS covers 8 row pairs x both column parities,
    // so with the row shift below its 16 lanes hit 16 distinct double-banks (one wavefront per phase);
    // the loads cover the same 256-B column segments as any other lane order
    const int p = lane >> 1, half = lane & 1;
    // 8-row groups are shifted by 2 doubles each (b32_row): with ld == 2 mod 4 the row pairs of one
    // STS otherwise land on 4 of 8 even double-banks (ncu: 75% of the shared wavefronts were
    // conflicts)
    double* tile = b32_smem + (size_t)warp * (kB32Rows * ldtile + kB32Pad);
    for (int e = lane; e < kB32Rows * ldtile + kB32Pad; e += 32) tile[e] = 0.0;
    __syncwarp();
    const int nchunks = (ncols + cw - 1) / cw;
    const int64_t ngroups = (rows + kB32Rows - 1) / kB32Rows;
    const int64_t nunits = ngroups * nchunks;
    constexpr int kJ = KJ;
    // Work distribution: with L.work (a zeroed counter after the workspace) warps take batches of
    // kGrab consecutive units from one atomic counter, so CTAs that start late (SMs still held by an
    // overlapping kernel, e.g. the previous batch's solve) just take fewer units; else static
    // round-robin.  Units are taken in increasing order either way (chunk-major slices stay hot).
    const int kGrab = L.grab;
    int64_t u, uend;
    {
        unsigned long long ub = 0;
        if (lane == 0) ub = atomicAdd(L.work, (unsigned long long)kGrab);
        ub = __shfl_sync(0xffffffffu, ub, 0);
        u = (int64_t)ub;
        uend = min(u + kGrab, nunits);
    }
    // Look-ahead order: tile i is stored into the warp's shared tile, then tile i+1's loads are
    // issued, and only then are tile i's 32 bulk reduce-adds issued -- the per-row issue loop (one
    // uniform-datapath UBLKRED per lane, ~20-30 cycles each, ncu r02) runs while the next tile's
    // loads are in flight instead of in front of them.  Registers hold one tile either way.
    int ch = 0, nc = 0;
    int64_t r0 = 0;
    uint32_t ca = 0, cb = 0, crow = 0;
    double2 v[kJ];
    auto fetch = [&]() {   // coordinates, codes and loads of unit u
        int64_t g;
        unit_coords(u, nchunks, ngroups, L.chunk_major, g, ch);
        const int c0 = ch * cw;
        nc = min(cw, ncols - c0);
        r0 = g * kB32Rows;
        const bool full = r0 + kB32Rows <= rows;
        const int64_t ra = min(r0 + 2 * p, rows - 1), rb = min(r0 + 2 * p + 1, rows - 1);
        if constexpr (HASH) {
            // CSK_PLAN_HASH (hash-based generation on the fly): lane r hashes row r0 + r
            // (one Philox4x32-10 block, the word of its row) and the pair rows come by shuffle --
            // no code array is read; the same function codes_kernel stores (R3)
            const uint64_t gr = (uint64_t)(L.g0 + min(r0 + lane, rows - 1));
            const uint4 x = hash_block(gr, L.hkey0, L.hkey1);
            const uint32_t jw = (uint32_t)gr & 3u;
            const uint32_t w = jw == 0 ? x.x : jw == 1 ? x.y : jw == 2 ? x.z : x.w;
            crow = code_from_word(w, (uint32_t)k1);
            ca = __shfl_sync(0xffffffffu, crow, 2 * p);
            cb = __shfl_sync(0xffffffffu, crow, 2 * p + 1);
        } else {
            ca = __ldg(code + ra);
            cb = __ldg(code + rb);
            crow = __ldg(code + min(r0 + lane, rows - 1));
        }
        if (full && !PRED) {
            // (nearly) full-width chunk (C2, C4): lanes past the chunk's last column re-read that
            // column (an L1 hit, no DRAM bytes) and drop the value.  Plain loads schedule better
            // than predicated inline PTX (1.5% at C2, same-box A/B).
#pragma unroll
            for (int j = 0; j < kJ; ++j) {
                const int c = 2 * j + half;
                const double2 x = (EXP & 2) ? make_double2((double)ra, (double)c)
                                            : __ldcs(reinterpret_cast<const double2*>(
                                                  cols.col(c0 + min(c, nc - 1)) + r0 + 2 * p));
                v[j] = (c < nc) ? x : make_double2(0.0, 0.0);
            }
        } else if (full) {
            // PRED (narrow chunks, C3: 52 of 66 slots): predicated loads -- the idle lanes issue
            // nothing (re-reading would add 27% load instructions; measured 2.22 vs 2.11 ms at C3).
            // A separate instantiation: one kernel holding both paths ran C2 1.5% slower.
#pragma unroll
            for (int j = 0; j < kJ; ++j) {
                const int c = 2 * j + half;
                v[j] = (EXP & 2) ? make_double2((double)ra, (double)c)
                                 : ldcs2_pred(cols.col(c0 + min(c, nc - 1)) + r0 + 2 * p, c < nc);
            }
        } else {
#pragma unroll
            for (int j = 0; j < kJ; ++j) {
                const int c = 2 * j + half;
                const double* col = cols.col(c0 + min(c, nc - 1));
                const double xa = __ldcs(col + ra), xb = __ldcs(col + rb);
                v[j] = (c < nc) ? make_double2(xa, r0 + 2 * p + 1 < rows ? xb : 0.0) : make_double2(0.0, 0.0);
            }
        }
    };
    auto advance = [&]() {
        if (++u >= uend) {
            unsigned long long ub = 0;
            if (lane == 0) ub = atomicAdd(L.work, (unsigned long long)kGrab);
            ub = __shfl_sync(0xffffffffu, ub, 0);
            u = (int64_t)ub;
            uend = min(u + kGrab, nunits);
        }
    };
    if (u < nunits) fetch();
    while (u < nunits) {
        // the TMA engine must have finished reading the tile (bulk ops of the previous unit)
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        double* ta = tile + b32_row(2 * p, ldtile);
        double* tb = tile + b32_row(2 * p + 1, ldtile);
        const long long sa = (long long)code_sign_mask64(ca), sb = (long long)code_sign_mask64(cb);
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            const int c = 2 * j + half;
            if (c < nc) {
                ta[c] = __longlong_as_double(__double_as_longlong(v[j].x) ^ sa);
                tb[c] = __longlong_as_double(__double_as_longlong(v[j].y) ^ sb);
            }
        }
        if ((nc & 1) && half == 0) {   // 16-B padding column
            ta[nc] = 0.0;
            tb[nc] = 0.0;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        // this tile's bulk reduce-adds: lane r reduces row r (its bucket's SA^T row, spread copy of the CTA)
        const bool bvalid = r0 + lane < rows && !(EXP & 1);
        const uint32_t bytes = (uint32_t)(((nc + 1) & ~1) * 8);
        double* dst = SAt + L.base(ch, code_bucket(crow)) + (int64_t)(blockIdx.x % L.nspread) * L.spread_stride;
        const uint32_t src = (uint32_t)__cvta_generic_to_shared(tile + b32_row(lane, ldtile));
        auto issue = [&]() {
            if (bvalid) {
                if constexpr (PRED) {
                    // narrow chunks (C3): the chunk's SA^T slice (54 MB) competes with the streamed A for
                    // L2; mark the reductions evict_last so the slice is not written back mid-pass
                    uint64_t pol;
                    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
                    asm volatile(
                        "cp.reduce.async.bulk.global.shared::cta.bulk_group.L2::cache_hint.add.f64 [%0], [%1], %2, %3;" ::"l"(
                            dst),
                        "r"(src), "r"(bytes), "l"(pol)
                        : "memory");
                } else {
                    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(dst),
                                 "r"(src), "r"(bytes)
                                 : "memory");
                }
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        };
        advance();
        if (u < nunits) fetch();   // next tile's loads in flight ...
        issue();                   // ... while this tile's reduce-adds are issued
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------ fp32 input, fp32 accumulation (variant B, default fp32)
// The fp64 row scatter is bound by the L2's fp64 reduction rate (~147 G sector-RMW/s,
// 17 sectors per 65-double row).  fp32 rows are 9 sectors and the L2 reduces them faster per sector
// (microbenchmark: 2^24 rows of 272 B in 0.82 ms vs 528-B fp64 rows in 1.93 ms), so fp32 input is
// summed in fp32 -- but a sequential fp32 sum over a whole bucket (2048 rows at C2) could reach
// ~1.2e-4 sum|terms|, above BASELINE's 1e-5.  The rows are therefore split into ncopies blocks, each
// reduced into its own float SA^T copy with a mean bucket depth <= 64 (an fp32 sum of m terms in any
// order errs by <= (m - 1) u32 sum|terms|, 3.8e-6 at m = 64), and the copies are added in fp64 by
// cs_combine_*_kernel (fixed order).
// Tile: 64 rows x cw (<= 66) columns per warp.  Lane (q, s) = (lane >> 2, lane & 3) loads rows
// 8q .. 8q+7 of column 4j + s with one 32-byte load (256 contiguous bytes per column per instruction),
// flips the signs (XOR) and stores row 8q+i of the row-major float tile at
// (8q+i) ldf + 4q + c: with ldf == 4 (mod 32) the 32 lanes of each store hit 32 distinct banks (rows stay
// 16-B aligned for the bulk copies).  Lane r then bulk-reduces rows r and r + 32 (.add.f32).
constexpr int kF32Rows = 64;
constexpr int kF32MaxCols = 68;   // 17 column quads

// predicated 32-B streaming load (branch-free: a lane with pred == false fetches nothing and gets 0;
// the address must still be legal)
__device__ __forceinline__ void ldcs_v8_pred(const float* p, bool pred, float (&v)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = 0.0f;
    asm("{ .reg .pred q; setp.ne.b32 q, %9, 0;\n\t"
        "@q ld.global.cs.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8]; }"
        : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]), "+f"(v[7])
        : "l"(p), "r"((int)pred));
}

// KJF = column quads a lane holds (4 KJF >= the chunk's columns + pad): the narrow instantiations
// (KJF = 5 / 9, n <= 16 / 32) run 3 / 2 CTAs per SM, as the fp64 B32 kernel does.
template <int KJF>
constexpr int f32_ctas_per_sm() { return KJF <= 5 ? 3 : KJF <= 9 ? 2 : 1; }
static int f32_kj(int cw) {
    const char* e = std::getenv("CSK_B32_NARROW");
    const bool off = e && std::atoi(e) == 0;
    const int slots = (cw + 3) & ~3;
    return off ? kF32MaxCols / 4 : slots <= 20 ? 5 : slots <= 36 ? 9 : kF32MaxCols / 4;
}
template <int W, int KJF = kF32MaxCols / 4>
__global__ void __launch_bounds__(W * 32, f32_ctas_per_sm<KJF>()) cs_bulk64f_kernel(const uint32_t* __restrict__ code, int64_t rows,
                                                                Cols<float> cols, int ncols, int ldf,
                                                                float* __restrict__ SAt, RowLayout L) {
    const int cw = L.cw;
    extern __shared__ __align__(16) float f32_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = lane >> 2, sq = lane & 3;
    // one tile buffer per warp (two buffers with 6 warps measured 30% slower: fewer loads in flight)
    float* tile = f32_smem + (size_t)warp * (kF32Rows * ldf + 32);
    for (int e = lane; e < kF32Rows * ldf + 32; e += 32) tile[e] = 0.0f;
    __syncwarp();
    const int nchunks = (ncols + cw - 1) / cw;
    const int64_t ngroups = (rows + kF32Rows - 1) / kF32Rows;
    const int64_t nunits = ngroups * nchunks;
    constexpr int kJ = KJF;
    const int kGrab = L.grab;
    const int64_t tailz = L.grab_tail ? 2 * (int64_t)kGrab * gridDim.x * W : 0;
    int64_t u, uend;
    {
        unsigned long long ub = 0;
        if (lane == 0) ub = atomicAdd(L.work, (unsigned long long)kGrab);
        ub = __shfl_sync(0xffffffffu, ub, 0);
        u = (int64_t)ub;
        uend = min(u + kGrab, nunits);
    }
    // look-ahead issue order as in cs_bulk32_kernel: store tile i, issue tile i+1's loads, then tile i's
    // 64 bulk reduce-adds (ncu r02: the per-row issue loop otherwise ran with no loads in flight)
    int ch = 0, nc = 0;
    int64_t r0 = 0;
    uint32_t ca = 0, cb = 0;
    float v[kJ][8];
    auto fetch = [&]() {
        int64_t g;
        unit_coords(u, nchunks, ngroups, L.chunk_major, g, ch);
        const int c0 = ch * cw;
        nc = min(cw, ncols - c0);
        r0 = g * kF32Rows;
        const bool full = r0 + kF32Rows <= rows;
        ca = __ldg(code + min(r0 + lane, rows - 1));
        cb = __ldg(code + min(r0 + 32 + lane, rows - 1));
        if (full) {   // one predicated 32-B load per column quad, no branches
#pragma unroll
            for (int j = 0; j < kJ; ++j) {
                const int c = 4 * j + sq;
                ldcs_v8_pred(cols.col(c0 + min(c, nc - 1)) + r0 + 8 * q, c < nc, v[j]);
            }
        } else {      // the ragged last tile: clamped scalar loads
#pragma unroll
            for (int j = 0; j < kJ; ++j) {
                const int c = 4 * j + sq;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const bool ok = c < nc && r0 + 8 * q + i < rows;
                    v[j][i] = ok ? __ldcs(cols.col(c0 + min(c, nc - 1)) + min(r0 + 8 * q + i, rows - 1)) : 0.0f;
                }
            }
        }
    };
    if (u < nunits) fetch();
    while (u < nunits) {
        // sign bits of the 64 rows (bit r = row r negative), one ballot per half
        const uint32_t sg_lo = __ballot_sync(0xffffffffu, (ca >> 31) != 0u);
        const uint32_t sg_hi = __ballot_sync(0xffffffffu, (cb >> 31) != 0u);
        const uint32_t sgw = q < 4 ? sg_lo : sg_hi;
        const int sh = (q & 3) * 8;
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        const int nc4 = (nc + 3) & ~3;
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            const int c = 4 * j + sq;
            if (c < nc4) {   // columns nc .. nc4 - 1 carry the zeros of the 16-B row padding
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint32_t neg = ((sgw >> (sh + i)) & 1u) << 31;
                    tile[(8 * q + i) * ldf + 4 * q + c] = __uint_as_float(__float_as_uint(v[j][i]) ^ neg);
                }
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        // this tile's reduce-adds: lane r reduces rows r and r + 32 into their row-block copies
        const uint32_t bytes = (uint32_t)(nc4 * 4);
        float* dst[2];
        bool ok[2];
        // row-block copy of the tile (rows_per_copy is a multiple of the 64-row tile): one 32-bit
        // division per tile instead of two 64-bit divisions per lane
        // interleaved in groups of S = L.f32_spread copies: tile g of a block of S * TPC tiles goes to copy
        // (block) S + g % S, so the tiles in flight at one time (consecutive g) spread over S copies
        // while each copy still takes TPC tiles (the depth bound is unchanged)
        const uint32_t gt = (uint32_t)(r0 / kF32Rows), tpc = (uint32_t)(L.rows_per_copy / kF32Rows);
        const uint32_t S = (uint32_t)L.f32_spread;
        const int64_t copy = (int64_t)((gt / (S * tpc)) * S + gt % S);
        float* cbase = SAt + copy * L.copy_stride + (int64_t)ch * L.cs;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = lane + 32 * h;
            ok[h] = r0 + r < rows;
            dst[h] = cbase + (int64_t)code_bucket(h ? cb : ca) * L.lc;
        }
        if (++u >= uend) {
            // near the end of the range a grab of kGrab 64-row units is ~kGrab tiles of one warp's time:
            // the last 2 * kGrab * (warps in the grid) units go out one at a time so the warps finish
            // together (u is this warp's previous range end, within one round of the counter).  Measured
            // (profiles/r02_grab_tail_ab.txt): fp32 C2 1.020 -> 1.008 ms; on the fp64 B32 kernel it
            // gained nothing (C2, C4, C3) or lost (n = 32: +1.8%), so only the fp32 kernel uses it
            const int g = nunits - u <= tailz ? 1 : kGrab;
            unsigned long long ub = 0;
            if (lane == 0) ub = atomicAdd(L.work, (unsigned long long)g);
            ub = __shfl_sync(0xffffffffu, ub, 0);
            u = (int64_t)ub;
            uend = min(u + g, nunits);
        }
        if (u < nunits) fetch();   // next tile's loads in flight while this tile is reduced
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t src = (uint32_t)__cvta_generic_to_shared(tile + (lane + 32 * h) * ldf + 4 * ((lane + 32 * h) >> 3));
            if (ok[h])
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst[h]),
                             "r"(src), "r"(bytes)
                             : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// the fp32 copies summed in fp64 (fixed order over the copies) into the fp64 row-major workspace of
// ms_apply (RowOut: regular layout, lc = lcd doubles)
__global__ void cs_combine_rows_kernel(const float* __restrict__ SAt, RowLayout L, int64_t k1, int ncols,
                                       double* __restrict__ Yt, int64_t lcd) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= k1 * lcd) return;
    const int64_t m = e / lcd;
    const int c = (int)(e - m * lcd);
    double acc = 0.0;
    if (c < ncols) {
        const int64_t off = (int64_t)(c / L.cw) * L.cs + m * L.lc + (c % L.cw);
        #pragma unroll 8   // the loads of 8 copies in flight; the adds stay in copy order
        for (int p = 0; p < L.ncopies; ++p) acc += (double)SAt[p * L.copy_stride + off];
    }
    Yt[e] = acc;
}

// many copies (small k1: rows / (64 k1) copies, e.g. 1024 at d = 2^23, k1 = 128): one warp per element,
// lane l sums copies l, l + 32, ... in fp64, then a fixed butterfly -- deterministic, and 32x shorter
// than the one-thread chain of the kernels above (which made the combine, not the sketch, the cost
// of the narrow fp32 shapes).  ROWOUT: fp64 row-major workspace (ms_apply), else column-major float SA.
template <bool ROWOUT>
__global__ void __launch_bounds__(256) cs_combine_warp_kernel(const float* __restrict__ SAt, RowLayout L, int64_t k1,
                                                              int ncols, int64_t lcd, double* __restrict__ Yt,
                                                              float* __restrict__ SA, int64_t ldsa) {
    const int lane = threadIdx.x & 31;
    const int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t ne = k1 * (ROWOUT ? lcd : (int64_t)ncols);
    if (e >= ne) return;
    int64_t m;
    int c;
    if (ROWOUT) {
        m = e / lcd;
        c = (int)(e - m * lcd);
    } else {   // column-major order: consecutive warps write consecutive rows of one column
        c = (int)(e / k1);
        m = e - (int64_t)c * k1;
    }
    double acc = 0.0;
    if (c < ncols) {
        const int64_t off = (int64_t)(c / L.cw) * L.cs + m * L.lc + (c % L.cw);
        #pragma unroll 8   // the loads of 8 copies in flight; the adds stay in copy order
        for (int p = lane; p < L.ncopies; p += 32) acc += (double)SAt[p * L.copy_stride + off];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
        if (ROWOUT)
            Yt[e] = acc;
        else
            SA[m + (int64_t)c * ldsa] = (float)acc;
    }
}
constexpr int kCombineWarpCopies = 64;   // ncopies from which the warp-per-element combine is used

// spread copies (fp64 B32): copy 0 <- sum_p copy_p, elementwise, fixed order p = 0, 1, ...
__global__ void cs_spread_combine_kernel(double* __restrict__ SAt, int64_t n, int nspread, int64_t stride) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        double acc = SAt[e];
        #pragma unroll 8   // the loads of 8 copies in flight; the adds stay in copy order
        for (int p = 1; p < nspread; ++p) acc += SAt[p * stride + e];
        SAt[e] = acc;
    }
}

// SA[m, c] = (float) sum_p (double) copy_p[m, c]  (fixed order over p)
__global__ void cs_combine_f32_kernel(const float* __restrict__ SAt, RowLayout L, int64_t k1, int ncols,
                                      float* __restrict__ SA, int64_t ldsa) {
    __shared__ float t[32][33];
    const int64_t m0 = blockIdx.x * 32;
    const int c0 = blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int64_t m = m0 + j;
        const int c = c0 + threadIdx.x;
        double acc = 0.0;
        if (m < k1 && c < ncols) {
            const int64_t off = (int64_t)(c / L.cw) * L.cs + m * L.lc + (c % L.cw);
            #pragma unroll 8   // the loads of 8 copies in flight; the adds stay in copy order
            for (int q = 0; q < L.ncopies; ++q) acc += (double)SAt[q * L.copy_stride + off];
        }
        t[j][threadIdx.x] = (float)acc;
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int c = c0 + j;
        const int64_t m = m0 + threadIdx.x;
        if (m < k1 && c < ncols) SA[m + (int64_t)c * ldsa] = t[threadIdx.x][j];
    }
}

// SA^T (row-major workspace, fp64) -> SA (column-major, ldsa, T)
template <typename T>
__global__ void transpose_out_kernel(const double* __restrict__ SAt, RowLayout L, int64_t k1, int ncols,
                                     T* __restrict__ SA, int64_t ldsa) {
    __shared__ double t[32][33];
    const int64_t m0 = blockIdx.x * 32;
    const int c0 = blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int64_t m = m0 + j;
        const int c = c0 + threadIdx.x;
        t[j][threadIdx.x] = (m < k1 && c < ncols) ? SAt[(int64_t)(c / L.cw) * L.cs + m * L.lc + (c % L.cw)] : 0.0;
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int c = c0 + j;
        const int64_t m = m0 + threadIdx.x;
        if (m < k1 && c < ncols) SA[m + (int64_t)c * ldsa] = (T)t[threadIdx.x][j];
    }
}

// fp64 column-major workspace -> fp32 SA
__global__ void narrow_kernel(const double* __restrict__ src, int64_t k1, int ncols, float* __restrict__ SA,
                              int64_t ldsa) {
    const int64_t total = k1 * ncols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / k1, m = e - c * k1;
        SA[m + c * ldsa] = (float)src[e];
    }
}

// ------------------------------------------------------------------ variant S
// Shared-memory privatised buckets.  Warp w of a CTA owns the k1 fp64 accumulators of
// one column for a contiguous range of rows: every update is a plain LDS/DADD/STS
// (sm_100a has no native shared fp64 atomic; ptxas emits a CAS loop), duplicates among
// the 32 rows of one iteration are merged in lane order with __match_any_sync, and the
// warp-uniform common case (no duplicate, >94% at k1 = 8192) skips the merge.  The
// arrays are warp-private, so the kernel has no block barrier at all.  Loads are
// prefetched kPrivDepth iterations ahead in registers (kPrivDepth * 384 B in flight per
// warp).  The (column, row) work space is split evenly over CTAs; each warp flushes its
// array with REDG once per column it touched.
constexpr int kPrivDepth = 24;

template <typename T>
__global__ void __launch_bounds__(128, 1) cs_smem_kernel(const uint32_t* __restrict__ code, int64_t rows,
                                                         Cols<T> cols, int ncols, int cpc, int k1,
                                                         double* __restrict__ out, int64_t ldo,
                                                         int64_t work_per_cta) {
    extern __shared__ double acc_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ngroups = (ncols + cpc - 1) / cpc;
    const int64_t total = (int64_t)ngroups * rows;
    int64_t w = blockIdx.x * work_per_cta;
    const int64_t w_end = min(total, w + work_per_cta);
    double* acc = acc_smem + (size_t)warp * k1;
    while (w < w_end) {
        const int g = (int)(w / rows);
        const int64_t r0 = w - (int64_t)g * rows;
        const int64_t r1 = min(rows, r0 + (w_end - w));
        w += r1 - r0;
        const int c = g * cpc + warp;
        if (c >= ncols) continue;
        for (int i = lane; i < k1; i += 32) acc[i] = 0.0;
        __syncwarp();
        const T* col = cols.col(c);
        double pv[kPrivDepth];
        uint32_t pc[kPrivDepth];
#pragma unroll
        for (int p = 0; p < kPrivDepth; ++p) {
            const int64_t r = min(r0 + p * 32 + lane, r1 - 1);   // clamped: masked by `valid` at use
            pv[p] = (double)ldg_stream(col + r);
            pc[p] = __ldg(code + r);
        }
        for (int64_t base = r0; base < r1; base += 32 * kPrivDepth) {
#pragma unroll
            for (int p = 0; p < kPrivDepth; ++p) {
                const int64_t r = base + p * 32 + lane;
                const bool valid = r < r1;
                const uint32_t cd = pc[p];
                const double val = valid ? apply_sign(pv[p], cd) : 0.0;
                const int64_t rn = min(r + 32 * kPrivDepth, r1 - 1);
                pv[p] = (double)ldg_stream(col + rn);
                pc[p] = __ldg(code + rn);
                const uint32_t key = valid ? code_bucket(cd) : 0x80000000u | lane;
                const uint32_t peers = __match_any_sync(0xffffffffu, key);
                if (__all_sync(0xffffffffu, peers == (1u << lane))) {
                    if (valid) acc[key] += val;
                } else {
                    // lanes sharing a bucket: the lowest lane adds their sum (lane order)
                    double sum = 0.0;
                    for (uint32_t m = peers; m; m &= m - 1) sum += __shfl_sync(peers, val, __ffs(m) - 1);
                    if (valid && lane == __ffs(peers) - 1) acc[key] += sum;
                }
                __syncwarp();
            }
        }
        // flush this column's partial sums (REDG; exact zeros skipped)
        for (int i = lane; i < k1; i += 32) {
            const double v = acc[i];
            if (v != 0.0) red_add_f64(out + i + (int64_t)c * ldo, v);
        }
        __syncwarp();
    }
}


// ------------------------------------------------------------------ variant G
// Warp per (bucket m, column c): SA[m,c] = sum over the bucket's segment of the
// sorted rows, lanes striding the segment, fixed-order shuffle tree at the end.
// Bitwise deterministic (no atomics, fixed order).
template <typename T>
__global__ void __launch_bounds__(256) cs_sorted_kernel(const uint32_t* __restrict__ code,
                                                        const int32_t* __restrict__ perm,
                                                        const int64_t* __restrict__ offsets, int64_t k1,
                                                        Cols<T> cols, int ncols, double* __restrict__ out,
                                                        int64_t ldo) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t m = gw; m < k1; m += nw) {
        const int64_t s0 = offsets[m], s1 = offsets[m + 1];
        for (int c = 0; c < ncols; ++c) {
            const T* col = cols.col(c);
            double sum = 0.0;
            for (int64_t p = s0 + lane; p < s1; p += 32) {
                const int32_t i = __ldg(perm + p);
                sum += apply_sign((double)__ldg(col + i), __ldg(code + i));
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            if (lane == 0) out[m + (int64_t)c * ldo] = sum;
        }
    }
}

// ------------------------------------------------------------------ dispatch
// Accumulation target of a variant: row-major SA^T workspace (T, B), or a
// column-major fp64 buffer (L, S, G) which is SA itself for fp64 output.
static bool variant_rowmajor(int v) {
    return v == CSK_VAR_ATOMIC_ROW || v == CSK_VAR_BULK_ROW || v == CSK_VAR_TMA_ROW;
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
        cudaGetLastError();
    });
    return fn;
}

// [A b] as one 2-D tensor for TMA: needs b == NULL or b == A + n*lda, 16-B aligned base and stride
template <typename T>
static bool tma_eligible(const Cols<T>& cols, int ncols) {
    const T* base = cols.n > 0 ? cols.A : cols.b;
    if (cols.n > 0 && cols.b != nullptr && cols.b != cols.A + (int64_t)cols.n * cols.lda) return false;
    if (((uintptr_t)base & 15) != 0) return false;
    if (ncols > 1 && ((cols.lda * (int64_t)sizeof(T)) & 15) != 0) return false;
    return tensor_map_encoder() != nullptr;
}

static int env_variant() {
    const char* e = std::getenv("CSK_VARIANT");
    if (!e || !*e) return CSK_VAR_AUTO;
    return std::atoi(e);
}

static int smem_cpc(int64_t k1, int ncols) {
    const DeviceInfo& di = device_info();
    const int64_t per_col = k1 * 8;
    int cpc = (int)std::min<int64_t>((int64_t)di.smem_optin / per_col, 4);   // <= 4 warps (launch bounds)
    return std::min(cpc, ncols);
}

// Variant selection (BASELINE north_star: "picked per (d, n, k1) from ncu-measured HBM GB/s").
// profiles/r02_variant_table.json (scripts/variant_table.py: all six variants at d = 2^20 and 2^23,
// n = 8 ... 256, k1 = 2 n^2, fp64 and fp32) is encoded below as rules on the dtype and
// the SA^T footprint k1 (n+1) w, the quantity that decides between the row-scatter variants: B wins
// every fp64 row and every fp32 row whose SA^T exceeds 64 KB; for a tiny fp32 SA^T the fp32 row-block
// copies of B contend in a few L2 lines and X (<= 8 KB) or T (<= 64 KB) is faster.  d did not change
// any winner (the one exception, fp64 n = 16 at d = 2^20, is T by 3%, within run-to-run noise).
struct VariantRule {
    csk_dtype dtype;
    int64_t max_sat_bytes;   // k1 * ncols * sizeof(element)
    int variant;
};
static const VariantRule kVariantTable[] = {
    // round-2 close: the narrow instantiations (2-3 CTAs per SM), interleaved fp32 copies and the
    // warp-per-element combine made B the fastest for every measured fp32 row as well
    // (profiles/r02_variant_table.json; fp32 d=2^23 n=8: B 0.191 ms vs X 0.962, n=16: B 0.206 vs T 0.625)
    {CSK_F32, INT64_MAX, CSK_VAR_BULK_ROW},
    {CSK_F64, INT64_MAX, CSK_VAR_BULK_ROW},   // every row (e.g. d=2^23 n=8 0.236 ms vs T 1.036, n=256 4.05 vs 8.57)
};

static int select_variant(int64_t d, int64_t k1, int ncols, csk_dtype dtype, bool has_sort) {
    (void)d;
    (void)has_sort;
    const int64_t bytes = k1 * ncols * (dtype == CSK_F64 ? 8 : 4);
    for (const VariantRule& r : kVariantTable)
        if (r.dtype == dtype && bytes <= r.max_sat_bytes) return r.variant;
    return CSK_VAR_BULK_ROW;
}

// 2-D tensor map of [A b] (rows x ncols, column stride lda) with a RB x cw box, 128B swizzle
template <typename T>
static bool make_tensor_map(CUtensorMap* tmap, const Cols<T>& cols, int64_t rows, int ncols, int cw) {
    constexpr int RB = 128 / sizeof(T);
    const T* base = cols.n > 0 ? cols.A : cols.b;
    const cuuint64_t gdim[2] = {(cuuint64_t)rows, (cuuint64_t)ncols};
    const cuuint64_t gstride[1] = {(cuuint64_t)(ncols > 1 ? cols.lda * (int64_t)sizeof(T)
                                                          : ((rows * (int64_t)sizeof(T) + 15) & ~(int64_t)15))};
    const cuuint32_t box[2] = {(cuuint32_t)RB, (cuuint32_t)cw};
    const cuuint32_t estride[2] = {1, 1};
    const CUresult cr = tensor_map_encoder()(
        tmap, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
        const_cast<T*>(base), gdim, gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return cr == CUDA_SUCCESS;
}

static int exp_switch() {   // CSK_EXP: roofline attribution of the B kernels (bench.py), 0 in production
    const char* e = std::getenv("CSK_EXP");
    return e ? std::atoi(e) : 0;
}

// fp64 B32 kernels need every column 16-B aligned; the fp32 kernel's 32-B loads need 32-B columns
template <typename T>
static bool cols_aligned(const Cols<T>& cols, size_t bytes) {
    const size_t elems = bytes / sizeof(T);
    return ((uintptr_t)cols.A % bytes) == 0 && (cols.n <= 1 || cols.lda % (int64_t)elems == 0) &&
           (cols.b == nullptr || ((uintptr_t)cols.b % bytes) == 0);
}

// For the row-scatter variants `out` is the SA^T workspace described by L (L.tma marks
// a TMA-eligible launch decided by cs_apply_impl); the others write column-major (out, ldo).
template <typename T>
static csk_status run_variant(int variant, csk_plan_t plan, int ncols, Cols<T> cols, int64_t row_begin,
                              int64_t row_end, double* out, int64_t ldo, const RowLayout& L, cudaStream_t st) {
    const DeviceInfo& di = device_info();
    const int64_t rows = row_end - row_begin;
    if (rows <= 0) return CSK_OK;
    // CSK_PLAN_HASH: only the default fp64 32-row kernels hash rows on the fly; every other
    // kernel reads the code array, materialised on first use
    const bool b32 = variant == CSK_VAR_BULK_ROW && sizeof(T) == 8 && cols_aligned(cols, 16) &&
                     (cols.n > 0 || cols.b != nullptr);
    if (plan->code == nullptr && !b32) {
        const csk_status es = ensure_codes(plan, st);
        if (es != CSK_OK) return es;
    }
    const uint32_t* code = plan->code ? reinterpret_cast<const uint32_t*>(plan->code) + row_begin : nullptr;
    switch (variant) {
        case CSK_VAR_ATOMIC_COL: {
            const int64_t blocks = std::min<int64_t>(ceil_div(rows, 256), (int64_t)di.num_sms * 8);
            prof_mark(st, true);   // right before the launch: host prep is not timed
            cs_col_kernel<T><<<(unsigned)blocks, 256, 0, st>>>(code, rows, cols, ncols, out, ldo);
            CSK_LAUNCH_CHECK();
            return CSK_OK;
        }
        case CSK_VAR_TMA_ROW: {
            constexpr int RB = 128 / sizeof(T);
            CSK_REQUIRE(L.tma, CSK_EINVAL, "variant X launched without a TMA layout");
            CUtensorMap tmap;
            CSK_REQUIRE(make_tensor_map(&tmap, cols, rows, ncols, L.cw), CSK_ECUDA, "cuTensorMapEncodeTiled failed");
            const int stage_bytes = (L.cw * 128 + 1023) & ~1023;
            const size_t smem = (size_t)kTmaWarps * kTmaStages * stage_bytes + (size_t)kTmaWarps * kTmaStages * RB * 4 +
                                (size_t)kTmaWarps * kTmaStages * 8 + 1024;
            CSK_REQUIRE(smem <= (size_t)di.smem_optin, CSK_EUNSUPPORTED, "variant X: tile does not fit smem");
            CSK_CUDA_TRY(cudaFuncSetAttribute(cs_tma_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            const int64_t units = ceil_div(rows, RB) * ceil_div(ncols, L.cw);
            const int64_t blocks = std::min<int64_t>(ceil_div(units, kTmaWarps), (int64_t)di.num_sms);
            prof_mark(st, true);
            cs_tma_kernel<T><<<(unsigned)blocks, kTmaWarps * 32, smem, st>>>(tmap, code, rows, ncols, stage_bytes, out, L);
            CSK_LAUNCH_CHECK();
            return CSK_OK;
        }
        case CSK_VAR_BULK_ROW: {
            const int cw = L.cw;   // set with the layout by cs_apply_impl
            const int expv = exp_switch();
            if constexpr (sizeof(T) == 4) {
                if (L.ncopies > 0) {   // fp32 accumulation into bounded-depth copies (default for fp32)
                    int ldf = (cw + 3) & ~3;
                    while (ldf % 32 != 4) ldf += 4;   // == 4 mod 32: conflict-free tile stores
                    constexpr int fw = 8;
                    const int kjf = f32_kj(cw);
                    auto fk = kjf == 5 ? cs_bulk64f_kernel<fw, 5> : kjf == 9 ? cs_bulk64f_kernel<fw, 9> : cs_bulk64f_kernel<fw>;
                    const int cps = kjf == 5 ? f32_ctas_per_sm<5>() : kjf == 9 ? f32_ctas_per_sm<9>() : 1;
                    const size_t smem = (size_t)fw * (kF32Rows * ldf + 32) * sizeof(float);
                    CSK_CUDA_TRY(cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                    const int64_t units = ceil_div(rows, kF32Rows) * ceil_div(ncols, cw);
                    const int64_t blocks = std::min<int64_t>(ceil_div(units, fw), (int64_t)di.num_sms * cps);
                    prof_mark(st, true);
                    fk<<<(unsigned)blocks, fw * 32, smem, st>>>(
                        code, rows, *reinterpret_cast<const Cols<float>*>(&cols), ncols, ldf,
                        reinterpret_cast<float*>(out), L);
                    CSK_LAUNCH_CHECK();
                    return CSK_OK;
                }
            }
            const int ldtile = (cw + 1) & ~1;
            if constexpr (sizeof(T) == 8) {
                if (b32) {
                    const int ld32 = ldtile % 4 == 0 ? ldtile + 2 : ldtile;   // == 2 mod 4
                    const int64_t units32 = ceil_div(rows, kB32Rows) * ceil_div(ncols, cw);
                    const size_t smem = (size_t)8 * (kB32Rows * ld32 + kB32Pad) * sizeof(double);
                    const bool narrow = cw < kBulkMaxCols - 3;   // predicated loads + evict_last (C3)
                    RowLayout LH = L;
                    if (code == nullptr) {   // CSK_PLAN_HASH plan: codes hashed in the kernel
                        LH.g0 = plan->row0 + row_begin;
                        LH.hkey0 = (uint32_t)plan->seed;
                        LH.hkey1 = (uint32_t)(plan->seed >> 32);
                    }
                    // narrow rows (chunk + pad <= 18 / 34 columns): the 2- / 3-CTA-per-SM instantiations
                    const int kjn = b32_kj(cw);
                    auto kern = code == nullptr ? (kjn == 9    ? cs_bulk32_kernel<8, 0, true, true, 9>
                                                   : kjn == 17 ? cs_bulk32_kernel<8, 0, true, true, 17>
                                                   : narrow    ? cs_bulk32_kernel<8, 0, true, true>
                                                               : cs_bulk32_kernel<8, 0, false, true>)
                                : expv == 1     ? cs_bulk32_kernel<8, 1>
                                : expv == 2     ? cs_bulk32_kernel<8, 2>
                                : expv == 3     ? cs_bulk32_kernel<8, 3>
                                : kjn == 9      ? cs_bulk32_kernel<8, 0, true, false, 9>
                                : kjn == 17     ? cs_bulk32_kernel<8, 0, true, false, 17>
                                : narrow        ? cs_bulk32_kernel<8, 0, true>
                                                : cs_bulk32_kernel<8, 0>;
                    const int cps = (expv != 0 && code != nullptr) ? 1 : kjn == 9 ? b32_ctas_per_sm<9>() : kjn == 17 ? b32_ctas_per_sm<17>() : 1;
                    CSK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                    const int64_t blocks = std::min<int64_t>(ceil_div(units32, 8), (int64_t)di.num_sms * cps);
                    prof_mark(st, true);   // right before the launch: host prep is not timed
                    kern<<<(unsigned)blocks, 256, smem, st>>>(code, rows, cols, ncols, ld32, out, LH, (int)plan->k1);
                    CSK_LAUNCH_CHECK();
                    return CSK_OK;
                }
            }
            // 16-row tiles: unaligned fp64 columns, or fp32 accumulated in fp64 (CSK_F32ACC=0, unaligned)
            const int64_t units = ceil_div(rows, kBulkRows) * ceil_div(ncols, cw);
            auto launch = [&](auto cfg) -> csk_status {
                using C = decltype(cfg);
                const size_t smem = (size_t)C::kWarps * C::kBufs * kBulkRows * ldtile * sizeof(double);
                if (smem > (size_t)di.smem_optin) return CSK_EUNSUPPORTED;
                auto kb = expv == 1 ? cs_bulk_kernel<T, C, 1>
                          : expv == 2 ? cs_bulk_kernel<T, C, 2>
                          : expv == 3 ? cs_bulk_kernel<T, C, 3> : cs_bulk_kernel<T, C, 0>;
                CSK_CUDA_TRY(cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                const int64_t blocks = std::min<int64_t>(ceil_div(units, C::kWarps), (int64_t)di.num_sms);
                prof_mark(st, true);
                kb<<<(unsigned)blocks, C::kWarps * 32, smem, st>>>(code, rows, cols, ncols, ldtile, out, L);
                CSK_LAUNCH_CHECK();
                return CSK_OK;
            };
            // measured at C2: 12/16 warps and register double-buffering were not faster than 8 x 2
            csk_status r = launch(BulkCfg<8, 2, false>{});
            if (r == CSK_EUNSUPPORTED) r = launch(BulkCfg<4, 2, false>{});
            CSK_REQUIRE(r != CSK_EUNSUPPORTED, CSK_EUNSUPPORTED, "variant B: tile does not fit smem");
            return r;
        }
        case CSK_VAR_ATOMIC_ROW: {
            const size_t smem = (size_t)kRowWarps * 32 * kTileLd * sizeof(double);
            const int64_t units = ceil_div(rows, 32) * ceil_div(ncols, 32);
            auto kern = cs_row_kernel<T>;
            CSK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int per_sm = 0;
            CSK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRowWarps * 32, smem));
            per_sm = std::max(per_sm, 1);
            const int64_t blocks = std::min<int64_t>(ceil_div(units, kRowWarps), (int64_t)di.num_sms * per_sm);
            prof_mark(st, true);
            kern<<<(unsigned)blocks, kRowWarps * 32, smem, st>>>(code, rows, cols, ncols, out, ldo);
            CSK_LAUNCH_CHECK();
            return CSK_OK;
        }
        case CSK_VAR_SMEM: {
            const int cpc = smem_cpc(plan->k1, ncols);
            CSK_REQUIRE(cpc >= 1, CSK_EUNSUPPORTED, "variant S: k1=%lld buckets do not fit shared memory",
                        (long long)plan->k1);
            const size_t smem = (size_t)cpc * plan->k1 * sizeof(double);
            CSK_CUDA_TRY(cudaFuncSetAttribute(cs_smem_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)smem));
            const int ngroups = (ncols + cpc - 1) / cpc;
            const int64_t total = (int64_t)ngroups * rows;
            int per_sm = 0;
            CSK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cs_smem_kernel<T>, cpc * 32, smem));
            per_sm = std::max(per_sm, 1);
            const int64_t grid = std::max<int64_t>(
                1, std::min<int64_t>((int64_t)di.num_sms * per_sm, ceil_div(total, 32 * kPrivDepth * 4)));
            const int64_t per_cta = ceil_div(total, grid);
            prof_mark(st, true);
            cs_smem_kernel<T><<<(unsigned)grid, cpc * 32, smem, st>>>(code, rows, cols, ncols, cpc,
                                                                        (int)plan->k1, out, ldo, per_cta);
            CSK_LAUNCH_CHECK();
            return CSK_OK;
        }
        case CSK_VAR_SORTED: {
            CSK_REQUIRE(plan->perm != nullptr, CSK_EUNSUPPORTED, "variant G needs a plan built with CSK_PLAN_SORT");
            CSK_REQUIRE(row_begin == 0 && row_end == plan->d, CSK_EUNSUPPORTED,
                        "variant G needs the whole block resident on the device");
            const int64_t blocks = std::min<int64_t>(ceil_div(plan->k1 * 32, 256), (int64_t)di.num_sms * 16);
            prof_mark(st, true);
            cs_sorted_kernel<T><<<(unsigned)blocks, 256, 0, st>>>(code, plan->perm, plan->offsets, plan->k1, cols,
                                                                  ncols, out, ldo);
            CSK_LAUNCH_CHECK();
            return CSK_OK;
        }
        default:
            set_error("unknown variant %d", variant);
            return CSK_EINVAL;
    }
}

struct ApplyTarget {
    double* buf = nullptr;   // accumulation buffer (fp64; floats for the fp32-accumulation copies)
    int64_t ld = 0;
    bool owned = false;
};

// Footprint the spread copies of a small SA^T should reach (CSK_SPREAD_KB overrides,
// 0 disables)
static int64_t spread_target_bytes() {
    if (const char* e = std::getenv("CSK_SPREAD_KB")) return std::atoll(e) * 1024;
    return kSpreadBytes;
}

// Row-major SA^T layout of the B kernels: all columns in one row when ncols <= 66, else the fewest
// chunks of <= 66 (even) columns; chunk-major (one slice per chunk) when the whole SA^T would take
// more than half of L2, with the chunk width cut so one slice fits half of L2.
// Units of lc / cs: elements of width esz.
static void bulk_layout(RowLayout& L, int64_t k1, int ncols, size_t esz, int align_elems) {
    L.cw = bulk_chunk_width(ncols);
    const int64_t l2h = (int64_t)device_info().l2_bytes / 2;
    if ((int64_t)k1 * ncols * (int64_t)esz > l2h) {
        const int64_t fit = std::max<int64_t>(2, (l2h / ((int64_t)esz * k1)) & ~1);
        const int nch = (int)std::max<int64_t>(ceil_div(ncols, kBulkMaxCols), ceil_div(ncols, fit));
        L.cw = std::min(kBulkMaxCols, (((ncols + nch - 1) / nch) + 1) & ~1);
    }
    const int nchunks = (ncols + L.cw - 1) / L.cw;
    const int64_t cwa = (L.cw + align_elems - 1) / align_elems * align_elems;
    if (nchunks > 1 && (int64_t)k1 * ncols * (int64_t)esz > l2h) {
        L.chunk_major = true;   // one L2-sized SA^T slice per column chunk
        L.lc = cwa;
        L.cs = k1 * L.lc;
    } else {
        // chunks start on aligned boundaries inside a row
        L.cs = nchunks > 1 ? cwa : L.cw;
        L.lc = std::max<int64_t>((ncols + align_elems - 1) / align_elems * align_elems, nchunks * cwa);
    }
}

csk_status cs_apply_impl(csk_plan_t plan, csk_dtype dtype, int64_t n, const void* A, int64_t lda, const void* b,
                         void* SA, int64_t ldsa, int variant, cudaStream_t st, int64_t row_begin, int64_t row_end,
                         bool accumulate, RowOut* rowout) {
    CSK_REQUIRE(plan != nullptr, CSK_EINVAL, "plan is NULL");
    CSK_REQUIRE(dtype == CSK_F64 || dtype == CSK_F32, CSK_EDTYPE, "dtype %d not supported", (int)dtype);
    CSK_REQUIRE(n >= 0, CSK_EINVAL, "n=%lld must be >= 0", (long long)n);
    const int64_t ncols64 = n + (b ? 1 : 0);
    CSK_REQUIRE(ncols64 >= 1 && ncols64 <= 65536, CSK_EINVAL, "n + (b != NULL) = %lld must be in [1, 65536]",
                (long long)ncols64);
    CSK_REQUIRE(n == 0 || A != nullptr, CSK_EINVAL, "A is NULL");
    CSK_REQUIRE(SA != nullptr || rowout != nullptr, CSK_EINVAL, "SA is NULL");
    if (rowout != nullptr) *rowout = RowOut{};
    CSK_REQUIRE(row_begin >= 0 && row_begin < row_end && row_end <= plan->d, CSK_EINVAL, "bad row range");
    CSK_REQUIRE(n == 0 || lda >= row_end - row_begin, CSK_ESHAPE, "lda=%lld < rows=%lld", (long long)lda,
                (long long)(row_end - row_begin));
    CSK_REQUIRE(ldsa >= plan->k1, CSK_ESHAPE, "ldsa=%lld < k1=%lld", (long long)ldsa, (long long)plan->k1);
    const int ncols = (int)ncols64;
    if (variant == CSK_VAR_AUTO) variant = env_variant();
    if (variant == CSK_VAR_AUTO) variant = select_variant(plan->d, plan->k1, ncols, dtype, plan->perm != nullptr);
    CSK_REQUIRE(variant >= CSK_VAR_ATOMIC_COL && variant <= CSK_VAR_TMA_ROW, CSK_EINVAL, "unknown variant %d",
                variant);
    if (variant == CSK_VAR_SMEM && smem_cpc(plan->k1, ncols) < 1) variant = CSK_VAR_BULK_ROW;
    if (accumulate) {
        // accumulating row blocks into SA (host streaming): SA itself must be the fp64 target
        CSK_REQUIRE(dtype == CSK_F64, CSK_EDTYPE, "row-block accumulation needs fp64");
        if (variant_rowmajor(variant) || variant == CSK_VAR_SORTED) variant = CSK_VAR_ATOMIC_COL;
    }
    const int64_t k1 = plan->k1;
    const int64_t rows = row_end - row_begin;
    const size_t esz = dtype == CSK_F64 ? 8 : 4;
    const void* base = n > 0 ? A : b;

    // variant X loads [A b] as one 2-D TMA tensor
    bool tma = variant == CSK_VAR_TMA_ROW && (n == 0 || b == nullptr ||
                                              (const char*)b == (const char*)A + (size_t)n * lda * esz);
    tma = tma && ((uintptr_t)base & 15) == 0 && (ncols == 1 || ((lda * (int64_t)esz) & 15) == 0);
    if (tma && plan->code == nullptr) {   // hash plan: the TMA kernel reads codes
        const csk_status es = ensure_codes(plan, st);
        if (es != CSK_OK) return es;
    }
    tma = tma && (((uintptr_t)(plan->code + row_begin)) & 15) == 0 && tensor_map_encoder() != nullptr;
    if (variant == CSK_VAR_TMA_ROW && !tma) variant = CSK_VAR_ATOMIC_ROW;

    ApplyTarget tgt;
    RowLayout L;
    size_t ws_doubles = 0;
    if (variant_rowmajor(variant)) {
        if (variant == CSK_VAR_TMA_ROW) {
            L.tma = true;
            L.cw = tma_chunk_width(ncols);
            L.cs = L.cw;
            L.lc = (ncols + 3) & ~3;
            ws_doubles = (size_t)k1 * L.lc;
        } else if (variant == CSK_VAR_BULK_ROW) {
            // fp32 input: fp32 sums in row-block copies of mean bucket depth <= 64, combined in fp64
            // (default; CSK_F32ACC=0 accumulates fp32 input in fp64 instead, for A/B measurements)
            const char* f32e = std::getenv("CSK_F32ACC");
            const bool f32acc = dtype == CSK_F32 && !(f32e && std::atoi(f32e) == 0) &&
                                cols_aligned(Cols<float>{static_cast<const float*>(A), static_cast<const float*>(b),
                                                         lda, (int)n},
                                             32);
            if (f32acc) {
                bulk_layout(L, k1, ncols, 4, 8);   // 32-B aligned rows and chunk starts
                // no cap on the copy count: a cap would let the mean depth exceed 64 at small k1 (the 1e-5 bound needs
                // every bucket sum of a copy to stay far below 1e-5 / u32 = 168 terms)
                int64_t ncp = std::max<int64_t>(1, ceil_div(rows, 64 * k1));
                // a small copy is spread: S consecutive tiles go to S different copies (kernel comment), S
                // chosen so the S copies in use reach the spread footprint
                {
                    const int64_t cbytes = (int64_t)k1 * L.lc * 4 * ((ncols + L.cw - 1) / L.cw);
                    const int64_t S = std::max<int64_t>(1, std::min<int64_t>(ncp, spread_target_bytes() / std::max<int64_t>(cbytes, 1)));
                    ncp = ceil_div(ncp, S) * S;
                    L.f32_spread = (int)S;
                }
                L.ncopies = (int)ncp;
                // whole 64-row tiles per copy (the kernel maps a tile to its copy with one division); the
                // mean bucket depth stays <= 64 + 64 / k1 (<= 128 for k1 = 1, where the depth is exact)
                L.rows_per_copy = ceil_div(ceil_div(rows, ncp), (int64_t)kF32Rows) * kF32Rows;
                L.copy_stride = L.chunk_major ? L.cs * ((ncols + L.cw - 1) / L.cw) : k1 * L.lc;   // floats
                ws_doubles = (size_t)ceil_div(ncp * L.copy_stride, 2);
            } else {
                bulk_layout(L, k1, ncols, 8, 4);
                const int nchunks = (ncols + L.cw - 1) / L.cw;
                ws_doubles = L.chunk_major ? (size_t)nchunks * L.cs : (size_t)k1 * L.lc;
                // spread copies for a small SA^T (fp64 B32 kernel only: 16-B aligned columns)
                const bool b32 = dtype == CSK_F64 && !accumulate &&
                                 cols_aligned(Cols<double>{static_cast<const double*>(A),
                                                           static_cast<const double*>(b), lda, (int)n},
                                              16);
                if (b32 && !L.chunk_major) {
                    const int64_t units32 = ceil_div(rows, kB32Rows) * nchunks;
                    const int64_t ctas = std::min<int64_t>(ceil_div(units32, 8), (int64_t)device_info().num_sms);
                    const int64_t want = spread_target_bytes() / (int64_t)(ws_doubles * 8);
                    L.nspread = (int)std::max<int64_t>(1, std::min<int64_t>(want, ctas));
                    L.spread_stride = (int64_t)ws_doubles;
                    ws_doubles *= (size_t)L.nspread;
                }
            }
        } else {
            L.cw = ncols;   // T: its own 32-column chunks, one row of SA^T
            L.lc = (ncols + 3) & ~3;
            L.cs = ncols;
            ws_doubles = (size_t)k1 * L.lc;
        }
        tgt.ld = L.lc;
        tgt.owned = true;
    } else if (dtype == CSK_F32 || SA == nullptr) {
        // fp32 output of a column-major variant, or the row-major hand-over: private fp64 target
        tgt.ld = k1;
        tgt.owned = true;
        ws_doubles = (size_t)k1 * ncols;
    } else {
        tgt.buf = static_cast<double*>(SA);
        tgt.ld = ldsa;
    }
    if (tgt.owned) {
        // + 2 doubles: the B kernels' work counter, zeroed by the same memset
        CSK_CUDA_TRY(csk_malloc_async(&tgt.buf, (ws_doubles + 2) * sizeof(double), st));
        CSK_CUDA_TRY(cudaMemsetAsync(tgt.buf, 0, (ws_doubles + 2) * sizeof(double), st));
        L.work = reinterpret_cast<unsigned long long*>(tgt.buf + ws_doubles);
        if (const char* ge = std::getenv("CSK_GRAB")) L.grab = std::max(1, std::atoi(ge));   // sweep hook
        if (const char* te = std::getenv("CSK_GRAB_TAIL")) L.grab_tail = std::atoi(te);     // A/B hook
    } else if (variant != CSK_VAR_SORTED && !accumulate) {
        // zero SA (ldsa may exceed k1: clear the k1 x ncols window only)
        if (ldsa == k1) {
            CSK_CUDA_TRY(cudaMemsetAsync(tgt.buf, 0, (size_t)k1 * ncols * sizeof(double), st));
        } else {
            CSK_CUDA_TRY(cudaMemset2DAsync(tgt.buf, ldsa * sizeof(double), 0, k1 * sizeof(double), ncols, st));
        }
    }
    auto release = on_exit([&] {
        if (tgt.owned && tgt.buf) cudaFreeAsync(tgt.buf, st);
    });
    csk_status s;
    if (dtype == CSK_F64) {
        Cols<double> cols{static_cast<const double*>(A), static_cast<const double*>(b), lda, (int)n};
        s = run_variant<double>(variant, plan, ncols, cols, row_begin, row_end, tgt.buf, tgt.ld, L, st);
    } else {
        Cols<float> cols{static_cast<const float*>(A), static_cast<const float*>(b), lda, (int)n};
        s = run_variant<float>(variant, plan, ncols, cols, row_begin, row_end, tgt.buf, tgt.ld, L, st);
    }
    prof_mark(st, false);
    if (s != CSK_OK) return s;
    auto launch_ok = [&](const char* what) -> csk_status {
        count_launch();
        if (cudaGetLastError() != cudaSuccess) {
            set_error("cs_apply %s launch failed", what);
            return CSK_ECUDA;
        }
        return CSK_OK;
    };
    if (L.nspread > 1) {   // fold the spread copies into copy 0 (the layout every consumer reads)
        const int64_t ne = L.spread_stride;
        cs_spread_combine_kernel<<<(unsigned)std::min<int64_t>(ceil_div(ne, 256), 4 * device_info().num_sms), 256, 0,
                                   st>>>(tgt.buf, ne, L.nspread, L.spread_stride);
        const csk_status ls = launch_ok("spread combine");
        if (ls != CSK_OK) return ls;
    }
    if (rowout != nullptr) {
        if (L.ncopies > 0) {   // fp32 copies -> fp64 row-major workspace (regular layout)
            const int64_t lcd = (ncols + 1) & ~1;
            double* Yt = nullptr;
            CSK_CUDA_TRY(csk_malloc_async(&Yt, (size_t)k1 * lcd * sizeof(double), st));
            if (L.ncopies >= kCombineWarpCopies)
                cs_combine_warp_kernel<true><<<(unsigned)ceil_div(k1 * lcd, 8), 256, 0, st>>>(
                    reinterpret_cast<const float*>(tgt.buf), L, k1, ncols, lcd, Yt, nullptr, 0);
            else
                cs_combine_rows_kernel<<<(unsigned)ceil_div(k1 * lcd, 256), 256, 0, st>>>(
                    reinterpret_cast<const float*>(tgt.buf), L, k1, ncols, Yt, lcd);
            const csk_status ls = launch_ok("fp32 combine");
            if (ls != CSK_OK) {
                cudaFreeAsync(Yt, st);
                return ls;
            }
            *rowout = RowOut{Yt, ncols, ncols, lcd, ncols};
            return CSK_OK;
        }
        if (variant_rowmajor(variant)) {
            // the caller (ms_apply) consumes the row-major SA^T directly (Z^T = Y^T G^T, no transpose)
            *rowout = RowOut{tgt.buf, L.cw, ncols, L.lc, L.cs};
            tgt.owned = false;   // handed over
            return CSK_OK;
        }
        return rows_from_colmajor(tgt.buf, tgt.ld, k1, ncols, rowout, st);   // L, S, G
    }
    if (!tgt.owned) return CSK_OK;
    dim3 grid((unsigned)ceil_div(k1, 32), (unsigned)ceil_div(ncols, 32));
    if (L.ncopies > 0) {
        if (L.ncopies >= kCombineWarpCopies)
            cs_combine_warp_kernel<false><<<(unsigned)ceil_div(k1 * ncols, 8), 256, 0, st>>>(
                reinterpret_cast<const float*>(tgt.buf), L, k1, ncols, 0, nullptr, static_cast<float*>(SA), ldsa);
        else
            cs_combine_f32_kernel<<<grid, dim3(32, 8), 0, st>>>(reinterpret_cast<const float*>(tgt.buf), L, k1, ncols,
                                                                static_cast<float*>(SA), ldsa);
        return launch_ok("fp32 combine");
    }
    if (variant_rowmajor(variant)) {
        if (dtype == CSK_F64)
            transpose_out_kernel<double><<<grid, dim3(32, 8), 0, st>>>(tgt.buf, L, k1, ncols, static_cast<double*>(SA),
                                                                       ldsa);
        else
            transpose_out_kernel<float><<<grid, dim3(32, 8), 0, st>>>(tgt.buf, L, k1, ncols, static_cast<float*>(SA),
                                                                      ldsa);
        return launch_ok("transpose");
    }
    narrow_kernel<<<(unsigned)std::min<int64_t>(ceil_div(k1 * ncols, 256), 4096), 256, 0, st>>>(
        tgt.buf, k1, ncols, static_cast<float*>(SA), ldsa);
    return launch_ok("narrow");
}

}  // namespace csk

extern "C" csk_status cs_apply(csk_plan_t plan, csk_dtype dtype, int64_t n, const void* A, int64_t lda,
                               const void* b, void* SA, int64_t ldsa, int variant, void* stream) {
    CSK_REQUIRE(plan != nullptr, CSK_EINVAL, "plan is NULL");
    return csk::cs_apply_impl(plan, dtype, n, A, lda, b, SA, ldsa, variant, (cudaStream_t)stream, 0, plan->d,
                              false);
}

// ------------------------------------------------------------- profiling
namespace csk {
static thread_local bool g_prof = false;
// pool of events created by csk_profile_enable (no cudaEventCreate on the launch path);
// g_prof_pairs[i] = (begin, end) indices of the i-th profiled launch
static thread_local std::vector<cudaEvent_t> g_prof_pool;
static thread_local size_t g_prof_next = 0;
static thread_local std::vector<std::pair<int, int>> g_prof_pairs;
constexpr size_t kProfPool = 4096;

void prof_mark(cudaStream_t st, bool begin) {
    if (!g_prof || g_prof_next >= g_prof_pool.size()) return;
    if (begin) {
        if (!g_prof_pairs.empty() && g_prof_pairs.back().second < 0) return;   // one open interval
        cudaEventRecord(g_prof_pool[g_prof_next], st);
        g_prof_pairs.push_back({(int)g_prof_next++, -1});
    } else if (!g_prof_pairs.empty() && g_prof_pairs.back().second < 0) {
        cudaEventRecord(g_prof_pool[g_prof_next], st);
        g_prof_pairs.back().second = (int)g_prof_next++;
    }
}
}  // namespace csk

extern "C" void csk_profile_enable(int on) {
    csk::g_prof = on != 0;
    if (csk::g_prof && csk::g_prof_pool.empty()) {
        csk::g_prof_pool.resize(csk::kProfPool);
        for (auto& e : csk::g_prof_pool)
            if (cudaEventCreate(&e) != cudaSuccess) {
                csk::g_prof = false;
                break;
            }
    }
    csk::g_prof_next = 0;
    csk::g_prof_pairs.clear();
}

extern "C" csk_status csk_profile_read(double* total_ms, uint64_t* launches) {
    double sum = 0.0;
    uint64_t cnt = 0;
    for (auto& p : csk::g_prof_pairs) {
        if (p.second < 0) continue;
        CSK_CUDA_TRY(cudaEventSynchronize(csk::g_prof_pool[p.second]));
        float ms = 0.f;
        CSK_CUDA_TRY(cudaEventElapsedTime(&ms, csk::g_prof_pool[p.first], csk::g_prof_pool[p.second]));
        sum += ms;
        ++cnt;
    }
    csk::g_prof_next = 0;
    csk::g_prof_pairs.clear();
    if (total_ms) *total_ms = sum;
    if (launches) *launches = cnt;
    return CSK_OK;
}
