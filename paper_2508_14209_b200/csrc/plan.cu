// plan.cu -- library status/bookkeeping and the CountSketch plan.
//
// a1 codes: bucket h(i) and sign s(i) of GLOBAL row i from Philox4x32-10
//   (Def 3; hash generation; R1, R3).
// a2 sort : stable LSD radix sort of rows by bucket -> offsets[k1+1], perm[d]
//   (BASELINE.json north_star form 1: "one-time integer counting-sort of h").
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "csk_internal.cuh"

namespace csk {

static thread_local std::string g_last_error;
static thread_local uint64_t g_launches = 0;

void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
}
const char* last_error() { return g_last_error.c_str(); }
void count_launch() { ++g_launches; }

const DeviceInfo& device_info() {
    static std::mutex mu;
    static std::map<int, DeviceInfo> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    DeviceInfo info;
    info.device = dev;
    cudaDeviceGetAttribute(&info.num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&info.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&info.l2_bytes, cudaDevAttrL2CacheSize, dev);
    // The library's own stream-ordered pool (workspaces of SA, Z, QR, ... are cudaMallocAsync'd per
    // call): freed blocks stay mapped (release threshold max), and a block freed on one stream is
    // reused on another only through an event dependency the caller made, never through hidden
    // internal dependencies or opportunistic reuse -- with those (the default pool's defaults) a
    // two-stream pipeline (bench --pipeline) saw single steps of 9-23 ms in 5 of 10 C3/C4 runs, none
    // in 10 runs without.  CSK_POOL_NODEP=0 restores the default behaviour.
    {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&info.pool, &props) != cudaSuccess) {
            info.pool = nullptr;
            cudaDeviceGetDefaultMemPool(&info.pool, dev);
        }
        if (info.pool) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(info.pool, cudaMemPoolAttrReleaseThreshold, &thr);
            const char* e = std::getenv("CSK_POOL_NODEP");
            if (!(e && std::atoi(e) == 0)) {
                int zero = 0;
                cudaMemPoolSetAttribute(info.pool, cudaMemPoolReuseAllowInternalDependencies, &zero);
                cudaMemPoolSetAttribute(info.pool, cudaMemPoolReuseAllowOpportunistic, &zero);
            }
        }
    }
    cudaGetLastError();
    return cache.emplace(dev, info).first->second;
}

cudaError_t csk_malloc_async(void** p, size_t bytes, cudaStream_t st) {
    const DeviceInfo& di = device_info();
    return di.pool ? cudaMallocFromPoolAsync(p, bytes, di.pool, st) : cudaMallocAsync(p, bytes, st);
}

bool is_device_pointer(const void* p) {
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

// ------------------------------------------------------------- a1: codes
// Thread t owns Philox block q (global rows 4q..4q+3); one 128-bit draw serves
// four rows (R3).  h = floor(w * k1 / 2^32) = umulhi(w, k1).
__global__ void __launch_bounds__(256) codes_kernel(int32_t* __restrict__ code, int64_t d, uint32_t k1,
                                                    uint32_t key_lo, uint32_t key_hi, int64_t row0) {
    const int64_t q_first = row0 >> 2;
    const int64_t q_last = (row0 + d - 1) >> 2;
    for (int64_t q = q_first + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q <= q_last;
         q += (int64_t)gridDim.x * blockDim.x) {
        const uint4 x = philox4x32_10(make_uint4((uint32_t)q, (uint32_t)(q >> 32), 0u, 0u),
                                      make_uint2(key_lo, key_hi));
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t i = 4 * q + j - row0;
            if (i >= 0 && i < d) code[i] = (int32_t)(__umulhi(w[j], k1) | ((w[j] & 1u) << 31));
        }
    }
}

// --------------------------------------------------------- a2: radix sort
// One LSD pass over an 8-bit digit of the bucket.  Stable: rows are assigned to
// CTAs and warps in index order, ranks within a warp come from __match_any_sync.
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;                        // per thread
constexpr int kSortTile = kSortThreads * kSortItems;  // rows per CTA

__global__ void __launch_bounds__(kSortThreads) radix_hist_kernel(const uint32_t* __restrict__ keys, int64_t d,
                                                                  int shift, uint32_t* __restrict__ hist,
                                                                  int64_t ntiles) {
    __shared__ uint32_t h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int k = 0; k < kSortItems; ++k) {
        const int64_t i = base + (int64_t)k * kSortThreads + threadIdx.x;
        if (i < d) atomicAdd(&h[((keys[i] & 0x7fffffffu) >> shift) & 255u], 1u);
    }
    __syncthreads();
    // digit-major layout: hist[digit * ntiles + tile]
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[(int64_t)i * ntiles + blockIdx.x] = h[i];
}

// exclusive scan of n uint32 counts into int64 (single CTA, sequential chunks)
__global__ void __launch_bounds__(1024) scan_kernel(const uint32_t* __restrict__ in, int64_t* __restrict__ out,
                                                    int64_t n) {
    __shared__ int64_t warp_sums[32];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t base = 0; base < n; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        int64_t v = i < n ? (int64_t)in[i] : 0;
        int64_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_sums[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            int64_t s = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int64_t t = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += t;
            }
            warp_sums[lane] = s;   // inclusive over warps
        }
        __syncthreads();
        const int64_t warp_prefix = warp ? warp_sums[warp - 1] : 0;
        if (i < n) out[i] = carry + warp_prefix + incl - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += warp_prefix + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[n] = carry;
}

__global__ void __launch_bounds__(kSortThreads) radix_scatter_kernel(
    const uint32_t* __restrict__ keys_in, const int32_t* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
    int32_t* __restrict__ vals_out, int64_t d, int shift, const int64_t* __restrict__ tile_offsets, int64_t ntiles) {
    constexpr int kWarps = kSortThreads / 32;
    __shared__ uint32_t warp_count[kWarps][256];
    __shared__ int64_t digit_base[256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kWarps * 256; i += blockDim.x) (&warp_count[0][0])[i] = 0;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) digit_base[i] = tile_offsets[(int64_t)i * ntiles + blockIdx.x];
    __syncthreads();
    // warp w owns rows [base + w*32*K, base + (w+1)*32*K), visited 32 at a time in order
    const int64_t wbase = (int64_t)blockIdx.x * kSortTile + (int64_t)warp * 32 * kSortItems;
    uint32_t digit[kSortItems];
    uint32_t rank[kSortItems];
#pragma unroll
    for (int k = 0; k < kSortItems; ++k) {
        const int64_t i = wbase + k * 32 + lane;
        const bool valid = i < d;
        const uint32_t dg = valid ? ((keys_in[i] & 0x7fffffffu) >> shift) & 255u : 256u + lane;
        const uint32_t peers = __match_any_sync(0xffffffffu, dg);
        const uint32_t lt = peers & ((1u << lane) - 1u);
        uint32_t before = 0;
        if (valid) before = warp_count[warp][dg];
        __syncwarp();
        rank[k] = before + __popc(lt);
        digit[k] = dg;
        // the highest lane of each peer group bumps the counter
        if (valid && (peers >> lane) == 1u) warp_count[warp][dg] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // exclusive scan over warps for each digit
    for (int dg = threadIdx.x; dg < 256; dg += blockDim.x) {
        uint32_t run = 0;
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = warp_count[w][dg];
            warp_count[w][dg] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kSortItems; ++k) {
        const int64_t i = wbase + k * 32 + lane;
        if (i < d) {
            const uint32_t dg = digit[k];
            const int64_t pos = digit_base[dg] + warp_count[warp][dg] + rank[k];
            keys_out[pos] = keys_in[i];
            vals_out[pos] = vals_in ? vals_in[i] : (int32_t)i;
        }
    }
}

__global__ void iota_kernel(int32_t* __restrict__ v, int64_t d) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (int32_t)i;
}

// bucket offsets from the sorted keys: offsets[m] = first position with bucket >= m
__global__ void bucket_offsets_kernel(const uint32_t* __restrict__ sorted, int64_t d, int64_t k1,
                                      int64_t* __restrict__ offsets) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= d; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = p == 0 ? 0 : (int64_t)(sorted[p - 1] & 0x7fffffffu) + 1;
        const int64_t hi = p == d ? k1 : (int64_t)(sorted[p] & 0x7fffffffu);
        for (int64_t m = lo; m <= hi; ++m) offsets[m] = p;
    }
}

static csk_status build_sort(csk_plan_t plan, cudaStream_t st) {
    const int64_t d = plan->d, k1 = plan->k1;
    int bits = 0;
    while (bits < 31 && ((int64_t)1 << bits) < k1) ++bits;
    const int passes = bits == 0 ? 0 : (bits + 7) / 8;
    const int64_t ntiles = ceil_div(d, kSortTile);
    uint32_t *k_a = nullptr, *k_b = nullptr, *hist = nullptr;
    int32_t* v_b = nullptr;
    int64_t* tile_off = nullptr;
    CSK_CUDA_TRY(csk_malloc_async(&k_a, d * 4, st));
    CSK_CUDA_TRY(csk_malloc_async(&k_b, d * 4, st));
    CSK_CUDA_TRY(csk_malloc_async(&v_b, d * 4, st));
    CSK_CUDA_TRY(csk_malloc_async(&hist, 256 * ntiles * 4, st));
    CSK_CUDA_TRY(csk_malloc_async(&tile_off, (256 * ntiles + 1) * 8, st));
    CSK_CUDA_TRY(cudaMemcpyAsync(k_a, plan->code, d * 4, cudaMemcpyDeviceToDevice, st));
    uint32_t* kin = k_a;
    uint32_t* kout = k_b;
    int32_t* vin = nullptr;     // identity on the first pass
    int32_t* vout = plan->perm;
    int32_t* vspare = v_b;
    if (passes == 0) {   // k1 == 1: every row is in bucket 0, the stable sort is the identity
        iota_kernel<<<256, 256, 0, st>>>(plan->perm, d);
        CSK_LAUNCH_CHECK();
    }
    for (int p = 0; p < passes; ++p) {
        radix_hist_kernel<<<(unsigned)ntiles, kSortThreads, 0, st>>>(kin, d, 8 * p, hist, ntiles);
        CSK_LAUNCH_CHECK();
        scan_kernel<<<1, 1024, 0, st>>>(hist, tile_off, 256 * ntiles);
        CSK_LAUNCH_CHECK();
        radix_scatter_kernel<<<(unsigned)ntiles, kSortThreads, 0, st>>>(kin, vin, kout, vout, d, 8 * p, tile_off,
                                                                         ntiles);
        CSK_LAUNCH_CHECK();
        std::swap(kin, kout);
        vin = vout;
        std::swap(vout, vspare);
    }
    // after the loop the sorted values are in vin; make sure they land in plan->perm
    if (passes > 0 && vin != plan->perm)
        CSK_CUDA_TRY(cudaMemcpyAsync(plan->perm, vin, d * 4, cudaMemcpyDeviceToDevice, st));
    bucket_offsets_kernel<<<256, 256, 0, st>>>(kin, d, k1, plan->offsets);
    CSK_LAUNCH_CHECK();
    CSK_CUDA_TRY(cudaFreeAsync(k_a, st));
    CSK_CUDA_TRY(cudaFreeAsync(k_b, st));
    CSK_CUDA_TRY(cudaFreeAsync(v_b, st));
    CSK_CUDA_TRY(cudaFreeAsync(hist, st));
    CSK_CUDA_TRY(cudaFreeAsync(tile_off, st));
    return CSK_OK;
}

static csk_status alloc_plan(int64_t d, int64_t k1, uint32_t flags, csk_plan_t* out, csk_plan_t* plan_out) {
    CSK_REQUIRE(out != nullptr, CSK_EINVAL, "out is NULL");
    *out = nullptr;
    CSK_REQUIRE(d >= 1 && d <= 2147483647LL, CSK_EINVAL, "d=%lld must be in [1, 2^31-1]", (long long)d);
    CSK_REQUIRE(k1 >= 1 && k1 <= 2147483647LL, CSK_EINVAL, "k1=%lld must be in [1, 2^31-1]", (long long)k1);
    CSK_REQUIRE((flags & ~(CSK_PLAN_SORT | CSK_PLAN_HASH)) == 0, CSK_EINVAL, "unknown plan flags 0x%x", flags);
    csk_plan_t plan = new (std::nothrow) csk_plan_s();
    CSK_REQUIRE(plan != nullptr, CSK_ENOMEM, "plan allocation failed");
    plan->d = d;
    plan->k1 = k1;
    cudaGetDevice(&plan->device);
    // codes are padded by 32 zero entries: 64/128-B bulk copies of a tile's codes never read past the end
    const bool hash = (flags & CSK_PLAN_HASH) && !(flags & CSK_PLAN_SORT);
    plan->hash = hash;
    if ((!hash && (cudaMalloc(&plan->code, (d + 32) * 4) != cudaSuccess ||
                   cudaMemset(plan->code + d, 0, 32 * 4) != cudaSuccess)) ||
        ((flags & CSK_PLAN_SORT) &&
         (cudaMalloc(&plan->offsets, (k1 + 1) * 8) != cudaSuccess || cudaMalloc(&plan->perm, d * 4) != cudaSuccess))) {
        cudaGetLastError();
        cs_plan_destroy(plan);
        set_error("device allocation of the plan failed (d=%lld, k1=%lld)", (long long)d, (long long)k1);
        return CSK_ENOMEM;
    }
    *plan_out = plan;
    return CSK_OK;
}

csk_status ensure_codes(csk_plan_t plan, cudaStream_t st) {
    // A CSK_PLAN_HASH plan materialises its codes on first use by a kernel that reads them.  The
    // codes are published (plan->code) only after the stream has finished writing them, so a
    // consumer on another stream or thread never sees a half-written array.
    std::lock_guard<std::mutex> lk(plan->mu);
    if (plan->code != nullptr) return CSK_OK;
    int32_t* code = nullptr;
    CSK_CUDA_TRY(cudaMalloc(&code, (plan->d + 32) * 4));
    const int64_t blocks4 = ceil_div(ceil_div(plan->d + 3, 4) + 1, 256);
    const unsigned grid = (unsigned)std::min<int64_t>(blocks4, 65535 * 4);
    cudaError_t e = cudaMemsetAsync(code + plan->d, 0, 32 * 4, st);
    if (e == cudaSuccess) {
        codes_kernel<<<grid, 256, 0, st>>>(code, plan->d, (uint32_t)plan->k1, (uint32_t)plan->seed,
                                           (uint32_t)(plan->seed >> 32), plan->row0);
        count_launch();
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaFree(code);
        set_error("materialising the codes of a hash plan failed: %s", cudaGetErrorString(e));
        return CSK_ECUDA;
    }
    plan->code = code;
    return CSK_OK;
}

}  // namespace csk

using namespace csk;

extern "C" {

csk_status cs_plan(int64_t d, int64_t k1, uint64_t seed, int64_t row0, uint32_t flags, void* stream,
                   csk_plan_t* out) {
    CSK_REQUIRE(row0 >= 0, CSK_EINVAL, "row0=%lld must be >= 0", (long long)row0);
    csk_plan_t plan = nullptr;
    csk_status s = alloc_plan(d, k1, flags, out, &plan);
    if (s != CSK_OK) return s;
    plan->seed = seed;
    plan->row0 = row0;
    cudaStream_t st = (cudaStream_t)stream;
    if (!plan->hash) {
        const int64_t blocks4 = ceil_div(ceil_div(d + 3, 4) + 1, 256);
        const unsigned grid = (unsigned)std::min<int64_t>(blocks4, 65535 * 4);
        codes_kernel<<<grid, 256, 0, st>>>(plan->code, d, (uint32_t)k1, (uint32_t)seed, (uint32_t)(seed >> 32), row0);
        count_launch();
        if (cudaGetLastError() != cudaSuccess) {
            set_error("codes_kernel launch failed");
            cs_plan_destroy(plan);
            return CSK_ECUDA;
        }
    }
    if (flags & CSK_PLAN_SORT) {
        s = build_sort(plan, st);
        if (s != CSK_OK) {
            cs_plan_destroy(plan);
            return s;
        }
    }
    *out = plan;
    return CSK_OK;
}

csk_status cs_plan_from_arrays(int64_t d, int64_t k1, const int32_t* h, const int8_t* s, uint32_t flags,
                               void* stream, csk_plan_t* out) {
    CSK_REQUIRE(h != nullptr && s != nullptr, CSK_EINVAL, "h and s must be non-NULL host arrays");
    csk_plan_t plan = nullptr;
    csk_status st_ = alloc_plan(d, k1, flags, out, &plan);
    if (st_ != CSK_OK) return st_;
    std::vector<int32_t> code((size_t)d);
    for (int64_t i = 0; i < d; ++i) {
        if (h[i] < 0 || h[i] >= k1 || (s[i] != 1 && s[i] != -1)) {
            cs_plan_destroy(plan);
            set_error("row %lld: bucket %d / sign %d out of range", (long long)i, h[i], (int)s[i]);
            return CSK_EINVAL;
        }
        code[i] = (int32_t)((uint32_t)h[i] | (s[i] < 0 ? 0x80000000u : 0u));
    }
    cudaStream_t st = (cudaStream_t)stream;
    plan->from_arrays = true;
    if (cudaMemcpyAsync(plan->code, code.data(), d * 4, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
        cudaGetLastError();
        cs_plan_destroy(plan);
        set_error("upload of forced codes failed");
        return CSK_ECUDA;
    }
    if (flags & CSK_PLAN_SORT) {
        st_ = build_sort(plan, st);
        if (st_ != CSK_OK) {
            cs_plan_destroy(plan);
            return st_;
        }
    }
    *out = plan;
    return CSK_OK;
}


csk_status cs_plan_export(csk_plan_t plan, int32_t* code, int64_t* offsets, int32_t* perm, void* stream) {
    CSK_REQUIRE(plan != nullptr, CSK_EINVAL, "plan is NULL");
    if (code) {
        const csk_status es = csk::ensure_codes(plan, (cudaStream_t)stream);
        if (es != CSK_OK) return es;
    }
    CSK_REQUIRE((offsets == nullptr && perm == nullptr) || plan->perm != nullptr, CSK_EUNSUPPORTED,
                "plan was built without CSK_PLAN_SORT");
    cudaStream_t st = (cudaStream_t)stream;
    if (code) CSK_CUDA_TRY(cudaMemcpyAsync(code, plan->code, plan->d * 4, cudaMemcpyDefault, st));
    if (offsets) CSK_CUDA_TRY(cudaMemcpyAsync(offsets, plan->offsets, (plan->k1 + 1) * 8, cudaMemcpyDefault, st));
    if (perm) CSK_CUDA_TRY(cudaMemcpyAsync(perm, plan->perm, plan->d * 4, cudaMemcpyDefault, st));
    CSK_CUDA_TRY(cudaStreamSynchronize(st));
    return CSK_OK;
}

csk_status cs_plan_info(csk_plan_t plan, int64_t* d, int64_t* k1, int64_t* row0) {
    CSK_REQUIRE(plan != nullptr, CSK_EINVAL, "plan is NULL");
    if (d) *d = plan->d;
    if (k1) *k1 = plan->k1;
    if (row0) *row0 = plan->row0;
    return CSK_OK;
}

void cs_plan_destroy(csk_plan_t plan) {
    if (!plan) return;
    cudaFree(plan->code);
    cudaFree(plan->offsets);
    cudaFree(plan->perm);
    for (auto& kv : plan->gauss64) cudaFree(kv.second);
    delete plan;
}

const char* csk_status_str(csk_status st) {
    switch (st) {
        case CSK_OK: return "CSK_OK";
        case CSK_EINVAL: return "CSK_EINVAL";
        case CSK_ESHAPE: return "CSK_ESHAPE";
        case CSK_EDTYPE: return "CSK_EDTYPE";
        case CSK_ENOMEM: return "CSK_ENOMEM";
        case CSK_ECUDA: return "CSK_ECUDA";
        case CSK_ENOTPD: return "CSK_ENOTPD";
        case CSK_ESINGULAR: return "CSK_ESINGULAR";
        case CSK_EUNSUPPORTED: return "CSK_EUNSUPPORTED";
    }
    return "CSK_UNKNOWN";
}

const char* csk_last_error(void) { return csk::last_error(); }

uint64_t csk_launch_count(int reset) {
    uint64_t v = csk::g_launches;
    if (reset) csk::g_launches = 0;
    return v;
}

const char* csk_version(void) { return "csk 0.1 (sm_100a)"; }

}  // extern "C"
