// Microbenchmarks behind the CountSketch dataflow decisions:
//   bulk   : the reduce path alone -- one cp.reduce.async.bulk .add.{f64,f32} of a ROWB-byte row per
//            sketch row into a random bucket row of an L2-resident k1-row table (what the B kernels
//            do, without the A loads); rows/s and sector-RMW/s for fp64 and fp32 rows
//   dsmem  : red.shared::cluster.add.f64 to random words of a cluster's distributed bucket table
//            (the cluster-privatised alternative of VERDICT r1 #5), ops/clk/SM
//   redg   : the same rows reduced by warp-wide red.global (16-B .v4.f32 or scalar .f64) from the LSU,
//            alone and mixed with the bulk path (a fraction of the rows on each engine)
//   smem   : private shared-memory buckets, random fp64 read-add-write (no atomics; one warp per
//            array) -- the per-SM scatter rate of the privatised variant
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2red_bench l2red_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <bool F32>
__global__ void __launch_bounds__(256, 1) bulk_kernel(char* table, int k1, int rowb, int64_t rows, int ldrow) {
    extern __shared__ __align__(16) char sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    char* row = sm + (warp * 32 + lane) * ldrow;
    for (int i = 0; i < rowb / 4; ++i) reinterpret_cast<float*>(row)[i] = F32 ? 1.0f : 0.0f;
    if (!F32) for (int i = 0; i < rowb / 8; ++i) reinterpret_cast<double*>(row)[i] = 1.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    const uint32_t src = (uint32_t)__cvta_generic_to_shared(row);
    for (int64_t u = blockIdx.x * 8 + warp; u * 32 < rows; u += nwarps) {
        const int64_t r = u * 32 + lane;
        if (r < rows) {
            const uint32_t m = ((uint64_t)mix((uint32_t)r) * (uint32_t)k1) >> 32;
            char* dst = table + (int64_t)m * ldrow;
            if (F32)
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
                             "r"(src), "r"(rowb) : "memory");
            else
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(dst),
                             "r"(src), "r"(rowb) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// LSU path: rows reduced by warp-wide red.global (REDG) instead of the TMA engine.  VEC = 4: 16-B
// red.global.add.v4.f32 chunks (REDG.E.ADD.F32x4), VEC = 1: scalar red.global.add.f64.  Each warp
// covers 32 rows per iteration, item e = it * 32 + lane -> (row e / cpr, chunk e % cpr).
// MIX > 0: rows with (r % 8) < MIX go through the bulk path instead (both engines at once).
template <int VEC, int MIX>
__global__ void __launch_bounds__(256, 1) redg_kernel(char* table, int k1, int rowb, int64_t rows, int ldrow) {
    extern __shared__ __align__(16) char sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    char* row = sm + (warp * 32 + lane) * ldrow;
    for (int i = 0; i < rowb / 4; ++i) reinterpret_cast<float*>(row)[i] = 1.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const uint32_t src = (uint32_t)__cvta_generic_to_shared(row);
    const int cb = VEC == 4 ? 16 : 8;
    const int cpr = rowb / cb;   // chunks per row
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    for (int64_t u = blockIdx.x * 8 + warp; u * 32 < rows; u += nwarps) {
        const int64_t rb = u * 32;
        if (MIX > 0) {
            const int64_t r = rb + lane;
            if ((lane & 7) < MIX && r < rows) {
                const uint32_t m = ((uint64_t)mix((uint32_t)r) * (uint32_t)k1) >> 32;
                char* dst = table + (int64_t)m * ldrow;
                if (VEC == 4)
                    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
                                 "r"(src), "r"(rowb) : "memory");
                else
                    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(dst),
                                 "r"(src), "r"(rowb) : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
        }
        for (int e = lane; e < 32 * cpr; e += 32) {
            const int rr = e / cpr, ch = e - rr * cpr;
            const int64_t r = rb + rr;
            if (r >= rows || (MIX > 0 && (rr & 7) < MIX)) continue;
            const uint32_t m = ((uint64_t)mix((uint32_t)r) * (uint32_t)k1) >> 32;
            char* dst = table + (int64_t)m * ldrow + ch * cb;
            if (VEC == 4)
                asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(1.0f), "f"(1.0f),
                             "f"(1.0f), "f"(1.0f) : "memory");
            else
                asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(dst), "d"(1.0) : "memory");
        }
    }
    if (MIX > 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// cluster of CL CTAs, each owning k1/CL fp64 buckets of one column in shared memory; every thread adds
// `per_thread` values to random buckets of the cluster (remote with probability (CL-1)/CL)
template <int CL>
__global__ void __launch_bounds__(256, 1) dsmem_kernel(int k1, int per_thread, double* out) {
    extern __shared__ __align__(16) double bk[];
    cg::cluster_group cl = cg::this_cluster();
    const int per = k1 / CL;
    for (int i = threadIdx.x; i < per; i += blockDim.x) bk[i] = 0.0;
    cl.sync();
    uint32_t x = mix(blockIdx.x * 1024 + threadIdx.x + 1);
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(bk);
    for (int i = 0; i < per_thread; ++i) {
        x = mix(x + i);
        const uint32_t m = ((uint64_t)x * (uint32_t)k1) >> 32;
        const uint32_t rank = m / per, off = m - rank * per;
        uint32_t addr;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(base + off * 8), "r"(rank));
        asm volatile("red.shared::cluster.add.f64 [%0], %1;" ::"r"(addr), "d"(1.0) : "memory");
    }
    cl.sync();
    if (threadIdx.x == 0) out[blockIdx.x] = bk[0];
}

// private buckets: warp w owns array w (k1 doubles); each lane does read-add-write of a random bucket
// (lanes of a warp use distinct buckets here: the duplicate case is handled apart in a real kernel)
__global__ void __launch_bounds__(128, 1) smem_kernel(int k1, int per_lane, double* out) {
    extern __shared__ __align__(16) double arr[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* a = arr + (size_t)warp * k1;
    for (int i = lane; i < k1; i += 32) a[i] = 0.0;
    __syncwarp();
    uint32_t x = mix(blockIdx.x * 1024 + threadIdx.x + 7);
    for (int i = 0; i < per_lane; ++i) {
        x = mix(x + i);
        const uint32_t m = (((uint64_t)x * (uint32_t)(k1 / 32)) >> 32) * 32 + lane;   // distinct per lane
        a[m] += 1.0;
    }
    __syncwarp();
    if (lane == 0) out[blockIdx.x * 4 + warp] = a[0];
}

int main(int argc, char** argv) {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    const int64_t rows = 1 << 24;
    const int k1 = 8192;
    char* table;
    cudaMalloc(&table, (size_t)k1 * 1024);
    cudaMemset(table, 0, (size_t)k1 * 1024);
    struct Case { bool f32; int rowb, ldrow; const char* name; };
    Case cases[] = {{false, 528, 544, "f64 65+1 cols (528 B, 17 sectors)"},
                    {false, 512, 544, "f64 64 cols (512 B, 16 sectors)"},
                    {true, 272, 288, "f32 65+3 cols (272 B, 9 sectors)"},
                    {true, 256, 288, "f32 64 cols (256 B, 8 sectors)"},
                    {false, 256, 288, "f64 32 cols (256 B, 8 sectors)"},
                    {true, 128, 144, "f32 32 cols (128 B, 4 sectors)"}};
    for (auto& c : cases) {
        const size_t smem = 256 * (size_t)c.ldrow;
        auto k = c.f32 ? bulk_kernel<true> : bulk_kernel<false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            k<<<nsm, 256, smem>>>(table, k1, c.rowb, rows, c.ldrow);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        const double sectors = (double)rows * ((c.rowb + 31) / 32);
        printf("bulk %-36s %8.3f ms  %7.2f Grows/s  %7.1f Gsector/s  %7.2f TB/s payload\n", c.name, ms,
               rows / ms / 1e6, sectors / ms / 1e6, rows * (double)c.rowb / ms / 1e9);
    }
    {   // same fp64 528-B rows into larger tables (k1 x 544 B: 4.5 / 17.8 / 35.7 / 71 MB): is the rate limited
        // by contention on the table's lines (then spread copies of SA^T would help at C2) or by the slices?
        char* big;
        cudaMalloc(&big, (size_t)131072 * 544);
        cudaMemset(big, 0, (size_t)131072 * 544);
        const size_t smem = 256 * (size_t)544;
        cudaFuncSetAttribute(bulk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int kk : {2048, 8192, 32768, 65536, 131072}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                bulk_kernel<false><<<nsm, 256, smem>>>(big, kk, 528, rows, 544);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            cudaEventElapsedTime(&ms, e0, e1);
            printf("bulk f64 528-B rows, table k1 = %6d (%6.1f MB): %8.3f ms  %7.2f TB/s payload\n", kk, kk * 544 / 1e6, ms,
                   rows * 528.0 / ms / 1e9);
        }
        cudaFree(big);
    }
    {
        struct RCase { void (*k)(char*, int, int, int64_t, int); int rowb, ldrow; const char* name; };
        RCase rc[] = {{redg_kernel<4, 0>, 272, 288, "REDG.F32x4 f32 68 cols (272 B)"},
                      {redg_kernel<4, 2>, 272, 288, "mix f32: 2/8 rows bulk, 6/8 REDG.F32x4"},
                      {redg_kernel<4, 4>, 272, 288, "mix f32: 4/8 rows bulk, 4/8 REDG.F32x4"},
                      {redg_kernel<4, 6>, 272, 288, "mix f32: 6/8 rows bulk, 2/8 REDG.F32x4"},
                      {redg_kernel<1, 0>, 528, 544, "REDG.F64 f64 66 cols (528 B)"},
                      {redg_kernel<1, 6>, 528, 544, "mix f64: 6/8 rows bulk, 2/8 REDG.F64"}};
        for (auto& c : rc) {
            const size_t smem = 256 * (size_t)c.ldrow;
            cudaFuncSetAttribute(c.k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                c.k<<<nsm, 256, smem>>>(table, k1, c.rowb, rows, c.ldrow);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            cudaEventElapsedTime(&ms, e0, e1);
            printf("redg %-40s %8.3f ms  %7.2f Grows/s  %7.2f TB/s payload  err=%s\n", c.name, ms, rows / ms / 1e6,
                   rows * (double)c.rowb / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    }
    double* out;
    cudaMalloc(&out, 4096 * 8);
    {
        const int per_thread = 4096;
        auto k = dsmem_kernel<8>;
        const size_t smem = (size_t)k1 / 8 * 8 * 8;   // 8 columns' worth of buckets per CTA
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((nsm / 8) * 8);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 8;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            cudaLaunchKernelEx(&cfg, k, k1 * 8, per_thread, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)cfg.gridDim.x * 256 * per_thread;
        int clk = 0;
        cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        printf("dsmem red.shared::cluster.add.f64 (cluster 8): %8.3f ms  %7.2f Gops/s  %.3f ops/clk/SM (at %d MHz)  err=%s\n",
               ms, ops / ms / 1e6, ops / (ms * 1e-3) / ((double)cfg.gridDim.x * clk * 1e3), clk / 1000,
               cudaGetErrorString(cudaGetLastError()));
    }
    {
        const int per_lane = 8192;
        const size_t smem = (size_t)4 * k1 * 8;   // 4 warps x k1 doubles = 256 KB at k1 = 8192: too big
        const int kk = 6144;                       // 4 x 6144 x 8 = 192 KB
        (void)smem;
        cudaFuncSetAttribute(smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kk * 8);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            smem_kernel<<<nsm, 128, 4 * kk * 8>>>(kk, per_lane, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)nsm * 128 * per_lane;
        int clk = 0;
        cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        printf("smem private fp64 read-add-write (4 warps/SM): %8.3f ms  %7.2f Gops/s  %.3f elem/clk/SM  err=%s\n", ms,
               ops / ms / 1e6, ops / (ms * 1e-3) / ((double)nsm * clk * 1e3), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
