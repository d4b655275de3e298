// Latency microbenchmarks for the small-solve design (one warp unless stated): dependent chains of
// DFMA, DADD, 64-bit butterfly shuffle + add, LDS, shared atomicAdd, fp64 sqrt and division,
// named barrier (4 warps), __syncthreads (8 warps), cluster barrier (P CTAs).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/lat_bench.cu -o scripts/lat_bench
#include <cooperative_groups.h>
#include <cstdio>

constexpr int N = 4096;

__global__ void k_dfma(double* out, long long* cyc, double a, double b) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = x;
}
__global__ void k_dadd(double* out, long long* cyc, double a, double b) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = x + b;
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = x;
}
__global__ void k_shfl(double* out, long long* cyc, double a, double b) {
    double x = a + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1 << (i & 4));
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = x;
}
__global__ void k_lds(double* out, long long* cyc, double a, double b) {
    __shared__ int s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 1) & 1023;
    __syncwarp();
    int p = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) p = s[p];
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = p;
}
__global__ void k_atoms(double* out, long long* cyc, double a, double b) {
    __shared__ int c;
    if (threadIdx.x == 0) c = 0;
    __syncwarp();
    int q = 0;
    long long t0 = clock64();
    for (int i = 0; i < N / 16; ++i) {
        if ((threadIdx.x & 31) == 0) q = atomicAdd(&c, 1 + (q & 0));
        q = __shfl_sync(0xffffffffu, q, 0);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 16;
    out[threadIdx.x] = q;
}
__global__ void k_sqrt(double* out, long long* cyc, double a, double b) {
    double x = a + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N / 16; ++i) x = sqrt(x) + b;
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 16;
    out[threadIdx.x] = x;
}
__global__ void k_div(double* out, long long* cyc, double a, double b) {
    double x = a + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N / 16; ++i) x = b / x + 1.0;
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 16;
    out[threadIdx.x] = x;
}
__global__ void k_namedbar(double* out, long long* cyc, double a, double b) {
    long long t0 = clock64();
    for (int i = 0; i < N / 16; ++i) asm volatile("bar.sync 1, 128;" ::: "memory");
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 16;
}
__global__ void k_sync(double* out, long long* cyc, double a, double b) {
    long long t0 = clock64();
    for (int i = 0; i < N / 16; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 16;
}
__global__ void k_clsync(double* out, long long* cyc, double a, double b) {
    auto cl = cooperative_groups::this_cluster();
    long long t0 = clock64();
    for (int i = 0; i < N / 16; ++i) cl.sync();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0) * 16;
}
// one warp: red of 8 doubles through the full butterfly (the per-column team reduction's first half)
__global__ void k_bfly8(double* out, long long* cyc, double a, double b) {
    double v[8];
    for (int i = 0; i < 8; ++i) v[i] = a * (threadIdx.x + i);
    long long t0 = clock64();
    for (int it = 0; it < N / 16; ++it) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
        v[0] *= b;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 16;
    double s = 0;
    for (int i = 0; i < 8; ++i) s += v[i];
    out[threadIdx.x] = s;
}

typedef void (*K)(double*, long long*, double, double);

static void run(const char* name, K k, int threads, int cluster = 0) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 4096 * 8);
    cudaMalloc(&cyc, 8);
    for (int rep = 0; rep < 2; ++rep) {
        if (cluster) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cluster);
            cfg.blockDim = dim3(threads);
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = cluster;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            if (cluster > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaLaunchKernelEx(&cfg, k, out, cyc, 1.0000001, 1e-9);
        } else {
            k<<<1, threads>>>(out, cyc, 1.0000001, 1e-9);
        }
        cudaDeviceSynchronize();
    }
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-34s %8.1f cycles per op  (%s)\n", name, (double)c / N, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run("DFMA dependent (1 warp)", k_dfma, 32);
    run("DADD dependent (1 warp)", k_dadd, 32);
    run("SHFL.BFLY f64 + DADD (1 warp)", k_shfl, 32);
    run("LDS pointer chase (1 warp)", k_lds, 32);
    run("ATOMS.ADD + SHFL bcast (1 warp)", k_atoms, 32);
    run("sqrt(f64) + add (1 warp)", k_sqrt, 32);
    run("f64 division + add (1 warp)", k_div, 32);
    run("8-value butterfly (5 levels)", k_bfly8, 32);
    run("bar.sync 1,128 (4 warps)", k_namedbar, 128);
    run("__syncthreads (8 warps)", k_sync, 256);
    run("__syncthreads (16 warps)", k_sync, 512);
    run("cluster.sync P=2 (8 warps)", k_clsync, 256, 2);
    run("cluster.sync P=8 (8 warps)", k_clsync, 256, 8);
    run("cluster.sync P=16 (8 warps)", k_clsync, 256, 16);
    return 0;
}
