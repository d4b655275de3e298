// Microbenchmark (not product code): read a column-major d x nc fp64 matrix in
// R-row x nc-column tiles (a warp per tile, grid-stride over tiles like the CountSketch
// kernels) and reduce into a per-warp sum, to measure how the tile height and the load
// width shape the achievable HBM read bandwidth on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tile_read_bench tile_read_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int R, int VEC>
__global__ void __launch_bounds__(256) tile_read(const double* __restrict__ A, int64_t d, int nc, int64_t lda,
                                                 double* __restrict__ out) {
    // lanes: VEC doubles per lane along rows; R/VEC lanes per column; 32*VEC/R columns per instruction
    constexpr int LPC = R / VEC;            // lanes per column
    constexpr int CPI = 32 / LPC;           // columns per instruction
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t ntiles = (d + R - 1) / R;
    const int64_t gw = blockIdx.x * 8ll + warp, nw = gridDim.x * 8ll;
    double acc = 0.0;
    const int rl = (lane % LPC) * VEC, cl = lane / LPC;
    for (int64_t t = gw; t < ntiles; t += nw) {
        const int64_t r = t * R + rl;
#pragma unroll 8
        for (int c = cl; c < nc; c += CPI) {
            const double* p = A + (int64_t)c * lda + r;
            if (VEC == 2) {
                const double2 v = __ldcs(reinterpret_cast<const double2*>(p));
                acc += v.x + v.y;
            } else {
                acc += __ldcs(p);
            }
        }
    }
    if (acc == 12345.678) out[0] = acc;   // keep the loads alive
}

__global__ void plain_read(const double2* __restrict__ A, int64_t n2, double* out) {
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
        const double2 v = __ldcs(A + i);
        acc += v.x + v.y;
    }
    if (acc == 12345.678) out[0] = acc;
}

template <int R, int VEC>
void run(const char* name, const double* A, int64_t d, int nc, double* out, int blocks) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) tile_read<R, VEC><<<blocks, 256>>>(A, d, nc, d, out);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) tile_read<R, VEC><<<blocks, 256>>>(A, d, nc, d, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-28s blocks=%5d  %.3f ms  %.1f GB/s\n", name, blocks, ms, d * nc * 8.0 / ms / 1e6);
    fflush(stdout);
}

int main() {
    const int64_t d = 1ll << 24;
    const int nc = 65;
    double *A, *out;
    cudaMalloc(&A, d * nc * 8);
    cudaMalloc(&out, 8);
    cudaMemset(A, 0, d * nc * 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int occ : {1, 2, 4, 8}) {
        const int blocks = sms * occ;
        run<16, 1>("R=16 LDG.64", A, d, nc, out, blocks);
        run<32, 1>("R=32 LDG.64", A, d, nc, out, blocks);
        run<32, 2>("R=32 LDG.128", A, d, nc, out, blocks);
        run<64, 2>("R=64 LDG.128", A, d, nc, out, blocks);
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) plain_read<<<sms * 8, 256>>>((const double2*)A, d * nc / 2, out);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) plain_read<<<sms * 8, 256>>>((const double2*)A, d * nc / 2, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("plain sequential LDG.128      %.3f ms  %.1f GB/s\n", ms / 10, d * nc * 8.0 / (ms / 10) / 1e6);
    return 0;
}
