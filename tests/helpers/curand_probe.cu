// Test-only probe: cuRAND's Philox4x32-10 (a library routine) for pinning the
// oracle's Philox on the GPU.  curand_init(seed, subsequence 0, offset 4q) then
// curand4() returns Philox(ctr = (lo32 q, hi32 q, 0, 0), key = seed).
#include <cstdint>
#include <curand_kernel.h>

__global__ void probe(uint64_t seed, const uint64_t* q, uint4* out, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    curandStatePhilox4_32_10_t st;
    curand_init(seed, 0ull, 4ull * q[i], &st);
    out[i] = curand4(&st);
}

extern "C" int curand_probe(uint64_t seed, const uint64_t* q_host, uint32_t* out_host, int n) {
    uint64_t* q; uint4* o;
    if (cudaMalloc(&q, n * 8) != cudaSuccess || cudaMalloc(&o, n * 16) != cudaSuccess) return 1;
    cudaMemcpy(q, q_host, n * 8, cudaMemcpyHostToDevice);
    probe<<<(n + 127) / 128, 128>>>(seed, q, o, n);
    cudaMemcpy(out_host, o, n * 16, cudaMemcpyDeviceToHost);
    cudaFree(q); cudaFree(o);
    return cudaGetLastError() != cudaSuccess;
}
