// Timeline of the small-solve kernel (csrc/qr_wy.cu built with CSK_QR_PROFILE): per panel step,
// clock64 stamps of the panel team and of a trailing-update warp in every CTA.
// Build (here):  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//   scripts/qr_wy_prof.cu -o scripts/qr_wy_prof -L paper_2508_14209_b200 -lcsk \
//   -Xlinker -rpath='$ORIGIN/../paper_2508_14209_b200'
// Run (GPU):     scripts/qr_wy_prof 512 256
#define CSK_QR_PROFILE
#include "../paper_2508_14209_b200/csrc/qr_wy.cu"

#include <cstdio>
#include <random>
#include <vector>

int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 512, n = argc > 2 ? atoi(argv[2]) : 256, nc = n + 1;
    const int npan = (nc + 3) / 4;
    std::vector<double> Z((size_t)m * nc);
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    for (auto& v : Z) v = nd(g);
    double *dZ, *dR, *dS, *dx;
    csk::SolveStatus* dst;
    long long* dp;
    const size_t profn = (size_t)16 * (npan + 1) * 8;
    cudaMalloc(&dZ, Z.size() * 8);
    cudaMalloc(&dR, (size_t)(nc + 1) * nc * 8);
    cudaMalloc(&dS, csk::qr_wy_scratch_doubles(m, nc) * 8);
    cudaMalloc(&dx, n * 8);
    cudaMalloc(&dst, sizeof(csk::SolveStatus));
    cudaMalloc(&dp, profn * 8);
    cudaMemcpy(dZ, Z.data(), Z.size() * 8, cudaMemcpyHostToDevice);
    csk::qr_wy_prof_buffer = dp;
    bool launched = false;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 4; ++it) {
        cudaMemset(dp, 0, profn * 8);
        cudaEventRecord(e0);
        csk::qr_wy_launch(dZ, m, m, nc, dR, (nc + 1) & ~1, dS, dx, dst, 0, &launched);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> pr(profn);
    cudaMemcpy(pr.data(), dp, profn * 8, cudaMemcpyDeviceToHost);
    int P = 0;
    for (int r = 0; r < 16; ++r)
        if (pr[((size_t)r * (npan + 1) + npan) * 8 + 0] != 0) P = r + 1;
    printf("m=%d n=%d launched=%d P=%d npan=%d kernel %.1f us (%s)\n", m, n, launched, P, npan, ms * 1e3,
           cudaGetErrorString(cudaGetLastError()));
    auto at = [&](int r, int k, int s) { return pr[((size_t)r * (npan + 1) + k) * 8 + s]; };
    const long long base = at(0, npan, 0);
    printf("rank0: load %lld  prologue factor %lld  (cycles)\n", at(0, npan, 1) - base, at(0, npan, 2) - at(0, npan, 1));
    double sum_step = 0, sum_stage = 0, sum_fac = 0, sum_upd0 = 0, sum_upd7 = 0, sum_upd7o = 0;
    int cnt = 0;
    printf("  k  own(k+1) step  stage factor upd(team) upd(w7) | other-CTA upd(w7)\n");
    for (int k = 0; k + 1 < npan; ++k) {
        const int o = (k + 1) % P, oth = (o + 1) % P;
        const long long step = at(o, k + 1, 0) - at(o, k, 0);
        const long long stage = at(o, k, 1) - at(o, k, 0);
        const long long fac = at(o, k, 2) - at(o, k, 1);
        const long long upd0 = at(o, k, 3) - at(o, k, 2);
        const long long upd7 = at(o, k, 5) - at(o, k, 4);
        const long long upd7o = at(oth, k, 5) - at(oth, k, 4);
        if (k < 6 || k % 16 == 0)
            printf("%3d %3d %7lld %6lld %6lld %7lld %7lld | %7lld\n", k, o, step, stage, fac, upd0, upd7, upd7o);
        sum_step += step;
        sum_stage += stage;
        sum_fac += fac;
        sum_upd0 += upd0;
        sum_upd7 += upd7;
        sum_upd7o += upd7o;
        ++cnt;
    }
    printf("mean    step %.0f stage %.0f factor %.0f upd(team) %.0f upd(w7) %.0f other upd(w7) %.0f\n",
           sum_step / cnt, sum_stage / cnt, sum_fac / cnt, sum_upd0 / cnt, sum_upd7 / cnt, sum_upd7o / cnt);
    printf("final sync -> backsub %lld cycles; total rank0 %lld cycles\n", at(0, npan, 4) - at(0, npan, 3),
           at(0, npan, 4) - base);
    return 0;
}
