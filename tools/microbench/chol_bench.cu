// chol_bench.cu -- time the b x b Cholesky + inverse kernels of smallla.cu in isolation.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2506_03859_b200/csrc \
//        -o tools/microbench/chol_bench tools/microbench/chol_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#ifdef FQB_CHOL_PROBE
__device__ long long g_stamps[512];
__device__ __forceinline__ void chol_probe_stamp(int k) { g_stamps[k] = clock64(); }
#endif
#include "smallla.cu"

namespace farqb {
bool pdl_enabled() { return false; }   // engine.cu owns the real switch
}

int main(int argc, char** argv) {
  for (int b : {16, 32, 50, 64, 100, 128}) {
    const int reps = 200;
    std::vector<double> h(size_t(b) * b), w(size_t(b) * 4 * b);
    srand(1);
    for (auto& x : w) x = double(rand()) / RAND_MAX - 0.5;
    for (int i = 0; i < b; ++i)
        for (int j = 0; j < b; ++j) {
            double s = 0;
            for (int k = 0; k < 4 * b; ++k) s += w[size_t(i) * 4 * b + k] * w[size_t(j) * 4 * b + k];
            h[size_t(j) * b + i] = s;
        }
    double *S, *R, *Ri, *md, *scratch;
    unsigned* st;
    cudaMalloc(&S, sizeof(double) * b * b);
    cudaMalloc(&R, sizeof(double) * b * b);
    cudaMalloc(&Ri, sizeof(double) * b * b);
    cudaMalloc(&md, sizeof(double));
    cudaMalloc(&scratch, sizeof(double) * b * (b + 1));
    cudaMalloc(&st, sizeof(unsigned));
    cudaMemset(st, 0, sizeof(unsigned));
    cudaMemcpy(S, h.data(), sizeof(double) * b * b, cudaMemcpyHostToDevice);
    farqb::LaunchCounter lc;
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int i = 0; i < 10; ++i)
        farqb::launch_chol_upper_inv(S, b, b, 1e-12, 0.0, nullptr, 0, R, Ri, md, scratch, st, 1, s, lc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int i = 0; i < reps; ++i)
        farqb::launch_chol_upper_inv(S, b, b, 1e-12, 0.0, nullptr, 0, R, Ri, md, scratch, st, 1, s, lc);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    // check R' R = S and R Ri = I
    std::vector<double> hr(size_t(b) * b), hri(size_t(b) * b);
    cudaMemcpy(hr.data(), R, sizeof(double) * b * b, cudaMemcpyDeviceToHost);
    cudaMemcpy(hri.data(), Ri, sizeof(double) * b * b, cudaMemcpyDeviceToHost);
    double e1max = 0, e2max = 0;
    for (int i = 0; i < b; ++i)
        for (int j = 0; j < b; ++j) {
            double s1 = 0, s2 = 0;
            for (int k = 0; k < b; ++k) {
                s1 += hr[size_t(i) * b + k] * hr[size_t(j) * b + k];   // (R'R)_ij = sum_k R_ki R_kj
                s2 += hr[size_t(k) * b + i] * hri[size_t(j) * b + k];  // (R Ri)_ij
            }
            e1max = std::max(e1max, std::abs(s1 - h[size_t(j) * b + i]));
            e2max = std::max(e2max, std::abs(s2 - (i == j)));
        }
    unsigned hst = 0;
    cudaMemcpy(&hst, st, sizeof(unsigned), cudaMemcpyDeviceToHost);
    printf("b=%d: %.2f us per factorization  |R'R-S|=%.2e |R Ri - I|=%.2e status=%u  (%s)\n", b, 1e3 * ms / reps,
           e1max, e2max, hst, cudaGetErrorString(cudaGetLastError()));
#ifdef FQB_CHOL_PROBE
    long long hs[512];
    cudaMemcpyFromSymbol(hs, g_stamps, sizeof hs);
    double work = 0, wait = 0;
    for (int j = 1; j < b; ++j) { work += hs[2 * j] - hs[2 * j - 1]; wait += hs[2 * j + 1] - hs[2 * j]; }
    printf("   thread %d: per step %.0f cycles of work, %.0f cycles at the barrier\n", FQB_CHOL_PROBE, work / (b - 1), wait / (b - 1));
#endif
  }
    return 0;
}
