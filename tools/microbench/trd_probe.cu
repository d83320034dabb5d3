// trd_probe.cu -- where a step of k_sytrd4 (eigsmall.cu) spends its cycles: per-phase
// clock64 sums of one thread (H = reflector + barrier, S = p sweep, S-bar, P = p / K / w,
// U = update sweep, U-bar), n = 200.
#include <cstdio>
#include <vector>
__device__ long long trd_probe_out[6];
#include "eigsmall.cu"
namespace farqb {
bool pdl_enabled() { return false; }
void gemm(bool, int64_t, int64_t, int64_t, double, const double*, int64_t, const double*, int64_t, double, double*,
          int64_t, GemmWorkspace&, int, cudaStream_t, LaunchCounter&) {}   // unused here
}
int main() {
    const int n = 200;
    std::vector<double> h(size_t(n) * n);
    srand(1);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) h[size_t(j) * n + i] = h[size_t(i) * n + j] = double(rand()) / RAND_MAX - 0.5;
    double *m, *d, *e, *tau, *vh;
    cudaMalloc(&m, 8 * n * n); cudaMalloc(&d, 8 * n); cudaMalloc(&e, 8 * n); cudaMalloc(&tau, 8 * n); cudaMalloc(&vh, 8 * n * n);
    cudaMemcpy(m, h.data(), 8 * n * n, cudaMemcpyHostToDevice);
    const size_t smem4 = sizeof(double) * size_t(n * (n + 1) / 2 + 4 * 224 + farqb::kTrd4Warps * 224 + 224);
    cudaFuncSetAttribute(farqb::k_sytrd5, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem4));
    for (int r = 0; r < 3; ++r) farqb::k_sytrd5<<<1, farqb::kTrd4Warps * 32, smem4>>>(m, n, d, e, tau, vh);
    cudaDeviceSynchronize();
    long long t[6];
    cudaMemcpyFromSymbol(t, trd_probe_out, sizeof t);
    const char* nm[6] = {"P (p,K,w)", "L (col+refl)", "F sweep", "F bar", "-", "-"};
    long long tot = 0;
    for (int x = 0; x < 6; ++x) tot += t[x];
    for (int x = 0; x < 6; ++x) printf("%-10s %8.0f cycles/step  %5.1f%%\n", nm[x], double(t[x]) / (n - 2), 100.0 * t[x] / tot);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
