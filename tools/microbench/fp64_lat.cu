// fp64_lat.cu -- dependent-chain latency of DFMA / DMUL / FP64 division / sqrt / LDS / bar.sync
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_lat tools/microbench/fp64_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k_chain(double* out, double x, int n, long long* cyc) {
    __shared__ double sh[64];
    double a = x + threadIdx.x, b = 1.0000001;
    sh[threadIdx.x & 63] = a;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (OP == 0) a = fma(a, b, 1e-30);
        if (OP == 1) a = a * b;
        if (OP == 2) a = 1.0 / a + 1.0;
        if (OP == 3) a = sqrt(a) + 1.0;
        if (OP == 4) a = sh[(int(a) + i) & 63] + 1.0;
        if (OP == 5) { __syncthreads(); a += 1.0; }
        if (OP == 6) a = __drcp_rn(a) + 1.0;
        if (OP == 7) a = __fmaf_rn(float(a), 1.0000001f, 1e-30f);
    }
    const long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int OP>
void run(const char* name, int threads) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8 * 1024);
    cudaMalloc(&cyc, 8);
    const int n = 4096;
    k_chain<OP><<<1, threads>>>(out, 1.5, n, cyc);
    k_chain<OP><<<1, threads>>>(out, 1.5, n, cyc);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s threads %4d: %.1f cycles per op\n", name, threads, double(h) / n);
}

int main() {
    for (int t : {32, 416}) {
        run<0>("DFMA", t);
        run<1>("DMUL", t);
        run<2>("1.0/x + 1 (FP64 div)", t);
        run<6>("__drcp_rn + 1", t);
        run<3>("sqrt + 1", t);
        run<4>("LDS -> DADD", t);
        run<5>("bar.sync + DADD", t);
        run<7>("FFMA (fp32 ref)", t);
    }
    return 0;
}
