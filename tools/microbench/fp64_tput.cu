// fp64_tput.cu -- CUDA-core throughput (not latency) of DFMA, DMUL, FFMA, IMAD, LDS.64 per SM
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_tput tools/microbench/fp64_tput.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k_tput(double* out, int n, long long* cyc) {
    __shared__ double sh[1024];
    sh[threadIdx.x] = threadIdx.x;
    __syncthreads();
    double a[8];
    float f[8];
    int ii[8];
    for (int q = 0; q < 8; ++q) { a[q] = threadIdx.x + q; f[q] = a[q]; ii[q] = threadIdx.x + q; }
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (OP == 0) a[q] = fma(a[q], 1.0000001, 1e-9);
            if (OP == 1) f[q] = __fmaf_rn(f[q], 1.0000001f, 1e-9f);
            if (OP == 2) ii[q] = ii[q] * 3 + 1;
            if (OP == 3) a[q] += sh[(threadIdx.x + q * 33 + i) & 1023];
        }
    }
    const long long t1 = clock64();
    double s = 0;
    for (int q = 0; q < 8; ++q) s += a[q] + f[q] + ii[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int OP>
void run(const char* name) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8 * 148 * 1024);
    cudaMalloc(&cyc, 8);
    const int n = 2048;
    k_tput<OP><<<148, 1024>>>(out, n, cyc);
    k_tput<OP><<<148, 1024>>>(out, n, cyc);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double ops_per_sm = 1024.0 * 8 * n;
    printf("%-10s: %.1f ops / clk / SM (lane ops)\n", name, ops_per_sm / double(h));
}

int main() {
    run<0>("DFMA");
    run<1>("FFMA");
    run<2>("IMAD");
    run<3>("LDS+DADD");
    return 0;
}
