// Does DMMA (FP64 tensor) overlap with DFMA (FP64 CUDA cores) on sm_100a?
#include <cstdio>
#include <cuda_runtime.h>

template <int ND, int NF>
__global__ void mixed(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[8][2], f[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ND; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
        for (int i = 0; i < NF; ++i) f[i] = fma(a, f[i], b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
#pragma unroll
    for (int i = 0; i < 16; ++i) s += f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ND, int NF>
void run(double* out, int sms) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 20000, blocks = sms * 2, threads = 256;
    mixed<ND, NF><<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    mixed<ND, NF><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warps = double(blocks) * threads / 32;
    double fl_d = 2.0 * 256 * ND * iters * warps, fl_f = 2.0 * 32 * NF * iters * warps;
    printf("ND=%d NF=%2d: dmma %.2f TF + dfma %.2f TF = %.2f TF\n", ND, NF, fl_d / ms / 1e9, fl_f / ms / 1e9,
           (fl_d + fl_f) / ms / 1e9);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, sizeof(double) * 148 * 2 * 256 * 4);
    run<8, 0>(out, sms); run<0, 16>(out, sms); run<8, 4>(out, sms); run<8, 8>(out, sms); run<8, 16>(out, sms);
    run<4, 16>(out, sms);
    return 0;
}
