#include <cstdio>
__global__ void k_a(double* out, int b, int mode) {
    __shared__ double pr[2][128];
    double v = threadIdx.x * 1e-3 + 1.0, acc = 0;
    for (int j = 0; j < b; ++j) {
        double* p = pr[j & 1];
        if (threadIdx.x < 64) p[threadIdx.x] = v + j;
        __syncthreads();
        const double d = p[j % 64];
        double invd;
        if (mode == 0) invd = 1.0 / d;
        else if (mode == 1) invd = __drcp_rn(d);
        else invd = d * 0.5;
        v = fma(-invd, p[threadIdx.x & 63], v);
        acc += v;
    }
    out[threadIdx.x] = acc;
}
int main() {
    double* o; cudaMalloc(&o, 8 * 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) for (int th : {32, 128, 416, 1024}) {
        k_a<<<1, th>>>(o, 50, mode);
        cudaEventRecord(e0);
        for (int r = 0; r < 100; ++r) k_a<<<1, th>>>(o, 50, mode);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("mode %d threads %4d: %.2f us per kernel (50 steps)\n", mode, th, ms * 10);
    }
}
