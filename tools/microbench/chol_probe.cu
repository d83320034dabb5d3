// chol_probe.cu -- where the time of the b x b Cholesky (k_chol_inv_reg, smallla.cu) goes:
// globaltimer stamps at the phase boundaries of a copy of the kernel, per launch.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/chol_probe tools/microbench/chol_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int kSmemMaxB = 128;

template <int MAXS, int VARIANT>
__global__ void __launch_bounds__(1024) k_probe(const double* __restrict__ S, int b, int64_t lds, double tol,
                                                double* __restrict__ R, double* __restrict__ Rinv,
                                                unsigned long long* stamps) {
    const unsigned long long t0 = gtime();
    extern __shared__ double smem[];
    __shared__ double prow[2][kSmemMaxB];
    __shared__ double pinv[2];
    __shared__ double sd[kSmemMaxB];
    __shared__ double red[32];
    constexpr int RG = 8;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int c = tid % b, rg = tid / b;
    const bool active = tid < RG * b;
    double v[MAXS];
#pragma unroll
    for (int s = 0; s < MAXS; ++s) {
        const int i = rg + s * RG;
        v[s] = (active && i < b) ? S[int64_t(c) * lds + i] : 0.0;
    }
    double local = 0.0;
    for (int i = tid; i < b; i += nt) local = fmax(local, S[int64_t(i) * lds + i]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) local = fmax(local, __shfl_down_sync(0xffffffffu, local, off));
    if ((tid & 31) == 0) red[tid >> 5] = local;
    __syncthreads();
    double max_diag = 0.0;
    for (int w = 0; w < (nt >> 5); ++w) max_diag = fmax(max_diag, red[w]);
    const double thresh = tol * max_diag;
    const unsigned long long t1 = gtime();
    bool failed = false;
    if (VARIANT == 4) {
        // branch-free steps: all slot loads first, selects instead of branches, one
        // STS for the publication (no jump table)
        for (int j = 0; j < b; ++j) {
            double* pr = prow[j & 1];
            if (active && rg == (j % RG)) {
                const int sj = j / RG;
                double val = v[0];
#pragma unroll
                for (int s = 1; s < MAXS; ++s) val = s == sj ? v[s] : val;
                pr[c] = val;
            }
            __syncthreads();
            const double d = pr[j];
            if (!(d > thresh)) { failed = true; break; }
            double pv[MAXS];
#pragma unroll
            for (int s = 0; s < MAXS; ++s) pv[s] = pr[min(rg + s * RG, b - 1)];
            const double pc = pr[c];
            const double invd = 1.0 / d;
            const bool diag_col = c == j;
#pragma unroll
            for (int s = 0; s < MAXS; ++s) {
                const int i = rg + s * RG;
                const double f = pv[s] * invd;
                const double nv = diag_col ? -f : fma(-f, pc, v[s]);
                v[s] = (i > j && i < b) ? nv : v[s];
            }
        }
    } else if (VARIANT == 0 || VARIANT == 2 || VARIANT == 3) {
        for (int j = 0; j < b; ++j) {
            double* pr = prow[j & 1];
            if (active && rg == (j % RG)) {
                const int sj = j / RG;
#pragma unroll
                for (int s = 0; s < MAXS; ++s)
                    if (s == sj) pr[c] = v[s];
            }
            __syncthreads();
            const double d = pr[j];
            if (!(d > thresh)) { failed = true; break; }
            // probes: 2 = no division, 3 = no update (barrier + publication only)
            const double invd = VARIANT == 2 ? 0.5 : 1.0 / d;
            const double pc = pr[c];
            if (active && VARIANT != 3) {
#pragma unroll
                for (int s = 0; s < MAXS; ++s) {
                    const int i = rg + s * RG;
                    if (i > j && i < b) {
                        const double f = pr[i] * invd;
                        v[s] = c == j ? -f : fma(-f, pc, v[s]);
                    }
                }
            }
        }
    } else {
        // VARIANT 1: the owner of the next pivot publishes 1/d with the row; row j+1 is
        // updated first so the publication leaves the step as early as possible
        if (active && rg == 0) {
            prow[0][c] = v[0];
            if (c == 0) pinv[0] = 1.0 / v[0];
        }
        __syncthreads();
        for (int j = 0; j < b; ++j) {
            const double* pr = prow[j & 1];
            double* nx = prow[(j + 1) & 1];
            const double d = pr[j];
            if (!(d > thresh)) { failed = true; break; }
            const double invd = pinv[j & 1];
            const double pc = pr[c];
            if (active) {
                const int jn = j + 1;
                const int sn = jn / RG;
#pragma unroll
                for (int s = 0; s < MAXS; ++s) {
                    const int i = rg + s * RG;
                    if (i > j && i < b) {
                        const double f = pr[i] * invd;
                        v[s] = c == j ? -f : fma(-f, pc, v[s]);
                        if (i == jn) {
                            nx[c] = v[s];
                            if (c == jn) pinv[jn & 1] = 1.0 / v[s];
                        }
                    }
                }
                (void)sn;
            }
            __syncthreads();
        }
    }
    const unsigned long long t2 = gtime();
    const int ld = b + 1;
    if (!failed) {
        if (active) {
#pragma unroll
            for (int s = 0; s < MAXS; ++s) {
                const int i = rg + s * RG;
                if (i < b) smem[i * ld + c] = v[s];
            }
        }
        __syncthreads();
        for (int i = tid; i < b; i += nt) sd[i] = sqrt(smem[i * ld + i]);
        __syncthreads();
        for (int e = tid; e < b * b; e += nt) {
            const int r = e % b, cc = e / b;
            R[e] = cc >= r ? smem[r * ld + cc] / sd[r] : 0.0;
            Rinv[e] = r < cc ? smem[cc * ld + r] / sd[cc] : (r == cc ? 1.0 / sd[cc] : 0.0);
        }
    }
    __syncthreads();
    const unsigned long long t3 = gtime();
    if (tid == 0) {
        stamps[0] = t0; stamps[1] = t1; stamps[2] = t2; stamps[3] = t3;
    }
}

template <int V>
void run(int b, const double* S, double* R, double* Ri, unsigned long long* st, const std::vector<double>& h) {
    const int threads = ((8 * b + 31) / 32) * 32;
    const size_t smem = size_t(b) * (b + 1) * 8;
    cudaFuncSetAttribute(k_probe<8, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    for (int i = 0; i < 5; ++i) k_probe<8, V><<<1, threads, smem>>>(S, b, b, 1e-12, R, Ri, st);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 200;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) k_probe<8, V><<<1, threads, smem>>>(S, b, b, 1e-12, R, Ri, st);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long hs[4];
    cudaMemcpy(hs, st, sizeof hs, cudaMemcpyDeviceToHost);
    std::vector<double> hr(size_t(b) * b);
    cudaMemcpy(hr.data(), R, sizeof(double) * b * b, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < b; ++i)
        for (int j = 0; j < b; ++j) {
            double s1 = 0;
            for (int k = 0; k < b; ++k) s1 += hr[size_t(i) * b + k] * hr[size_t(j) * b + k];
            err = std::max(err, std::abs(s1 - h[size_t(j) * b + i]));
        }
    printf("variant %d b=%d: %.2f us/launch (back to back) | setup %.2f  loop %.2f  tail %.2f us | err %.1e %s\n", V, b,
           1e3 * ms / reps, (hs[1] - hs[0]) * 1e-3, (hs[2] - hs[1]) * 1e-3, (hs[3] - hs[2]) * 1e-3, err,
           cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
    for (int b : {32, 50, 64}) {
        std::vector<double> h(size_t(b) * b), w(size_t(b) * 4 * b);
        srand(1);
        for (auto& x : w) x = double(rand()) / RAND_MAX - 0.5;
        for (int i = 0; i < b; ++i)
            for (int j = 0; j < b; ++j) {
                double s = 0;
                for (int k = 0; k < 4 * b; ++k) s += w[size_t(i) * 4 * b + k] * w[size_t(j) * 4 * b + k];
                h[size_t(j) * b + i] = s;
            }
        double *S, *R, *Ri;
        unsigned long long* st;
        cudaMalloc(&S, 8 * b * b);
        cudaMalloc(&R, 8 * b * b);
        cudaMalloc(&Ri, 8 * b * b);
        cudaMalloc(&st, 64);
        cudaMemcpy(S, h.data(), 8 * b * b, cudaMemcpyHostToDevice);
        run<0>(b, S, R, Ri, st, h);
        run<1>(b, S, R, Ri, st, h);
        run<4>(b, S, R, Ri, st, h);
    }
    return 0;
}
