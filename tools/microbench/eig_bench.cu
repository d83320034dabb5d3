// eig_bench.cu -- cuSOLVER symmetric eigensolvers at the SVD-assembly sizes (l x l,
// l = 100..400): Dsyevd, XsyevBatched (batch 1), Dsyevj (tol 1e-14), and Dsytrd alone.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/eig_bench tools/microbench/eig_bench.cu -lcusolver
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <algorithm>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#define CK(x) do { auto _e = (x); if (int(_e) != 0) { printf("error %d at %s:%d\n", int(_e), __FILE__, __LINE__); exit(1); } } while (0)

int main() {
    cusolverDnHandle_t h;
    CK(cusolverDnCreate(&h));
    cudaStream_t s;
    cudaStreamCreate(&s);
    CK(cusolverDnSetStream(h, s));
    cusolverDnParams_t params;
    CK(cusolverDnCreateParams(&params));
    for (int n : {100, 200, 400}) {
        std::vector<double> w(size_t(n) * 3 * n), a(size_t(n) * n);
        srand(3);
        for (auto& x : w) x = double(rand()) / RAND_MAX - 0.5;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                double acc = 0;
                for (int k = 0; k < 3 * n; ++k) acc += w[size_t(i) * 3 * n + k] * w[size_t(j) * 3 * n + k] * std::pow(0.97, k);
                a[size_t(j) * n + i] = acc;
            }
        double *A, *A0, *W, *work;
        int* info;
        cudaMalloc(&A, 8 * n * n);
        cudaMalloc(&A0, 8 * n * n);
        cudaMalloc(&W, 8 * n);
        cudaMalloc(&info, 4);
        cudaMemcpy(A0, a.data(), 8 * n * n, cudaMemcpyHostToDevice);
        int lw = 0;
        CK(cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, &lw));
        int lw2 = 0;
        syevjInfo_t sj;
        CK(cusolverDnCreateSyevjInfo(&sj));
        CK(cusolverDnXsyevjSetTolerance(sj, 1e-14));
        CK(cusolverDnXsyevjSetMaxSweeps(sj, 30));
        CK(cusolverDnDsyevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, &lw2, sj));
        size_t dbytes = 0, hbytes = 0;
        CK(cusolverDnXsyevBatched_bufferSize(h, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A,
                                             n, CUDA_R_64F, W, CUDA_R_64F, &dbytes, &hbytes, 1));
        int lw3 = 0;
        double *d_, *e_, *tau;
        cudaMalloc(&d_, 8 * n);
        cudaMalloc(&e_, 8 * n);
        cudaMalloc(&tau, 8 * n);
        CK(cusolverDnDsytrd_bufferSize(h, CUBLAS_FILL_MODE_LOWER, n, A, n, d_, e_, tau, &lw3));
        size_t wbytes = std::max<size_t>({size_t(lw) * 8, size_t(lw2) * 8, dbytes, size_t(lw3) * 8});
        cudaMalloc(&work, wbytes);
        std::vector<char> hbuf(hbytes + 1);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        auto timeit = [&](const char* name, auto&& fn) {
            for (int i = 0; i < 3; ++i) { cudaMemcpyAsync(A, A0, 8 * n * n, cudaMemcpyDeviceToDevice, s); fn(); }
            cudaStreamSynchronize(s);
            float tot = 0;
            const int reps = 10;
            for (int i = 0; i < reps; ++i) {
                cudaMemcpyAsync(A, A0, 8 * n * n, cudaMemcpyDeviceToDevice, s);
                cudaEventRecord(e0, s);
                fn();
                cudaEventRecord(e1, s);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                tot += ms;
            }
            int hi = 0;
            cudaMemcpy(&hi, info, 4, cudaMemcpyDeviceToHost);
            printf("n=%d %-22s %8.1f us  info=%d\n", n, name, 1e3 * tot / reps, hi);
        };
        timeit("Dsyevd", [&] { CK(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, work, lw, info)); });
        timeit("Dsyevd (values only)", [&] { CK(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, work, lw, info)); });
        timeit("XsyevBatched(1)", [&] {
            CK(cusolverDnXsyevBatched(h, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n,
                                      CUDA_R_64F, W, CUDA_R_64F, work, dbytes, hbuf.data(), hbytes, info, 1));
        });
        size_t xd = 0, xh = 0;
        CK(cusolverDnXsyevd_bufferSize(h, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n,
                                       CUDA_R_64F, W, CUDA_R_64F, &xd, &xh));
        double* xwork;
        cudaMalloc(&xwork, std::max<size_t>(xd, 8));
        std::vector<char> xhb(xh + 1);
        timeit("Xsyevd", [&] {
            CK(cusolverDnXsyevd(h, params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n,
                                CUDA_R_64F, W, CUDA_R_64F, xwork, xd, xhb.data(), xh, info));
        });
        timeit("Dsyevd UPPER", [&] { CK(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, A, n, W, work, lw, info)); });
        timeit("Dsyevj tol 1e-14", [&] { CK(cusolverDnDsyevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, A, n, W, work, lw2, info, sj)); });
        timeit("Dsytrd only", [&] { CK(cusolverDnDsytrd(h, CUBLAS_FILL_MODE_LOWER, n, A, n, d_, e_, tau, work, lw3, info)); });
        cudaFree(A); cudaFree(A0); cudaFree(W); cudaFree(work); cudaFree(d_); cudaFree(e_); cudaFree(tau);
    }
    return 0;
}
