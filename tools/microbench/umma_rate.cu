// umma_rate.cu -- issue-rate probe for tcgen05.mma.cta_group::1 kind::i8 / kind::f16.
//
// One CTA per SM; lane 0 of warp 0 issues R back-to-back MMAs (M = 128, N given,
// K = 32 bytes) on resident shared memory, commits, waits, and reports cycles per
// MMA.  The floor in the B300 notes is 128 * N / 256 cycles per dispatch.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate umma_rate.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t smem_desc(unsigned addr) {
    return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) |
           (uint64_t(2) << 61);
}

__device__ __forceinline__ void mma_i8(unsigned d, uint64_t a, uint64_t b, unsigned id, unsigned acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a), "l"(b), "r"(id),
                 "r"(acc));
}

// Ozaki-shaped sequence: per "slice" sp, MMAs of N = 64 * min(4, 8 - sp - sq0) into TMEM column
// (sp + sq0) * 64; mode bit 0: commit after each sp; bit 1: fence after each sp
__global__ void __launch_bounds__(128, 1) k_oz(int mode, int reps, long long* out, int fill) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar, bar2;
    __shared__ unsigned tbase;
    const unsigned base = (smem_u32(sm) + 1023u) & ~1023u;
    for (int i = threadIdx.x; i < 208 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<unsigned*>(sm)[i] = fill ? (unsigned(i) * 2654435761u) ^ (unsigned(i) >> 7) * 40503u : 0u;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar2)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (threadIdx.x == 0) {
        const unsigned tmem = tbase;
        const unsigned idesc = (2u << 4) | (1u << 7) | (1u << 10) | (8u << 24);
        const uint64_t da0 = smem_desc(base), db0 = smem_desc(base + 81920);
        long long t0 = clock64();
        long long nmma = 0;
        for (int r = 0; r < reps; ++r) {
            for (int sp = 0; sp < 8; ++sp) {
                if (mode & 2) asm volatile("tcgen05.fence::after_thread_sync;\n");
                const uint64_t da = da0 + uint64_t((((mode & 64) ? (r * 8 + sp) % 5 : sp % 5) * 16384) >> 4);
                uint64_t db = db0 + ((mode & 8) ? uint64_t(((r & 1) * 65536) >> 4) : 0) + ((mode & 32) ? uint64_t(65536 >> 4) : 0);
                for (int sq0 = 0; sq0 < 8 - sp; sq0 += 4, db += uint64_t((4 * 64 * 128) >> 4)) {
                    const int ns = (8 - sp - sq0) < 4 ? (8 - sp - sq0) : 4;
                    const unsigned id = (mode & 4) ? (idesc | (32u << 17)) : (idesc | (unsigned(ns * 8) << 17));
                    const unsigned d = (mode & 4) ? tmem + unsigned(sq0 * 64) : tmem + unsigned((sp + sq0) * 64);
                    mma_i8(d, da, db, id, 1u);
                    mma_i8(d, da + 2, db + 2, id, 1u);
                    mma_i8(d, da + 4, db + 4, id, 1u);
                    mma_i8(d, da + 6, db + 6, id, 1u);
                    nmma += 4;
                }
                if (mode & 1)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                        smem_u32(&bar2)) : "memory");
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(&bar)) : "memory");
        unsigned done = 0;
        do {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
        } while (!done);
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

template <int KIND>
__global__ void __launch_bounds__(128, 1) k_rate(int n, int reps, int b_stride, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ unsigned tbase;
    const unsigned base = (smem_u32(sm) + 1023u) & ~1023u;
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<unsigned*>(sm)[i] = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (threadIdx.x == 0) {
        const unsigned tmem = tbase;
        const unsigned idesc = KIND == 0 ? ((2u << 4) | (1u << 7) | (1u << 10) | (unsigned(n >> 3) << 17) | (8u << 24))
                                         : ((1u << 4) | (unsigned(n >> 3) << 17) | (8u << 24));  // f16 -> f32
        const uint64_t da = smem_desc(base), db = smem_desc(base + 32768);
        long long t0 = clock64();
        for (int r = 0; r < reps; r += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t a = da + uint64_t(2 * u);
                const uint64_t b = db + uint64_t((u * b_stride) >> 4) + uint64_t(2 * u);
                if (KIND == 0)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
                                 ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(1));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                                 ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(1));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(&bar)) : "memory");
        unsigned done = 0;
        do {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
        } while (!done);
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d;
    cudaMalloc(&d, sizeof(long long) * sms);
    std::vector<long long> h(sms);
    const size_t smem = 160 * 1024 + 1024;
    cudaFuncSetAttribute(k_rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(k_rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const int reps = 4096;
    for (int kind = 0; kind < 2; ++kind)
        for (int n : {64, 128, 192, 256}) {
            for (int it = 0; it < 2; ++it) {
                if (kind == 0) k_rate<0><<<sms, 128, smem>>>(n, reps, n * 128, d);
                else k_rate<1><<<sms, 128, smem>>>(n, reps, n * 128, d);
            }
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            cudaMemcpy(h.data(), d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
            long long mx = 0, sum = 0;
            for (auto v : h) mx = v > mx ? v : mx, sum += v;
            const double cyc = double(sum) / sms / reps;
            const double floor_cyc = 128.0 * n / 256.0;
            printf("%s M=128 N=%3d: %7.1f cycles/MMA (floor %5.1f) -> %4.0f%% of floor rate (max SM %.1f)\n",
                   kind == 0 ? "i8 " : "f16", n, cyc, floor_cyc, 100.0 * floor_cyc / cyc, double(mx) / reps);
        }
    cudaFuncSetAttribute(k_oz, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const size_t smem2 = 209 * 1024;
    cudaFuncSetAttribute(k_oz, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2));
    for (int mode : {3, 3 + 8, 3 + 32, 3 + 64, 3 + 8 + 64}) {
        const int r2 = 256;
        for (int it = 0; it < 2; ++it) k_oz<<<sms, 128, smem2>>>(mode, r2, d, 1);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("k_oz error\n"); return 1; }
        cudaMemcpy(h.data(), d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
        long long sum = 0;
        for (auto v : h) sum += v;
        // floor per k-step (4 MMAs per group): sum over groups of N/2 cycles
        printf("ozaki sequence mode %d (random smem %d): %7.1f cycles per k32-step (floor %s)\n", mode, 1, double(sum) / sms / r2 / 4,
               mode & 4 ? "1536: all N=256" : "1184");
    }
    return 0;
}
