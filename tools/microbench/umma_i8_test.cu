// umma_i8_test.cu -- minimal tcgen05 kind::i8 GEMM, validated on the host.
//
// C[M x N] (int32) = X' Z,  X: K x M int8 (K-major, ld = K), Z: K x N int8 (K-major).
// One CTA per 128-row tile, N = 64, K multiple of 128.  Warp 0: TMA producer,
// warp 1: MMA issuer, warps 2..5: epilogue (TMEM -> registers -> global).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);       \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

constexpr int BM = 128, BN = 64, BK = 128, STAGES = 4;
constexpr int A_BYTES = BM * BK, B_BYTES = BN * BK, STAGE_BYTES = A_BYTES + B_BYTES;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned done = 0;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}\n"
                     : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    } while (!done);
}
__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, int x, int y, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar) : "memory");
}
// K-major, 128B swizzle canonical layout: 8-row atoms of 1024 B (SBO), version 1
__device__ __forceinline__ uint64_t smem_desc(unsigned addr) {
    uint64_t d = 0;
    d |= uint64_t((addr >> 4) & 0x3FFF);
    d |= uint64_t(1) << 16;                 // LBO (unused for swizzled K-major)
    d |= uint64_t(1024 >> 4) << 32;         // SBO
    d |= uint64_t(1) << 46;                 // version
    d |= uint64_t(2) << 61;                 // SWIZZLE_128B
    return d;
}
__device__ __forceinline__ void umma_i8(unsigned tmem_d, uint64_t da, uint64_t db, unsigned idesc, unsigned acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n"
        ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
}
__device__ __forceinline__ void umma_commit(unsigned bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
                 : "memory");
}

__global__ void __launch_bounds__(192, 1)
    k_i8(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mz, int M, int K, int* C,
         int ldc) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t bars[2 * STAGES + 1];
    __shared__ unsigned tmem_base_s;
    const unsigned raw = smem_u32(smem_raw);
    const unsigned base = (raw + 1023u) & ~1023u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned full0 = smem_u32(&bars[0]), empty0 = smem_u32(&bars[STAGES]), done = smem_u32(&bars[2 * STAGES]);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_s)),
                     "r"(BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const unsigned tmem = tmem_base_s;
    const int m0 = blockIdx.x * BM;
    const int ktiles = K / BK;

    if (warp == 0 && lane == 0) {
        for (int kt = 0; kt < ktiles; ++kt) {
            const int s = kt % STAGES;
            mbar_wait(empty0 + 8 * s, ((kt / STAGES) & 1) ^ 1);
            mbar_expect_tx(full0 + 8 * s, STAGE_BYTES);
            tma_load_2d(base + s * STAGE_BYTES, &mx, kt * BK, m0, full0 + 8 * s);
            tma_load_2d(base + s * STAGE_BYTES + A_BYTES, &mz, kt * BK, 0, full0 + 8 * s);
        }
    } else if (warp == 1 && lane == 0) {
        // M = 128, N = 64, S32 accumulate, signed int8 A/B, both K-major
        const unsigned idesc = (2u << 4) | (1u << 7) | (1u << 10) | (unsigned(BN >> 3) << 17) | (unsigned(BM >> 4) << 24);
        for (int kt = 0; kt < ktiles; ++kt) {
            const int s = kt % STAGES;
            mbar_wait(full0 + 8 * s, (kt / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            const unsigned sa = base + s * STAGE_BYTES, sb = sa + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 32; ++k)
                umma_i8(tmem, smem_desc(sa + 32 * k), smem_desc(sb + 32 * k), idesc, (kt | k) != 0);
            umma_commit(empty0 + 8 * s);
        }
        umma_commit(done);
    } else if (warp >= 2) {
        mbar_wait(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const int quarter = warp & 3;
        const int row = m0 + quarter * 32 + lane;
        for (int c0 = 0; c0 < BN; c0 += 16) {
            unsigned v[16];
            const unsigned taddr = tmem + (unsigned(quarter * 32) << 16) + c0;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            if (row < M)
                for (int j = 0; j < 16; ++j) C[int64_t(c0 + j) * ldc + row] = int(v[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(BN));
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

CUtensorMap map_i8(void* p, int K, int rows, int box_rows) {
    static EncodeFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn), cudaEnableDefault, &q));
    }
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(K)};
    cuuint32_t box[2] = {128, cuuint32_t(box_rows)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", int(r));
        exit(1);
    }
    return m;
}

int main() {
    const int M = 512, N = BN, K = 1024;
    std::vector<int8_t> hx(size_t(K) * M), hz(size_t(K) * N);
    srand(1);
    for (auto& v : hx) v = int8_t((rand() % 129) - 64);
    for (auto& v : hz) v = int8_t((rand() % 129) - 64);
    int8_t *dx, *dz;
    int* dc;
    CK(cudaMalloc(&dx, hx.size()));
    CK(cudaMalloc(&dz, hz.size()));
    CK(cudaMalloc(&dc, sizeof(int) * M * N));
    CK(cudaMemcpy(dx, hx.data(), hx.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dz, hz.data(), hz.size(), cudaMemcpyHostToDevice));
    CK(cudaMemset(dc, 0, sizeof(int) * M * N));
    CUtensorMap mx = map_i8(dx, K, M, BM), mz = map_i8(dz, K, N, BN);
    const size_t smem = STAGES * STAGE_BYTES + 1024;
    CK(cudaFuncSetAttribute(k_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_i8<<<M / BM, 192, smem>>>(mx, mz, M, K, dc, M);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int> hc(size_t(M) * N);
    CK(cudaMemcpy(hc.data(), dc, sizeof(int) * M * N, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            long s = 0;
            for (int k = 0; k < K; ++k) s += long(hx[size_t(i) * K + k]) * long(hz[size_t(j) * K + k]);
            if (s != hc[size_t(j) * M + i]) {
                if (bad < 5) printf("mismatch (%d,%d): got %d want %ld\n", i, j, hc[size_t(j) * M + i], s);
                ++bad;
            }
        }
    printf("%s: %ld mismatches of %d\n", bad ? "FAIL" : "PASS", bad, M * N);
    return bad != 0;
}
