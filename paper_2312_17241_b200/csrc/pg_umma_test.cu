// Self-tests of the tcgen05 building blocks (pg_umma.cuh), one CTA each.
//
// Layout "RG" (row-group contiguous, no swizzle) for an R x K fp32 matrix:
//     off(r, k) = (r/8)*K*32 + (k/4)*128 + (r%8)*16 + (k%4)*4
// It is a K-major UMMA operand (rows r = M or N, K = k): per MMA (8 k)
// start += 256 B, LBO = 128 B, SBO = K*32 B.
// mode 0: D[128x64]  = A[128x32] . B[64x32]^T        (K-major A, K-major B)
// mode 2: D[128x64]  = A[128x64] . B[64x64]^T        (K-major, K = 64)
// mode 4: D[64x64]   = A[64x64] . B[64x64]^T         (M = 64 accumulator)
// split != 0 (mode 0): 2-term hi/lo expansion of A.
// D is returned as the raw TMEM contents: 128 lanes x 64 columns.
#include "pg_common.cuh"
#include "pg_umma.cuh"

namespace pg {

__device__ __forceinline__ uint32_t rg_off(int r, int k, int K) {
    return (uint32_t)((r >> 3) * K * 32 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

__global__ void __launch_bounds__(128) umma_selftest_kernel(const float *__restrict__ A,
                                                            const float *__restrict__ B,
                                                            float *__restrict__ D, int split, int mode) {
    extern __shared__ __align__(1024) unsigned char dsm[];  // A hi 32K | A lo 16K | B 32K
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    char *a0 = reinterpret_cast<char *>(dsm);
    char *a1 = a0 + 128 * 128 * 4;
    char *b0 = a1 + 128 * 32 * 4;
    // operand shapes as stored (rows x cols, RG layout)
    const int ar = mode == 4 ? 64 : 128, ac = mode == 0 ? 32 : 64;
    const int br = 64, bc = mode == 0 ? 32 : 64;
    for (int i = tid; i < ar * ac; i += 128) {
        const int r = i / ac, k = i % ac;
        float hi = A[i], lo = 0.0f;
        if (split) umma::split_tf32(A[i], hi, lo);
        *reinterpret_cast<float *>(a0 + rg_off(r, k, ac)) = hi;
        *reinterpret_cast<float *>(a1 + rg_off(r, k, ac)) = lo;
    }
    for (int i = tid; i < br * bc; i += 128) {
        const int r = i / bc, k = i % bc;
        *reinterpret_cast<float *>(b0 + rg_off(r, k, bc)) = B[i];
    }
    if (warp == 0) umma::tmem_alloc<64>(&tmem_base);
    if (tid == 0) {
        umma::mbar_init(&mbar, 1);
        umma::mbar_init_fence();
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        int n = 0;
        if (mode == 0 || mode == 2) {
            const int K = ac;
            const uint32_t idesc = umma::idesc_tf32(128, 64);
            const int passes = split ? 2 : 1;
            for (int p = 0; p < passes; ++p)
                for (int kb = 0; kb < K / 8; ++kb, ++n) {
                    const uint64_t ad = umma::smem_desc(umma::smem_u32(p ? a1 : a0) + kb * 256, 128, K * 32);
                    const uint64_t bd = umma::smem_desc(umma::smem_u32(b0) + kb * 256, 128, K * 32);
                    umma::mma_tf32(tmem, ad, bd, idesc, n > 0 ? 1u : 0u);
                }
        } else if (mode == 4) {
            const uint32_t idesc = umma::idesc_tf32(64, 64);
            for (int kb = 0; kb < 64 / 8; ++kb, ++n) {
                const uint64_t ad = umma::smem_desc(umma::smem_u32(a0) + kb * 256, 128, 64 * 32);
                const uint64_t bd = umma::smem_desc(umma::smem_u32(b0) + kb * 256, 128, 64 * 32);
                umma::mma_tf32(tmem, ad, bd, idesc, n > 0 ? 1u : 0u);
            }
        }
        umma::commit(&mbar);
    }
    umma::mbar_wait(&mbar, 0);
    umma::fence_after_sync();
    const int row = warp * 32 + (tid & 31);
#pragma unroll
    for (int c = 0; c < 64; c += 32) {
        float v[32];
        umma::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) D[row * 64 + c + j] = v[j];
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free<64>(tmem);
}

}  // namespace pg

extern "C" int pg_selftest_umma_tf32(const float *A, const float *B, float *D, int split,
                                     void *stream) {
    // split: bit 0 = hi/lo expansion (mode 0); bits 4.. = mode
    const int mode = split >> 4;
    PG_REQUIRE(mode == 0 || mode == 2 || mode == 4, "selftest_umma_tf32: mode must be 0, 2 or 4");
    const int smem = (128 * 128 + 128 * 32 + 128 * 64) * 4;
    cudaFuncSetAttribute(pg::umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    pg::umma_selftest_kernel<<<1, 128, smem, pg::as_stream(stream)>>>(A, B, D, split & 1, split >> 4);
    return pg::check_launch("selftest_umma_tf32");
}
