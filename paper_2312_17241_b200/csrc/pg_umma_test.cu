// Self-test of the tcgen05 building blocks (pg_umma.cuh): one CTA computes
// D[128x64] = A[128x32] . B[64x32]^T with kind::tf32 UMMA, accumulator in
// TMEM, read back with tcgen05.ld.  split != 0 uses the 2-term (hi + lo)
// expansion of A the fused kernels rely on for fp32-level accuracy.
#include "pg_common.cuh"
#include "pg_umma.cuh"

namespace pg {

__global__ void __launch_bounds__(128) umma_selftest_kernel(const float *__restrict__ A,
                                                            const float *__restrict__ B,
                                                            float *__restrict__ D, int split) {
    constexpr int M = 128, N = 64, K = 32;
    __shared__ __align__(1024) float sA[2][M * K];  // hi, lo
    __shared__ __align__(1024) float sB[N * K];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    char *a0 = reinterpret_cast<char *>(sA[0]);
    char *a1 = reinterpret_cast<char *>(sA[1]);
    char *b0 = reinterpret_cast<char *>(sB);
    for (int i = tid; i < M * K; i += 128) {
        const int r = i / K, k = i % K;
        float hi = A[i], lo = 0.0f;
        if (split) umma::split_tf32(A[i], hi, lo);
        *reinterpret_cast<float *>(a0 + umma::kmaj_off(r, k, M)) = hi;
        *reinterpret_cast<float *>(a1 + umma::kmaj_off(r, k, M)) = lo;
    }
    for (int i = tid; i < N * K; i += 128) {
        const int n = i / K, k = i % K;
        *reinterpret_cast<float *>(b0 + umma::kmaj_off(n, k, N)) = B[i];
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
        const uint32_t idesc = umma::idesc_tf32(M, N);
        const int passes = split ? 2 : 1;
        int n = 0;
        for (int p = 0; p < passes; ++p)
            for (int kb = 0; kb < K / 8; ++kb, ++n) {
                const uint64_t ad = umma::smem_desc(umma::smem_u32(p ? a1 : a0) + kb * M * 32, 128, 256);
                const uint64_t bd = umma::smem_desc(umma::smem_u32(b0) + kb * N * 32, 128, 256);
                umma::mma_tf32(tmem, ad, bd, idesc, n > 0 ? 1u : 0u);
            }
        umma::commit(&mbar);
    }
    umma::mbar_wait(&mbar, 0);
    umma::fence_after_sync();
    const int row = warp * 32 + (tid & 31);
#pragma unroll
    for (int c = 0; c < N; c += 32) {
        float v[32];
        umma::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) D[row * N + c + j] = v[j];
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free<64>(tmem);
}

}  // namespace pg

extern "C" int pg_selftest_umma_tf32(const float *A, const float *B, float *D, int split,
                                     void *stream) {
    pg::umma_selftest_kernel<<<1, 128, 0, pg::as_stream(stream)>>>(A, B, D, split);
    return pg::check_launch("selftest_umma_tf32");
}
