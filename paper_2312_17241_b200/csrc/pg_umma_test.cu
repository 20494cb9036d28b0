// Self-tests of the tcgen05 building blocks (pg_umma.cuh), one CTA each.
//
// Layout "RG" (row-group contiguous, no swizzle) for an R x K fp32 matrix:
//     off(r, k) = (r/8)*K*32 + (k/4)*128 + (r%8)*16 + (k%4)*4
// It is a K-major UMMA operand (rows r = M or N, K = k): per MMA (8 k)
// start += 256 B, LBO = 128 B, SBO = K*32 B.
// mode 0: D[128x64]  = A[128x32] . B[64x32]^T        (K-major A, K-major B)
// mode 2: D[128x64]  = A[128x64] . B[64x64]^T        (K-major, K = 64)
// mode 4: D[64x64]   = A[64x64] . B[64x64]^T        (M = 64 accumulator)
// mode 6: D[128x64]  = A[128x32] . B[64x32]^T with A stored MN-MAJOR (the
//         layout a weight-gradient GEMM reads its K = samples operand in):
//         no-swizzle canonical MN-major, core matrix = 8 K-rows x 16 bytes
//         (4 MN elements), off(m, k) = (m/4)*128 + (k/8)*(R*32) + (k%8)*16 +
//         (m%4)*4; descriptor LBO = R*32 B (K-group stride), SBO = 128 B
//         (MN-group stride); instruction descriptor a_major (bit 15) = 1
// mode 8: same with B stored MN-major (b_major, bit 16), A K-major
// mode 10: positive control of the MN-major path: kind::f16 (inputs rounded
//         to binary16), A MN-major no-swizzle (core matrix 8 K-rows x 8
//         halves), B K-major — measured: correct, while kind::tf32 with
//         either major bit set writes zeros for every layout tried (modes
//         6 / 8, variants 0-3), so tf32 operands must be K-major here
// split != 0 (mode 0): 2-term hi/lo expansion of A.
// D is returned as the raw TMEM contents: 128 lanes x 64 columns.
#include "pg_common.cuh"
#include "pg_umma.cuh"

namespace pg {

__device__ __forceinline__ uint32_t rg_off(int r, int k, int K) {
    return (uint32_t)((r >> 3) * K * 32 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}
// MN-major no-swizzle canonical layout of an R x K operand (R = M or N)
__device__ __forceinline__ uint32_t mn_off(int r, int k, int R) {
    return (uint32_t)((r >> 2) * 128 + (k >> 3) * (R * 32) + (k & 7) * 16 + (r & 3) * 4);
}
// MN-major 128-byte-swizzle canonical layout (CUTLASS Layout_MN_SW128_Atom):
// 1 KB atoms of 8 K-rows x 128 B (32 tf32 along MN), 16-byte chunk c of row
// r stored at chunk c ^ r; atoms along MN every 1 KB, K-groups every R*32 B
__device__ __forceinline__ uint32_t mn_sw128_off(int r, int k, int R) {
    const uint32_t row = (uint32_t)(k & 7), chunk = (uint32_t)((r & 31) >> 2);
    return (uint32_t)((r >> 5) * 1024 + (k >> 3) * (R * 32)) + row * 128 + ((chunk ^ row) << 4) + (r & 3) * 4;
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
    const bool mn_a = mode == 6, mn_b = mode == 8;
    const int ar = mode == 4 ? 64 : 128, ac = (mode == 0 || mn_a || mn_b) ? 32 : 64;
    const int br = 64, bc = (mode == 0 || mn_a || mn_b) ? 32 : 64;
    if (mode == 10) {   // binary16 operands: A [128 x 32] MN-major, B [64 x 32] K-major
        for (int i = tid; i < 128 * 32; i += 128) {
            const int m = i / 32, k = i % 32;
            // MN-major: core = 8 K-rows x 16 B (8 MN halves); MN groups of 8
            // every 128 B, K groups of 8 every 128 * 16 B
            const uint32_t o = (uint32_t)((m >> 3) * 128 + (k >> 3) * (128 * 16) + (k & 7) * 16 + (m & 7) * 2);
            *reinterpret_cast<__half *>(a0 + o) = __float2half(A[i]);
        }
        for (int i = tid; i < 64 * 32; i += 128) {
            const int nn = i / 32, k = i % 32;
            // K-major: core = 8 N-rows x 16 B (8 K halves); K chunks of 8 every
            // 128 B, N groups of 8 every 32 * 16 B
            const uint32_t o = (uint32_t)((nn >> 3) * (32 * 16) + (k >> 3) * 128 + (nn & 7) * 16 + (k & 7) * 2);
            *reinterpret_cast<__half *>(b0 + o) = __float2half(B[i]);
        }
    }
    for (int i = tid; i < ar * ac && mode != 10; i += 128) {
        const int r = i / ac, k = i % ac;
        float hi = A[i], lo = 0.0f;
        if (split & 1) umma::split_tf32(A[i], hi, lo);
        const bool sw = ((split >> 1) & 3) == 3;
        const uint32_t o = mn_a ? (sw ? mn_sw128_off(r, k, ar) : mn_off(r, k, ar)) : rg_off(r, k, ac);
        *reinterpret_cast<float *>(a0 + o) = hi;
        *reinterpret_cast<float *>(a1 + o) = lo;
    }
    for (int i = tid; i < br * bc && mode != 10; i += 128) {
        const int r = i / bc, k = i % bc;
        *reinterpret_cast<float *>(b0 + (mn_b ? mn_off(r, k, br) : rg_off(r, k, bc))) = B[i];
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
            const int passes = (split & 1) ? 2 : 1;
            for (int p = 0; p < passes; ++p)
                for (int kb = 0; kb < K / 8; ++kb, ++n) {
                    const uint64_t ad = umma::smem_desc(umma::smem_u32(p ? a1 : a0) + kb * 256, 128, K * 32);
                    const uint64_t bd = umma::smem_desc(umma::smem_u32(b0) + kb * 256, 128, K * 32);
                    umma::mma_tf32(tmem, ad, bd, idesc, n > 0 ? 1u : 0u);
                }
        } else if (mode == 10) {
            // f16 operands written below as halves: A MN-major (off16_mn),
            // B K-major (off16_k); K = 16 per MMA, two MMAs for K = 32
            const uint32_t idesc = (1u << 4) | (0u << 7) | (0u << 10) | (1u << 15) | ((uint32_t)(64 >> 3) << 17) |
                                   ((uint32_t)(128 >> 4) << 24);
            for (int kb = 0; kb < 2; ++kb, ++n) {
                const uint64_t ad = umma::smem_desc(umma::smem_u32(a0) + kb * 2 * 128 * 16, 128 * 16, 128);
                const uint64_t bd = umma::smem_desc(umma::smem_u32(b0) + kb * 2 * 128, 128, 32 * 16);
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(n > 0 ? 1u : 0u));
            }
        } else if (mn_a || mn_b) {
            // a_major (bit 15) / b_major (bit 16): MN-major operand
            // variant (split bits 1-2, experiments): 0 LBO = K-group stride,
            // SBO = MN-group stride (CUTLASS make_umma_desc<MN>); 1 swapped;
            // 2 as 0 without the major bit (control)
            const int var = (split >> 1) & 3;
            const uint32_t idesc = umma::idesc_tf32(128, 64) |
                                   (var != 2 ? ((mn_a ? 1u << 15 : 0u) | (mn_b ? 1u << 16 : 0u)) : 0u);
            for (int kb = 0; kb < 32 / 8; ++kb, ++n) {
                const uint32_t ka = 128 * 32, kbs = 64 * 32;
                // variant 3: A in the 128-B swizzled MN-major layout; descriptor
                // layout type SWIZZLE_128B (2, bits 61-63), LBO = MN-atom stride
                // 1 KB, SBO = K-group stride
                uint64_t ad = mn_a ? (var == 1 ? umma::smem_desc(umma::smem_u32(a0) + kb * ka, 128, ka)
                                               : umma::smem_desc(umma::smem_u32(a0) + kb * ka, ka, 128))
                                   : umma::smem_desc(umma::smem_u32(a0) + kb * 256, 128, 32 * 32);
                if (mn_a && var == 3)
                    ad = umma::smem_desc(umma::smem_u32(a0) + kb * ka, 1024, ka) | ((uint64_t)2 << 61);
                const uint64_t bd = mn_b ? (var == 1 ? umma::smem_desc(umma::smem_u32(b0) + kb * kbs, 128, kbs)
                                                     : umma::smem_desc(umma::smem_u32(b0) + kb * kbs, kbs, 128))
                                         : umma::smem_desc(umma::smem_u32(b0) + kb * 256, 128, 32 * 32);
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
    PG_REQUIRE(mode == 0 || mode == 2 || mode == 4 || mode == 6 || mode == 8 || mode == 10,
               "selftest_umma_tf32: mode must be 0, 2, 4, 6, 8 or 10");
    const int smem = (128 * 128 + 128 * 32 + 128 * 64) * 4;
    cudaFuncSetAttribute(pg::umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    pg::umma_selftest_kernel<<<1, 128, smem, pg::as_stream(stream)>>>(A, B, D, split & 15, split >> 4);
    return pg::check_launch("selftest_umma_tf32");
}
