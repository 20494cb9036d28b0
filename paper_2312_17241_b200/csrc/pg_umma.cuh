// Thin inline-PTX layer over the sm_100a 5th-generation tensor core
// (tcgen05 / UMMA): TMEM allocation, shared-memory matrix descriptors,
// kind::tf32 MMA issue, commit-to-mbarrier, and TMEM -> register loads.
//
// Operand layout used throughout (no swizzle, K-major "interleaved" canonical
// layout): a matrix of R rows x K fp32/tf32 values is stored as core matrices
// of 8 rows x 16 bytes; for one MMA (K = 8 tf32) the two 16-byte K-chunks are
// LBO = 128 B apart and successive 8-row groups SBO = 256 B apart; successive
// K = 8 blocks follow each other every R*32 bytes:
//     off(r, k) = (k/8)*R*32 + (r/8)*256 + ((k/4)%2)*128 + (r%8)*16 + (k%4)*4
#pragma once

#include <stdint.h>

namespace pg {
namespace umma {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// byte offset of element (r, k) inside a K-major interleaved operand of R rows
__device__ __forceinline__ uint32_t kmaj_off(int r, int k, int R) {
    return (uint32_t)((k >> 3) * R * 32 + (r >> 3) * 256 + ((k >> 2) & 1) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

// shared-memory matrix descriptor (tcgen05 "version 1"), SWIZZLE_NONE
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // version = 1 (Blackwell)
    return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

// instruction descriptor: D f32, A/B tf32, both K-major, shape M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4)                       // c_format  = F32
           | (2u << 7)                     // a_format  = TF32
           | (2u << 10)                    // b_format  = TF32
           | ((uint32_t)(N >> 3) << 17)    // n_dim
           | ((uint32_t)(M >> 4) << 24);   // m_dim
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// all previously issued MMAs of this thread arrive on the mbarrier when done
__device__ __forceinline__ void commit(uint64_t *mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(mbar))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
        "r"(parity)
        : "memory");
}

// ReLU that propagates NaN like numpy's maximum(x, 0): one FMNMX.NAN
// (the x < 0 ? 0 : x select is two instructions)
__device__ __forceinline__ float relu_nan(float x) {
    float r;
    asm("max.NaN.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(x));
    return r;
}

// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_before_sync() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// TMEM allocation: one full warp; the base address is written to *dst (smem)
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t *dst) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
                 "n"(NCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_free(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS)
                 : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x N consecutive 32-bit columns <-> N registers per thread
// (N = 4, 8, 16), for parking per-thread state in TMEM between tiles
#define PG_TMEM_LDST(N, REGS_OUT, REGS_IN, LIST_LD, LIST_ST)                                           \
    __device__ __forceinline__ void tmem_ld##N(uint32_t taddr, float (&v)[N]) {                        \
        uint32_t r[N];                                                                                 \
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x" #N ".b32 " LIST_LD ", [%" #N "];"              \
                     : REGS_OUT                                                                        \
                     : "r"(taddr));                                                                    \
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");                                    \
        for (int i = 0; i < N; ++i) v[i] = __uint_as_float(r[i]);                                      \
    }                                                                                                  \
    __device__ __forceinline__ void tmem_st##N(uint32_t taddr, const float (&v)[N]) {                  \
        uint32_t r[N];                                                                                 \
        for (int i = 0; i < N; ++i) r[i] = __float_as_uint(v[i]);                                      \
        asm volatile("tcgen05.st.sync.aligned.32x32b.x" #N ".b32 [%0], " LIST_ST ";"                   \
                     ::"r"(taddr), REGS_IN                                                             \
                     : "memory");                                                                      \
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");                                    \
    }
#define PG_O4 "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
#define PG_I4 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3])
#define PG_O8 PG_O4, "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
#define PG_I8 PG_I4, "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
#define PG_O16 PG_O8, "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
#define PG_I16 PG_I8, "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
PG_TMEM_LDST(4, PG_O4, PG_I4, "{%0,%1,%2,%3}", "{%1,%2,%3,%4}")
PG_TMEM_LDST(8, PG_O8, PG_I8, "{%0,%1,%2,%3,%4,%5,%6,%7}", "{%1,%2,%3,%4,%5,%6,%7,%8}")
PG_TMEM_LDST(16, PG_O16, PG_I16, "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}",
             "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16}")
#undef PG_O4
#undef PG_I4
#undef PG_O8
#undef PG_I8
#undef PG_O16
#undef PG_I16
#undef PG_TMEM_LDST

// fp32 -> (hi, lo) with hi exactly representable in tf32 (round to nearest
// even on the 10-bit mantissa) and lo = x - hi (exact), itself rounded to tf32 by
// the MMA: hi*w + lo*w carries ~22 significand bits of x.
__device__ __forceinline__ void split_tf32(float x, float &hi, float &lo) {
    uint32_t h;
#ifdef PG_TF32_RNA
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
#else
    asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));   // one F2FP.TF32 (.rna: three instructions)
#endif
    hi = __uint_as_float(h);
    lo = __fsub_rn(x, hi);
}

}  // namespace umma
}  // namespace pg
