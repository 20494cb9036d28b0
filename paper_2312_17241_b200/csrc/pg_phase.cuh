// Optional per-phase cycle accounting for the fused training kernels (build
// with -DPG_PHASE_PROF: make -C paper_2312_17241_b200/csrc prof).  Thread 0 of
// every CTA adds the clock64() time between consecutive barriers to this
// translation unit's g_phase_cycles[phase]; tools/phase_prof.py reads it.
#pragma once
#ifdef PG_PHASE_PROF
static __device__ unsigned long long g_phase_cycles[16];
#define PG_PH_INIT                  \
    long long ph_t = clock64();     \
    unsigned long long ph_acc[12] = {};
#define PG_PH(i)                                        \
    do {                                                \
        const long long ph_n = clock64();               \
        ph_acc[i] += (unsigned long long)(ph_n - ph_t); \
        ph_t = ph_n;                                    \
    } while (0)
#define PG_PH_FLUSH                                                         \
    if (threadIdx.x == 0)                                                   \
        for (int i = 0; i < 12; ++i) atomicAdd(&g_phase_cycles[i], ph_acc[i]);
#define PG_PH_READER(name)                                                              \
    extern "C" int name(unsigned long long *out16, int reset) {                         \
        cudaMemcpyFromSymbol(out16, g_phase_cycles, 16 * sizeof(unsigned long long));   \
        if (reset) {                                                                    \
            static const unsigned long long zero[16] = {};                              \
            cudaMemcpyToSymbol(g_phase_cycles, zero, sizeof(zero));                     \
        }                                                                               \
        return (int)cudaGetLastError();                                                 \
    }
#else
#define PG_PH_INIT
#define PG_PH(i)
#define PG_PH_FLUSH
#define PG_PH_READER(name)
#endif
