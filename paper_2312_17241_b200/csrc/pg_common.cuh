// Shared device helpers for the probegrid B200 kernels (sm_100a).
//
// Bit-exactness contract: wherever a result must equal the reference's
// (/root/reference/pkg/src/probegrid/backends/_core.pyx, compiled without
// FMA contraction — pkg/setup.py:27-33) the code uses the explicitly rounded
// intrinsics below (Ar<T>::mul/add/...), which nvcc never contracts.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/probegrid_b200.h"

namespace pg {

// ---------------------------------------------------------------- errors
void set_error(const std::string &msg);
int check_launch(const char *what);

#define PG_REQUIRE(cond, msg)            \
    do {                                 \
        if (!(cond)) {                   \
            ::pg::set_error(msg);        \
            return PG_ERR_ARG;           \
        }                                \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- per-device state: the library launches on the caller's current
// device, so every cached device property and every one-time kernel
// attribute (cudaFuncSetAttribute is per device) is keyed by it
constexpr int kMaxDevices = 64;
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d >= 0 && d < kMaxDevices ? d : 0;
}
inline int device_sms() {
    static int sms[kMaxDevices] = {};
    const int d = current_device();
    if (!sms[d]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
        sms[d] = v > 0 ? v : 148;
    }
    return sms[d];
}
inline int device_optin_smem() {
    static int optin[kMaxDevices] = {};
    const int d = current_device();
    if (!optin[d]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
        optin[d] = v > 0 ? v : 48 * 1024;
    }
    return optin[d];
}
// true the first time it is asked on the current device
struct DeviceOnce {
    bool done[kMaxDevices] = {};
    bool first() {
        const int d = current_device();
        if (done[d]) return false;
        done[d] = true;
        return true;
    }
};

inline int grid_for(int64_t n, int block, int64_t cap = (int64_t)1 << 30) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

// ------------------------------------------------- explicitly rounded math
template <typename T> struct Ar;
template <> struct Ar<float> {
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
    static __device__ __forceinline__ float sqrt(float a) { return __fsqrt_rn(a); }
    static __device__ __forceinline__ float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
    static __device__ __forceinline__ float exp(float a) { return expf(a); }
};
template <> struct Ar<double> {
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
    static __device__ __forceinline__ double sqrt(double a) { return __dsqrt_rn(a); }
    static __device__ __forceinline__ double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
    static __device__ __forceinline__ double exp(double a) { return ::exp(a); }
};

// ------------------------------------------------------------ geometry
// _core.pyx:17-23 + 38-40: cell = clamp(floor((double)x * res), 0, res-1),
// t = x*(T)res - (T)cell in T.
//
// float: x*res is exact in 48 bits, so floor((double)x*res) equals the floor
// of the exact product.  We get it in fp32: p = RN(x*res), e = x*res - p
// (exact via FMA); floor(exact) = floor(p) - [p integral and e < 0].  p cannot
// jump over an integer because integers below 2^24 are representable.
__device__ __forceinline__ int cell_coord(float x, int res, float &t) {
    const float rf = (float)res;
    const float p = __fmul_rn(x, rf);
    const float e = __fmaf_rn(x, rf, -p);
    float fl = floorf(p);
    if (p == fl && e < 0.0f) fl -= 1.0f;
    int c = (int)fl;
    c = c > res - 1 ? res - 1 : c;
    c = c < 0 ? 0 : c;
    t = __fsub_rn(p, (float)c);
    return c;
}
// double: the reference rounds the double product, then floors it.
__device__ __forceinline__ int cell_coord(double x, int res, double &t) {
    const double p = __dmul_rn(x, (double)res);
    double fl = floor(p);
    int c = (int)fl;
    c = c > res - 1 ? res - 1 : c;
    c = c < 0 ? 0 : c;
    t = __dsub_rn(p, (double)c);
    return c;
}

// corner k has offset bit (d-1-i) on axis i (numpy_backend.py:10, 37-41);
// w = ((1*a_0)*a_1)*a_2 with a_i = t_i or 1-t_i (_core.pyx:44-47).
template <typename T, int D>
__device__ __forceinline__ T corner_weight(int k, const T (&t)[D], const T (&omt)[D]) {
    T w = ((k >> (D - 1)) & 1) ? t[0] : omt[0];
#pragma unroll
    for (int i = 1; i < D; ++i) w = Ar<T>::mul(w, ((k >> (D - 1 - i)) & 1) ? t[i] : omt[i]);
    return w;
}

template <int D>
__device__ __forceinline__ uint32_t corner_hash(int k, const int (&c)[D], const uint32_t *pr) {
    uint32_t h = 0;
#pragma unroll
    for (int i = 0; i < D; ++i) h ^= (uint32_t)(c[i] + ((k >> (D - 1 - i)) & 1)) * pr[i];
    return h;
}

// row-major dense vertex index v_0 + s*(v_1 + s*v_2), s = res+1 (_core.pyx:48-50)
template <int D>
__device__ __forceinline__ int corner_dense(int k, const int (&c)[D], int stride) {
    int lin = 0;
#pragma unroll
    for (int i = D - 1; i >= 0; --i) lin = lin * stride + (c[i] + ((k >> (D - 1 - i)) & 1));
    return lin;
}

// ------------------------------------------------- feature row loads
template <typename FT> struct Feat;
template <> struct Feat<float> {
    static __device__ __forceinline__ float ld(const float *p) { return __ldg(p); }
    static __device__ __forceinline__ float2 ld2(const float *p) {
        return __ldg(reinterpret_cast<const float2 *>(p));
    }
};
template <> struct Feat<double> {
    static __device__ __forceinline__ double ld(const double *p) { return __ldg(p); }
};
template <> struct Feat<__half> {
    static __device__ __forceinline__ float ld(const __half *p) { return __half2float(__ldg(p)); }
    static __device__ __forceinline__ float2 ld2(const __half *p) {
        return __half22float2(__ldg(reinterpret_cast<const __half2 *>(p)));
    }
};

// ------------------------------------------------------ vector reductions
// sm_90+ vector float reductions straight into L2 (REDG.E.ADD.F32x4).  No
// "memory" clobber on purpose: the gradient buffers they target are never
// read by the issuing kernels, so loads may be scheduled across them (a
// clobber would serialise every corner's L2 round trip behind the previous
// corner's reductions).  Kernel boundaries order them for later readers.
__device__ __forceinline__ void red_add_v4(float *p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
                 "f"(d));
}
__device__ __forceinline__ void red_add_v2(float *p, float a, float b) {
    asm volatile("red.global.add.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(a), "f"(b));
}
__device__ __forceinline__ void red_add(float *p, float a) { atomicAdd(p, a); }
__device__ __forceinline__ void red_add(double *p, double a) { atomicAdd(p, a); }

// ------------------------------------------------ deterministic accumulation
// Deterministic mode (PG_DETERMINISTIC) accumulates every cross-thread sum in
// 64-bit fixed point: integer addition is associative, so the result does not
// depend on the order the GPU happens to schedule the adds.  Gradients use
// 2^-56 resolution (range +-128), loss sums 2^-32 (range +-2^31).
typedef unsigned long long fx_t;
#define PG_FX_SHIFT 56
#define PG_FX_LOSS_SHIFT 32
__device__ __forceinline__ fx_t to_fx(double v, int shift) {
    return (fx_t)__double2ll_rn(ldexp(v, shift));
}
__device__ __forceinline__ void red_add(fx_t *p, float a) {
    atomicAdd(p, to_fx((double)a, PG_FX_SHIFT));
}
__device__ __forceinline__ void red_add(fx_t *p, double a) {
    atomicAdd(p, to_fx(a, PG_FX_SHIFT));
}
__device__ __forceinline__ void red_add_v4(fx_t *p, float a, float b, float c, float d) {
    red_add(p, a);
    red_add(p + 1, b);
    red_add(p + 2, c);
    red_add(p + 3, d);
}
__device__ __forceinline__ void red_add_v2(fx_t *p, float a, float b) {
    red_add(p, a);
    red_add(p + 1, b);
}
__device__ __forceinline__ void loss_add(double *p, double v) { atomicAdd(p, v); }
__device__ __forceinline__ void loss_add(fx_t *p, double v) { atomicAdd(p, to_fx(v, PG_FX_LOSS_SHIFT)); }

// ------------------------------------------------------- level table
struct LevelTab {
    int res[PG_MAX_LEVELS];
    int kind[PG_MAX_LEVELS];
    int slot[PG_MAX_LEVELS];
};

int validate_grid(const pg_grid *g);

// Streaming decode (pg_decode_host_stream_f32): one kernel over the whole
// batch consumes chunks as the copy engine lands them.  ready[c] is written
// non-zero (cuStreamWriteValue32) after chunk c's H2D copy; the kernel bumps
// done[c] once per finished tile, and the D2H stream waits (cuStreamWaitValue32
// GEQ) for done[c] == tiles of chunk c.  Null pointers: ordinary launch.
struct DecodeStream {
    const uint32_t *ready = nullptr;
    uint32_t *done = nullptr;
    int chunk_tiles_log2 = 0;   // chunks are 2^k tiles of 128 queries
    uint64_t timeout_ns = 0;
    const float *host_xs = nullptr;   // pinned host copy of the inputs (fallback)
    uint32_t *fallbacks = nullptr;    // groups that took the host fallback (counted)
};

// poll a flag written by the stream front end after a copy; false if it
// does not arrive within timeout_ns.  Relaxed polling (an acquire invalidates
// L1 — the tables' cache — CCTL.IVALL in SASS, so not on every check); once
// the flag is seen set, ONE ld.acquire of it orders the caller's later loads
// of the data behind it (the chunk's coordinates, read by the whole group
// after a bar.sync) after the copy that preceded the flag write.
__device__ __forceinline__ bool acquire_flag(const uint32_t *f) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    return v != 0;
}
__device__ __forceinline__ bool wait_flag(const uint32_t *f, uint64_t timeout_ns) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if (v) return acquire_flag(f);
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        __nanosleep(128);
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (v) return acquire_flag(f);
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns) return false;
    }
}

// count n finished tiles; the caller has fenced every thread's output
// stores (gpu scope: the copy engine reads through L2) and synchronised
__device__ __forceinline__ void signal_done(uint32_t *f, uint32_t n) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(f), "r"(n) : "memory");
}

}  // namespace pg
