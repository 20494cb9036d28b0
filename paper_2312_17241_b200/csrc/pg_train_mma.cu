// Fused training pass, fast path: the same per-tile pipeline as pg_train.cu
// (encode fwd -> MLP fwd -> loss -> MLP bwd -> encode bwd, activations in
// shared memory, weight gradients held in registers across tiles), but every
// GEMM of the MLP — the two hidden layers, the output layer, both data
// gradients and all three weight gradients — runs on the tensor cores as
// warp-level mma.sync.m16n8k8 tf32 with a 3-term split (a_hi*b_hi + a_lo*b_hi
// + a_hi*b_lo, "3xTF32"), which keeps fp32-level accuracy (~1e-6 relative).
//
// Why mma.sync and not tcgen05 here: the step is bound by the L1/shared-memory
// data pipe that the table gathers/scatters also use.  The FFMA kernel spends
// ~22k shared-memory wavefronts per 64-sample tile on GEMM operands (LDS.128
// broadcast loads cost 4 wavefronts each); register fragments loaded with
// conflict-free LDS.32 cut that ~4x.  Fragments can be read from ANY layout,
// so one [feature][sample] copy of each activation serves the forward GEMMs
// (K = features) and the weight-gradient GEMMs (K = samples) alike — tcgen05
// kind::tf32 accepts only K-major operands and would need transposed copies
// of every activation, which do not fit next to two CTAs' tiles.
//
// Results are NOT in OpenBLAS order: the bit-exact path is pg_train.cu
// (PG_EXACT_MLP / reference-order mode); tests bound this one at 1e-5.
#include "pg_encode_dev.cuh"
#include "pg_phase.cuh"
#include "pg_umma.cuh"

namespace pg {
namespace tm {
constexpr int kT = 64;    // samples per tile
constexpr int kNT = 256;  // threads (8 warps), 2 CTAs per SM
constexpr int kI = 32;    // L*F
constexpr int kH = 64;    // hidden width
constexpr int kO = 4;     // max output width
constexpr int kAggRanges = 8;   // warp-aggregate feature reductions up to this many ranges per level
constexpr int kS = 72;    // row stride (floats) of [feature][sample] tiles and weights:
                          // 72 = 8 mod 32 makes the fragment loads that walk
                          // rows 4 at a time (c) and columns 8 at a time (g)
                          // bank-conflict free ...
// ... and the XOR swizzle (column ^ 12 in rows with bit 2 set) makes the
// transposed walk (rows 8 at a time, columns 4 at a time: the weight-gradient
// GEMMs, whose K is the sample index, and the W^T data-gradient GEMMs) and
// the C-fragment stores (rows 2c, columns g) conflict free too (^4 left the
// stores 2-way conflicted); every access to a [row][column] tile goes
// through sw()
__device__ __forceinline__ int sw(int row, int col) { return row * kS + (col ^ ((row & 4) * 3)); }

struct SmemW {            // weights: shared by the tile pipelines of a CTA
    // W0 / W1 in fp32, split into their 3xTF32 terms at the fragment load.
    // PG_W_PRESPLIT keeps hi and lo copies instead (split once per CTA): that
    // won while a split cost three instructions (cvt.rna; C1 0.5247 ->
    // 0.5175 ms), and loses now that it is one F2FP and L1TEX is the busiest
    // unit (twice the weight wavefronts, 28 KB less L1: 0.4516 vs 0.4435 ms)
#ifdef PG_W_PRESPLIT
    float w0[kI * kS], w0l[kI * kS];
    float w1[kH * kS], w1l[kH * kS];
#else
    float w0[kI * kS];
    float w1[kH * kS];
#endif
    float w2[kH * 8];     // W2 [in k][out j], columns >= od zero
    float b0[kH], b1[kH], b2[8];
};
struct SmemG {            // one tile pipeline's activations
    float y[kI * kS];     // y^T [f][q] of the current tile, then of the next
    float h1[kH * kS];    // relu(z1)^T [i][q], later delta1^T
    float h2[kH * kS];    // relu(z2)^T [k][q], later delta2^T, then dL/dy^T (rows < 32)
    float d3[kT * 8];     // dL/d(out) [q][j], columns >= od zero
    float xs[kT * 3];
    float tg[kT * kO];
    double lred[kNT / 32];
};
template <int NG>
struct SmemT {
    SmemW w;
    SmemG g[NG];
    uint32_t tmem_base;
};
using Smem = SmemT<1>;

// per-thread weight-gradient accumulators live in TMEM between tiles (28
// columns per warp: dW1 fragment 16, dW0 8, dW2 4), leaving the registers to
// the encode loops; acc[] is added to the parked values
template <int N>
__device__ __forceinline__ void tmem_accumulate(uint32_t taddr, const float *acc) {
    float v[N];
    if constexpr (N == 16) umma::tmem_ld16(taddr, v);
    else if constexpr (N == 8) umma::tmem_ld8(taddr, v);
    else umma::tmem_ld4(taddr, v);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] += acc[i];
    if constexpr (N == 16) umma::tmem_st16(taddr, v);
    else if constexpr (N == 8) umma::tmem_st8(taddr, v);
    else umma::tmem_st4(taddr, v);
}

// cvt.rn.tf32.f32 is one F2FP.TF32 instruction on sm_100a; cvt.rna (ties
// away) is a three-instruction software sequence (FSETP, IADD, LOP3), and
// the 3xTF32 splits are most of the MLP phase's non-MMA instructions
// (tools/micro/tf32_cvt_check.cu checks the .rn result is a clean,
// round-to-nearest-even tf32): C1 step 0.510 -> 0.483 ms
__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t r;
#ifdef PG_TF32_RNA
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
#else
    asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
#endif
    return r;
}
__device__ __forceinline__ void split(float x, uint32_t &hi, uint32_t &lo) {
    hi = to_tf32(x);
#ifndef PG_TF32_LO_RND
    // lo unrounded: the MMA reads its upper 19 bits (truncation: <= 2^-21
    // relative to x, as the decode's split); C1 0.483 -> 0.479 ms
    lo = __float_as_uint(__fsub_rn(x, __uint_as_float(hi)));
#else
    lo = to_tf32(__fsub_rn(x, __uint_as_float(hi)));
#endif
}
__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// acc[t] (16 x 8 tile at rows m0, columns n0 + 8t) += A[m][k] * B[k][n] over
// k < K, A(m, k) = pa[m*am + k*ak], B(k, n) = pb[k*bk + n*bn]; 3xTF32.
// Fragment layouts (PTX mma.m16n8k8 .tf32): g = lane/4, c = lane%4;
// A: (g, c) (g+8, c) (g, c+4) (g+8, c+4); B: (c, g) (c+4, g);
// C: (g, 2c) (g, 2c+1) (g+8, 2c) (g+8, 2c+1).
// Per-lane fragment offsets, hoisted out of the K loop: element k0 + ... of
// the fragment sits at o[i] + k0 * ks (+ t * ts for B's n-tile t).  Operands
// are swizzled kS tiles (one stride 1, the other kS; m0, n0, k0 multiples of
// 8, so the swizzle reduces to lane-constant XORs) or, SW = false, plain
// arrays.  Same addresses as sw() element by element.
// K loops fully unrolled (8 steps): the scheduler hoists the next steps'
// fragment loads over the HMMAs (C1 0.4735 -> 0.467 ms; unroll 2: 0.4735,
// 4: 0.471, 1: 0.482)
#ifndef PG_GEMM_UNROLL
#define PG_GEMM_UNROLL 8
#endif
#define PG_STR_(x) #x
#define PG_UNROLL_(n) _Pragma(PG_STR_(unroll n))
#define PG_GEMM_UNROLL_PRAGMA PG_UNROLL_(PG_GEMM_UNROLL)
// o[kp][i]: element i at k0 = kp * 8 (k0 & 8 selects kp; the rest of k0
// adds (k0 & ~15) * ks: the swizzle flips column bits 2-3, so offsets are
// lane-constant per 16-column group)
struct FragA { int o[2][4], ks; };
__device__ __forceinline__ FragA frag_a(int am, int m0, int g, int c) {
    FragA f;
    if (am == 1) {          // [k][m] tile: rows k0+c (unswizzled), k0+c+4 (^12); columns m0+g, m0+g+8
        f.o[0][0] = c * kS + m0 + g;
        f.o[0][1] = c * kS + m0 + 8 + g;
        f.o[0][2] = (c + 4) * kS + m0 + (g ^ 12);
        f.o[0][3] = (c + 4) * kS + m0 + (g ^ 4);
#pragma unroll
        for (int i = 0; i < 4; ++i) f.o[1][i] = f.o[0][i] + 8 * kS;
        f.ks = kS;
    } else {                // [m][k] tile: rows m0+g, m0+g+8 (swizzle s); columns k0+c, k0+c+4
        const int s = (g & 4) * 3, r0 = (m0 + g) * kS, r1 = r0 + 8 * kS;
        f.o[0][0] = r0 + (c ^ s);
        f.o[0][1] = r1 + (c ^ s);
        f.o[0][2] = r0 + ((c + 4) ^ s);
        f.o[0][3] = r1 + ((c + 4) ^ s);
        f.o[1][0] = r0 + ((c + 8) ^ s);
        f.o[1][1] = r1 + ((c + 8) ^ s);
        f.o[1][2] = r0 + ((c + 12) ^ s);
        f.o[1][3] = r1 + ((c + 12) ^ s);
        f.ks = 1;
    }
    return f;
}
// o[kp][tp][j]: element j of n-tile t at k0 = kp * 8, t = tp; add
// (k0 & ~15) * ks + (t & ~1) * ts
struct FragB { int o[2][2][2], ks, ts; };
template <bool SW>
__device__ __forceinline__ FragB frag_b(int bk, int bn, int n0, int g, int c) {
    FragB f;
    if constexpr (!SW) {
#pragma unroll
        for (int kp = 0; kp < 2; ++kp)
#pragma unroll
            for (int tp = 0; tp < 2; ++tp) {
                f.o[kp][tp][0] = (8 * kp + c) * bk + (n0 + 8 * tp + g) * bn;
                f.o[kp][tp][1] = (8 * kp + c + 4) * bk + (n0 + 8 * tp + g) * bn;
            }
        f.ks = bk;
        f.ts = 8 * bn;
    } else if (bn == 1) {   // [k][n] tile: rows k0+c, k0+c+4 (^12); columns n0+8t+g (n0 % 16 == 0)
#pragma unroll
        for (int kp = 0; kp < 2; ++kp) {
            f.o[kp][0][0] = (8 * kp + c) * kS + n0 + g;
            f.o[kp][1][0] = (8 * kp + c) * kS + n0 + 8 + g;
            f.o[kp][0][1] = (8 * kp + c + 4) * kS + n0 + (g ^ 12);
            f.o[kp][1][1] = (8 * kp + c + 4) * kS + n0 + (g ^ 4);
        }
        f.ks = kS;
        f.ts = 8;
    } else {                // [n][k] tile: rows n0+8t+g (swizzle s); columns k0+c, k0+c+4
        const int s = (g & 4) * 3, r0 = (n0 + g) * kS;
#pragma unroll
        for (int tp = 0; tp < 2; ++tp) {
            f.o[0][tp][0] = r0 + 8 * tp * kS + (c ^ s);
            f.o[0][tp][1] = r0 + 8 * tp * kS + ((c + 4) ^ s);
            f.o[1][tp][0] = r0 + 8 * tp * kS + ((c + 8) ^ s);
            f.o[1][tp][1] = r0 + 8 * tp * kS + ((c + 12) ^ s);
        }
        f.ks = 1;
        f.ts = 8 * kS;
    }
    return f;
}
template <int NT, int K, bool SWB = true>
__device__ __forceinline__ void warp_gemm(float (&acc)[NT][4], const float *pa, int am, int ak, int m0,
                                          const float *pb, int bk, int bn, int n0) {
    const int lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
    const FragA fa = frag_a(am, m0, g, c);
    const FragB fb = frag_b<SWB>(bk, bn, n0, g, c);
PG_GEMM_UNROLL_PRAGMA
    for (int k0 = 0; k0 < K; k0 += 8) {
        uint32_t ah[4], al[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) split(pa[fa.o[(k0 >> 3) & 1][i] + (k0 & ~15) * fa.ks], ah[i], al[i]);
        // term-major issue: NT independent HMMAs between dependent ones
        // (0.5545 -> 0.5521 ms per C1 step vs the three terms of one tile
        // back to back)
        uint32_t bh[NT][2], bl[NT][2];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int kp = (k0 >> 3) & 1, kb = (k0 & ~15) * fb.ks + (t & ~1) * fb.ts;
            split(pb[fb.o[kp][t & 1][0] + kb], bh[t][0], bl[t][0]);
            split(pb[fb.o[kp][t & 1][1] + kb], bh[t][1], bl[t][1]);
        }
#pragma unroll
        for (int t = 0; t < NT; ++t) hmma(acc[t], al, bh[t][0], bh[t][1]);  // small terms first
#pragma unroll
        for (int t = 0; t < NT; ++t) hmma(acc[t], ah, bl[t][0], bl[t][1]);
#pragma unroll
        for (int t = 0; t < NT; ++t) hmma(acc[t], ah, bh[t][0], bh[t][1]);
    }
}

// warp_gemm with B given as its pre-split tf32 hi / lo terms (same products,
// same accumulation order: bit-identical to splitting at the load)
template <int NT, int K>
__device__ __forceinline__ void warp_gemm_bs(float (&acc)[NT][4], const float *pa, int am, int ak, int m0,
                                             const float *pbh, const float *pbl, int bk, int bn, int n0) {
    const int lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
    const FragA fa = frag_a(am, m0, g, c);
    const FragB fb = frag_b<true>(bk, bn, n0, g, c);
PG_GEMM_UNROLL_PRAGMA
    for (int k0 = 0; k0 < K; k0 += 8) {
        uint32_t ah[4], al[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) split(pa[fa.o[(k0 >> 3) & 1][i] + (k0 & ~15) * fa.ks], ah[i], al[i]);
        uint32_t bh[NT][2], bl[NT][2];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int kp = (k0 >> 3) & 1, kb = (k0 & ~15) * fb.ks + (t & ~1) * fb.ts;
            const int o0 = fb.o[kp][t & 1][0] + kb, o1 = fb.o[kp][t & 1][1] + kb;
            bh[t][0] = __float_as_uint(pbh[o0]);
            bl[t][0] = __float_as_uint(pbl[o0]);
            bh[t][1] = __float_as_uint(pbh[o1]);
            bl[t][1] = __float_as_uint(pbl[o1]);
        }
#pragma unroll
        for (int t = 0; t < NT; ++t) hmma(acc[t], al, bh[t][0], bh[t][1]);
#pragma unroll
        for (int t = 0; t < NT; ++t) hmma(acc[t], ah, bl[t][0], bl[t][1]);
#pragma unroll
        for (int t = 0; t < NT; ++t) hmma(acc[t], ah, bh[t][0], bh[t][1]);
    }
}

// GEMM with a weight operand: pre-split hi/lo copies (PG_W_PRESPLIT) or
// one fp32 copy split at the fragment load
#ifdef PG_W_PRESPLIT
#define PG_WGEMM(NT, K, acc, pa, am, ak, m0, wh, wl, bk, bn, n0) \
    warp_gemm_bs<NT, K>(acc, pa, am, ak, m0, wh, wl, bk, bn, n0)
#else
#define PG_WGEMM(NT, K, acc, pa, am, ak, m0, wh, wl, bk, bn, n0) warp_gemm<NT, K>(acc, pa, am, ak, m0, wh, bk, bn, n0)
#endif

// store a warp's C fragments (rows = samples m, columns = features n) into a
// [feature][sample] tile, optionally through f(value, feature, sample)
template <int NT, typename F>
__device__ __forceinline__ void store_frags_T(float *dstT, const float (&acc)[NT][4], int m0, int n0, F f) {
    const int lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int n = n0 + 8 * t + 2 * c;
        dstT[sw(n, m0 + g)] = f(acc[t][0], n, m0 + g);
        dstT[sw(n + 1, m0 + g)] = f(acc[t][1], n + 1, m0 + g);
        dstT[sw(n, m0 + g + 8)] = f(acc[t][2], n, m0 + g + 8);
        dstT[sw(n + 1, m0 + g + 8)] = f(acc[t][3], n + 1, m0 + g + 8);
    }
}

// bias gradient partial: sum over the tile's samples of row r of a
// [feature][sample] tile; 4 threads per row, result valid in lane%4 == 0
__device__ __forceinline__ float row_sum4(const float *srcT, int r, int qq) {
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < kT / 4; ++i) s += srcT[sw(r, qq + 4 * i)];
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    return s;
}
}  // namespace tm

// Volume compositing of one ray = one 64-sample tile (PG_COMPOSITE, the
// NeRF-style head of SURVEY 8f row 4): G.d3[q*8 + 0..3] holds the raw MLP
// outputs (sigma_raw, r, g, b) of sample q, G.tg[q*4] its segment length and
// G.tg[1..3] the ray's target colour.  One warp: lane l owns samples 2l and
// 2l+1; transmittance by a multiplicative warp scan, the colour by a warp
// sum, the backward's "colour behind sample i" by an additive scan (same
// equations as pg_mlp.cu composite_loss_kernel).  Overwrites G.d3 with
// dL/d(raw); returns the ray's squared error (lane 0).
__device__ __forceinline__ float tile_softplus(float x) { return x > 20.0f ? x : log1pf(expf(x)); }
__device__ __forceinline__ float tile_logistic(float x) { return 1.0f / (1.0f + expf(-x)); }

__device__ __forceinline__ double composite_tile(float *d3, const float *tg, float scale, int lane) {
    float raw[2][4], tr[2], c[2][3], dl[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int q = 2 * lane + u;
        const float4 v = *reinterpret_cast<const float4 *>(d3 + q * 8);
        raw[u][0] = v.x; raw[u][1] = v.y; raw[u][2] = v.z; raw[u][3] = v.w;
        dl[u] = tg[q * 4];
        tr[u] = expf(-tile_softplus(v.x) * dl[u]);
#pragma unroll
        for (int k = 0; k < 3; ++k) c[u][k] = tile_logistic(raw[u][k + 1]);
    }
    // exclusive prefix product of the transmittances over the 64 samples
    float p = tr[0] * tr[1], incl = p;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl *= t;
    }
    float T0 = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) T0 = 1.0f;
    const float T[2] = {T0, T0 * tr[0]};
    const float w[2] = {T[0] * (1.0f - tr[0]), T[1] * (1.0f - tr[1])};
    float C[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float v = w[0] * c[0][k] + w[1] * c[1][k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        C[k] = v;
    }
    double sq = 0.0;
    float gC[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float diff = C[k] - tg[1 + k];
        sq += (double)diff * (double)diff;
        gC[k] = diff * scale;
    }
    const float cg = C[0] * gC[0] + C[1] * gC[1] + C[2] * gC[2];
    float ci_g[2], v[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        ci_g[u] = c[u][0] * gC[0] + c[u][1] * gC[1] + c[u][2] * gC[2];
        v[u] = w[u] * ci_g[u];
    }
    float s = v[0] + v[1];   // inclusive prefix sum over lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float t = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += t;
    }
    const float pre[2] = {s - v[1], s};             // prefix through samples 2l, 2l+1
    const float Tn[2] = {T[1], T[1] * tr[1]};        // T_{i+1}
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int q = 2 * lane + u;
        const float dsig = dl[u] * (Tn[u] * ci_g[u] - (cg - pre[u]));
        float4 d;
        d.x = dsig * tile_logistic(raw[u][0]);
        d.y = w[u] * gC[0] * c[u][0] * (1.0f - c[u][0]);
        d.z = w[u] * gC[1] * c[u][1] * (1.0f - c[u][1]);
        d.w = w[u] * gC[2] * c[u][2] * (1.0f - c[u][2]);
        *reinterpret_cast<float4 *>(d3 + q * 8) = d;
    }
    return lane == 0 ? sq : 0.0;
}

// NG = 1: one 8-warp tile pipeline per CTA, two CTAs per SM.  NG = 2: one
// CTA per SM running two 8-warp pipelines that share the weights and are
// held in anti-phase by a CTA-wide barrier at every phase switch, so one
// pipeline's MLP (shared memory + tensor pipe) always runs beside the
// other's table gathers/scatters (L1/L2).
// AGG: warp-aggregated feature-gradient reductions for probed levels with
// few probing ranges (n_f / N_p <= kAggRanges).  Every lookup of such a
// level lands in one of a handful of ranges, so per-lane reductions from all
// SMs serialise on the same L2 addresses (C5 / default-HyperParams shapes:
// 2-9x slower steps); instead the lanes of a warp that share a range sum
// their contributions with a shuffle reduce-scatter and one coalesced
// reduction per range and warp is issued (encode_level_bwd2<..., AGG>).
template <typename FT, int D, int NPM, typename ACC, typename LACC, int NG, bool AGG = false>
__global__ void __launch_bounds__(tm::kNT *NG, 2 / NG)
    train_mma_kernel(const pg_grid g, const float *__restrict__ xs, const float *__restrict__ targets,
                     int64_t B, const FT *__restrict__ feats_fwd, const float *__restrict__ feats,
                     const uint8_t *__restrict__ baked, const float *__restrict__ conf,
                     const float *__restrict__ params, int od, float scale,
                     int mode_flags,   // bits 0-1: 1 logistic output, 2 volume compositing (one ray
                                       // per tile); bit 2: flag every probed lookup as touched;
                                       // bits 8-15: feature-gradient replicas - 1 (gfeat then
                                       // holds that many copies; CTA b adds into copy b % reps)
                     ACC *__restrict__ gfeat, ACC *__restrict__ gconf, uint8_t *__restrict__ touched,
                     ACC *__restrict__ gparams, LACC *__restrict__ loss_sum, float *__restrict__ dy_out,
                     const CellMap cmap) {
    using namespace tm;
    const int sigmoid = mode_flags & 3;
    const bool touch_all = (mode_flags & 4) != 0;
    const int reps = ((mode_flags >> 8) & 255) + 1;
    ACC *const gfeat_cta = gfeat + (int64_t)(blockIdx.x % reps) * g.n_levels * g.n_f * 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmemT<NG> &S = *reinterpret_cast<SmemT<NG> *>(smem_raw);
    const int gid = NG == 1 ? 0 : (int)(threadIdx.x >> 8);   // tile pipeline
    const int tid = threadIdx.x & (kNT - 1), warp = tid >> 5, lane = tid & 31;
    SmemW &W = S.w;
    SmemG &G = S.g[gid];
    // dL/dy^T [f][q] lives in h2's rows 0..31: delta2 is dead when dy is
    // stored, and h2 is rewritten only by the next tile's layer 2 (saves 9 KB
    // per pipeline of shared memory for L1: 0.548 vs 0.551 ms per C1 step)
    float *const GDY = G.h2;
    // barrier of this pipeline's 256 threads / of the whole CTA
    auto gsync = [&]() {
        if constexpr (NG == 1) __syncthreads();
        else asm volatile("bar.sync %0, %1;" ::"r"(1 + gid), "r"(kNT) : "memory");
    };
    // ping-pong between the two pipelines (NG = 2): named barrier 3 = "pipeline
    // 1's MLP done", 4 = "pipeline 0's MLP done"; a pipeline arrives (no
    // wait) when its MLP ends and waits only before starting its next MLP, so
    // the two MLP phases never overlap and each runs beside the other
    // pipeline's encode.  Measured per C1 step: 0.551 ms; a symmetric CTA
    // barrier at both phase switches 0.567, at one 0.558; no coupling 0.656.
    auto bar_sync = [&](int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(2 * kNT) : "memory"); };
    auto bar_arrive = [&](int id) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(2 * kNT) : "memory"); };
    {
        const float *p = params;
        const int nt = kNT * NG, t0 = threadIdx.x;
        for (int i = t0; i < kI * kH; i += nt) {
#ifdef PG_W_PRESPLIT
            uint32_t h, l;
            split(p[i], h, l);
            W.w0[sw(i / kH, i % kH)] = __uint_as_float(h);
            W.w0l[sw(i / kH, i % kH)] = __uint_as_float(l);
#else
            W.w0[sw(i / kH, i % kH)] = p[i];
#endif
        }
        p += kI * kH;
        for (int i = t0; i < kH; i += nt) W.b0[i] = p[i];
        p += kH;
        for (int i = t0; i < kH * kH; i += nt) {
#ifdef PG_W_PRESPLIT
            uint32_t h, l;
            split(p[i], h, l);
            W.w1[sw(i / kH, i % kH)] = __uint_as_float(h);
            W.w1l[sw(i / kH, i % kH)] = __uint_as_float(l);
#else
            W.w1[sw(i / kH, i % kH)] = p[i];
#endif
        }
        p += kH * kH;
        for (int i = t0; i < kH; i += nt) W.b1[i] = p[i];
        p += kH;
        for (int i = t0; i < kH * 8; i += nt) {
            const int k = i / 8, j = i % 8;
            W.w2[i] = j < od ? p[k * od + j] : 0.0f;
        }
        p += kH * od;
        for (int i = t0; i < 8; i += nt) W.b2[i] = i < od ? p[i] : 0.0f;
    }
    // weight-gradient fragments (dW1 rows i = 16*(warp&3).., columns j =
    // 32*(warp>>2)..; dW0 rows f = 16*(warp&1).., columns i = 16*(warp>>1)..;
    // dW2 rows k = 16*warp (warps 0-3), columns j < 8), parked in TMEM
    if (threadIdx.x < 32) umma::tmem_alloc<64 * NG>(&S.tmem_base);
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tm = S.tmem_base + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 32) +
                        (uint32_t)(64 * gid);

    {
        const float z16[16] = {}, z8[8] = {}, z4[4] = {};
        umma::tmem_st16(tm, z16);
        umma::tmem_st8(tm + 16, z8);
        umma::tmem_st4(tm + 24, z4);
    }
    float gb0 = 0.0f, gb1 = 0.0f, gb2 = 0.0f;   // biases: row tid>>2 (lane%4 == 0); b2: tid < 8
    double lsum = 0.0;
    PG_PH_INIT

    const int64_t ntiles = (B + kT - 1) / kT;
    static_assert(kT * 3 <= kNT && kT * kO == kNT, "one prefetched value per thread");
    auto fetch = [&](int64_t t, float &fx, float &ft) {
        const int64_t q0 = t * kT;
        const int n = t < ntiles ? (int)((B - q0) < kT ? (B - q0) : kT) : 0;
        fx = (tid < kT * D && tid < n * D) ? __ldg(xs + q0 * D + tid) : 0.5f;
        const int q = tid / kO, j = tid % kO;
        ft = (q < n && j < od) ? __ldg(targets + (q0 + q) * od + j) : 0.0f;
    };
    float pf_x, pf_t;
    const int pl = tid & (kT - 1), lsub = tid >> 6;
    const int mt = warp & 3;           // 16-sample m-tile of the sample-major GEMMs
    const int rr = tid >> 2, qq = tid & 3;  // bias row-sum role
    // tiles of this pipeline: first, first + stride, ...; every pipeline of
    // a CTA runs as many iterations as its first one (the most), so the
    // CTA-wide phase barriers match up
    const int64_t first = (int64_t)blockIdx.x * NG + gid, stride = (int64_t)gridDim.x * NG;
    const int64_t base0 = (int64_t)blockIdx.x * NG;
    const int64_t n_iter = base0 < ntiles ? (ntiles - base0 + stride - 1) / stride : 0;
    // prologue: the first tile's inputs and encode forward
    float x[D];
    fetch(first, pf_x, pf_t);
    if (tid < kT * D) G.xs[tid] = pf_x;
    G.tg[tid] = pf_t;
    fetch(first + stride, pf_x, pf_t);
    gsync();
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = G.xs[pl * D + a];
    if (first < ntiles) {
#pragma unroll 2
        for (int it = 0; it < 4; ++it) {
            const int l = lsub + 4 * it;
            const float2 yv = cmap.off[l] >= 0 ? encode_level_fwd2_cell32<D>(g, l, x, cmap.cells + cmap.off[l])
                                               : encode_level_fwd2_rng<FT, D>(g, l, x, feats_fwd, baked);
            G.y[sw(2 * l, pl)] = yv.x;
            G.y[sw(2 * l + 1, pl)] = yv.y;
        }
    }
    for (int64_t iter = 0; iter < n_iter; ++iter) {
        const int64_t tile = first + iter * stride;
        if (NG > 1) {   // wait for the other pipeline's previous MLP to end
            if (gid == 0) bar_sync(3);
            else if (iter > 0) bar_sync(4);
        }
        if (tile >= ntiles) {    // (only pipeline 1's last iteration) keep the barrier count
            if (NG > 1 && gid == 1) bar_arrive(3);
            continue;
        }
        const int64_t p0 = tile * kT;
        const int nv = (int)((B - p0) < kT ? (B - p0) : kT);
        gsync();
        PG_PH(1);
        // ---- layer 1: h1 = relu(y W0 + b0) ----
        {
            float acc[4][4] = {};
            PG_WGEMM(4, kI, acc, G.y, 1, kS, 16 * mt, W.w0, W.w0l, kS, 1, 32 * (warp >> 2));
            const int c = lane & 3;
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float z = acc[t][e] + W.b0[32 * (warp >> 2) + 8 * t + 2 * c + (e & 1)];
                    acc[t][e] = z > 0.0f ? z : 0.0f;
                }
            store_frags_T<4>(G.h1, acc, 16 * mt, 32 * (warp >> 2), [](float v, int, int) { return v; });
        }
        gsync();
        PG_PH(2);
        // ---- layer 2: h2 = relu(h1 W1 + b1) ----
        float po[4] = {};   // this warp's partial output layer (its 32 hidden units)
        {
            float acc[4][4] = {};
            PG_WGEMM(4, kH, acc, G.h1, 1, kS, 16 * mt, W.w1, W.w1l, kS, 1, 32 * (warp >> 2));
#ifdef PG_OUT_SEPARATE
            store_frags_T<4>(G.h2, acc, 16 * mt, 32 * (warp >> 2), [&](float v, int n, int) {
                const float z = v + W.b1[n];
                return z > 0.0f ? z : 0.0f;
            });
#else
            // ReLU in registers: the C fragments are also the A fragments of
            // the output layer over this warp's 32 hidden units (k-slot c ->
            // unit 2c, c + 4 -> 2c + 1), so each warp of an m-tile pair
            // computes a K-half of the output from registers; the halves meet
            // in G.d3 across the barrier (output phase 7.5% of a tile)
            const int nb = 32 * (warp >> 2), g = lane >> 2, c = lane & 3;
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float z = acc[t][e] + W.b1[nb + 8 * t + 2 * c + (e & 1)];
                    acc[t][e] = z > 0.0f ? z : 0.0f;
                }
            store_frags_T<4>(G.h2, acc, 16 * mt, nb, [](float v, int, int) { return v; });
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                uint32_t ah[4], al[4], bh0, bl0, bh1, bl1;
                split(acc[t][0], ah[0], al[0]);
                split(acc[t][2], ah[1], al[1]);
                split(acc[t][1], ah[2], al[2]);
                split(acc[t][3], ah[3], al[3]);
                split(W.w2[(nb + 8 * t + 2 * c) * 8 + g], bh0, bl0);
                split(W.w2[(nb + 8 * t + 2 * c + 1) * 8 + g], bh1, bl1);
                hmma(po, al, bh0, bh1);
                hmma(po, ah, bl0, bl1);
                hmma(po, ah, bh0, bh1);
            }
            if (warp >= 4) {
#pragma unroll
                for (int e = 0; e < 4; ++e) G.d3[(16 * mt + g + (e >> 1) * 8) * 8 + 2 * c + (e & 1)] = po[e];
            }
#endif
        }
        gsync();
        PG_PH(3);
        // ---- output layer, loss, dL/dout (warps 0-3: one 16-sample tile each) ----
        if (warp < 4) {
            float acc[1][4] = {};
            const int gq = lane >> 2, c = lane & 3;
#ifdef PG_OUT_SEPARATE
            warp_gemm<1, kH, false>(acc, G.h2, 1, kS, 16 * warp, W.w2, 8, 1, 0);
#else
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[0][e] = po[e] + G.d3[(16 * warp + gq + (e >> 1) * 8) * 8 + 2 * c + (e & 1)];
#endif
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int q = 16 * warp + gq + (e >> 1) * 8, j = 2 * c + (e & 1);
                float d = 0.0f;
                if (sigmoid == 2) {
                    d = j < od ? acc[0][e] + W.b2[j] : 0.0f;   // raw output, composited below
                } else if (j < od && q < nv) {
                    const float o = acc[0][e] + W.b2[j];
                    const float pred = sigmoid == 1 ? 1.0f / (1.0f + expf(-o)) : o;
                    const float diff = pred - G.tg[q * kO + j];
                    lsum += (double)diff * (double)diff;
                    d = diff * scale;
                    if (sigmoid == 1) d *= pred * (1.0f - pred);
                }
                G.d3[q * 8 + j] = d;
            }
        }
        gsync();
        if (sigmoid == 2) {
            if (warp == 0) lsum += composite_tile(G.d3, G.tg, scale, lane);
            gsync();
        }
        PG_PH(4);
        // ---- dW2 += h2^T d3 (warps 0-3), db2; delta2 = (d3 W2^T) * (h2 > 0) ----
        if (warp < 4) {
            float t2[1][4] = {};
            warp_gemm<1, kT, false>(t2, G.h2, kS, 1, 16 * warp, G.d3, 8, 1, 0);
            tmem_accumulate<4>(tm + 24, &t2[0][0]);
        }
        if (tid < 8) {
            float s = 0.0f;
            for (int q = 0; q < kT; ++q) s += G.d3[q * 8 + tid];
            gb2 += s;
        }
        {
            // thread (sample q = tid & 63, 16 hidden units k = 16*(tid>>6)..)
            const int q = tid & (kT - 1), k0 = 16 * (tid >> 6);
            const float4 dq = *reinterpret_cast<const float4 *>(G.d3 + q * 8);
            float dl[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int k = k0 + u;
                const float4 w = *reinterpret_cast<const float4 *>(W.w2 + k * 8);
                const float s = dq.x * w.x + dq.y * w.y + dq.z * w.z + dq.w * w.w;
                dl[u] = G.h2[sw(k, q)] > 0.0f ? s : 0.0f;
            }
            gsync();  // dW2 reads h2 above
            PG_PH(5);
#pragma unroll
            for (int u = 0; u < 16; ++u) G.h2[sw(k0 + u, q)] = dl[u];
        }
        gsync();
        PG_PH(6);
        {
            const float s = row_sum4(G.h2, rr, qq);
            if (qq == 0) gb1 += s;
        }
        // ---- dW1 += h1^T delta2 ; delta1' = delta2 W1^T (kept in registers) ----
        float dacc[4][4] = {};
        {
            float t1[4][4] = {};
            warp_gemm<4, kT>(t1, G.h1, kS, 1, 16 * (warp & 3), G.h2, 1, kS, 32 * (warp >> 2));
            PG_WGEMM(4, kH, dacc, G.h2, 1, kS, 16 * mt, W.w1, W.w1l, 1, kS, 32 * (warp >> 2));
            tmem_accumulate<16>(tm, &t1[0][0]);   // after the independent GEMM: they interleave
        }
        gsync();
        PG_PH(7);
        // delta1 = delta1' * (h1 > 0), in place over h1; its bias gradient
        // (column sums over the tile's samples) from the same registers:
        // rows g, g+8 per lane, then a reduce-scatter over the 8 lanes of a
        // column group — lane (g, c) ends with column 8*(g>>1) + 2c + (g&1)
        // (vs a row sum re-reading delta1 from shared memory: C1 0.4368 ->
        // 0.4272 ms; keeping h1 > 0 as a register bit mask instead of
        // re-reading h1 spills at the 128-register cap: 0.449)
        {
            float x[8];
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (!(G.h1[sw(32 * (warp >> 2) + 8 * t + 2 * (lane & 3) + (e & 1), 16 * mt + (lane >> 2) + (e >> 1) * 8)] > 0.0f))
                        dacc[t][e] = 0.0f;
#pragma unroll
            for (int v = 0; v < 8; ++v) x[v] = dacc[v >> 1][v & 1] + dacc[v >> 1][2 + (v & 1)];
#pragma unroll
            for (int sh = 4; sh >= 1; sh >>= 1) {
                const bool up = (lane & (4 * sh)) != 0;
#pragma unroll
                for (int i = 0; i < sh; ++i) {
                    const float send = up ? x[i] : x[i + sh], keep = up ? x[i + sh] : x[i];
                    x[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4 * sh);
                }
            }
            gb0 += x[0];
        }
        store_frags_T<4>(G.h1, dacc, 16 * mt, 32 * (warp >> 2), [](float v, int, int) { return v; });
        gsync();
        PG_PH(8);
        // ---- dW0 += y^T delta1 ; dy = delta1 W0^T ----
        {
            float yacc[2][4] = {};
            {
                float t0[2][4] = {};
                warp_gemm<2, kT>(t0, G.y, kS, 1, 16 * (warp & 1), G.h1, 1, kS, 16 * (warp >> 1));
                PG_WGEMM(2, kH, yacc, G.h1, 1, kS, 16 * mt, W.w0, W.w0l, 1, kS, 16 * (warp >> 2));
                tmem_accumulate<8>(tm + 16, &t0[0][0]);
            }
            PG_PH(9);
            store_frags_T<2>(GDY, yacc, 16 * mt, 16 * (warp >> 2), [](float v, int, int) { return v; });
        }
        gsync();   // dy complete; y, xs, tg free for the next tile
        PG_PH(10);
        if (dy_out) {
            for (int i = tid; i < nv * kI; i += kNT) {
                const int q = i / kI, c = i % kI;
                dy_out[(p0 + q) * kI + c] = GDY[sw(c, q)];
            }
        }
        // ---- stage the next tile's inputs (prefetched into registers) ----
        const int64_t nxt = tile + stride;
        if (tid < kT * D) G.xs[tid] = pf_x;
        G.tg[tid] = pf_t;
        fetch(nxt + stride, pf_x, pf_t);
        gsync();
        if (NG > 1) bar_arrive(gid == 0 ? 4 : 3);   // MLP done: the other pipeline may start its own
        PG_PH(0);
        float xn[D];
#pragma unroll
        for (int a = 0; a < D; ++a) xn[a] = G.xs[pl * D + a];
        // ---- encode backward of this tile fused with encode forward of the
        //      next: both use the (sample, level) thread mapping, so one loop
        //      keeps both tiles' L2 round trips in flight together ----
        const bool has_next = nxt < ntiles;
#pragma unroll 1
        for (int it = 0; it < 4; ++it) {
            const int l = lsub + 4 * it;
            if (has_next) {
                // N_p = 4: the probing range fetched whole beside the baked
                // byte (one L2 round trip, not two): 0.5499 -> 0.5473 ms (C1)
                // levels in the step's cell cache: one 32-byte record load
                const float2 yv = cmap.off[l] >= 0 ? encode_level_fwd2_cell32<D>(g, l, xn, cmap.cells + cmap.off[l])
                                                   : encode_level_fwd2_rng<FT, D>(g, l, xn, feats_fwd, baked);
                G.y[sw(2 * l, pl)] = yv.x;
                G.y[sw(2 * l + 1, pl)] = yv.y;
            }
            constexpr bool lazy = std::is_same<ACC, float>::value;
            if constexpr (AGG) {
                // every lane of the warp takes part (the shuffles); lanes past
                // the batch end contribute nothing
                encode_level_bwd2<D, NPM, ACC, lazy, true>(g, l, x, GDY[sw(2 * l, pl)],
                                                           GDY[sw(2 * l + 1, pl)], feats, conf, gfeat_cta, gconf,
                                                           touched, touch_all, pl < nv);
            } else if (pl < nv) {
                encode_level_bwd2<D, NPM, ACC, lazy>(g, l, x, GDY[sw(2 * l, pl)], GDY[sw(2 * l + 1, pl)],
                                                     feats, conf, gfeat_cta, gconf, touched, touch_all);
            }
        }
#pragma unroll
        for (int a = 0; a < D; ++a) x[a] = xn[a];
        PG_PH(11);
    }
    if (NG > 1 && gid == 1 && n_iter > 0) bar_sync(4);   // consume pipeline 0's last MLP-done
    PG_PH_FLUSH
    // ---- flush ----
    ACC *gW0p = gparams, *gb0p = gW0p + kI * kH, *gW1p = gb0p + kH, *gb1p = gW1p + kH * kH;
    ACC *gW2p = gb1p + kH, *gb2p = gW2p + kH * od;
    {
        float gW1[4][4], gW0[2][4], gW2[1][4];
        umma::tmem_ld16(tm, *reinterpret_cast<float(*)[16]>(&gW1[0][0]));
        umma::tmem_ld8(tm + 16, *reinterpret_cast<float(*)[8]>(&gW0[0][0]));
        umma::tmem_ld4(tm + 24, *reinterpret_cast<float(*)[4]>(&gW2[0][0]));
        const int gq = lane >> 2, c = lane & 3;
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = 16 * (warp & 3) + gq + (e >> 1) * 8, j = 32 * (warp >> 2) + 8 * t + 2 * c + (e & 1);
                red_add(gW1p + i * kH + j, gW1[t][e]);
            }
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int f = 16 * (warp & 1) + gq + (e >> 1) * 8, i = 16 * (warp >> 1) + 8 * t + 2 * c + (e & 1);
                red_add(gW0p + f * kH + i, gW0[t][e]);
            }
        if (warp < 4) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = 16 * warp + gq + (e >> 1) * 8, j = 2 * c + (e & 1);
                if (j < od) red_add(gW2p + k * od + j, gW2[0][e]);
            }
        }
        red_add(gb0p + 32 * (warp >> 2) + 8 * (gq >> 1) + 2 * c + (gq & 1), gb0);
        if (qq == 0) red_add(gb1p + rr, gb1);
        if (tid < od) red_add(gb2p + tid, gb2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    if (lane == 0) G.lred[warp] = lsum;
    gsync();
    if (tid < 32) {
        double v = tid < kNT / 32 ? G.lred[tid] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (tid == 0 && loss_sum) loss_add(loss_sum, v);
    }
    umma::fence_before_sync();
    __syncthreads();
    if (threadIdx.x < 32) umma::tmem_free<64 * NG>(S.tmem_base);
}

PG_PH_READER(pg_phase_prof_read_mma)

template <typename ACC, typename LACC>
int train_mma(const pg_grid *g, int od, const float *xs, const float *targets, int64_t B, const float *feats,
              const uint8_t *baked, const float *conf, const float *params, float scale, int sig, ACC *gfeat,
              ACC *gconf, uint8_t *touched, ACC *gparams, LACC *loss_sum, float *dy_out, cudaStream_t s,
              const pg_cells *cells) {
    static DeviceOnce configured[18];
    CellMap cmap;
    cmap.cells = nullptr;
    for (int l = 0; l < PG_MAX_LEVELS; ++l) cmap.off[l] = -1;
    if (cells && cells->data) {
        cmap.cells = reinterpret_cast<const uint4 *>(cells->data);
        for (int l = 0; l < g->n_levels; ++l) cmap.off[l] = cells->off[l] >= 0 ? (int32_t)cells->off[l] : -1;
    }
    const int sms = device_sms();
    // tile pipelines per CTA (1 or 2)
    static const int groups = getenv("PG_TRAIN_GROUPS") && atoi(getenv("PG_TRAIN_GROUPS")) == 1 ? 1 : 2;
    const int64_t ntiles = (B + tm::kT - 1) / tm::kT;
    const int npm = g->log2_np <= 2 ? 4 : g->log2_np == 3 ? 8 : 16;   // probing range held in registers
    // warp-aggregated feature reductions (fast fp32 path, two pipelines per
    // CTA) when the probed levels have at most kAggRanges probing ranges
    static const int agg_ranges = getenv("PG_TRAIN_AGG_RANGES") ? atoi(getenv("PG_TRAIN_AGG_RANGES"))
                                                                 : tm::kAggRanges;   // 0 disables
    const bool agg = std::is_same<ACC, float>::value && groups == 2 && (g->n_f >> g->log2_np) <= agg_ranges;
#define PG_TRAIN_MMA(D_, NP_, NG_, IDX)                                                               \
    do {                                                                                              \
        auto kern = train_mma_kernel<float, D_, NP_, ACC, LACC, NG_>;                                 \
        const int smem = (int)sizeof(tm::SmemT<NG_>);                                                 \
        if (configured[IDX].first())                                                                  \
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);            \
        const int64_t want = (ntiles + NG_ - 1) / NG_, cap = (int64_t)sms * (2 / NG_);                \
        const int grd = (int)(want < cap ? want : cap);                                               \
        kern<<<grd, tm::kNT * NG_, smem, s>>>(*g, xs, targets, B, feats, feats, baked, conf, params, od, \
                                              scale, sig, gfeat, gconf, touched, gparams, loss_sum, dy_out, cmap); \
    } while (0)
#define PG_TRAIN_MMA_AGG(D_, NP_, IDX)                                                                \
    do {                                                                                              \
        auto kern = train_mma_kernel<float, D_, NP_, ACC, LACC, 2, true>;                             \
        const int smem = (int)sizeof(tm::SmemT<2>);                                                   \
        if (configured[IDX].first())                                                                  \
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);            \
        const int64_t want = (ntiles + 1) / 2, cap = (int64_t)sms;                                    \
        const int grd = (int)(want < cap ? want : cap);                                               \
        kern<<<grd, tm::kNT * 2, smem, s>>>(*g, xs, targets, B, feats, feats, baked, conf, params, od,   \
                                            scale, sig, gfeat, gconf, touched, gparams, loss_sum, dy_out, cmap); \
    } while (0)
#define PG_TRAIN_MMA_NG(D_, NP_, IDX)                                                                 \
    do {                                                                                              \
        if (agg) {                                                                                    \
            if constexpr (std::is_same<ACC, float>::value) PG_TRAIN_MMA_AGG(D_, NP_, (IDX) + 12);     \
        }                                                                                             \
        else if (groups == 2) PG_TRAIN_MMA(D_, NP_, 2, (IDX) + 6);                                    \
        else PG_TRAIN_MMA(D_, NP_, 1, IDX);                                                           \
    } while (0)
    if (g->d == 2) {
        if (npm == 4) PG_TRAIN_MMA_NG(2, 4, 0); else if (npm == 8) PG_TRAIN_MMA_NG(2, 8, 4); else PG_TRAIN_MMA_NG(2, 16, 1);
    } else {
        if (npm == 4) PG_TRAIN_MMA_NG(3, 4, 2); else if (npm == 8) PG_TRAIN_MMA_NG(3, 8, 5); else PG_TRAIN_MMA_NG(3, 16, 3);
    }
#undef PG_TRAIN_MMA_NG
#undef PG_TRAIN_MMA_AGG
#undef PG_TRAIN_MMA
    return check_launch("train_mma");
}

template int train_mma<float, double>(const pg_grid *, int, const float *, const float *, int64_t,
                                      const float *, const uint8_t *, const float *, const float *, float,
                                      int, float *, float *, uint8_t *, float *, double *, float *,
                                      cudaStream_t, const pg_cells *);
template int train_mma<fx_t, fx_t>(const pg_grid *, int, const float *, const float *, int64_t,
                                   const float *, const uint8_t *, const float *, const float *, float, int,
                                   fx_t *, fx_t *, uint8_t *, fx_t *, fx_t *, float *, cudaStream_t,
                                   const pg_cells *);

}  // namespace pg
