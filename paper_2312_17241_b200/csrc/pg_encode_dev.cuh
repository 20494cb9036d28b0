// Per-(point, level) encode forward / backward device routines for F = 2,
// shared by the fused decode and fused training kernels.  Arithmetic is the
// reference's (_core.pyx:36-54 forward blend order; straight-through
// backward, _core.pyx:179-202 / PAPER.md:403-409).
#pragma once

#include "pg_common.cuh"

namespace pg {
// 2^x by the SFU (MUFU.EX2; x <= 0 here, so no overflow handling needed)
__device__ __forceinline__ float exp2f_approx(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// 256-bit read-only global load (sm_100: LDG.E.ENL2.256); p 32-byte aligned
__device__ __forceinline__ void ld_nc_v8(const float *p, float (&v)[8]) {
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
        : "l"(p));
}

// Decode cell cache (pg_cells): per-level record offsets (uint4 units, -1 =
// not cached) into one buffer of per-cell records holding the 2^d resolved
// corner rows (binary16 F = 2, 4 B each) in corner order.
struct CellMap {
    const uint4 *cells;
    int32_t off[PG_MAX_LEVELS];
};

// Forward of a cached level: ONE 16 B (2-D) / 32 B (3-D) record load instead
// of 2^d index + row gathers; same weights, values and blend order as
// encode_level_fwd2, so bit-identical.
// L2 eviction-priority policies (createpolicy): the decode keeps its tables
// and cell records L2-resident (evict_last) while its 20 B/query of inputs
// and outputs stream through (evict_first)
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint4 ld_nc_v4_hint(const uint4 *p, uint64_t pol) {
    uint4 v;
    asm("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
        : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_nc_hint(const float *p, uint64_t pol) {
    float v;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_hint(float *p, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}

template <int D>
__device__ __forceinline__ float2 encode_level_fwd2_cell(const pg_grid &g, int l, const float (&x)[D],
                                                         const uint4 *__restrict__ rec, uint64_t pol = 0) {
    constexpr int C = 1 << D;
    const int res = g.res[l];
    int c[D];
    float t[D], omt[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        c[a] = cell_coord(x[a], res, t[a]);
        omt[a] = __fsub_rn(1.0f, t[a]);
    }
    // cached levels hold res^D <= 2^27 cells (the cache budget), so 32-bit
    // index math suffices
    int cell = c[D - 1];
#pragma unroll
    for (int a = D - 2; a >= 0; --a) cell = cell * res + c[a];
    uint32_t r[C];
    if constexpr (D == 2) {
        const uint4 v = pol ? ld_nc_v4_hint(rec + cell, pol) : __ldg(rec + cell);
        r[0] = v.x; r[1 % C] = v.y; r[2 % C] = v.z; r[3 % C] = v.w;
    } else {
        float v8[8];
        ld_nc_v8(reinterpret_cast<const float *>(rec + 2 * cell), v8);
#pragma unroll
        for (int k = 0; k < C; ++k) r[k] = __float_as_uint(v8[k % 8]);
    }
    float y0 = 0.0f, y1 = 0.0f;
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const float w = corner_weight<float, D>(k, t, omt);
        const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&r[k]));
        y0 = __fadd_rn(y0, __fmul_rn(w, f.x));
        y1 = __fadd_rn(y1, __fmul_rn(w, f.y));
    }
    return make_float2(y0, y1);
}

// fp32 cell records (the training tables, rebuilt every step): 2^d corners x
// 8 B per cell, read as 32-byte loads; same weights, values and blend order
// as encode_level_fwd2, so bit-identical
template <int D>
__device__ __forceinline__ float2 encode_level_fwd2_cell32(const pg_grid &g, int l, const float (&x)[D],
                                                           const uint4 *__restrict__ rec) {
    constexpr int C = 1 << D;
    const int res = g.res[l];
    int c[D];
    float t[D], omt[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        c[a] = cell_coord(x[a], res, t[a]);
        omt[a] = __fsub_rn(1.0f, t[a]);
    }
    int64_t cell = c[D - 1];
#pragma unroll
    for (int a = D - 2; a >= 0; --a) cell = cell * res + c[a];
    const float *p = reinterpret_cast<const float *>(rec + (int64_t)(C / 2) * cell);
    float f[2 * C];
#pragma unroll
    for (int h = 0; h < C / 4; ++h) {
        float f8[8];
        ld_nc_v8(p + 8 * h, f8);
#pragma unroll
        for (int i = 0; i < 8; ++i) f[8 * h + i] = f8[i];
    }
    float y0 = 0.0f, y1 = 0.0f;
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const float w = corner_weight<float, D>(k, t, omt);
        y0 = __fadd_rn(y0, __fmul_rn(w, f[2 * k]));
        y1 = __fadd_rn(y1, __fmul_rn(w, f[2 * k + 1]));
    }
    return make_float2(y0, y1);
}

// Forward: blended F=2 feature of point x at level l (bit-exact vs _core).
template <typename FT, int D>
__device__ __forceinline__ float2 encode_level_fwd2(const pg_grid &g, int l, const float (&x)[D],
                                                    const FT *__restrict__ feats,
                                                    const uint8_t *__restrict__ baked) {
    constexpr int C = 1 << D;
    const uint32_t nf_mask = (uint32_t)g.n_f - 1u, nc_mask = (uint32_t)g.n_c - 1u;
    const int res = g.res[l], kind = g.kind[l];
    int c[D];
    float t[D], omt[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        c[a] = cell_coord(x[a], res, t[a]);
        omt[a] = __fsub_rn(1.0f, t[a]);
    }
    int idx[C];
    float w[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
        w[k] = corner_weight<float, D>(k, t, omt);
        if (kind == PG_LEVEL_DENSE) {
            idx[k] = corner_dense<D>(k, c, res + 1);
        } else {
            const uint32_t h = corner_hash<D>(k, c, g.primary);
            if (kind == PG_LEVEL_HASHED) {
                idx[k] = (int)(h & nf_mask);
            } else {
                const int r = (int)(corner_hash<D>(k, c, g.aux) & nc_mask);
                idx[k] = (int)((h << g.log2_np) & nf_mask) +
                         (int)__ldg(baked + (int64_t)g.slot[l] * g.n_c + r);
            }
        }
    }
    const FT *tab = feats + (int64_t)l * g.n_f * 2;
    float2 f[C];
#pragma unroll
    for (int k = 0; k < C; ++k) f[k] = Feat<FT>::ld2(tab + (int64_t)idx[k] * 2);
    float y0 = 0.0f, y1 = 0.0f;
#pragma unroll
    for (int k = 0; k < C; ++k) {
        y0 = __fadd_rn(y0, __fmul_rn(w[k], f[k].x));
        y1 = __fadd_rn(y1, __fmul_rn(w[k], f[k].y));
    }
    return make_float2(y0, y1);
}

// encode_level_fwd2 for N_p = 4 probed levels with the probing range fetched
// whole (4 rows x F = 2: 32 B fp32 / 16 B fp16 — one sector) in parallel
// with the baked byte, the probe selected in registers: one L2 round trip
// instead of the dependent baked -> feature pair.  Identical arithmetic.
template <typename FT, int D>
__device__ __forceinline__ float2 encode_level_fwd2_rng(const pg_grid &g, int l, const float (&x)[D],
                                                        const FT *__restrict__ feats,
                                                        const uint8_t *__restrict__ baked) {
    if (g.kind[l] != PG_LEVEL_PROBED || g.log2_np != 2) return encode_level_fwd2<FT, D>(g, l, x, feats, baked);
    constexpr int C = 1 << D;
    const uint32_t nf_mask = (uint32_t)g.n_f - 1u, nc_mask = (uint32_t)g.n_c - 1u;
    const int res = g.res[l];
    int c[D];
    float t[D], omt[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        c[a] = cell_coord(x[a], res, t[a]);
        omt[a] = __fsub_rn(1.0f, t[a]);
    }
    const FT *tab = feats + (int64_t)l * g.n_f * 2;
    const uint8_t *bt = baked + (int64_t)g.slot[l] * g.n_c;
    float2 f[C];
    int bk[C];
    if constexpr (sizeof(FT) == 4) {
        float r[C][8];
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const uint32_t base = (corner_hash<D>(k, c, g.primary) << 2) & nf_mask;
            ld_nc_v8(reinterpret_cast<const float *>(tab) + (int64_t)base * 2, r[k]);
            bk[k] = (int)__ldg(bt + (corner_hash<D>(k, c, g.aux) & nc_mask));
        }
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const int j = bk[k];
            f[k].x = j == 0 ? r[k][0] : j == 1 ? r[k][2] : j == 2 ? r[k][4] : r[k][6];
            f[k].y = j == 0 ? r[k][1] : j == 1 ? r[k][3] : j == 2 ? r[k][5] : r[k][7];
        }
    } else {
        uint4 r[C];
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const uint32_t base = (corner_hash<D>(k, c, g.primary) << 2) & nf_mask;
            r[k] = __ldg(reinterpret_cast<const uint4 *>(tab + (int64_t)base * 2));
            bk[k] = (int)__ldg(bt + (corner_hash<D>(k, c, g.aux) & nc_mask));
        }
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const int j = bk[k];
            const uint32_t w = j == 0 ? r[k].x : j == 1 ? r[k].y : j == 2 ? r[k].z : r[k].w;
            f[k] = __half22float2(*reinterpret_cast<const __half2 *>(&w));
        }
    }
    float y0 = 0.0f, y1 = 0.0f;
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const float w = corner_weight<float, D>(k, t, omt);
        y0 = __fadd_rn(y0, __fmul_rn(w, f[k].x));
        y1 = __fadd_rn(y1, __fmul_rn(w, f[k].y));
    }
    return make_float2(y0, y1);
}

// Backward for one (point, level), F = 2, fp32: scatter w*up into the
// feature-gradient table (all N_p probes, softmax-weighted, for probed
// levels), the softmax-Jacobian term into gconf, and flag the row touched.
// ACC = float (vector reductions into L2) or fx_t (deterministic fixed point).
template <int NPMAX, typename ACC, bool FEATS = true>
__device__ __forceinline__ void encode_probe_reds(ACC *gb, ACC *gc, int n_p, const float (&sg)[NPMAX],
                                                  const float (&dots)[NPMAX], float s, float g0, float g1);

// Warp-aggregated feature-gradient reduction of one corner's probing range
// (AGG): lanes whose ranges start at the same row `base` (key; -1 = lane
// contributes nothing) are summed by a shuffle reduce-scatter of the
// range's 2*n_p floats (element i = sg[i/2] * (i odd ? g1 : g0)), then ONE
// coalesced reduction per distinct range and warp.  Called by all 32 lanes.
template <int NPMAX>
__device__ __forceinline__ void warp_agg_range_reds(float *gtab, int key, int n_p, const float (&sg)[NPMAX],
                                                    float g0, float g1) {
    static_assert(NPMAX <= 16, "a probing range of 2*N_p floats must fit one warp");
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned grp = __match_any_sync(full, key);
    unsigned todo = full;
    while (todo) {
        const int lead = __ffs(todo) - 1;
        const unsigned gmask = __shfl_sync(full, grp, lead);
        const int kb = __shfl_sync(full, key, lead);
        todo &= ~gmask;
        if (kb < 0) continue;
        const bool in = (gmask >> lane) & 1u;
        // step 1 (xor 16) from the contributions directly, then 8, 4, 2, 1:
        // lane l ends with the group's sum of element l
        float x[16];
        const bool u16 = (lane & 16) != 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            float lo = 0.0f, hi = 0.0f;
            if ((i >> 1) < NPMAX && in) lo = sg[(i >> 1) % NPMAX] * ((i & 1) ? g1 : g0);
            if (((i + 16) >> 1) < NPMAX && in) hi = sg[((i + 16) >> 1) % NPMAX] * ((i & 1) ? g1 : g0);
            const float send = u16 ? lo : hi, keep = u16 ? hi : lo;
            x[i] = keep + __shfl_xor_sync(full, send, 16);
        }
#pragma unroll
        for (int s = 8; s >= 1; s >>= 1) {
            const bool up = (lane & s) != 0;
#pragma unroll
            for (int i = 0; i < s; ++i) {
                const float send = up ? x[i] : x[i + s], keep = up ? x[i + s] : x[i];
                x[i] = keep + __shfl_xor_sync(full, send, s);
            }
        }
        if (lane < 2 * n_p) red_add(gtab + (int64_t)kb * 2 + lane, x[0]);
    }
}

// AGG: feature reductions of probed levels through warp_agg_range_reds (all
// 32 lanes must call; `valid` = this lane has a sample).  Dense / hashed
// levels and the confidence rows keep per-lane reductions.
template <int D, int NPMAX, typename ACC = float, bool LAZY = false, bool AGG = false>
__device__ __forceinline__ void encode_level_bwd2(const pg_grid &g, int l, const float (&x)[D],
                                                  float up0, float up1,
                                                  const float *__restrict__ feats,
                                                  const float *__restrict__ conf,
                                                  ACC *__restrict__ gfeat,
                                                  ACC *__restrict__ gconf,
                                                  uint8_t *__restrict__ touched,
                                                  bool touch_all = false, bool valid = true) {
    constexpr int C = 1 << D;
    const uint32_t nf_mask = (uint32_t)g.n_f - 1u, nc_mask = (uint32_t)g.n_c - 1u;
    const int res = g.res[l], kind = g.kind[l];
    const int n_p = 1 << g.log2_np;
    int c[D];
    float t[D], omt[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        c[a] = cell_coord(x[a], res, t[a]);
        omt[a] = __fsub_rn(1.0f, t[a]);
    }
    ACC *gtab = gfeat + (int64_t)l * g.n_f * 2;
    const float *ftab = feats + (int64_t)l * g.n_f * 2;
    float wk[C];
#pragma unroll
    for (int k = 0; k < C; ++k) wk[k] = corner_weight<float, D>(k, t, omt);
    if (kind != PG_LEVEL_PROBED) {
        if (!valid) return;
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const int lin = kind == PG_LEVEL_DENSE ? corner_dense<D>(k, c, res + 1)
                                                   : (int)(corner_hash<D>(k, c, g.primary) & nf_mask);
            red_add_v2(gtab + (int64_t)lin * 2, __fmul_rn(wk[k], up0), __fmul_rn(wk[k], up1));
        }
        return;
    }
    // Probed: resolve every corner's probing range and confidence row first
    // and issue ALL their loads before any arithmetic or reduction, so the
    // 2^d corners' L2 round trips overlap instead of serialising.
    // corners prefetched together (all 2^d: 0.576 vs 0.548 ms per C1 step,
    // spills at the 128-register cap)
    constexpr int PF = NPMAX <= 4 ? 2 : 1;
    int bs[C];
    int64_t crow[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
        bs[k] = (int)((corner_hash<D>(k, c, g.primary) << g.log2_np) & nf_mask);
        crow[k] = (int64_t)g.slot[l] * g.n_c + (int)(corner_hash<D>(k, c, g.aux) & nc_mask);
    }
#pragma unroll
    for (int k0 = 0; k0 < C; k0 += PF) {
        float cv[PF][NPMAX], fv[PF][NPMAX][2];
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const float *cr = conf + crow[k0 + u] * n_p;
            const float2 *fb = reinterpret_cast<const float2 *>(ftab + (int64_t)bs[k0 + u] * 2);
            if (NPMAX == 4 && n_p == 4) {
                // conf row: 16 B; probing range (4 probes x F=2): ONE 32-byte load
                const float4 c4 = __ldg(reinterpret_cast<const float4 *>(cr));
                float f8[8];
                ld_nc_v8(reinterpret_cast<const float *>(fb), f8);
                cv[u][0] = c4.x; cv[u][1 % NPMAX] = c4.y; cv[u][2 % NPMAX] = c4.z; cv[u][3 % NPMAX] = c4.w;
                fv[u][0][0] = f8[0]; fv[u][0][1] = f8[1]; fv[u][1 % NPMAX][0] = f8[2]; fv[u][1 % NPMAX][1] = f8[3];
                fv[u][2 % NPMAX][0] = f8[4]; fv[u][2 % NPMAX][1] = f8[5];
                fv[u][3 % NPMAX][0] = f8[6]; fv[u][3 % NPMAX][1] = f8[7];
            } else if (NPMAX >= 4 && n_p >= 4) {
                // groups of 4 probes: 16-byte conf load + 32-byte feature load
#pragma unroll
                for (int j0 = 0; j0 < NPMAX; j0 += 4)
                    if (j0 < n_p) {
                        const float4 c4 = __ldg(reinterpret_cast<const float4 *>(cr + j0));
                        float f8[8];
                        ld_nc_v8(reinterpret_cast<const float *>(fb + j0), f8);
                        cv[u][j0] = c4.x; cv[u][(j0 + 1) % NPMAX] = c4.y;
                        cv[u][(j0 + 2) % NPMAX] = c4.z; cv[u][(j0 + 3) % NPMAX] = c4.w;
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            fv[u][(j0 + i) % NPMAX][0] = f8[2 * i];
                            fv[u][(j0 + i) % NPMAX][1] = f8[2 * i + 1];
                        }
                    }
            } else {
#pragma unroll
                for (int j = 0; j < NPMAX; ++j)
                    if (j < n_p) {
                        cv[u][j] = __ldg(cr + j);
                        const float2 f = __ldg(fb + j);
                        fv[u][j][0] = f.x;
                        fv[u][j][1] = f.y;
                    }
            }
        }
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const int k = k0 + u;
            if (!LAZY && valid) touched[crow[k]] = 1;
            const float g0 = __fmul_rn(wk[k], up0), g1 = __fmul_rn(wk[k], up1);
            ACC *gc = gconf + crow[k] * n_p;
            ACC *gb = gtab + (int64_t)bs[k] * 2;
            float sg[NPMAX], dots[NPMAX];
            float mx = cv[u][0];
#pragma unroll
            for (int j = 1; j < NPMAX; ++j)
                if (j < n_p) mx = fmaxf(mx, cv[u][j]);
            // LAZY (the fast fp32 step): exp as one ex2.approx of a scaled
            // argument and one reciprocal instead of n_p IEEE divisions
            // (relative error ~1e-6 on the probe weights, inside the 1e-5
            // gradient bars; the parity-mode kernels keep the reference's
            // expf and division)
#ifndef PG_SM_EXACT
            constexpr bool kFastSm = LAZY;
#else
            constexpr bool kFastSm = false;
#endif
            float sum = 0.0f;
#pragma unroll
            for (int j = 0; j < NPMAX; ++j)
                if (j < n_p) {
                    sg[j] = kFastSm ? exp2f_approx(__fmul_rn(cv[u][j] - mx, 1.4426950408889634f))
                                    : expf(cv[u][j] - mx);
                    sum += sg[j];
                }
            const float inv = kFastSm ? __frcp_rn(sum) : 0.0f;
            // the reference's rounding: z /= sums (numpy_backend.py:128-130);
            // dot = f0*g0 + f1*g1 and s += sj*dot without FMA (_core.pyx:196-201)
            float s = 0.0f;
#pragma unroll
            for (int j = 0; j < NPMAX; ++j)
                if (j < n_p) {
                    sg[j] = kFastSm ? __fmul_rn(sg[j], inv) : __fdiv_rn(sg[j], sum);
                    dots[j] = __fadd_rn(__fmul_rn(fv[u][j][0], g0), __fmul_rn(fv[u][j][1], g1));
                    s = __fadd_rn(s, __fmul_rn(sg[j], dots[j]));
                }
            if (LAZY) {
                // A lookup that adds a normal (non-zero, non-subnormal: the
                // vector reductions flush subnormals) value to its gconf row
                // needs no flag: the lazy Adam also visits every row whose
                // gradient is non-zero.  Only all-zero contributions (zero
                // corner weight or upstream, equal dots, exp underflow) are
                // flagged -- a byte store on ~0% of lookups instead of all.
                bool live = false;
#pragma unroll
                for (int j = 0; j < NPMAX; ++j)
                    if (j < n_p) live |= fabsf(sg[j] * (dots[j] - s)) >= 1.17549435e-38f;
                // touch_all (data-parallel steps): every lookup flags its
                // row, so a row whose replicas' contributions cancel to an
                // exact 0.0 after the all-reduce is still updated, as the
                // reference's lazy Adam updates every touched row
                if ((!live || touch_all) && valid) touched[crow[k]] = 1;
            }
            if constexpr (AGG) {
                static_assert(std::is_same<ACC, float>::value, "AGG: fp32 reductions only");
                // confidence rows first: dots are dead during the shuffles
                if (valid) encode_probe_reds<NPMAX, ACC, false>(gb, gc, n_p, sg, dots, s, g0, g1);
                warp_agg_range_reds<NPMAX>(gtab, valid ? bs[k] : -1, n_p, sg, g0, g1);
            } else {
                encode_probe_reds<NPMAX, ACC>(gb, gc, n_p, sg, dots, s, g0, g1);
            }
        }
    }
}

// scatter of one probed corner: softmax-weighted feature grads over the
// probing range (16-byte vector reductions) + confidence-row gradient
template <int NPMAX, typename ACC, bool FEATS>
__device__ __forceinline__ void encode_probe_reds(ACC *gb, ACC *gc, int n_p, const float (&sg)[NPMAX],
                                                  const float (&dots)[NPMAX], float s, float g0, float g1) {
    if constexpr (FEATS) {
        if (n_p >= 2) {
#pragma unroll
            for (int j = 0; j < NPMAX; j += 2)
                if (j < n_p)
                    red_add_v4(gb + 2 * j, sg[j] * g0, sg[j] * g1, sg[j + 1] * g0, sg[j + 1] * g1);
        } else {
            red_add_v2(gb, sg[0] * g0, sg[0] * g1);
        }
    }
    {
        if (n_p >= 4) {
#pragma unroll
            for (int j = 0; j < NPMAX; j += 4)
                if (j < n_p)
                    red_add_v4(gc + j, sg[j] * (dots[j] - s), sg[j + 1] * (dots[j + 1] - s),
                               sg[j + 2] * (dots[j + 2] - s), sg[j + 3] * (dots[j + 3] - s));
        } else if (n_p == 2) {
            red_add_v2(gc, sg[0] * (dots[0] - s), sg[1] * (dots[1] - s));
        } else {
            red_add(gc, sg[0] * (dots[0] - s));
        }
    }
}

}  // namespace pg
