// Per-(point, level) encode forward / backward device routines for F = 2,
// shared by the fused decode and fused training kernels.  Arithmetic is the
// reference's (_core.pyx:36-54 forward blend order; straight-through
// backward, _core.pyx:179-202 / PAPER.md:403-409).
#pragma once

#include "pg_common.cuh"

namespace pg {

struct LevelGeo2 {
    int res, kind, slot;
};

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

// Backward for one (point, level), F = 2, fp32: scatter w*up into the
// feature-gradient table (all N_p probes, softmax-weighted, for probed
// levels), the softmax-Jacobian term into gconf, and flag the row touched.
template <int D, int NPMAX>
__device__ __forceinline__ void encode_level_bwd2(const pg_grid &g, int l, const float (&x)[D],
                                                  float up0, float up1,
                                                  const float *__restrict__ feats,
                                                  const float *__restrict__ conf,
                                                  float *__restrict__ gfeat,
                                                  float *__restrict__ gconf,
                                                  uint8_t *__restrict__ touched) {
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
    float *gtab = gfeat + (int64_t)l * g.n_f * 2;
    const float *ftab = feats + (int64_t)l * g.n_f * 2;
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const float w = corner_weight<float, D>(k, t, omt);
        const float g0 = __fmul_rn(w, up0), g1 = __fmul_rn(w, up1);
        if (kind != PG_LEVEL_PROBED) {
            const int lin = kind == PG_LEVEL_DENSE ? corner_dense<D>(k, c, res + 1)
                                                   : (int)(corner_hash<D>(k, c, g.primary) & nf_mask);
            red_add_v2(gtab + (int64_t)lin * 2, g0, g1);
            continue;
        }
        const int bs = (int)((corner_hash<D>(k, c, g.primary) << g.log2_np) & nf_mask);
        const int r = (int)(corner_hash<D>(k, c, g.aux) & nc_mask);
        const int64_t crow = (int64_t)g.slot[l] * g.n_c + r;
        touched[crow] = 1;
        const float *cr = conf + crow * n_p;
        float *gc = gconf + crow * n_p;
        const float *fb = ftab + (int64_t)bs * 2;
        float *gb = gtab + (int64_t)bs * 2;
        float sg[NPMAX], dots[NPMAX];
        float mx = cr[0];
#pragma unroll
        for (int j = 1; j < NPMAX; ++j)
            if (j < n_p) mx = fmaxf(mx, cr[j]);
        float sum = 0.0f;
#pragma unroll
        for (int j = 0; j < NPMAX; ++j)
            if (j < n_p) {
                sg[j] = expf(cr[j] - mx);
                sum += sg[j];
            }
        const float inv = 1.0f / sum;
        float s = 0.0f;
#pragma unroll
        for (int j = 0; j < NPMAX; ++j)
            if (j < n_p) {
                sg[j] *= inv;
                const float2 f = __ldg(reinterpret_cast<const float2 *>(fb) + j);
                dots[j] = f.x * g0 + f.y * g1;
                s += sg[j] * dots[j];
            }
        if (n_p >= 2) {
#pragma unroll
            for (int j = 0; j < NPMAX; j += 2)
                if (j < n_p)
                    red_add_v4(gb + 2 * j, sg[j] * g0, sg[j] * g1, sg[j + 1] * g0, sg[j + 1] * g1);
        } else {
            red_add_v2(gb, sg[0] * g0, sg[0] * g1);
        }
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
