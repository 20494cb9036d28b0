// Fused all-level encode backward (encoding.py:89-133 in one launch).
#include "pg_common.cuh"

namespace pg {

constexpr int kChunk = 128;

// =========================================================================
// Fused all-level backward (encoding.py:119-133 + trainer.py:138-148):
// recompute geometry, scatter d-linear-weighted upstream into gfeat; for
// probed levels spread over all N_p probes with the row softmax and add the
// softmax-Jacobian term to gconf (straight-through), and
// flag the row as touched (every lookup, including zero-weight corners —
// encoding.py:111 dedups over all B*2^d rows).
// Softmax uses the per-row max (the reference shifts by the global max of the
// gathered rows, numpy_backend.py:115-131: mathematically identical).
// =========================================================================
template <typename T, int D, int FC, int NPMAX, typename ACC>
__global__ void __launch_bounds__(256) encode_bwd_kernel(
    const pg_grid g, const T *__restrict__ xs, int64_t B, const T *__restrict__ dy,
    const T *__restrict__ feats, const T *__restrict__ conf, ACC *__restrict__ gfeat,
    ACC *__restrict__ gconf, uint8_t *__restrict__ touched) {
    __shared__ LevelTab lt;
    const int L = g.n_levels;
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        lt.res[i] = g.res[i];
        lt.kind[i] = g.kind[i];
        lt.slot[i] = g.slot[i];
    }
    __syncthreads();
    constexpr int C = 1 << D;
    const int F = FC ? FC : g.feature_dim;
    const uint32_t nf_mask = (uint32_t)g.n_f - 1u, nc_mask = (uint32_t)g.n_c - 1u;
    const int n_p = 1 << g.log2_np;
    const int64_t nchunks = (B + kChunk - 1) / kChunk;
    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        for (int i = threadIdx.x; i < L * kChunk; i += blockDim.x) {
            const int l = i / kChunk;
            const int64_t p = ch * kChunk + (i - l * kChunk);
            if (p >= B) continue;
            const int res = lt.res[l], kind = lt.kind[l];
            int c[D];
            T t[D], omt[D];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                c[a] = cell_coord(xs[p * D + a], res, t[a]);
                omt[a] = Ar<T>::sub(T(1), t[a]);
            }
            T up[FC ? FC : PG_MAX_FEATURE];
            const T *dyp = dy + p * (int64_t)L * F + (int64_t)l * F;
            for (int q = 0; q < F; ++q) up[q] = dyp[q];
            ACC *gtab = gfeat + (int64_t)l * g.n_f * F;
            const T *ftab = feats + (int64_t)l * g.n_f * F;
#pragma unroll(FC == 2 && NPMAX > 0 ? C : 1)
            for (int k = 0; k < C; ++k) {
                const T w = corner_weight<T, D>(k, t, omt);
                T gq[FC ? FC : PG_MAX_FEATURE];
                for (int q = 0; q < F; ++q) gq[q] = Ar<T>::mul(w, up[q]);
                if (kind != PG_LEVEL_PROBED) {
                    const int lin = kind == PG_LEVEL_DENSE
                                        ? corner_dense<D>(k, c, res + 1)
                                        : (int)(corner_hash<D>(k, c, g.primary) & nf_mask);
                    ACC *dst = gtab + (int64_t)lin * F;
                    if constexpr (FC == 2 && sizeof(T) == 4) {
                        red_add_v2((ACC *)dst, gq[0], gq[1]);
                    } else {
                        for (int q = 0; q < F; ++q) red_add(dst + q, gq[q]);
                    }
                    continue;
                }
                const int bs = (int)((corner_hash<D>(k, c, g.primary) << g.log2_np) & nf_mask);
                const int r = (int)(corner_hash<D>(k, c, g.aux) & nc_mask);
                const int64_t crow = (int64_t)lt.slot[l] * g.n_c + r;
                touched[crow] = 1;
                const T *cr = conf + crow * n_p;
                ACC *gc = gconf + crow * n_p;
                const T *fb = ftab + (int64_t)bs * F;
                ACC *gb = gtab + (int64_t)bs * F;
                if constexpr (NPMAX > 0) {
                    T sg[NPMAX], dots[NPMAX];
                    T mx = cr[0];
#pragma unroll
                    for (int j = 1; j < NPMAX; ++j)
                        if (j < n_p) mx = cr[j] > mx ? cr[j] : mx;
                    T sum = T(0);
#pragma unroll
                    for (int j = 0; j < NPMAX; ++j)
                        if (j < n_p) {
                            sg[j] = Ar<T>::exp(cr[j] - mx);
                            sum += sg[j];
                        }
                    // reference rounding: z /= sums; dot and s without FMA
                    T s = T(0);
#pragma unroll
                    for (int j = 0; j < NPMAX; ++j)
                        if (j < n_p) {
                            sg[j] = Ar<T>::div(sg[j], sum);
                            T dot = T(0);
                            for (int q = 0; q < F; ++q) dot = Ar<T>::add(dot, Ar<T>::mul(fb[j * F + q], gq[q]));
                            dots[j] = dot;
                            s = Ar<T>::add(s, Ar<T>::mul(sg[j], dot));
                        }
                    if constexpr (FC == 2 && sizeof(T) == 4) {
                        // N_p*F contiguous floats, 16B aligned when n_p >= 2
                        if (n_p >= 2) {
#pragma unroll
                            for (int j = 0; j < NPMAX; j += 2)
                                if (j < n_p)
                                    red_add_v4((ACC *)gb + 2 * j, sg[j] * gq[0], sg[j] * gq[1],
                                               sg[j + 1] * gq[0], sg[j + 1] * gq[1]);
                        } else {
                            red_add_v2((ACC *)gb, sg[0] * gq[0], sg[0] * gq[1]);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < NPMAX; ++j)
                            if (j < n_p)
                                for (int q = 0; q < F; ++q) red_add(gb + j * F + q, sg[j] * gq[q]);
                    }
                    if constexpr (sizeof(T) == 4) {
                        if (n_p >= 4) {
#pragma unroll
                            for (int j = 0; j < NPMAX; j += 4)
                                if (j < n_p)
                                    red_add_v4((ACC *)gc + j, sg[j] * (dots[j] - s),
                                               sg[j + 1] * (dots[j + 1] - s),
                                               sg[j + 2] * (dots[j + 2] - s),
                                               sg[j + 3] * (dots[j + 3] - s));
                        } else if (n_p == 2) {
                            red_add_v2((ACC *)gc, sg[0] * (dots[0] - s), sg[1] * (dots[1] - s));
                        } else {
                            red_add(gc, sg[0] * (dots[0] - s));
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < NPMAX; ++j)
                            if (j < n_p) red_add(gc + j, sg[j] * (dots[j] - s));
                    }
                } else {
                    // long probing ranges: three passes, nothing kept per probe
                    T mx = cr[0];
                    for (int j = 1; j < n_p; ++j) mx = cr[j] > mx ? cr[j] : mx;
                    T sum = T(0);
                    for (int j = 0; j < n_p; ++j) sum += Ar<T>::exp(cr[j] - mx);
                    T s = T(0);
                    for (int j = 0; j < n_p; ++j) {
                        T dot = T(0);
                        for (int q = 0; q < F; ++q) dot = Ar<T>::add(dot, Ar<T>::mul(fb[j * F + q], gq[q]));
                        s = Ar<T>::add(s, Ar<T>::mul(Ar<T>::div(Ar<T>::exp(cr[j] - mx), sum), dot));
                    }
                    for (int j = 0; j < n_p; ++j) {
                        const T sj = Ar<T>::div(Ar<T>::exp(cr[j] - mx), sum);
                        T dot = T(0);
                        for (int q = 0; q < F; ++q) {
                            dot = Ar<T>::add(dot, Ar<T>::mul(fb[j * F + q], gq[q]));
                            red_add(gb + j * F + q, sj * gq[q]);
                        }
                        red_add(gc + j, sj * (dot - s));
                    }
                }
            }
        }
    }
}


static int encode_blocks(int64_t B) {
    const int sms = device_sms();
    const int64_t nchunks = (B + kChunk - 1) / kChunk;
    const int64_t cap = (int64_t)sms * 8;
    return (int)(nchunks < cap ? nchunks : cap);
}


template <typename T, typename ACC = T>
static int launch_encode_bwd(const pg_grid *g, const T *xs, int64_t B, const T *dy,
                             const T *feats, const T *conf, ACC *gfeat, ACC *gconf, uint8_t *touched,
                             void *stream) {
    if (int e = validate_grid(g)) return e;
    bool any_probed = false;
    for (int l = 0; l < g->n_levels; ++l) any_probed |= g->kind[l] == PG_LEVEL_PROBED;
    PG_REQUIRE(!any_probed || (conf && gconf && touched), "probed levels need conf/gconf/touched");
    if (B == 0) return PG_OK;
    const int grd = encode_blocks(B);
    cudaStream_t s = as_stream(stream);
    const bool f2 = g->feature_dim == 2;
    const int n_p = 1 << g->log2_np;
#define PG_ENC_BWD(D_, FC_, NP_) \
    encode_bwd_kernel<T, D_, FC_, NP_, ACC><<<grd, 256, 0, s>>>(*g, xs, B, dy, feats, conf, gfeat, gconf, touched)
#define PG_ENC_BWD_NP(D_, FC_)                   \
    do {                                         \
        if (FC_ == 0) PG_ENC_BWD(D_, 0, 0);       \
        else if (n_p <= 4) PG_ENC_BWD(D_, 2, 4);   \
        else if (n_p <= 16) PG_ENC_BWD(D_, 2, 16); \
        else PG_ENC_BWD(D_, FC_, 0);             \
    } while (0)
    if (g->d == 2) {
        if (f2) PG_ENC_BWD_NP(2, 2); else PG_ENC_BWD_NP(2, 0);
    } else {
        if (f2) PG_ENC_BWD_NP(3, 2); else PG_ENC_BWD_NP(3, 0);
    }
#undef PG_ENC_BWD_NP
#undef PG_ENC_BWD
    return check_launch("encode_bwd");
}


}  // namespace pg

using namespace pg;

extern "C" {

int pg_encode_bwd_f32(const pg_grid *grid, const float *xs, int64_t B, const float *dy,
                      const float *feats, const float *conf, float *gfeat, float *gconf,
                      uint8_t *touched, void *stream) {
    return launch_encode_bwd<float>(grid, xs, B, dy, feats, conf, gfeat, gconf, touched, stream);
}
int pg_encode_bwd_f64(const pg_grid *grid, const double *xs, int64_t B, const double *dy,
                      const double *feats, const double *conf, double *gfeat, double *gconf,
                      uint8_t *touched, void *stream) {
    return launch_encode_bwd<double>(grid, xs, B, dy, feats, conf, gfeat, gconf, touched, stream);
}
int pg_encode_bwd_det_f32(const pg_grid *grid, const float *xs, int64_t B, const float *dy,
                          const float *feats, const float *conf, uint64_t *gfeat_fx,
                          uint64_t *gconf_fx, uint8_t *touched, void *stream) {
    return launch_encode_bwd<float, fx_t>(grid, xs, B, dy, feats, conf, (fx_t *)gfeat_fx,
                                          (fx_t *)gconf_fx, touched, stream);
}

}  // extern "C"
