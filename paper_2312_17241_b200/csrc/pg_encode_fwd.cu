// Fused all-level encode forward (encoding.py:42-86 in one launch).
#include "pg_common.cuh"

namespace pg {

constexpr int kChunk = 128;

// =========================================================================
// Fused all-level forward.  Thread task = (point, level) mapped level-major
// inside a 128-point chunk so each warp serves 32 points of ONE level
// (uniform dense/hashed/probed branch, one table per warp).
// =========================================================================

template <typename T, typename FT, int D, int FC>
__global__ void __launch_bounds__(256) encode_fwd_kernel(const pg_grid g, const T *__restrict__ xs,
                                                         int64_t B, const FT *__restrict__ feats,
                                                         const uint8_t *__restrict__ baked,
                                                         const T *__restrict__ conf,
                                                         unsigned flags, T *__restrict__ y,
                                                         int32_t *__restrict__ bad) {
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
    const bool surrogate = (flags & PG_SURROGATE) != 0;
    const int64_t nchunks = (B + kChunk - 1) / kChunk;
    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        for (int i = threadIdx.x; i < L * kChunk; i += blockDim.x) {
            const int l = i / kChunk;
            const int64_t p = ch * kChunk + (i - l * kChunk);
            if (p >= B) continue;
            T x[D];
            bool oob = false;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                x[a] = xs[p * D + a];
                oob |= !(x[a] >= T(0) && x[a] <= T(1));
            }
            if (l == 0 && oob && bad) *bad = 1;
            const int res = lt.res[l], kind = lt.kind[l];
            int c[D];
            T t[D], omt[D];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                c[a] = cell_coord(x[a], res, t[a]);
                omt[a] = Ar<T>::sub(T(1), t[a]);
            }
            const FT *tab = feats + (int64_t)l * g.n_f * F;
            T acc[FC ? FC : PG_MAX_FEATURE];
#pragma unroll
            for (int q = 0; q < (FC ? FC : PG_MAX_FEATURE); ++q) acc[q] = T(0);
            int idx[C];
            T w[C];
#pragma unroll
            for (int k = 0; k < C; ++k) {
                w[k] = corner_weight<T, D>(k, t, omt);
                if (kind == PG_LEVEL_DENSE) {
                    idx[k] = corner_dense<D>(k, c, res + 1);
                } else {
                    const uint32_t h = corner_hash<D>(k, c, g.primary);
                    if (kind == PG_LEVEL_HASHED) {
                        idx[k] = (int)(h & nf_mask);
                    } else {
                        const int bs = (int)((h << g.log2_np) & nf_mask);
                        const int r = (int)(corner_hash<D>(k, c, g.aux) & nc_mask);
                        if (surrogate) {
                            idx[k] = -1 - r;  // remember the row; base re-derived below
                        } else {
                            idx[k] = bs + (int)__ldg(baked + (int64_t)lt.slot[l] * g.n_c + r);
                        }
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < C; ++k) {
                if (idx[k] >= 0) {
                    const FT *f = tab + (int64_t)idx[k] * F;
                    for (int q = 0; q < F; ++q)
                        acc[q] = Ar<T>::add(acc[q], Ar<T>::mul(w[k], (T)Feat<FT>::ld(f + q)));
                } else {
                    // softmax-mixture surrogate (numpy_backend.py:94-112), f64 checks
                    const int r = -1 - idx[k];
                    const int bs =
                        (int)((corner_hash<D>(k, c, g.primary) << g.log2_np) & nf_mask);
                    const T *cr = conf + ((int64_t)lt.slot[l] * g.n_c + r) * n_p;
                    T mx = cr[0];
                    for (int j = 1; j < n_p; ++j) mx = cr[j] > mx ? cr[j] : mx;
                    T sum = T(0);
                    for (int j = 0; j < n_p; ++j) sum += Ar<T>::exp(cr[j] - mx);
                    for (int q = 0; q < F; ++q) {
                        T mix = T(0);
                        for (int j = 0; j < n_p; ++j)
                            mix += (Ar<T>::exp(cr[j] - mx) / sum) *
                                   (T)Feat<FT>::ld(tab + (int64_t)(bs + j) * F + q);
                        acc[q] = Ar<T>::add(acc[q], Ar<T>::mul(w[k], mix));
                    }
                }
            }
            T *yo = y + p * (int64_t)L * F + (int64_t)l * F;
            for (int q = 0; q < F; ++q) yo[q] = acc[q];
        }
    }
}


static int encode_blocks(int64_t B) {
    const int sms = device_sms();
    const int64_t nchunks = (B + kChunk - 1) / kChunk;
    const int64_t cap = (int64_t)sms * 8;
    return (int)(nchunks < cap ? nchunks : cap);
}


template <typename T, typename FT>
static int launch_encode_fwd(const pg_grid *g, const T *xs, int64_t B, const FT *feats,
                             const uint8_t *baked, const T *conf, unsigned flags, T *y,
                             int32_t *bad, void *stream) {
    if (int e = validate_grid(g)) return e;
    PG_REQUIRE(!(flags & PG_SURROGATE) || conf != nullptr, "surrogate encoding needs confidences");
    if (B == 0) return PG_OK;
    const int grd = encode_blocks(B);
    cudaStream_t s = as_stream(stream);
    const bool f2 = g->feature_dim == 2;
#define PG_ENC_FWD(D_, FC_) \
    encode_fwd_kernel<T, FT, D_, FC_><<<grd, 256, 0, s>>>(*g, xs, B, feats, baked, conf, flags, y, bad)
    if (g->d == 2) {
        if (f2) PG_ENC_FWD(2, 2); else PG_ENC_FWD(2, 0);
    } else {
        if (f2) PG_ENC_FWD(3, 2); else PG_ENC_FWD(3, 0);
    }
#undef PG_ENC_FWD
    return check_launch("encode_fwd");
}


}  // namespace pg

using namespace pg;

extern "C" {

int pg_encode_fwd_f32(const pg_grid *grid, const float *xs, int64_t B, const void *feats,
                      const uint8_t *baked, const float *conf, unsigned flags, float *y,
                      int32_t *d_bad, void *stream) {
    if (flags & PG_HALF_FEATS)
        return launch_encode_fwd<float, __half>(grid, xs, B, (const __half *)feats, baked, conf,
                                                flags, y, d_bad, stream);
    return launch_encode_fwd<float, float>(grid, xs, B, (const float *)feats, baked, conf, flags, y,
                                           d_bad, stream);
}
int pg_encode_fwd_f64(const pg_grid *grid, const double *xs, int64_t B, const void *feats,
                      const uint8_t *baked, const double *conf, unsigned flags, double *y,
                      int32_t *d_bad, void *stream) {
    PG_REQUIRE(!(flags & PG_HALF_FEATS), "binary16 tables are float32-only");
    return launch_encode_fwd<double, double>(grid, xs, B, (const double *)feats, baked, conf, flags,
                                             y, d_bad, stream);
}
}  // extern "C"
