/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the probegrid hot path.
 *
 * A plain-C restatement of the reference's compiled kernels
 * (/root/reference/pkg/src/probegrid/backends/_core.pyx).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this
 * library, and only as the checker.  The product path (the CUDA library in
 * paper_2312_17241_b200/) never links or calls it.
 *
 * Arithmetic contract, copied from the reference build (pkg/setup.py:27-33):
 * compiled without FMA contraction or reassociation (see oracle/Makefile:
 * -ffp-contract=off, no -ffast-math), so float results are bit-identical to
 * the reference Cython core for the same inputs.  Loops run in batch order,
 * single-threaded, exactly as _core.pyx:4-6 documents.
 *
 * Every kernel exists for float (suffix _f32) and double (_f64).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* _core.pyx:17-23 — floor of the double product, clamped to [0, res-1]. */
static inline long orc_cell(double scaled, long res)
{
    long c = (long)floor(scaled);
    if (c > res - 1) c = res - 1;
    if (c < 0) c = 0;
    return c;
}

/* corner k carries offset bit (d-1-i) on axis i (numpy_backend.py:10,37-41) */
#define ORC_BIT(k, d, i) (((k) >> ((d) - 1 - (i))) & 1)

#define ORC_KERNELS(T, SFX, SQRT)                                              \
                                                                               \
/* _core.pyx:26-54 (dense_fwd): row-major vertex index, d-linear blend. */     \
void orc_dense_fwd_##SFX(const T *xs, int64_t B, int d, long res,              \
                         const T *feats, int F, T *out, int32_t *idx, T *wgt)  \
{                                                                              \
    const int C = 1 << d;                                                      \
    const long stride = res + 1;                                               \
    for (int64_t b = 0; b < B; ++b) {                                          \
        long cell[3];                                                          \
        T t[3];                                                                \
        for (int i = 0; i < d; ++i) {                                          \
            T x = xs[b * d + i];                                               \
            cell[i] = orc_cell((double)x * res, res);                          \
            t[i] = x * (T)res - (T)cell[i];                                    \
        }                                                                      \
        for (int k = 0; k < C; ++k) {                                          \
            T w = (T)1.0;                                                      \
            long lin = 0;                                                      \
            for (int i = 0; i < d; ++i) {                                      \
                int bit = ORC_BIT(k, d, i);                                    \
                w = w * (bit ? t[i] : ((T)1.0 - t[i]));                        \
            }                                                                  \
            for (int i = d - 1; i >= 0; --i)                                   \
                lin = lin * stride + (cell[i] + ORC_BIT(k, d, i));             \
            idx[b * C + k] = (int32_t)lin;                                     \
            wgt[b * C + k] = w;                                                \
            for (int q = 0; q < F; ++q)                                        \
                out[b * F + q] += w * feats[lin * F + q];                      \
        }                                                                      \
    }                                                                          \
}                                                                              \
                                                                               \
/* _core.pyx:57-84 (hashed_fwd): idx = XOR_i(v_i * pi_i) & (n_f - 1). */       \
void orc_hashed_fwd_##SFX(const T *xs, int64_t B, int d, long res,             \
                          uint32_t nf_mask, const T *feats, int F,             \
                          const uint32_t *primary, T *out, int32_t *idx,       \
                          T *wgt)                                              \
{                                                                              \
    const int C = 1 << d;                                                      \
    for (int64_t b = 0; b < B; ++b) {                                          \
        long cell[3];                                                          \
        T t[3];                                                                \
        for (int i = 0; i < d; ++i) {                                          \
            T x = xs[b * d + i];                                               \
            cell[i] = orc_cell((double)x * res, res);                          \
            t[i] = x * (T)res - (T)cell[i];                                    \
        }                                                                      \
        for (int k = 0; k < C; ++k) {                                          \
            T w = (T)1.0;                                                      \
            uint32_t h = 0;                                                    \
            for (int i = 0; i < d; ++i) {                                      \
                int bit = ORC_BIT(k, d, i);                                    \
                w = w * (bit ? t[i] : ((T)1.0 - t[i]));                        \
                h ^= (uint32_t)(cell[i] + bit) * primary[i];                   \
            }                                                                  \
            long lin = (long)(h & nf_mask);                                    \
            idx[b * C + k] = (int32_t)lin;                                     \
            wgt[b * C + k] = w;                                                \
            for (int q = 0; q < F; ++q)                                        \
                out[b * F + q] += w * feats[lin * F + q];                      \
        }                                                                      \
    }                                                                          \
}                                                                              \
                                                                               \
/* _core.pyx:87-122 (probed_fwd): base=(h<<log2Np)&(n_f-1),                    \
 * row=h2&(n_c-1), idx=base+baked[row] (paper Eq. 6). */                       \
void orc_probed_fwd_##SFX(const T *xs, int64_t B, int d, long res,             \
                          uint32_t nf_mask, uint32_t nc_mask, int log2_np,     \
                          const T *feats, int F, const uint8_t *baked,         \
                          const uint32_t *primary, const uint32_t *aux,        \
                          T *out, int32_t *base, int32_t *row, T *wgt)         \
{                                                                              \
    const int C = 1 << d;                                                      \
    for (int64_t b = 0; b < B; ++b) {                                          \
        long cell[3];                                                          \
        T t[3];                                                                \
        for (int i = 0; i < d; ++i) {                                          \
            T x = xs[b * d + i];                                               \
            cell[i] = orc_cell((double)x * res, res);                          \
            t[i] = x * (T)res - (T)cell[i];                                    \
        }                                                                      \
        for (int k = 0; k < C; ++k) {                                          \
            T w = (T)1.0;                                                      \
            uint32_t h = 0, h2 = 0;                                            \
            for (int i = 0; i < d; ++i) {                                      \
                int bit = ORC_BIT(k, d, i);                                    \
                uint32_t v = (uint32_t)(cell[i] + bit);                        \
                w = w * (bit ? t[i] : ((T)1.0 - t[i]));                        \
                h ^= v * primary[i];                                           \
                h2 ^= v * aux[i];                                              \
            }                                                                  \
            long bs = (long)((h << log2_np) & nf_mask);                        \
            long r = (long)(h2 & nc_mask);                                     \
            long lin = bs + (long)baked[r];                                    \
            base[b * C + k] = (int32_t)bs;                                     \
            row[b * C + k] = (int32_t)r;                                       \
            wgt[b * C + k] = w;                                                \
            for (int q = 0; q < F; ++q)                                        \
                out[b * F + q] += w * feats[lin * F + q];                      \
        }                                                                      \
    }                                                                          \
}                                                                              \
                                                                               \
/* _core.pyx:125-137 (indexed_bwd): gfeat[idx] += w * up, batch order. */      \
void orc_indexed_bwd_##SFX(const T *up, int64_t B, int F, const int32_t *idx,  \
                           const T *wgt, int C, T *gfeat)                      \
{                                                                              \
    for (int64_t b = 0; b < B; ++b)                                            \
        for (int k = 0; k < C; ++k) {                                          \
            long lin = idx[b * C + k];                                         \
            T w = wgt[b * C + k];                                              \
            for (int q = 0; q < F; ++q)                                        \
                gfeat[lin * F + q] += w * up[b * F + q];                       \
        }                                                                      \
}                                                                              \
                                                                               \
/* _core.pyx:163-221 (probed_bwd): straight-through scatter.  F == 2 takes     \
 * the reference's flat-pointer path (179-202), others the generic one         \
 * (203-221); both are restated so rounding matches term for term. */          \
void orc_probed_bwd_##SFX(const T *up, int64_t B, int F, const int32_t *base,  \
                          const int32_t *inv, const T *wgt, int C,             \
                          const T *smu, int n_p, const T *feats, T *gfeat,     \
                          T *gconf_u)                                          \
{                                                                              \
    T dots[256];                                                               \
    T g[16];                                                                   \
    for (int64_t b = 0; b < B; ++b)                                            \
        for (int k = 0; k < C; ++k) {                                          \
            long bs = base[b * C + k];                                         \
            long iv = inv[b * C + k];                                          \
            T w = wgt[b * C + k];                                              \
            const T *sp = smu + iv * n_p;                                      \
            T *cp = gconf_u + iv * n_p;                                        \
            T s = (T)0.0;                                                      \
            if (F == 2) {                                                      \
                T g0 = w * up[b * 2 + 0];                                      \
                T g1 = w * up[b * 2 + 1];                                      \
                const T *fp = feats + bs * 2;                                  \
                T *gp = gfeat + bs * 2;                                        \
                for (int j = 0; j < n_p; ++j) {                                \
                    T sj = sp[j];                                              \
                    T dot = fp[2 * j] * g0 + fp[2 * j + 1] * g1;               \
                    gp[2 * j] += sj * g0;                                      \
                    gp[2 * j + 1] += sj * g1;                                  \
                    dots[j] = dot;                                             \
                    s += sj * dot;                                             \
                }                                                              \
            } else {                                                           \
                for (int q = 0; q < F; ++q) g[q] = w * up[b * F + q];          \
                for (int j = 0; j < n_p; ++j) {                                \
                    T sj = sp[j];                                              \
                    T dot = (T)0.0;                                            \
                    for (int q = 0; q < F; ++q) {                              \
                        dot += feats[(bs + j) * F + q] * g[q];                 \
                        gfeat[(bs + j) * F + q] += sj * g[q];                  \
                    }                                                          \
                    dots[j] = dot;                                             \
                    s += sj * dot;                                             \
                }                                                              \
            }                                                                  \
            for (int j = 0; j < n_p; ++j) cp[j] += sp[j] * (dots[j] - s);      \
        }                                                                      \
}                                                                              \
                                                                               \
/* _core.pyx:224-272 (adam_rebake_rows): lazy Adam on touched rows with        \
 * bias correction by reciprocal multiply, then strict-'>' argmax re-bake. */  \
void orc_adam_rebake_rows_##SFX(T *conf, T *m, T *v, int n_p, uint8_t *baked,  \
                                const int32_t *rows_u, int64_t U,              \
                                const T *gconf_u, double corr1, double corr2,  \
                                double lr, double beta1, double beta2,         \
                                double eps)                                    \
{                                                                              \
    const T b1 = (T)beta1, b2 = (T)beta2;                                      \
    const T nb1 = (T)(1.0 - beta1), nb2 = (T)(1.0 - beta2);                    \
    const T ic1 = (T)(1.0 / corr1), ic2 = (T)(1.0 / corr2);                    \
    const T flr = (T)lr, feps = (T)eps;                                        \
    for (int64_t i = 0; i < U; ++i) {                                          \
        long r = rows_u[i];                                                    \
        T *mp = m + r * n_p, *vp = v + r * n_p, *cp = conf + r * n_p;          \
        const T *gp = gconf_u + i * n_p;                                       \
        for (int j = 0; j < n_p; ++j) {                                        \
            T gj = gp[j];                                                      \
            mp[j] = b1 * mp[j] + nb1 * gj;                                     \
            vp[j] = b2 * vp[j] + nb2 * (gj * gj);                              \
        }                                                                      \
        for (int j = 0; j < n_p; ++j) {                                        \
            T mm = mp[j] * ic1;                                                \
            T vv = vp[j] * ic2;                                                \
            cp[j] = cp[j] - flr * mm / (SQRT(vv) + feps);                      \
        }                                                                      \
        T best = cp[0];                                                        \
        uint8_t best_j = 0;                                                    \
        for (int j = 1; j < n_p; ++j)                                          \
            if (cp[j] > best) { best = cp[j]; best_j = (uint8_t)j; }           \
        baked[r] = best_j;                                                     \
    }                                                                          \
}                                                                              \
                                                                               \
/* _core.pyx:275-289 (linear_rows): out = x @ W + b row by row, bias first,    \
 * inputs summed in order, optional ReLU. */                                   \
void orc_linear_rows_##SFX(const T *xs, int64_t B, int fin, const T *w,        \
                           const T *bias, int fout, T *out, int relu)          \
{                                                                              \
    for (int64_t b = 0; b < B; ++b)                                            \
        for (int j = 0; j < fout; ++j) {                                       \
            T acc = bias[j];                                                   \
            for (int i = 0; i < fin; ++i) acc += xs[b * fin + i] * w[i * fout + j]; \
            if (relu && acc < 0) acc = (T)0.0;                                 \
            out[b * fout + j] = acc;                                           \
        }                                                                      \
}                                                                              \
                                                                               \
/* _core.pyx:292-298 (sigmoid_rows): logistic evaluated in double. */          \
void orc_sigmoid_rows_##SFX(T *xs, int64_t n)                                  \
{                                                                              \
    for (int64_t i = 0; i < n; ++i)                                            \
        xs[i] = (T)(1.0 / (1.0 + exp(-(double)xs[i])));                        \
}

ORC_KERNELS(float, f32, sqrtf)
ORC_KERNELS(double, f64, sqrt)

/* _core.pyx:140-160 (dedup_rows): first-encounter unique rows + inverse.
 * `mark` is caller scratch of n_c int32; returns U. */
int64_t orc_dedup_rows(const int32_t *row, int64_t n, int32_t *mark, int64_t n_c,
                       int32_t *rows_u, int32_t *inv)
{
    for (int64_t i = 0; i < n_c; ++i) mark[i] = -1;
    int32_t u = 0;
    for (int64_t i = 0; i < n; ++i) {
        int32_t r = row[i];
        if (mark[r] < 0) {
            mark[r] = u;
            rows_u[u] = r;
            ++u;
        }
        inv[i] = mark[r];
    }
    return u;
}

/* OpenBLAS 0.3.30 (SkylakeX) sgemm order for the MLP weight gradient
 * W_grad += a^T @ delta (mlp.py:81; OpenBLAS is a numpy dependency, not part
 * of the reference tree): C = 0; the K loop (samples) is blocked by Q = 448,
 * the last two blocks balanced (a remainder in (Q, 2Q) is split in half,
 * driver/level3 GEMM_Q logic); inside a block each C element is ONE
 * sequential fused-multiply-add chain from 0; block results are added to C in
 * order.  Then the numpy in-place add into gw.  Bias: delta.sum(axis=0) is a
 * sequential sum over rows (mlp.py:82).  Pinned against numpy in
 * tests/test_oracle.py::test_openblas_wgrad_order. */
void orc_wgrad_blas_f32(const float *a, int64_t K, int fin, const float *d, int fout,
                        float *gw, float *gb)
{
    const int64_t Q = 448;
    for (int i = 0; i < fin; ++i)
        for (int j = 0; j < fout; ++j) {
            float c = 0.0f;
            for (int64_t ls = 0; ls < K;) {
                int64_t ml = K - ls;
                if (ml >= 2 * Q) ml = Q;
                else if (ml > Q) ml = ml / 2;
                float acc = 0.0f;
                for (int64_t k = ls; k < ls + ml; ++k) acc = fmaf(a[k * fin + i], d[k * fout + j], acc);
                c = c + acc;
                ls += ml;
            }
            gw[(int64_t)i * fout + j] = gw[(int64_t)i * fout + j] + c;
        }
    for (int j = 0; j < fout; ++j) {
        float s = 0.0f;
        for (int64_t k = 0; k < K; ++k) s = s + d[k * fout + j];
        gb[j] = gb[j] + s;
    }
}
