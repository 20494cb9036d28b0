// Multiresolution learned-hash-probing encoding on sm_100a: per-level
// protocol kernels (replacing _core.pyx's dense/hashed/probed_fwd,
// indexed_bwd, probed_bwd, dedup_rows) and the fused all-level encode
// forward / backward used by the device-resident API.
#include "pg_common.cuh"

namespace pg {

// =========================================================================
// Protocol forward: one level, one thread per point, corners in order
// (_core.pyx:26-122).  out is accumulated in place (the reference wrapper
// zero-initialises it, cython_backend.py:27).
// =========================================================================
template <typename T, int D, int KIND>
__global__ void level_fwd_kernel(const T *__restrict__ xs, int64_t B, int res, uint32_t nf_mask,
                                 uint32_t nc_mask, int log2_np, const T *__restrict__ feats, int F,
                                 const uint8_t *__restrict__ baked, uint3 pr, uint3 ax,
                                 T *__restrict__ out, int32_t *__restrict__ ib,
                                 int32_t *__restrict__ row, T *__restrict__ wgt) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    constexpr int C = 1 << D;
    const uint32_t prim[3] = {pr.x, pr.y, pr.z};
    const uint32_t auxp[3] = {ax.x, ax.y, ax.z};
    int c[D];
    T t[D], omt[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
        c[i] = cell_coord(xs[b * D + i], res, t[i]);
        omt[i] = Ar<T>::sub(T(1), t[i]);
    }
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const T w = corner_weight<T, D>(k, t, omt);
        int lin;
        if (KIND == PG_LEVEL_DENSE) {
            lin = corner_dense<D>(k, c, res + 1);
            ib[b * C + k] = lin;
        } else if (KIND == PG_LEVEL_HASHED) {
            lin = (int)(corner_hash<D>(k, c, prim) & nf_mask);
            ib[b * C + k] = lin;
        } else {
            const int bs = (int)((corner_hash<D>(k, c, prim) << log2_np) & nf_mask);
            const int r = (int)(corner_hash<D>(k, c, auxp) & nc_mask);
            lin = bs + (int)baked[r];
            ib[b * C + k] = bs;
            row[b * C + k] = r;
        }
        wgt[b * C + k] = w;
        for (int q = 0; q < F; ++q)
            out[b * F + q] = Ar<T>::add(out[b * F + q], Ar<T>::mul(w, feats[(int64_t)lin * F + q]));
    }
}

template <typename T, int KIND>
static int launch_level_fwd(const T *xs, int64_t B, int d, int64_t res, uint32_t nf_mask,
                            uint32_t nc_mask, int log2_np, const T *feats, int F,
                            const uint8_t *baked, const uint32_t *pr, const uint32_t *ax, T *out,
                            int32_t *ib, int32_t *row, T *wgt, void *stream) {
    PG_REQUIRE(d == 2 || d == 3, "d must be 2 or 3");
    PG_REQUIRE(F >= 1, "feature dim must be positive");
    PG_REQUIRE(res >= 1 && res < (1 << 24), "resolution out of range");
    if (B == 0) return PG_OK;
    uint3 p3 = make_uint3(0, 0, 0), a3 = make_uint3(0, 0, 0);
    if (pr) p3 = make_uint3(pr[0], pr[1], d > 2 ? pr[2] : 0);
    if (ax) a3 = make_uint3(ax[0], ax[1], d > 2 ? ax[2] : 0);
    const int blk = 128;
    const int grd = grid_for(B, blk);
    if (d == 2)
        level_fwd_kernel<T, 2, KIND><<<grd, blk, 0, as_stream(stream)>>>(
            xs, B, (int)res, nf_mask, nc_mask, log2_np, feats, F, baked, p3, a3, out, ib, row, wgt);
    else
        level_fwd_kernel<T, 3, KIND><<<grd, blk, 0, as_stream(stream)>>>(
            xs, B, (int)res, nf_mask, nc_mask, log2_np, feats, F, baked, p3, a3, out, ib, row, wgt);
    return check_launch("level_fwd");
}

// =========================================================================
// Protocol backward (_core.pyx:125-137, 163-221): one thread per (b, k);
// accumulation by atomics, so only the set of adds matches the reference,
// not their order (the reference's own cross-backend bar, test_backends.py:
// 67-106, is rtol=atol=1e-5 in fp32).
// =========================================================================
template <typename T>
__global__ void indexed_bwd_kernel(const T *__restrict__ up, int64_t B, int F,
                                   const int32_t *__restrict__ idx, const T *__restrict__ wgt,
                                   int C, T *__restrict__ gfeat) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B * C) return;
    const int64_t b = i / C;
    const int64_t lin = idx[i];
    const T w = wgt[i];
    for (int q = 0; q < F; ++q) red_add(gfeat + lin * F + q, Ar<T>::mul(w, up[b * F + q]));
}

template <typename T>
__global__ void probed_bwd_kernel(const T *__restrict__ up, int64_t B, int F,
                                  const int32_t *__restrict__ base, const int32_t *__restrict__ inv,
                                  const T *__restrict__ wgt, int C, const T *__restrict__ smu,
                                  int n_p, const T *__restrict__ feats, T *__restrict__ gfeat,
                                  T *__restrict__ gconf_u) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B * C) return;
    const int64_t b = i / C;
    const int64_t bs = base[i];
    const int64_t iv = inv[i];
    const T w = wgt[i];
    T g[PG_MAX_FEATURE];
    for (int q = 0; q < F; ++q) g[q] = Ar<T>::mul(w, up[b * F + q]);
    // pass 1: s = sum_j sigma_j <f_{base+j}, g>
    T s = T(0);
    for (int j = 0; j < n_p; ++j) {
        T dot = T(0);
        for (int q = 0; q < F; ++q) dot = Ar<T>::add(dot, Ar<T>::mul(feats[(bs + j) * F + q], g[q]));
        s = Ar<T>::add(s, Ar<T>::mul(smu[iv * n_p + j], dot));
    }
    // pass 2: scatter
    for (int j = 0; j < n_p; ++j) {
        const T sj = smu[iv * n_p + j];
        T dot = T(0);
        for (int q = 0; q < F; ++q) {
            dot = Ar<T>::add(dot, Ar<T>::mul(feats[(bs + j) * F + q], g[q]));
            red_add(gfeat + (bs + j) * F + q, Ar<T>::mul(sj, g[q]));
        }
        red_add(gconf_u + iv * n_p + j, Ar<T>::mul(sj, Ar<T>::sub(dot, s)));
    }
}

// =========================================================================
// dedup_rows with the reference's first-encounter order (_core.pyx:140-160):
//   first[r] = min position of r;  keep[i] = (first[row[i]] == i);
//   u(i) = exclusive scan of keep;  rows_u[u(i)] = row[i] for kept i;
//   inv[i] = u(first[row[i]]).
// =========================================================================
__global__ void dedup_init_kernel(int32_t *first, int64_t n_c) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_c) first[i] = INT32_MAX;
}
__global__ void dedup_first_kernel(const int32_t *row, int64_t n, int32_t *first) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicMin(first + row[i], (int32_t)i);
}
// block-wide exclusive scan of keep flags; block totals to sums[]
__global__ void dedup_scan_kernel(const int32_t *row, int64_t n, const int32_t *first,
                                  int32_t *pos, int32_t *sums) {
    __shared__ int32_t warp_tot[32];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int keep = (i < n) && first[row[i]] == (int32_t)i;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    const int in_warp = __popc(bal & ((1u << lane) - 1u));
    if (lane == 31) warp_tot[wid] = in_warp + keep;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        int v = lane < nw ? warp_tot[lane] : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane < nw) warp_tot[lane] = incl - v;
        if (lane == nw - 1) sums[blockIdx.x] = incl;
    }
    __syncthreads();
    if (i < n) pos[i] = warp_tot[wid] + in_warp;
}
// sequential scan of block totals by one block (chunks of blockDim with carry)
__global__ void dedup_scan_sums_kernel(int32_t *sums, int64_t nb, int32_t *total) {
    __shared__ int32_t buf[1024];
    __shared__ int32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < nb; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const int v = i < nb ? sums[i] : 0;
        buf[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < (int)blockDim.x; o <<= 1) {
            const int u = threadIdx.x >= (unsigned)o ? buf[threadIdx.x - o] : 0;
            __syncthreads();
            buf[threadIdx.x] += u;
            __syncthreads();
        }
        if (i < nb) sums[i] = carry + buf[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += buf[threadIdx.x];
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = carry;
}
__global__ void dedup_emit_kernel(const int32_t *row, int64_t n, const int32_t *first,
                                  const int32_t *pos, const int32_t *sums, int32_t *rows_u,
                                  int32_t *inv, int blk) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = row[i];
    const int32_t f = first[r];
    const int32_t uf = sums[f / blk] + pos[f];
    if (f == (int32_t)i) rows_u[uf] = r;
    inv[i] = uf;
}

// =========================================================================
// Fused all-level forward.  Thread task = (point, level) mapped level-major
// inside a 128-point chunk so each warp serves 32 points of ONE level
// (uniform dense/hashed/probed branch, one table per warp).
// =========================================================================
constexpr int kChunk = 128;

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
template <typename T, int D, int FC, int NPMAX>
__global__ void __launch_bounds__(256) encode_bwd_kernel(
    const pg_grid g, const T *__restrict__ xs, int64_t B, const T *__restrict__ dy,
    const T *__restrict__ feats, const T *__restrict__ conf, T *__restrict__ gfeat,
    T *__restrict__ gconf, uint8_t *__restrict__ touched) {
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
            T *gtab = gfeat + (int64_t)l * g.n_f * F;
            const T *ftab = feats + (int64_t)l * g.n_f * F;
#pragma unroll
            for (int k = 0; k < C; ++k) {
                const T w = corner_weight<T, D>(k, t, omt);
                T gq[FC ? FC : PG_MAX_FEATURE];
                for (int q = 0; q < F; ++q) gq[q] = Ar<T>::mul(w, up[q]);
                if (kind != PG_LEVEL_PROBED) {
                    const int lin = kind == PG_LEVEL_DENSE
                                        ? corner_dense<D>(k, c, res + 1)
                                        : (int)(corner_hash<D>(k, c, g.primary) & nf_mask);
                    T *dst = gtab + (int64_t)lin * F;
                    if constexpr (FC == 2 && sizeof(T) == 4) {
                        red_add_v2((float *)dst, gq[0], gq[1]);
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
                T *gc = gconf + crow * n_p;
                const T *fb = ftab + (int64_t)bs * F;
                T *gb = gtab + (int64_t)bs * F;
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
                    const T inv_sum = T(1) / sum;
                    T s = T(0);
#pragma unroll
                    for (int j = 0; j < NPMAX; ++j)
                        if (j < n_p) {
                            sg[j] = sg[j] * inv_sum;
                            T dot = T(0);
                            for (int q = 0; q < F; ++q) dot += fb[j * F + q] * gq[q];
                            dots[j] = dot;
                            s += sg[j] * dot;
                        }
                    if constexpr (FC == 2 && sizeof(T) == 4) {
                        // N_p*F contiguous floats, 16B aligned when n_p >= 2
                        if (n_p >= 2) {
#pragma unroll
                            for (int j = 0; j < NPMAX; j += 2)
                                if (j < n_p)
                                    red_add_v4((float *)gb + 2 * j, sg[j] * gq[0], sg[j] * gq[1],
                                               sg[j + 1] * gq[0], sg[j + 1] * gq[1]);
                        } else {
                            red_add_v2((float *)gb, sg[0] * gq[0], sg[0] * gq[1]);
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
                                    red_add_v4((float *)gc + j, sg[j] * (dots[j] - s),
                                               sg[j + 1] * (dots[j + 1] - s),
                                               sg[j + 2] * (dots[j + 2] - s),
                                               sg[j + 3] * (dots[j + 3] - s));
                        } else if (n_p == 2) {
                            red_add_v2((float *)gc, sg[0] * (dots[0] - s), sg[1] * (dots[1] - s));
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
                    const T inv_sum = T(1) / sum;
                    T s = T(0);
                    for (int j = 0; j < n_p; ++j) {
                        T dot = T(0);
                        for (int q = 0; q < F; ++q) dot += fb[j * F + q] * gq[q];
                        s += Ar<T>::exp(cr[j] - mx) * inv_sum * dot;
                    }
                    for (int j = 0; j < n_p; ++j) {
                        const T sj = Ar<T>::exp(cr[j] - mx) * inv_sum;
                        T dot = T(0);
                        for (int q = 0; q < F; ++q) {
                            dot += fb[j * F + q] * gq[q];
                            red_add(gb + j * F + q, sj * gq[q]);
                        }
                        red_add(gc + j, sj * (dot - s));
                    }
                }
            }
        }
    }
}

int validate_grid(const pg_grid *g) {
    PG_REQUIRE(g != nullptr, "null grid");
    PG_REQUIRE(g->d == 2 || g->d == 3, "grid.d must be 2 or 3");
    PG_REQUIRE(g->n_levels >= 1 && g->n_levels <= PG_MAX_LEVELS, "grid.n_levels out of range");
    PG_REQUIRE(g->feature_dim >= 1 && g->feature_dim <= PG_MAX_FEATURE, "feature dim beyond compiled limit");
    PG_REQUIRE(g->n_f >= 1 && (g->n_f & (g->n_f - 1)) == 0, "n_f must be a power of two");
    PG_REQUIRE(g->n_c >= 1 && (g->n_c & (g->n_c - 1)) == 0, "n_c must be a power of two");
    PG_REQUIRE(g->log2_np >= 0 && g->log2_np <= 8, "probing range beyond compiled limit");
    for (int l = 0; l < g->n_levels; ++l) {
        PG_REQUIRE(g->res[l] >= 1 && g->res[l] < (1 << 24), "resolution out of range");
        PG_REQUIRE(g->kind[l] >= 0 && g->kind[l] <= 2, "bad level kind");
        if (g->kind[l] == PG_LEVEL_DENSE) {
            int64_t v = 1;
            for (int a = 0; a < g->d; ++a) v *= (int64_t)g->res[l] + 1;
            PG_REQUIRE(v <= g->n_f, "dense level does not fit its table");
        }
        if (g->kind[l] == PG_LEVEL_PROBED) PG_REQUIRE(g->slot[l] >= 0, "probed level without slot");
    }
    return PG_OK;
}

static int encode_blocks(int64_t B) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
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

template <typename T>
static int launch_encode_bwd(const pg_grid *g, const T *xs, int64_t B, const T *dy,
                             const T *feats, const T *conf, T *gfeat, T *gconf, uint8_t *touched,
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
    encode_bwd_kernel<T, D_, FC_, NP_><<<grd, 256, 0, s>>>(*g, xs, B, dy, feats, conf, gfeat, gconf, touched)
#define PG_ENC_BWD_NP(D_, FC_)                   \
    do {                                         \
        if (n_p <= 4) PG_ENC_BWD(D_, FC_, 4);     \
        else if (n_p <= 16) PG_ENC_BWD(D_, FC_, 16); \
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

int pg_dense_fwd_f32(const float *xs, int64_t B, int d, int64_t res, const float *feats, int F,
                     float *out, int32_t *idx, float *wgt, void *stream) {
    return launch_level_fwd<float, PG_LEVEL_DENSE>(xs, B, d, res, 0, 0, 0, feats, F, nullptr,
                                                   nullptr, nullptr, out, idx, nullptr, wgt, stream);
}
int pg_dense_fwd_f64(const double *xs, int64_t B, int d, int64_t res, const double *feats, int F,
                     double *out, int32_t *idx, double *wgt, void *stream) {
    return launch_level_fwd<double, PG_LEVEL_DENSE>(xs, B, d, res, 0, 0, 0, feats, F, nullptr,
                                                    nullptr, nullptr, out, idx, nullptr, wgt, stream);
}
int pg_hashed_fwd_f32(const float *xs, int64_t B, int d, int64_t res, uint32_t nf_mask,
                      const float *feats, int F, const uint32_t *h_primary, float *out,
                      int32_t *idx, float *wgt, void *stream) {
    return launch_level_fwd<float, PG_LEVEL_HASHED>(xs, B, d, res, nf_mask, 0, 0, feats, F, nullptr,
                                                    h_primary, nullptr, out, idx, nullptr, wgt, stream);
}
int pg_hashed_fwd_f64(const double *xs, int64_t B, int d, int64_t res, uint32_t nf_mask,
                      const double *feats, int F, const uint32_t *h_primary, double *out,
                      int32_t *idx, double *wgt, void *stream) {
    return launch_level_fwd<double, PG_LEVEL_HASHED>(xs, B, d, res, nf_mask, 0, 0, feats, F,
                                                     nullptr, h_primary, nullptr, out, idx, nullptr,
                                                     wgt, stream);
}
int pg_probed_fwd_f32(const float *xs, int64_t B, int d, int64_t res, uint32_t nf_mask,
                      uint32_t nc_mask, int log2_np, const float *feats, int F,
                      const uint8_t *baked, const uint32_t *h_primary, const uint32_t *h_aux,
                      float *out, int32_t *base, int32_t *row, float *wgt, void *stream) {
    return launch_level_fwd<float, PG_LEVEL_PROBED>(xs, B, d, res, nf_mask, nc_mask, log2_np, feats,
                                                    F, baked, h_primary, h_aux, out, base, row, wgt,
                                                    stream);
}
int pg_probed_fwd_f64(const double *xs, int64_t B, int d, int64_t res, uint32_t nf_mask,
                      uint32_t nc_mask, int log2_np, const double *feats, int F,
                      const uint8_t *baked, const uint32_t *h_primary, const uint32_t *h_aux,
                      double *out, int32_t *base, int32_t *row, double *wgt, void *stream) {
    return launch_level_fwd<double, PG_LEVEL_PROBED>(xs, B, d, res, nf_mask, nc_mask, log2_np,
                                                     feats, F, baked, h_primary, h_aux, out, base,
                                                     row, wgt, stream);
}

#define PG_IDX_BWD(T, SFX)                                                                      \
    int pg_indexed_bwd_##SFX(const T *up, int64_t B, int F, const int32_t *idx, const T *wgt,   \
                             int C, T *gfeat, void *stream) {                                   \
        PG_REQUIRE(F >= 1 && F <= PG_MAX_FEATURE, "feature dim beyond compiled limit");         \
        if (B * C == 0) return PG_OK;                                                           \
        indexed_bwd_kernel<T><<<grid_for(B * C, 256), 256, 0, as_stream(stream)>>>(             \
            up, B, F, idx, wgt, C, gfeat);                                                      \
        return check_launch("indexed_bwd");                                                     \
    }
PG_IDX_BWD(float, f32)
PG_IDX_BWD(double, f64)
#undef PG_IDX_BWD

#define PG_PROBED_BWD(T, SFX)                                                                    \
    int pg_probed_bwd_##SFX(const T *up, int64_t B, int F, const int32_t *base,                  \
                            const int32_t *inv, const T *wgt, int C, const T *smu, int n_p,      \
                            const T *feats, T *gfeat, T *gconf_u, void *stream) {                \
        PG_REQUIRE(F >= 1 && F <= PG_MAX_FEATURE, "feature dim beyond compiled limit");          \
        PG_REQUIRE(n_p >= 1 && n_p <= PG_MAX_PROBES, "probing range beyond compiled limit");     \
        if (B * C == 0) return PG_OK;                                                            \
        probed_bwd_kernel<T><<<grid_for(B * C, 256), 256, 0, as_stream(stream)>>>(               \
            up, B, F, base, inv, wgt, C, smu, n_p, feats, gfeat, gconf_u);                       \
        return check_launch("probed_bwd");                                                       \
    }
PG_PROBED_BWD(float, f32)
PG_PROBED_BWD(double, f64)
#undef PG_PROBED_BWD

int64_t pg_dedup_workspace_bytes(int64_t n, int64_t n_c) {
    const int64_t nb = (n + 255) / 256;
    return 4 * (n_c + n + nb + 1) + 64;
}

int pg_dedup_rows(const int32_t *row, int64_t n, int64_t n_c, void *workspace, int32_t *rows_u,
                  int32_t *inv, int32_t *d_count, void *stream) {
    PG_REQUIRE(n >= 0 && n < INT32_MAX && n_c >= 1, "dedup sizes out of range");
    PG_REQUIRE(workspace != nullptr, "dedup needs workspace");
    cudaStream_t s = as_stream(stream);
    int32_t *first = (int32_t *)workspace;
    int32_t *pos = first + n_c;
    const int64_t nb = (n + 255) / 256;
    int32_t *sums = pos + n;
    if (n == 0) {
        cudaMemsetAsync(d_count, 0, sizeof(int32_t), s);
        return check_launch("dedup_rows");
    }
    dedup_init_kernel<<<grid_for(n_c, 256), 256, 0, s>>>(first, n_c);
    dedup_first_kernel<<<grid_for(n, 256), 256, 0, s>>>(row, n, first);
    dedup_scan_kernel<<<(int)nb, 256, 0, s>>>(row, n, first, pos, sums);
    dedup_scan_sums_kernel<<<1, 1024, 0, s>>>(sums, nb, d_count);
    dedup_emit_kernel<<<grid_for(n, 256), 256, 0, s>>>(row, n, first, pos, sums, rows_u, inv, 256);
    return check_launch("dedup_rows");
}

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

}  // extern "C"
