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

}  // extern "C"
