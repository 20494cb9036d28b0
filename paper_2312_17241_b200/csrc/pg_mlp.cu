// The tiny decoder MLP on sm_100a (mlp.py:16-85, _core.pyx:275-298):
//  * generic row-wise kernels for any widths (protocol mlp_infer_rows, and
//    the training pass for shapes the fused kernels do not cover);
//  * the fused decode kernel: all-level encode + [32,64,64,<=4] MLP per
//    128-query tile, activations resident in shared memory.
#include <cuda.h>

#include "pg_encode_dev.cuh"

namespace pg {

// =========================================================================
// Generic row-wise linear layer in the reference's order: acc = b_j, then
// acc += x_i * W_ij for i ascending (no FMA unless !exact), optional ReLU
// (acc < 0 -> 0, so NaN/-0 pass like _core.pyx:287-288) and logistic
// evaluated in double (_core.pyx:292-298).
// =========================================================================
template <typename T, bool EXACT>
__global__ void linear_rows_kernel(const T *__restrict__ a, int64_t B, int fin,
                                   const T *__restrict__ W, const T *__restrict__ bias, int fout,
                                   T *__restrict__ out, int relu, int sigmoid) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B * fout) return;
    const int64_t b = i / fout;
    const int j = (int)(i - b * fout);
    const T *ar = a + b * fin;
    T acc = bias[j];
    for (int k = 0; k < fin; ++k) {
        if (EXACT)
            acc = Ar<T>::add(acc, Ar<T>::mul(ar[k], W[(int64_t)k * fout + j]));
        else
            acc = Ar<T>::fma(ar[k], W[(int64_t)k * fout + j], acc);
    }
    if (relu && acc < T(0)) acc = T(0);
    if (sigmoid) acc = (T)(1.0 / (1.0 + ::exp(-(double)acc)));
    out[i] = acc;
}

static int64_t mlp_param_count(const pg_mlp *m) {
    int64_t n = 0;
    for (int l = 0; l < m->n_layers; ++l) n += (int64_t)m->widths[l] * m->widths[l + 1] + m->widths[l + 1];
    return n;
}
static int mlp_max_width(const pg_mlp *m) {
    int w = 0;
    for (int l = 0; l <= m->n_layers; ++l) w = m->widths[l] > w ? m->widths[l] : w;
    return w;
}
static int validate_mlp(const pg_mlp *m) {
    PG_REQUIRE(m != nullptr, "null mlp");
    PG_REQUIRE(m->n_layers >= 1 && m->n_layers <= PG_MAX_LAYERS, "mlp layer count out of range");
    for (int l = 0; l <= m->n_layers; ++l) PG_REQUIRE(m->widths[l] >= 1, "mlp width must be positive");
    return PG_OK;
}

template <typename T>
static int mlp_infer_rows_generic(const T *xs, int64_t B, const pg_mlp *mlp, const T *params,
                                  unsigned flags, T *act_ws, T *out, cudaStream_t s) {
    if (int e = validate_mlp(mlp)) return e;
    if (B == 0) return PG_OK;
    PG_REQUIRE(act_ws != nullptr || mlp->n_layers == 1, "mlp_infer_rows needs activation workspace");
    const int maxw = mlp_max_width(mlp);
    const T *a = xs;
    const T *p = params;
    const bool exact = (flags & PG_EXACT_MLP) != 0;
    for (int l = 0; l < mlp->n_layers; ++l) {
        const int fin = mlp->widths[l], fout = mlp->widths[l + 1];
        const bool last = l == mlp->n_layers - 1;
        T *dst = last ? out : act_ws + (int64_t)(l & 1) * B * maxw;
        const int relu = last ? 0 : 1;
        const int sig = (last && (flags & PG_SIGMOID)) ? 1 : 0;
        const int grd = grid_for(B * fout, 256);
        if (exact)
            linear_rows_kernel<T, true><<<grd, 256, 0, s>>>(a, B, fin, p, p + (int64_t)fin * fout, fout, dst, relu, sig);
        else
            linear_rows_kernel<T, false><<<grd, 256, 0, s>>>(a, B, fin, p, p + (int64_t)fin * fout, fout, dst, relu, sig);
        p += (int64_t)fin * fout + fout;
        a = dst;
    }
    return check_launch("mlp_infer_rows");
}

// =========================================================================
// Fused decode: encode all 16 levels (F = 2) of a 128-query tile into
// shared memory, then run the [32, 64, 64, out] MLP on it.
//
// Activation tiles are stored transposed, act[feature][query], 128 floats
// per row with the 16-byte chunk index XOR-swizzled by (row >> 2) & 7, so
//   - encode writes (32 consecutive queries of one feature) and
//   - the MMA-style reads (one feature row, 4 chunks per warp) and
//   - the epilogue writes (8 feature rows x 1 chunk per quarter-warp)
// are all bank-conflict free.
// Layer math: thread (og = tid % 16, pg = tid / 16) owns queries pg*8..+7 and
// outputs og*4..+3 of a 128x64 layer tile (32 accumulators).
// =========================================================================
constexpr int kTP = 128;   // queries per tile
constexpr int kIn = 32;    // L * F
constexpr int kHid = 64;
constexpr int kOutMax = 4;

struct DecodeSmemW {       // weights, shared by the CTA's tile pipelines
    float w0[kIn * kHid];
    float w1[kHid * kHid];
    float w2[kHid * kOutMax];
    float b0[kHid];
    float b1[kHid];
    float b2[kOutMax];
};
struct DecodeSmemG {       // one tile pipeline
    float actA[kHid * kTP];  // y^T (rows 0..31) for layer 1, then h2^T for layer 3
    float actB[kHid * kTP];  // h1^T
    float outs[kTP * kOutMax];
    float xs[kTP * 3];
};
struct DecodeSmem {        // two ping-pong pipelines per CTA
    DecodeSmemW w;
    DecodeSmemG g[2];
};

__device__ __forceinline__ int swz(int row, int col) {
    // element offset of act[row][col] in a swizzled 128-float row
    const int chunk = (col >> 2) ^ ((row >> 2) & 7);
    return row * kTP + (chunk << 2) + (col & 3);
}

template <bool EXACT>
__device__ __forceinline__ float mac(float acc, float a, float w) {
    return EXACT ? __fadd_rn(acc, __fmul_rn(a, w)) : __fmaf_rn(a, w, acc);
}

// Paired fp32 FMA (sm_100 FFMA2: two fp32 lanes per instruction) for the
// non-exact MLP.  The exact (reference-order) MLP stays on scalar
// __fmul_rn/__fadd_rn: ptxas (12.9) contracts mul.rn.f32x2 + add.rn.f32x2
// into FFMA2 even with --fmad=false, which would change the rounding.
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float &a, float &b) {
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t acc, uint64_t a, uint64_t w) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(w), "l"(acc));
    return r;
}

// 128 x 64 layer: out^T = act(in^T)^T W + b, K = fan_in.
template <int K, bool EXACT>
__device__ __forceinline__ void layer_tile(const float *__restrict__ in_t, const float *__restrict__ W,
                                           const float *__restrict__ bias, float *__restrict__ out_t) {
    const int og = threadIdx.x & 15, pg = (threadIdx.x & 255) >> 4;   // within the 256-thread pipeline
    float acc[8][4];
    if (EXACT) {
        const float4 bb = *reinterpret_cast<const float4 *>(bias + og * 4);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            acc[i][0] = bb.x;
            acc[i][1] = bb.y;
            acc[i][2] = bb.z;
            acc[i][3] = bb.w;
        }
#pragma unroll 8
        for (int k = 0; k < K; ++k) {
            const float4 a0 = *reinterpret_cast<const float4 *>(in_t + swz(k, pg * 8));
            const float4 a1 = *reinterpret_cast<const float4 *>(in_t + swz(k, pg * 8 + 4));
            const float4 w = *reinterpret_cast<const float4 *>(W + k * kHid + og * 4);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                acc[i][0] = mac<true>(acc[i][0], a[i], w.x);
                acc[i][1] = mac<true>(acc[i][1], a[i], w.y);
                acc[i][2] = mac<true>(acc[i][2], a[i], w.z);
                acc[i][3] = mac<true>(acc[i][3], a[i], w.w);
            }
        }
    } else {
    // accumulators as output pairs (j0, j1), (j2, j3): paired fp32 FMA
    uint64_t acc2[8][2];
    const float4 bb = *reinterpret_cast<const float4 *>(bias + og * 4);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        acc2[i][0] = f2pack(bb.x, bb.y);
        acc2[i][1] = f2pack(bb.z, bb.w);
    }
#pragma unroll 8
    for (int k = 0; k < K; ++k) {
        const float4 a0 = *reinterpret_cast<const float4 *>(in_t + swz(k, pg * 8));
        const float4 a1 = *reinterpret_cast<const float4 *>(in_t + swz(k, pg * 8 + 4));
        const float4 w = *reinterpret_cast<const float4 *>(W + k * kHid + og * 4);
        const uint64_t w01 = f2pack(w.x, w.y), w23 = f2pack(w.z, w.w);
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint64_t aa = f2pack(a[i], a[i]);
            acc2[i][0] = ffma2(acc2[i][0], aa, w01);
            acc2[i][1] = ffma2(acc2[i][1], aa, w23);
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        f2unpack(acc2[i][0], acc[i][0], acc[i][1]);
        f2unpack(acc2[i][1], acc[i][2], acc[i][3]);
    }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float r[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = acc[i][j] < 0.0f ? 0.0f : acc[i][j];  // ReLU
        const int row = og * 4 + j;
        *reinterpret_cast<float4 *>(out_t + swz(row, pg * 8)) = make_float4(r[0], r[1], r[2], r[3]);
        *reinterpret_cast<float4 *>(out_t + swz(row, pg * 8 + 4)) = make_float4(r[4], r[5], r[6], r[7]);
    }
}

// Two 256-thread tile pipelines per CTA (one CTA per SM) sharing the weights,
// in ping-pong over their MLP phases (named barriers 3/4: a pipeline arrives
// when its MLP ends and waits before its next one), so one pipeline's MLP
// always runs beside the other's gathers.
template <typename FT, int D, bool EXACT>
__global__ void __launch_bounds__(512, 1)
    decode_fused_kernel(const pg_grid g, const float *__restrict__ xs, int64_t B,
                        const FT *__restrict__ feats, const uint8_t *__restrict__ baked,
                        const float *__restrict__ params, int out_dim, int sigmoid,
                        float *__restrict__ out, int32_t *__restrict__ bad, const CellMap cmap) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    DecodeSmem &S = *reinterpret_cast<DecodeSmem *>(smem_raw);
    const int gid = threadIdx.x >> 8, tid = threadIdx.x & 255;
    DecodeSmemW &W = S.w;
    DecodeSmemG &sm = S.g[gid];
    auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + gid), "r"(256) : "memory"); };
    // ---- weights to shared memory once per CTA (params = [W0|b0|W1|b1|W2|b2]) ----
    {
        const float *p = params;
        const int t0 = threadIdx.x;
        for (int i = t0; i < kIn * kHid; i += 512) W.w0[i] = p[i];
        p += kIn * kHid;
        for (int i = t0; i < kHid; i += 512) W.b0[i] = p[i];
        p += kHid;
        for (int i = t0; i < kHid * kHid; i += 512) W.w1[i] = p[i];
        p += kHid * kHid;
        for (int i = t0; i < kHid; i += 512) W.b1[i] = p[i];
        p += kHid;
        for (int i = t0; i < kHid * kOutMax; i += 512) {
            const int k = i / kOutMax, j = i % kOutMax;
            W.w2[i] = j < out_dim ? p[k * out_dim + j] : 0.0f;
        }
        p += kHid * out_dim;
        for (int i = t0; i < kOutMax; i += 512) W.b2[i] = i < out_dim ? p[i] : 0.0f;
    }
    __syncthreads();
    const int64_t ntiles = (B + kTP - 1) / kTP;
    const int pl = tid & (kTP - 1);
    const int lhalf = tid >> 7;  // 0/1: which of the two levels per iteration
    const int64_t stride = (int64_t)gridDim.x * 2, first = (int64_t)blockIdx.x * 2 + gid;
    const int64_t base0 = (int64_t)blockIdx.x * 2;
    const int64_t n_iter = base0 < ntiles ? (ntiles - base0 + stride - 1) / stride : 0;
    for (int64_t iter = 0; iter < n_iter; ++iter) {
        const int64_t tile = first + iter * stride;
        if (tile >= ntiles) {   // pipeline 1's last iteration: keep the ping-pong count
            if (iter > 0) asm volatile("bar.sync 4, 512;" ::: "memory");
            asm volatile("bar.arrive 3, 512;" ::: "memory");
            continue;
        }
        const int64_t p0 = tile * kTP;
        const int nvalid = (int)((B - p0) < kTP ? (B - p0) : kTP);
        gsync();  // previous tile's layer 3 finished reading actA / outs
        for (int i = tid; i < kTP * D; i += 256) sm.xs[i] = i < nvalid * D ? xs[p0 * D + i] : 0.0f;
        gsync();
        // ---------------- encode: thread = (query pl, levels lhalf, lhalf+2, ...) --------
        float x[D];
        bool oob = false;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            x[a] = sm.xs[pl * D + a];
            oob |= !(x[a] >= 0.0f && x[a] <= 1.0f);
        }
        if (bad && oob && pl < nvalid && lhalf == 0) *bad = 1;
#pragma unroll 2
        for (int it = 0; it < 8; ++it) {
            const int l = 2 * it + lhalf;  // warp-uniform
            float2 yv;
            if (std::is_same<FT, __half>::value && cmap.off[l] >= 0)
                yv = encode_level_fwd2_cell<D>(g, l, x, cmap.cells + cmap.off[l]);
            else
                yv = encode_level_fwd2_rng<FT, D>(g, l, x, feats, baked);
            const float y0 = yv.x, y1 = yv.y;
            sm.actA[swz(2 * l, pl)] = y0;
            sm.actA[swz(2 * l + 1, pl)] = y1;
        }
        gsync();
        // MLP phase: wait for the other pipeline's previous MLP to end
        if (gid == 0) asm volatile("bar.sync 3, 512;" ::: "memory");
        else if (iter > 0) asm volatile("bar.sync 4, 512;" ::: "memory");
        layer_tile<kIn, EXACT>(sm.actA, W.w0, W.b0, sm.actB);
        gsync();
        layer_tile<kHid, EXACT>(sm.actB, W.w1, W.b1, sm.actA);
        gsync();
        // ---------------- output layer: thread = (query, pair of outputs) -------------
        {
            const int q = tid & (kTP - 1);
            const int j0 = (tid >> 7) * 2;
            float acc0 = W.b2[j0], acc1 = W.b2[j0 + 1];
#pragma unroll 16
            for (int k = 0; k < kHid; ++k) {
                const float a = sm.actA[swz(k, q)];
                acc0 = mac<EXACT>(acc0, a, W.w2[k * kOutMax + j0]);
                acc1 = mac<EXACT>(acc1, a, W.w2[k * kOutMax + j0 + 1]);
            }
            if (sigmoid) {
                acc0 = (float)(1.0 / (1.0 + exp(-(double)acc0)));
                acc1 = (float)(1.0 / (1.0 + exp(-(double)acc1)));
            }
            sm.outs[q * kOutMax + j0] = acc0;
            sm.outs[q * kOutMax + j0 + 1] = acc1;
        }
        gsync();
        asm volatile("bar.arrive %0, 512;" ::"r"(gid == 0 ? 4 : 3) : "memory");   // MLP done
        float *dst = out + p0 * out_dim;
        for (int i = tid; i < nvalid * out_dim; i += 256) {
            const int q = i / out_dim, j = i - q * out_dim;
            dst[i] = sm.outs[q * kOutMax + j];
        }
    }
    if (gid == 1 && n_iter > 0) asm volatile("bar.sync 4, 512;" ::: "memory");   // pipeline 0's last MLP-done
}

static bool decode_fast_ok(const pg_grid *g, const pg_mlp *m) {
    return g->feature_dim == 2 && g->n_levels == 16 && m->n_layers == 3 && m->widths[0] == kIn &&
           m->widths[1] == kHid && m->widths[2] == kHid && m->widths[3] >= 1 && m->widths[3] <= kOutMax;
}

static int sm_count() { return device_sms(); }

template <typename FT, int D, bool EXACT>
static void launch_decode(const pg_grid *g, const float *xs, int64_t B, const void *feats,
                          const uint8_t *baked, const float *params, int out_dim, int sig,
                          float *out, int32_t *bad, cudaStream_t s, const CellMap &cmap) {
    static DeviceOnce configured;
    const int smem = (int)sizeof(DecodeSmem);
    if (configured.first())
        cudaFuncSetAttribute(decode_fused_kernel<FT, D, EXACT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int64_t ntiles = (B + kTP - 1) / kTP;
    const int64_t want = (ntiles + 1) / 2, cap = (int64_t)sm_count();
    const int grd = (int)(want < cap ? want : cap);
    decode_fused_kernel<FT, D, EXACT><<<grd, 512, smem, s>>>(*g, xs, B, (const FT *)feats, baked,
                                                            params, out_dim, sig, out, bad, cmap);
}

int decode_umma(const pg_grid *g, int od, const float *xs, int64_t B, const void *feats, bool half,
                const uint8_t *baked, const float *params, int sig, int table_flags, float *out, cudaStream_t s,
                const DecodeStream &st = DecodeStream(), const pg_cells *cells = nullptr);

int decode_device(const pg_grid *g, const pg_mlp *m, const float *xs, int64_t B,
                  const void *feats, const uint8_t *baked, const float *params, unsigned flags,
                  float *ws, float *out, int32_t *bad, cudaStream_t s, const pg_cells *cells = nullptr) {
    if (int e = validate_grid(g)) return e;
    if (int e = validate_mlp(m)) return e;
    PG_REQUIRE(m->widths[0] == g->n_levels * g->feature_dim, "MLP input width != L*F");
    if (B == 0) return PG_OK;
    const bool half = (flags & PG_HALF_FEATS) != 0;
    const bool exact = (flags & PG_EXACT_MLP) != 0;
    const int sig = (flags & PG_SIGMOID) ? 1 : 0;
    if (decode_fast_ok(g, m)) {
        const int od = m->widths[3];
        if (!exact && !(flags & PG_NO_TENSOR))  // tcgen05 path (pg_decode_tc.cu)
            return decode_umma(g, od, xs, B, feats, half, baked, params, sig, (int)(flags & (PG_SMEM_TABLES | PG_NO_SMEM_TABLES)),
                               out, s, DecodeStream(), cells);
        CellMap cmap;
        cmap.cells = nullptr;
        for (int l = 0; l < PG_MAX_LEVELS; ++l) cmap.off[l] = -1;
        if (half && cells && cells->data) {
            cmap.cells = reinterpret_cast<const uint4 *>(cells->data);
            for (int l = 0; l < g->n_levels; ++l) cmap.off[l] = cells->off[l] >= 0 ? (int32_t)cells->off[l] : -1;
        }
#define PG_DEC(FT_, D_)                                                                    \
    (exact ? launch_decode<FT_, D_, true>(g, xs, B, feats, baked, params, od, sig, out, bad, s, cmap) \
           : launch_decode<FT_, D_, false>(g, xs, B, feats, baked, params, od, sig, out, bad, s, cmap))
        if (half) {
            if (g->d == 2) PG_DEC(__half, 2); else PG_DEC(__half, 3);
        } else {
            if (g->d == 2) PG_DEC(float, 2); else PG_DEC(float, 3);
        }
#undef PG_DEC
        return check_launch("decode_fused");
    }
    // generic shapes: fused encode, then row-wise MLP
    PG_REQUIRE(ws != nullptr, "generic decode needs workspace");
    float *y = ws;
    if (int e = pg_encode_fwd_f32(g, xs, B, feats, baked, nullptr, flags & PG_HALF_FEATS, y, bad, s)) return e;
    return mlp_infer_rows_generic<float>(y, B, m, params, flags, ws + B * g->n_levels * g->feature_dim,
                                         out, s);
}

// =========================================================================
// Generic training pass (any widths, float or double).  ws layout:
//   z_l (pre-activations) for every layer: B * sum(widths[1:])
//   two delta buffers:                     2 * B * max(widths)
// =========================================================================
template <typename T>
__global__ void train_linear_fwd_kernel(const T *__restrict__ a, int relu_in, int64_t B, int fin,
                                        const T *__restrict__ W, const T *__restrict__ bias,
                                        int fout, T *__restrict__ z) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B * fout) return;
    const int64_t b = i / fout;
    const int j = (int)(i - b * fout);
    // numpy `a @ W + b` on OpenBLAS: FMA chain over k from zero, then the
    // bias as a separate rounded add (same bits as mlp.py:66 in fp32/fp64)
    T acc = T(0);
    for (int k = 0; k < fin; ++k) {
        T v = a[b * fin + k];
        if (relu_in && v < T(0)) v = T(0);
        acc = Ar<T>::fma(v, W[(int64_t)k * fout + j], acc);
    }
    z[i] = Ar<T>::add(acc, bias[j]);
}

template <typename T, typename LACC>
__global__ void train_loss_kernel(const T *__restrict__ zout, const T *__restrict__ targets,
                                  int64_t n, T scale, int sigmoid, T *__restrict__ delta,
                                  LACC *__restrict__ loss_sum) {
    __shared__ double red[32];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double sq = 0.0;
    if (i < n) {
        const T o = zout[i];
        const T pred = sigmoid ? T(1) / (T(1) + Ar<T>::exp(-o)) : o;
        const T diff = pred - targets[i];
        sq = (double)diff * (double)diff;
        T dp = Ar<T>::mul(diff, scale);
        if (sigmoid) dp = dp * (pred * (T(1) - pred));
        delta[i] = dp;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0 && loss_sum) loss_add(loss_sum, v);
    }
}

// dW[k][j] += sum_b a[b][k] * delta[b][j] (k == fin -> bias row), rows split
// over blockIdx.y in chunks, partial sums added atomically (fixed point in
// deterministic mode).
template <typename T, typename ACC>
__global__ void train_wgrad_kernel(const T *__restrict__ a, int relu_in, int64_t B, int fin,
                                   const T *__restrict__ delta, int fout, ACC *__restrict__ gW,
                                   ACC *__restrict__ gb, int64_t rows_per_chunk) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)(fin + 1) * fout) return;
    const int k = (int)(i / fout), j = (int)(i % fout);
    const int64_t b0 = (int64_t)blockIdx.y * rows_per_chunk;
    const int64_t b1 = b0 + rows_per_chunk < B ? b0 + rows_per_chunk : B;
    T acc = T(0);
    for (int64_t b = b0; b < b1; ++b) {
        T v = T(1);
        if (k < fin) {
            v = a[b * fin + k];
            if (relu_in && v < T(0)) v = T(0);
        }
        acc = Ar<T>::fma(v, delta[b * fout + j], acc);
    }
    if (k < fin) red_add(gW + (int64_t)k * fout + j, acc);
    else red_add(gb + j, acc);
}

// out[b][k] = (sum_j delta[b][j] W[k][j]) * (mask ? z[b][k] > 0 : 1)
template <typename T>
__global__ void train_dgrad_kernel(const T *__restrict__ delta, int64_t B, int fout,
                                   const T *__restrict__ W, int fin, const T *__restrict__ zmask,
                                   T *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B * fin) return;
    const int64_t b = i / fin;
    const int k = (int)(i - b * fin);
    // numpy `(delta @ W.T) * (pre > 0)`: FMA chain over j from zero, then a
    // rounded multiply by the 0/1 mask (mlp.py:83-85)
    T acc = T(0);
    for (int j = 0; j < fout; ++j) acc = Ar<T>::fma(delta[b * fout + j], W[(int64_t)k * fout + j], acc);
    if (zmask) acc = Ar<T>::mul(acc, zmask[i] > T(0) ? T(1) : T(0));
    out[i] = acc;
}

// forward layers -> loss(z_out, delta) -> backward layers; the loss stage
// writes dL/d(output pre-activation) for all B rows into delta
template <typename T, typename ACC, typename LossFn>
int mlp_train_core(const pg_mlp *m, const T *y, int64_t B, const T *params, ACC *gparams, T *dy,
                   T *ws, cudaStream_t s, LossFn loss) {
    if (int e = validate_mlp(m)) return e;
    if (B == 0) return PG_OK;
    PG_REQUIRE(ws != nullptr, "mlp_train needs workspace");
    const int nl = m->n_layers;
    const int maxw = mlp_max_width(m);
    const T *Wp[PG_MAX_LAYERS], *bp[PG_MAX_LAYERS];
    ACC *gWp[PG_MAX_LAYERS], *gbp[PG_MAX_LAYERS];
    T *z[PG_MAX_LAYERS];
    {
        int64_t off = 0, zoff = 0;
        for (int l = 0; l < nl; ++l) {
            const int fi = m->widths[l], fo = m->widths[l + 1];
            Wp[l] = params + off;
            gWp[l] = gparams + off;
            off += (int64_t)fi * fo;
            bp[l] = params + off;
            gbp[l] = gparams + off;
            off += fo;
            z[l] = ws + zoff;
            zoff += B * fo;
        }
        T *d0 = ws + zoff;
        T *d1 = d0 + B * maxw;
        // forward
        for (int l = 0; l < nl; ++l) {
            const int fi = m->widths[l], fo = m->widths[l + 1];
            const T *a = l == 0 ? y : z[l - 1];
            train_linear_fwd_kernel<T><<<grid_for(B * fo, 256), 256, 0, s>>>(a, l > 0, B, fi, Wp[l], bp[l], fo, z[l]);
        }
        loss(z[nl - 1], d0);
        // backward
        T *dcur = d0, *dnext = d1;
        for (int l = nl - 1; l >= 0; --l) {
            const int fi = m->widths[l], fo = m->widths[l + 1];
            const T *a = l == 0 ? y : z[l - 1];
            const int64_t chunk = 4096;
            dim3 gg(grid_for((int64_t)(fi + 1) * fo, 128), (unsigned)((B + chunk - 1) / chunk));
            train_wgrad_kernel<T, ACC><<<gg, 128, 0, s>>>(a, l > 0, B, fi, dcur, fo, gWp[l], gbp[l], chunk);
            T *dst = l > 0 ? dnext : dy;
            train_dgrad_kernel<T><<<grid_for(B * fi, 256), 256, 0, s>>>(dcur, B, fo, Wp[l], fi,
                                                                       l > 0 ? z[l - 1] : nullptr, dst);
            T *tmp = dcur;
            dcur = dnext;
            dnext = tmp;
        }
    }
    return check_launch("mlp_train");
}

template <typename T, typename ACC = T, typename LACC = double>
int mlp_train_generic(const pg_mlp *m, const T *y, const T *targets, int64_t B, const T *params,
                      T scale, unsigned flags, ACC *gparams, T *dy, LACC *loss_sum, T *ws,
                      cudaStream_t s) {
    const int od = m->widths[m->n_layers];
    return mlp_train_core<T, ACC>(m, y, B, params, gparams, dy, ws, s, [&](const T *zout, T *delta) {
        train_loss_kernel<T, LACC><<<grid_for(B * od, 256), 256, 0, s>>>(
            zout, targets, B * od, scale, (flags & PG_SIGMOID) ? 1 : 0, delta, loss_sum);
    });
}

// =========================================================================
// Volume compositing head (beyond the reference, which has
// no renderer): per ray, S samples of raw MLP outputs (sigma_raw, r, g, b),
// density sigma = softplus(sigma_raw), colour c = logistic(rgb_raw),
// alpha_i = 1 - exp(-sigma_i delta_i), T_i = prod_{j<i} (1 - alpha_j),
// C = sum_i T_i alpha_i c_i.  One thread per ray, samples in order.
// Backward (derivation in DESIGN.md 4): with w_i = T_i alpha_i and the
// prefix C_<=i, dC/dc_i = w_i and dC/dsigma_i = delta_i (T_{i+1} c_i -
// (C - C_<=i)).
// =========================================================================
// midpoint samples along each ray inside the unit cube (slab test); rays
// that miss get zero-length segments at their clamped origin
// t4 (optional): the fused NeRF step's per-sample targets (segment length,
// ray colour) written alongside, rgb (R, 3) the rays' target colours
__global__ void ray_samples_kernel(const float *__restrict__ o, const float *__restrict__ dir, int64_t R,
                                   int S, float *__restrict__ pts, float *__restrict__ deltas,
                                   const float *__restrict__ rgb = nullptr, float *__restrict__ t4 = nullptr) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R * S) return;
    const int64_t r = i / S;
    const int k = (int)(i - r * S);
    float ov[3], dv[3], nr = 0.0f, fr = 3.4e38f;
    for (int a = 0; a < 3; ++a) {
        ov[a] = o[r * 3 + a];
        dv[a] = dir[r * 3 + a];
        const float inv = 1.0f / (fabsf(dv[a]) < 1e-12f ? 1e-12f : dv[a]);
        const float t0 = (0.0f - ov[a]) * inv, t1 = (1.0f - ov[a]) * inv;
        nr = fmaxf(nr, fminf(t0, t1));
        fr = fminf(fr, fmaxf(t0, t1));
    }
    if (!(fr > nr)) nr = fr = 0.0f;
    const float step = (fr - nr) / (float)S;
    const float t = nr + ((float)k + 0.5f) * step;
    for (int a = 0; a < 3; ++a) pts[i * 3 + a] = fminf(fmaxf(ov[a] + t * dv[a], 0.0f), 1.0f);
    deltas[i] = step;
    if (t4) *reinterpret_cast<float4 *>(t4 + i * 4) = make_float4(step, rgb[r * 3], rgb[r * 3 + 1], rgb[r * 3 + 2]);
}

__device__ __forceinline__ float softplus_f(float x) { return x > 20.0f ? x : log1pf(expf(x)); }
__device__ __forceinline__ float logistic_f(float x) { return 1.0f / (1.0f + expf(-x)); }

__global__ void composite_fwd_kernel(const float *__restrict__ raw, const float *__restrict__ deltas,
                                     int64_t R, int S, float *__restrict__ rgb, float *__restrict__ wts) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    float T = 1.0f, c0 = 0.0f, c1 = 0.0f, c2 = 0.0f;
    for (int i = 0; i < S; ++i) {
        const int64_t q = r * S + i;
        const float4 v = *reinterpret_cast<const float4 *>(raw + q * 4);
        const float tr = expf(-softplus_f(v.x) * deltas[q]);
        const float w = T * (1.0f - tr);
        c0 += w * logistic_f(v.y);
        c1 += w * logistic_f(v.z);
        c2 += w * logistic_f(v.w);
        if (wts) wts[q] = w;
        T *= tr;
    }
    rgb[r * 3 + 0] = c0;
    rgb[r * 3 + 1] = c1;
    rgb[r * 3 + 2] = c2;
}

// loss = sum over rays and channels of (C - target)^2 (fp64, into loss_sum);
// delta (R*S, 4) = dL/d(raw) with dL/dC = scale * (C - target)
template <typename LACC>
__global__ void composite_loss_kernel(const float *__restrict__ raw, const float *__restrict__ deltas,
                                      const float *__restrict__ target, int64_t R, int S, float scale,
                                      float *__restrict__ draw, LACC *__restrict__ loss_sum) {
    __shared__ double red[32];
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double sq = 0.0;
    if (r < R) {
        float T = 1.0f, C[3] = {0.0f, 0.0f, 0.0f};
        for (int i = 0; i < S; ++i) {
            const int64_t q = r * S + i;
            const float4 v = *reinterpret_cast<const float4 *>(raw + q * 4);
            const float tr = expf(-softplus_f(v.x) * deltas[q]);
            const float w = T * (1.0f - tr);
            C[0] += w * logistic_f(v.y);
            C[1] += w * logistic_f(v.z);
            C[2] += w * logistic_f(v.w);
            T *= tr;
        }
        float gC[3];
        for (int k = 0; k < 3; ++k) {
            const float diff = C[k] - target[r * 3 + k];
            sq += (double)diff * (double)diff;
            gC[k] = diff * scale;
        }
        const float cg = C[0] * gC[0] + C[1] * gC[1] + C[2] * gC[2];
        float Tc = 1.0f, pre = 0.0f;   // T_i and (C_<=i . gC)
        for (int i = 0; i < S; ++i) {
            const int64_t q = r * S + i;
            const float4 v = *reinterpret_cast<const float4 *>(raw + q * 4);
            const float dl = deltas[q];
            const float tr = expf(-softplus_f(v.x) * dl);
            const float w = Tc * (1.0f - tr);
            const float l0 = logistic_f(v.y), l1 = logistic_f(v.z), l2 = logistic_f(v.w);
            const float ci_g = l0 * gC[0] + l1 * gC[1] + l2 * gC[2];
            pre += w * ci_g;
            Tc *= tr;                                   // now T_{i+1}
            const float dsig = dl * (Tc * ci_g - (cg - pre));
            float4 d;
            d.x = dsig * logistic_f(v.x);               // softplus' = logistic
            d.y = w * gC[0] * l0 * (1.0f - l0);
            d.z = w * gC[1] * l1 * (1.0f - l1);
            d.w = w * gC[2] * l2 * (1.0f - l2);
            *reinterpret_cast<float4 *>(draw + q * 4) = d;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0 && loss_sum) loss_add(loss_sum, v);
    }
}


// standalone batched MLP (mlp.py:55-85): forward into the pre-activation
// workspace (the "cache"), and a backward that re-runs the forward from x and
// seeds the backward with a caller-supplied dL/d(output)
template <typename T>
int mlp_forward_generic(const pg_mlp *m, const T *x, int64_t B, const T *params, T *ws, T *out,
                        cudaStream_t s) {
    if (int e = validate_mlp(m)) return e;
    if (B == 0) return PG_OK;
    PG_REQUIRE(ws != nullptr && out != nullptr, "mlp_forward: null buffer");
    const int nl = m->n_layers;
    int64_t off = 0, zoff = 0;
    const T *a = x;
    for (int l = 0; l < nl; ++l) {
        const int fi = m->widths[l], fo = m->widths[l + 1];
        T *z = l == nl - 1 ? out : ws + zoff;
        train_linear_fwd_kernel<T><<<grid_for(B * fo, 256), 256, 0, s>>>(a, l > 0, B, fi, params + off,
                                                                        params + off + (int64_t)fi * fo, fo, z);
        off += (int64_t)fi * fo + fo;
        zoff += B * fo;
        a = z;
    }
    return check_launch("mlp_forward");
}

template <typename T>
int mlp_backward_generic(const pg_mlp *m, const T *x, int64_t B, const T *params, const T *upstream,
                         T *gparams, T *dx, T *ws, cudaStream_t s) {
    PG_REQUIRE(B == 0 || upstream != nullptr, "mlp_backward: null upstream");
    const int od = m->widths[m->n_layers];
    return mlp_train_core<T, T>(m, x, B, params, gparams, dx, ws, s, [&](const T *, T *delta) {
        cudaMemcpyAsync(delta, upstream, sizeof(T) * B * od, cudaMemcpyDeviceToDevice, s);
    });
}

int64_t mlp_train_ws(int64_t B, const pg_mlp *m) {
    int64_t zsum = 0;
    for (int l = 0; l < m->n_layers; ++l) zsum += m->widths[l + 1];
    return B * zsum + 2 * B * mlp_max_width(m);
}
int64_t mlp_params(const pg_mlp *m) { return mlp_param_count(m); }

// =========================================================================
// Reference-order weight/bias gradients (parity mode, mlp.py:80-84):
//   W_grad[l] += a_l^T @ delta_l     via OpenBLAS sgemm: C = 0; K (= samples)
//                                    blocked by kBlasQ, the last two blocks
//                                    balanced; per block one sequential FMA
//                                    chain from 0; C += block, in order
//   b_grad[l] += delta_l.sum(axis=0) sequential over samples
// One thread per gradient element.  The blocking was pinned against numpy
// 2.3 / OpenBLAS 0.3.30 (SkylakeX) in this image for K from 128 to 2^18,
// 1 to 8 BLAS threads (the CPU test test_openblas_wgrad_order pins it).
// =========================================================================
constexpr int64_t kBlasQ = 448;

// K (= sample) blocking of OpenBLAS's sgemm: Q-blocks while at least 2Q
// samples remain, then the rest in one block (<= Q) or two balanced halves
__host__ __device__ inline int64_t blas_nblocks(int64_t B) {
    const int64_t nq = B >= 2 * kBlasQ ? (B - 2 * kBlasQ) / kBlasQ + 1 : 0;
    const int64_t r = B - nq * kBlasQ;
    return nq + (r > kBlasQ ? 2 : r > 0 ? 1 : 0);
}
__device__ inline void blas_block(int64_t B, int64_t blk, int64_t &start, int64_t &len) {
    const int64_t nq = B >= 2 * kBlasQ ? (B - 2 * kBlasQ) / kBlasQ + 1 : 0;
    if (blk < nq) {
        start = blk * kBlasQ;
        len = kBlasQ;
        return;
    }
    const int64_t r = B - nq * kBlasQ;
    if (r > kBlasQ) {
        const int64_t h = r / 2;
        start = nq * kBlasQ + (blk == nq ? 0 : h);
        len = blk == nq ? h : r - h;
    } else {
        start = nq * kBlasQ;
        len = r;
    }
}

// pass 2: C = 0; C += block partial, blocks in order; then gW += C.
__global__ void wgrad_blas_reduce_kernel(const float *__restrict__ part, int64_t nblk, int fin, int fout,
                                         const float *__restrict__ d, int64_t B, float *__restrict__ gW,
                                         float *__restrict__ gb) {
    const int64_t E = (int64_t)fin * fout;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < E) {
        float c = 0.0f;
        for (int64_t b = 0; b < nblk; ++b) c = __fadd_rn(c, part[b * E + e]);
        gW[e] = __fadd_rn(gW[e], c);
    }
}

// Bias chains, warp edition: ONE warp per output column runs the column's
// in-order add chain over all B rows.  The 32 lanes load 32 consecutive rows
// of the column per instruction, 8 such loads in flight per lane (256 rows
// ahead of the chain, > the L2 latency at ~4 cycles per add); each round's
// 256 rows go through a 1 KB shared-memory stage and the chain reads them
// in row order with broadcast 16-byte loads (a shuffle per row measured
// ~14 cycles per add: the shuffles' latency sat on the chain); every lane
// carries the same chain (no divergence), lane 0 stores it.  Same additions in the same order
// as numpy's delta.sum(axis=0) (rows in order): bit-identical.  Round 1 ran
// the chains from a cp.async ring in shared memory, 2 columns per CTA (~2 ms
// of a 3.3 ms reference-order C1 step).
constexpr int kChainDepth = 8;   // float4 loads in flight per lane (1024 rows ahead)
constexpr int kWT = 128;         // threads per CTA of wgrad_bias_kernel
__device__ __forceinline__ void bias_chain_warp(const float *__restrict__ dT, int64_t B,
                                                float *__restrict__ gbj, float *__restrict__ stage) {
    // dT: this column's B values, contiguous (column-major copy written by
    // the training kernel); 16-byte aligned when B % 4 == 0
    const int lane = threadIdx.x & 31;
    constexpr int kRows = kChainDepth * 128;   // rows staged per round
    float acc = 0.0f;
    if ((B & 3) == 0 && ((uintptr_t)dT & 15) == 0) {
        const float4 *d4 = reinterpret_cast<const float4 *>(dT);
        const int64_t n4 = B >> 2;
        float4 cur[kChainDepth];
#pragma unroll
        for (int k = 0; k < kChainDepth; ++k) {
            const int64_t r4 = (int64_t)k * 32 + lane;
            cur[k] = r4 < n4 ? __ldg(d4 + r4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float4 *s4 = reinterpret_cast<float4 *>(stage);
        for (int64_t b0 = 0; b0 < B; b0 += kRows) {
            __syncwarp();
#pragma unroll
            for (int k = 0; k < kChainDepth; ++k) s4[k * 32 + lane] = cur[k];
            __syncwarp();
#pragma unroll
            for (int k = 0; k < kChainDepth; ++k) {
                const int64_t r4 = (b0 + kRows) / 4 + (int64_t)k * 32 + lane;
                cur[k] = r4 < n4 ? __ldg(d4 + r4) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            const int nr = (int)(B - b0 < kRows ? B - b0 : kRows);
            if (nr == kRows) {
#pragma unroll 16
                for (int q = 0; q < kRows / 4; ++q) {
                    const float4 v = s4[q];
                    acc = __fadd_rn(acc, v.x);
                    acc = __fadd_rn(acc, v.y);
                    acc = __fadd_rn(acc, v.z);
                    acc = __fadd_rn(acc, v.w);
                }
            } else {
                for (int r = 0; r < nr; ++r) acc = __fadd_rn(acc, stage[r]);
            }
        }
    } else {   // ragged batch: scalar loads, same order
        for (int64_t b0 = 0; b0 < B; b0 += 32) {
            const float v = b0 + lane < B ? __ldg(dT + b0 + lane) : 0.0f;
            const int n = (int)(B - b0 < 32 ? B - b0 : 32);
            for (int i = 0; i < n; ++i) acc = __fadd_rn(acc, __shfl_sync(0xffffffffu, v, i));
        }
    }
    if (lane == 0) *gbj = __fadd_rn(*gbj, acc);
}

// Pass 1 of the reference-order weight gradients and the bias chains in ONE
// launch (no side stream, no allocation): CTAs [0, nbias) run one bias chain
// per warp (all columns of all layers), the rest run the per-layer K-block
// partials (every (block, element) FMA chain of OpenBLAS's K-blocking starts
// from 0, so they are independent; tiled 4 x 4 per thread where the widths
// allow), so the serial chains (~0.5 ms) overlap the parallel partial sums.
struct WgradJob {
    const float *a[3], *d[3], *dT[3];
    float *gb[3], *part[3];
    int fin[3], fout[3], tiled[3];
    int64_t first_cta[4];   // CTA ranges of the partial-sum work per layer
    int n_layers, n_cols, nbias_ctas;
};
__global__ void __launch_bounds__(kWT) wgrad_bias_kernel(const WgradJob job, int64_t B, int64_t nblk) {
    __shared__ __align__(16) float stage[kWT / 32][kChainDepth * 128];
    if ((int64_t)blockIdx.x < job.nbias_ctas) {
        const int w = blockIdx.x * (kWT / 32) + (threadIdx.x >> 5);
        if (w >= job.n_cols) return;
        int l = 0, j = w;
        while (l < job.n_layers - 1 && j >= job.fout[l]) {
            j -= job.fout[l];
            ++l;
        }
        bias_chain_warp(job.dT[l] + (int64_t)j * B, B, job.gb[l] + j, stage[threadIdx.x >> 5]);
        return;
    }
    int l = 0;
    while (l < job.n_layers - 1 && (int64_t)blockIdx.x >= job.first_cta[l + 1]) ++l;
    const int64_t t = ((int64_t)blockIdx.x - job.first_cta[l]) * kWT + threadIdx.x;
    const int fin = job.fin[l], fout = job.fout[l];
    const float *a = job.a[l], *d = job.d[l];
    const int64_t E = (int64_t)fin * fout;
    if (job.tiled[l]) {   // 4 x 4 chains per thread, two float4 loads per 16 FMAs
        const int tj = fout >> 2;
        const int64_t T = (int64_t)(fin >> 2) * tj;
        if (t >= nblk * T) return;
        const int64_t blk = t / T;
        const int e = (int)(t - blk * T);
        const int i0 = (e / tj) * 4, j0 = (e - (e / tj) * tj) * 4;
        int64_t ls, ml;
        blas_block(B, blk, ls, ml);
        float acc[4][4] = {};
#pragma unroll 4
        for (int64_t k = ls; k < ls + ml; ++k) {
            const float4 av = __ldg(reinterpret_cast<const float4 *>(a + k * fin + i0));
            const float4 dv = __ldg(reinterpret_cast<const float4 *>(d + k * fout + j0));
            const float au[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                acc[u][0] = __fmaf_rn(au[u], dv.x, acc[u][0]);
                acc[u][1] = __fmaf_rn(au[u], dv.y, acc[u][1]);
                acc[u][2] = __fmaf_rn(au[u], dv.z, acc[u][2]);
                acc[u][3] = __fmaf_rn(au[u], dv.w, acc[u][3]);
            }
        }
        float *p = job.part[l] + blk * E + (int64_t)i0 * fout + j0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            *reinterpret_cast<float4 *>(p + (int64_t)u * fout) =
                make_float4(acc[u][0], acc[u][1], acc[u][2], acc[u][3]);
    } else {              // one chain per thread
        if (t >= nblk * E) return;
        const int64_t blk = t / E;
        const int e = (int)(t - blk * E);
        const int i = e / fout, j = e - i * fout;
        int64_t ls, ml;
        blas_block(B, blk, ls, ml);
        float acc = 0.0f;
#pragma unroll 8
        for (int64_t k = ls; k < ls + ml; ++k) acc = __fmaf_rn(__ldg(a + k * fin + i), __ldg(d + k * fout + j), acc);
        job.part[l][t] = acc;
    }
}

int64_t mlp_acts_floats(int64_t B, const pg_mlp *m) {
    int64_t w = 0, e = 0;
    for (int l = 0; l < m->n_layers; ++l) {
        w += m->widths[l] + m->widths[l + 1];
        const int64_t el = (int64_t)m->widths[l] * m->widths[l + 1];
        e = el > e ? el : e;
    }
    int64_t cols = 0;
    for (int l = 0; l < m->n_layers; ++l) cols += m->widths[l + 1];
    // + the deltas again, column-major (bias chains) + the per-block partial
    // sums of pass 1, one region per layer
    return B * w + B * cols + (int64_t)m->n_layers * blas_nblocks(B) * e;
}

int mlp_wgrad_blas(const pg_mlp *m, const float *acts, int64_t B, float *gparams, cudaStream_t s) {
    if (int e = validate_mlp(m)) return e;
    if (B == 0) return PG_OK;
    PG_REQUIRE(m->n_layers <= 3, "reference-order weight gradients: at most 3 layers");
    // acts = [a_0 .. a_{n-1} | delta_0 .. delta_{n-1} | delta_l^T (column-major) | partials per layer]
    int64_t a_off = 0, d_off = 0, w = 0, emax = 0;
    for (int l = 0; l < m->n_layers; ++l) {
        d_off += B * m->widths[l];
        w += m->widths[l] + m->widths[l + 1];
        const int64_t el = (int64_t)m->widths[l] * m->widths[l + 1];
        emax = el > emax ? el : emax;
    }
    const int64_t nblk = blas_nblocks(B);
    int64_t cols = 0;
    for (int l = 0; l < m->n_layers; ++l) cols += m->widths[l + 1];
    const float *dT0 = acts + B * w;                              // [delta_l^T ...] column-major
    float *part0 = const_cast<float *>(acts) + B * w + B * cols;
    WgradJob job{};
    job.n_layers = m->n_layers;
    job.n_cols = 0;
    int64_t cta = 0;
    float *g = gparams;
    float *gW[3] = {nullptr, nullptr, nullptr};
    for (int l = 0; l < m->n_layers; ++l) job.n_cols += m->widths[l + 1];
    job.nbias_ctas = (job.n_cols + kWT / 32 - 1) / (kWT / 32);
    cta = job.nbias_ctas;
    for (int l = 0; l < m->n_layers; ++l) {
        const int fin = m->widths[l], fout = m->widths[l + 1];
        const int64_t E = (int64_t)fin * fout;
        const float *av = acts + a_off, *dv = acts + d_off;
        float *part = part0 + (int64_t)l * nblk * emax;
        const bool tiled = fin % 4 == 0 && fout % 4 == 0 && ((uintptr_t)av & 15) == 0 &&
                           ((uintptr_t)dv & 15) == 0 && ((uintptr_t)part & 15) == 0;
        job.a[l] = av;
        job.d[l] = dv;
        job.dT[l] = dT0;
        dT0 += B * fout;
        job.part[l] = part;
        job.fin[l] = fin;
        job.fout[l] = fout;
        job.tiled[l] = tiled ? 1 : 0;
        job.first_cta[l] = cta;
        const int64_t work = tiled ? nblk * E / 16 : nblk * E;
        cta += (work + kWT - 1) / kWT;
        gW[l] = g;
        job.gb[l] = g + E;
        a_off += B * fin;
        d_off += B * fout;
        g += E + fout;
    }
    job.first_cta[m->n_layers] = cta;
    wgrad_bias_kernel<<<(unsigned)cta, kWT, 0, s>>>(job, B, nblk);
    for (int l = 0; l < m->n_layers; ++l) {
        const int64_t E = (int64_t)job.fin[l] * job.fout[l];
        wgrad_blas_reduce_kernel<<<(unsigned)((E + 127) / 128), 128, 0, s>>>(job.part[l], nblk, job.fin[l],
                                                                             job.fout[l], job.d[l], B, gW[l],
                                                                             job.gb[l]);
    }
    return check_launch("mlp_wgrad_blas");
}

}  // namespace pg

using namespace pg;

extern "C" {

int pg_mlp_infer_rows_f32(const float *xs, int64_t B, const pg_mlp *mlp, const float *params,
                          unsigned flags, float *act_ws, float *out, void *stream) {
    return mlp_infer_rows_generic<float>(xs, B, mlp, params, flags, act_ws, out, as_stream(stream));
}
int pg_mlp_infer_rows_f64(const double *xs, int64_t B, const pg_mlp *mlp, const double *params,
                          unsigned flags, double *act_ws, double *out, void *stream) {
    return mlp_infer_rows_generic<double>(xs, B, mlp, params, flags, act_ws, out, as_stream(stream));
}

int pg_decode_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs, int64_t B,
                  const void *feats, const uint8_t *baked, const float *params, unsigned flags,
                  float *ws, float *out, void *stream) {
    return decode_device(grid, mlp, xs, B, feats, baked, params, flags, ws, out, nullptr,
                         as_stream(stream));
}
int pg_decode_cells_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs, int64_t B,
                        const void *feats, const uint8_t *baked, const float *params, unsigned flags,
                        const pg_cells *cells, float *ws, float *out, void *stream) {
    return decode_device(grid, mlp, xs, B, feats, baked, params, flags, ws, out, nullptr,
                         as_stream(stream), cells);
}

static int decode_host_chunked(const pg_grid *grid, const pg_mlp *mlp, const float *h_xs, int64_t B,
                       const void *feats, const uint8_t *baked, const float *params,
                       unsigned flags, int64_t chunk, float *d_xs, float *d_out, float *h_out,
                       void *stream_in, void *stream_compute, void *stream_out, const pg_cells *cells) {
    if (int e = validate_grid(grid)) return e;
    if (int e = validate_mlp(mlp)) return e;
    PG_REQUIRE(decode_fast_ok(grid, mlp), "host decode needs the fused [32,64,64,<=4] shape");
    PG_REQUIRE(chunk >= 1, "chunk must be positive");
    const int d = grid->d, od = mlp->widths[mlp->n_layers];
    cudaStream_t si = as_stream(stream_in), sk = as_stream(stream_compute), so = as_stream(stream_out);
    // Three streams, two buffer slots: H2D on si, kernels on sk, D2H on so,
    // ordered by events — copy-in of chunk c+2 needs only kernel c done (its
    // input slot), kernel c+2 needs only copy-out c done (its output slot), so
    // both copy directions run under the kernels.
    cudaEvent_t ev_in[2], ev_k[2], ev_out[2];
    for (int i = 0; i < 2; ++i) {
        cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev_k[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming);
    }
    // chunk sizes ramp up from chunk/8 and back down at the end: the first
    // H2D and the last D2H are the only transfers nothing overlaps
    const int64_t head[3] = {chunk / 8, chunk / 4, chunk / 2};
    int64_t c = 0, n = 0;
    int err = PG_OK;
    for (int64_t off = 0; off < B; off += n, ++c) {
        const int64_t rem = B - off;
        n = chunk;
        if (c < 3 && head[c] > 0) n = head[c];
        if (rem <= chunk + chunk / 2 && rem > chunk / 8) {
            n = rem / 2 > chunk / 8 ? (rem + 1) / 2 : rem;
            if (n > chunk) n = chunk;
        }
        if (n > rem) n = rem;
        if (n < 1) n = rem;
        const int slot = (int)(c & 1);
        float *dx = d_xs + (int64_t)slot * chunk * d;
        float *dout = d_out + (int64_t)slot * chunk * od;
        if (c >= 2) cudaStreamWaitEvent(si, ev_k[slot], 0);     // kernel c-2 has read this input slot
        cudaMemcpyAsync(dx, h_xs + off * d, sizeof(float) * n * d, cudaMemcpyHostToDevice, si);
        cudaEventRecord(ev_in[slot], si);
        cudaStreamWaitEvent(sk, ev_in[slot], 0);
        if (c >= 2) cudaStreamWaitEvent(sk, ev_out[slot], 0);   // copy-out c-2 has drained this output slot
        if ((err = decode_device(grid, mlp, dx, n, feats, baked, params, flags, nullptr, dout, nullptr, sk, cells)))
            break;
        cudaEventRecord(ev_k[slot], sk);
        cudaStreamWaitEvent(so, ev_k[slot], 0);
        cudaMemcpyAsync(h_out + off * od, dout, sizeof(float) * n * od, cudaMemcpyDeviceToHost, so);
        cudaEventRecord(ev_out[slot], so);
    }
    cudaStreamSynchronize(si);
    cudaStreamSynchronize(sk);
    cudaStreamSynchronize(so);
    for (int i = 0; i < 2; ++i) {
        cudaEventDestroy(ev_in[i]);
        cudaEventDestroy(ev_k[i]);
        cudaEventDestroy(ev_out[i]);
    }
    if (err) return err;
    return check_launch("decode_host");
}
int pg_decode_host_f32(const pg_grid *grid, const pg_mlp *mlp, const float *h_xs, int64_t B,
                       const void *feats, const uint8_t *baked, const float *params,
                       unsigned flags, int64_t chunk, float *d_xs, float *d_out, float *h_out,
                       void *stream_in, void *stream_compute, void *stream_out) {
    return decode_host_chunked(grid, mlp, h_xs, B, feats, baked, params, flags, chunk, d_xs, d_out, h_out,
                               stream_in, stream_compute, stream_out, nullptr);
}
int pg_decode_host_cells_f32(const pg_grid *grid, const pg_mlp *mlp, const float *h_xs, int64_t B,
                             const void *feats, const uint8_t *baked, const float *params, unsigned flags,
                             const pg_cells *cells, int64_t chunk, float *d_xs, float *d_out, float *h_out,
                             void *stream_in, void *stream_compute, void *stream_out) {
    return decode_host_chunked(grid, mlp, h_xs, B, feats, baked, params, flags, chunk, d_xs, d_out, h_out,
                               stream_in, stream_compute, stream_out, cells);
}

// Streaming end-to-end decode: ONE tcgen05 decode launch over the whole
// batch, fed chunk by chunk by the copy engine (see DecodeStream): removes
// the per-launch prologue (weights, shared-memory tables, TMEM) and tail
// that chunked launches pay (~35 us each), and lets the first tiles start
// as soon as the first chunk lands.
typedef CUresult (*pg_write_value_fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*pg_wait_value_fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static pg_write_value_fn g_write_value = nullptr;
static pg_wait_value_fn g_wait_value = nullptr;
static bool stream_memops() {
    // stream memory operations (CUDA >= 12: always available; the v1
    // capability attribute is deprecated), resolved through the runtime's
    // driver entry-point query so the library needs no link against libcuda
    static int state = 0;   // 0 unknown, 1 ok, -1 unavailable
    if (state == 0) {
        cudaDriverEntryPointQueryResult q1 = cudaDriverEntryPointSymbolNotFound, q2 = q1;
        cudaGetDriverEntryPoint("cuStreamWriteValue32", (void **)&g_write_value, cudaEnableDefault, &q1);
        cudaGetDriverEntryPoint("cuStreamWaitValue32", (void **)&g_wait_value, cudaEnableDefault, &q2);
        state = (q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && g_write_value &&
                 g_wait_value)
                    ? 1
                    : -1;
        if (getenv("PG_DEBUG_MEMOPS"))
            fprintf(stderr, "pg: stream memops q1=%d q2=%d write=%p wait=%p\n", (int)q1, (int)q2,
                    (void *)g_write_value, (void *)g_wait_value);
        cudaGetLastError();
    }
    return state == 1;
}

int pg_decode_stream_supported(const pg_grid *grid, const pg_mlp *mlp, unsigned flags) {
    return grid && mlp && decode_fast_ok(grid, mlp) && !(flags & (PG_EXACT_MLP | PG_NO_TENSOR)) && stream_memops();
}

static bool is_pinned_host(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

static int decode_host_stream(const pg_grid *grid, const pg_mlp *mlp, const float *h_xs, int64_t B,
                              const void *feats, const uint8_t *baked, const float *params, unsigned flags,
                              int64_t chunk, float *d_xs, float *d_out, uint32_t *d_flags, float *h_out,
                              void *stream_in, void *stream_compute, void *stream_out, const pg_cells *cells) {
    if (int e = validate_grid(grid)) return e;
    if (int e = validate_mlp(mlp)) return e;
    PG_REQUIRE(pg_decode_stream_supported(grid, mlp, flags),
               "streaming decode needs the tcgen05 [32,64,64,<=4] path and stream memory operations");
    PG_REQUIRE(chunk >= 128 && (chunk & (chunk - 1)) == 0, "chunk must be a power of two >= 128 queries");
    PG_REQUIRE(B >= 0 && (B == 0 || (h_xs && d_xs && d_out && d_flags && h_out)), "null buffer");
    if (B == 0) return PG_OK;
    // a group whose chunk flag times out reads the inputs from h_xs through
    // UVA: it must be page-locked host memory
    PG_REQUIRE(is_pinned_host(h_xs) && is_pinned_host(h_out),
               "streaming decode needs page-locked (pinned) host buffers");
    const int d = grid->d, od = mlp->widths[3];
    const int64_t nch = (B + chunk - 1) / chunk;
    cudaStream_t si = as_stream(stream_in), sk = as_stream(stream_compute), so = as_stream(stream_out);
    uint32_t *ready = d_flags, *done = d_flags + nch;
    cudaEvent_t ev0;
    cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming);
    const bool dbg_nocopy = getenv("PG_DEBUG_STREAM_NOCOPY") != nullptr;   // kernel-only probe
    cudaMemsetAsync(d_flags, 0, sizeof(uint32_t) * (2 * nch + 1), sk);
    if (dbg_nocopy) cudaMemsetAsync(d_flags, 1, sizeof(uint32_t) * nch, sk);
    cudaEventRecord(ev0, sk);
    cudaStreamWaitEvent(si, ev0, 0);
    cudaStreamWaitEvent(so, ev0, 0);
    DecodeStream st;
    st.ready = ready;
    st.done = done;
    while ((128ll << st.chunk_tiles_log2) < chunk) ++st.chunk_tiles_log2;
    st.timeout_ns = 2ull * 1000 * 1000;   // then read from host memory (see the kernel)
    st.host_xs = h_xs;
    st.fallbacks = d_flags + 2 * nch;
    const bool half = (flags & PG_HALF_FEATS) != 0;
    static const bool dbg = getenv("PG_DEBUG_STREAM") != nullptr;
    cudaEvent_t dk0 = nullptr, dk1 = nullptr, dend = nullptr;
    if (dbg) {
        cudaEventCreate(&dk0);
        cudaEventCreate(&dk1);
        cudaEventCreate(&dend);
        cudaEventRecord(dk0, sk);
    }
    int err = decode_umma(grid, od, d_xs, B, feats, half, baked, params, (flags & PG_SIGMOID) ? 1 : 0,
                          (int)(flags & (PG_SMEM_TABLES | PG_NO_SMEM_TABLES)), d_out, sk, st, cells);
    if (dbg) cudaEventRecord(dk1, sk);
    for (int64_t c = 0; c < nch && !err && !dbg_nocopy; ++c) {
        const int64_t off = c * chunk, n = B - off < chunk ? B - off : chunk;
        cudaMemcpyAsync(d_xs + off * d, h_xs + off * d, sizeof(float) * n * d, cudaMemcpyHostToDevice, si);
        CUresult r1 = g_write_value((CUstream)si, (CUdeviceptr)(ready + c), 1u, 0);
        CUresult r2 = g_wait_value((CUstream)so, (CUdeviceptr)(done + c), (cuuint32_t)((n + 127) / 128),
                                   CU_STREAM_WAIT_VALUE_GEQ);
        if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS) {
            // cannot feed the running kernel: it would time out; report instead
            set_error("stream memory operation failed (" + std::to_string((int)r1) + ", " +
                      std::to_string((int)r2) + ")");
            err = PG_ERR_CUDA;
        }
        cudaMemcpyAsync(h_out + off * od, d_out + off * od, sizeof(float) * n * od, cudaMemcpyDeviceToHost, so);
    }
    if (dbg) cudaEventRecord(dend, so);
    cudaStreamSynchronize(si);
    cudaStreamSynchronize(sk);
    cudaStreamSynchronize(so);
    cudaEventDestroy(ev0);
    if (dbg) {
        float k = 0, t = 0;
        cudaEventElapsedTime(&k, dk0, dk1);
        cudaEventElapsedTime(&t, dk0, dend);
        fprintf(stderr, "pg stream decode: kernel %.3f ms, kernel start -> last D2H %.3f ms\n", k, t);
        cudaEventDestroy(dk0);
        cudaEventDestroy(dk1);
        cudaEventDestroy(dend);
    }
    if (err) return err;
    return check_launch("decode_host_stream");
}
int pg_decode_host_stream_f32(const pg_grid *grid, const pg_mlp *mlp, const float *h_xs, int64_t B,
                              const void *feats, const uint8_t *baked, const float *params, unsigned flags,
                              int64_t chunk, float *d_xs, float *d_out, uint32_t *d_flags, float *h_out,
                              void *stream_in, void *stream_compute, void *stream_out) {
    return decode_host_stream(grid, mlp, h_xs, B, feats, baked, params, flags, chunk, d_xs, d_out, d_flags, h_out,
                              stream_in, stream_compute, stream_out, nullptr);
}
int pg_decode_host_stream_cells_f32(const pg_grid *grid, const pg_mlp *mlp, const float *h_xs, int64_t B,
                                    const void *feats, const uint8_t *baked, const float *params, unsigned flags,
                                    const pg_cells *cells, int64_t chunk, float *d_xs, float *d_out,
                                    uint32_t *d_flags, float *h_out, void *stream_in, void *stream_compute,
                                    void *stream_out) {
    return decode_host_stream(grid, mlp, h_xs, B, feats, baked, params, flags, chunk, d_xs, d_out, d_flags, h_out,
                              stream_in, stream_compute, stream_out, cells);
}

// Zero-copy end-to-end decode: the decode kernel reads the coordinates from
// and writes the outputs to pinned host memory directly (UVA).  No copies,
// flags or extra device memory (measured 5.50 ms per 2^24 queries vs 5.22
// for the streaming path; a variant prefetching each tile's coordinates a
// tile ahead spilled at the 80-register cap and ran 5.62 ms).

int pg_decode_host_zc_f32(const pg_grid *grid, const pg_mlp *mlp, const float *h_xs, int64_t B,
                          const void *feats, const uint8_t *baked, const float *params, unsigned flags,
                          float *h_out, void *stream) {
    if (int e = validate_grid(grid)) return e;
    if (int e = validate_mlp(mlp)) return e;
    PG_REQUIRE(decode_fast_ok(grid, mlp) && !(flags & (PG_EXACT_MLP | PG_NO_TENSOR)) && (flags & PG_HALF_FEATS),
               "zero-copy decode needs the tcgen05 [32,64,64,<=4] path on fp16 tables");
    if (B == 0) return PG_OK;
    PG_REQUIRE(is_pinned_host(h_xs) && is_pinned_host(h_out),
               "zero-copy decode needs page-locked (pinned) host buffers");
    cudaStream_t s = as_stream(stream);
    if (int e = decode_umma(grid, mlp->widths[3], h_xs, B, feats, true, baked, params,
                            (flags & PG_SIGMOID) ? 1 : 0, (int)(flags & (PG_SMEM_TABLES | PG_NO_SMEM_TABLES)),
                            h_out, s))
        return e;
    cudaStreamSynchronize(s);
    return check_launch("decode_host_zc");
}

int64_t pg_mlp_train_workspace_floats(int64_t B, const pg_mlp *mlp) { return mlp_train_ws(B, mlp); }

int pg_mlp_train_f32(const pg_mlp *mlp, const float *y, const float *targets, int64_t B,
                     const float *params, float scale, unsigned flags, float *gparams, float *dy,
                     double *loss_sum, float *ws, void *stream) {
    return mlp_train_generic<float>(mlp, y, targets, B, params, scale, flags, gparams, dy, loss_sum,
                                    ws, as_stream(stream));
}
int pg_mlp_train_det_f32(const pg_mlp *mlp, const float *y, const float *targets, int64_t B,
                         const float *params, float scale, unsigned flags, uint64_t *gparams_fx,
                         float *dy, uint64_t *loss_fx, float *ws, void *stream) {
    return mlp_train_generic<float, fx_t, fx_t>(mlp, y, targets, B, params, scale, flags,
                                                (fx_t *)gparams_fx, dy, (fx_t *)loss_fx, ws,
                                                as_stream(stream));
}
int pg_ray_samples_f32(const float *origins, const float *dirs, int64_t R, int S, float *pts,
                       float *deltas, void *stream) {
    PG_REQUIRE(R >= 0 && S >= 1, "ray_samples: R >= 0 and S >= 1");
    if (R == 0) return PG_OK;
    ray_samples_kernel<<<grid_for(R * S, 256), 256, 0, as_stream(stream)>>>(origins, dirs, R, S, pts, deltas);
    return check_launch("ray_samples");
}
int pg_ray_samples_targets_f32(const float *origins, const float *dirs, const float *rgb, int64_t R, int S,
                               float *pts, float *deltas, float *t4, void *stream) {
    PG_REQUIRE(R >= 0 && S >= 1, "ray_samples: R >= 0 and S >= 1");
    PG_REQUIRE(R == 0 || (rgb && t4 && ((uintptr_t)t4 & 15) == 0), "ray_samples: rgb / 16-byte aligned t4");
    if (R == 0) return PG_OK;
    ray_samples_kernel<<<grid_for(R * S, 256), 256, 0, as_stream(stream)>>>(origins, dirs, R, S, pts, deltas,
                                                                          rgb, t4);
    return check_launch("ray_samples_targets");
}
int pg_composite_fwd_f32(const float *raw, const float *deltas, int64_t R, int S, float *rgb,
                         float *weights, void *stream) {
    PG_REQUIRE(R >= 0 && S >= 1, "composite: R >= 0 and S >= 1");
    PG_REQUIRE(R == 0 || (raw && deltas && rgb), "composite: null buffer");
    if (R == 0) return PG_OK;
    composite_fwd_kernel<<<grid_for(R, 128), 128, 0, as_stream(stream)>>>(raw, deltas, R, S, rgb, weights);
    return check_launch("composite_fwd");
}
int pg_nerf_train_f32(const pg_mlp *mlp, const float *y, const float *deltas, const float *target_rgb,
                      int64_t R, int S, const float *params, float scale, float *gparams, float *dy,
                      double *loss_sum, float *ws, void *stream) {
    PG_REQUIRE(R >= 0 && S >= 1, "nerf_train: R >= 0 and S >= 1");
    PG_REQUIRE(mlp && mlp->n_layers >= 1 && mlp->widths[mlp->n_layers] == 4,
               "nerf_train: the MLP must output (sigma, r, g, b)");
    if (R == 0) return PG_OK;
    cudaStream_t s = as_stream(stream);
    return mlp_train_core<float, float>(mlp, y, R * S, params, gparams, dy, ws, s, [&](const float *zout, float *delta) {
        composite_loss_kernel<double><<<grid_for(R, 128), 128, 0, s>>>(zout, deltas, target_rgb, R, S, scale,
                                                                      delta, loss_sum);
    });
}
int64_t pg_mlp_acts_floats(int64_t B, const pg_mlp *mlp) { return mlp_acts_floats(B, mlp); }
int pg_mlp_wgrad_blas_f32(const pg_mlp *mlp, const float *acts, int64_t B, float *gparams, void *stream) {
    return mlp_wgrad_blas(mlp, acts, B, gparams, as_stream(stream));
}
int pg_mlp_train_f64(const pg_mlp *mlp, const double *y, const double *targets, int64_t B,
                     const double *params, double scale, unsigned flags, double *gparams,
                     double *dy, double *loss_sum, double *ws, void *stream) {
    return mlp_train_generic<double>(mlp, y, targets, B, params, scale, flags, gparams, dy,
                                     loss_sum, ws, as_stream(stream));
}
int pg_mlp_forward_f32(const pg_mlp *mlp, const float *x, int64_t B, const float *params, float *ws,
                       float *out, void *stream) {
    return mlp_forward_generic<float>(mlp, x, B, params, ws, out, as_stream(stream));
}
int pg_mlp_forward_f64(const pg_mlp *mlp, const double *x, int64_t B, const double *params, double *ws,
                       double *out, void *stream) {
    return mlp_forward_generic<double>(mlp, x, B, params, ws, out, as_stream(stream));
}
int pg_mlp_backward_f32(const pg_mlp *mlp, const float *x, int64_t B, const float *params,
                        const float *upstream, float *gparams, float *dx, float *ws, void *stream) {
    return mlp_backward_generic<float>(mlp, x, B, params, upstream, gparams, dx, ws, as_stream(stream));
}
int pg_mlp_backward_f64(const pg_mlp *mlp, const double *x, int64_t B, const double *params,
                        const double *upstream, double *gparams, double *dx, double *ws, void *stream) {
    return mlp_backward_generic<double>(mlp, x, B, params, upstream, gparams, dx, ws, as_stream(stream));
}

}  // extern "C"
