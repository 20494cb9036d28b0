// Fused training pass on sm_100a, OpenBLAS-order (exact) variant — selected by
// PG_EXACT_MLP and by reference-order mode; the default fast path with the
// MLP on the tensor cores is pg_train_mma.cu.  For every 64-sample tile, ONE
// kernel does
//   encode fwd (16 levels, F=2)  ->  MLP [32,64,64,out<=4] fwd  ->  squared
//   error + dpred  ->  MLP bwd (weight grads held in registers across tiles,
//   dgrads)  ->  encode bwd (straight-through scatter into gfeat/gconf)
// with every activation in shared memory (trainer.py:118-148, mlp.py:55-85,
// encoding.py:89-133 of the reference).
//
// Forward GEMMs and the data-gradient GEMMs reproduce numpy/OpenBLAS's
// arithmetic exactly: OpenBLAS sgemm (SkylakeX kernel, K <= 64) computes each
// output as a sequential fused multiply-add chain over k starting from 0, and
// numpy then adds the bias / multiplies the ReLU mask as separate rounded
// operations (verified bit-for-bit in the build container).  So y, the
// activations, the loss terms and dy = dL/dy are bit-identical to the
// reference for the same parameters and batch; only the cross-sample sums
// (weight/bias gradients, table scatters) are reordered.
#include <cstdlib>

#include "pg_encode_dev.cuh"
#include "pg_phase.cuh"

namespace pg {


constexpr int kT = 64;    // samples per tile
constexpr int kNT = 256;  // threads per CTA (2 CTAs per SM: one's memory-bound
                          // encode phases overlap the other's FFMA MLP phases)
constexpr int kI = 32;    // L*F
constexpr int kH = 64;    // hidden width
constexpr int kO = 4;     // padded output width

struct TrainW {           // weights: shared by the tile pipelines of a CTA
    float w0[kI * kH], w1[kH * kH], w2[kH * kO];      // [in][out]
    float w0t[kH * kI], w1t[kH * kH];                 // [out][in]
    float b0[kH], b1[kH], b2[kO];
};
struct TrainG {           // one tile pipeline's activations
    float yT[kI * kT];    // encodings, later dL/dy       (swizzled rows)
    float z1T[kH * kT];   // layer-1 activations relu(z1), later delta_1
    float z2T[kH * kT];   // layer-2 activations relu(z2), later delta_2
    float d3[kT * kO];    // dL/d(out), sample-major
    float xs[kT * 3];
    float tg[kT * kO];
    double red[kNT / 32];
};
// NG tile pipelines of kNT threads per CTA (pg_train_mma.cu's layout)
template <int NG>
struct TrainSmemT {
    TrainW w;
    TrainG g[NG];
};

__device__ __forceinline__ int sw(int row, int col) {
    const int chunk = (col >> 2) ^ ((row >> 2) & 7);
    return row * kT + (chunk << 2) + (col & 3);
}
// parity mode: copy a transposed smem tile (rows = features) to acts rows
__device__ __forceinline__ void dump_tile(const float *srcT, int width, int nv, float *dst, int tid) {
    for (int i = tid; i < nv * width; i += kNT) {
        const int q = i / width, c = i - q * width;
        dst[(int64_t)q * width + c] = srcT[sw(c, q)];
    }
}
// ... and column-major ([feature][sample], stride B) for the in-order bias
// chains, which then read each column as one contiguous stream
__device__ __forceinline__ void dump_tile_T(const float *srcT, int width, int nv, float *dstT, int64_t B, int tid) {
    for (int i = tid; i < nv * width; i += kNT) {
        const int c = i / nv, q = i - c * nv;
        dstT[(int64_t)c * B + q] = srcT[sw(c, q)];
    }
}
__device__ __forceinline__ float relu_np(float z) { return z < 0.0f ? 0.0f : z; }  // np.maximum(z, 0)
__device__ __forceinline__ float mask_np(float z) { return z > 0.0f ? 1.0f : 0.0f; }  // (pre > 0)

// out^T[j][q] = relu( fma-chain_k( in^T[k][q] * W[k][j] ) + b[j] )   (j < 64, q < 64)
// The ReLU is applied once at the write (np.maximum(z, 0) of the reference);
// the backward masks test h > 0, the same predicate as z > 0.
template <int K>
__device__ __forceinline__ void fwd_layer(const float *__restrict__ inT, const float *__restrict__ W,
                                          const float *__restrict__ b, float *__restrict__ outT) {
    const int t = threadIdx.x & (kNT - 1), og = t & 15, pg = t >> 4;  // 4 outputs x 4 samples (pipeline-local thread)
    float acc[4][4] = {};
#pragma unroll 8
    for (int k = 0; k < K; ++k) {
        const float4 a = *reinterpret_cast<const float4 *>(inT + sw(k, pg * 4));
        const float4 w = *reinterpret_cast<const float4 *>(W + k * kH + og * 4);
        const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            acc[i][0] = __fmaf_rn(av[i], w.x, acc[i][0]);
            acc[i][1] = __fmaf_rn(av[i], w.y, acc[i][1]);
            acc[i][2] = __fmaf_rn(av[i], w.z, acc[i][2]);
            acc[i][3] = __fmaf_rn(av[i], w.w, acc[i][3]);
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float bj = b[og * 4 + j];
        *reinterpret_cast<float4 *>(outT + sw(og * 4 + j, pg * 4)) =
            make_float4(relu_np(__fadd_rn(acc[0][j], bj)), relu_np(__fadd_rn(acc[1][j], bj)),
                        relu_np(__fadd_rn(acc[2][j], bj)), relu_np(__fadd_rn(acc[3][j], bj)));
    }
}

// NG = 1: one 8-warp tile pipeline per CTA, two CTAs per SM.  NG = 2: one
// CTA per SM running two 8-warp pipelines that share the weights (50 KB less
// shared memory per SM) and ping-pong their FFMA MLP phases (named barriers
// 3/4, as in pg_train_mma.cu), so one pipeline's MLP always runs beside the
// other's encode.  The per-element arithmetic is the same in both.
template <typename FT, int D, int NPM, typename ACC, typename LACC, int NG>
__global__ void __launch_bounds__(kNT *NG, 2 / NG)
    train_fused_kernel(const pg_grid g, const float *__restrict__ xs, const float *__restrict__ targets,
                       int64_t B, const FT *__restrict__ feats_fwd, const float *__restrict__ feats,
                       const uint8_t *__restrict__ baked, const float *__restrict__ conf,
                       const float *__restrict__ params, int od, float scale, int sigmoid,
                       ACC *__restrict__ gfeat, ACC *__restrict__ gconf,
                       uint8_t *__restrict__ touched, ACC *__restrict__ gparams,
                       LACC *__restrict__ loss_sum, float *__restrict__ dy_out,
                       float *__restrict__ acts) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TrainSmemT<NG> &S = *reinterpret_cast<TrainSmemT<NG> *>(smem_raw);
    const int gid = NG == 1 ? 0 : (int)(threadIdx.x >> 8);   // tile pipeline
    const int tid = threadIdx.x & (kNT - 1);
    TrainW &W = S.w;
    TrainG &G = S.g[gid];
    auto gsync = [&]() {   // barrier of this pipeline's threads
        if constexpr (NG == 1) __syncthreads();
        else asm volatile("bar.sync %0, %1;" ::"r"(1 + gid), "r"(kNT) : "memory");
    };
    auto bar_sync = [&](int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(2 * kNT) : "memory"); };
    auto bar_arrive = [&](int id) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(2 * kNT) : "memory"); };
    // ---- parameters -> shared (both layouts), by all NG pipelines ----
    {
        const int tid = threadIdx.x;
        constexpr int kNT = ::pg::kNT * NG;
        const float *p = params;
        for (int i = tid; i < kI * kH; i += kNT) {
            const float v = p[i];
            W.w0[i] = v;
            W.w0t[(i % kH) * kI + i / kH] = v;
        }
        p += kI * kH;
        for (int i = tid; i < kH; i += kNT) W.b0[i] = p[i];
        p += kH;
        for (int i = tid; i < kH * kH; i += kNT) {
            const float v = p[i];
            W.w1[i] = v;
            W.w1t[(i % kH) * kH + i / kH] = v;
        }
        p += kH * kH;
        for (int i = tid; i < kH; i += kNT) W.b1[i] = p[i];
        p += kH;
        for (int i = tid; i < kH * kO; i += kNT) {
            const int k = i / kO, j = i % kO;
            const float v = j < od ? p[k * od + j] : 0.0f;
            W.w2[i] = v;
        }
        p += kH * od;
        for (int i = tid; i < kO; i += kNT) W.b2[i] = i < od ? p[i] : 0.0f;
    }
    // persistent per-thread gradient accumulators
    float gW2 = 0.0f;                 // (k = tid&63, j = tid>>6)
    float gB2 = 0.0f;                 // j = tid>>6 (threads with tid&63 == 0)
    float gW1[4][4] = {};             // i = (tid>>4)*4 + u, j = (tid&15)*4 + v
    float gB1[4] = {};                // j = tid*4 + v (tid < 16)
    float gW0[2][4] = {};             // i = (tid>>4)*2 + u, j = (tid&15)*4 + v
    float gB0[4] = {};                // j = tid*4 + v (tid < 16)
    double lsum = 0.0;
    PG_PH_INIT

    const int64_t ntiles = (B + kT - 1) / kT;
    // a tile's coordinates and targets (one value of each per thread, since
    // kT*D <= kNT and kT*kO == kNT) are fetched one tile ahead into registers
    static_assert(kT * 3 <= kNT && kT * kO == kNT, "one prefetched value per thread");
    auto fetch = [&](int64_t t, float &fx, float &ft) {
        const int64_t q0 = t * kT;
        const int n = t < ntiles ? (int)((B - q0) < kT ? (B - q0) : kT) : 0;
        fx = (tid < kT * D && tid < n * D) ? __ldg(xs + q0 * D + tid) : 0.5f;
        const int q = tid / kO, j = tid % kO;
        ft = (q < n && j < od) ? __ldg(targets + (q0 + q) * od + j) : 0.0f;
    };
    // tiles of this pipeline: first, first + stride, ...; every pipeline of a
    // CTA runs as many iterations as its first one (the most), so the
    // ping-pong barrier counts match up
    const int64_t first = (int64_t)blockIdx.x * NG + gid, stride = (int64_t)gridDim.x * NG;
    const int64_t base0 = (int64_t)blockIdx.x * NG;
    const int64_t n_iter = base0 < ntiles ? (ntiles - base0 + stride - 1) / stride : 0;
    float pf_x, pf_t;
    fetch(first, pf_x, pf_t);
    __syncthreads();   // weights staged
    for (int64_t iter = 0; iter < n_iter; ++iter) {
        const int64_t tile = first + iter * stride;
        if (tile >= ntiles) {   // (only pipeline 1's last iteration) keep the barrier counts
            if (NG > 1) {
                if (iter > 0) bar_sync(4);
                bar_arrive(3);
            }
            continue;
        }
        const int64_t p0 = tile * kT;
        const int nv = (int)((B - p0) < kT ? (B - p0) : kT);
        gsync();
        PG_PH(11);
        if (tid < kT * D) G.xs[tid] = pf_x;
        G.tg[tid] = pf_t;
        fetch(tile + stride, pf_x, pf_t);
        gsync();
        PG_PH(0);
        // ---- encode forward: thread = (sample pl, levels lsub + 4*it) ----
        const int pl = tid & (kT - 1), lsub = tid >> 6;
        float x[D];
#pragma unroll
        for (int a = 0; a < D; ++a) x[a] = G.xs[pl * D + a];
#pragma unroll 2
        for (int it = 0; it < 4; ++it) {
            const int l = lsub + 4 * it;
            const float2 yv = encode_level_fwd2_rng<FT, D>(g, l, x, feats_fwd, baked);
            G.yT[sw(2 * l, pl)] = yv.x;
            G.yT[sw(2 * l + 1, pl)] = yv.y;
        }
        gsync();
        if (NG > 1) {   // wait for the other pipeline's previous MLP to end
            if (gid == 0) bar_sync(3);
            else if (iter > 0) bar_sync(4);
        }
        PG_PH(1);
        if (acts) dump_tile(G.yT, kI, nv, acts + p0 * kI, tid);
        fwd_layer<kI>(G.yT, W.w0, W.b0, G.z1T);
        gsync();
        PG_PH(2);
        if (acts) dump_tile(G.z1T, kH, nv, acts + B * kI + p0 * kH, tid);
        fwd_layer<kH>(G.z1T, W.w1, W.b1, G.z2T);
        gsync();
        PG_PH(3);
        if (acts) dump_tile(G.z2T, kH, nv, acts + B * (kI + kH) + p0 * kH, tid);
        // ---- output layer, loss, dpred (trainer.py:122-136) ----
        {
            const int q = tid & (kT - 1), j = tid >> 6;
            float d = 0.0f;
            if (j < od && q < nv) {
                float acc = 0.0f;
#pragma unroll 16
                for (int k = 0; k < kH; ++k) acc = __fmaf_rn(G.z2T[sw(k, q)], W.w2[k * kO + j], acc);
                const float o = __fadd_rn(acc, W.b2[j]);
                const float pred = sigmoid ? 1.0f / (1.0f + expf(-o)) : o;
                const float diff = __fsub_rn(pred, G.tg[q * kO + j]);
                lsum += (double)diff * (double)diff;
                d = __fmul_rn(diff, scale);
                if (sigmoid) d = __fmul_rn(d, __fmul_rn(pred, __fsub_rn(1.0f, pred)));
            }
            G.d3[q * kO + j] = d;
        }
        gsync();
        PG_PH(4);
        if (acts) {
            for (int i = tid; i < nv * od; i += kNT)
                acts[B * (kI + 4 * kH) + p0 * od + i] = G.d3[(i / od) * kO + i % od];
            // column-major copy for the bias chains: [d0^T | d1^T | d2^T] after the activations
            float *d2T = acts + B * (kI + 4 * kH + od) + 2 * B * kH + p0;
            for (int i = tid; i < nv * od; i += kNT) {
                const int j = i / nv, q = i - j * nv;
                d2T[(int64_t)j * B + q] = G.d3[q * kO + j];
            }
        }
        // ---- dW2 += h2^T d3, db2 += sum d3 (4 samples per shared load) ----
        {
            const int k = tid & 63, j = tid >> 6;
            float acc = 0.0f, bs = 0.0f;
#pragma unroll 4
            for (int q = 0; q < kT; q += 4) {
                const float4 h = *reinterpret_cast<const float4 *>(G.z2T + sw(k, q));
                const float d0 = G.d3[q * kO + j], d1 = G.d3[(q + 1) * kO + j];
                const float d2 = G.d3[(q + 2) * kO + j], d3v = G.d3[(q + 3) * kO + j];
                acc = __fmaf_rn(h.x, d0, acc);
                acc = __fmaf_rn(h.y, d1, acc);
                acc = __fmaf_rn(h.z, d2, acc);
                acc = __fmaf_rn(h.w, d3v, acc);
                bs += (d0 + d1) + (d2 + d3v);
            }
            gW2 += acc;
            if (k == 0) gB2 += bs;
        }
        gsync();
        PG_PH(5);
        // ---- delta2 = (d3 @ W2^T) * (z2 > 0), in place over z2 ----
        {
            const int og = tid & 15, pg = tid >> 4;
            float dq[4][kO];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float4 v = *reinterpret_cast<const float4 *>(G.d3 + (pg * 4 + i) * kO);
                dq[i][0] = v.x; dq[i][1] = v.y; dq[i][2] = v.z; dq[i][3] = v.w;
            }
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int k = og * 4 + jj;
                const float4 wv = *reinterpret_cast<const float4 *>(W.w2 + k * kO);
                const float w[kO] = {wv.x, wv.y, wv.z, wv.w};
                float4 z = *reinterpret_cast<float4 *>(G.z2T + sw(k, pg * 4));
                float zv[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    float acc = 0.0f;   // fma chain over j < od, as the sgemm kernel
#pragma unroll
                    for (int j = 0; j < kO; ++j)
                        if (j < od) acc = __fmaf_rn(dq[i][j], w[j], acc);
                    zv[i] = __fmul_rn(acc, mask_np(zv[i]));
                }
                *reinterpret_cast<float4 *>(G.z2T + sw(k, pg * 4)) = make_float4(zv[0], zv[1], zv[2], zv[3]);
            }
        }
        gsync();
        PG_PH(6);
        if (acts) {
            dump_tile(G.z2T, kH, nv, acts + B * (kI + 3 * kH) + p0 * kH, tid);
            dump_tile_T(G.z2T, kH, nv, acts + B * (kI + 4 * kH + od) + B * kH + p0, B, tid);
        }
        // ---- dW1 += h1^T delta2, db1 += sum delta2 (summed by the ig == 0 threads) ----
        {
            const int jg = tid & 15, ig = tid >> 4;
            float bs[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            for (int q = 0; q < kT; q += 4) {
                float4 a[4], dd[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) a[u] = *reinterpret_cast<const float4 *>(G.z1T + sw(ig * 4 + u, q));
#pragma unroll
                for (int v = 0; v < 4; ++v) dd[v] = *reinterpret_cast<const float4 *>(G.z2T + sw(jg * 4 + v, q));
                if (ig == 0) {
#pragma unroll
                    for (int v = 0; v < 4; ++v) bs[v] += (dd[v].x + dd[v].y) + (dd[v].z + dd[v].w);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        float s = gW1[u][v];
                        s = __fmaf_rn(a[u].x, dd[v].x, s);
                        s = __fmaf_rn(a[u].y, dd[v].y, s);
                        s = __fmaf_rn(a[u].z, dd[v].z, s);
                        s = __fmaf_rn(a[u].w, dd[v].w, s);
                        gW1[u][v] = s;
                    }
            }
            if (ig == 0) {
#pragma unroll
                for (int v = 0; v < 4; ++v) gB1[v] += bs[v];
            }
        }
        gsync();
        PG_PH(7);
        // ---- delta1 = (delta2 @ W1^T) * (z1 > 0), in place over z1 ----
        {
            const int og = tid & 15, pg = tid >> 4;
            float acc[4][4] = {};
#pragma unroll 8
            for (int j = 0; j < kH; ++j) {
                const float4 a = *reinterpret_cast<const float4 *>(G.z2T + sw(j, pg * 4));
                const float4 w = *reinterpret_cast<const float4 *>(W.w1t + j * kH + og * 4);
                const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    acc[i][0] = __fmaf_rn(av[i], w.x, acc[i][0]);
                    acc[i][1] = __fmaf_rn(av[i], w.y, acc[i][1]);
                    acc[i][2] = __fmaf_rn(av[i], w.z, acc[i][2]);
                    acc[i][3] = __fmaf_rn(av[i], w.w, acc[i][3]);
                }
            }
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                float *dst = G.z1T + sw(og * 4 + jj, pg * 4);
                const float4 z = *reinterpret_cast<float4 *>(dst);
                *reinterpret_cast<float4 *>(dst) =
                    make_float4(__fmul_rn(acc[0][jj], mask_np(z.x)), __fmul_rn(acc[1][jj], mask_np(z.y)),
                                __fmul_rn(acc[2][jj], mask_np(z.z)), __fmul_rn(acc[3][jj], mask_np(z.w)));
            }
        }
        gsync();
        PG_PH(8);
        if (acts) {
            dump_tile(G.z1T, kH, nv, acts + B * (kI + 2 * kH) + p0 * kH, tid);
            dump_tile_T(G.z1T, kH, nv, acts + B * (kI + 4 * kH + od) + p0, B, tid);
        }
        // ---- dW0 += y^T delta1, db0 += sum delta1 (summed by the ig == 0 threads) ----
        {
            const int jg = tid & 15, ig = tid >> 4;
            float bs[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            for (int q = 0; q < kT; q += 4) {
                float4 a[2], dd[4];
#pragma unroll
                for (int u = 0; u < 2; ++u) a[u] = *reinterpret_cast<const float4 *>(G.yT + sw(ig * 2 + u, q));
#pragma unroll
                for (int v = 0; v < 4; ++v) dd[v] = *reinterpret_cast<const float4 *>(G.z1T + sw(jg * 4 + v, q));
                if (ig == 0) {
#pragma unroll
                    for (int v = 0; v < 4; ++v) bs[v] += (dd[v].x + dd[v].y) + (dd[v].z + dd[v].w);
                }
#pragma unroll
                for (int u = 0; u < 2; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        float s = gW0[u][v];
                        s = __fmaf_rn(a[u].x, dd[v].x, s);
                        s = __fmaf_rn(a[u].y, dd[v].y, s);
                        s = __fmaf_rn(a[u].z, dd[v].z, s);
                        s = __fmaf_rn(a[u].w, dd[v].w, s);
                        gW0[u][v] = s;
                    }
            }
            if (ig == 0) {
#pragma unroll
                for (int v = 0; v < 4; ++v) gB0[v] += bs[v];
            }
        }
        gsync();
        PG_PH(9);
        // ---- dy = delta1 @ W0^T (fma chain over j), over yT ----
        {
            const int og = tid & 7, pg = tid >> 3;  // 4 inputs x 2 samples
            float acc[2][4] = {};
#pragma unroll 8
            for (int j = 0; j < kH; ++j) {
                const float2 a = *reinterpret_cast<const float2 *>(G.z1T + sw(j, pg * 2));
                const float4 w = *reinterpret_cast<const float4 *>(W.w0t + j * kI + og * 4);
                acc[0][0] = __fmaf_rn(a.x, w.x, acc[0][0]);
                acc[0][1] = __fmaf_rn(a.x, w.y, acc[0][1]);
                acc[0][2] = __fmaf_rn(a.x, w.z, acc[0][2]);
                acc[0][3] = __fmaf_rn(a.x, w.w, acc[0][3]);
                acc[1][0] = __fmaf_rn(a.y, w.x, acc[1][0]);
                acc[1][1] = __fmaf_rn(a.y, w.y, acc[1][1]);
                acc[1][2] = __fmaf_rn(a.y, w.z, acc[1][2]);
                acc[1][3] = __fmaf_rn(a.y, w.w, acc[1][3]);
            }
            gsync();  // all reads of yT (dW0) finished before overwrite
#pragma unroll
            for (int ii = 0; ii < 4; ++ii)
                *reinterpret_cast<float2 *>(G.yT + sw(og * 4 + ii, pg * 2)) = make_float2(acc[0][ii], acc[1][ii]);
        }
        gsync();
        if (NG > 1) bar_arrive(gid == 0 ? 4 : 3);   // MLP done: the other pipeline may start its own
        PG_PH(10);
        if (dy_out) {  // optional copy of dL/dy (parity tests)
            for (int i = tid; i < nv * kI; i += kNT) {
                const int q = i / kI, c = i % kI;
                dy_out[(p0 + q) * kI + c] = G.yT[sw(c, q)];
            }
        }
        // ---- encode backward: scatter dy ----
        if (pl < nv) {
#pragma unroll 1
            for (int it = 0; it < 4; ++it) {
                const int l = lsub + 4 * it;
                encode_level_bwd2<D, NPM, ACC>(g, l, x, G.yT[sw(2 * l, pl)], G.yT[sw(2 * l + 1, pl)], feats,
                                         conf, gfeat, gconf, touched);
            }
        }
    }
    if (NG > 1 && gid == 1 && n_iter > 0) bar_sync(4);   // consume pipeline 0's last MLP-done
    PG_PH_FLUSH
    // ---- flush gradient accumulators ----
    ACC *gW0p = gparams, *gb0p = gW0p + kI * kH, *gW1p = gb0p + kH, *gb1p = gW1p + kH * kH;
    ACC *gW2p = gb1p + kH, *gb2p = gW2p + kH * od;
    if (!acts) {  // (parity mode: pg_mlp_wgrad_blas_f32 forms them from acts)
        const int jg = tid & 15, ig = tid >> 4;
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) red_add(gW0p + (ig * 2 + u) * kH + jg * 4 + v, gW0[u][v]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) red_add(gW1p + (ig * 4 + u) * kH + jg * 4 + v, gW1[u][v]);
        const int k = tid & 63, j = tid >> 6;
        if (j < od) red_add(gW2p + k * od + j, gW2);
        if (tid < 16) {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                red_add(gb0p + tid * 4 + v, gB0[v]);
                red_add(gb1p + tid * 4 + v, gB1[v]);
            }
        }
        if (k == 0 && j < od) red_add(gb2p + j, gB2);
    }
    // loss: block reduce in fp64
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    if ((tid & 31) == 0) G.red[tid >> 5] = lsum;
    gsync();
    if (tid < 32) {
        double v = tid < kNT / 32 ? G.red[tid] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (tid == 0 && loss_sum) loss_add(loss_sum, v);
    }
}

bool train_fast_ok(const pg_grid *g, const pg_mlp *m) {
    return g->feature_dim == 2 && g->n_levels == 16 && g->log2_np <= 4 && m->n_layers == 3 &&
           m->widths[0] == kI && m->widths[1] == kH && m->widths[2] == kH && m->widths[3] >= 1 &&
           m->widths[3] <= kO;
}

template <typename ACC, typename LACC>
int train_mma(const pg_grid *g, int od, const float *xs, const float *targets, int64_t B, const float *feats,
              const uint8_t *baked, const float *conf, const float *params, float scale, int sig, ACC *gfeat,
              ACC *gconf, uint8_t *touched, ACC *gparams, LACC *loss_sum, float *dy_out, cudaStream_t s,
              const pg_cells *cells = nullptr);

// gfeat += sum of the `reps` replica tables (each n floats), replicas zeroed
__global__ void reduce_replicas_kernel(float *__restrict__ rep, int reps, int64_t n, float *__restrict__ gfeat) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float s = 0.0f;
        for (int r = 0; r < reps; ++r) {
            s += rep[r * n + i];
            rep[r * n + i] = 0.0f;
        }
        if (s != 0.0f) gfeat[i] += s;
    }
}

template <typename ACC, typename LACC>
int train_fused(const pg_grid *g, const pg_mlp *m, const float *xs, const float *targets, int64_t B,
                const float *feats, const uint8_t *baked, const float *conf, const float *params,
                float scale, unsigned flags, ACC *gfeat, ACC *gconf, uint8_t *touched,
                ACC *gparams, LACC *loss_sum, float *dy_out, float *acts, cudaStream_t s,
                float *gfeat_rep = nullptr, int reps = 1, const pg_cells *cells = nullptr) {
    if (int e = validate_grid(g)) return e;
    PG_REQUIRE(train_fast_ok(g, m), "fused training needs F=2, 16 levels, N_p<=16, MLP [32,64,64,<=4]");
    if (B == 0) return PG_OK;
    const int od = m->widths[3];
    const int sig = (flags & PG_SIGMOID) ? 1 : 0;
    int touch_all = (flags & PG_TOUCH_ALL) ? 4 : 0;
    // replicated feature-gradient tables (fast fp32 path): the kernel adds
    // into gfeat_rep copy (CTA % reps), one pass then folds them into gfeat
    const bool rep = std::is_same<ACC, float>::value && gfeat_rep && reps > 1 && !acts && !(flags & PG_EXACT_MLP);
    PG_REQUIRE(reps >= 1 && reps <= 256, "reps must be in [1, 256]");
    ACC *gf = gfeat;
    if (rep) {
        touch_all |= (reps - 1) << 8;
        gf = reinterpret_cast<ACC *>(gfeat_rep);
    }
    auto fold = [&](int rc) {
        if (rc || !rep) return rc;
        const int64_t n = (int64_t)g->n_levels * g->n_f * 2;
        reduce_replicas_kernel<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(gfeat_rep, reps, n,
                                                                        reinterpret_cast<float *>(gfeat));
        return check_launch("reduce_replicas");
    };
    if (flags & PG_COMPOSITE) {
        // one 64-sample tile = one ray of 64 samples (pg_train_mma.cu)
        PG_REQUIRE(od == 4 && !sig && !(flags & PG_EXACT_MLP) && !acts && B % 64 == 0,
                   "PG_COMPOSITE: out_dim 4, no sigmoid, tensor-core MLP, B a multiple of 64 samples");
        return fold(train_mma<ACC, LACC>(g, od, xs, targets, B, feats, baked, conf, params, scale, 2 | touch_all, gf, gconf,
                                    touched, gparams, loss_sum, dy_out, s, cells));
    }
    // fast path: tensor-core MLP (pg_train_mma.cu); this file's FFMA kernel is
    // the OpenBLAS-order path (PG_EXACT_MLP, reference-order mode)
    if (!acts && !(flags & PG_EXACT_MLP))
        return fold(train_mma<ACC, LACC>(g, od, xs, targets, B, feats, baked, conf, params, scale, sig | touch_all, gf, gconf,
                                    touched, gparams, loss_sum, dy_out, s, cells));
    static DeviceOnce configured[8];
    const int sms = device_sms();
    // tile pipelines per CTA (1 or 2)
    static const int groups = getenv("PG_TRAIN_GROUPS") && atoi(getenv("PG_TRAIN_GROUPS")) == 1 ? 1 : 2;
    const int64_t ntiles = (B + kT - 1) / kT;
    const bool np4 = g->log2_np <= 2;
#define PG_TRAIN_LAUNCH1(D_, NP_, NG_, IDX)                                                           \
    do {                                                                                              \
        auto kern = train_fused_kernel<float, D_, NP_, ACC, LACC, NG_>;                               \
        const int smem = (int)sizeof(TrainSmemT<NG_>);                                                \
        if (configured[IDX].first())                                                                  \
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);            \
        const int64_t want = (ntiles + NG_ - 1) / NG_, cap = (int64_t)sms * (2 / NG_);                \
        const int grd = (int)(want < cap ? want : cap);                                               \
        kern<<<grd, kNT * NG_, smem, s>>>(*g, xs, targets, B, feats, feats, baked, conf, params, od,   \
                                          scale, sig, gfeat, gconf, touched, gparams, loss_sum, dy_out, acts); \
    } while (0)
#define PG_TRAIN_LAUNCH(D_, NP_, IDX)                                                                 \
    do {                                                                                              \
        if (groups == 2) PG_TRAIN_LAUNCH1(D_, NP_, 2, (IDX) + 4); else PG_TRAIN_LAUNCH1(D_, NP_, 1, IDX); \
    } while (0)
    if (g->d == 2) {
        if (np4) PG_TRAIN_LAUNCH(2, 4, 0); else PG_TRAIN_LAUNCH(2, 16, 1);
    } else {
        if (np4) PG_TRAIN_LAUNCH(3, 4, 2); else PG_TRAIN_LAUNCH(3, 16, 3);
    }
#undef PG_TRAIN_LAUNCH1
#undef PG_TRAIN_LAUNCH
    return check_launch("train_fused");
}

}  // namespace pg

PG_PH_READER(pg_phase_prof_read)

extern "C" int pg_train_fused_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs,
                                  const float *targets, int64_t B, const float *feats,
                                  const uint8_t *baked, const float *conf, const float *params,
                                  float scale, unsigned flags, float *gfeat, float *gconf,
                                  uint8_t *touched, float *gparams, double *loss_sum, float *dy_out,
                                  void *stream) {
    return pg::train_fused<float, double>(grid, mlp, xs, targets, B, feats, baked, conf, params, scale,
                                          flags, gfeat, gconf, touched, gparams, loss_sum, dy_out,
                                          nullptr, pg::as_stream(stream));
}

extern "C" int pg_train_fused_rep_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs,
                                      const float *targets, int64_t B, const float *feats,
                                      const uint8_t *baked, const float *conf, const float *params,
                                      float scale, unsigned flags, float *gfeat, float *gconf,
                                      uint8_t *touched, float *gparams, double *loss_sum, float *dy_out,
                                      float *gfeat_rep, int reps, void *stream) {
    return pg::train_fused<float, double>(grid, mlp, xs, targets, B, feats, baked, conf, params, scale,
                                          flags, gfeat, gconf, touched, gparams, loss_sum, dy_out,
                                          nullptr, pg::as_stream(stream), gfeat_rep, reps);
}
extern "C" int pg_train_fused_ex_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs,
                                     const float *targets, int64_t B, const float *feats,
                                     const uint8_t *baked, const float *conf, const float *params,
                                     float scale, unsigned flags, float *gfeat, float *gconf,
                                     uint8_t *touched, float *gparams, double *loss_sum, float *dy_out,
                                     float *gfeat_rep, int reps, const pg_cells *cells, void *stream) {
    return pg::train_fused<float, double>(grid, mlp, xs, targets, B, feats, baked, conf, params, scale,
                                          flags, gfeat, gconf, touched, gparams, loss_sum, dy_out,
                                          nullptr, pg::as_stream(stream), gfeat_rep, reps, cells);
}

extern "C" int pg_train_fused_ref_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs,
                                      const float *targets, int64_t B, const float *feats,
                                      const uint8_t *baked, const float *conf, const float *params,
                                      float scale, unsigned flags, float *gfeat, float *gconf,
                                      uint8_t *touched, double *loss_sum, float *acts, void *stream) {
    PG_REQUIRE(acts != nullptr, "pg_train_fused_ref_f32: acts is required");
    return pg::train_fused<float, double>(grid, mlp, xs, targets, B, feats, baked, conf, params, scale,
                                          flags, gfeat, gconf, touched, nullptr, loss_sum, nullptr, acts,
                                          pg::as_stream(stream));
}

extern "C" int pg_train_fused_ref_det_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs,
                                          const float *targets, int64_t B, const float *feats,
                                          const uint8_t *baked, const float *conf, const float *params,
                                          float scale, unsigned flags, uint64_t *gfeat_fx,
                                          uint64_t *gconf_fx, uint8_t *touched, uint64_t *loss_fx,
                                          float *acts, void *stream) {
    using pg::fx_t;
    PG_REQUIRE(acts != nullptr, "pg_train_fused_ref_det_f32: acts is required");
    return pg::train_fused<fx_t, fx_t>(grid, mlp, xs, targets, B, feats, baked, conf, params, scale, flags,
                                       (fx_t *)gfeat_fx, (fx_t *)gconf_fx, touched, nullptr, (fx_t *)loss_fx,
                                       nullptr, acts, pg::as_stream(stream));
}

extern "C" int pg_train_fused_det_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs,
                                      const float *targets, int64_t B, const float *feats,
                                      const uint8_t *baked, const float *conf, const float *params,
                                      float scale, unsigned flags, uint64_t *gfeat_fx,
                                      uint64_t *gconf_fx, uint8_t *touched, uint64_t *gparams_fx,
                                      uint64_t *loss_fx, float *dy_out, void *stream) {
    using pg::fx_t;
    return pg::train_fused<fx_t, fx_t>(grid, mlp, xs, targets, B, feats, baked, conf, params, scale,
                                       flags, (fx_t *)gfeat_fx, (fx_t *)gconf_fx, touched,
                                       (fx_t *)gparams_fx, (fx_t *)loss_fx, dy_out, nullptr,
                                       pg::as_stream(stream));
}
