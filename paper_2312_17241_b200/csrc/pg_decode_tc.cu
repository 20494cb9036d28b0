// Fused decode on the 5th-generation tensor core (tcgen05 / UMMA), the
// headline kernel.  Per 128-query tile: 16-level encode (fp16 tables) ->
// layers 1 and 2 of the MLP as kind::tf32 UMMA (M = 128, N = 64, fp32
// accumulators in TMEM) -> bias/ReLU epilogues from TMEM (tcgen05.ld) ->
// output layer (64 -> <= 4) in registers.
//
// Accuracy: activations go in as a 2-term tf32 expansion (hi + lo, ~22
// significand bits); the weights of an inference model are fp16-rounded
// (to_inference, model_io.py:130-147), hence exact in tf32, so each layer is
// 2 UMMA passes and matches fp32 to ~1e-6 relative (tests bound it at 1e-5).
//
// Throughput: the encode is ~100 random 4-byte L2 gathers per query (64
// feature rows + 36 baked bytes at C2), and random gathers retire at ~1 per
// SM per clock on B200 (pg_probe_gather: 2.8e11/s, independent of table size
// and of loads in flight) — that, not HBM or the MMA, is this kernel's
// ceiling.  The layout therefore maximises warps per SM and L1 capacity:
// * a tile pipeline ("group") is 256 threads with a 32 KB operand buffer
//   (one 128 x 32 K-block, hi | lo) and 128 TMEM columns; layer 2's 64-wide
//   A operand is fed as two K = 32 blocks through that buffer, and the
//   output-layer partial sums reuse it too -> ~60 KB of shared memory;
// * default: one group per CTA, three CTAs per SM (24 warps, <= 80 regs);
// * PG_SMEM_TABLES: three groups in ONE CTA (named barriers 1..3) sharing
//   weights and a few KB of the probed levels' baked indices bit-packed to
//   log2(N_p) bits, which removes those levels' dependent baked-byte L2
//   round trip.  Dense-level feature tables can be placed too (ablation
//   knob); they are not, because every KB of shared memory comes out of the
//   L1 that caches the coarse levels' rows.
#include <type_traits>

#include "pg_encode_dev.cuh"
#include "pg_umma.cuh"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace pg {

namespace tc {
constexpr int kTP = 128;  // queries per tile == UMMA M
constexpr int kIn = 32;
constexpr int kHid = 64;
constexpr int kOutMax = 4;
constexpr int kGT = 256;  // threads per group

struct Group {
    // one 128 x 32 K-block, hi | lo; after layer 2 it holds the output-layer
    // partial sums part[2][kTP][kOutMax]
    alignas(128) float opA[2 * kTP * 32];
    float xs[kTP * 3];
    uint64_t mbar[3];
    int seen;            // streaming: chunk of the group's current tile
    uint32_t pending;    // streaming: finished tiles of chunk `seen` not yet counted
    int host;            // streaming: a flag timed out -> read inputs from host memory
};
template <int NG>
struct Smem {
    alignas(128) float b1[kHid * kIn];   // W0^T, K-major
    alignas(128) float b2[kHid * kHid];  // W1^T, K-major
    float w2[kHid * kOutMax];
    float bias0[kHid], bias1[kHid], bias2[kOutMax];
    Group grp[NG];
    uint32_t tmem_base;
};
template <int NG>
__host__ __device__ constexpr int tab_offset() { return (int)((sizeof(Smem<NG>) + 127) / 128 * 128); }

// which levels live in shared memory (byte offsets into the table region)
struct TabPlan {
    int32_t off[PG_MAX_LEVELS];  // -1: global memory
    int32_t pbits;               // packed bits per baked index; 0 when N_p == 1
    int32_t bytes;
    const uint4 *cells;          // decode cell cache (pg_cells), or null
    int32_t cell[PG_MAX_LEVELS]; // level's record offset in uint4 units, -1: not cached
    int32_t l2_hints;            // evict_last tables/cells, evict_first inputs/outputs
};
using Stream = DecodeStream;
using pg::wait_flag;
using pg::signal_done;
}  // namespace tc

template <typename FT> struct FeatS;
template <> struct FeatS<__half> {
    static __device__ __forceinline__ float2 ld2(const unsigned char *p) {
        return __half22float2(*reinterpret_cast<const __half2 *>(p));
    }
};
template <> struct FeatS<float> {
    static __device__ __forceinline__ float2 ld2(const unsigned char *p) {
        return *reinterpret_cast<const float2 *>(p);
    }
};

template <typename FT> struct RangeLoad {
    static constexpr bool ok = false;
    static __device__ __forceinline__ float2 widen(uint32_t) { return make_float2(0.f, 0.f); }
};
template <> struct RangeLoad<__half> {
    static constexpr bool ok = true;
    static __device__ __forceinline__ float2 widen(uint32_t w) {
        return __half22float2(*reinterpret_cast<const __half2 *>(&w));
    }
};

// encode_level_fwd2 (pg_encode_dev.cuh) with optional on-chip tables and
// the decode cell cache: identical indices, weights and blend order, so the
// result is bit-identical.
template <typename FT, int D>
__device__ __forceinline__ float2 encode_level_fwd2_tab(const pg_grid &g, int l, const float (&x)[D],
                                                        const FT *__restrict__ feats,
                                                        const uint8_t *__restrict__ baked,
                                                        const unsigned char *tabs, int off, int pbits,
                                                        const uint4 *__restrict__ cellrec = nullptr,
                                                        uint64_t pol = 0) {
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
    if (RangeLoad<FT>::ok && cellrec != nullptr) return encode_level_fwd2_cell<D>(g, l, x, cellrec, pol);
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
                idx[k] = (int)((h << g.log2_np) & nf_mask);
                if (pbits != 0) {
                    const uint32_t r = corner_hash<D>(k, c, g.aux) & nc_mask;
                    if (off >= 0) {
                        const int lg = 5 - __ffs(pbits) + 1;  // log2(32 / pbits)
                        const uint32_t word = reinterpret_cast<const uint32_t *>(tabs + off)[r >> lg];
                        idx[k] += (int)((word >> ((r & ((1u << lg) - 1u)) * pbits)) & ((1u << pbits) - 1u));
                    } else if (!(RangeLoad<FT>::ok && g.log2_np == 2)) {
                        idx[k] += (int)__ldg(baked + (int64_t)g.slot[l] * g.n_c + r);
                    }
                }
            }
        }
    }
    float2 f[C];
    if (kind == PG_LEVEL_DENSE && off >= 0) {
#pragma unroll
        for (int k = 0; k < C; ++k) f[k] = FeatS<FT>::ld2(tabs + off + idx[k] * (int)(2 * sizeof(FT)));
    } else if (RangeLoad<FT>::ok && kind == PG_LEVEL_PROBED && off < 0 && g.log2_np == 2) {
        // baked offsets in global memory (N_p = 4): fetch the whole probing
        // range (4 binary16 rows = 16 B, one sector) together with the baked
        // byte instead of after it and select the probe in registers — one L2
        // round trip instead of two.  (A generic N_p = 2/4/8 version of this
        // measured slower: register pressure at the 80-register budget.)
        const FT *tab = feats + (int64_t)l * g.n_f * 2;
        const uint8_t *bt = baked + (int64_t)g.slot[l] * g.n_c;
        uint4 rng[C];
        int bk[C];
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const uint32_t base = (corner_hash<D>(k, c, g.primary) << 2) & nf_mask;
            rng[k] = __ldg(reinterpret_cast<const uint4 *>(tab + (int64_t)base * 2));
            bk[k] = (int)__ldg(bt + (corner_hash<D>(k, c, g.aux) & nc_mask));
        }
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const uint32_t w = bk[k] == 0 ? rng[k].x : bk[k] == 1 ? rng[k].y : bk[k] == 2 ? rng[k].z : rng[k].w;
            f[k] = RangeLoad<FT>::widen(w);
        }
    } else {
        const FT *tab = feats + (int64_t)l * g.n_f * 2;
#pragma unroll
        for (int k = 0; k < C; ++k) f[k] = Feat<FT>::ld2(tab + (int64_t)idx[k] * 2);
    }
    float y0 = 0.0f, y1 = 0.0f;
#pragma unroll
    for (int k = 0; k < C; ++k) {
        y0 = __fadd_rn(y0, __fmul_rn(w[k], f[k].x));
        y1 = __fadd_rn(y1, __fmul_rn(w[k], f[k].y));
    }
    return make_float2(y0, y1);
}

__device__ __forceinline__ void group_sync(int grp) {
    asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "r"(tc::kGT) : "memory");
}

// MODE 0: ordinary launch (inputs/outputs in device memory, or in pinned
// host memory for the zero-copy entry point); 1: streaming (inputs landed by
// the copy engine behind per-chunk flags, outputs counted per chunk for the
// D2H stream)
template <typename FT, int D, int NG, int MINB, int MODE>
__global__ void __launch_bounds__(tc::kGT *NG, MINB)
    decode_umma_kernel(const pg_grid g, const tc::TabPlan plan, const float *__restrict__ xs, int64_t B,
                        const FT *__restrict__ feats, const uint8_t *__restrict__ baked,
                        const float *__restrict__ params, int od, int sigmoid, float *__restrict__ out,
                        tc::Stream st) {
    using namespace tc;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    constexpr int kThreads = kGT * NG, kGroups = NG;
    Smem<NG> &S = *reinterpret_cast<Smem<NG> *>(smem_raw);
    unsigned char *tabs = smem_raw + tab_offset<NG>();
    const int tid = threadIdx.x, lane = tid & 31;
    const uint64_t pol_last = plan.l2_hints ? l2_policy_evict_last() : 0;
    const uint64_t pol_first = plan.l2_hints && MODE == 0 ? l2_policy_evict_first() : 0;

    // ---- weights: B operands (K-major W^T) + epilogue constants ----
    {
        const float *p = params;
        char *b1 = reinterpret_cast<char *>(S.b1);
        char *b2 = reinterpret_cast<char *>(S.b2);
        for (int i = tid; i < kIn * kHid; i += kThreads) {  // W0[k][n]
            const int k = i / kHid, n = i % kHid;
            *reinterpret_cast<float *>(b1 + umma::kmaj_off(n, k, kHid)) = p[i];
        }
        p += kIn * kHid;
        for (int i = tid; i < kHid; i += kThreads) S.bias0[i] = p[i];
        p += kHid;
        for (int i = tid; i < kHid * kHid; i += kThreads) {  // W1[k][n]
            const int k = i / kHid, n = i % kHid;
            *reinterpret_cast<float *>(b2 + umma::kmaj_off(n, k, kHid)) = p[i];
        }
        p += kHid * kHid;
        for (int i = tid; i < kHid; i += kThreads) S.bias1[i] = p[i];
        p += kHid;
        for (int i = tid; i < kHid * kOutMax; i += kThreads) {
            const int k = i / kOutMax, j = i % kOutMax;
            S.w2[i] = j < od ? p[k * od + j] : 0.0f;
        }
        p += kHid * od;
        for (int i = tid; i < kOutMax; i += kThreads) S.bias2[i] = i < od ? p[i] : 0.0f;
    }
    // ---- on-chip tables ----
    for (int l = 0; l < g.n_levels; ++l) {
        const int o = plan.off[l];
        if (o < 0) continue;
        uint32_t *dst = reinterpret_cast<uint32_t *>(tabs + o);
        if (g.kind[l] == PG_LEVEL_DENSE) {
            int n = g.res[l] + 1, e = n;
            for (int a = 1; a < D; ++a) e *= n;
            const int words = e * (int)(2 * sizeof(FT)) / 4;
            const uint32_t *src = reinterpret_cast<const uint32_t *>(feats + (int64_t)l * g.n_f * 2);
            for (int i = tid; i < words; i += kThreads) dst[i] = __ldg(src + i);
        } else {  // probed: pack baked indices, R = 32 / pbits per word
            const int pb = plan.pbits, R = 32 / pb;
            const int words = g.n_c / R;
            const uint2 *src = reinterpret_cast<const uint2 *>(baked + (int64_t)g.slot[l] * g.n_c);
            for (int wi = tid; wi < words; wi += kThreads) {
                uint32_t word = 0;
                for (int c8 = 0; c8 < R / 8; ++c8) {
                    const uint2 v = __ldg(src + (int64_t)wi * (R / 8) + c8);
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const uint32_t byte = ((b < 4 ? v.x : v.y) >> ((b & 3) * 8)) & 0xFFu;
                        word |= byte << ((c8 * 8 + b) * pb);
                    }
                }
                dst[wi] = word;
            }
        }
    }
    constexpr bool STREAM = MODE == 1;
    if (STREAM && tid < kGroups) {
        S.grp[tid].seen = -1;
        S.grp[tid].pending = 0;
        S.grp[tid].host = 0;
    }
    if ((tid >> 5) == 0) umma::tmem_alloc<(NG == 1 ? 128 : NG == 2 ? 256 : 512)>(&S.tmem_base);
    if (tid == 0) {
        for (int gi = 0; gi < kGroups; ++gi)
            for (int m = 0; m < 3; ++m) umma::mbar_init(&S.grp[gi].mbar[m], 1);
        umma::mbar_init_fence();
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();

    const int grp = tid >> 8, gt = tid & (kGT - 1), gw = gt >> 5;
    // i / od in the output store by a 16-bit reciprocal: exact for i < nv * od <= 512
    const uint32_t od_mag = (65536u + (uint32_t)od - 1u) / (uint32_t)od;
    Group &G = S.grp[grp];
    const uint32_t tm_d1 = S.tmem_base + (uint32_t)(grp * 128), tm_d2 = tm_d1 + kHid;
    const uint32_t idesc = umma::idesc_tf32(kTP, kHid);
    char *opA = reinterpret_cast<char *>(G.opA);
    const uint32_t a_s = umma::smem_u32(opA);
    const uint32_t b1_s = umma::smem_u32(S.b1), b2_s = umma::smem_u32(S.b2);
    constexpr int kLoOff = kTP * 32 * 4;  // lo half of the operand buffer
    // epilogue role: row (TMEM lane; a warp may only touch lanes 32*(warp%4)..) and column half
    const int erow = (gw & 3) * 32 + lane;
    const int ehalf = gw >> 2;
    const uint32_t lane_off = (uint32_t)((gw & 3) * 32) << 16;

    const int64_t ntiles = (B + kTP - 1) / kTP;
    uint32_t phase = 0;
    // Token ring over the pipelines' MLP phases (named barriers 4..4+NG-1):
    // pipeline g starts its tensor-core MLP only after pipeline g-1 finished
    // its own (bar.arrive at an MLP's end, bar.sync before the next), so the
    // MLP phases of a CTA's pipelines never overlap and the L1 gather pipe
    // always has the other pipelines' encodes: 3.71e9 vs 3.43e9 q/s free-
    // running (C2).  All pipelines run as many iterations as pipeline 0.
    constexpr bool RING = NG > 1;
    const int64_t stride_t = (int64_t)gridDim.x * kGroups, first_t = (int64_t)blockIdx.x * kGroups + grp;
    const int64_t base0 = (int64_t)blockIdx.x * kGroups;
    const int64_t n_iter = base0 < ntiles ? (ntiles - base0 + stride_t - 1) / stride_t : 0;
    for (int64_t iter = 0; iter < n_iter; ++iter) {
        const int64_t tile = first_t + iter * stride_t;
        if (tile >= ntiles) {
            if (RING) {
                if (grp > 0 || iter > 0) asm volatile("bar.sync %0, %1;" ::"r"(4 + grp), "r"(2 * kGT) : "memory");
                asm volatile("bar.arrive %0, %1;" ::"r"(4 + (grp + 1) % NG), "r"(2 * kGT) : "memory");
            }
            continue;
        }
        phase = (uint32_t)(iter & 1);
        const int64_t p0 = tile * kTP;
        const int nv = (int)((B - p0) < kTP ? (B - p0) : kTP);
        if (STREAM && (int)(tile >> st.chunk_tiles_log2) != G.seen) {
            // streaming, entering a new chunk: publish the finished tiles of
            // the previous one (fence each thread's output stores, then one
            // counter add per group and chunk), then wait for this chunk's
            // inputs to land.  The bookkeeping lives in shared memory: the
            // 3-pipeline variant is at its register cap.
            __threadfence();
            group_sync(grp);
            if (gt == 0) {
                if (G.pending) tc::signal_done(st.done + G.seen, G.pending);
                G.pending = 0;
                G.seen = (int)(tile >> st.chunk_tiles_log2);
                // a flag that does not come (the copies serialised behind
                // this kernel: profilers, CUDA_LAUNCH_BLOCKING) is not an
                // error: the group then reads its inputs from pinned host
                // memory directly (they are there already)
                if (!G.host && !tc::wait_flag(st.ready + G.seen, st.timeout_ns)) {
                    G.host = 1;
                    atomicAdd(st.fallbacks, 1u);
                }
            }
            group_sync(grp);
        }
        // streaming: L2-coherent loads (the copy engine writes xs while the
        // kernel runs, so the non-coherent path must not be used)
        {
            // streaming: L2-coherent loads from the landed chunk, or straight
            // from pinned host memory for a group whose flag never came
            const float *src = STREAM && G.host ? st.host_xs : xs;
            for (int i = gt; i < kTP * D; i += kGT)
                G.xs[i] = i < nv * D ? (STREAM ? __ldcg(src + p0 * D + i)
                                               : pol_first ? ld_nc_hint(xs + p0 * D + i, pol_first) : xs[p0 * D + i])
                                     : 0.5f;
        }
        group_sync(grp);
        // ---------------- encode -> layer-1 A operand (hi | lo) ----------------
        {
            const int q = gt & (kTP - 1), lsub = gt >> 7;
            float x[D];
#pragma unroll
            for (int a = 0; a < D; ++a) x[a] = G.xs[q * D + a];
#pragma unroll 2
            for (int it = 0; it < 4; ++it) {
                const int P = lsub + 2 * it;  // warp-uniform level pair (2P, 2P+1)
                const int ca = plan.cell[2 * P], cb = plan.cell[2 * P + 1];
                const float2 ya = encode_level_fwd2_tab<FT, D>(g, 2 * P, x, feats, baked, tabs,
                                                               plan.off[2 * P], plan.pbits,
                                                               ca >= 0 ? plan.cells + ca : nullptr, pol_last);
                const float2 yb = encode_level_fwd2_tab<FT, D>(g, 2 * P + 1, x, feats, baked, tabs,
                                                               plan.off[2 * P + 1], plan.pbits,
                                                               cb >= 0 ? plan.cells + cb : nullptr, pol_last);
                float h[4], lo[4];
                umma::split_tf32(ya.x, h[0], lo[0]);
                umma::split_tf32(ya.y, h[1], lo[1]);
                umma::split_tf32(yb.x, h[2], lo[2]);
                umma::split_tf32(yb.y, h[3], lo[3]);
                const uint32_t off = umma::kmaj_off(q, 4 * P, kTP);
                *reinterpret_cast<float4 *>(opA + off) = make_float4(h[0], h[1], h[2], h[3]);
                *reinterpret_cast<float4 *>(opA + kLoOff + off) = make_float4(lo[0], lo[1], lo[2], lo[3]);
            }
        }
        umma::fence_async_smem();
        umma::fence_before_sync();
        group_sync(grp);
        if (RING && (grp > 0 || iter > 0)) asm volatile("bar.sync %0, %1;" ::"r"(4 + grp), "r"(2 * kGT) : "memory");
        // ---------------- layer 1: D1 = (Y_hi + Y_lo) . W0 ----------------
        if (gt == 0) {
            umma::fence_after_sync();
#pragma unroll
            for (int pass = 0; pass < 2; ++pass)
#pragma unroll
                for (int kb = 0; kb < kIn / 8; ++kb) {
                    const uint64_t ad = umma::smem_desc(a_s + pass * kLoOff + kb * kTP * 32, 128, 256);
                    const uint64_t bd = umma::smem_desc(b1_s + kb * kHid * 32, 128, 256);
                    umma::mma_tf32(tm_d1, ad, bd, idesc, (pass | kb) ? 1u : 0u);
                }
            umma::commit(&G.mbar[0]);
        }
        umma::mbar_wait(&G.mbar[0], phase);
        umma::fence_after_sync();
        // ------- epilogue 1: bias + ReLU -> layer-2 A operand, two K = 32 blocks -------
        // With NG > 1 (80-register budget) each column half reads its
        // accumulators right before its block is written, so no registers
        // are held across the first block's MMAs; NG = 1 reads both up front.
        float v[32];
        auto load_h1 = [&]() {
            umma::tmem_ld32(tm_d1 + lane_off + ehalf * 32, v);
#pragma unroll
            for (int c = 0; c < 32; c += 4) {
                const float4 b4 = *reinterpret_cast<const float4 *>(S.bias0 + ehalf * 32 + c);
                v[c] = umma::relu_nan(v[c] + b4.x);   // one FMNMX (1.5% of the decode vs a select)
                v[c + 1] = umma::relu_nan(v[c + 1] + b4.y);
                v[c + 2] = umma::relu_nan(v[c + 2] + b4.z);
                v[c + 3] = umma::relu_nan(v[c + 3] + b4.w);
            }
        };
        if (NG == 1) load_h1();
#pragma unroll
        for (int blk = 0; blk < 2; ++blk) {
            if (ehalf == blk) {
                if (NG > 1) load_h1();
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    float hi[4], lo[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) umma::split_tf32(v[c + u], hi[u], lo[u]);
                    const uint32_t off = umma::kmaj_off(erow, c, kTP);
                    *reinterpret_cast<float4 *>(opA + off) = make_float4(hi[0], hi[1], hi[2], hi[3]);
                    *reinterpret_cast<float4 *>(opA + kLoOff + off) = make_float4(lo[0], lo[1], lo[2], lo[3]);
                }
            }
            umma::fence_async_smem();
            umma::fence_before_sync();
            group_sync(grp);
            if (gt == 0) {
                umma::fence_after_sync();
#pragma unroll
                for (int pass = 0; pass < 2; ++pass)
#pragma unroll
                    for (int kb = 0; kb < 4; ++kb) {
                        const uint64_t ad = umma::smem_desc(a_s + pass * kLoOff + kb * kTP * 32, 128, 256);
                        const uint64_t bd = umma::smem_desc(b2_s + (blk * 4 + kb) * kHid * 32, 128, 256);
                        umma::mma_tf32(tm_d2, ad, bd, idesc, (blk | pass | kb) ? 1u : 0u);
                    }
                umma::commit(&G.mbar[1 + blk]);
            }
            umma::mbar_wait(&G.mbar[1 + blk], phase);
            umma::fence_after_sync();
        }
        // ---------------- epilogue 2: bias + ReLU + output layer ----------------
        {
            umma::tmem_ld32(tm_d2 + lane_off + ehalf * 32, v);
            float acc[kOutMax] = {0.0f, 0.0f, 0.0f, 0.0f};
            // biases by float4; the fourth output column only when od > 3
            // (its weights are zero otherwise)
            auto out_layer = [&](auto four) {
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    const float4 b4 = *reinterpret_cast<const float4 *>(S.bias1 + ehalf * 32 + c);
                    const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int k = ehalf * 32 + c + u;
                        const float h = umma::relu_nan(v[c + u] + bb[u]);
                        const float4 w = *reinterpret_cast<const float4 *>(S.w2 + k * kOutMax);
                        acc[0] = fmaf(h, w.x, acc[0]);
                        acc[1] = fmaf(h, w.y, acc[1]);
                        acc[2] = fmaf(h, w.z, acc[2]);
                        if (decltype(four)::value) acc[3] = fmaf(h, w.w, acc[3]);
                    }
                }
            };
            if (od > 3) out_layer(std::true_type{});
            else out_layer(std::false_type{});
            // packed [half][query][od]: the output loop below then reads
            // consecutive words (a [query][4] float4 layout left its reads
            // 2-way bank conflicted)
#pragma unroll
            for (int j = 0; j < kOutMax; ++j)
                if (j < od) G.opA[(ehalf * kTP + erow) * od + j] = acc[j];
        }
        umma::fence_before_sync();
        group_sync(grp);
        if (RING) asm volatile("bar.arrive %0, %1;" ::"r"(4 + (grp + 1) % NG), "r"(2 * kGT) : "memory");
        {
            float *dst = out + p0 * od;
            for (int i = gt; i < nv * od; i += kGT) {
                const int q = (int)(((uint32_t)i * od_mag) >> 16), j = i - q * od;   // 1.1% vs i / od
                float o = S.bias2[j] + G.opA[i] + G.opA[kTP * od + i];
                if (sigmoid) o = (float)(1.0 / (1.0 + exp(-(double)o)));
                if (pol_first) st_hint(dst + i, o, pol_first);
                else dst[i] = o;
            }
        }
        if (STREAM && gt == 0) ++G.pending;
    }
    if (STREAM) {
        __threadfence();
        group_sync(grp);
        if (gt == 0 && G.pending) tc::signal_done(st.done + G.seen, G.pending);
    }
    if (RING && grp == 0 && n_iter > 0) asm volatile("bar.sync %0, %1;" ::"r"(4), "r"(2 * kGT) : "memory");
    umma::fence_after_sync();
    __syncthreads();
    if ((tid >> 5) == 0) umma::tmem_free<(NG == 1 ? 128 : NG == 2 ? 256 : 512)>(S.tmem_base);
}

// Host: choose the on-chip tables (smallest first, they save the same 2^d
// gathers per query each) within the shared-memory budget.
static tc::TabPlan plan_tables(const pg_grid *g, size_t feat_bytes, int budget, int kinds, const pg_cells *cells) {
    tc::TabPlan p;
    p.cells = nullptr;
    static const bool hints = !(getenv("PG_DECODE_L2_HINTS") && atoi(getenv("PG_DECODE_L2_HINTS")) == 0);
    p.l2_hints = hints ? 1 : 0;
    for (int l = 0; l < PG_MAX_LEVELS; ++l) {
        p.off[l] = -1;
        p.cell[l] = -1;
    }
    if (cells && cells->data && feat_bytes == 2) {
        p.cells = reinterpret_cast<const uint4 *>(cells->data);
        for (int l = 0; l < g->n_levels; ++l) p.cell[l] = cells->off[l] >= 0 ? (int32_t)cells->off[l] : -1;
    }
    p.pbits = g->log2_np == 0 ? 0 : g->log2_np == 1 ? 1 : g->log2_np == 2 ? 2 : g->log2_np <= 4 ? 4 : -1;
    p.bytes = 0;
    std::vector<std::pair<int64_t, int>> cand;
    for (int l = 0; l < g->n_levels; ++l) {
        int64_t bytes = -1;
        if (p.cell[l] >= 0) continue;   // served by the cell cache
        if (g->kind[l] == PG_LEVEL_DENSE && (kinds & 1)) {
            int64_t e = 1;
            for (int a = 0; a < g->d; ++a) e *= (int64_t)(g->res[l] + 1);
            bytes = e * 2 * (int64_t)feat_bytes;
        } else if (g->kind[l] == PG_LEVEL_PROBED && (kinds & 2) && p.pbits > 0 && g->n_c % (32 / p.pbits) == 0 &&
                   (32 / p.pbits) % 8 == 0) {
            bytes = (int64_t)g->n_c * p.pbits / 8;
        }
        if (bytes > 0) cand.push_back({(bytes + 15) / 16 * 16, l});
    }
    std::sort(cand.begin(), cand.end());
    for (auto &c : cand) {
        if (p.bytes + c.first > budget) break;
        p.off[c.second] = p.bytes;
        p.bytes += (int)c.first;
    }
    if (p.pbits < 0) p.pbits = 8;  // N_p > 16: never packed, global byte loads
    return p;
}

template <typename FT, int D, int NG, int MINB, int MODE>
static void launch_umma(const pg_grid *g, const tc::TabPlan &plan, int smem, int grd, const float *xs,
                         int64_t B, const void *feats, const uint8_t *baked, const float *params, int od,
                         int sig, float *out, const tc::Stream &st, cudaStream_t s) {
    static DeviceOnce configured;
    if (configured.first())
        cudaFuncSetAttribute(decode_umma_kernel<FT, D, NG, MINB, MODE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, device_optin_smem());
    decode_umma_kernel<FT, D, NG, MINB, MODE><<<grd, tc::kGT * NG, smem, s>>>(*g, plan, xs, B, (const FT *)feats,
                                                                           baked, params, od, sig, out, st);
}

int decode_umma(const pg_grid *g, int od, const float *xs, int64_t B, const void *feats, bool half,
                const uint8_t *baked, const float *params, int sig, int table_flags, float *out, cudaStream_t s,
                const tc::Stream &st, const pg_cells *cells) {
    // tuning knobs for the table variant (ablations in tools/gpu_decode_ab.sh)
    static const int env_budget = getenv("PG_DECODE_TABLE_BYTES") ? atoi(getenv("PG_DECODE_TABLE_BYTES")) : -1;
    static const int env_kinds = getenv("PG_DECODE_TABLE_KINDS") ? atoi(getenv("PG_DECODE_TABLE_KINDS")) : 2;
    const int sms = device_sms(), optin = device_optin_smem();
    // Shared-memory tables: the three pipelines of a CTA share <= 64 KB of
    // bit-packed baked indices, so that smem + L1 stay inside the 196 KB
    // carve-out and L1 keeps ~60 KB.  On for N_p = 2 and 4 (measured with the
    // token ring: 3.99 vs 3.11e9 at N_p = 2, 3.72 vs 3.38e9 at N_p = 4;
    // none or a wash at N_p = 1, 8, 16).
    const bool tables = (table_flags & PG_SMEM_TABLES) ||
                        (!(table_flags & PG_NO_SMEM_TABLES) && g->log2_np >= 1 && g->log2_np <= 2);
    // three token-ring pipelines per CTA (one CTA per SM) with or without
    // tables: measured faster than three independent CTAs per SM for every
    // C2/C5 shape (N_p 1: 4.72 vs 4.44e9, 8: 2.84 vs 2.61e9, 16: 2.84 vs
    // 2.59e9 q/s); PG_DECODE_GROUPS=1 restores the independent CTAs
    static const int env_groups = getenv("PG_DECODE_GROUPS") ? atoi(getenv("PG_DECODE_GROUPS")) : 3;
    const int ng = (tables || env_groups != 1) ? 3 : 1;
    const int fixed = ng == 3 ? tc::tab_offset<3>() : tc::tab_offset<1>();
    int budget = 0;
    if (tables) {
        const int room = optin - fixed - 1024;
        budget = env_budget >= 0 ? env_budget : 65536;
        if (budget > room) budget = room;
    }
    const tc::TabPlan plan = plan_tables(g, half ? 2 : 4, budget, env_kinds, cells);
    const int smem = fixed + plan.bytes;
    const int per_sm = ng == 3 ? 1 : 3;
    const int64_t ntiles = (B + tc::kTP - 1) / tc::kTP;
    const int64_t want = (ntiles + ng - 1) / ng;
    const int64_t cap = (int64_t)sms * per_sm;
    const int grd = (int)(want < cap ? want : cap);
    // streaming (pg_decode_host_stream_f32) is its own instantiation, so the
    // ordinary kernel carries none of its registers; fp16 tables only (the
    // inference model's storage)
    const int mode = st.ready ? 1 : 0;
    PG_REQUIRE(!mode || half, "streaming decode runs on fp16 tables");
#define PG_DEC_TC2(FT_, D_, S_)                                                                       \
    (ng == 3 ? launch_umma<FT_, D_, 3, 1, S_>(g, plan, smem, grd, xs, B, feats, baked, params, od, sig, out, st, s) \
             : launch_umma<FT_, D_, 1, 3, S_>(g, plan, smem, grd, xs, B, feats, baked, params, od, sig, out, st, s))
    if (half) {
        if (mode == 1) {
            if (g->d == 2) PG_DEC_TC2(__half, 2, 1); else PG_DEC_TC2(__half, 3, 1);
        } else {
            if (g->d == 2) PG_DEC_TC2(__half, 2, 0); else PG_DEC_TC2(__half, 3, 0);
        }
    } else {
        if (g->d == 2) PG_DEC_TC2(float, 2, 0); else PG_DEC_TC2(float, 3, 0);
    }
#undef PG_DEC_TC2
    return check_launch("decode_umma");
}

// ---- cell cache (pg_cells): records of the 2^d resolved corner rows per
// cell of the coarsest levels; R = the row type (uint32_t: binary16 F = 2 of
// the inference tables; uint2: fp32 F = 2 of the training tables).  One
// launch builds every cached level (flattened (level, cell) index).
struct CellLevels {
    int n;
    int level[PG_MAX_LEVELS];
    int64_t start[PG_MAX_LEVELS + 1];   // first flattened cell index of each entry
    int64_t rec[PG_MAX_LEVELS];         // record offset of the level, in rows
};
template <int D, typename R>
__global__ void build_cells_kernel(const pg_grid g, const CellLevels cl, const R *__restrict__ feats,
                                   const uint8_t *__restrict__ baked, R *__restrict__ out) {
    constexpr int C = 1 << D;
    const uint32_t nf_mask = (uint32_t)g.n_f - 1u, nc_mask = (uint32_t)g.n_c - 1u;
    const int64_t total = cl.start[cl.n];
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int e = 0;
        while (e + 1 < cl.n && t >= cl.start[e + 1]) ++e;
        const int l = cl.level[e], res = g.res[l], kind = g.kind[l];
        const int64_t i = t - cl.start[e];
        const R *tab = feats + (int64_t)l * g.n_f;
        int c[D];
        int64_t rem = i;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            c[a] = (int)(rem % res);
            rem /= res;
        }
        R *rec = out + cl.rec[e] + i * C;
#pragma unroll
        for (int k = 0; k < C; ++k) {
            int idx;
            if (kind == PG_LEVEL_DENSE) {
                idx = corner_dense<D>(k, c, res + 1);
            } else {
                const uint32_t h = corner_hash<D>(k, c, g.primary);
                if (kind == PG_LEVEL_HASHED) {
                    idx = (int)(h & nf_mask);
                } else {
                    const uint32_t r = corner_hash<D>(k, c, g.aux) & nc_mask;
                    idx = (int)((h << g.log2_np) & nf_mask) + (int)baked[(int64_t)g.slot[l] * g.n_c + r];
                }
            }
            rec[k] = tab[idx];
        }
    }
}

template <typename R>
static int build_cells(const pg_grid *grid, const void *feats, const uint8_t *baked, const pg_cells *cells,
                       cudaStream_t s) {
    if (int e = validate_grid(grid)) return e;
    PG_REQUIRE(cells != nullptr, "cells: null");
    PG_REQUIRE(grid->feature_dim == 2, "cell cache: F = 2 tables only");
    CellLevels cl;
    cl.n = 0;
    cl.start[0] = 0;
    for (int l = 0; l < grid->n_levels; ++l) {
        if (cells->off[l] < 0) continue;
        PG_REQUIRE(cells->data != nullptr, "cells: null data with cached levels");
        int64_t ncells = 1;
        for (int a = 0; a < grid->d; ++a) ncells *= grid->res[l];
        cl.level[cl.n] = l;
        cl.rec[cl.n] = cells->off[l] * 16 / (int64_t)sizeof(R);
        cl.start[cl.n + 1] = cl.start[cl.n] + ncells;
        ++cl.n;
    }
    if (cl.n == 0) return PG_OK;
    const int grd = grid_for(cl.start[cl.n], 256, 148 * 32);
    R *out = reinterpret_cast<R *>(const_cast<void *>(cells->data));
    if (grid->d == 2)
        build_cells_kernel<2, R><<<grd, 256, 0, s>>>(*grid, cl, (const R *)feats, baked, out);
    else
        build_cells_kernel<3, R><<<grd, 256, 0, s>>>(*grid, cl, (const R *)feats, baked, out);
    return check_launch("cells_build");
}

}  // namespace pg

using namespace pg;

extern "C" {

int64_t pg_cells_plan_rows(const pg_grid *grid, int64_t budget_bytes, int row_bytes, pg_cells *plan) {
    if (!grid || !plan || (row_bytes != 4 && row_bytes != 8)) return -1;
    const int C = 1 << grid->d;
    int64_t total = 0;
    bool open = true;
    plan->data = nullptr;
    for (int l = 0; l < PG_MAX_LEVELS; ++l) {
        plan->off[l] = -1;
        if (!open || l >= grid->n_levels) continue;
        int64_t cells = 1;
        for (int a = 0; a < grid->d; ++a) cells *= grid->res[l];
        const int64_t bytes = cells * C * row_bytes;
        // the decode indexes a level's records with 32-bit math
        if (total + bytes > budget_bytes || cells > ((int64_t)1 << 30)) {
            open = false;
            continue;
        }
        plan->off[l] = total / 16;
        total += bytes;
    }
    return total;
}
int64_t pg_cells_plan(const pg_grid *grid, int64_t budget_bytes, pg_cells *plan) {
    return pg_cells_plan_rows(grid, budget_bytes, 4, plan);
}
int pg_cells_build(const pg_grid *grid, const void *feats16, const uint8_t *baked, const pg_cells *cells,
                   void *stream) {
    return build_cells<uint32_t>(grid, feats16, baked, cells, as_stream(stream));
}
int pg_cells_build_f32(const pg_grid *grid, const float *feats, const uint8_t *baked, const pg_cells *cells,
                       void *stream) {
    return build_cells<uint2>(grid, feats, baked, cells, as_stream(stream));
}

}  // extern "C"
