// Fused decode on the 5th-generation tensor core (tcgen05 / UMMA):
//   per 128-query tile: 16-level encode (fp16 tables) -> layer 1 and layer 2
//   of the MLP as kind::tf32 UMMA (M=128, N=64, accumulators in TMEM) ->
//   bias/ReLU epilogues from TMEM -> output layer (64 -> <=4) in registers.
//
// Accuracy: activations are fed as a 2-term tf32 expansion (hi + lo, ~22
// significand bits); the weights of an inference model are fp16-rounded
// (to_inference, model_io.py:130-147), hence exactly representable in tf32.
// Each layer is therefore 2 passes of UMMA and matches fp32 to ~1e-6
// relative (tests/test_gpu_parity.py bounds it at rtol 1e-5).
#include "pg_encode_dev.cuh"
#include "pg_umma.cuh"

namespace pg {

namespace tc {
constexpr int kTP = 128;  // queries per tile == UMMA M
constexpr int kIn = 32;
constexpr int kHid = 64;
constexpr int kOutMax = 4;
constexpr int kThreads = 256;

struct Smem {
    // operand region: layer-1 A (hi | lo, 128x32 each) then layer-2 A (hi | lo, 128x64 each)
    alignas(16) float opA[2 * kTP * kHid];
    alignas(16) float b1[kHid * kIn];   // W0^T, K-major
    alignas(16) float b2[kHid * kHid];  // W1^T, K-major
    float w2[kHid * kOutMax];
    float bias0[kHid], bias1[kHid], bias2[kOutMax];
    float part[2][kTP][kOutMax];
    float xs[kTP * 3];
    uint64_t mbar[2];
    uint32_t tmem_base;
};
}  // namespace tc

template <typename FT, int D>
__global__ void __launch_bounds__(tc::kThreads, 2)
    decode_umma_kernel(const pg_grid g, const float *__restrict__ xs, int64_t B,
                       const FT *__restrict__ feats, const uint8_t *__restrict__ baked,
                       const float *__restrict__ params, int od, int sigmoid,
                       float *__restrict__ out) {
    using namespace tc;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

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
    if (warp == 0) umma::tmem_alloc<128>(&S.tmem_base);
    if (tid == 0) {
        umma::mbar_init(&S.mbar[0], 1);
        umma::mbar_init(&S.mbar[1], 1);
        umma::mbar_init_fence();
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = S.tmem_base;
    const uint32_t tm_d1 = tmem, tm_d2 = tmem + kHid;   // columns [0,64) and [64,128)
    const uint32_t idesc = umma::idesc_tf32(kTP, kHid);
    char *opA = reinterpret_cast<char *>(S.opA);
    const uint32_t a_s = umma::smem_u32(opA);
    const uint32_t b1_s = umma::smem_u32(S.b1), b2_s = umma::smem_u32(S.b2);
    // epilogue role: row (TMEM lane) and column half
    const int erow = (warp & 3) * 32 + lane;
    const int ehalf = warp >> 2;  // 0: columns 0..31, 1: columns 32..63
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;

    const int64_t ntiles = (B + kTP - 1) / kTP;
    uint32_t phase = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, phase ^= 1u) {
        const int64_t p0 = tile * kTP;
        const int nv = (int)((B - p0) < kTP ? (B - p0) : kTP);
        for (int i = tid; i < kTP * D; i += kThreads) S.xs[i] = i < nv * D ? xs[p0 * D + i] : 0.5f;
        __syncthreads();
        // ---------------- encode -> layer-1 A operand (hi | lo) ----------------
        {
            const int q = tid & (kTP - 1), lsub = tid >> 7;
            float x[D];
#pragma unroll
            for (int a = 0; a < D; ++a) x[a] = S.xs[q * D + a];
            // a thread encodes level PAIRS (2P, 2P+1): their 4 features fill one
            // 16-byte K-chunk, so the operand stores are float4 and a warp's
            // 32 queries hit 4 full wavefronts (no bank conflicts)
#pragma unroll 2
            for (int it = 0; it < 4; ++it) {
                const int P = lsub + 2 * it;  // warp-uniform
                const float2 ya = encode_level_fwd2<FT, D>(g, 2 * P, x, feats, baked);
                const float2 yb = encode_level_fwd2<FT, D>(g, 2 * P + 1, x, feats, baked);
                float h[4], lo[4];
                umma::split_tf32(ya.x, h[0], lo[0]);
                umma::split_tf32(ya.y, h[1], lo[1]);
                umma::split_tf32(yb.x, h[2], lo[2]);
                umma::split_tf32(yb.y, h[3], lo[3]);
                const uint32_t off = umma::kmaj_off(q, 4 * P, kTP);
                *reinterpret_cast<float4 *>(opA + off) = make_float4(h[0], h[1], h[2], h[3]);
                *reinterpret_cast<float4 *>(opA + kTP * kIn * 4 + off) = make_float4(lo[0], lo[1], lo[2], lo[3]);
            }
        }
        umma::fence_async_smem();
        umma::fence_before_sync();
        __syncthreads();
        // ---------------- layer 1: D1 = (Y_hi + Y_lo) . W0 ----------------
        if (tid == 0) {
            umma::fence_after_sync();
#pragma unroll
            for (int pass = 0; pass < 2; ++pass)
#pragma unroll
                for (int kb = 0; kb < kIn / 8; ++kb) {
                    const uint64_t ad = umma::smem_desc(a_s + pass * kTP * kIn * 4 + kb * kTP * 32, 128, 256);
                    const uint64_t bd = umma::smem_desc(b1_s + kb * kHid * 32, 128, 256);
                    umma::mma_tf32(tm_d1, ad, bd, idesc, (pass | kb) ? 1u : 0u);
                }
            umma::commit(&S.mbar[0]);
        }
        umma::mbar_wait(&S.mbar[0], phase);
        umma::fence_after_sync();
        // ---------------- epilogue 1: bias + ReLU -> layer-2 A operand ----------------
        {
            float v[32];
            umma::tmem_ld32(tm_d1 + lane_off + ehalf * 32, v);
#pragma unroll
            for (int c = 0; c < 32; c += 4) {
                float hi[4], lo[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    float z = v[c + u] + S.bias0[ehalf * 32 + c + u];
                    z = z < 0.0f ? 0.0f : z;
                    umma::split_tf32(z, hi[u], lo[u]);
                }
                const uint32_t off = umma::kmaj_off(erow, ehalf * 32 + c, kTP);
                *reinterpret_cast<float4 *>(opA + off) = make_float4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<float4 *>(opA + kTP * kHid * 4 + off) = make_float4(lo[0], lo[1], lo[2], lo[3]);
            }
        }
        umma::fence_async_smem();
        umma::fence_before_sync();
        __syncthreads();
        // ---------------- layer 2: D2 = (H1_hi + H1_lo) . W1 ----------------
        if (tid == 0) {
            umma::fence_after_sync();
#pragma unroll
            for (int pass = 0; pass < 2; ++pass)
#pragma unroll
                for (int kb = 0; kb < kHid / 8; ++kb) {
                    const uint64_t ad = umma::smem_desc(a_s + pass * kTP * kHid * 4 + kb * kTP * 32, 128, 256);
                    const uint64_t bd = umma::smem_desc(b2_s + kb * kHid * 32, 128, 256);
                    umma::mma_tf32(tm_d2, ad, bd, idesc, (pass | kb) ? 1u : 0u);
                }
            umma::commit(&S.mbar[1]);
        }
        umma::mbar_wait(&S.mbar[1], phase);
        umma::fence_after_sync();
        // ---------------- epilogue 2: bias + ReLU + output layer ----------------
        {
            float v[32];
            umma::tmem_ld32(tm_d2 + lane_off + ehalf * 32, v);
            float acc[kOutMax] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const int k = ehalf * 32 + c;
                float h = v[c] + S.bias1[k];
                h = h < 0.0f ? 0.0f : h;
                const float4 w = *reinterpret_cast<const float4 *>(S.w2 + k * kOutMax);
                acc[0] = fmaf(h, w.x, acc[0]);
                acc[1] = fmaf(h, w.y, acc[1]);
                acc[2] = fmaf(h, w.z, acc[2]);
                acc[3] = fmaf(h, w.w, acc[3]);
            }
#pragma unroll
            for (int j = 0; j < kOutMax; ++j) S.part[ehalf][erow][j] = acc[j];
        }
        umma::fence_before_sync();
        __syncthreads();
        {
            float *dst = out + p0 * od;
            for (int i = tid; i < nv * od; i += kThreads) {
                const int q = i / od, j = i - q * od;
                float o = S.bias2[j] + S.part[0][q][j] + S.part[1][q][j];
                if (sigmoid) o = (float)(1.0 / (1.0 + exp(-(double)o)));
                dst[i] = o;
            }
        }
    }
    umma::fence_after_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free<128>(tmem);
}

int decode_umma(const pg_grid *g, int od, const float *xs, int64_t B, const void *feats, bool half,
                const uint8_t *baked, const float *params, int sig, float *out, cudaStream_t s) {
    const int smem = (int)sizeof(tc::Smem);
    static bool configured[4] = {false, false, false, false};
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ntiles = (B + tc::kTP - 1) / tc::kTP;
    const int64_t cap = (int64_t)sms * 2;
    const int grd = (int)(ntiles < cap ? ntiles : cap);
#define PG_DEC_TC(FT_, D_, IDX)                                                                   \
    do {                                                                                          \
        if (!configured[IDX]) {                                                                   \
            cudaFuncSetAttribute(decode_umma_kernel<FT_, D_>,                                     \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem);              \
            configured[IDX] = true;                                                               \
        }                                                                                         \
        decode_umma_kernel<FT_, D_><<<grd, tc::kThreads, smem, s>>>(*g, xs, B, (const FT_ *)feats, \
                                                                   baked, params, od, sig, out);  \
    } while (0)
    if (half) {
        if (g->d == 2) PG_DEC_TC(__half, 2, 0); else PG_DEC_TC(__half, 3, 1);
    } else {
        if (g->d == 2) PG_DEC_TC(float, 2, 2); else PG_DEC_TC(float, 3, 3);
    }
#undef PG_DEC_TC
    return check_launch("decode_umma");
}

}  // namespace pg
