// Microbenchmark: random 16-byte row fetches from an
// L2-resident table through the TMA engine (cp.async.bulk.tensor.2d ...
// tile::gather4: four rows per instruction, landing in shared memory,
// completion on an mbarrier) against per-lane LSU gathers (ld.global.nc.v4).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_gather tools/micro/tma_gather_bench.cu -lcuda
//   /tmp/tma_gather [rows_log2=16]
//
// A 16-byte row = one N_p = 4 probing range of fp16 F = 2 features (the
// decode's whole-range fetch).  Reports rows/s for: LSU (every lane its own
// row), TMA with 1 issuing thread per CTA, and TMA with 4 issuing threads
// (one per warp) per CTA, each with an S-stage ring of 64-byte slots.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);       \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t i, uint32_t s) {
    uint32_t h = i * 2654435761u ^ s;
    h ^= h >> 15;
    h *= 0x2c1b3c6du;
    h ^= h >> 12;
    return h;
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void lsu_kernel(const uint4 *tab, uint32_t mask, int64_t n_rows, uint32_t *sink) {
    uint32_t acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_rows; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            v[u] = __ldg(tab + (hash32((uint32_t)(i + u * stride), 7) & mask));
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

// ISSUERS threads per CTA (lane 0 of warps 0..ISSUERS-1) each run an S-slot
// ring: wait slot free -> expect_tx(64) -> gather4; the whole warp then waits
// for completion of the oldest slot and reads it (as a consumer would).
template <int ISSUERS, int S>
__global__ void tma_kernel(const __grid_constant__ CUtensorMap map, uint32_t mask, int64_t n_instr,
                           uint32_t *sink) {
    __shared__ __align__(128) uint4 slots[ISSUERS][S][8];   // 64 B used, 128-B aligned slots
    __shared__ __align__(8) uint64_t full[ISSUERS][S];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp >= ISSUERS) return;
    if (lane == 0)
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t per = n_instr / ((int64_t)gridDim.x * ISSUERS);
    const uint32_t seed = (uint32_t)(blockIdx.x * ISSUERS + warp) * 0x9E3779B9u;
    uint32_t acc = 0;
    auto issue = [&](int64_t k) {
        const int s = (int)(k % S);
        const uint32_t mb = smem_u32(&full[warp][s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 64;" ::"r"(mb) : "memory");
        const int r0 = (int)(hash32((uint32_t)(4 * k), seed) & mask), r1 = (int)(hash32((uint32_t)(4 * k + 1), seed) & mask);
        const int r2 = (int)(hash32((uint32_t)(4 * k + 2), seed) & mask), r3 = (int)(hash32((uint32_t)(4 * k + 3), seed) & mask);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(&slots[warp][s][0])),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(mb), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
            : "memory");
    };
    if (lane == 0)
        for (int64_t k = 0; k < S && k < per; ++k) issue(k);
    for (int64_t k = 0; k < per; ++k) {
        const int s = (int)(k % S);
        const uint32_t mb = smem_u32(&full[warp][s]), par = (uint32_t)((k / S) & 1);
        asm volatile(
            "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra W_%=;\n\t}\n" ::"r"(mb),
            "r"(par)
            : "memory");
        if (lane < 4) {
            const uint4 v = slots[warp][s][lane];
            acc += v.x ^ v.w;
        }
        __syncwarp();
        if (lane == 0 && k + S < per) issue(k + S);
    }
    if (acc == 0x12345678u) *sink = acc;
}

typedef CUresult (*encode_fn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
    const int lg = argc > 1 ? atoi(argv[1]) : 16;
    const int64_t rows = (int64_t)1 << lg;
    uint4 *tab;
    uint32_t *sink;
    CK(cudaMalloc(&tab, rows * 16));
    CK(cudaMemset(tab, 1, rows * 16));
    CK(cudaMalloc(&sink, 4));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float ms;
    const int64_t n = (int64_t)1 << 28;
    lsu_kernel<<<sms * 8, 256>>>(tab, (uint32_t)(rows - 1), n, sink);
    CK(cudaEventRecord(e0));
    lsu_kernel<<<sms * 8, 256>>>(tab, (uint32_t)(rows - 1), n, sink);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("LSU ld.global.nc.v4 random 16-B rows: %.3e rows/s (%.2f rows/SM/clk at 1.965 GHz)\n", n / (ms * 1e-3),
           n / (ms * 1e-3) / sms / 1.965e9);

    encode_fn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
    CUtensorMap map;
    const cuuint64_t dims[2] = {8, (cuuint64_t)rows};          // 8 halfs (16 B) x rows
    const cuuint64_t strides[1] = {16};
    const cuuint32_t box[2] = {8, 1};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, tab, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("cuTensorMapEncodeTiled(box 8x1): %d\n", (int)r);
    if (r != CUDA_SUCCESS) return 1;
    const int64_t ni = (int64_t)1 << 25;   // instructions (4 rows each)
#define RUN(ISS, S, CTAS)                                                                                      \
    do {                                                                                                       \
        tma_kernel<ISS, S><<<sms * CTAS, 32 * ISS>>>(map, (uint32_t)(rows - 1), ni, sink);                      \
        CK(cudaGetLastError());                                                                                \
        CK(cudaEventRecord(e0));                                                                               \
        tma_kernel<ISS, S><<<sms * CTAS, 32 * ISS>>>(map, (uint32_t)(rows - 1), ni, sink);                      \
        CK(cudaEventRecord(e1));                                                                               \
        CK(cudaEventSynchronize(e1));                                                                          \
        CK(cudaEventElapsedTime(&ms, e0, e1));                                                                 \
        printf("TMA gather4: %d issuers/CTA x %d CTAs/SM, %2d-slot ring: %.3e rows/s (%.2f rows/SM/clk)\n", ISS, \
               CTAS, S, 4.0 * ni / (ms * 1e-3), 4.0 * ni / (ms * 1e-3) / sms / 1.965e9);                    \
    } while (0)
    RUN(1, 8, 1);
    RUN(1, 16, 1);
    RUN(4, 8, 1);
    RUN(4, 16, 1);
    RUN(4, 16, 4);
    RUN(8, 16, 2);
    RUN(16, 16, 1);
    RUN(16, 16, 2);
    return 0;
}
