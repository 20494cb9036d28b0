// Microbenchmark: scattered 32-byte fp32 reductions into an L2-resident
// table, as two red.global.add.v4.f32 vs one cp.reduce.async.bulk (TMA unit),
// alone and mixed with random 8-byte gathers (the training backward's mix).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_red_bench bulk_red_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE, int GATHERS>
__global__ void __launch_bounds__(256) bench(float *tab, const float2 *src, uint32_t mask_rec, uint32_t mask_g,
                                             int iters, float *sink) {
    __shared__ __align__(128) float stage[256 * 4 * 8];   // 4 slots of 32 B per thread
    float acc = 0.f;
    uint32_t st = blockIdx.x * 256 + threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        st = mix(st + i);
#pragma unroll
        for (int gi = 0; gi < GATHERS; ++gi) {
            const float2 v = __ldg(src + (mix(st + 77 * gi) & mask_g));
            acc += v.x + v.y;
        }
        const uint32_t rec = st & mask_rec;
        float *dst = tab + (size_t)rec * 8;
        const float a = 1e-7f * (float)(i & 7) + acc * 1e-30f;
        if (MODE == 0) {
            asm volatile("red.global.add.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(dst), "f"(a) : "memory");
            asm volatile("red.global.add.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(dst + 4), "f"(a) : "memory");
        } else {
            const int slot = i & 3;
            float *s = stage + (threadIdx.x * 4 + slot) * 8;
            // slot reuse: wait until the bulk op 4 back has read its source
            asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
            reinterpret_cast<float4 *>(s)[0] = make_float4(a, a, a, a);
            reinterpret_cast<float4 *>(s)[1] = make_float4(a, a, a, a);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 32;"
                         ::"l"(dst), "r"(sa) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (MODE == 1) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (acc == 12345.f) sink[0] = acc;
}

template <int MODE, int G>
static void run(const char *name, float *tab, const float2 *src, float *sink, uint32_t mrec, uint32_t mg) {
    const int blocks = 148 * 4, iters = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    bench<MODE, G><<<blocks, 256>>>(tab, src, mrec, mg, iters, sink);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) bench<MODE, G><<<blocks, 256>>>(tab, src, mrec, mg, iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double recs = 10.0 * blocks * 256 * iters;
    printf("%-28s %8.3f ms  %.3e records/s  %.3e gathers/s  err=%s\n", name, ms, recs / (ms * 1e-3),
           recs * G / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
}

int main() {
    float *tab, *sink; float2 *src;
    const uint32_t nrec = 1u << 17;     // 4 MiB of 32-byte records
    const uint32_t ng = 1u << 19;       // 4 MiB of 8-byte gather rows
    cudaMalloc(&tab, (size_t)nrec * 32); cudaMemset(tab, 0, (size_t)nrec * 32);
    cudaMalloc(&src, (size_t)ng * 8); cudaMemset(src, 0, (size_t)ng * 8);
    cudaMalloc(&sink, 4);
    run<0, 0>("red.v4 x2", tab, src, sink, nrec - 1, ng - 1);
    run<1, 0>("bulk reduce 32B", tab, src, sink, nrec - 1, ng - 1);
    run<0, 4>("red.v4 x2 + 4 gathers", tab, src, sink, nrec - 1, ng - 1);
    run<1, 4>("bulk reduce + 4 gathers", tab, src, sink, nrec - 1, ng - 1);
    run<0, 8>("red.v4 x2 + 8 gathers", tab, src, sink, nrec - 1, ng - 1);
    run<1, 8>("bulk reduce + 8 gathers", tab, src, sink, nrec - 1, ng - 1);
    // correctness: sum of the table equals the sum of all added values
    return 0;
}
