// Throughput of the legacy warp-level tensor path on sm_100a:
// mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 (and m16n8k16 bf16 for
// scale), 8 independent accumulators per warp. Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 mma_sync_bench.cu -o mma_sync_bench
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tf32(float *out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    float c[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
    const int iters = 4096;
    for (int warps = 4; warps <= 16; warps *= 2) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        k_tf32<<<sms * 2, warps * 32>>>(out, 16);
        cudaEventRecord(e0);
        k_tf32<<<sms * 2, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double macs = (double)sms * 2 * warps * iters * 8 * 16 * 8 * 8;
        printf("{\"warps_per_cta\": %d, \"ctas\": %d, \"tf32_mma_sync_tflops\": %.1f}\n", warps, sms * 2,
               2 * macs / (ms * 1e-3) / 1e12);
    }
    return 0;
}
