// Latency vs chain count of mma.sync m16n8k8 tf32 on sm_100a: one CTA per
// SM, W warps per scheduler, each warp issuing NC independent accumulator
// chains.  Prints cycles per HMMA per warp and HMMAs per SM per clock.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 mma_chain_bench.cu -o mma_chain_bench
#include <cstdio>
#include <cuda_runtime.h>

template <int NC>
__global__ void k(float *out, long long *cyc, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    float c[NC][4] = {};
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < NC; ++j)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    long long t1 = clock64();
    float s = 0;
    for (int j = 0; j < NC; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NC>
void run(int sms, float *out, long long *cyc, int wps) {
    const int iters = 2048, threads = 4 * wps * 32;
    k<NC><<<sms, threads>>>(out, cyc, 16);
    k<NC><<<sms, threads>>>(out, cyc, iters);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double per = (double)h / ((double)iters * NC);
    printf("chains %2d warps/SMSP %d: %6.2f cyc per HMMA per warp, %5.3f HMMA/SM/clk\n", NC, wps, per,
           4.0 * wps / per);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    long long *cyc;
    cudaMalloc(&out, sizeof(float) * sms * 2048);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    for (int w = 1; w <= 4; w *= 2) {
        run<1>(sms, out, cyc, w);
        run<2>(sms, out, cyc, w);
        run<4>(sms, out, cyc, w);
        run<8>(sms, out, cyc, w);
        run<12>(sms, out, cyc, w);
    }
    return 0;
}
