// .cngp index blocks on the device (FORMAT.md "Index block packing",
// model_io.py:150-165 pack_indices / unpack_indices): each probed level's n_c
// baked probe offsets are stored at w = log2(N_p) bits, entry k in bits
// [k*w, (k+1)*w) counted LSB-first within little-endian bytes, the last byte
// zero-padded.  A file's blocks are uploaded as they lie and expanded here,
// one thread per entry (unpack) / per output byte (pack); both are exact
// integer transforms.
#include "pg_common.cuh"

namespace pg {

__global__ void unpack_indices_kernel(const uint8_t *__restrict__ packed, int64_t n_rows, int64_t n_c, int w,
                                      int64_t block_bytes, uint8_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rows * n_c) return;
    const int64_t r = i / n_c, k = i - r * n_c;
    const uint8_t *blk = packed + r * block_bytes;
    const int64_t bit = k * w, byte = bit >> 3;
    const int sh = (int)(bit & 7);
    uint32_t v = blk[byte];
    if (sh + w > 8) v |= (uint32_t)blk[byte + 1] << 8;  // entry straddles a byte boundary
    out[i] = (uint8_t)((v >> sh) & ((1u << w) - 1u));
}

__global__ void pack_indices_kernel(const uint8_t *__restrict__ entries, int64_t n_rows, int64_t n_c, int w,
                                    int64_t block_bytes, uint8_t *__restrict__ packed) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rows * block_bytes) return;
    const int64_t r = i / block_bytes, j = i - r * block_bytes;
    const uint8_t *e = entries + r * n_c;
    const int64_t lo = j * 8, hi = lo + 8;  // bits of this byte
    uint32_t byte = 0;
    for (int64_t k = lo / w; k < n_c && k * w < hi; ++k) {
        const int64_t b0 = k * w;
        const uint32_t v = e[k] & ((1u << w) - 1u);
        if (b0 >= lo) byte |= v << (b0 - lo);
        else byte |= v >> (lo - b0);
    }
    packed[i] = (uint8_t)(byte & 0xFFu);
}

// Pixel centres of a rectangle of a W x H image in raster order
// (model_io.py:321-325 _grid_coords: float32((c + 0.5) / W) with the division
// in double, as numpy does), so decode_rect / decode_image need no host-side
// coordinate arrays.
__global__ void raster_coords_kernel(int x0, int y0, int w, int64_t n, int W, int H, float *__restrict__ xs) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t r = i / w, c = i - r * w;
    const double u = ((double)(x0 + c) + 0.5) / (double)W;
    const double v = ((double)(y0 + r) + 0.5) / (double)H;
    reinterpret_cast<float2 *>(xs)[i] = make_float2(__double2float_rn(u), __double2float_rn(v));
}

}  // namespace pg

namespace pg {
// pngio.py:39: np.rint(np.clip(p, 0, 1) * 255).astype(uint8) on a float32
// array: float32 clip, rounded float32 multiply, round half to even
__global__ void quantize_u8_kernel(const float *__restrict__ x, int64_t n, uint8_t *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float v = fminf(fmaxf(x[i], 0.0f), 1.0f);
        out[i] = (uint8_t)rintf(__fmul_rn(v, 255.0f));
    }
}
}  // namespace pg

extern "C" {

int pg_raster_coords_f32(int x0, int y0, int w, int h, int width, int height, float *xs, void *stream) {
    PG_REQUIRE(width >= 1 && height >= 1, "raster_coords: empty image");
    PG_REQUIRE(0 <= x0 && x0 + w <= width && 0 <= y0 && y0 + h <= height && w >= 0 && h >= 0,
               "raster_coords: rectangle outside the image");
    const int64_t n = (int64_t)w * h;
    if (n == 0) return PG_OK;
    pg::raster_coords_kernel<<<(unsigned)((n + 255) / 256), 256, 0, pg::as_stream(stream)>>>(x0, y0, w, n, width,
                                                                                            height, xs);
    return pg::check_launch("raster_coords");
}


int pg_unpack_indices(const uint8_t *packed, int64_t n_rows, int64_t n_c, int log2_np, uint8_t *entries,
                      void *stream) {
    PG_REQUIRE(log2_np >= 1 && log2_np <= 8, "unpack_indices: log2_np must be in [1, 8]");
    PG_REQUIRE(n_rows >= 0 && n_c >= 0, "unpack_indices: negative size");
    const int64_t n = n_rows * n_c;
    if (n == 0) return PG_OK;
    const int64_t block_bytes = (n_c * log2_np + 7) / 8;
    pg::unpack_indices_kernel<<<(unsigned)((n + 255) / 256), 256, 0, pg::as_stream(stream)>>>(
        packed, n_rows, n_c, log2_np, block_bytes, entries);
    return pg::check_launch("unpack_indices");
}

int pg_pack_indices(const uint8_t *entries, int64_t n_rows, int64_t n_c, int log2_np, uint8_t *packed,
                    void *stream) {
    PG_REQUIRE(log2_np >= 1 && log2_np <= 8, "pack_indices: log2_np must be in [1, 8]");
    PG_REQUIRE(n_rows >= 0 && n_c >= 0, "pack_indices: negative size");
    const int64_t block_bytes = (n_c * log2_np + 7) / 8;
    const int64_t n = n_rows * block_bytes;
    if (n == 0) return PG_OK;
    pg::pack_indices_kernel<<<(unsigned)((n + 255) / 256), 256, 0, pg::as_stream(stream)>>>(
        entries, n_rows, n_c, log2_np, block_bytes, packed);
    return pg::check_launch("pack_indices");
}

int pg_quantize_u8_f32(const float *x, int64_t n, uint8_t *out, void *stream) {
    PG_REQUIRE(n >= 0, "quantize: negative size");
    if (n == 0) return PG_OK;
    pg::quantize_u8_kernel<<<pg::grid_for(n, 256, 148 * 16), 256, 0, pg::as_stream(stream)>>>(x, n, out);
    return pg::check_launch("quantize_u8");
}

}  // extern "C"
