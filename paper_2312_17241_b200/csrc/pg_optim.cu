// Optimizer and batch kernels for the device-resident training step
// (trainer.py:63-171) plus the protocol adam_rebake_rows (_core.pyx:224-272).
#include "pg_common.cuh"

namespace pg {

// ---- dense Adam (trainer.py:73-84), numpy's rounding order in T:
//   m = m*b1; m = m + (1-b1)*g; v = v*b2; v = v + (1-b2)*(g*g);
//   p = p - (lr*(m/c1)) / (sqrt(v/c2) + eps)         then g = 0
template <typename T>
__global__ void adam_kernel(T *__restrict__ p, T *__restrict__ g, T *__restrict__ m,
                            T *__restrict__ v, int64_t n, T b1, T nb1, T b2, T nb2, T c1, T c2,
                            T lr, T eps, const double *guard) {
    const bool skip = guard && !isfinite(*guard);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (skip) {
            g[i] = T(0);
            continue;
        }
        const T gi = g[i];
        T mi = Ar<T>::add(Ar<T>::mul(m[i], b1), Ar<T>::mul(nb1, gi));
        T vi = Ar<T>::add(Ar<T>::mul(v[i], b2), Ar<T>::mul(nb2, Ar<T>::mul(gi, gi)));
        m[i] = mi;
        v[i] = vi;
        const T mhat = Ar<T>::div(mi, c1);
        const T vhat = Ar<T>::div(vi, c2);
        p[i] = Ar<T>::sub(p[i], Ar<T>::div(Ar<T>::mul(lr, mhat), Ar<T>::add(Ar<T>::sqrt(vhat), eps)));
        g[i] = T(0);
    }
}

// ---- one confidence row: _core.pyx:246-272 arithmetic (reciprocal bias
// correction), strict '>' argmax from probe 0.
template <typename T>
__device__ __forceinline__ void adam_row(T *cp, T *mp, T *vp, const T *gp, int n_p, T b1, T nb1,
                                         T b2, T nb2, T ic1, T ic2, T lr, T eps, uint8_t *bk) {
    for (int j = 0; j < n_p; ++j) {
        const T gj = gp[j];
        mp[j] = Ar<T>::add(Ar<T>::mul(b1, mp[j]), Ar<T>::mul(nb1, gj));
        vp[j] = Ar<T>::add(Ar<T>::mul(b2, vp[j]), Ar<T>::mul(nb2, Ar<T>::mul(gj, gj)));
    }
    T best = T(0);
    int best_j = 0;
    for (int j = 0; j < n_p; ++j) {
        const T mm = Ar<T>::mul(mp[j], ic1);
        const T vv = Ar<T>::mul(vp[j], ic2);
        const T c = Ar<T>::sub(cp[j], Ar<T>::div(Ar<T>::mul(lr, mm), Ar<T>::add(Ar<T>::sqrt(vv), eps)));
        cp[j] = c;
        if (j == 0 || c > best) {
            best = c;
            best_j = j;
        }
    }
    *bk = (uint8_t)best_j;
}

template <typename T>
__global__ void adam_rebake_rows_kernel(T *conf, T *m, T *v, int n_p, uint8_t *baked,
                                        const int32_t *rows_u, int64_t U, const T *gconf_u, T b1,
                                        T nb1, T b2, T nb2, T ic1, T ic2, T lr, T eps) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= U) return;
    const int64_t r = rows_u[i];
    adam_row<T>(conf + r * n_p, m + r * n_p, v + r * n_p, gconf_u + i * n_p, n_p, b1, nb1, b2, nb2,
                ic1, ic2, lr, eps, baked + r);
}

// lazy variant over touched flags; consumes (zeroes) the gradient row + flag
template <typename T>
__global__ void lazy_adam_rebake_kernel(T *conf, T *m, T *v, uint8_t *baked, T *gconf,
                                        uint8_t *touched, int64_t rows, int n_p, T b1, T nb1, T b2,
                                        T nb2, T ic1, T ic2, T lr, T eps, const double *guard) {
    const bool skip = guard && !isfinite(*guard);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        // a row is due when flagged or when its gradient is non-zero (the
        // fused fp32 training pass flags only all-zero lookups,
        // encode_level_bwd2<..., LAZY>); every lookup of a flagged-or-
        // non-zero row is exactly the reference's touched set up to an
        // exact cancellation of its summed gradient
        T *gp = gconf + r * n_p;
        bool due = touched[r] != 0;
        for (int j = 0; j < n_p && !due; ++j) due = gp[j] != T(0);
        if (!due) continue;
        if (!skip)
            adam_row<T>(conf + r * n_p, m + r * n_p, v + r * n_p, gp, n_p, b1, nb1, b2, nb2, ic1,
                        ic2, lr, eps, baked + r);
        for (int j = 0; j < n_p; ++j) gp[j] = T(0);
        touched[r] = 0;
    }
}

// full bake (codebooks.py:147-152): np.argmax over each row, i.e. the first
// maximum, or the first NaN if the row holds one (numpy's argmax treats NaN
// as the maximum).  The incremental re-bake in adam_row is the Cython core's
// strict '>' scan (_core.pyx:265-272); the two agree on every finite row.
template <typename T>
__global__ void bake_rows_kernel(const T *conf, int64_t rows, int n_p, uint8_t *baked) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const T *cp = conf + r * n_p;
        T best = cp[0];
        int best_j = 0;
        if (!isnan(best)) {
            for (int j = 1; j < n_p; ++j) {
                const T c = cp[j];
                if (isnan(c)) {
                    best_j = j;
                    break;
                }
                if (c > best) {
                    best = c;
                    best_j = j;
                }
            }
        }
        baked[r] = (uint8_t)best_j;
    }
}

// deterministic mode: fixed-point accumulators -> float gradients (added),
// accumulators cleared for the next step
__global__ void fx_accumulate_kernel(fx_t *fx, int64_t n, float *dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const long long v = (long long)fx[i];
        if (v != 0) {
            dst[i] = __fadd_rn(dst[i], (float)ldexp((double)v, -PG_FX_SHIFT));
            fx[i] = 0;
        }
    }
}
__global__ void fx_loss_kernel(fx_t *fx, double *loss) {
    loss[0] = ldexp((double)(long long)fx[0], -PG_FX_LOSS_SHIFT);
    fx[0] = 0;
}

// touched flags <-> slots of the exchange buffer, in the buffer's own
// element type (a float64 model's gradient buffer holds doubles)
template <typename T>
__global__ void touched_to_kernel(const uint8_t *t, int64_t n, T *o) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) o[i] = (T)t[i];
}
template <typename T>
__global__ void touched_from_kernel(const T *in, int64_t n, uint8_t *t) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) t[i] = in[i] > (T)0 ? 1 : 0;
}

// ---- pixel batch (trainer.py:109-116): x = ((col+.5)/W, (row+.5)/H) in
// double then cast, targets = image[pix].  Device draws: splitmix64 of
// (seed, step, i) reduced to [0, W*H) by 128-bit multiply-high.
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <typename T>
__global__ void pixel_batch_kernel(const int64_t *pix_in, int64_t B, int width, int height,
                                   const T *image, int channels, uint64_t seed, uint64_t step,
                                   int64_t *pix_out, T *xs, T *targets) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B) return;
    const uint64_t npix = (uint64_t)width * (uint64_t)height;
    int64_t pix;
    if (pix_in) {
        pix = pix_in[i];
    } else {
        const uint64_t r = splitmix64(seed ^ splitmix64(step * 0x100000001B3ull + (uint64_t)i));
        pix = (int64_t)__umul64hi(r, npix);
        if (pix_out) pix_out[i] = pix;
    }
    const int64_t row = pix / width, col = pix - row * width;
    xs[2 * i] = (T)(((double)col + 0.5) / (double)width);
    xs[2 * i + 1] = (T)(((double)row + 0.5) / (double)height);
    for (int c = 0; c < channels; ++c) targets[i * channels + c] = image[pix * channels + c];
}

struct AdamConsts {
    double b1, nb1, b2, nb2, c1, c2;
};
static AdamConsts adam_consts(int64_t t, double beta1, double beta2) {
    AdamConsts k;
    k.b1 = beta1;
    k.nb1 = 1.0 - beta1;
    k.b2 = beta2;
    k.nb2 = 1.0 - beta2;
    k.c1 = 1.0 - pow(beta1, (double)t);
    k.c2 = 1.0 - pow(beta2, (double)t);
    return k;
}

template <typename T>
static int launch_adam(T *p, T *g, T *m, T *v, int64_t n, int64_t t, double lr, double b1,
                       double b2, double eps, const double *guard, void *stream) {
    PG_REQUIRE(t >= 1, "adam step must be >= 1");
    if (n == 0) return PG_OK;
    const AdamConsts k = adam_consts(t, b1, b2);
    adam_kernel<T><<<grid_for(n, 256, 148 * 16), 256, 0, as_stream(stream)>>>(
        p, g, m, v, n, (T)k.b1, (T)k.nb1, (T)k.b2, (T)k.nb2, (T)k.c1, (T)k.c2, (T)lr, (T)eps, guard);
    return check_launch("adam");
}

template <typename T>
static int launch_lazy(T *conf, T *m, T *v, uint8_t *baked, T *gconf, uint8_t *touched,
                       int64_t rows, int n_p, int64_t t, double lr, double b1, double b2,
                       double eps, const double *guard, void *stream) {
    PG_REQUIRE(t >= 1, "adam step must be >= 1");
    PG_REQUIRE(n_p >= 1 && n_p <= PG_MAX_PROBES, "probing range beyond compiled limit");
    if (rows == 0) return PG_OK;
    const AdamConsts k = adam_consts(t, b1, b2);
    lazy_adam_rebake_kernel<T><<<grid_for(rows, 256, 148 * 16), 256, 0, as_stream(stream)>>>(
        conf, m, v, baked, gconf, touched, rows, n_p, (T)k.b1, (T)k.nb1, (T)k.b2, (T)k.nb2,
        (T)(1.0 / k.c1), (T)(1.0 / k.c2), (T)lr, (T)eps, guard);
    return check_launch("lazy_adam_rebake");
}

template <typename T>
static int launch_rows(T *conf, T *m, T *v, int n_p, uint8_t *baked, const int32_t *rows_u,
                       int64_t U, const T *g, double corr1, double corr2, double lr, double b1,
                       double b2, double eps, void *stream) {
    PG_REQUIRE(n_p >= 1 && n_p <= PG_MAX_PROBES, "probing range beyond compiled limit");
    if (U == 0) return PG_OK;
    adam_rebake_rows_kernel<T><<<grid_for(U, 128), 128, 0, as_stream(stream)>>>(
        conf, m, v, n_p, baked, rows_u, U, g, (T)b1, (T)(1.0 - b1), (T)b2, (T)(1.0 - b2),
        (T)(1.0 / corr1), (T)(1.0 / corr2), (T)lr, (T)eps);
    return check_launch("adam_rebake_rows");
}

template <typename T>
static int launch_pixels(const int64_t *pix_in, int64_t B, int width, int height, const T *image,
                         int channels, uint64_t seed, uint64_t step, int64_t *pix_out, T *xs,
                         T *targets, void *stream) {
    PG_REQUIRE(width >= 1 && height >= 1 && channels >= 1, "bad image shape");
    if (B == 0) return PG_OK;
    pixel_batch_kernel<T><<<grid_for(B, 256), 256, 0, as_stream(stream)>>>(
        pix_in, B, width, height, image, channels, seed, step, pix_out, xs, targets);
    return check_launch("pixel_batch");
}

}  // namespace pg

using namespace pg;

extern "C" {

int pg_adam_f32(float *p, float *g, float *m, float *v, int64_t n, int64_t t, double lr,
                double b1, double b2, double eps, const double *guard, void *stream) {
    return launch_adam<float>(p, g, m, v, n, t, lr, b1, b2, eps, guard, stream);
}
int pg_adam_f64(double *p, double *g, double *m, double *v, int64_t n, int64_t t, double lr,
                double b1, double b2, double eps, const double *guard, void *stream) {
    return launch_adam<double>(p, g, m, v, n, t, lr, b1, b2, eps, guard, stream);
}
int pg_lazy_adam_rebake_f32(float *conf, float *m, float *v, uint8_t *baked, float *gconf,
                            uint8_t *touched, int64_t rows, int n_p, int64_t t, double lr,
                            double b1, double b2, double eps, const double *guard, void *stream) {
    return launch_lazy<float>(conf, m, v, baked, gconf, touched, rows, n_p, t, lr, b1, b2, eps, guard, stream);
}
int pg_lazy_adam_rebake_f64(double *conf, double *m, double *v, uint8_t *baked, double *gconf,
                            uint8_t *touched, int64_t rows, int n_p, int64_t t, double lr,
                            double b1, double b2, double eps, const double *guard, void *stream) {
    return launch_lazy<double>(conf, m, v, baked, gconf, touched, rows, n_p, t, lr, b1, b2, eps, guard, stream);
}
int pg_adam_rebake_rows_f32(float *conf, float *m, float *v, int n_p, uint8_t *baked,
                            const int32_t *rows_u, int64_t U, const float *gconf_u, double corr1,
                            double corr2, double lr, double b1, double b2, double eps,
                            void *stream) {
    return launch_rows<float>(conf, m, v, n_p, baked, rows_u, U, gconf_u, corr1, corr2, lr, b1, b2,
                              eps, stream);
}
int pg_adam_rebake_rows_f64(double *conf, double *m, double *v, int n_p, uint8_t *baked,
                            const int32_t *rows_u, int64_t U, const double *gconf_u, double corr1,
                            double corr2, double lr, double b1, double b2, double eps,
                            void *stream) {
    return launch_rows<double>(conf, m, v, n_p, baked, rows_u, U, gconf_u, corr1, corr2, lr, b1, b2,
                               eps, stream);
}
int pg_bake_rows_f32(const float *conf, int64_t rows, int n_p, uint8_t *baked, void *stream) {
    PG_REQUIRE(n_p >= 1 && n_p <= PG_MAX_PROBES, "n_p out of range");
    if (rows == 0) return PG_OK;
    bake_rows_kernel<float><<<grid_for(rows, 256, 148 * 16), 256, 0, as_stream(stream)>>>(conf, rows, n_p, baked);
    return check_launch("bake_rows");
}
int pg_bake_rows_f64(const double *conf, int64_t rows, int n_p, uint8_t *baked, void *stream) {
    PG_REQUIRE(n_p >= 1 && n_p <= PG_MAX_PROBES, "n_p out of range");
    if (rows == 0) return PG_OK;
    bake_rows_kernel<double><<<grid_for(rows, 256, 148 * 16), 256, 0, as_stream(stream)>>>(conf, rows, n_p, baked);
    return check_launch("bake_rows");
}
int pg_fx_accumulate_f32(uint64_t *fx, int64_t n, float *dst, void *stream) {
    if (n == 0) return PG_OK;
    fx_accumulate_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, as_stream(stream)>>>((fx_t *)fx, n, dst);
    return check_launch("fx_accumulate");
}
int pg_fx_loss(uint64_t *fx, double *loss_sum, void *stream) {
    fx_loss_kernel<<<1, 1, 0, as_stream(stream)>>>((fx_t *)fx, loss_sum);
    return check_launch("fx_loss");
}
int pg_touched_to_f32(const uint8_t *touched, int64_t n, float *out, void *stream) {
    if (n == 0) return PG_OK;
    touched_to_kernel<float><<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(touched, n, out);
    return check_launch("touched_to_f32");
}
int pg_touched_from_f32(const float *in, int64_t n, uint8_t *touched, void *stream) {
    if (n == 0) return PG_OK;
    touched_from_kernel<float><<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(in, n, touched);
    return check_launch("touched_from_f32");
}
int pg_touched_to_f64(const uint8_t *touched, int64_t n, double *out, void *stream) {
    if (n == 0) return PG_OK;
    touched_to_kernel<double><<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(touched, n, out);
    return check_launch("touched_to_f64");
}
int pg_touched_from_f64(const double *in, int64_t n, uint8_t *touched, void *stream) {
    if (n == 0) return PG_OK;
    touched_from_kernel<double><<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(in, n, touched);
    return check_launch("touched_from_f64");
}
int pg_pixel_batch_f32(const int64_t *pix_in, int64_t B, int width, int height, const float *image,
                       int channels, uint64_t seed, uint64_t step, int64_t *pix_out, float *xs,
                       float *targets, void *stream) {
    return launch_pixels<float>(pix_in, B, width, height, image, channels, seed, step, pix_out, xs,
                                targets, stream);
}
int pg_pixel_batch_f64(const int64_t *pix_in, int64_t B, int width, int height,
                       const double *image, int channels, uint64_t seed, uint64_t step,
                       int64_t *pix_out, double *xs, double *targets, void *stream) {
    return launch_pixels<double>(pix_in, B, width, height, image, channels, seed, step, pix_out, xs,
                                 targets, stream);
}

}  // extern "C"
