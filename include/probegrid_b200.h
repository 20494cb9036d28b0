/*
 * probegrid_b200 — C ABI of the B200 (sm_100a) learned-hash-probing hot path.
 *
 * Drop-in boundary for the reference package `probegrid`
 * (/root/reference/pkg).  The reference's only native seam is its compiled
 * Cython core, bound through the backend protocol
 * (src/probegrid/backends/__init__.py:12-50, cython_backend.py:24-89).  Each
 * "protocol" entry point below replaces one of those bindings with the same
 * argument meaning; the "fused" entry points replace the Python orchestration
 * above them (encoding.py, mlp.py, trainer.py, model_io.py) with whole-path
 * kernels.  A maintainer binds them with ctypes exactly as
 * paper_2312_17241_b200/_lib.py does.
 *
 * Conventions
 *  - Every array argument is a DEVICE pointer unless its name starts with h_.
 *  - Shapes are C-contiguous row-major, as the reference's memoryviews require.
 *  - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *  - Calls are asynchronous on `stream`; they return PG_OK or an error code,
 *    with a message available from pg_last_error() (thread-local).
 *  - The library never allocates device memory on these paths; callers own
 *    every buffer, including workspaces sized by the *_workspace_bytes calls.
 *  - Suffix _f32 / _f64 selects float / double storage and arithmetic.
 */
#ifndef PROBEGRID_B200_H
#define PROBEGRID_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PG_OK 0
#define PG_ERR_ARG 1      /* invalid argument (shape, limit, null pointer)     */
#define PG_ERR_CUDA 2     /* CUDA launch / runtime failure                     */
#define PG_ERR_DOMAIN 3   /* a coordinate lies outside [0,1]^d                 */

#define PG_MAX_LEVELS 64    /* model file limit, model_io.py:207              */
#define PG_MAX_FEATURE 16   /* compiled limit, cython_backend.py:9            */
#define PG_MAX_PROBES 256   /* 8-bit baked storage, model.py:61-62            */
#define PG_MAX_LAYERS 17    /* n_hidden_layers <= 16, model_io.py:213         */

/* level kinds: indexing.py:26-41 + model.py:150 (probing iff hashed & conf) */
#define PG_LEVEL_DENSE 0
#define PG_LEVEL_HASHED 1
#define PG_LEVEL_PROBED 2

/* flags */
#define PG_EXACT_MLP 1u   /* MLP in the reference's operation order, no FMA   */
#define PG_SIGMOID 2u     /* logistic output (HyperParams.out_sigmoid)        */
#define PG_SURROGATE 4u   /* softmax-mixture forward (encoding.py:45-47)      */
#define PG_HALF_FEATS 8u  /* feature tables stored as IEEE binary16           */
#define PG_NO_TENSOR 16u  /* decode: FFMA MLP instead of tcgen05 (ablation)   */
#define PG_SMEM_TABLES 32u    /* decode: force the shared-memory baked-index
                               * variant (default: automatic, N_p = 2 or 4) */
#define PG_NO_SMEM_TABLES 64u /* decode: never use it                       */
#define PG_TOUCH_ALL 256u     /* fused fp32 training: flag every probed lookup
                                 as touched (data-parallel steps; see
                                 pg_train_fused_f32) */
#define PG_COMPOSITE 128u     /* fused training: volume compositing, one ray
                               * of 64 samples per tile; targets (B, 4) =
                               * (segment length, ray r, g, b) per sample */

/* Geometry of one multiresolution grid (HyperParams + build_level_specs,
 * model.py:35-87, indexing.py:93-101).  Feature tables of all levels are one
 * buffer [n_levels][n_f][feature_dim]; probed levels additionally own slot
 * `slot[l]` of conf [n_probed][n_c][n_p] and baked [n_probed][n_c]. */
typedef struct pg_grid {
    int32_t d;            /* 2 or 3                                          */
    int32_t n_levels;
    int32_t feature_dim;  /* F                                               */
    int32_t n_f;          /* rows per feature table (power of two)           */
    int32_t n_c;          /* rows per index/confidence table (power of two)  */
    int32_t log2_np;      /* log2 of the probing range N_p                   */
    int32_t res[PG_MAX_LEVELS];
    int32_t kind[PG_MAX_LEVELS];
    int32_t slot[PG_MAX_LEVELS];
    uint32_t primary[3];  /* indexing.py:22 */
    uint32_t aux[3];      /* indexing.py:23 */
} pg_grid;

/* Tiny MLP shape (mlp.py:16-52): weights (fan_in, fan_out) row-major; the
 * parameter buffer is [W0 | b0 | W1 | b1 | ...] in that order. */
typedef struct pg_mlp {
    int32_t n_layers;
    int32_t widths[PG_MAX_LAYERS + 1];
} pg_mlp;

/* Decode cell cache (inference-time acceleration structure, not part of the
 * model file): for the coarsest levels, one record per grid cell holding
 * the 2^d corners' RESOLVED fp16 feature rows (dense index, or probed base +
 * baked offset) in corner order — one 16-byte (2-D) / 32-byte (3-D) load per
 * query and level instead of 2^d dependent index + row gathers.  The values
 * are copies of the table rows, so a cached decode is bit-identical to an
 * uncached one.  off[l]: record offset of level l in 16-byte units, -1 when
 * the level is not cached. */
typedef struct pg_cells {
    const void *data;
    int64_t off[PG_MAX_LEVELS];
} pg_cells;

const char *pg_last_error(void);
const char *pg_version(void);
int pg_device_sm_count(int device);

/* ------------------------------------------------------------------------
 * Protocol kernels: one level / one layer per call, numpy-backend semantics.
 * ---------------------------------------------------------------------- */

/* replaces _core.dense_fwd (_core.pyx:26-54) via cython_backend.dense_fwd
 * (cython_backend.py:24-31).  out must be zero-initialised by the caller. */
int pg_dense_fwd_f32(const float *xs, int64_t B, int d, int64_t res,
                     const float *feats, int F, float *out, int32_t *idx,
                     float *wgt, void *stream);
int pg_dense_fwd_f64(const double *xs, int64_t B, int d, int64_t res,
                     const double *feats, int F, double *out, int32_t *idx,
                     double *wgt, void *stream);

/* replaces _core.hashed_fwd (_core.pyx:57-84), cython_backend.py:34-42;
 * primary points to d host uint32 primes. */
int pg_hashed_fwd_f32(const float *xs, int64_t B, int d, int64_t res,
                      uint32_t nf_mask, const float *feats, int F,
                      const uint32_t *h_primary, float *out, int32_t *idx,
                      float *wgt, void *stream);
int pg_hashed_fwd_f64(const double *xs, int64_t B, int d, int64_t res,
                      uint32_t nf_mask, const double *feats, int F,
                      const uint32_t *h_primary, double *out, int32_t *idx,
                      double *wgt, void *stream);

/* replaces _core.probed_fwd (_core.pyx:87-122), cython_backend.py:45-55 */
int pg_probed_fwd_f32(const float *xs, int64_t B, int d, int64_t res,
                      uint32_t nf_mask, uint32_t nc_mask, int log2_np,
                      const float *feats, int F, const uint8_t *baked,
                      const uint32_t *h_primary, const uint32_t *h_aux,
                      float *out, int32_t *base, int32_t *row, float *wgt,
                      void *stream);
int pg_probed_fwd_f64(const double *xs, int64_t B, int d, int64_t res,
                      uint32_t nf_mask, uint32_t nc_mask, int log2_np,
                      const double *feats, int F, const uint8_t *baked,
                      const uint32_t *h_primary, const uint32_t *h_aux,
                      double *out, int32_t *base, int32_t *row, double *wgt,
                      void *stream);

/* replaces _core.indexed_bwd (_core.pyx:125-137): gfeat[idx] += w*up */
int pg_indexed_bwd_f32(const float *up, int64_t B, int F, const int32_t *idx,
                       const float *wgt, int C, float *gfeat, void *stream);
int pg_indexed_bwd_f64(const double *up, int64_t B, int F, const int32_t *idx,
                       const double *wgt, int C, double *gfeat, void *stream);

/* replaces _core.dedup_rows (_core.pyx:140-160): same first-encounter order.
 * Workspace: pg_dedup_workspace_bytes(n, n_c).  *d_count receives U. */
int64_t pg_dedup_workspace_bytes(int64_t n, int64_t n_c);
int pg_dedup_rows(const int32_t *row, int64_t n, int64_t n_c, void *workspace,
                  int32_t *rows_u, int32_t *inv, int32_t *d_count,
                  void *stream);

/* replaces _core.probed_bwd (_core.pyx:163-221) */
int pg_probed_bwd_f32(const float *up, int64_t B, int F, const int32_t *base,
                      const int32_t *inv, const float *wgt, int C,
                      const float *smu, int n_p, const float *feats,
                      float *gfeat, float *gconf_u, void *stream);
int pg_probed_bwd_f64(const double *up, int64_t B, int F, const int32_t *base,
                      const int32_t *inv, const double *wgt, int C,
                      const double *smu, int n_p, const double *feats,
                      double *gfeat, double *gconf_u, void *stream);

/* replaces _core.adam_rebake_rows (_core.pyx:224-272); corr1/corr2 are
 * 1-beta^t as cython_backend.py:73-77 passes them. */
int pg_adam_rebake_rows_f32(float *conf, float *m, float *v, int n_p,
                            uint8_t *baked, const int32_t *rows_u, int64_t U,
                            const float *gconf_u, double corr1, double corr2,
                            double lr, double beta1, double beta2, double eps,
                            void *stream);
int pg_adam_rebake_rows_f64(double *conf, double *m, double *v, int n_p,
                            uint8_t *baked, const int32_t *rows_u, int64_t U,
                            const double *gconf_u, double corr1, double corr2,
                            double lr, double beta1, double beta2, double eps,
                            void *stream);

/* replaces cython_backend.mlp_infer_rows (cython_backend.py:80-89, i.e.
 * _core.linear_rows/_core.sigmoid_rows, _core.pyx:275-298): row-wise, in the
 * reference's operation order (bit-identical), any widths.  act_ws needs
 * 2*B*max(widths) elements. */
int pg_mlp_infer_rows_f32(const float *xs, int64_t B, const pg_mlp *mlp,
                          const float *params, unsigned flags, float *act_ws,
                          float *out, void *stream);
int pg_mlp_infer_rows_f64(const double *xs, int64_t B, const pg_mlp *mlp,
                          const double *params, unsigned flags,
                          double *act_ws, double *out, void *stream);

/* ------------------------------------------------------------------------
 * Fused B200 kernels (all levels / the whole MLP per launch).
 * ---------------------------------------------------------------------- */

/* encoding.encode_forward (encoding.py:42-86) for all levels at once:
 * y (B, L*F).  flags: PG_SURROGATE (needs conf), PG_HALF_FEATS (feats is
 * binary16).  *d_bad (optional) is set to 1 if any coordinate is outside
 * [0,1] (encoding.py:33-39). */
int pg_encode_fwd_f32(const pg_grid *grid, const float *xs, int64_t B,
                      const void *feats, const uint8_t *baked,
                      const float *conf, unsigned flags, float *y,
                      int32_t *d_bad, void *stream);
int pg_encode_fwd_f64(const pg_grid *grid, const double *xs, int64_t B,
                      const void *feats, const uint8_t *baked,
                      const double *conf, unsigned flags, double *y,
                      int32_t *d_bad, void *stream);

/* encoding.encode_backward (encoding.py:89-133) for all levels at once.
 * Recomputes geometry from xs; accumulates into gfeat [L][n_f][F] and
 * gconf [P][n_c][N_p]; marks every looked-up confidence row in
 * touched [P][n_c] (uint8, set to 1), including zero-weight corners. */
int pg_encode_bwd_f32(const pg_grid *grid, const float *xs, int64_t B,
                      const float *dy, const float *feats, const float *conf,
                      float *gfeat, float *gconf, uint8_t *touched,
                      void *stream);
int pg_encode_bwd_f64(const pg_grid *grid, const double *xs, int64_t B,
                      const double *dy, const double *feats,
                      const double *conf, double *gfeat, double *gconf,
                      uint8_t *touched, void *stream);

/* model_io.decode_pixels (model_io.py:292-311): fused encode + MLP forward
 * per 128-query tile; out (B, out_dim).  Fast path for widths
 * [L*F = 32, 64, 64, out_dim <= 4]; other shapes run the generic kernels
 * (then ws must hold B*(L*F) + 2*B*max(widths) floats, else ws may be 0).
 * PG_EXACT_MLP reproduces _core.linear_rows bit for bit. */
int pg_decode_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs,
                  int64_t B, const void *feats, const uint8_t *baked,
                  const float *params, unsigned flags, float *ws, float *out,
                  void *stream);

/* End-to-end decode from HOST memory (pinned for overlap): chunks of up to
 * `chunk` queries, H2D copies on stream_in, fused decodes on stream_compute,
 * D2H copies on stream_out, two buffer slots ordered by events so both copy
 * directions overlap the kernels.  d_xs must hold 2*chunk*d floats, d_out
 * 2*chunk*out_dim floats.  Returns after all three streams drain. */
int pg_decode_host_f32(const pg_grid *grid, const pg_mlp *mlp,
                       const float *h_xs, int64_t B, const void *feats,
                       const uint8_t *baked, const float *params,
                       unsigned flags, int64_t chunk, float *d_xs,
                       float *d_out, float *h_out, void *stream_in,
                       void *stream_compute, void *stream_out);

/* Cell cache: pg_cells_plan fills plan->off for the coarsest levels whose
 * records fit `budget_bytes` (levels in order, stopping at the first that
 * does not fit) and returns the bytes needed (0: nothing cached);
 * pg_cells_build writes the records of fp16 tables feats16/baked (the
 * InferenceModel's) into cells->data.  Rebuild after the tables change. */
int64_t pg_cells_plan(const pg_grid *grid, int64_t budget_bytes, pg_cells *plan);
int pg_cells_build(const pg_grid *grid, const void *feats16, const uint8_t *baked,
                   const pg_cells *cells, void *stream);
/* The same for fp32 F = 2 rows (8 bytes per corner: the training tables;
 * row_bytes 4 = pg_cells_plan).  The fused training step reads its forward
 * levels from such a cache (pg_train_fused_ex_f32), rebuilt every step. */
int64_t pg_cells_plan_rows(const pg_grid *grid, int64_t budget_bytes, int row_bytes,
                           pg_cells *plan);
int pg_cells_build_f32(const pg_grid *grid, const float *feats, const uint8_t *baked,
                       const pg_cells *cells, void *stream);
/* pg_decode_f32 / pg_decode_host_f32 / pg_decode_host_stream_f32 reading the
 * cached levels from `cells` (NULL = none); every fused engine (tcgen05,
 * FFMA, exact reference order) uses it on fp16 tables. */
int pg_decode_cells_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs,
                        int64_t B, const void *feats, const uint8_t *baked,
                        const float *params, unsigned flags, const pg_cells *cells,
                        float *ws, float *out, void *stream);
int pg_decode_host_cells_f32(const pg_grid *grid, const pg_mlp *mlp,
                             const float *h_xs, int64_t B, const void *feats,
                             const uint8_t *baked, const float *params,
                             unsigned flags, const pg_cells *cells, int64_t chunk,
                             float *d_xs, float *d_out, float *h_out,
                             void *stream_in, void *stream_compute,
                             void *stream_out);
int pg_decode_host_stream_cells_f32(const pg_grid *grid, const pg_mlp *mlp,
                                    const float *h_xs, int64_t B, const void *feats,
                                    const uint8_t *baked, const float *params,
                                    unsigned flags, const pg_cells *cells, int64_t chunk,
                                    float *d_xs, float *d_out, uint32_t *d_flags,
                                    float *h_out, void *stream_in,
                                    void *stream_compute, void *stream_out);

/* Streaming end-to-end decode from HOST memory: one tcgen05 decode launch
 * over the whole batch consumes `chunk`-query pieces as
 * the copy engine lands them (flag written by the stream after each H2D
 * copy), and the D2H copy of each piece starts as soon as the kernel has
 * counted all of its tiles done (stream wait on a device counter).  chunk:
 * a power of two >= 128.  d_xs
 * holds B*d floats, d_out B*out_dim floats, d_flags 2*ceil(B/chunk) + 1
 * uint32 (per-chunk ready flags, per-chunk done counters, and in the last
 * slot the number of tile pipelines that took the host fallback below).
 * h_xs and h_out must be page-locked (checked; ValueError otherwise).
 * Needs the fused shape, the tensor-core MLP and stream memory operations:
 * pg_decode_stream_supported() says whether this call can run.  A chunk
 * whose flag has not arrived 2 ms after the kernel reached it (copies
 * serialised behind the kernel by a profiler or CUDA_LAUNCH_BLOCKING) is
 * read from h_xs directly (pinned, so device-accessible): never a hang. */
int pg_decode_stream_supported(const pg_grid *grid, const pg_mlp *mlp,
                               unsigned flags);
int pg_decode_host_stream_f32(const pg_grid *grid, const pg_mlp *mlp,
                              const float *h_xs, int64_t B, const void *feats,
                              const uint8_t *baked, const float *params,
                              unsigned flags, int64_t chunk, float *d_xs,
                              float *d_out, uint32_t *d_flags, float *h_out,
                              void *stream_in, void *stream_compute,
                              void *stream_out);

/* Zero-copy end-to-end decode: the tcgen05 decode kernel reads h_xs and
 * writes h_out in pinned host memory directly over PCIe (UVA); no copies,
 * flags or device buffers.
 * h_xs / h_out must be page-locked (checked).  Returns after completion. */
int pg_decode_host_zc_f32(const pg_grid *grid, const pg_mlp *mlp,
                          const float *h_xs, int64_t B, const void *feats,
                          const uint8_t *baked, const float *params,
                          unsigned flags, float *h_out, void *stream);

/* Training MLP pass (trainer.py:122-137 + mlp.py:55-85): forward, squared
 * error loss (sum in fp64 into *loss_sum), dpred = diff*scale, backward.
 * Accumulates parameter grads into gparams (same layout as params) and
 * writes dy (B, widths[0]).  targets (B, out_dim).  flags: PG_SIGMOID.
 * ws: pg_mlp_train_workspace_floats(B, mlp) floats (0 for the fast path). */
int64_t pg_mlp_train_workspace_floats(int64_t B, const pg_mlp *mlp);
int pg_mlp_train_f32(const pg_mlp *mlp, const float *y, const float *targets,
                     int64_t B, const float *params, float scale,
                     unsigned flags, float *gparams, float *dy,
                     double *loss_sum, float *ws, void *stream);
int pg_mlp_train_f64(const pg_mlp *mlp, const double *y, const double *targets,
                     int64_t B, const double *params, double scale,
                     unsigned flags, double *gparams, double *dy,
                     double *loss_sum, double *ws, void *stream);

/* Fused training pass (trainer.py:118-148): per 64-sample tile one kernel
 * runs encode fwd -> MLP fwd -> squared error -> MLP bwd -> encode bwd with
 * activations in shared memory.  Shape: F = 2, 16 levels, N_p <= 16, MLP
 * [32, 64, 64, out_dim <= 4].
 * Default: every MLP GEMM on tensor cores (mma.sync tf32, 3-term split,
 * fp32-level accuracy), the next tile's encode fwd fused with this tile's
 * encode bwd.  Table gradients (gfeat, gconf) are accumulated as
 * pg_encode_bwd does; touched[] is set only for lookups whose gconf
 * contribution is all zero/subnormal -- pg_lazy_adam_rebake_f32 also visits
 * every row with a non-zero gradient, which together is the reference's
 * touched set up to a row whose summed gradient cancels to exactly 0.0;
 * flags & PG_TOUCH_ALL sets touched[] for every lookup instead (what a
 * data-parallel step uses: the replicas' sums are added by the all-reduce).
 * flags & PG_EXACT_MLP: CUDA-core MLP in numpy/OpenBLAS's FMA-chain order, so
 * y, the loss terms and dL/dy equal the reference's bit for bit; touched[]
 * is set for every lookup.
 * loss_sum += sum of squared errors (fp64).  dy_out (optional, B x 32)
 * receives dL/dy for parity checks. */
int pg_train_fused_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs,
                       const float *targets, int64_t B, const float *feats,
                       const uint8_t *baked, const float *conf,
                       const float *params, float scale, unsigned flags,
                       float *gfeat, float *gconf, uint8_t *touched,
                       float *gparams, double *loss_sum, float *dy_out,
                       void *stream);
/* pg_train_fused_f32 with replicated feature-gradient tables: the fused
 * kernel's CTA b adds its feature gradients into copy b % reps of gfeat_rep
 * (reps x L x n_f x 2 floats, zero on entry, left zeroed), then one pass adds
 * the copies into gfeat.  Divides the same-address reduction traffic of
 * small tables by reps (reference default / C5 shapes); exact-MLP and
 * reference-order modes ignore it.  reps in [1, 256]. */
int pg_train_fused_rep_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs,
                           const float *targets, int64_t B, const float *feats,
                           const uint8_t *baked, const float *conf,
                           const float *params, float scale, unsigned flags,
                           float *gfeat, float *gconf, uint8_t *touched,
                           float *gparams, double *loss_sum, float *dy_out,
                           float *gfeat_rep, int reps, void *stream);
/* pg_train_fused_rep_f32 whose encode FORWARD reads the levels in `cells`
 * (an fp32 cell cache of these tables built by pg_cells_build_f32 for this
 * step; NULL = none): one 32-byte record per cached level and sample instead
 * of the dependent index and row gathers; identical values. */
int pg_train_fused_ex_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs,
                          const float *targets, int64_t B, const float *feats,
                          const uint8_t *baked, const float *conf,
                          const float *params, float scale, unsigned flags,
                          float *gfeat, float *gconf, uint8_t *touched,
                          float *gparams, double *loss_sum, float *dy_out,
                          float *gfeat_rep, int reps, const pg_cells *cells,
                          void *stream);

/* Standalone batched MLP, mlp.py:55-85 (mlp_forward / mlp_backward with an
 * arbitrary upstream gradient; ReLU hidden layers, linear output; numpy /
 * OpenBLAS operation order: each output an FMA chain over k from zero, the
 * bias a separate rounded add).  pg_mlp_forward: out (B, widths[-1]); ws
 * holds the hidden pre-activations, pg_mlp_train_workspace_floats(B, mlp)
 * floats.  pg_mlp_backward: re-runs the forward from x, then
 * gparams += parameter grads (params layout) for dL/d(out) = upstream
 * (B, widths[-1]) and writes dx (B, widths[0]). */
int pg_mlp_forward_f32(const pg_mlp *mlp, const float *x, int64_t B,
                       const float *params, float *ws, float *out, void *stream);
int pg_mlp_forward_f64(const pg_mlp *mlp, const double *x, int64_t B,
                       const double *params, double *ws, double *out, void *stream);
int pg_mlp_backward_f32(const pg_mlp *mlp, const float *x, int64_t B,
                        const float *params, const float *upstream,
                        float *gparams, float *dx, float *ws, void *stream);
int pg_mlp_backward_f64(const pg_mlp *mlp, const double *x, int64_t B,
                        const double *params, const double *upstream,
                        double *gparams, double *dx, double *ws, void *stream);

/* Output quantisation for PNG (pngio.py:34-41): out[i] = uint8(rint(clip(x[i],
 * 0, 1) * 255)) in float32 arithmetic, half-to-even (numpy on a float32 array). */
int pg_quantize_u8_f32(const float *x, int64_t n, uint8_t *out, void *stream);

/* Volume-compositing head (the reference has no
 * renderer, so these are checked against the numpy restatement in
 * oracle/oracle.py and finite differences).  raw (R*S, 4) = per-sample MLP
 * outputs (sigma_raw, r, g, b) of R rays x S samples in ray-major order;
 * sigma = softplus(sigma_raw), colour = logistic(rgb_raw),
 * alpha_i = 1 - exp(-sigma_i * deltas_i), T_i = prod_{j<i}(1 - alpha_j),
 * rgb = sum_i T_i alpha_i c_i.  weights (optional, R*S) = T_i alpha_i. */
int pg_composite_fwd_f32(const float *raw, const float *deltas, int64_t R,
                         int S, float *rgb, float *weights, void *stream);
/* S midpoint samples per ray inside [0,1]^3 (slab entry/exit; a ray that
 * misses gets zero-length segments): pts (R*S, 3) clamped to [0,1],
 * deltas (R*S) = segment length.  origins/dirs (R, 3). */
int pg_ray_samples_f32(const float *origins, const float *dirs, int64_t R,
                       int S, float *pts, float *deltas, void *stream);
/* pg_ray_samples_f32 plus the fused NeRF step's targets in one pass:
 * t4 (R*S, 4) = (segment length, target r, g, b) per sample (16-byte
 * aligned), rgb (R, 3) the rays' target colours. */
int pg_ray_samples_targets_f32(const float *origins, const float *dirs,
                               const float *rgb, int64_t R, int S, float *pts,
                               float *deltas, float *t4, void *stream);
/* NeRF-style training pass over R rays x S samples: y (R*S, widths[0]) are
 * the samples' encodings (pg_encode_fwd_f32); MLP forward (widths[-1] = 4),
 * compositing, loss = sum (rgb - target_rgb)^2 into *loss_sum (fp64),
 * dL/drgb = scale * (rgb - target), backward through compositing and the
 * MLP: gparams += parameter grads, dy (R*S, widths[0]) = dL/dy for
 * pg_encode_bwd_f32.  ws: pg_mlp_train_workspace_floats(R*S, mlp). */
int pg_nerf_train_f32(const pg_mlp *mlp, const float *y, const float *deltas,
                      const float *target_rgb, int64_t R, int S,
                      const float *params, float scale, float *gparams,
                      float *dy, double *loss_sum, float *ws, void *stream);

/* .cngp index blocks (model_io.py:150-165, FORMAT.md "Index block packing"):
 * n_rows blocks of n_c probe offsets at w = log2_np bits each, entry k in
 * bits [k*w, (k+1)*w) LSB-first within bytes, each block padded to
 * ceil(n_c*w/8) bytes.  Device pointers; exact integer transforms. */
int pg_unpack_indices(const uint8_t *packed, int64_t n_rows, int64_t n_c,
                      int log2_np, uint8_t *entries, void *stream);
int pg_pack_indices(const uint8_t *entries, int64_t n_rows, int64_t n_c,
                    int log2_np, uint8_t *packed, void *stream);

/* Pixel centres of the rectangle [x0, x0+w) x [y0, y0+h) of a width x height
 * image in raster order, (w*h, 2) floats on the device, bit-identical to
 * model_io.py:321-325 _grid_coords (decode_rect / decode_image input). */
int pg_raster_coords_f32(int x0, int y0, int w, int h, int width, int height,
                         float *xs, void *stream);

/* Reference-order MLP gradients (parity mode).  pg_train_fused_ref_f32 is
 * pg_train_fused_f32 except that it leaves gparams untouched and writes, per
 * sample, every layer's input and output delta to acts, laid out as
 * [a_0 | a_1 | .. | a_{n-1} | delta_0 | .. | delta_{n-1}], each block B rows
 * of its width (a_0 = y, a_l = relu activations, delta_l = dL/d(pre-activation
 * of layer l)), followed by the deltas again column-major (one contiguous
 * B-float column per output, for the in-order bias chains);
 * pg_mlp_acts_floats(B, mlp) floats (which include the scratch
 * pg_mlp_wgrad_blas_f32 uses after them).  pg_mlp_wgrad_blas_f32
 * then forms gparams += every weight and bias gradient in numpy/OpenBLAS
 * order (mlp.py:80-84): the sgemm K loop over samples is blocked by 448 (the
 * last two blocks balanced), each block one sequential FMA chain from 0,
 * blocks added in order; bias sums sequential over samples.  With the forward
 * already in OpenBLAS order this makes the MLP gradients bit-identical to the
 * reference's for out_dim >= 2 (out_dim 1 goes through sgemv there) and even
 * B >= 8192 (odd K and small products take other OpenBLAS paths:
 * rounding-level agreement only). */
int64_t pg_mlp_acts_floats(int64_t B, const pg_mlp *mlp);
int pg_train_fused_ref_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs,
                           const float *targets, int64_t B, const float *feats,
                           const uint8_t *baked, const float *conf,
                           const float *params, float scale, unsigned flags,
                           float *gfeat, float *gconf, uint8_t *touched,
                           double *loss_sum, float *acts, void *stream);
int pg_mlp_wgrad_blas_f32(const pg_mlp *mlp, const float *acts, int64_t B,
                          float *gparams, void *stream);
/* the same with the table gradients and the loss in 64-bit fixed point
 * (deterministic mode; flush with pg_fx_accumulate_f32 / pg_fx_loss) */
int pg_train_fused_ref_det_f32(const pg_grid *grid, const pg_mlp *mlp, const float *xs,
                               const float *targets, int64_t B, const float *feats,
                               const uint8_t *baked, const float *conf,
                               const float *params, float scale, unsigned flags,
                               uint64_t *gfeat_fx, uint64_t *gconf_fx, uint8_t *touched,
                               uint64_t *loss_fx, float *acts, void *stream);

/* Deterministic mode.  Same passes as pg_encode_bwd_f32 / pg_mlp_train_f32 /
 * pg_train_fused_f32, but every cross-thread sum (table scatters, weight
 * gradients, the loss) is accumulated in 64-bit fixed point (2^-56 for
 * gradients, range +-128; 2^-32 for the loss), which is order-independent:
 * results are bit-identical run to run, and identical contributions give
 * identical sums (the reference's N_p=1 probed == plain-hash equivalence,
 * test_trainer.py:131-141).  Accumulators (uint64, zeroed by the caller the
 * first time) use the float buffers' element layout; pg_fx_accumulate_f32
 * adds them into the float gradients and clears them, pg_fx_loss converts
 * the loss accumulator. */
int pg_encode_bwd_det_f32(const pg_grid *grid, const float *xs, int64_t B,
                          const float *dy, const float *feats,
                          const float *conf, uint64_t *gfeat_fx,
                          uint64_t *gconf_fx, uint8_t *touched, void *stream);
int pg_mlp_train_det_f32(const pg_mlp *mlp, const float *y,
                         const float *targets, int64_t B, const float *params,
                         float scale, unsigned flags, uint64_t *gparams_fx,
                         float *dy, uint64_t *loss_fx, float *ws, void *stream);
int pg_train_fused_det_f32(const pg_grid *grid, const pg_mlp *mlp,
                           const float *xs, const float *targets, int64_t B,
                           const float *feats, const uint8_t *baked,
                           const float *conf, const float *params, float scale,
                           unsigned flags, uint64_t *gfeat_fx,
                           uint64_t *gconf_fx, uint8_t *touched,
                           uint64_t *gparams_fx, uint64_t *loss_fx,
                           float *dy_out, void *stream);
int pg_fx_accumulate_f32(uint64_t *fx, int64_t n, float *dst, void *stream);
int pg_fx_loss(uint64_t *fx, double *loss_sum, void *stream);

/* Pixel batch for the image trainer (trainer.py:109-116): xs from pixel
 * indices pix (host-drawn for reference parity, or drawn on device from
 * (seed, step) when pix_in is NULL and pix_out receives them), targets
 * gathered from the HxWxC image. */
int pg_pixel_batch_f32(const int64_t *pix_in, int64_t B, int width,
                       int height, const float *image, int channels,
                       uint64_t seed, uint64_t step, int64_t *pix_out,
                       float *xs, float *targets, void *stream);
int pg_pixel_batch_f64(const int64_t *pix_in, int64_t B, int width,
                       int height, const double *image, int channels,
                       uint64_t seed, uint64_t step, int64_t *pix_out,
                       double *xs, double *targets, void *stream);

/* trainer.adam_update (trainer.py:73-84) over one flat buffer, reference
 * rounding order; zeroes grad afterwards (trainer.py:157-161).
 * d_guard (optional): when *d_guard is not finite (a diverged loss,
 * trainer.py:130-132) the update is skipped and only the gradient cleared. */
int pg_adam_f32(float *param, float *grad, float *m, float *v, int64_t n,
                int64_t t, double lr, double beta1, double beta2, double eps,
                const double *d_guard, void *stream);
int pg_adam_f64(double *param, double *grad, double *m, double *v, int64_t n,
                int64_t t, double lr, double beta1, double beta2, double eps,
                const double *d_guard, void *stream);

/* Lazy Adam + incremental re-bake over every confidence row whose touched
 * flag is set or whose gradient row is non-zero (trainer.py:162-167 with
 * _core.pyx:224-272 arithmetic), then clears that row's gradient and flag.
 * rows = n_probed*n_c. */
int pg_lazy_adam_rebake_f32(float *conf, float *m, float *v, uint8_t *baked,
                            float *gconf, uint8_t *touched, int64_t rows,
                            int n_p, int64_t t, double lr, double beta1,
                            double beta2, double eps, const double *d_guard,
                            void *stream);
int pg_lazy_adam_rebake_f64(double *conf, double *m, double *v,
                            uint8_t *baked, double *gconf, uint8_t *touched,
                            int64_t rows, int n_p, int64_t t, double lr,
                            double beta1, double beta2, double eps,
                            const double *d_guard, void *stream);

/* Full bake of `rows` confidence rows into baked indices: codebooks.py:147-152
 * (np.argmax per row: first maximum, first NaN if any).  Replaces the
 * reference's `bake` in init_model (model.py:150-156) and
 * TrainState.check_bake_consistency (trainer.py:173-180). */
int pg_bake_rows_f32(const float *conf, int64_t rows, int n_p, uint8_t *baked,
                     void *stream);
int pg_bake_rows_f64(const double *conf, int64_t rows, int n_p, uint8_t *baked,
                     void *stream);

/* touched flags as counts in the exchange buffer's element type (for the
 * data-parallel allreduce: a float64 model's buffer holds doubles) and back
 * (count > 0 -> touched: the union over replicas) */
int pg_touched_to_f32(const uint8_t *touched, int64_t n, float *out,
                      void *stream);
int pg_touched_from_f32(const float *in, int64_t n, uint8_t *touched,
                        void *stream);
int pg_touched_to_f64(const uint8_t *touched, int64_t n, double *out,
                      void *stream);
int pg_touched_from_f64(const double *in, int64_t n, uint8_t *touched,
                        void *stream);

/* Self-test of the tcgen05 (UMMA) path: one CTA computes
 * D[128x64] = A[128x32] . B[64x32]^T with kind::tf32 MMA into TMEM;
 * split != 0 uses the 2-term hi/lo expansion of A. */
int pg_selftest_umma_tf32(const float *A, const float *B, float *D, int split,
                          void *stream);

/* Roofline probes (bench.py): L2 streaming read of `bytes` from buf, `reps`
 * times; `nq` random 8-byte gathers from a table of entries_pow2 float2. */
int pg_probe_stream_read(const void *buf, int64_t bytes, int reps, float *sink,
                         void *stream);
int pg_probe_gather(const void *table, int64_t entries_pow2, int64_t nq,
                    uint32_t seed, float *sink, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* PROBEGRID_B200_H */
