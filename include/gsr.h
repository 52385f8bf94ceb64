/* gsr.h -- C ABI of the B200-native GSFusion rasterizer hot path (libgsr.so).
 *
 * GSFusion (arXiv 2408.12677) optimises 3D Gaussians online with "a tile-based
 * rasterizer which divides the screen into multiple tiles.  3D Gaussians lying in
 * the current view frustum are sorted based on depth in each tile" (PAPER.md:139,
 * §III-B3), renders Eq. 11, minimises Eq. 12 with "explicitly
 * derived" gradients and updates every parameter by a
 * first-order method.  The five calls below are that problem
 * statement, one call per step (BASELINE.json north_star):
 *
 *   gs_project    Eqs. 2, 4, 5 + SH colour
 *   gs_bin_tiles  per-tile depth sort
 *   gs_render_fwd Eq. 11 + depth channel
 *   gs_render_bwd dEq.11 -> dEq.5/4/2
 *   gs_adam_step  first-order update          (Adam per north_star)
 *
 * plus the harness call gs_l1_loss_grad (Eq. 12) and diagnostics.
 *
 * CONVENTIONS (apply to every call)
 *  - Pointers are DEVICE pointers unless marked HOST.  Every buffer is allocated and
 *    owned by the caller; the library never allocates, frees or retains device
 *    memory and keeps no state between calls except a process-wide launch counter.
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*; NULL =
 *    the legacy default stream).  The only exception is gs_bin_tiles with a non-NULL
 *    num_keys_host, which synchronises `stream` to report the key count.
 *  - Float buffers used with 128-bit access must be 16-byte aligned and P_stride must
 *    be a multiple of 4; violations return GS_ERR_ALIGN before anything is launched.
 *  - Errors: every call returns a gs_status; no C++ exception crosses the ABI.
 *    Argument errors are detected on the host before any launch.  A failed kernel
 *    launch returns GS_ERR_CUDA; gs_last_error() then holds a thread-local message.
 *    Culling is not an error: a culled Gaussian gets radius = tiles = 0 and exactly
 *    zero gradient (readings R6, R23 in DESIGN.md).
 *  - Precision: fp32 everywhere (R25).  All calls are re-entrant.
 *  - The camera model, parameter layout and every reading (R1-R27) are documented
 *    in DESIGN.md; the readings are frozen and shared with the CPU oracle's tests.
 */
#ifndef GSR_H_
#define GSR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSR_VERSION 2
#define GS_TILE 16         /* 16x16-pixel tiles (north_star) */
#define GS_MAX_SH_DEGREE 3
#define GS_MAX_TILES 65536 /* tile ids are sorted as 16-bit keys */
#define GS_REC_FLOATS 12   /* floats per projected-Gaussian record */
#define GS_SGRAD_FLOATS 12 /* floats per Gaussian in the render_bwd workspace */

typedef enum {
  GS_OK = 0,
  GS_ERR_ARG = -1,      /* invalid argument (NULL, negative size, bad degree, ...) */
  GS_ERR_ALIGN = -2,    /* pointer not 16-byte aligned or P_stride % 4 != 0 */
  GS_ERR_CAPACITY = -3, /* gs_bin_tiles: K > key_capacity (required K reported) */
  GS_ERR_STATE = -4,    /* backward given buffers / sizes of another forward (SPEC StateMismatch) */
  GS_ERR_EMPTY = -5,    /* gs_adam_step with P == 0 (SPEC NoGaussians) */
  GS_ERR_CUDA = -6      /* a CUDA launch or runtime call failed; see gs_last_error() */
} gs_status;

/* Pinhole camera, OpenCV axes (x right, y down, z forward).  R_cw/t_cw map world to
 * camera: the rotation W and translation of T_WC^{-1}, row-major.
 * Pixel (i, j) is sampled at continuous (i, j) (R1).  Gaussians with camera-space
 * z <= z_near are culled (R6).  bg is the background colour (R26). */
typedef struct {
  int32_t width, height;
  float fx, fy, cx, cy;
  float R_cw[9];
  float t_cw[3];
  float z_near;
  float bg[3];
} gs_camera;

/* Parameters: float[F][P_stride], F = 11 + 3(deg+1)^2 rows (R3-R5):
 *   rows 0-2 mean xyz (m) | 3-5 log-scale | 6-9 quaternion (w,x,y,z), need not be unit
 *   10 opacity logit       | 11 + 3k + ch  SH coefficient k (k = 0 is DC), channel ch.
 * The same layout is used for grad, Adam's m and v.  Columns >= P are never read. */
typedef struct {
  int64_t P;
  int64_t P_stride;
  int32_t sh_degree; /* 0..3 */
} gs_scene;

/* Per-view projection outputs (written by gs_project, read by every later call).
 *  rec:    float[P][12] records, 48 B each (16-B aligned):
 *            0 mu_x  1 mu_y  2 z  3 opacity  4 conic A  5 conic B  6 conic C
 *            7 r  8 g  9 b  10-11 reserved
 *          conic (A, B, C) is Sigma_hat^{-1} = [[A, B], [B, C]] (Eq. 3).  Records of
 *          culled Gaussians are left untouched (undefined).
 *  radius: int32[P]  ceil(3 sqrt(lambda_max)) in pixels, 0 = culled (R10)
 *  tiles:  int32[P]  number of 16x16 tiles touched, 0 = culled (R11)
 *  flags:  uint8[P]  bit0-2 colour channel clamped at 0 (R13), bit3/4 J x/y tangent
 *                    clamp active (R7), bit7 culled */
typedef struct {
  float* rec;
  int32_t* radius;
  int32_t* tiles;
  uint8_t* flags;
} gs_proj;

#define GS_FLAG_CLAMP_R 1
#define GS_FLAG_CLAMP_G 2
#define GS_FLAG_CLAMP_B 4
#define GS_FLAG_JCLAMP_X 8
#define GS_FLAG_JCLAMP_Y 16
#define GS_FLAG_CULLED 128

/* ---------------------------------------------------------------- diagnostics */
int gs_version(void);
const char* gs_last_error(void);  /* thread-local text of the last failure ("" if none) */
int64_t gs_launch_count(void);    /* kernels launched by this library (process-wide) */
/* Performance switch of gs_render_fwd / gs_render_bwd_screen(_l1) (process-wide, read at
 * each launch; results are identical either way, tests/test_gpu_keymask.py):
 * 0 (default) = each key evaluates all four 8x4-block rows of its tile, straight-line;
 * 1 = each key visits only the block rows its block mask touches (a warp-uniform branch
 * per row): faster for scenes of small Gaussians (config 4: step 76.5 -> 73.6 ms), slower
 * for large ones (scannetpp +2%).  pipeline.Trainer.autotune_render picks it per scene by
 * timing both.  Only the default one-warp-per-CTA kernels have the row walk. */
gs_status gs_set_render_rows(int enable);
int gs_render_rows(void);
int gs_exact_exp(void);           /* 1 in the GSR_EXACT_EXP debug build (libgsr_exact.so) */

/* ---------------------------------------------------------------- gs_project
 * Steps O1-O8: activations (R3-R5, R9), Sigma = R S S^T R^T (Eq. 2),
 * p_c = W p + t and mu = pi(p_c) (Eq. 4), Sigma_hat = J W Sigma W^T J^T + 0.3 I
 * (Eq. 5, R7, R8), conic, 3-sigma radius and tile rectangle (R10, R11), SH colour
 * at the mean (R13).  In: params (see gs_scene).  Out: `out` (see gs_proj).
 * Integer outputs and mu, z, conic, opacity are computed with a fixed fp32
 * operation order (R9) and match the oracle bit for bit.
 * P == 0 is valid (nothing launched). */
gs_status gs_project(const gs_camera* cam /*HOST*/, const gs_scene* scene /*HOST*/, const float* params,
                     gs_proj out, void* stream);

/* gs_project for n_views cameras in one pass over the parameters (the projection of a
 * batch of views, R21): outs[v] receives exactly what gs_project(&cams[v], ...) would
 * write (bit-identical: the per-view arithmetic is the same), but the parameter rows
 * are read once per batch of up to 8 views instead of once per view.  cams, outs:
 * HOST arrays of n_views.  Errors as gs_project (per camera and output). */
gs_status gs_project_views(int n_views, const gs_camera* cams /*HOST[n_views]*/, const gs_scene* scene /*HOST*/,
                           const float* params, const gs_proj* outs /*HOST[n_views]*/, void* stream);

/* ---------------------------------------------------------------- gs_bin_tiles
 * Duplicates every visible Gaussian into one key per touched tile and orders the
 * keys by (tile id = ty * tiles_x + tx, depth z, Gaussian index) (R12):
 * an order-preserving compaction of the visible set, a 4-pass onesweep LSD radix
 * sort of the depths, key emission in depth order, and a 1-2-pass onesweep radix
 * sort of the 16-bit tile ids.
 *  ws / ws_bytes:   scratch of at least gs_bin_tiles_workspace() bytes (16-B aligned)
 *  sorted_ids:      int32[key_capacity] Gaussian index of each sorted key
 *  tile_ranges:     int32[num_tiles][2] [start, end) of each tile's keys
 *  num_keys_dev:    nullable DEVICE int64: receives K asynchronously
 *  num_keys_host:   nullable HOST int64: if set, the call synchronises `stream`
 *                   and writes K; returns GS_ERR_CAPACITY if K > key_capacity
 * If K > key_capacity no key is written past key_capacity and every tile range is
 * empty (renders give background); in async mode the caller detects this from
 * num_keys_dev and retries with a larger buffer.  num_tiles must be <= 65536. */
size_t gs_bin_tiles_workspace(const gs_camera* cam /*HOST*/, int64_t P, int64_t key_capacity);
gs_status gs_bin_tiles(const gs_camera* cam /*HOST*/, const gs_scene* scene /*HOST*/, gs_proj proj, void* ws,
                       size_t ws_bytes, int64_t key_capacity, int32_t* sorted_ids, int32_t* tile_ranges,
                       int64_t* num_keys_dev, int64_t* num_keys_host /*HOST*/, void* stream);

/* ---------------------------------------------------------------- gs_tile_order
 * Scheduling order of the tiles for the render calls: the tile ids sorted by
 * decreasing key count (min(count, 4095) / 4 buckets; order inside a bucket is
 * unspecified), so that the longest tiles start first and the short ones fill the
 * tail (longest-processing-time-first).  Not a step of the method: a work order.
 *  tile_ranges: int32[num_tiles][2] from gs_bin_tiles (same stream)
 *  tile_order:  int32[num_tiles] output permutation.  num_tiles <= 65536. */
gs_status gs_tile_order(const gs_camera* cam /*HOST*/, const int32_t* tile_ranges, int32_t* tile_order, void* stream);

/* ---------------------------------------------------------------- forward state
 * What a backward consumes from its forward (SPEC.md:345-353 render_backward ->
 * StateMismatch): gs_render_fwd fills a caller-owned HOST gs_fwd_state (fwd_out) with a
 * process-unique id and the buffers and image size it used, and records, in a small
 * process-wide table keyed by the n_contrib buffer, which forward call wrote that
 * buffer last.  A backward given that state (gs_bwd_opts.fwd) returns GS_ERR_STATE,
 * launching nothing, if
 *   - its camera's width / height differ from the forward's,
 *   - any of proj.rec, sorted_ids, tile_ranges, T_final, n_contrib (and key_blocks,
 *     when the backward uses masks; rgb and depth for the fused-loss backward) is not
 *     the buffer that forward used (e.g. the key masks or n_contrib of another view), or
 *   - a later gs_render_fwd has rewritten n_contrib (the state is stale).
 * Checks run on the host at call (or graph-capture) time; NULL skips them. */
typedef struct {
  uint64_t id; /* never 0 once written */
  int32_t width, height;
  const float* rec;
  const int32_t* sorted_ids;
  const int32_t* tile_ranges;
  const float* rgb;
  const float* depth;
  const float* T_final;
  const int32_t* n_contrib;
  const uint8_t* key_blocks;
} gs_fwd_state;

/* Options of the backward calls (nullable pointer = all defaults):
 *  fwd:      the forward's state (above): consistency check -> GS_ERR_STATE.
 *  det_ws:   non-NULL selects the DETERMINISTIC reduction mode: every
 *            (tile, Gaussian) pair's warp-reduced 10 screen-gradient components are
 *            stored to det_ws[key][12] (no atomics), then one thread per Gaussian sums
 *            its pairs in a fixed order (the tiles of its rectangle, row-major) into
 *            sgrad.  Results are then bit-reproducible: independent of scheduling,
 *            streams, graph replay and tile_order.  det_ws: DEVICE float[det_keys][12],
 *            16-B aligned; det_keys >= the key_capacity given to gs_bin_tiles.  Costs
 *            48 B per key of traffic and one binary search per key (a test mode).
 *            The K13 port (gs_naive_render_bwd_screen) rejects it (GS_ERR_ARG). */
typedef struct {
  const gs_fwd_state* fwd;
  float* det_ws;
  int64_t det_keys;
} gs_bwd_opts;

/* ---------------------------------------------------------------- gs_render_fwd
 * Eq. 11 per pixel over its tile's depth-sorted list, front to back: alpha =
 * min(0.99, o exp(power)), skip alpha < 1/255 (and power > 0), stop before a
 * Gaussian that would take T below 1e-4 (R15, R16, R27); C += c alpha T,
 * D += z alpha T (R17); finally C += T bg.
 *  rgb: float[3][H][W]   depth, T_final: float[H][W]   n_contrib: int32[H][W]
 *       (1 + position in the tile list of the last composited Gaussian, 0 if none)
 *  blended: nullable u64 counter, += number of composited (pixel, Gaussian) pairs.
 *  key_blocks: nullable uint8[key_capacity]: for every sorted key the forward
 *       visited, the mask of its tile's 8x4 pixel blocks (bit b: x offset 8 (b & 1),
 *       y offset 4 (b >> 1)) in which that Gaussian was composited into >= 1 pixel.
 *       Passing it to the backward lets it skip (tile, Gaussian) pairs that
 *       contributed nothing (an exact property of this forward pass).
 *  tile_order: nullable int32[num_tiles], a permutation of the tile ids: the order in
 *       which tiles are scheduled (gs_tile_order).  Results do not depend on it. */
gs_status gs_render_fwd(const gs_camera* cam /*HOST*/, const gs_scene* scene /*HOST*/, gs_proj proj,
                        const int32_t* sorted_ids, const int32_t* tile_ranges, const int32_t* tile_order /*nullable*/,
                        float* rgb, float* depth,
                        float* T_final, int32_t* n_contrib, unsigned long long* blended, uint8_t* key_blocks,
                        gs_fwd_state* fwd_out /*HOST, nullable*/, void* stream);

/* ---------------------------------------------------------------- gs_render_bwd
 * Exact derivative of gs_project + gs_render_fwd (R18) for upstream
 * dL/drgb float[3][H][W] and dL/ddepth float[H][W] (nullable = 0).  Consumes the
 * forward's T_final and n_contrib (it does not re-render).  Reverses each pixel's
 * composite per tile, reduces per-Gaussian screen-space gradients across each warp
 * and scatters them with one atomic per (warp, Gaussian, component), then chains
 * them to every parameter row.
 *  ws: float[P][12] screen-space gradients (dmu_x, dmu_y, dA, dB, dC, dopacity,
 *      dr, dg, db, dz, pad, pad); >= gs_render_bwd_workspace() bytes; cleared here.
 *  key_blocks: nullable, the forward's key masks for the SAME forward call (see
 *      gs_render_fwd); NULL = derive the pixel blocks geometrically.
 *  tile_order: nullable, as in gs_render_fwd.
 *  grad: float[F][P_stride], ACCUMULATED (+=) so that views sum (R21).
 *  opts: nullable gs_bwd_opts (forward-state check -> GS_ERR_STATE; deterministic mode).
 * Float atomics make grad order-dependent in the last bits unless opts->det_ws is set. */
size_t gs_render_bwd_workspace(const gs_scene* scene /*HOST*/);
gs_status gs_render_bwd(const gs_camera* cam /*HOST*/, const gs_scene* scene /*HOST*/, const float* params,
                        gs_proj proj, const int32_t* sorted_ids, const int32_t* tile_ranges,
                        const int32_t* tile_order /*nullable*/, const float* T_final,
                        const int32_t* n_contrib, const float* dL_drgb, const float* dL_ddepth,
                        const uint8_t* key_blocks /*nullable*/, void* ws, size_t ws_bytes, float* grad,
                        const gs_bwd_opts* opts /*HOST, nullable*/, void* stream);

/* ---------------------------------------------------------------- batched backward
 * gs_render_bwd split in its two halves so that a batch of views (R21) chains the
 * projection backward ONCE per up to 8 views instead of once per view:
 *
 *  gs_render_bwd_screen: the raster half of gs_render_bwd for one view.  Accumulates
 *    (+=) the view's screen-space gradients into sgrad float[P][12] (layout of the
 *    gs_render_bwd workspace).  sgrad must be zero at every visible Gaussian's entry
 *    before the first call (cudaMemset once at allocation); gs_project_bwd_views
 *    leaves it zero again.
 *  gs_project_bwd_views: grad += sum over the n_views views of d(projection_v)^T sgrad_v
 *    (exact derivative of gs_project, R18).  cams: HOST array of n_views cameras;
 *    flags: HOST array of n_views DEVICE pointers to each view's gs_proj.flags (uint8[P],
 *    as written by gs_project for that view); sgrads: HOST array of n_views DEVICE
 *    pointers to float[P][12].  Each params row is read and each grad row updated once
 *    per call for up to 64 views (<= 8 views: unrolled per-view registers; more: the
 *    views in the inner loop of each Gaussian); every consumed sgrad entry is reset to
 *    zero (floats 10-11 of the first view's records, unused by the render backward,
 *    carry the wide pass's per-Gaussian visibility mask between its two kernels and
 *    are zero again on return; the n_views buffers must be distinct).  accumulate != 0:
 *    grad += the batch's gradient; accumulate == 0: grad := the batch's gradient
 *    (every row of every Gaussian written, none read -- the first batch of an
 *    iteration, so that the optimiser need not zero grad). */
gs_status gs_render_bwd_screen(const gs_camera* cam /*HOST*/, const gs_scene* scene /*HOST*/, gs_proj proj,
                               const int32_t* sorted_ids, const int32_t* tile_ranges,
                               const int32_t* tile_order /*nullable*/, const float* T_final,
                               const int32_t* n_contrib, const float* dL_drgb, const float* dL_ddepth,
                               const uint8_t* key_blocks /*nullable*/, float* sgrad,
                               const gs_bwd_opts* opts /*HOST, nullable*/, void* stream);
gs_status gs_project_bwd_views(int n_views, const gs_camera* cams /*HOST[n_views]*/, const gs_scene* scene /*HOST*/,
                               const float* params, const uint8_t* const* flags /*HOST[n_views] of DEVICE*/,
                               float* const* sgrads /*HOST[n_views] of DEVICE*/, float* grad, int accumulate,
                               void* stream);

/* The end of one optimisation iteration (the explicitly derived
 * gradient, then the first-order update; Adam per north_star, R20):
 * gs_project_bwd_views (overwrite when accumulate == 0) followed by gs_adam_step_dev's
 * update of every row (step counter *step_dev advanced once, first; grad not zeroed),
 * with the optimiser split at the geometry / SH-row boundary: the SH rows (11..F-1,
 * final once the chain's colour half has run) are updated on `side_stream` while the
 * geometry half of the chain runs on `stream`, then rows 0..10 on `stream`, which
 * finally waits for the side stream.  Same results as gs_project_bwd_views +
 * gs_adam_step_dev (Adam is element-wise); graph-capturable (the side stream forks from
 * and joins `stream`).  side_stream NULL: no split.  Not thread-safe (two library-owned
 * events).  n_views >= 1; params, m, v, grad: the model's full [F][P_stride] arrays.
 * Errors: GS_ERR_ARG (NULL array, n_views < 1, step_dev NULL, betas outside [0, 1)),
 * GS_ERR_ALIGN (an sgrad not 16-byte aligned), as gs_project_bwd_views otherwise. */
gs_status gs_project_bwd_views_adam_dev(int n_views, const gs_camera* cams /*HOST[n_views]*/,
                                        const gs_scene* scene /*HOST*/, float* params,
                                        const uint8_t* const* flags /*HOST[n_views] of DEVICE*/,
                                        float* const* sgrads /*HOST[n_views] of DEVICE*/, float* grad, int accumulate,
                                        float* m, float* v, const float* lr_per_row /*HOST*/, float beta1,
                                        float beta2, float eps, int64_t* step_dev, void* stream, void* side_stream);

/* ---------------------------------------------------------------- K13 comparison baseline
 * The "straightforward per-pixel GPU port" the north_star's >= 10x target is measured
 * against (BASELINE.json north_star).  NOT the product path: drop-in
 * replacements of gs_render_fwd (without key_blocks) and gs_render_bwd_screen with the
 * same arguments, layouts, outputs and error behaviour, computed by one thread per
 * pixel that reads every Gaussian record from global memory (no shared-memory staging,
 * no warp cooperation) and, in the backward, issues 10 atomicAdd per composited
 * (pixel, Gaussian) pair.  Results equal the product calls up to fp32 rounding. */
gs_status gs_naive_render_fwd(const gs_camera* cam /*HOST*/, const gs_scene* scene /*HOST*/, gs_proj proj,
                              const int32_t* sorted_ids, const int32_t* tile_ranges, float* rgb, float* depth,
                              float* T_final, int32_t* n_contrib, unsigned long long* blended,
                              gs_fwd_state* fwd_out /*HOST, nullable*/, void* stream);
gs_status gs_naive_render_bwd_screen(const gs_camera* cam /*HOST*/, const gs_scene* scene /*HOST*/, gs_proj proj,
                                     const int32_t* sorted_ids, const int32_t* tile_ranges, const float* T_final,
                                     const int32_t* n_contrib, const float* dL_drgb, const float* dL_ddepth,
                                     float* sgrad, const gs_bwd_opts* opts /*HOST, nullable*/, void* stream);

/* gs_render_bwd_screen with the harness loss of Eq. 12 fused in: the upstream gradient
 * of every pixel is computed inside the backward from the rendered rgb / depth (as
 * written by gs_render_fwd) and the target images, with exactly the values
 * gs_l1_loss_grad writes (sign(residual) / (3 npix) per colour channel, w_depth
 * sign / npix for depth, sign(0) = 0, invalid target samples masked as there, R43),
 * and the loss (nullable DEVICE float) += L.
 * One kernel instead of gs_l1_loss_grad + gs_render_bwd_screen; no dL/d-image buffers.
 * P == 0 is valid (background-only images; the loss is still accumulated). */
gs_status gs_render_bwd_screen_l1(const gs_camera* cam /*HOST*/, const gs_scene* scene /*HOST*/, gs_proj proj,
                                  const int32_t* sorted_ids, const int32_t* tile_ranges,
                                  const int32_t* tile_order /*nullable*/, const float* T_final,
                                  const int32_t* n_contrib, const float* rgb, const float* depth,
                                  const float* target_rgb, const float* target_depth, float w_depth,
                                  float* loss /*nullable*/, const uint8_t* key_blocks /*nullable*/, float* sgrad,
                                  const gs_bwd_opts* opts /*HOST, nullable*/, void* stream);

/* ---------------------------------------------------------------- gs_adam_step
 * Dense bias-corrected Adam over all F x P scalars of the live Gaussians [0, P) (R20;
 * columns P..P_stride-1, the room a growing map has left, are not touched):
 *   m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2;
 *   p -= lr_row * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)
 *  lr_per_row: HOST float[F].  step: 1-based t.  zero_grad != 0 also writes grad = 0.
 *  Returns GS_ERR_EMPTY if P == 0. */
gs_status gs_adam_step(const gs_scene* scene /*HOST*/, float* params, float* grad, float* m, float* v,
                       const float* lr_per_row /*HOST*/, float beta1, float beta2, float eps, int64_t step,
                       int zero_grad, void* stream);

/* gs_adam_step with the 1-based step counter in DEVICE memory: *step_dev (int64) is
 * incremented on the stream first and the bias corrections are computed from it on
 * the device, so the call can be captured in a CUDA graph and replayed (bench.py's
 * graph mode).  On entry *step_dev = t - 1. */
gs_status gs_adam_step_dev(const gs_scene* scene /*HOST*/, float* params, float* grad, float* m, float* v,
                           const float* lr_per_row /*HOST*/, float beta1, float beta2, float eps, int64_t* step_dev,
                           int zero_grad, void* stream);

/* gs_adam_step restricted to the scalars [begin, end) of the flattened [F][P_stride]
 * arrays (row r = index / P_stride keeps its learning rate): the optimiser half of a
 * reduce-scatter -> sharded Adam -> all-gather step across ranks (SURVEY.md §8(f)
 * NEXT-2).  params, m, v: the FULL arrays (only the range is read or
 * written); grad_range: float[end - begin], the (reduce-scattered) gradient of the
 * range.  begin and end must be multiples of 4 (GS_ERR_ALIGN).  The gradient is not
 * zeroed.  Same hyper-parameters and update as gs_adam_step. */
gs_status gs_adam_step_range(const gs_scene* scene /*HOST*/, float* params, const float* grad_range, float* m, float* v,
                             const float* lr_per_row /*HOST*/, float beta1, float beta2, float eps, int64_t step,
                             int64_t begin, int64_t end, void* stream);

/* gs_adam_step_range with the 1-based step counter in DEVICE memory (as gs_adam_step_dev:
 * *step_dev is incremented on the stream first; graph-capturable).  Every rank calls it,
 * also one whose range is empty (it then only advances its counter). */
gs_status gs_adam_step_range_dev(const gs_scene* scene /*HOST*/, float* params, const float* grad_range, float* m,
                                 float* v, const float* lr_per_row /*HOST*/, float beta1, float beta2, float eps,
                                 int64_t* step_dev, int64_t begin, int64_t end, void* stream);

/* Reduce-scatter + Adam + all-gather fused in ONE kernel over peer memory (SURVEY.md
 * §8(f) NEXT-2): for the scalars [begin, end) this rank owns, sum every rank's
 * gradient (P2P loads over NVLink from grad_peers[0..world-1], in rank order), apply
 * Adam to the local m, v and param_peers[rank], and store the new parameters into
 * every rank's param_peers[r] (P2P stores).  grad_peers / param_peers: HOST arrays of
 * world DEVICE pointers to each rank's full [F][P_stride] buffers (symmetric memory
 * mapped into this process); m, v: this rank's full arrays (only the range is
 * touched).  world <= 8; begin, end multiples of 4.  The caller must order the ranks
 * around the call (all gradients final before, all parameter stores done after),
 * e.g. with a symmetric-memory barrier on the same stream. */
gs_status gs_adam_step_peers(const gs_scene* scene /*HOST*/, int world, int rank,
                             const float* const* grad_peers /*HOST[world]*/, float* const* param_peers /*HOST[world]*/,
                             float* m, float* v, const float* lr_per_row /*HOST*/, float beta1, float beta2, float eps,
                             int64_t step, int64_t begin, int64_t end, void* stream);
/* gs_adam_step_peers with the step counter in DEVICE memory (*step_dev incremented first;
 * graph-capturable, so the multi-GPU iteration replays as one CUDA graph per rank). */
gs_status gs_adam_step_peers_dev(const gs_scene* scene /*HOST*/, int world, int rank,
                                 const float* const* grad_peers /*HOST[world]*/, float* const* param_peers /*HOST[world]*/,
                                 float* m, float* v, const float* lr_per_row /*HOST*/, float beta1, float beta2,
                                 float eps, int64_t* step_dev, int64_t begin, int64_t end, void* stream);

/* The same step with the reduction and the broadcast done by the NVSwitch (NVLS,
 * SURVEY.md §8(f) NEXT-2): for the scalars [begin, end) this rank owns, one
 * multimem.ld_reduce (add, fp32) on the MULTICAST address of the symmetric gradient
 * buffer returns the sum over all ranks, Adam updates the local m, v and this rank's
 * parameter copy `param` (read only), and one multimem.st on the MULTICAST address of
 * the symmetric parameter buffer writes the new values into every rank's copy.
 *  mc_grad, mc_param: DEVICE multicast addresses (e.g. torch symmetric memory's
 *  multicast_ptr, which exists only on NVSwitch systems with multicast support);
 *  param: this rank's unicast view of the parameter buffer.
 *  step_dev: nullable DEVICE int64; non-NULL: the step counter on the device
 *  (incremented first, as gs_adam_step_dev), else `step` (>= 1).
 * The caller orders the ranks around the call as for gs_adam_step_peers.  begin, end
 * multiples of 4 (GS_ERR_ALIGN). */
gs_status gs_adam_step_multimem(const gs_scene* scene /*HOST*/, const float* mc_grad, float* mc_param,
                                const float* param, float* m, float* v, const float* lr_per_row /*HOST*/, float beta1,
                                float beta2, float eps, int64_t step, int64_t* step_dev, int64_t begin, int64_t end,
                                void* stream);

/* ---------------------------------------------------------------- visibility-sparse exchange/* ---------------------------------------------------------------- visibility-sparse exchange
 * (SURVEY.md §8(f) NEXT-2 "visibility-sparse gradient exchange: union of visible masks,
 * then compaction").  A Gaussian culled in every view of every rank has
 * an exactly zero gradient on every rank, so only the columns of the union of the
 * ranks' visible sets need to cross the wire:
 *   gs_visibility_union: visible[i] = 1 if flags[v][i] lacks GS_FLAG_CULLED for some
 *     v < n_views, else 0; accumulate != 0 ORs into the existing visible[i] instead
 *     (flags: HOST array of n_views DEVICE uint8[P], gs_project's flags; visible:
 *     DEVICE uint8[P]).  The ranks then combine their masks (an all-reduce MAX of P
 *     bytes).
 *   gs_compact_index: idx[0..M) = the i with visible[i] != 0, ascending (so every rank
 *     derives the same list from the same mask); *count_dev (DEVICE int64) = M.
 *     ws: scratch of gs_compact_workspace(P) bytes.  idx: DEVICE int32[P] (capacity).
 *   gs_gather_columns: packed[r][j] = full[r][idx[j]] for r < F, j < M (full: [F][S],
 *     packed: [F][M], both DEVICE float).
 *   gs_scatter_columns: full[r][idx[j]] = packed[r][j] (other columns untouched).
 * M is read by the host between the calls (the collective's size); P, F >= 0, S >= P,
 * else GS_ERR_ARG; NULL pointers with a nonzero size, GS_ERR_ARG. */
gs_status gs_visibility_union(int n_views, const uint8_t* const* flags /*HOST[n_views]*/, int64_t P, int accumulate,
                              uint8_t* visible, void* stream);
size_t gs_compact_workspace(int64_t P);
gs_status gs_compact_index(const uint8_t* visible, int64_t P, void* ws, size_t ws_bytes, int32_t* idx,
                           int64_t* count_dev, void* stream);
gs_status gs_gather_columns(const float* full, int64_t F, int64_t S, const int32_t* idx, int64_t M, float* packed,
                            void* stream);
gs_status gs_scatter_columns(const float* packed, int64_t F, int64_t S, const int32_t* idx, int64_t M, float* full,
                             void* stream);

/* ---------------------------------------------------------------- layout (setup)
 * gs_spatial_order: params_out = params_in with the Gaussians (columns) permuted into
 * Morton (Z-curve) order of their means, 10 bits per axis inside the means'
 * bounding box; ties keep the input order.  perm (nullable) int32[P] receives, for
 * each new index, the old index.  A one-off layout transform (not a step of the
 * method): the visible subset of a view then occupies contiguous sectors of every
 * SoA row, which is what the per-view projection kernels stream.  Synchronous only
 * in the sense of stream order; params_in and params_out must not alias.
 *  ws: >= gs_spatial_order_workspace() bytes. */
size_t gs_spatial_order_workspace(const gs_scene* scene /*HOST*/);
gs_status gs_spatial_order(const gs_scene* scene /*HOST*/, const float* params_in, float* params_out, int32_t* perm,
                           void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- keyframe schedule (host)
 * The online optimisation strategy of PAPER.md:149 (§III-B3 "Online Optimization")
 * with the settings of PAPER.md:174, as a plan of iterations; each iteration is then
 * one fwd + bwd + Adam step over one view.  Frame t is a
 * keyframe iff new_prims[t] > threshold; keyframes get m iterations on themselves;
 * non-keyframes get n, plus one iteration on each of the first (m - n) keyframes of
 * the shuffled keyframe list (the current frame excluded); after the last frame,
 * global_iters passes over the keyframe list, each in a freshly shuffled order.
 * store_all_frames != 0 puts every frame in the list (the paper's ScanNet++ setting)
 * while the m / n split still follows the threshold.  Shuffles: Fisher-Yates with
 * the counter-based generator documented in DESIGN.md (R31).  All pointers HOST.
 *  iter_view[i]:  view (frame) optimised by iteration i
 *  iter_frame[i]: frame during which iteration i runs, -1 for the global passes
 *  n_iters:       number of iterations of the plan (always written)
 *  is_keyframe:   nullable uint8[n_frames]
 * Returns GS_ERR_CAPACITY (n_iters = the required capacity) if capacity is too small,
 * GS_ERR_ARG on invalid parameters (n > m, negative counts, NULL). */
typedef struct {
  int64_t threshold;        /* 50 */
  int32_t m, n;             /* Replica 5 / 3, ScanNet++ 10 / 1 */
  int32_t global_iters;     /* 10 */
  int32_t store_all_frames; /* 1 for the ScanNet++ setting */
  uint64_t seed;
} gs_kf_params;
gs_status gs_keyframe_schedule(const gs_kf_params* prm /*HOST*/, int64_t n_frames, const int64_t* new_prims /*HOST*/,
                               int32_t* iter_view /*HOST*/, int32_t* iter_frame /*HOST*/, int64_t capacity,
                               int64_t* n_iters /*HOST*/, uint8_t* is_keyframe /*HOST, nullable*/);

/* ================================================================ TSDF fusion (NEXT-3)
 * GSFusion's TSDF grid (§III-A1) and its fusion step (PAPER.md:105-115,
 * §III-B1, Eqs. 6-9) on the GPU: single-resolution voxels
 * (tsdf, weight) in 8^3-voxel blocks, indexed by the 63-bit Morton code of the block
 * coordinates through an open-addressing hash table (the octree is used "as a spatial
 * index" only).  Readings R32-R36 in DESIGN.md.
 *
 * Coordinates: voxel index v = floor(p / voxel_size) + origin (per axis, must lie in
 * [0, 2^21)); block b = v >> 3; voxel centre p_v = (v - origin + 0.5) voxel_size. */
typedef struct {
  float voxel_size; /* m (1 cm) */
  float trunc;      /* epsilon, m (band half-width; default 6 voxels, R33) */
  float w_max;      /* weight cap of Eq. 8 */
  float step;       /* allocation ray-march step, m (default voxel_size / 2, R34) */
  int32_t origin[3];
} gs_tsdf_params;

/* Caller-owned DEVICE buffers.  keys/slots: int64/int32 [table_cap] (table_cap a power
 * of two, >= 2 x blocks); pool_keys: uint64 [block_cap] (Morton key of each pool
 * block); tsdf, weight: float [block_cap][512] (voxel x-fastest inside a block);
 * num_blocks: int64 counter.  gs_tsdf_reset initialises everything (empty table,
 * zero voxels); allocated blocks are never freed, so pool entries are zero until
 * first allocated. */
typedef struct {
  uint64_t* keys;
  int32_t* slots;
  uint64_t* pool_keys;
  float* tsdf;
  float* weight;
  int64_t table_cap;
  int64_t block_cap;
  int64_t* num_blocks;
} gs_tsdf_volume;

#define GS_TSDF_EMPTY_KEY 0xFFFFFFFFFFFFFFFFull

gs_status gs_tsdf_reset(gs_tsdf_volume vol, void* stream);

/* Band allocation: for every pixel with valid depth d (> 0, metres of
 * camera z), samples the pixel's line of sight at z = d - eps + k step (k = 0..n, the
 * last sample clamped to d + eps) and allocates the block of every sample.
 * depth: float[H][W] DEVICE.  new_blocks: nullable DEVICE int64, += blocks created.
 * Returns GS_ERR_CAPACITY (synchronising) if the pool or table overflowed; the volume
 * is then unusable until reset. */
gs_status gs_tsdf_allocate(const gs_tsdf_params* prm /*HOST*/, gs_tsdf_volume vol, const gs_camera* cam /*HOST*/,
                           const float* depth, int64_t* new_blocks, void* stream);

/* Integration (Eqs. 6-9): every voxel of every allocated block whose
 * centre projects (camera z > 0, nearest pixel under R1) onto a valid depth d gets
 * sdf = d - z_c (Eq. 6); voxels with sdf < -eps are skipped (R35); tsdf = min(1,
 * sdf/eps) if sdf > 0 else max(-1, sdf/eps) (Eq. 7); w_k = min(w_max, w_{k-1} + 1)
 * (Eq. 8); tsdf_k = (tsdf_{k-1} w_{k-1} + tsdf w_k) / (w_{k-1} + w_k) (Eq. 9).
 * updated: nullable DEVICE int64, += voxels updated.  fp32 with a fixed operation
 * order (bit-exact against the oracle). */
gs_status gs_tsdf_integrate(const gs_tsdf_params* prm /*HOST*/, gs_tsdf_volume vol, const gs_camera* cam /*HOST*/,
                            const float* depth, int64_t* updated, void* stream);

/* ================================================================ seeding (NEXT-4)
 * Quadtree decomposition of the RGB frame and weight-gated Gaussian initialisation
 * (§III-B2, Eq. 10).  Readings R37-R40.
 *
 * gs_quadtree: a cell (x, y, w, h) splits into NW (x, y, w/2, h/2), NE (x + w/2, y,
 *   w - w/2, h/2), SW, SE (integer halves) iff w > min_cell, h > min_cell and its
 *   contrast max(L) - min(L) > threshold, L = 0.299 R + 0.587 G + 0.114 B (fp32, in
 *   that order).  rgb: float[3][H][W] in [0, 1] DEVICE.  leaves: int32[leaf_capacity][4]
 *   (x, y, w, h) DEVICE, in depth-first NW, NE, SW, SE order; num_leaves: DEVICE int64
 *   (the full count even if it exceeds the capacity).  ws: gs_quadtree_workspace bytes.
 *   A leaf side is at least ceil((min_cell + 1) / 2) pixels, so (W / s + 1)(H / s + 1)
 *   leaves with that s always fit; gs_seed_gaussians reads num_leaves leaves, so size
 *   the buffer for that bound.
 * gs_seed_gaussians: for every leaf in order, the centre pixel u = (x + w/2, y + h/2)
 *   with depth d > 0 is back-projected, p_q = T_WC pi^-1(u, d) (Eq. 10); if the voxel
 *   containing p_q (TSDF grid of the same frame, fused BEFORE seeding) has weight
 *   exactly 1, a Gaussian is appended at column scene->P + (index among the accepted
 *   leaves): mean p_q, log-scale log(s) x 3 with s = |pi^-1(corner (x, y), d) -
 *   pi^-1(u, d)|, quaternion (1, 0, 0, 0), opacity logit 0 (alpha 0.5), SH DC
 *   (rgb(u) - 0.5) / Y00, higher SH 0.  Columns past P_stride are not written.
 *   num_new: DEVICE int64 = accepted count (the keyframe signal of PAPER.md:149); the
 *   caller advances P. */
size_t gs_quadtree_workspace(int32_t width, int32_t height, int32_t min_cell);
gs_status gs_quadtree(int32_t width, int32_t height, const float* rgb, float threshold, int32_t min_cell, void* ws,
                      size_t ws_bytes, int32_t* leaves, int64_t leaf_capacity, int64_t* num_leaves, void* stream);
gs_status gs_seed_gaussians(const gs_camera* cam /*HOST*/, const gs_tsdf_params* prm /*HOST*/, gs_tsdf_volume vol,
                            const float* depth, const float* rgb, const int32_t* leaves, const int64_t* num_leaves,
                            const gs_scene* scene /*HOST*/, float* params, int64_t* num_new, void* stream);

/* ---------------------------------------------------------------- harness: Eq. 12
 * L = mean_{pixel,ch} |C - C*| + w_depth mean_pixel |D - D*| (R19), sign(0) = 0.
 * A target sample that is not a measurement -- a non-finite colour, or a depth <= 0
 * (the sensor's "invalid", R41) or non-finite -- contributes neither loss nor
 * gradient (R43; the means still divide by npix).
 * Writes dL/drgb [3][npix], dL/ddepth [npix]; loss (nullable DEVICE float) += L. */
gs_status gs_l1_loss_grad(int64_t npix, const float* rgb, const float* depth, const float* target_rgb,
                          const float* target_depth, float w_depth, float* dL_drgb, float* dL_ddepth, float* loss,
                          void* stream);

/* ---------------------------------------------------------------- harness: input frames
 * The method "takes a pair of RGB-D images as input" at every time step (PAPER.md:58,
 * Fig. 2); Eq. 12's C* and D* and the depth map D_k of Eqs. 6 and 10 are that frame.
 * A sensor frame is an 8-bit RGB image and a 16-bit depth image whose units times
 * depth_scale are metres, 0 = invalid (reading R41).  This call turns
 * one frame, as it arrives from the host, into the planar float images the other calls
 * take:  out_rgb[c][y][x] = rgb[y][x][c] / 255 (IEEE division, correctly rounded),
 * out_depth[y][x] = depth[y][x] * depth_scale (one rounded fp32 product; 0 stays 0).
 *   rgb       DEVICE uint8 [H][W][3] (interleaved, as decoded from the sensor / file)
 *   depth     DEVICE uint16 [H][W]
 *   out_rgb   DEVICE float [3][H][W];  out_depth DEVICE float [H][W]  (caller-owned)
 * width, height > 0 and depth_scale > 0 (finite), else GS_ERR_ARG.  Vectorised 4 pixels
 * per thread when W*H % 4 == 0 and the buffers are 16-B (rgb 4-B, depth 8-B) aligned,
 * else one pixel per thread; same values either way. */
gs_status gs_decode_rgbd(int32_t width, int32_t height, const uint8_t* rgb, const uint16_t* depth,
                         float depth_scale, float* out_rgb, float* out_depth, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GSR_H_ */
