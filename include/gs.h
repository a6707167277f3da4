/*
 * gs.h -- C ABI of libgs.so, the B200 (sm_100a) hot path of Photo-SLAM's photorealistic
 * mapping (arXiv 2311.16728): render the hyper-primitive map with a tile-based Gaussian
 * splatting rasteriser (Eq. 3), evaluate the photometric loss (Eq. 4,
 * PAPER.md:181-184), back-propagate it to the primitive parameters, build the
 * Gaussian pyramid (Eq. 5) and apply the optimiser step.
 * Citations are /root/reference lines; readings R1..R26 are listed in DESIGN.md.
 *
 * Conventions for every entry point
 *  - Pointers are DEVICE pointers unless marked (host).  The caller allocates every buffer
 *    (including the workspace sized by gs_workspace_size); the library never allocates,
 *    frees or synchronises, except gs_query_status which synchronises `stream`.
 *  - All work is enqueued on `stream` (a cudaStream_t; NULL = legacy default stream) and the
 *    call returns immediately; CUDA-graph capture of any call sequence is allowed.
 *  - Argument and shape errors are returned synchronously (GS_ERR_INVALID_ARG /
 *    GS_ERR_SHAPE) and nothing is enqueued.  A failed kernel launch returns GS_ERR_CUDA.
 *    Pair-capacity overflow is detected on the device: it sets a flag that
 *    gs_query_status reports as GS_ERR_CAPACITY (that call's outputs are then invalid).
 *  - No exception or C++ type crosses the ABI.  Calls are re-entrant given distinct
 *    workspaces; concurrent calls on one workspace are a caller error.
 *  - Precision: fp32 everywhere (R23); decision quantities follow the fp32 recipe of
 *    DESIGN.md so that binning and sort order are bit-exact to the CPU oracle.
 */
#ifndef GS_H
#define GS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *gs_stream_t; /* identical to cudaStream_t */

typedef enum {
    GS_OK = 0,
    GS_ERR_INVALID_ARG = 1,  /* NULL pointer, non-positive size, bad degree/level count      */
    GS_ERR_SHAPE = 2,        /* DimensionMismatch, TooManyLevels, */
                             /* views of different sizes, workspace too small                  */
    GS_ERR_CAPACITY = 3,     /* (from gs_query_status) more tile pairs than the workspace holds */
    GS_ERR_STALE_STATE = 4,  /* backward without a matching forward             */
    GS_ERR_CUDA = 5,         /* kernel launch / CUDA runtime failure                           */
    GS_ERR_NOT_SUPPORTED = 6 /* e.g. more than GS_MAX_VIEWS views in one call                 */
} gs_status;

#define GS_TILE 16      /* 16x16-pixel tiles */
#define GS_MAX_VIEWS 64 /* views per call (keyframe batch on one GPU) */

/* Pinhole camera of one keyframe view.  World->camera p_c = R P + t with R row-major
   (SPEC.md:38); pixel (x, y) is centred at integer (x, y) (R12); at pyramid level l the
   caller passes fx, fy, cx, cy scaled by 2^-l and the ceil-halved size (R12, R19).
   znear: cull z_c <= znear (R14).  lim_x, lim_y: |x_c/z_c|, |y_c/z_c| clamp used inside the
   EWA Jacobian (R15); +INF disables the clamp. */
typedef struct {
    float R[9];
    float t[3];
    float fx, fy, cx, cy;
    int32_t width, height;
    float znear, lim_x, lim_y;
} gs_camera;

/* Gaussian parameters (position P, rotation r, scaling s, density sigma, SH),
   fp32 structure-of-arrays: row r occupies data[r*ld .. r*ld+n).  K = gs_param_rows(D):
     rows 0..2   P (x, y, z)
     rows 3..6   raw quaternion (w, x, y, z), normalised inside (R5)
     rows 7..9   log scales (R4)
     row  10     opacity logit (R3)
     rows 11..   SH, coefficient-major: row 11 + 3*l + c, l = 0..(D+1)^2-1, c = R,G,B (R2)
   ld >= n and ld % 4 == 0 (gs_param_ld gives the recommended value).  Gradients and the
   Adam moments use the identical layout. */
typedef struct {
    float *data;
    int64_t n;
    int64_t ld;
    int32_t sh_degree; /* 0..3 */
} gs_params;

/* Optimiser hyper-parameters (PAPER.md:568 fixed learning rate; R20).  lr per class:
   [0] P, [1] quaternion, [2] log scale, [3] opacity logit, [4] SH DC (l = 0), [5] SH rest. */
typedef struct {
    float lr[6];
    float beta1, beta2, eps;
    int32_t sgd_mode; /* 1: p -= lr * g (no moments) */
} gs_adam_hparams;

/* Rows K of the parameter layout: 11 + 3 (D+1)^2 (14 at D = 0, 59 at D = 3). */
int32_t gs_param_rows(int32_t sh_degree);
/* Recommended leading dimension: n rounded up to a multiple of 64 floats (256-byte rows). */
int64_t gs_param_ld(int64_t n);

/* Bytes of the render workspace for n Gaussians, n_views views of width x height and a
   capacity of pair_capacity (Gaussian, tile) pairs summed over the views (rounded up to a
   multiple of 4096).  *bytes is host memory. */
gs_status gs_workspace_size(int64_t n, int32_t n_views, int32_t width, int32_t height,
                            int64_t pair_capacity, size_t *bytes);

/* A1 + A2: per (view, Gaussian) projection, culling, EWA 2D covariance + 0.3 px^2 floor,
   conic, radius r = ceil(3 sqrt(lambda_max)), tile rect, depth, SH colour and sigmoid
   opacity; then the exclusive scan of tiles touched.
   cams: host array [n_views]; all views must share width and height. */
gs_status gs_preprocess(const gs_params *params, const gs_camera *cams, int32_t n_views, void *ws,
                        size_t ws_bytes, gs_stream_t stream);

/* A3-A6: the pairs of every (view, tile) in the order of a stable sort by key = (view*tiles +
   tile) << 32 | float_bits(depth), value = Gaussian index (SPEC.md:348 (2)-(3)) -- by default
   tile buckets filled by a scatter and each sorted by (depth, id) (bin.cu); gs_set_binning(1)
   selects key duplication + a stable onesweep LSD radix sort; both give the same pairs bit for
   bit -- tile ranges, and per-tile front-to-back alpha
   compositing of Eq. 3: alpha = min(0.99, sigma e^power),
   power cut at Mahalanobis^2 > 9 (R9), skip alpha < 1/255, stop when T (1 - alpha) < 1e-4
   (R7, R8).  Requires gs_preprocess on the same params/cams/workspace first.
   bg: host float[3] background (R16).  out_rgb [n_views][3][H][W], out_T [n_views][H][W]
   (final transmittance; may be NULL). */
gs_status gs_render_forward(const gs_params *params, const gs_camera *cams, int32_t n_views, void *ws,
                            size_t ws_bytes, const float bg[3], float *out_rgb, float *out_T,
                            gs_stream_t stream);

/* Workspace bytes for gs_photometric_loss on V images of H x W. */
gs_status gs_loss_workspace_size(int32_t V, int32_t H, int32_t W, size_t *bytes);

/* A7: Eq. 4 per view, L_v = (1 - lambda) mean|I_r - I_gt| + lambda (1 - mean SSIM) with an
   11x11 Gaussian window (sigma 1.5), C1 = 0.01^2, C2 = 0.03^2, zero-padded 'same' (R17), and
   its exact gradient (L1 subgradient 0 at 0).  render, gt, dL_drender:
   [V][3][H][W]; loss: device float[V]. */
gs_status gs_photometric_loss(const float *render, const float *gt, int32_t V, int32_t H, int32_t W,
                              float lambda, float *loss, float *dL_drender, void *ws, size_t ws_bytes,
                              gs_stream_t stream);

/* A8 + A9: reverse-mode gradient of sum_v <dL_drgb_v, I_v> through the compositing of the
   last gs_render_forward on this workspace and through the projection to P, quaternion,
   log scale, opacity logit and SH, summed over views (R22).
   grads (param layout, += accumulate), grad2d_norm_accum (float[n], += sum over views of
   ||dL/dmean2d|| in pixels, R24; may be NULL).  Returns GS_ERR_STALE_STATE if the last
   forward on ws used other params, n, views or cameras. */
gs_status gs_render_backward(const gs_params *params, const gs_camera *cams, int32_t n_views, void *ws,
                             size_t ws_bytes, const float bg[3], const float *dL_drgb, float *grads,
                             float *grad2d_norm_accum, gs_stream_t stream);

/* A8 + A9 + A11 fused for one optimiser step without a materialised gradient: the
   backward of gs_render_backward (same definition) followed by the Adam / SGD step of
   gs_adam_step over ALL Gaussians (Gaussians invisible in every view get g = 0, as in the
   dense step, R20), in place on params, m, v.  Equivalent to gs_render_backward into a zeroed
   gradient buffer followed by gs_adam_step(..., 0, n, ...) -- up to the summation order of the
   raster backward's fp32 atomics -- but never writes or reads the N x K gradient array
   (fused backward + Adam).  Single-GPU path: with data
   parallelism the gradient must be all-reduced, use the two separate calls.  After this call
   the forward state of ws is stale (the parameters changed).
   step > 0: the 1-based step number.  step == 0: device-resident step counter (for CUDA-graph
   replay): the call increments *step_dev (int64, device) on the device and uses the new value. */
gs_status gs_render_backward_adam(gs_params *params, const gs_camera *cams, int32_t n_views, void *ws,
                                  size_t ws_bytes, const float bg[3], const float *dL_drgb, float *m, float *v,
                                  const gs_adam_hparams *hp, int64_t step, int64_t *step_dev,
                                  float *grad2d_norm_accum, gs_stream_t stream);

/* ---- densify and prune ("splitting or cloning
   hyper primitives with large loss gradients similar to [kerbl2023]").  Readings R27-R30 in
   DESIGN.md.  Statistics of a densify interval, per Gaussian: grad_accum = the backward's
   grad2d_norm_accum (sum of ||dL/dmean2d|| in pixels over visible (iteration, view) pairs),
   vis_count = number of those pairs, max_radius = largest pixel radius (gs_densify_stats). */
typedef struct {
    float grad_threshold;    /* mean ||dL/dmean2d|| (pixels) at or above which a Gaussian densifies */
    float percent_dense;     /* "large" = max scale > percent_dense * scene_extent (SPEC: 1 %) */
    float scene_extent;
    float opacity_threshold; /* prune sigmoid(logit) < this (SPEC default 0.005) */
    int32_t max_screen_px;   /* prune max_radius > this (SPEC: 0.5 x image dimension) */
} gs_densify_cfg;

/* Bytes of the temp buffer gs_densify_plan / gs_densify_apply use for n Gaussians. */
gs_status gs_densify_temp_size(int64_t n, size_t *bytes);

/* After gs_preprocess (or a forward) on ws: vis_count[i] += number of views Gaussian i is
   visible in, max_radius[i] = max(max_radius[i], its pixel radius).  float[n] / int32[n],
   device.  GS_ERR_STALE_STATE if ws was not preprocessed with these params and cameras. */
gs_status gs_densify_stats(const gs_params *params, const gs_camera *cams, int32_t n_views, const void *ws,
                           size_t ws_bytes, float *vis_count, int32_t *max_radius, gs_stream_t stream);

/* Classify every Gaussian (decisions in fp32: mean = grad_accum / vis_count (0 if never visible),
   high = mean >= grad_threshold, large = max_j (float)exp((double)log s_j) > percent_dense *
   scene_extent, prune = logit < (float)log(t / (1 - t)) or max_radius > max_screen_px; prune
   wins, else high && !large = clone, high && large = split) into temp and return, on the host,
   counts = {n_clone, n_split, n_prune, n_new} (n_new = n - n_prune + n_clone + n_split).
   Synchronises the stream (the caller must allocate the new map). */
gs_status gs_densify_plan(const gs_params *params, const float *grad_accum, const float *vis_count,
                          const int32_t *max_radius, const gs_densify_cfg *cfg, void *temp, size_t temp_bytes,
                          int64_t counts[4], gs_stream_t stream);

/* Write the densified map planned in temp into out (out->n = counts[3], same sh_degree, its own
   ld): kept and cloned originals in index order (bitwise copies, with their Adam moments m, v),
   then one clone per clone parent, then two children per split parent (parent order).  A new
   Gaussian is its parent with position P + R(q) diag(e^s) z[i][c] and zero moments; split
   children also get log s - ln 1.6 (scale / 1.6).  z: device float[n][2][3] standard-normal
   samples (the method's randomness, an input).  m, v, out_m, out_v may all be NULL (no
   optimiser state). */
gs_status gs_densify_apply(const gs_params *params, const float *m, const float *v, const float *z, const void *temp,
                           size_t temp_bytes, gs_params *out, float *out_m, float *out_v, gs_stream_t stream);

/* Carry a per-Gaussian byte tag (e.g. the temporary flag of geometry densification) through the
   densification planned in temp: tags_out[new row] = tags_in[source Gaussian] for kept and cloned
   originals, clones and split children.  tags_out: device uint8[n_new]. */
gs_status gs_densify_tags(int64_t n, const void *temp, size_t temp_bytes, const uint8_t *tags_in, uint8_t *tags_out,
                          gs_stream_t stream);

/* ---- geometry-based densification ("actively
   create additional temporary hyper primitives based on the inactive 2D feature points").
   Readings R31-R33 in DESIGN.md.  For each INACTIVE keypoint (active[k] == 0), in index order,
   at its nearest pixel (round-half-even; skipped outside the image): depth d from depth_map
   (mode 1, RGB-D; skipped if <= 0) or (mode 0, mono) the inverse-distance-weighted depth of the
   <= 4 nearest active keypoints within rho pixels (kp_depth[j]: camera-space depth of active
   keypoint j; skipped if none); new primitive (create_map_points): P = R^T (d K^-1
   (u, v, 1) - t), q = (1, 0, 0, 0), log s = log(d / fx) x 3, logit(0.1), SH DC = (pixel colour -
   0.5) / C0, higher SH 0.  cam: host, one view; uv: device float[n][2]; active: device int32[n];
   kp_depth: device float[n] (mono); depth_map: device float[H][W] (RGB-D); image: device float
   [3][H][W].  out: parameter layout with capacity out->n >= n_keypoints rows (same sh_degree as
   the map); rows [0, *count) are written; src[r] = keypoint of row r; count: device int32. */
gs_status gs_geometry_densify(const gs_camera *cam, const float *uv, const int32_t *active, const float *kp_depth,
                              const float *depth_map, const float *image, int32_t n_keypoints, int32_t mode, float rho,
                              gs_params *out, int32_t *src, int32_t *count, gs_stream_t stream);

/* A0: Gaussian pyramid (Eq. 5): level l+1 = even rows/cols of the level-l
   image blurred by [1,4,6,4,1]/16 horizontally then vertically with a reflect-101 border
   (R18); sizes ceil-halved.  img [n_images][C][H][W]; out = levels 1..n_levels concatenated,
   level-major, each [n_images][C][H_l][W_l].  GS_ERR_SHAPE if min(H, W) <= 2^n_levels
   (TooManyLevels). */
gs_status gs_pyramid(const float *img, int32_t n_images, int32_t C, int32_t H, int32_t W, int32_t n_levels,
                     float *out, gs_stream_t stream);

/* A11: fused optimiser step over Gaussians [g_begin, g_end) of every row: bias-corrected
   Adam with per-class lr (R20) or SGD, in place on params, m, v; step is 1-based; if
   zero_grads, grads of the range are zeroed after use. */
gs_status gs_adam_step(gs_params *params, float *grads, float *m, float *v, const gs_adam_hparams *hp,
                       int64_t step, int64_t g_begin, int64_t g_end, int32_t zero_grads, gs_stream_t stream);

/* A11 on a parameter-row shard (reduce-scatter -> sharded Adam -> all-gather):
   the step of gs_adam_step over all n Gaussians of parameter rows [row_begin, row_end) of the
   [K][ld] layout (K = gs_param_rows; each row's class decides its learning rate).  params and
   grads are the full layout; m_rows, v_rows hold only the shard's moments, row r at
   (r - row_begin) * ld (a rank keeps 1/G of the optimiser state).  Same arithmetic as
   gs_adam_step, element for element.  GS_ERR_INVALID_ARG for a range outside [0, K]. */
gs_status gs_adam_step_rows(gs_params *params, float *grads, float *m_rows, float *v_rows, const gs_adam_hparams *hp,
                            int64_t step, int32_t row_begin, int32_t row_end, int32_t zero_grads,
                            gs_stream_t stream);

/* gs_adam_step_rows with the step counter on the device, for a data-parallel step captured in a
   CUDA graph (the counter advances on every replay): step_dev (device, int64) holds the number
   of steps taken; the call takes step *step_dev + 1 (bias corrections from it) and leaves
   *step_dev incremented (stream-ordered: a one-thread kernel, then the step).  Otherwise as
   gs_adam_step_rows.  GS_ERR_INVALID_ARG for a NULL step_dev. */
gs_status gs_adam_step_rows_dev(gs_params *params, float *grads, float *m_rows, float *v_rows,
                                const gs_adam_hparams *hp, int64_t *step_dev, int32_t row_begin, int32_t row_end,
                                int32_t zero_grads, gs_stream_t stream);

/* Synchronises stream, then reads the workspace status: *flags (host) bit 0 = pair capacity
   overflow; *pairs (host, may be NULL) = pair count of the last gs_preprocess.  Returns
   GS_ERR_CAPACITY if bit 0 is set. */
gs_status gs_query_status(const void *ws, size_t ws_bytes, gs_stream_t stream, int32_t *flags, int64_t *pairs);

/* ---- A10 + A11 fused over peer memory (SURVEY §8(e) extension f3; north_star: "Gaussian-
   parameter gradients are summed ... over NVLink"; the optimiser step PAPER.md:568, R20).
   Data parallelism over keyframe views: every rank's backward adds its views' gradient into its
   own [K][ld] gradient buffer; the step's gradient is the sum over ranks (R22).  Rank g owns the
   flat element range [e_begin, e_end) of the [K][ld] layout (gs_comm_shard: world ranges of
   whole float4s, the last one shorter).

   gs_reduce_adam_bcast: for every element of the rank's range, g = sum over ranks of
   grad_peers[q][e] (with grad_mc / param_mc -- multicast addresses of NVLink SHARP groups -- one
   multimem.ld_reduce; else peer loads summed in rank order 0..world-1), the Adam update of
   gs_adam_step (same arithmetic, same bits; columns >= n left as they are) on m_shard / v_shard
   (device, the range's moments, index e - e_begin), then the new value is stored into
   param_peers[q][e] and 0 into grad_peers[q][e] for every rank q (multimem.st on the multicast
   addresses, else one peer store per rank).  param_peers / grad_peers: host arrays of `world`
   device pointers valid on this device (this rank's own buffers at index `rank`;
   param_peers[rank] must equal params->data); the buffers are symmetric (same n, ld on every
   rank) and owned by the caller.  step >= 1, or step_dev (device int64, read by the kernel:
   the bias corrections of graph replays) with step ignored.
   gs_peer_barrier: every rank's earlier work on its stream completes and becomes visible to all
   ranks before any rank's later work starts: flag_peers = host array of `world` device
   pointers to each rank's uint32[world] flag array (zeroed by the caller before the first call,
   symmetric), epoch = this rank's device uint32 barrier count; step_dev (optional) is
   incremented once the barrier passed.  A step is: backward -> gs_peer_barrier(step_dev) ->
   gs_reduce_adam_bcast(step_dev) -> gs_peer_barrier(NULL).  Both calls only enqueue (graph
   capturable).  GS_ERR_INVALID_ARG for a NULL pointer, world outside [1, 8] or rank outside
   [0, world); GS_ERR_SHAPE for ld % 4 != 0.  Errors not detected: peers calling with different
   shapes or barrier counts (the barrier then waits forever -- a caller contract). */
gs_status gs_comm_shard(int64_t n, int32_t sh_degree, int32_t rank, int32_t world, int64_t *e_begin, int64_t *e_end);
gs_status gs_peer_barrier(uint32_t *const *flag_peers, int32_t rank, int32_t world, uint32_t *epoch,
                          int64_t *step_dev, gs_stream_t stream);
gs_status gs_reduce_adam_bcast(const gs_params *params, float *const *param_peers, float *const *grad_peers,
                               float *param_mc, float *grad_mc, float *m_shard, float *v_shard,
                               const gs_adam_hparams *hp, int64_t step, const int64_t *step_dev, int32_t rank,
                               int32_t world, gs_stream_t stream);

/* Enqueues on stream a copy of the workspace status into dst[0..1] (device or pinned host
   int32): dst[0] = flags (bit 0 = pair capacity overflow of the last gs_preprocess: that call's
   outputs are invalid), dst[1] = its pair count.  Does not synchronise, so it can sit inside a
   captured CUDA graph (the end-to-end step reads it back with its losses).
   GS_ERR_INVALID_ARG for a NULL pointer or a buffer smaller than a workspace header. */
gs_status gs_status_async(const void *ws, size_t ws_bytes, int32_t *dst, gs_stream_t stream);

/* Forgets the forward-state token of ws (SPEC.md:355-359 StaleRenderState check): call before
   freeing a workspace, so that a new workspace allocated at the same address cannot pass the
   check with the old one's token.  GS_ERR_INVALID_ARG for NULL. */
gs_status gs_workspace_release(const void *ws);

const char *gs_status_str(gs_status s);

/* ---- Map layout (not a step of the method): spatial order.
   Eq. 3 does not depend on where a Gaussian sits in memory -- its index only
   breaks ties between equal depths (SPEC.md:348 (3)) -- but the memory behaviour of the
   per-Gaussian kernels (A1, A9, A11, bin scatter) and of the raster backward's atomics does.
   gs_spatial_order writes perm[k] (device uint32[n]) = index of the Gaussian placed at position
   k: ascending 30-bit Morton code of its mean (x in bits 0, 3, ..., y in 1, 4, ..., z in 2, 5,
   ...), each axis cell = min(1023, (int)((x - lo) * (1024 / (hi - lo)))) in fp32 IEEE operations
   over the means' bounding box [lo, hi] (cell 0 for a flat axis); equal codes keep index order.
   temp: device bytes >= gs_spatial_order_temp_size.  GS_ERR_NOT_SUPPORTED for n >= 2^30.
   gs_permute_columns: dst[r * ld + k] = src[r * ld + perm[k]] for r < rows, k < n (src and dst
   distinct device buffers; the parameter layout has rows = gs_param_rows(D), a per-Gaussian
   array rows = 1).  Applying the same perm to params, Adam m and v keeps the optimiser state
   with its Gaussians. */
gs_status gs_spatial_order_temp_size(int64_t n, size_t *bytes);
gs_status gs_spatial_order(const gs_params *params, uint32_t *perm, void *temp, size_t temp_bytes,
                           gs_stream_t stream);
gs_status gs_permute_columns(const float *src, float *dst, int64_t ld, int32_t rows, int64_t n, const uint32_t *perm,
                             gs_stream_t stream);

/* ---- test / benchmark entry points ------------------------------------------------------ */
/* Stable LSD radix sort of n (key, value) pairs on key bits [0, key_bits) (8-bit digits,
   one decoupled-look-back pass per digit).  Sorted in place in keys/vals; keys_alt/vals_alt
   are ping-pong buffers of n entries; temp of gs_sort_temp_size bytes. */
/* Diagnostics: with on != 0 the forward also writes each pixel's number of composited
   Gaussians (gs_debug_workspace_view n_composited); off (the default) it leaves that array as it
   was -- the count costs ~6 % of the forward's instructions.  Process-wide setting. */
gs_status gs_set_render_stats(int32_t on);

gs_status gs_sort_temp_size(int64_t n, int32_t key_bits, size_t *bytes);
gs_status gs_debug_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *keys_alt, uint32_t *vals_alt, int64_t n,
                              int32_t key_bits, void *temp, size_t temp_bytes, gs_stream_t stream);

/* Device pointers to the per-(view, Gaussian) and binning buffers of a workspace, for
   bit-exact comparison with the oracle.  Valid after gs_preprocess / gs_render_forward. */
typedef struct {
    const float *rec0;            /* [n_views*n][4] (u, v, A, B): mean2d, conic A, B */
    const float *rec1;            /* [n_views*n][4] (C, sigma, r, g)                 */
    const float *rec2;            /* [n_views*n][4] (b, 3-sigma x/y extents, -)      */
    const float *depth;           /* [n_views*n] view-space z                        */
    const int32_t *radius;        /* [n_views*n] 0 = culled                          */
    const int32_t *rect;          /* [n_views*n][4] tile x0, y0, x1, y1 (exclusive)  */
    const uint32_t *tiles_touched; /* [n_views*n]                                    */
    const uint32_t *offsets;       /* [n_views*n] exclusive scan of tiles_touched     */
    const uint64_t *keys;          /* [capacity] sorted keys (after render_forward)   */
    const uint32_t *vals;          /* [capacity] sorted values                        */
    const uint32_t *ranges;        /* [n_views*tiles][2] [start, end) per tile        */
    const uint32_t *n_contrib;     /* [n_views][H][W] list position of the last composited */
    const uint32_t *n_composited;  /* [n_views][H][W] number of composited Gaussians   */
    int64_t capacity;
} gs_ws_view;
gs_status gs_debug_workspace_view(void *ws, size_t ws_bytes, int64_t n, int32_t n_views, int32_t width,
                                  int32_t height, gs_ws_view *out);
/* Binning path for subsequent gs_preprocess / gs_render_forward calls (process-wide):
   0 (default) = per-(view, tile) pair counts in A1, scan to tile ranges, scatter into tile
   buckets and an in-tile bitonic sort by (depth bits, id) in shared memory (MSD radix on the
   tile digit); 1 = key duplication + the global onesweep LSD radix sort + range extraction.
   Both produce the identical keys, values and ranges (bit-exact to the oracle). */
gs_status gs_set_binning(int32_t mode);

/* Live timing of one kernel inside a benchmark: after gs_profile_kernel("k_raster_bwd") every
   launch of that kernel (any call, any stream) is bracketed by CUDA events recorded on its
   launching stream; gs_profile_read synchronises on them and returns the summed duration and
   the launch count, then resets.  gs_profile_kernel(NULL) turns it off.  Names:
   k_preprocess, k_raster_fwd, k_raster_bwd, k_preprocess_bwd, k_adam, k_adam_fused, k_sort_pass,
   k_tile_sort. */
gs_status gs_profile_kernel(const char *kernel);
gs_status gs_profile_read(double *total_ms /*host*/, int64_t *launches /*host*/);
/* (float)exp((double)s) exactly as the preprocess kernel evaluates it, for the exhaustive
   check against the oracle (DESIGN.md fp32 recipe). */
gs_status gs_debug_exp_scale(const float *s, float *out, int64_t n, gs_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* GS_H */
