/*
 * splatstream_b200.h -- C ABI of the B200 (sm_100a) mapping hot path.
 *
 * Drop-in boundary for the reference package `splatstream`
 * (/root/reference/pkg/src/splatstream).  The reference has no FFI: its
 * boundary is the Python operator API listed in SURVEY.md 8b.  Each entry
 * point below replaces the compute inside one of those calls; the Python
 * package paper_2410_00486_b200 keeps the reference's names, argument
 * meaning and error behaviour and binds these symbols with ctypes
 * (INTEGRATION.md shows the binding).
 *
 * Conventions:
 *   - every pointer argument named d_* is DEVICE memory owned by the caller;
 *     host structs are passed by pointer and read before return;
 *   - functions never allocate: scratch comes from the caller, sized by the
 *     matching *_workspace_bytes query;
 *   - work is enqueued on `stream` (a cudaStream_t, NULL = legacy default)
 *     and the call returns without synchronising;
 *   - return value: SS_OK, or a negative SS_E* code (invalid argument,
 *     capacity overflow, CUDA launch error); data-dependent failures that
 *     the reference raises as exceptions (non-finite parameters, zero-norm
 *     quaternions, non-finite gradients, pair-capacity overflow) are
 *     reported through a device error block (ss_status) that the caller
 *     reads at its next synchronisation point, so a whole iteration stays
 *     capturable in one CUDA graph;
 *   - no global mutable state: calls are thread-compatible.
 */
#ifndef SPLATSTREAM_B200_H
#define SPLATSTREAM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_OK 0
#define SS_EINVAL (-1)
#define SS_ECUDA (-2)
#define SS_ECAPACITY (-3)

#define SS_ABI_VERSION 2

/* Device status block, zeroed/initialised by ss_status_reset.  Index words
 * hold INT64_MAX when no failure was seen. */
typedef struct ss_status {
    int64_t first_nonfinite_param;  /* api.py:127-129  ValueError("non-finite parameter in primitive i") */
    int64_t first_zero_quat;        /* projection.py:99-102 ValueError("zero-norm quaternion at primitive i") */
    int64_t first_nonfinite_grad;   /* api.py:74-79 / optimizer.py:111-113 FloatingPointError */
    int64_t pair_count;             /* P of the last binning (tiles.py:48-50) */
    int64_t pair_overflow;          /* 1 when P exceeded the caller's pair capacity */
    int64_t bucket_count;           /* number of (tile, bucket) backward work units */
    int64_t visible_count;          /* M = rows of the reference's Projection */
    int64_t reserved;               /* backward work-unit counter */
    double opacity_sum;             /* sum of sigmoid(opacity logit) over all Gaussians at
                                       ss_preprocess, i.e. before the step's update
                                       (opacity regulariser value, losses.py:157-168) */
    int64_t reserved2;
} ss_status;

/* Gaussian map in structure-of-arrays float32 (core.py:120-128; SH split
 * into the optimizer's sh_dc / sh_rest views, optimizer.py:79-87). */
typedef struct ss_map {
    int64_t n;
    float *d_positions;      /* (n,3) */
    float *d_rotations;      /* (n,4) w,x,y,z */
    float *d_log_scales;     /* (n,3) */
    float *d_opacity_logits; /* (n,)  */
    float *d_sh_dc;          /* (n,3) coefficient 0 */
    float *d_sh_rest;        /* (n,45) coefficients 1..15, coefficient-major */
    float *d_grad2d_accum;   /* (n,)  densify statistics (core.py:126-128) */
    float *d_grad3d_accum;   /* (n,3) */
    int32_t *d_obs_count;    /* (n,)  */
} ss_map;

/* Pinhole camera, x_cam = R x_world + t (core.py:244-274). */
typedef struct ss_camera {
    float fx, fy, cx, cy;
    int32_t width, height;
    float R[9];
    float t[3];
    float center[3]; /* -R^T t */
} ss_camera;

/* RasterOpts (api.py:37-52) plus the extensions. */
typedef struct ss_raster_opts {
    int32_t tile_size;   /* must be 16 */
    int32_t bucket_size; /* must be 32 */
    float t_min;
    float alpha_min;
    float alpha_max;
    float background[3];
    int32_t sh_degree;
    float near_plane;
    float dilation;
    int32_t with_depth;  /* builder extension A15: blend D = sum z a T */
} ss_raster_opts;

/* Per-Gaussian preprocess outputs (K1). */
typedef struct ss_splats {
    void *d_rec;          /* SplatRec[n], 48 B each (see csrc/common.cuh) */
    uint32_t *d_depth_key;/* [n] float bits of camera z; 0xFFFFFFFF when culled */
    uint32_t *d_tiles;    /* [n] touched-tile count (0 when culled) */
    uint32_t *d_rect;     /* [n*2] (x0 | y0<<16, x1 | y1<<16) inclusive tile rect */
    uint8_t *d_flags;     /* [n] bit0 visible, bits1..3 rgb_active (projection.py:154) */
    float *d_aux;         /* optional [n*8]: t_cam xyz, cov2d a b c, radius, 0 */
} ss_splats;

/* Binning outputs (K2-K4b). */
typedef struct ss_bins {
    int64_t pair_capacity;
    uint32_t *d_pair_splat;  /* [pair_capacity] Gaussian index, sorted by (tile, depth, index) */
    uint32_t *d_tile_start;  /* [n_tiles] */
    uint32_t *d_tile_end;    /* [n_tiles] */
    uint32_t *d_ckpt_base;   /* [n_tiles+1] exclusive scan of ceil(len/32) */
    /* Optional forward schedule (both or neither; n_tiles <= SS_ORDER_MAX_TILES):
     * d_tile_cost receives each tile's blend cost from ss_blend_forward
     * (SM cycles), ss_bin_sort turns the last costs into d_tile_order (the
     * permutation of tiles the forward's CTAs take, costliest first).  The
     * caller initialises d_tile_order to the identity and d_tile_cost to 0.
     * Results do not depend on the order; only the kernel's tail does. */
    uint32_t *d_tile_order;  /* [n_tiles] */
    uint32_t *d_tile_cost;   /* [n_tiles] */
} ss_bins;
#define SS_ORDER_MAX_TILES 16384

/* ---------------------------------------------------------------- status */
int ss_abi_version(void);
/* Initialise a device ss_status block. */
int ss_status_reset(ss_status *d_status, void *stream);

/* ------------------------------------------------------------ preprocess */
/* Replaces project_map (projection.py:73-163) + the finite check of
 * rasterize_forward (api.py:127-129, core.py:231-241).  d_cam (optional):
 * a DEVICE copy of the camera read by the kernel instead of *cam, so a
 * captured CUDA graph can be replayed for a new view after a host->device
 * copy of the camera. */
int ss_preprocess(const ss_map *map, const ss_camera *cam, const ss_camera *d_cam,
                  const ss_raster_opts *opts, const ss_splats *out, ss_status *d_status,
                  void *stream);

/* ----------------------------------------------------------------- binning */
/* Replaces build_tile_index (tiles.py:29-65): duplicate-with-keys, stable
 * radix sort equal to np.lexsort((index, depth, tile)) (tiles.py:58), tile
 * ranges, plus the checkpoint slot bases rasterize_forward sizes per tile
 * (api.py:168-185). */
size_t ss_bin_workspace_bytes(int64_t n, int64_t pair_capacity, int32_t n_tiles);
int ss_bin_sort(int64_t n, const ss_splats *splats, const ss_camera *cam, const ss_bins *bins,
                void *d_workspace, size_t workspace_bytes, ss_status *d_status, void *stream);
/* The forward's tile order alone (d_tile_cost -> d_tile_order, costliest
 * first), so a caller can compute it off the critical path -- e.g. on a
 * side stream during ss_preprocess -- and pass ss_bin_sort a ss_bins with
 * d_tile_cost = NULL (ss_bin_sort then leaves d_tile_order as it is).
 * Needs both pointers and n_tiles <= SS_ORDER_MAX_TILES. */
int ss_tile_order(const ss_camera *cam, const ss_bins *bins, void *stream);

/* Parity / drop-in entry for build_tile_index (tiles.py:29-65) fed an
 * EXTERNAL projection (e.g. the oracle's, or a reference-shaped Projection
 * built elsewhere): writes the K1 outputs ss_bin_sort reads (inclusive tile
 * rect in float32 arithmetic as numpy does, tile count, depth key) for m
 * rows of float32 (mean2d (m,2), radius (m,), depth (m,) > 0); the pair list
 * then holds row indices, exactly as the reference's pair_splat. */
int ss_splats_from_projection(int64_t m, const float *d_mean2d, const float *d_radius,
                              const float *d_depth, const ss_camera *cam, const ss_splats *out,
                              void *stream);

/* ------------------------------------------------------------ blend fwd */
/* Replaces rasterize_forward's blend (api.py:135-206; forward_tile
 * kernels.py:34-109 and checkpoint_tile kernels.py:112-152).
 * Checkpoint slots (d_bins->d_ckpt_base): d_ckpt holds (T,r,g,b) float4 per
 * pixel per slot; d_ckpt_depth (depth extension) holds D; d_ckpt_mask holds,
 * per pixel per slot, the 32-bit mask of the bucket's list positions that
 * were blended into the pixel (read by the backward).  d_contributed
 * (optional, [n] uint8) marks splats blended into >= 1 pixel.
 * d_work/d_status->bucket_count receive the (tile, bucket) work units of
 * the splat-wise backward. */
int ss_blend_forward(const ss_camera *cam, const ss_raster_opts *opts, const ss_splats *splats,
                     const ss_bins *bins, float *d_image, float *d_final_t, int32_t *d_n_contrib,
                     float *d_depth, int32_t *d_k_eff, uint8_t *d_contributed, void *d_ckpt,
                     float *d_ckpt_depth, uint32_t *d_ckpt_mask, uint32_t *d_work,
                     int64_t work_capacity, ss_status *d_status, void *stream);

/* RenderOutput.contributed (api.py:82-105; set in forward_tile,
 * kernels.py:94-95) from the forward's blend masks: d_contributed[i] = 1
 * for every Gaussian that was blended into at least one pixel, else 0
 * (n entries).  d_work / work_capacity / d_status are the work list and
 * status ss_blend_forward filled.  ss_blend_forward with d_contributed ==
 * NULL skips the per-pair flag in its blend loop; this entry derives the
 * same set afterwards. */
int ss_contributed_from_masks(const ss_camera *cam, const ss_bins *bins,
                              const int32_t *d_n_contrib, const int32_t *d_k_eff,
                              const uint32_t *d_ckpt_mask, const uint32_t *d_work,
                              int64_t work_capacity, const ss_status *d_status, int64_t n,
                              uint8_t *d_contributed, void *stream);

/* Replaces replay_pixel_states (api.py:340-368; replay_tile
 * kernels.py:155-178): advance tile `tile`'s archived (T, r, g, b) from
 * checkpoint bucket from_bucket to list position pos_to with the forward's
 * arithmetic.  d_out receives (th*tw, 4) floats, the tile's in-image pixels
 * in row-major order.  d_image/d_final_t/d_n_contrib are the forward's
 * outputs (a pixel stopped before the bucket has no archived state: its
 * final state is used). */
int ss_replay_pixel_states(const ss_camera *cam, const ss_raster_opts *opts,
                           const ss_splats *splats, const ss_bins *bins, const float *d_image,
                           const float *d_final_t, const int32_t *d_n_contrib, const void *d_ckpt,
                           int32_t tile, int32_t from_bucket, int32_t pos_to, float *d_out,
                           void *stream);

/* -------------------------------------------------------------- losses */
/* Replaces compute_losses' photometric part (losses.py:137-154,198-218):
 * (1-l) mean|x-y| + l (1 - SSIM), 11x11 Gaussian window, mirror padding.
 * d_sums receives (sum |x-y|, sum SSIM) as doubles; d_grad (h,w,3) the
 * analytic gradient; optional d_pixgrad (h,w,4) float4 (g_r, g_g, g_b,
 * g . x) for ss_backward_splat (lambda_ssim != 0 only; d_grad may then be
 * NULL).  Needs height, width >= 6 when lambda_ssim != 0. */
size_t ss_loss_workspace_bytes(int32_t height, int32_t width);
int ss_loss_l1_ssim(int32_t height, int32_t width, const float *d_x, const float *d_y,
                    float lambda_ssim, float *d_grad, float *d_pixgrad, double *d_sums,
                    void *d_workspace, size_t workspace_bytes, void *stream);
/* opacity_reg (losses.py:157-168) chained through the logistic
 * (losses.py:220-223): d_grad[i] = lambda_o sigma(1-sigma)/n (written or
 * added; d_grad may be NULL); d_sum[0] receives sum sigma.  d_sum must hold
 * SS_REDUCE_DOUBLES doubles (result + per-CTA partials). */
#define SS_REDUCE_DOUBLES (2 + 2 * 592)
int ss_opacity_reg(int64_t n, const float *d_logits, float lambda_o, float *d_grad,
                   int32_t accumulate, double *d_sum, void *stream);
/* Builder extension A15: mean |D - D*| over pixels with D* > 0; gradient
 * weight * sign(D-D*) / n_valid written to d_grad_depth; d_sums[0] = sum
 * |D - D*|, d_sums[1] = n_valid; d_sums holds SS_REDUCE_DOUBLES doubles. */
int ss_depth_l1(int32_t height, int32_t width, const float *d_depth, const float *d_target,
                float weight, float *d_grad_depth, double *d_sums, void *stream);

/* --------------------------------------------------------- backward */
/* Longest-units-first schedule of the splat-wise backward's work units,
 * built from the forward's d_k_eff by one CTA (tiles counting-sorted by
 * unit count; units handed out unit-index-major) into the tail of d_work;
 * ss_backward_splat uses it when present in d_status (reset by
 * ss_status_reset / ss_status_begin_step), else the forward's list.  May run
 * concurrently with the loss kernels (it reads only d_k_eff). */
int ss_backward_schedule(const ss_camera *cam, const int32_t *d_k_eff, uint32_t *d_work,
                         int64_t work_capacity, ss_status *d_status, void *stream);

/* Replaces backward_splatwise up to the screen-space rows g2d
 * (api.py:275-336; backward_splat_tile / _splat_bucket_inner
 * kernels.py:271-373).  d_pixgrad (optional, from ss_loss_l1_ssim; its .w
 * must include g_D . D with depth) replaces reading d_grad_image/d_image.
 * d_g2d [n * g2d_cols] float, g2d_cols = 9 (10 with
 * depth), columns [rgb(3), mean2d(2), conic(3), opacity(, z)], zeroed
 * here and accumulated with one red.add row per (tile, splat). */
int ss_backward_splat(const ss_camera *cam, const ss_raster_opts *opts, const ss_splats *splats,
                      const ss_bins *bins, const float *d_image, const float *d_grad_image,
                      const float *d_pixgrad, const float *d_depth, const float *d_grad_depth,
                      const int32_t *d_n_contrib, const int32_t *d_k_eff, const void *d_ckpt,
                      const float *d_ckpt_depth, const uint32_t *d_ckpt_mask,
                      const uint32_t *d_work, int64_t work_capacity,
                      int64_t n, float *d_g2d, uint8_t *d_contributed, const ss_status *d_status,
                      void *stream);
/* The clearing ss_backward_splat does first (d_g2d rows, d_contributed when
 * non-NULL, the work-unit counter in d_status), as its own launch: run it
 * ahead of time -- e.g. on a second stream beside the loss kernels, after
 * ss_backward_schedule on that stream -- and call ss_backward_splat_ex with
 * SS_BWD_SKIP_CLEAR.  g2d_cols 9 or 10 (with depth). */
int ss_backward_clear(int64_t n, int32_t g2d_cols, float *d_g2d, uint8_t *d_contributed,
                      ss_status *d_status, void *stream);
#define SS_BWD_SKIP_CLEAR 1
/* ss_backward_splat with flags (0 or SS_BWD_SKIP_CLEAR: the rows were
 * cleared by ss_backward_clear, stream-ordered before this call). */
int ss_backward_splat_ex(const ss_camera *cam, const ss_raster_opts *opts,
                         const ss_splats *splats, const ss_bins *bins, const float *d_image,
                         const float *d_grad_image, const float *d_pixgrad,
                         const float *d_depth, const float *d_grad_depth,
                         const int32_t *d_n_contrib, const int32_t *d_k_eff, const void *d_ckpt,
                         const float *d_ckpt_depth, const uint32_t *d_ckpt_mask,
                         const uint32_t *d_work, int64_t work_capacity, int64_t n,
                         float *d_g2d, uint8_t *d_contributed, const ss_status *d_status,
                         int32_t flags, void *stream);

/* Flat per-Gaussian gradient / moment layout (planes of n floats):
 * position 3, rotation 4, log_scale 3, opacity 1, sh_dc 3, sh_rest 45. */
typedef struct ss_param_grads {
    float *d_position;
    float *d_rotation;
    float *d_log_scale;
    float *d_opacity;
    float *d_sh_dc;
    float *d_sh_rest;      /* may be NULL when sh_degree == 0 */
    float *d_pos2d_norm;   /* (n,) projection.py:294-298 */
    /* multi-view statistics increments (optional): sum over views of
     * [contributed] * pos2d_norm, [contributed] * position grad, [contributed] */
    float *d_stat_g2d;     /* (n,)  */
    float *d_stat_g3d;     /* (n,3) */
    float *d_stat_cnt;     /* (n,)  */
} ss_param_grads;

#define SS_CHAIN_STATS 1       /* fold accumulate_grad_stats into the map's statistics */
#define SS_CHAIN_ACCUMULATE 2  /* add into grads (multi-view sum) instead of overwriting */
#define SS_CHAIN_STAT_PLANES 4 /* add statistics increments into grads->d_stat_* */

/* Replaces backward_pixelwise up to g2d (api.py:227-272,
 * backward_pixel_tile kernels.py:181-268): pixel-parallel, no checkpoints
 * needed -- every pixel re-runs its forward prefix up to n_contrib; per
 * splat, the tile's pixel contributions are reduced across each warp and
 * merged as one row per (tile, list position).  The paper's ablation
 * baseline for ss_backward_splat (same per-(pixel, splat) terms).  d_g2d
 * [n * 9] float is zeroed here.  opts->with_depth must be 0. */
int ss_backward_pixel(const ss_camera *cam, const ss_raster_opts *opts, const ss_splats *splats,
                      const ss_bins *bins, const float *d_image, const float *d_grad_image,
                      const int32_t *d_n_contrib, const int32_t *d_k_eff, int64_t n,
                      float *d_g2d, void *stream);

/* Replaces chain_backward (projection.py:200-299) + _finish_backward
 * (api.py:217-224).  Options: add the opacity regulariser's gradient
 * lambda_o sigma(1-sigma)/n to every Gaussian (trainer.py:206,
 * losses.py:220-223) when lambda_o_over_n != 0; fold
 * accumulate_grad_stats (densify.py:86-100) when d_contributed != NULL and
 * accumulate_stats != 0.  Non-finite gradients are reported in d_status. */
int ss_chain_backward(const ss_map *map, const ss_camera *cam, const ss_raster_opts *opts,
                      const float *d_g2d, const uint8_t *d_flags, const uint8_t *d_contributed,
                      float lambda_o_over_n, int32_t mode /* SS_CHAIN_* bits */,
                      const ss_param_grads *grads, ss_status *d_status, void *stream);
/* After a multi-view (all-reduced) step: grad2d_accum += stat_g2d,
 * grad3d_accum += stat_g3d, obs_count += stat_cnt (densify.py:96-99). */
int ss_apply_stat_planes(const ss_map *map, const ss_param_grads *grads, void *stream);
/* Start-of-iteration status reset that keeps the sticky error and
 * pair-overflow words (the fused step skips its update while overflow is
 * set, so the host can grow the buffers and replay). */
int ss_status_begin_step(ss_status *d_status, void *stream);
/* Keyframe-sharded step: d_flags[0] = 1.0f if the pair buffers
 * overflowed, d_flags[1] = 1.0f if any error word (non-finite parameter,
 * zero-norm quaternion, non-finite gradient) is set, else 0.0f.  The two
 * floats sit at the tail of the flat gradient buffer, so the one gradient
 * all-reduce also tells every rank whether ANY rank must redo or raise. */
int ss_status_flags(const ss_status *d_status, float *d_flags, void *stream);

/* Host snapshot of one step, for reading the step's outcome without
 * stalling the stream: h_row (page-locked host memory, 11 doubles) receives
 * the 8 status words as doubles, opacity_sum, and the two loss sums of
 * ss_loss_l1_ssim (sum |x - y|, sum SSIM; zeros when d_loss_sums is NULL).
 * One kernel writes through the mapped host pointer. */
#define SS_SNAPSHOT_DOUBLES 11
int ss_step_snapshot(const ss_status *d_status, const double *d_loss_sums, double *h_row,
                     void *stream);

/* Adam hyper-parameters of one step (optimizer.py:40-76,101-133), resolved
 * on the host for the post-increment step count t. */
typedef struct ss_adam_hparams {
    float lr_position, lr_rotation, lr_log_scale, lr_opacity, lr_sh_dc, lr_sh_rest;
    float beta1, beta2, eps;
    float bias1, bias2; /* 1 - beta^t */
    int32_t update_sh_rest;
} ss_adam_hparams;

/* Replaces adam_step (optimizer.py:101-133) incl. normalize_rotations
 * (core.py:225-229), in place on the map and the moments. */
int ss_adam_step(const ss_map *map, const ss_param_grads *grads, const ss_param_grads *m,
                 const ss_param_grads *v, const ss_adam_hparams *hp, ss_status *d_status,
                 void *stream);

/* Fused K8+K9 (+stats, +opacity reg): chain -> Adam for one view without
 * materialising the gradients (single-GPU mapping iteration).  Does nothing
 * while d_status->pair_overflow is set. */
int ss_chain_adam(const ss_map *map, const ss_camera *cam, const ss_camera *d_cam,
                  const ss_raster_opts *opts, const float *d_g2d, const uint8_t *d_flags,
                  const uint8_t *d_contributed, float lambda_o_over_n, const ss_param_grads *m,
                  const ss_param_grads *v, const ss_adam_hparams *hp,
                  const ss_adam_hparams *d_hp /* optional device copy, as d_cam */,
                  ss_status *d_status, void *stream);

/* accumulate_grad_stats (densify.py:86-100). */
int ss_accumulate_grad_stats(const ss_map *map, const ss_param_grads *grads,
                             const uint8_t *d_contributed, void *stream);

/* ----------------------------------------------------------- seeding */
/* Replaces seed_from_points (densify.py:53-83) for a keyframe's point
 * cloud: d_points / d_colors (n,3) float32; outputs position (n,3),
 * rotation (n,4) = (1,0,0,0), log_scale (n,3) = log(max(mean distance to the
 * 3 nearest neighbours within the cloud, 1e-4)) (0.01 * scene_extent for a
 * lone point), opacity logit (n) = logit(0.1), sh_dc (n,3) = (c - 0.5) /
 * SH_C0.  Exact kNN (float64 distances) on a uniform cell grid.
 * *d_nonfinite (device int32) is set to 1 when a point is non-finite
 * (ValueError("non-finite point in seed cloud") in the reference). */
size_t ss_seed_workspace_bytes(int64_t n);
int ss_seed_from_points(int64_t n, const float *d_points, const float *d_colors,
                        float scene_extent, float *d_positions, float *d_rotations,
                        float *d_log_scales, float *d_opacity_logits, float *d_sh_dc,
                        int32_t *d_nonfinite, void *d_workspace, size_t workspace_bytes,
                        void *stream);

/* ------------------------------------------------------------- densify */
/* densify_and_prune (densify.py:103-173) as stream compaction, phase 1:
 * masks in float64 from the stored values (densify.py:110-117,148,158) and
 * order-preserving scans kept in d_workspace.  d_counts (int64[5], device):
 * kept, cloned, split, pruned, n_new (DensifyResult fields, densify.py:42-50).
 * d_mask (optional, [n] uint8): bit0 clone, bit1 split, bit2 keep, bit3 fresh. */
size_t ss_densify_workspace_bytes(int64_t n);
int ss_densify_count(const ss_map *map, float grad_threshold, float prune_opacity,
                     double split_scale_limit, void *d_workspace, size_t workspace_bytes,
                     int64_t *d_counts, uint8_t *d_mask, void *stream);
/* Phase 2 (same workspace): writes the new map `out` (survivors in order,
 * then clones, then split children in repeat(split_idx, 2) order;
 * capacity kept + n_new) and gathers `n_planes` extra per-Gaussian planes
 * (Adam moments, resize_for_densify optimizer.py:136-146) for survivors;
 * the caller zeroes the planes' new-entry tail and the new stats.
 * d_normals: (2 n_split, 3) standard normals (densify.py:137), or NULL to
 * draw them on the device from `seed`.  d_survivors: [kept] original indices. */
int ss_densify_apply(const ss_map *map, void *d_workspace, const float *d_normals, uint64_t seed,
                     float clone_step, float shrink_log, const ss_map *out, int32_t n_planes,
                     const float *const *planes_in, float *const *planes_out,
                     const int32_t *plane_floats, int64_t *d_survivors, void *stream);

/* The drop-in API's finite checks (ParamGrads.validate_finite, api.py:74-79;
 * adam_step, optimizer.py:111-113) in one launch over up to 8 float32
 * tensors (host arrays of device pointers and element counts): d_flags[t] =
 * 1 if tensor t holds a non-finite value, d_flags[n + t] = 1 if it holds a
 * non-zero value, else 0 (2 n int32, zeroed by the call). */
int ss_check_finite(int32_t n_tensors, const float *const *d_tensors, const int64_t *counts,
                    int32_t *d_flags, void *stream);

/* Replaces resize_for_densify (optimizer.py:136-146): for each of n_planes
 * per-Gaussian float planes (plane_floats[p] floats per row), rows
 * [0, n_surv) of planes_out[p] = rows d_survivors[i] (int64) of planes_in[p],
 * rows [n_surv, n_out) zeroed (the n_new fresh primitives); n_planes <= 16. */
int ss_resize_moments(int64_t n_out, const int64_t *d_survivors, int64_t n_surv,
                      int32_t n_planes, const float *const *planes_in, float *const *planes_out,
                      const int32_t *plane_floats, void *stream);

/* Builder extension A16: logit <- logit(min(sigma, ceiling)); opacity moments
 * zeroed (3DGS convention; absent from the reference). */
int ss_opacity_reset(const ss_map *map, float ceiling, float *d_m_opacity, float *d_v_opacity,
                     void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SPLATSTREAM_B200_H */
