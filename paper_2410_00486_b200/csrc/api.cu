// api.cu -- extern "C" entry points declared in include/splatstream_b200.h.
// Each validates its arguments, enqueues the kernels of one stage on the
// caller's stream and maps CUDA errors to SS_ECUDA.  No allocation, no
// global state.
#include <climits>

#include "common.cuh"

namespace ss {
cudaError_t launch_preprocess(const ss_map*, const ss_camera*, const ss_camera*,
                              const ss_raster_opts*, const ss_splats*, ss_status*, cudaStream_t);
size_t bin_workspace_bytes(int64_t, int64_t, int);
cudaError_t launch_tile_order(const ss_camera*, const ss_bins*, cudaStream_t);
cudaError_t launch_bin_sort(int64_t, const ss_splats*, const ss_camera*, const ss_bins*, void*,
                            size_t, ss_status*, cudaStream_t);
cudaError_t launch_blend_forward(const ss_camera*, const ss_raster_opts*, const ss_splats*,
                                 const ss_bins*, float*, float*, int32_t*, float*, int32_t*,
                                 uint8_t*, void*, float*, uint32_t*, uint32_t*, int64_t,
                                 ss_status*, cudaStream_t);
cudaError_t launch_backward_splat(const ss_camera*, const ss_raster_opts*, const ss_splats*,
                                  const ss_bins*, const float*, const float*, const float4*,
                                  const float*, const float*, const int32_t*, const int32_t*,
                                  const void*, const float*, const uint32_t*, const uint32_t*,
                                  int64_t, int64_t, float*, uint8_t*, const ss_status*, uint32_t*,
                                  bool, cudaStream_t);
cudaError_t launch_backward_clear(int64_t, int, float*, uint8_t*, uint32_t*, cudaStream_t);
cudaError_t launch_backward_pixel(const ss_camera*, const ss_raster_opts*, const ss_splats*,
                                  const ss_bins*, const float*, const float*, const int32_t*,
                                  const int32_t*, int64_t, float*, cudaStream_t);
cudaError_t launch_splats_from_projection(int64_t, const float*, const float*, const float*,
                                          const ss_camera*, const ss_splats*, cudaStream_t);
cudaError_t launch_replay(const ss_camera*, const ss_raster_opts*, const ss_splats*,
                          const ss_bins*, const float*, const float*, const int32_t*, const void*,
                          int, int, int, float*, cudaStream_t);
cudaError_t launch_contributed(const ss_camera* cam, const ss_bins* bins, const int32_t* n_contrib,
                               const int32_t* k_eff, const uint32_t* ckpt_mask,
                               const uint32_t* work, int64_t work_cap, const ss_status* st,
                               uint8_t* contributed, int64_t n, cudaStream_t s);
size_t seed_workspace_bytes(int64_t);
cudaError_t launch_seed(int64_t, const float*, const float*, float, float*, float*, float*,
                        float*, float*, int32_t*, void*, size_t, cudaStream_t);
cudaError_t launch_backward_schedule(const ss_camera*, const int32_t*, uint32_t*, int64_t,
                                     ss_status*, cudaStream_t);
size_t loss_workspace_bytes(int, int);
cudaError_t launch_loss(int, int, const float*, const float*, float, float*, float*, double*,
                        void*, size_t, cudaStream_t);
cudaError_t launch_opacity_reg(int64_t, const float*, float, float*, int, double*, double*,
                               cudaStream_t);
cudaError_t launch_depth_l1(int, int, const float*, const float*, float, float*, double*,
                            double*, cudaStream_t);
cudaError_t launch_chain(const ss_map*, const ss_camera*, const ss_raster_opts*, const float*,
                         const uint8_t*, const uint8_t*, float, int, const ss_param_grads*,
                         ss_status*, cudaStream_t);
cudaError_t launch_adam(const ss_map*, const ss_param_grads*, const ss_param_grads*,
                        const ss_param_grads*, const ss_adam_hparams*, ss_status*, cudaStream_t);
cudaError_t launch_chain_adam(const ss_map*, const ss_camera*, const ss_camera*,
                              const ss_raster_opts*, const float*, const uint8_t*, const uint8_t*,
                              float, const ss_param_grads*, const ss_param_grads*,
                              const ss_adam_hparams*, const ss_adam_hparams*, ss_status*,
                              cudaStream_t);
cudaError_t launch_stats(const ss_map*, const ss_param_grads*, const uint8_t*, cudaStream_t);
cudaError_t launch_apply_stat_planes(const ss_map*, const ss_param_grads*, cudaStream_t);
cudaError_t launch_opacity_reset(const ss_map*, float, float*, float*, cudaStream_t);
size_t densify_workspace_bytes(int64_t);
cudaError_t launch_check_finite(int, const float* const*, const int64_t*, int32_t*,
                                cudaStream_t);
cudaError_t launch_resize_moments(int64_t, const int64_t*, int64_t, int, const float* const*,
                                  float* const*, const int32_t*, cudaStream_t);
cudaError_t launch_densify_count(const ss_map*, float, float, double, void*, int64_t*, uint8_t*,
                                 cudaStream_t);
cudaError_t launch_densify_apply(const ss_map*, void*, const float*, uint64_t, float, float,
                                 const ss_map*, int, const float* const*, float* const*,
                                 const int*, int64_t, int64_t*, cudaStream_t);

__global__ void status_reset_kernel(ss_status* st) {
    st->first_nonfinite_param = LLONG_MAX;
    st->first_zero_quat = LLONG_MAX;
    st->first_nonfinite_grad = LLONG_MAX;
    st->pair_count = 0;
    st->pair_overflow = 0;
    st->bucket_count = 0;
    st->visible_count = 0;
    st->reserved = 0;
    st->opacity_sum = 0.0;
    st->reserved2 = 0;
}

__global__ void status_begin_step_kernel(ss_status* st) {
    st->pair_count = 0;
    st->bucket_count = 0;
    st->visible_count = 0;
    st->reserved = 0;
    st->opacity_sum = 0.0;
}

__global__ void status_flags_kernel(const ss_status* st, float* flags) {
    flags[0] = st->pair_overflow ? 1.f : 0.f;
    flags[1] = (st->first_nonfinite_param != LLONG_MAX || st->first_zero_quat != LLONG_MAX ||
                st->first_nonfinite_grad != LLONG_MAX) ? 1.f : 0.f;
}

__global__ void step_snapshot_kernel(const ss_status* st, const double* sums, double* row) {
    PDL_WAIT();
    const int t = threadIdx.x;
    const int64_t* w = reinterpret_cast<const int64_t*>(st);
    if (t < 8) row[t] = (double)w[t];
    if (t == 8) row[8] = st->opacity_sum;
    if (t == 9 || t == 10) row[t] = sums ? sums[t - 9] : 0.0;
}
}  // namespace ss

using namespace ss;

static inline int rc(cudaError_t e) { return e == cudaSuccess ? SS_OK : SS_ECUDA; }
static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static bool opts_ok(const ss_raster_opts* o) {
    return o && o->tile_size == kTile && o->bucket_size == kBucket && o->sh_degree >= 0 &&
           o->sh_degree <= 3;
}

extern "C" {

int ss_abi_version(void) { return SS_ABI_VERSION; }

int ss_status_reset(ss_status* d_status, void* stream) {
    if (!d_status) return SS_EINVAL;
    status_reset_kernel<<<1, 1, 0, S(stream)>>>(d_status);
    return rc(cudaGetLastError());
}

int ss_status_begin_step(ss_status* d_status, void* stream) {
    if (!d_status) return SS_EINVAL;
    status_begin_step_kernel<<<1, 1, 0, S(stream)>>>(d_status);
    return rc(cudaGetLastError());
}

int ss_status_flags(const ss_status* d_status, float* d_flags, void* stream) {
    if (!d_status || !d_flags) return SS_EINVAL;
    status_flags_kernel<<<1, 1, 0, S(stream)>>>(d_status, d_flags);
    return rc(cudaGetLastError());
}

int ss_step_snapshot(const ss_status* d_status, const double* d_loss_sums, double* h_row,
                     void* stream) {
    if (!d_status || !h_row) return SS_EINVAL;
    void* dev_row = nullptr;
    if (cudaHostGetDevicePointer(&dev_row, h_row, 0) != cudaSuccess) {
        cudaGetLastError();
        return SS_EINVAL;  // not page-locked / mapped host memory
    }
    launch_pdl(step_snapshot_kernel, dim3(1), dim3(32), 0, S(stream), d_status, d_loss_sums,
               reinterpret_cast<double*>(dev_row));
    return rc(cudaGetLastError());
}

int ss_apply_stat_planes(const ss_map* map, const ss_param_grads* grads, void* stream) {
    if (!map || !grads || !grads->d_stat_cnt || !grads->d_stat_g2d || !grads->d_stat_g3d)
        return SS_EINVAL;
    return rc(launch_apply_stat_planes(map, grads, S(stream)));
}

int ss_preprocess(const ss_map* map, const ss_camera* cam, const ss_camera* d_cam,
                  const ss_raster_opts* opts, const ss_splats* out, ss_status* d_status,
                  void* stream) {
    if (!map || !cam || !opts_ok(opts) || !out || !d_status) return SS_EINVAL;
    if (map->n < 0 || map->n > 0x7fffffffLL) return SS_EINVAL;
    return rc(launch_preprocess(map, cam, d_cam, opts, out, d_status, S(stream)));
}

size_t ss_bin_workspace_bytes(int64_t n, int64_t pair_capacity, int32_t n_tiles) {
    return bin_workspace_bytes(n, pair_capacity, n_tiles);
}

int ss_tile_order(const ss_camera* cam, const ss_bins* bins, void* stream) {
    if (!cam || !bins) return SS_EINVAL;
    return rc(launch_tile_order(cam, bins, S(stream)));
}

int ss_bin_sort(int64_t n, const ss_splats* splats, const ss_camera* cam, const ss_bins* bins,
                void* d_workspace, size_t workspace_bytes, ss_status* d_status, void* stream) {
    if (!splats || !cam || !bins || !d_status || n < 0) return SS_EINVAL;
    if (bins->pair_capacity < 0 || bins->pair_capacity > 0x3fffffffLL) return SS_EINVAL;
    int n_tiles = div_up(cam->width, kTile) * div_up(cam->height, kTile);
    if (ss_bin_workspace_bytes(n, bins->pair_capacity, n_tiles) > workspace_bytes)
        return SS_ECAPACITY;
    return rc(launch_bin_sort(n, splats, cam, bins, d_workspace, workspace_bytes, d_status,
                              S(stream)));
}

int ss_blend_forward(const ss_camera* cam, const ss_raster_opts* opts, const ss_splats* splats,
                     const ss_bins* bins, float* d_image, float* d_final_t, int32_t* d_n_contrib,
                     float* d_depth, int32_t* d_k_eff, uint8_t* d_contributed, void* d_ckpt,
                     float* d_ckpt_depth, uint32_t* d_ckpt_mask, uint32_t* d_work,
                     int64_t work_capacity, ss_status* d_status, void* stream) {
    if (!cam || !opts_ok(opts) || !splats || !bins || !d_image || !d_final_t || !d_n_contrib ||
        !d_k_eff || !d_ckpt || !d_ckpt_mask || !d_status)
        return SS_EINVAL;
    if (opts->with_depth && (!d_depth || !d_ckpt_depth)) return SS_EINVAL;
    return rc(launch_blend_forward(cam, opts, splats, bins, d_image, d_final_t, d_n_contrib,
                                   d_depth, d_k_eff, d_contributed, d_ckpt, d_ckpt_depth,
                                   d_ckpt_mask, d_work, work_capacity, d_status, S(stream)));
}

int ss_splats_from_projection(int64_t m, const float* d_mean2d, const float* d_radius,
                              const float* d_depth, const ss_camera* cam, const ss_splats* out,
                              void* stream) {
    if (!cam || !out || m < 0 || m > 0x7fffffffLL) return SS_EINVAL;
    if (m && (!d_mean2d || !d_radius || !d_depth || !out->d_rec || !out->d_depth_key ||
              !out->d_tiles || !out->d_rect || !out->d_flags))
        return SS_EINVAL;
    return rc(launch_splats_from_projection(m, d_mean2d, d_radius, d_depth, cam, out, S(stream)));
}

int ss_replay_pixel_states(const ss_camera* cam, const ss_raster_opts* opts,
                           const ss_splats* splats, const ss_bins* bins, const float* d_image,
                           const float* d_final_t, const int32_t* d_n_contrib, const void* d_ckpt,
                           int32_t tile, int32_t from_bucket, int32_t pos_to, float* d_out,
                           void* stream) {
    if (!cam || !opts_ok(opts) || !splats || !bins || !d_image || !d_final_t || !d_n_contrib ||
        !d_ckpt || !d_out || tile < 0 || from_bucket < 0 || pos_to < 0)
        return SS_EINVAL;
    if (tile >= div_up(cam->width, kTile) * div_up(cam->height, kTile)) return SS_EINVAL;
    return rc(launch_replay(cam, opts, splats, bins, d_image, d_final_t, d_n_contrib, d_ckpt, tile,
                            from_bucket, pos_to, d_out, S(stream)));
}

int ss_contributed_from_masks(const ss_camera* cam, const ss_bins* bins,
                              const int32_t* d_n_contrib, const int32_t* d_k_eff,
                              const uint32_t* d_ckpt_mask, const uint32_t* d_work,
                              int64_t work_capacity, const ss_status* d_status, int64_t n,
                              uint8_t* d_contributed, void* stream) {
    if (!cam || !bins || !d_n_contrib || !d_k_eff || !d_ckpt_mask || !d_work || !d_status ||
        !d_contributed || n < 0 || work_capacity < 0)
        return SS_EINVAL;
    if (n == 0) return SS_OK;
    return rc(launch_contributed(cam, bins, d_n_contrib, d_k_eff, d_ckpt_mask, d_work,
                                 work_capacity, d_status, d_contributed, n, S(stream)));
}

size_t ss_loss_workspace_bytes(int32_t height, int32_t width) {
    return loss_workspace_bytes(height, width);
}

int ss_loss_l1_ssim(int32_t height, int32_t width, const float* d_x, const float* d_y,
                    float lambda_ssim, float* d_grad, float* d_pixgrad, double* d_sums,
                    void* d_workspace, size_t workspace_bytes, void* stream) {
    if (!d_x || !d_y || !d_sums || height <= 0 || width <= 0) return SS_EINVAL;
    if (!d_grad && !d_pixgrad) return SS_EINVAL;  // d_grad may be NULL when d_pixgrad is given
    if (lambda_ssim != 0.0f && (height < 6 || width < 6)) return SS_EINVAL;
    if (workspace_bytes < loss_workspace_bytes(height, width)) return SS_ECAPACITY;
    if (d_pixgrad && lambda_ssim == 0.0f) return SS_EINVAL;
    return rc(launch_loss(height, width, d_x, d_y, lambda_ssim, d_grad, d_pixgrad, d_sums,
                          d_workspace, workspace_bytes, S(stream)));
}

int ss_opacity_reg(int64_t n, const float* d_logits, float lambda_o, float* d_grad,
                   int32_t accumulate, double* d_sum, void* stream) {
    // d_sum must hold 2 + 2*592 doubles (result + per-CTA partials)
    if (!d_sum || n < 0 || (n > 0 && !d_logits)) return SS_EINVAL;
    return rc(launch_opacity_reg(n, d_logits, lambda_o, d_grad, accumulate, d_sum, d_sum + 2,
                                 S(stream)));
}

int ss_depth_l1(int32_t height, int32_t width, const float* d_depth, const float* d_target,
                float weight, float* d_grad_depth, double* d_sums, void* stream) {
    // d_sums must hold 2 + 2*592 doubles
    if (!d_depth || !d_target || !d_grad_depth || !d_sums) return SS_EINVAL;
    return rc(launch_depth_l1(height, width, d_depth, d_target, weight, d_grad_depth, d_sums,
                              d_sums + 2, S(stream)));
}

int ss_backward_schedule(const ss_camera* cam, const int32_t* d_k_eff, uint32_t* d_work,
                         int64_t work_capacity, ss_status* d_status, void* stream) {
    if (!cam || !d_k_eff || !d_work || work_capacity <= 0 || !d_status) return SS_EINVAL;
    return rc(launch_backward_schedule(cam, d_k_eff, d_work, work_capacity, d_status,
                                       S(stream)));
}

int ss_backward_clear(int64_t n, int32_t g2d_cols, float* d_g2d, uint8_t* d_contributed,
                      ss_status* d_status, void* stream) {
    if (n < 0 || (g2d_cols != 9 && g2d_cols != 10) || !d_g2d || !d_status) return SS_EINVAL;
    uint32_t* counter = reinterpret_cast<uint32_t*>(&d_status->reserved);
    return rc(launch_backward_clear(n, g2d_cols, d_g2d, d_contributed, counter, S(stream)));
}

int ss_backward_splat(const ss_camera* cam, const ss_raster_opts* opts, const ss_splats* splats,
                      const ss_bins* bins, const float* d_image, const float* d_grad_image,
                      const float* d_pixgrad, const float* d_depth, const float* d_grad_depth,
                      const int32_t* d_n_contrib, const int32_t* d_k_eff, const void* d_ckpt,
                      const float* d_ckpt_depth, const uint32_t* d_ckpt_mask,
                      const uint32_t* d_work, int64_t work_capacity,
                      int64_t n, float* d_g2d, uint8_t* d_contributed, const ss_status* d_status,
                      void* stream) {
    return ss_backward_splat_ex(cam, opts, splats, bins, d_image, d_grad_image, d_pixgrad,
                                d_depth, d_grad_depth, d_n_contrib, d_k_eff, d_ckpt,
                                d_ckpt_depth, d_ckpt_mask, d_work, work_capacity, n, d_g2d,
                                d_contributed, d_status, 0, stream);
}

int ss_backward_splat_ex(const ss_camera* cam, const ss_raster_opts* opts,
                         const ss_splats* splats, const ss_bins* bins, const float* d_image,
                         const float* d_grad_image, const float* d_pixgrad,
                         const float* d_depth, const float* d_grad_depth,
                         const int32_t* d_n_contrib, const int32_t* d_k_eff, const void* d_ckpt,
                         const float* d_ckpt_depth, const uint32_t* d_ckpt_mask,
                         const uint32_t* d_work, int64_t work_capacity, int64_t n,
                         float* d_g2d, uint8_t* d_contributed, const ss_status* d_status,
                         int32_t flags, void* stream) {
    if (flags & ~SS_BWD_SKIP_CLEAR) return SS_EINVAL;
    if (!cam || !opts_ok(opts) || !splats || !bins || !d_image || !d_grad_image ||
        !d_n_contrib || !d_k_eff || !d_ckpt || !d_ckpt_mask || !d_work || !d_g2d || !d_status)
        return SS_EINVAL;
    if (opts->with_depth && (!d_depth || !d_ckpt_depth)) return SS_EINVAL;
    // the work counter lives in the status block's reserved word
    uint32_t* counter = reinterpret_cast<uint32_t*>(const_cast<int64_t*>(&d_status->reserved));
    return rc(launch_backward_splat(cam, opts, splats, bins, d_image, d_grad_image,
                                    reinterpret_cast<const float4*>(d_pixgrad), d_depth,
                                    d_grad_depth, d_n_contrib, d_k_eff, d_ckpt, d_ckpt_depth,
                                    d_ckpt_mask, d_work, work_capacity, n, d_g2d, d_contributed,
                                    d_status, counter, !(flags & SS_BWD_SKIP_CLEAR), S(stream)));
}

int ss_backward_pixel(const ss_camera* cam, const ss_raster_opts* opts, const ss_splats* splats,
                      const ss_bins* bins, const float* d_image, const float* d_grad_image,
                      const int32_t* d_n_contrib, const int32_t* d_k_eff, int64_t n,
                      float* d_g2d, void* stream) {
    if (!cam || !opts_ok(opts) || opts->with_depth || !splats || !bins || !d_image ||
        !d_grad_image || !d_n_contrib || !d_k_eff || !d_g2d || n < 0)
        return SS_EINVAL;
    return rc(launch_backward_pixel(cam, opts, splats, bins, d_image, d_grad_image, d_n_contrib,
                                    d_k_eff, n, d_g2d, S(stream)));
}

int ss_chain_backward(const ss_map* map, const ss_camera* cam, const ss_raster_opts* opts,
                      const float* d_g2d, const uint8_t* d_flags, const uint8_t* d_contributed,
                      float lambda_o_over_n, int32_t mode,
                      const ss_param_grads* grads, ss_status* d_status, void* stream) {
    if (!map || !cam || !opts_ok(opts) || !d_g2d || !d_flags || !grads || !d_status)
        return SS_EINVAL;
    return rc(launch_chain(map, cam, opts, d_g2d, d_flags, d_contributed, lambda_o_over_n, mode,
                           grads, d_status, S(stream)));
}

int ss_adam_step(const ss_map* map, const ss_param_grads* grads, const ss_param_grads* m,
                 const ss_param_grads* v, const ss_adam_hparams* hp, ss_status* d_status,
                 void* stream) {
    if (!map || !grads || !m || !v || !hp || !d_status) return SS_EINVAL;
    return rc(launch_adam(map, grads, m, v, hp, d_status, S(stream)));
}

int ss_chain_adam(const ss_map* map, const ss_camera* cam, const ss_camera* d_cam,
                  const ss_raster_opts* opts, const float* d_g2d, const uint8_t* d_flags,
                  const uint8_t* d_contributed, float lambda_o_over_n, const ss_param_grads* m,
                  const ss_param_grads* v, const ss_adam_hparams* hp,
                  const ss_adam_hparams* d_hp, ss_status* d_status, void* stream) {
    if (!map || !cam || !opts_ok(opts) || !d_g2d || !d_flags || !m || !v || !hp || !d_status)
        return SS_EINVAL;
    return rc(launch_chain_adam(map, cam, d_cam, opts, d_g2d, d_flags, d_contributed,
                                lambda_o_over_n, m, v, hp, d_hp, d_status, S(stream)));
}

int ss_accumulate_grad_stats(const ss_map* map, const ss_param_grads* grads,
                             const uint8_t* d_contributed, void* stream) {
    if (!map || !grads || !d_contributed || !grads->d_pos2d_norm) return SS_EINVAL;
    return rc(launch_stats(map, grads, d_contributed, S(stream)));
}

size_t ss_densify_workspace_bytes(int64_t n) { return densify_workspace_bytes(n); }

int ss_densify_count(const ss_map* map, float grad_threshold, float prune_opacity,
                     double split_scale_limit, void* d_workspace, size_t workspace_bytes,
                     int64_t* d_counts, uint8_t* d_mask, void* stream) {
    if (!map || !d_workspace || !d_counts) return SS_EINVAL;
    if (workspace_bytes < densify_workspace_bytes(map->n)) return SS_ECAPACITY;
    return rc(launch_densify_count(map, grad_threshold, prune_opacity, split_scale_limit,
                                   d_workspace, d_counts, d_mask, S(stream)));
}

int ss_densify_apply(const ss_map* map, void* d_workspace, const float* d_normals,
                     uint64_t seed, float clone_step, float shrink_log, const ss_map* out,
                     int32_t n_planes, const float* const* planes_in, float* const* planes_out,
                     const int32_t* plane_floats, int64_t* d_survivors, void* stream) {
    if (!map || !d_workspace || !out || n_planes < 0 || n_planes > 16) return SS_EINVAL;
    return rc(launch_densify_apply(map, d_workspace, d_normals, seed, clone_step, shrink_log,
                                   out, n_planes, planes_in, planes_out, plane_floats, 0,
                                   d_survivors, S(stream)));
}

int ss_check_finite(int32_t n_tensors, const float* const* d_tensors, const int64_t* counts,
                    int32_t* d_flags, void* stream) {
    if (n_tensors < 1 || n_tensors > 8 || !d_tensors || !counts || !d_flags) return SS_EINVAL;
    for (int t = 0; t < n_tensors; ++t)
        if (counts[t] < 0 || (counts[t] > 0 && !d_tensors[t])) return SS_EINVAL;
    return rc(launch_check_finite(n_tensors, d_tensors, counts, d_flags, S(stream)));
}

int ss_resize_moments(int64_t n_out, const int64_t* d_survivors, int64_t n_surv,
                      int32_t n_planes, const float* const* planes_in, float* const* planes_out,
                      const int32_t* plane_floats, void* stream) {
    if (n_out < 0 || n_surv < 0 || n_surv > n_out || n_planes < 0 || n_planes > 16)
        return SS_EINVAL;
    if (n_surv > 0 && !d_survivors) return SS_EINVAL;
    for (int p = 0; p < n_planes; ++p)
        if (!planes_out[p] || (n_surv > 0 && !planes_in[p]) || plane_floats[p] < 1)
            return SS_EINVAL;
    return rc(launch_resize_moments(n_out, d_survivors, n_surv, n_planes, planes_in, planes_out,
                                    plane_floats, S(stream)));
}

int ss_opacity_reset(const ss_map* map, float ceiling, float* d_m_opacity, float* d_v_opacity,
                     void* stream) {
    if (!map || !(ceiling > 0.f && ceiling < 1.f)) return SS_EINVAL;
    return rc(launch_opacity_reset(map, ceiling, d_m_opacity, d_v_opacity, S(stream)));
}

}  // extern "C"

size_t ss_seed_workspace_bytes(int64_t n) { return n < 0 ? 0 : seed_workspace_bytes(n); }

int ss_seed_from_points(int64_t n, const float* d_points, const float* d_colors,
                        float scene_extent, float* d_positions, float* d_rotations,
                        float* d_log_scales, float* d_opacity_logits, float* d_sh_dc,
                        int32_t* d_nonfinite, void* d_workspace, size_t workspace_bytes,
                        void* stream) {
    if (n < 0 || !d_nonfinite || !d_workspace) return SS_EINVAL;
    if (n > 0 && (!d_points || !d_colors || !d_positions || !d_rotations || !d_log_scales ||
                  !d_opacity_logits || !d_sh_dc))
        return SS_EINVAL;
    if (n >= (int64_t)1 << 31) return SS_EINVAL;
    if (workspace_bytes < seed_workspace_bytes(n)) return SS_ECAPACITY;
    return rc(launch_seed(n, d_points, d_colors, scene_extent, d_positions, d_rotations,
                          d_log_scales, d_opacity_logits, d_sh_dc, d_nonfinite, d_workspace,
                          workspace_bytes, S(stream)));
}
