/*
 * splat_oracle.c -- CPU restatement of the splatstream mapping hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle for the CUDA
 * product path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product package
 * never links or calls it.
 *
 * It restates, in float64 (the reference trainer's working dtype,
 * rasterizer/api.py:50 and trainer.py:147-151), the algorithms of the
 * reference package `splatstream` under /root/reference/pkg/src/splatstream:
 *
 *   orc_project          rasterizer/projection.py:73-163   (project_map)
 *   orc_tile_index_*     rasterizer/tiles.py:29-65         (build_tile_index)
 *   orc_forward          rasterizer/kernels.py:14-109      (_alpha, forward_tile)
 *                        + rasterizer/api.py:118-206       (rasterize_forward tile loop)
 *   orc_replay           rasterizer/kernels.py:155-178     (replay_tile)
 *   orc_backward_splat   rasterizer/kernels.py:271-373     (backward_splat_tile)
 *                        + rasterizer/api.py:275-337       (ordered tile merge)
 *   orc_backward_pixel   rasterizer/kernels.py:181-268     (backward_pixel_tile)
 *                        + rasterizer/api.py:227-272
 *   orc_loss             losses.py:23-134,198-228          (L1 + SSIM with analytic grad)
 *   orc_chain            rasterizer/projection.py:200-325  (chain_backward, _quat_grad)
 *   orc_adam             optimizer.py:101-133              (adam_step)
 *
 * Extensions the reference does not define,
 * restated here by the builder and therefore "parity unpinned" against
 * the reference: the depth channel of the blend (D = sum z_i a_i T_i,
 * SURVEY 8a A15) in orc_forward / orc_backward_splat when `depth` buffers
 * are non-NULL.
 *
 * Compiled with -ffp-contract=off so that no fused multiply-add changes
 * the rounding of the reference's separate numpy/numba operations.
 * Parallelism mirrors the reference's tile thread pool (api.py:25-34):
 * OpenMP over tiles, with the per-tile gradient partials merged in tile
 * order so results do not depend on the thread count (api.py:331-336).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- SH */
/* Constants: sh.py:11-28 */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792,
                                0.31539156525252005, -1.0925484305920792,
                                0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554,
                                -0.4570457994644658, 0.3731763325901154,
                                -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* Real SH basis up to degree 3 at a unit direction; sh.py:37-70. */
static void sh_basis(const double d[3], int degree, double b[16]) {
    for (int k = 0; k < 16; ++k) b[k] = 0.0;
    b[0] = SH_C0;
    if (degree < 1) return;
    double x = d[0], y = d[1], z = d[2];
    b[1] = -SH_C1 * y;
    b[2] = SH_C1 * z;
    b[3] = -SH_C1 * x;
    if (degree < 2) return;
    double xx = x * x, yy = y * y, zz = z * z;
    double xy = x * y, yz = y * z, xz = x * z;
    b[4] = SH_C2[0] * xy;
    b[5] = SH_C2[1] * yz;
    b[6] = SH_C2[2] * (2 * zz - xx - yy);
    b[7] = SH_C2[3] * xz;
    b[8] = SH_C2[4] * (xx - yy);
    if (degree < 3) return;
    b[9] = SH_C3[0] * y * (3 * xx - yy);
    b[10] = SH_C3[1] * xy * z;
    b[11] = SH_C3[2] * y * (4 * zz - xx - yy);
    b[12] = SH_C3[3] * z * (2 * zz - 3 * xx - 3 * yy);
    b[13] = SH_C3[4] * x * (4 * zz - xx - yy);
    b[14] = SH_C3[5] * z * (xx - yy);
    b[15] = SH_C3[6] * x * (xx - 3 * yy);
}

/* d basis / d direction, (16,3); sh.py:73-119. */
static void sh_basis_grad(const double d[3], int degree, double g[16][3]) {
    memset(g, 0, sizeof(double) * 48);
    if (degree < 1) return;
    double x = d[0], y = d[1], z = d[2];
    g[1][1] = -SH_C1;
    g[2][2] = SH_C1;
    g[3][0] = -SH_C1;
    if (degree < 2) return;
    g[4][0] = SH_C2[0] * y;
    g[4][1] = SH_C2[0] * x;
    g[5][1] = SH_C2[1] * z;
    g[5][2] = SH_C2[1] * y;
    g[6][0] = SH_C2[2] * -2 * x;
    g[6][1] = SH_C2[2] * -2 * y;
    g[6][2] = SH_C2[2] * 4 * z;
    g[7][0] = SH_C2[3] * z;
    g[7][2] = SH_C2[3] * x;
    g[8][0] = SH_C2[4] * 2 * x;
    g[8][1] = SH_C2[4] * -2 * y;
    if (degree < 3) return;
    double xx = x * x, yy = y * y, zz = z * z;
    g[9][0] = SH_C3[0] * 6 * x * y;
    g[9][1] = SH_C3[0] * (3 * xx - 3 * yy);
    g[10][0] = SH_C3[1] * y * z;
    g[10][1] = SH_C3[1] * x * z;
    g[10][2] = SH_C3[1] * x * y;
    g[11][0] = SH_C3[2] * -2 * x * y;
    g[11][1] = SH_C3[2] * (4 * zz - xx - 3 * yy);
    g[11][2] = SH_C3[2] * 8 * y * z;
    g[12][0] = SH_C3[3] * -6 * x * z;
    g[12][1] = SH_C3[3] * -6 * y * z;
    g[12][2] = SH_C3[3] * (6 * zz - 3 * xx - 3 * yy);
    g[13][0] = SH_C3[4] * (4 * zz - 3 * xx - yy);
    g[13][1] = SH_C3[4] * -2 * x * y;
    g[13][2] = SH_C3[4] * 8 * x * z;
    g[14][0] = SH_C3[5] * 2 * x * z;
    g[14][1] = SH_C3[5] * -2 * y * z;
    g[14][2] = SH_C3[5] * (xx - yy);
    g[15][0] = SH_C3[6] * (3 * xx - 3 * yy);
    g[15][1] = SH_C3[6] * -6 * x * y;
}

/* ------------------------------------------------------------ camera */
/* cam[] layout (filled by oracle/__init__.py from a Camera, core.py:244-301):
 *   0 fx, 1 fy, 2 cx, 3 cy, 4 width, 5 height, 6..14 R (row-major),
 *   15..17 t, 18..20 camera centre (-R^T t, core.py:271-274). */
#define CAM_FX 0
#define CAM_FY 1
#define CAM_CX 2
#define CAM_CY 3
#define CAM_W 4
#define CAM_H 5
#define CAM_R 6
#define CAM_T 15
#define CAM_C 18

/* Rotation from a unit quaternion (w,x,y,z); projection.py:166-178. */
static void rot_from_unit_quat(const double q[4], double R[3][3]) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    R[0][0] = 1 - 2 * (y * y + z * z);
    R[0][1] = 2 * (x * y - w * z);
    R[0][2] = 2 * (x * z + w * y);
    R[1][0] = 2 * (x * y + w * z);
    R[1][1] = 1 - 2 * (x * x + z * z);
    R[1][2] = 2 * (y * z - w * x);
    R[2][0] = 2 * (x * z - w * y);
    R[2][1] = 2 * (y * z + w * x);
    R[2][2] = 1 - 2 * (x * x + y * y);
}

/* Numerically stable logistic; projection.py:68-70. */
static double sigmoid(double x) {
    double e = exp(-fabs(x));
    return x >= 0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
}

/* Per-primitive projection context shared by orc_project and orc_chain. */
typedef struct {
    double t[3];       /* camera-frame centre */
    double qn, qh[4];  /* |q|, q/|q| */
    double rot[3][3];
    double s2[3];      /* exp(2 log_scale) */
    double covc[3][3]; /* camera-frame covariance */
    double a, b, c;    /* dilated 2D covariance (packed) */
} proj_ctx;

/* World->camera, quaternion normalisation, world and camera covariance,
 * perspective Jacobian and dilated 2D covariance: projection.py:86-121. */
static void project_ctx(const double *pos, const double *q, const double *ls,
                        const double *cam, double dilation, proj_ctx *o) {
    const double *R = cam + CAM_R, *tt = cam + CAM_T;
    for (int i = 0; i < 3; ++i)
        o->t[i] = pos[0] * R[3 * i + 0] + pos[1] * R[3 * i + 1] + pos[2] * R[3 * i + 2] + tt[i];
    o->qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    for (int k = 0; k < 4; ++k) o->qh[k] = q[k] / o->qn;
    rot_from_unit_quat(o->qh, o->rot);
    for (int k = 0; k < 3; ++k) o->s2[k] = exp(2.0 * ls[k]);
    double cov3[3][3];
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) {
            double s = 0.0;
            for (int j = 0; j < 3; ++j) s += o->rot[i][j] * o->s2[j] * o->rot[k][j];
            cov3[i][k] = s;
        }
    double tmp[3][3];
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) {
            double s = 0.0;
            for (int j = 0; j < 3; ++j) s += R[3 * i + j] * cov3[j][k];
            tmp[i][k] = s;
        }
    for (int i = 0; i < 3; ++i)
        for (int l = 0; l < 3; ++l) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += tmp[i][k] * R[3 * l + k];
            o->covc[i][l] = s;
        }
    double fx = cam[CAM_FX], fy = cam[CAM_FY];
    double iz = 1.0 / o->t[2], iz2 = iz * iz;
    double J[2][3] = {{fx * iz, 0.0, -fx * o->t[0] * iz2}, {0.0, fy * iz, -fy * o->t[1] * iz2}};
    double JC[2][3];
    for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 3; ++k) {
            double s = 0.0;
            for (int j = 0; j < 3; ++j) s += J[i][j] * o->covc[j][k];
            JC[i][k] = s;
        }
    double c2[2][2];
    for (int i = 0; i < 2; ++i)
        for (int l = 0; l < 2; ++l) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += JC[i][k] * J[l][k];
            c2[i][l] = s;
        }
    o->a = c2[0][0] + dilation;
    o->b = c2[0][1];
    o->c = c2[1][1] + dilation;
}

/* project_map (projection.py:73-163), per primitive, without compaction:
 * visible[i] = 1 for rows the reference keeps; the caller compacts with
 * flatnonzero to obtain map_index.  Returns 0, or -(1+i) for the first
 * primitive in front of the near plane with a zero-norm quaternion
 * (projection.py:99-102). */
int64_t orc_project(int64_t n, const double *pos, const double *rot, const double *ls,
                    const double *opl, const double *sh, const double *cam, int sh_degree,
                    double near_, double dilation, double alpha_min,
                    uint8_t *visible, double *t_cam, double *mean2d, double *cov2d,
                    double *conic, double *radius, double *sigma_out, double *rgb,
                    uint8_t *rgb_active) {
    const double *Rw = cam + CAM_R, *tt = cam + CAM_T, *ctr = cam + CAM_C;
    /* zero-norm quaternion check over the near-plane survivors, in index order */
    for (int64_t i = 0; i < n; ++i) {
        double z = pos[3 * i] * Rw[6] + pos[3 * i + 1] * Rw[7] + pos[3 * i + 2] * Rw[8] + tt[2];
        if (!(z > near_)) continue;
        const double *q = rot + 4 * i;
        if (sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) == 0.0) return -(1 + i);
    }
    const double W = cam[CAM_W], H = cam[CAM_H];
    const double lam = log(alpha_min);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        visible[i] = 0;
        double z = pos[3 * i] * Rw[6] + pos[3 * i + 1] * Rw[7] + pos[3 * i + 2] * Rw[8] + tt[2];
        if (!(z > near_)) continue;
        proj_ctx P;
        project_ctx(pos + 3 * i, rot + 4 * i, ls + 3 * i, cam, dilation, &P);
        double mx = cam[CAM_FX] * P.t[0] / P.t[2] + cam[CAM_CX];
        double my = cam[CAM_FY] * P.t[1] / P.t[2] + cam[CAM_CY];
        double det = P.a * P.c - P.b * P.b;
        double mid = (P.a + P.c) / 2;
        double disc = mid * mid - det;
        double lmax = mid + sqrt(disc > 0 ? disc : 0);
        double sg = sigmoid(opl[i]);
        double mcut = 2.0 * (log(sg) - lam);
        double r = ceil(sqrt((mcut > 0 ? mcut : 0) * lmax));
        int vis = (det > 0) && (mcut > 0) && (mx + r >= 0) && (mx - r <= W - 1) &&
                  (my + r >= 0) && (my - r <= H - 1);
        if (!vis) continue;
        visible[i] = 1;
        for (int k = 0; k < 3; ++k) t_cam[3 * i + k] = P.t[k];
        mean2d[2 * i] = mx;
        mean2d[2 * i + 1] = my;
        cov2d[3 * i] = P.a;
        cov2d[3 * i + 1] = P.b;
        cov2d[3 * i + 2] = P.c;
        conic[3 * i] = P.c / det;
        conic[3 * i + 1] = -P.b / det;
        conic[3 * i + 2] = P.a / det;
        radius[i] = r;
        sigma_out[i] = sg;
        double u[3], vl;
        for (int k = 0; k < 3; ++k) u[k] = pos[3 * i + k] - ctr[k];
        vl = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
        if (vl < 1e-12) vl = 1e-12;
        double d[3] = {u[0] / vl, u[1] / vl, u[2] / vl};
        double bs[16];
        sh_basis(d, sh_degree, bs);
        const double *s = sh + 48 * i;
        for (int ch = 0; ch < 3; ++ch) {
            double raw = 0.0;
            for (int k = 0; k < 16; ++k) raw += bs[k] * s[3 * k + ch];
            raw += 0.5;
            rgb_active[3 * i + ch] = raw > 0;
            rgb[3 * i + ch] = raw > 0 ? raw : 0.0;
        }
    }
    return 0;
}

/* ------------------------------------------------------------- tiles */
/* build_tile_index (tiles.py:29-65): inclusive tile rectangles
 * floor((m -/+ r) / tile) clipped to the grid, one (tile, depth, row)
 * triple per touched tile, ordered by tile, then depth, then row.  The
 * rectangle arithmetic runs in the dtype of the projection it is given
 * (numpy keeps float32 inputs in float32), hence the two variants. */
#define RECT_BODY(T)                                                                  \
    for (int64_t i = 0; i < m; ++i) {                                                 \
        T mx = mean2d[2 * i], my = mean2d[2 * i + 1], r = radius[i];                  \
        T ts = (T)tile;                                                               \
        double fx0 = floor((double)((T)(mx - r) / ts));                               \
        double fx1 = floor((double)((T)(mx + r) / ts));                               \
        double fy0 = floor((double)((T)(my - r) / ts));                               \
        double fy1 = floor((double)((T)(my + r) / ts));                               \
        int64_t x0 = (int64_t)(fx0 < 0 ? 0 : (fx0 > tx - 1 ? tx - 1 : fx0));          \
        int64_t x1 = (int64_t)(fx1 < 0 ? 0 : (fx1 > tx - 1 ? tx - 1 : fx1));          \
        int64_t y0 = (int64_t)(fy0 < 0 ? 0 : (fy0 > ty - 1 ? ty - 1 : fy0));          \
        int64_t y1 = (int64_t)(fy1 < 0 ? 0 : (fy1 > ty - 1 ? ty - 1 : fy1));          \
        rect[4 * i] = x0;                                                             \
        rect[4 * i + 1] = y0;                                                         \
        rect[4 * i + 2] = x1;                                                         \
        rect[4 * i + 3] = y1;                                                         \
        total += (x1 - x0 + 1) * (y1 - y0 + 1);                                       \
    }

int64_t orc_tile_rects_f64(int64_t m, const double *mean2d, const double *radius, int tile,
                           int64_t tx, int64_t ty, int64_t *rect) {
    int64_t total = 0;
    RECT_BODY(double)
    return total;
}

int64_t orc_tile_rects_f32(int64_t m, const float *mean2d, const float *radius, int tile,
                           int64_t tx, int64_t ty, int64_t *rect) {
    int64_t total = 0;
    RECT_BODY(float)
    return total;
}

typedef struct {
    int64_t tile;
    double depth;
    int32_t row;
} pair_key;

static int pair_cmp(const void *pa, const void *pb) {
    const pair_key *a = (const pair_key *)pa, *b = (const pair_key *)pb;
    if (a->tile != b->tile) return a->tile < b->tile ? -1 : 1;
    if (a->depth != b->depth) return a->depth < b->depth ? -1 : 1;
    return (a->row > b->row) - (a->row < b->row);
}

/* Emit and order the (tile, row) pairs; writes pair_splat[total] and
 * tile_range[n_tiles+1].  depth is compared as double (exact for float32
 * inputs, so the order equals numpy's on either dtype). */
void orc_tile_sort(int64_t m, const int64_t *rect, const double *depth, int64_t tx,
                   int64_t n_tiles, int64_t total, int32_t *pair_splat, int64_t *tile_range) {
    pair_key *keys = (pair_key *)malloc(sizeof(pair_key) * (total > 0 ? total : 1));
    int64_t w = 0;
    for (int64_t i = 0; i < m; ++i) {
        for (int64_t y = rect[4 * i + 1]; y <= rect[4 * i + 3]; ++y)
            for (int64_t x = rect[4 * i]; x <= rect[4 * i + 2]; ++x) {
                keys[w].tile = y * tx + x;
                keys[w].depth = depth[i];
                keys[w].row = (int32_t)i;
                ++w;
            }
    }
    qsort(keys, (size_t)total, sizeof(pair_key), pair_cmp);
    for (int64_t t = 0; t <= n_tiles; ++t) tile_range[t] = 0;
    for (int64_t k = 0; k < total; ++k) {
        pair_splat[k] = keys[k].row;
        tile_range[keys[k].tile + 1] += 1;
    }
    for (int64_t t = 0; t < n_tiles; ++t) tile_range[t + 1] += tile_range[t];
    free(keys);
}

/* ------------------------------------------------------------- blend */
typedef struct {
    const int32_t *order;
    const double *mean2d, *conic, *rgb, *sigma, *mcut, *depth;
    double amin, amax, tmin;
} splat_set;

/* _alpha (kernels.py:14-31): < 0 means "skip this pair". */
static inline double alpha_at(const splat_set *S, int32_t s, double px, double py) {
    double dx = px - S->mean2d[2 * s];
    double dy = py - S->mean2d[2 * s + 1];
    const double *c = S->conic + 3 * s;
    double m = c[0] * dx * dx + 2.0 * c[1] * dx * dy + c[2] * dy * dy;
    if (m > S->mcut[s]) return -1.0;
    double a = S->sigma[s] * exp(-0.5 * m);
    if (a < S->amin) return -1.0;
    if (a > S->amax) a = S->amax;
    return a;
}

/* Parity support (test infrastructure, not in the reference): 1 when this
 * (pixel, splat) evaluation sits within a relative `band` of one of the
 * blend's discrete decisions -- the m_cut cull, the alpha_min skip
 * (kernels.py:14-31) or the t_min termination (kernels.py:93-99) -- so a
 * float32 evaluation of the same inputs may decide it the other way.
 * "n_contrib equal except flagged threshold pixels". */
static inline int near_threshold(const splat_set *S, int32_t s, double px, double py, double T,
                                 double band) {
    double dx = px - S->mean2d[2 * s];
    double dy = py - S->mean2d[2 * s + 1];
    const double *c = S->conic + 3 * s;
    double m = c[0] * dx * dx + 2.0 * c[1] * dx * dy + c[2] * dy * dy;
    double mc = S->mcut[s];
    if (fabs(m - mc) <= band * (fabs(mc) > 1.0 ? fabs(mc) : 1.0)) return 1;
    if (m > mc) return 0;
    double a = S->sigma[s] * exp(-0.5 * m);
    if (fabs(a - S->amin) <= band * S->amin) return 1;
    if (a < S->amin) return 0;
    if (a > S->amax) a = S->amax;
    double Tn = T * (1.0 - a);
    return fabs(Tn - S->tmin) <= band * S->tmin;
}

static inline void tile_geom(int64_t tile_id, int tile, int64_t tx, int W, int H,
                             int *x0, int *y0, int *tw, int *th) {
    *y0 = (int)(tile_id / tx) * tile;
    *x0 = (int)(tile_id % tx) * tile;
    *tw = W - *x0 < tile ? W - *x0 : tile;
    *th = H - *y0 < tile ? H - *y0 : tile;
}

/* rasterize_forward's per-tile loop (api.py:153-196) around forward_tile
 * (kernels.py:34-109), with checkpoints archived eagerly in the same pass
 * for every list length (the reference's replay path, checkpoint_tile
 * kernels.py:112-152, reproduces the same states bitwise).
 *
 * ckpt_off[a] is the capacity offset (in doubles) of active tile a,
 * sized by the caller as ceil(len/bucket) * npx * stride, stride 4
 * (T, r, g, b) or 5 (T, r, g, b, D) with the depth channel.  When `depth` is
 * non-NULL a fourth accumulator D = sum z a T is blended (builder-defined
 * extension A15) into out_depth.  Returns nothing; k_eff[a] holds the
 * largest per-pixel contributing prefix (kernels.py:86-87,109). */
void orc_forward(const int32_t *order, const int64_t *tile_range, int64_t n_active,
                 const int64_t *active, const double *mean2d, const double *conic,
                 const double *rgb, const double *sigma, const double *mcut, const double *depth,
                 int W, int H, int tile, int bucket, double tmin, double amin, double amax,
                 const double *bg, double *image, double *acc, double *final_t,
                 int32_t *n_contrib, int64_t *k_eff, uint8_t *contributed, double *ckpt,
                 const int64_t *ckpt_off, double *out_depth, double band, uint8_t *thr_px) {
    splat_set S = {order, mean2d, conic, rgb, sigma, mcut, depth, amin, amax, tmin};
    int64_t tx = (W + tile - 1) / tile;
    int npx_max = tile * tile;
    int cks = depth ? 5 : 4; /* checkpoint stride: (T, r, g, b[, D]) */
#pragma omp parallel
    {
        double *st = (double *)malloc(sizeof(double) * npx_max);
        double *sc = (double *)malloc(sizeof(double) * npx_max * 4);
        int64_t *alive = (int64_t *)malloc(sizeof(int64_t) * npx_max);
#pragma omp for schedule(dynamic, 1)
        for (int64_t ai = 0; ai < n_active; ++ai) {
            int64_t tid = active[ai];
            int x0, y0, tw, th;
            tile_geom(tid, tile, tx, W, H, &x0, &y0, &tw, &th);
            int npx = tw * th;
            int64_t start = tile_range[tid], end = tile_range[tid + 1];
            double *ck = ckpt ? ckpt + ckpt_off[ai] : NULL;
            for (int p = 0; p < npx; ++p) {
                st[p] = 1.0;
                sc[4 * p] = sc[4 * p + 1] = sc[4 * p + 2] = sc[4 * p + 3] = 0.0;
                alive[p] = p;
            }
            int64_t n_alive = npx, maxc = 0;
            for (int64_t k = start; k < end; ++k) {
                int64_t q = k - start;
                if (ck && q % bucket == 0) {
                    double *cb = ck + (q / bucket) * npx * cks;
                    for (int p = 0; p < npx; ++p) {
                        cb[cks * p] = st[p];
                        cb[cks * p + 1] = sc[4 * p];
                        cb[cks * p + 2] = sc[4 * p + 1];
                        cb[cks * p + 3] = sc[4 * p + 2];
                        if (depth) cb[cks * p + 4] = sc[4 * p + 3];
                    }
                }
                int32_t s = order[k];
                int blended = 0;
                int64_t ii = 0;
                while (ii < n_alive) {
                    int64_t p = alive[ii];
                    double px = (double)(x0 + p % tw), py = (double)(y0 + p / tw);
                    double a = alpha_at(&S, s, px, py);
                    if (thr_px && near_threshold(&S, s, px, py, st[p], band))
                        thr_px[(int64_t)(y0 + p / tw) * W + x0 + p % tw] = 1;
                    if (a < 0.0) {
                        ++ii;
                        continue;
                    }
                    double T = st[p];
                    double w = a * T;
                    sc[4 * p] += rgb[3 * s] * w;
                    sc[4 * p + 1] += rgb[3 * s + 1] * w;
                    sc[4 * p + 2] += rgb[3 * s + 2] * w;
                    if (depth) sc[4 * p + 3] += depth[s] * w;
                    double Tn = T * (1.0 - a);
                    st[p] = Tn;
                    n_contrib[(int64_t)(y0 + p / tw) * W + x0 + p % tw] = (int32_t)(q + 1);
                    if (q + 1 > maxc) maxc = q + 1;
                    blended = 1;
                    if (Tn < tmin) {
                        --n_alive;
                        alive[ii] = alive[n_alive];
                    } else {
                        ++ii;
                    }
                }
                if (blended) contributed[s] = 1; /* benign same-value race, as api.py:142 */
                if (n_alive == 0) break;
            }
            for (int i = 0; i < th; ++i)
                for (int j = 0; j < tw; ++j) {
                    int p = i * tw + j;
                    int64_t o = (int64_t)(y0 + i) * W + x0 + j;
                    double T = st[p];
                    final_t[o] = T;
                    for (int c = 0; c < 3; ++c) {
                        acc[3 * o + c] = sc[4 * p + c];
                        image[3 * o + c] = sc[4 * p + c] + bg[c] * T;
                    }
                    if (out_depth) out_depth[o] = sc[4 * p + 3];
                }
            k_eff[ai] = maxc;
        }
        free(st);
        free(sc);
        free(alive);
    }
}

/* replay_tile (kernels.py:155-178): advance archived states of one tile
 * from list position pos_from to pos_to.  state is (npx, 4) = (T,r,g,b). */
void orc_replay(const int32_t *order, int64_t start, int64_t pos_from, int64_t pos_to,
                const double *mean2d, const double *conic, const double *rgb,
                const double *sigma, const double *mcut, int x0, int y0, int tw, int th,
                double tmin, double amin, double amax, double *state) {
    splat_set S = {order, mean2d, conic, rgb, sigma, mcut, NULL, amin, amax, tmin};
    for (int64_t k = pos_from; k < pos_to; ++k) {
        int32_t s = order[start + k];
        for (int i = 0; i < th; ++i)
            for (int j = 0; j < tw; ++j) {
                double *sp = state + 4 * (i * tw + j);
                double T = sp[0];
                if (T < tmin) continue;
                double a = alpha_at(&S, s, (double)(x0 + j), (double)(y0 + i));
                if (a < 0.0) continue;
                double w = a * T;
                sp[1] += rgb[3 * s] * w;
                sp[2] += rgb[3 * s + 1] * w;
                sp[3] += rgb[3 * s + 2] * w;
                sp[0] = T * (1.0 - a);
            }
    }
}

/* Ordered merge of per-tile partial rows into g2d (api.py:331-336). */
static void merge_partials(const int32_t *order, const int64_t *tile_range, int64_t n_active,
                           const int64_t *active, const int64_t *k_eff, const int64_t *poff,
                           const double *partial, int ncol, double *g2d) {
    for (int64_t ai = 0; ai < n_active; ++ai) {
        int64_t start = tile_range[active[ai]];
        for (int64_t k = 0; k < k_eff[ai]; ++k) {
            int32_t s = order[start + k];
            for (int c = 0; c < ncol; ++c) g2d[(int64_t)s * ncol + c] += partial[poff[ai] + k * ncol + c];
        }
    }
}

/* backward_splatwise (api.py:275-337) over backward_splat_tile /
 * _splat_bucket_inner (kernels.py:271-373): each (tile, bucket) restores
 * pixel states from its checkpoint, replays its splats over the tile's
 * pixels and accumulates each splat's 9 screen-space gradients privately
 * [rgb(3), mean2d(2), conic(3), opacity]; partial rows merge in tile order.
 * With `depth` (extension A15) a 10th column dL/dz and the depth
 * channel's term in dL/dalpha are added (ncol = 10). */
void orc_backward_splat(const int32_t *order, const int64_t *tile_range, int64_t n_active,
                        const int64_t *active, const int64_t *k_eff, const double *ckpt,
                        const int64_t *ckpt_off, const double *mean2d, const double *conic,
                        const double *rgb, const double *sigma, const double *mcut,
                        const double *depth, int W, int H, int tile, int bucket, double amin,
                        double amax, const double *grad_image, const double *image,
                        const int32_t *n_contrib, const double *grad_depth,
                        const double *out_depth, int64_t m, double *g2d) {
    splat_set S = {order, mean2d, conic, rgb, sigma, mcut, depth, amin, amax, 0.0};
    int ncol = depth ? 10 : 9;
    int cks = depth ? 5 : 4;
    int64_t tx = (W + tile - 1) / tile;
    int64_t *poff = (int64_t *)malloc(sizeof(int64_t) * (n_active + 1));
    poff[0] = 0;
    for (int64_t ai = 0; ai < n_active; ++ai) poff[ai + 1] = poff[ai] + k_eff[ai] * ncol;
    double *partial = (double *)calloc((size_t)(poff[n_active] > 0 ? poff[n_active] : 1), sizeof(double));
    int npx_max = tile * tile;
#pragma omp parallel
    {
        double *st = (double *)malloc(sizeof(double) * npx_max * 5);
#pragma omp for schedule(dynamic, 1)
        for (int64_t ai = 0; ai < n_active; ++ai) {
            int64_t ke = k_eff[ai];
            int64_t nb = (ke + bucket - 1) / bucket;
            if (nb == 0) continue;
            int x0, y0, tw, th;
            tile_geom(active[ai], tile, tx, W, H, &x0, &y0, &tw, &th);
            int npx = tw * th;
            int64_t start = tile_range[active[ai]];
            double *part = partial + poff[ai];
            for (int64_t b = 0; b < nb; ++b) {
                const double *cb = ckpt + ckpt_off[ai] + b * npx * cks;
                for (int p = 0; p < npx; ++p)
                    for (int e = 0; e < 5; ++e) st[5 * p + e] = e < cks ? cb[cks * p + e] : 0.0;
                int64_t lo = b * bucket, hi = lo + bucket < ke ? lo + bucket : ke;
                for (int64_t k = lo; k < hi; ++k) {
                    int32_t s = order[start + k];
                    double acc[10] = {0};
                    for (int c = 0; c < ncol; ++c) acc[c] = part[k * ncol + c];
                    for (int i = 0; i < th; ++i) {
                        double py = (double)(y0 + i);
                        for (int j = 0; j < tw; ++j) {
                            int p = i * tw + j;
                            int64_t o = (int64_t)(y0 + i) * W + x0 + j;
                            if (k >= n_contrib[o]) continue;
                            double px = (double)(x0 + j);
                            double a = alpha_at(&S, s, px, py);
                            if (a < 0.0) continue;
                            double *sp = st + 5 * p;
                            double T = sp[0];
                            double w = a * T;
                            sp[1] = sp[1] + rgb[3 * s] * w;
                            sp[2] = sp[2] + rgb[3 * s + 1] * w;
                            sp[3] = sp[3] + rgb[3 * s + 2] * w;
                            if (depth) sp[4] = sp[4] + depth[s] * w;
                            sp[0] = T * (1.0 - a);
                            double g0 = grad_image[3 * o], g1 = grad_image[3 * o + 1],
                                   g2 = grad_image[3 * o + 2];
                            double gd = grad_depth ? grad_depth[o] : 0.0;
                            if (g0 == 0.0 && g1 == 0.0 && g2 == 0.0 && gd == 0.0) continue;
                            acc[0] += w * g0;
                            acc[1] += w * g1;
                            acc[2] += w * g2;
                            if (depth) acc[9] += w * gd;
                            double am1 = 1.0 - a;
                            if (am1 > 0.0 && a != amax) {
                                double s0 = image[3 * o] - sp[1];
                                double s1 = image[3 * o + 1] - sp[2];
                                double s2c = image[3 * o + 2] - sp[3];
                                double dal = (rgb[3 * s] * T - s0 / am1) * g0 +
                                             (rgb[3 * s + 1] * T - s1 / am1) * g1 +
                                             (rgb[3 * s + 2] * T - s2c / am1) * g2;
                                if (depth) /* depth channel: D = sum z a T, no background */
                                    dal += (depth[s] * T - (out_depth[o] - sp[4]) / am1) * gd;
                                double dx = px - mean2d[2 * s], dy = py - mean2d[2 * s + 1];
                                acc[8] += dal * (a / sigma[s]);
                                const double *cq = conic + 3 * s;
                                double qdx = cq[0] * dx + cq[1] * dy;
                                double qdy = cq[1] * dx + cq[2] * dy;
                                double da = dal * a;
                                acc[3] += da * qdx;
                                acc[4] += da * qdy;
                                double h = -0.5 * da;
                                acc[5] += h * dx * dx;
                                acc[6] += h * 2.0 * dx * dy;
                                acc[7] += h * dy * dy;
                            }
                        }
                    }
                    for (int c = 0; c < ncol; ++c) part[k * ncol + c] = acc[c];
                }
            }
        }
        free(st);
    }
    memset(g2d, 0, sizeof(double) * (size_t)m * ncol);
    merge_partials(order, tile_range, n_active, active, k_eff, poff, partial, ncol, g2d);
    free(partial);
    free(poff);
    (void)H;
}

/* backward_pixelwise (api.py:227-272) over backward_pixel_tile
 * (kernels.py:181-268): per pixel, re-run the forward prefix stashing
 * (alpha, T, colour-after), then walk it in reverse adding into the
 * tile's shared rows. */
void orc_backward_pixel(const int32_t *order, const int64_t *tile_range, int64_t n_active,
                        const int64_t *active, const int64_t *k_eff, const double *mean2d,
                        const double *conic, const double *rgb, const double *sigma,
                        const double *mcut, int W, int H, int tile, double amin, double amax,
                        const double *grad_image, const double *image, const int32_t *n_contrib,
                        int64_t m, double *g2d) {
    splat_set S = {order, mean2d, conic, rgb, sigma, mcut, NULL, amin, amax, 0.0};
    int64_t tx = (W + tile - 1) / tile;
    int64_t *poff = (int64_t *)malloc(sizeof(int64_t) * (n_active + 1));
    int64_t kmax = 0;
    poff[0] = 0;
    for (int64_t ai = 0; ai < n_active; ++ai) {
        poff[ai + 1] = poff[ai] + k_eff[ai] * 9;
        if (k_eff[ai] > kmax) kmax = k_eff[ai];
    }
    double *partial = (double *)calloc((size_t)(poff[n_active] > 0 ? poff[n_active] : 1), sizeof(double));
#pragma omp parallel
    {
        double *sa = (double *)malloc(sizeof(double) * (kmax + 1));
        double *stt = (double *)malloc(sizeof(double) * (kmax + 1));
        double *scc = (double *)malloc(sizeof(double) * 3 * (kmax + 1));
#pragma omp for schedule(dynamic, 1)
        for (int64_t ai = 0; ai < n_active; ++ai) {
            int x0, y0, tw, th;
            tile_geom(active[ai], tile, tx, W, H, &x0, &y0, &tw, &th);
            int64_t start = tile_range[active[ai]];
            double *part = partial + poff[ai];
            for (int i = 0; i < th; ++i) {
                double py = (double)(y0 + i);
                for (int j = 0; j < tw; ++j) {
                    int64_t o = (int64_t)(y0 + i) * W + x0 + j;
                    int64_t nj = n_contrib[o];
                    if (nj == 0) continue;
                    double g0 = grad_image[3 * o], g1 = grad_image[3 * o + 1], g2 = grad_image[3 * o + 2];
                    if (g0 == 0.0 && g1 == 0.0 && g2 == 0.0) continue;
                    double px = (double)(x0 + j);
                    double T = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
                    for (int64_t k = 0; k < nj; ++k) {
                        int32_t s = order[start + k];
                        double a = alpha_at(&S, s, px, py);
                        if (a < 0.0) {
                            sa[k] = 0.0;
                        } else {
                            sa[k] = a;
                            stt[k] = T;
                            double w = a * T;
                            scc[3 * k] = c0 + rgb[3 * s] * w;
                            scc[3 * k + 1] = c1 + rgb[3 * s + 1] * w;
                            scc[3 * k + 2] = c2 + rgb[3 * s + 2] * w;
                            c0 = scc[3 * k];
                            c1 = scc[3 * k + 1];
                            c2 = scc[3 * k + 2];
                            T = stt[k] * (1.0 - a);
                        }
                    }
                    for (int64_t k = nj - 1; k >= 0; --k) {
                        double a = sa[k];
                        if (a == 0.0) continue;
                        int32_t s = order[start + k];
                        double Tk = stt[k], w = a * Tk;
                        double *r = part + k * 9;
                        r[0] += w * g0;
                        r[1] += w * g1;
                        r[2] += w * g2;
                        double am1 = 1.0 - a;
                        if (am1 > 0.0 && a != amax) {
                            double s0 = image[3 * o] - scc[3 * k];
                            double s1 = image[3 * o + 1] - scc[3 * k + 1];
                            double s2c = image[3 * o + 2] - scc[3 * k + 2];
                            double dal = (rgb[3 * s] * Tk - s0 / am1) * g0 +
                                         (rgb[3 * s + 1] * Tk - s1 / am1) * g1 +
                                         (rgb[3 * s + 2] * Tk - s2c / am1) * g2;
                            double dx = px - mean2d[2 * s], dy = py - mean2d[2 * s + 1];
                            r[8] += dal * (a / sigma[s]);
                            const double *cq = conic + 3 * s;
                            double qdx = cq[0] * dx + cq[1] * dy;
                            double qdy = cq[1] * dx + cq[2] * dy;
                            double da = dal * a;
                            r[3] += da * qdx;
                            r[4] += da * qdy;
                            double h = -0.5 * da;
                            r[5] += h * dx * dx;
                            r[6] += h * 2.0 * dx * dy;
                            r[7] += h * dy * dy;
                        }
                    }
                }
            }
        }
        free(sa);
        free(stt);
        free(scc);
    }
    memset(g2d, 0, sizeof(double) * (size_t)m * 9);
    merge_partials(order, tile_range, n_active, active, k_eff, poff, partial, 9, g2d);
    free(partial);
    free(poff);
    (void)H;
}

/* -------------------------------------------------------------- loss */
/* SSIM window and reflection padding: losses.py:16-41. */
#define SSIM_WIN 11
static void ssim_window(double w[SSIM_WIN]) {
    double s = 0.0;
    for (int m = 0; m < SSIM_WIN; ++m) {
        double x = m - (SSIM_WIN - 1) / 2.0;
        w[m] = exp(-(x * x) / (2 * 1.5 * 1.5));
        s += w[m];
    }
    for (int m = 0; m < SSIM_WIN; ++m) w[m] /= s;
}

/* symmetric (mirror, no edge repeat) reflection of index i into [0, n) */
static int64_t reflect_idx(int64_t i, int64_t n) {
    if (n == 1) return 0;
    for (;;) {
        if (i < 0) i = -i;
        if (i >= n) i = 2 * n - 2 - i;
        else return i;
    }
}

/* Filter one axis of an (H, W, 3) image: axis 0 = rows (H), 1 = cols (W). */
static void filt_axis(const double *x, double *out, int64_t H, int64_t W, int axis, const double *w) {
    int64_t n = axis == 0 ? H : W;
#pragma omp parallel for schedule(static)
    for (int64_t y = 0; y < H; ++y)
        for (int64_t xx = 0; xx < W; ++xx)
            for (int c = 0; c < 3; ++c) {
                double s = 0.0;
                int64_t i = axis == 0 ? y : xx;
                for (int m = 0; m < SSIM_WIN; ++m) {
                    int64_t j = reflect_idx(i + m - SSIM_WIN / 2, n);
                    int64_t o = axis == 0 ? (j * W + xx) : (y * W + j);
                    s += w[m] * x[3 * o + c];
                }
                out[3 * (y * W + xx) + c] = s;
            }
}

/* Adjoint of filt_axis (losses.py:69-80): spread each g[j] by the window,
 * then fold the padded positions back through the reflection. */
static void filt_axis_adj(const double *g, double *out, int64_t H, int64_t W, int axis, const double *w) {
    int64_t n = axis == 0 ? H : W;
    memset(out, 0, sizeof(double) * H * W * 3);
    for (int64_t y = 0; y < H; ++y)
        for (int64_t xx = 0; xx < W; ++xx)
            for (int c = 0; c < 3; ++c) {
                int64_t i = axis == 0 ? y : xx;
                double gv = g[3 * (y * W + xx) + c];
                for (int m = 0; m < SSIM_WIN; ++m) {
                    int64_t j = reflect_idx(i + m - SSIM_WIN / 2, n);
                    int64_t o = axis == 0 ? (j * W + xx) : (y * W + j);
                    out[3 * o + c] += w[m] * gv;
                }
            }
}

static void filt2(const double *x, double *tmp, double *out, int64_t H, int64_t W, const double *w) {
    filt_axis(x, tmp, H, W, 0, w);
    filt_axis(tmp, out, H, W, 1, w);
}

static void filt2_adj(const double *g, double *tmp, double *out, int64_t H, int64_t W, const double *w) {
    filt_axis_adj(g, tmp, H, W, 1, w);
    filt_axis_adj(tmp, out, H, W, 0, w);
}

/* compute_losses' photometric part (losses.py:198-218 with _ssim_terms
 * :99-109 and _ssim_with_grad :119-134).  out[0] = l1, out[1] = mean SSIM.
 * grad (H,W,3) = d rendered_loss / d x. */
void orc_loss(int64_t H, int64_t W, const double *x, const double *y, double lambda_ssim,
              double *out, double *grad) {
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
    int64_t n = H * W * 3;
    double w[SSIM_WIN];
    ssim_window(w);
    double l1 = 0.0;
    for (int64_t i = 0; i < n; ++i) l1 += fabs(x[i] - y[i]);
    l1 /= (double)n;
    for (int64_t i = 0; i < n; ++i) {
        double d = x[i] - y[i];
        double sg = d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0);
        grad[i] = (1.0 - lambda_ssim) * sg / (double)n;
    }
    out[0] = l1;
    out[1] = 0.0;
    if (lambda_ssim == 0.0) return;
    double *buf = (double *)malloc(sizeof(double) * n * 12);
    double *tmp = buf, *mx = buf + n, *my = buf + 2 * n, *fxx = buf + 3 * n, *fyy = buf + 4 * n,
           *fxy = buf + 5 * n, *prod = buf + 6 * n, *gmx = buf + 7 * n, *gw2 = buf + 8 * n,
           *gwxy = buf + 9 * n, *adj = buf + 10 * n, *adj2 = buf + 11 * n;
    filt2(x, tmp, mx, H, W, w);
    filt2(y, tmp, my, H, W, w);
    for (int64_t i = 0; i < n; ++i) prod[i] = x[i] * x[i];
    filt2(prod, tmp, fxx, H, W, w);
    for (int64_t i = 0; i < n; ++i) prod[i] = y[i] * y[i];
    filt2(prod, tmp, fyy, H, W, w);
    for (int64_t i = 0; i < n; ++i) prod[i] = x[i] * y[i];
    filt2(prod, tmp, fxy, H, W, w);
    double ssum = 0.0;
    double gs = 1.0 / (double)n;
    for (int64_t i = 0; i < n; ++i) {
        double sxx = fxx[i] - mx[i] * mx[i];
        double syy = fyy[i] - my[i] * my[i];
        double sxy = fxy[i] - mx[i] * my[i];
        double a1 = 2 * mx[i] * my[i] + C1;
        double a2 = 2 * sxy + C2;
        double b1 = mx[i] * mx[i] + my[i] * my[i] + C1;
        double b2 = sxx + syy + C2;
        double s = a1 * a2 / (b1 * b2);
        ssum += s;
        double ga1 = gs * a2 / (b1 * b2);
        double ga2 = gs * a1 / (b1 * b2);
        double gb1 = -gs * s / b1;
        double gb2 = -gs * s / b2;
        gmx[i] = 2 * my[i] * ga1 + 2 * mx[i] * gb1 - 2 * mx[i] * gb2 - my[i] * 2 * ga2;
        gw2[i] = gb2;
        gwxy[i] = 2 * ga2;
    }
    out[1] = ssum / (double)n;
    /* gx = F*(g_mx) + F*(g_wx2) * 2x + F*(g_wxy) * y */
    filt2_adj(gmx, tmp, adj, H, W, w);
    for (int64_t i = 0; i < n; ++i) prod[i] = adj[i];
    filt2_adj(gw2, tmp, adj, H, W, w);
    filt2_adj(gwxy, tmp, adj2, H, W, w);
    for (int64_t i = 0; i < n; ++i) {
        double gx = prod[i] + adj[i] * 2 * x[i] + adj2[i] * y[i];
        grad[i] = grad[i] - lambda_ssim * gx;
    }
    free(buf);
}

/* ------------------------------------------------------------- chain */
/* _quat_grad (projection.py:302-325). */
static void quat_grad(double dR[3][3], const double q[4], double g[4]) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    g[0] = 2 * (-dR[0][1] * z + dR[0][2] * y + dR[1][0] * z - dR[1][2] * x - dR[2][0] * y + dR[2][1] * x);
    g[1] = 2 * (dR[0][1] * y + dR[0][2] * z + dR[1][0] * y - 2 * dR[1][1] * x - dR[1][2] * w +
                dR[2][0] * z + dR[2][1] * w - 2 * dR[2][2] * x);
    g[2] = 2 * (-2 * dR[0][0] * y + dR[0][1] * x + dR[0][2] * w + dR[1][0] * x + dR[1][2] * z -
                dR[2][0] * w + dR[2][1] * z - 2 * dR[2][2] * y);
    g[3] = 2 * (-2 * dR[0][0] * z - dR[0][1] * w + dR[0][2] * x + dR[1][0] * w - 2 * dR[1][1] * z +
                dR[1][2] * y + dR[2][0] * x + dR[2][1] * y);
}

/* chain_backward (projection.py:200-299): per visible row r with map index
 * mi[r], chain g2d[r] = [rgb(3), mean2d(2), conic(3), opacity] to the
 * primitive's parameters.  The projection context is recomputed from the
 * parameters with the same formulas project_map uses.  Outputs are dense
 * over the map (zeros for culled primitives): g_pos (n,3), g_rot (n,4),
 * g_ls (n,3), g_op (n), g_sh (n,48), pos2d_norm (n). */
void orc_chain(int64_t n, const double *pos, const double *rot, const double *ls,
               const double *opl, const double *sh, const double *cam, int sh_degree,
               double dilation, int64_t m, const int64_t *mi, const double *g2d,
               double *g_pos, double *g_rot, double *g_ls, double *g_op, double *g_sh,
               double *pos2d_norm) {
    memset(g_pos, 0, sizeof(double) * n * 3);
    memset(g_rot, 0, sizeof(double) * n * 4);
    memset(g_ls, 0, sizeof(double) * n * 3);
    memset(g_op, 0, sizeof(double) * n);
    memset(g_sh, 0, sizeof(double) * n * 48);
    memset(pos2d_norm, 0, sizeof(double) * n);
    const double *Rw = cam + CAM_R, *ctr = cam + CAM_C;
    double fx = cam[CAM_FX], fy = cam[CAM_FY];
    int nbc = (sh_degree + 1) * (sh_degree + 1);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < m; ++r) {
        int64_t i = mi[r];
        const double *g = g2d + 9 * r;
        proj_ctx P;
        project_ctx(pos + 3 * i, rot + 4 * i, ls + 3 * i, cam, dilation, &P);
        double det = P.a * P.c - P.b * P.b;
        double Q[2][2] = {{P.c / det, -P.b / det}, {-P.b / det, P.a / det}};
        double sg = sigmoid(opl[i]);
        /* rgb_active from the colour forward */
        double u[3];
        for (int k = 0; k < 3; ++k) u[k] = pos[3 * i + k] - ctr[k];
        double vl = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
        if (vl < 1e-12) vl = 1e-12;
        double d[3] = {u[0] / vl, u[1] / vl, u[2] / vl};
        double bs[16];
        sh_basis(d, sh_degree, bs);
        const double *s = sh + 48 * i;
        double grgb[3];
        for (int ch = 0; ch < 3; ++ch) {
            double raw = 0.0;
            for (int k = 0; k < 16; ++k) raw += bs[k] * s[3 * k + ch];
            raw += 0.5;
            grgb[ch] = raw > 0 ? g[ch] : 0.0;
        }
        double gm0 = g[3], gm1 = g[4];
        g_op[i] = g[8] * sg * (1.0 - sg);
        /* conic -> cov2d: GC = -Q GQ Q */
        double GQ[2][2] = {{g[5], g[6] / 2}, {g[6] / 2, g[7]}};
        double QG[2][2], GC[2][2];
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) QG[a][b] = Q[a][0] * GQ[0][b] + Q[a][1] * GQ[1][b];
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) GC[a][b] = -(QG[a][0] * Q[0][b] + QG[a][1] * Q[1][b]);
        double tz = P.t[2], iz = 1.0 / tz, iz2 = iz * iz;
        double J[2][3] = {{fx * iz, 0.0, -fx * P.t[0] * iz2}, {0.0, fy * iz, -fy * P.t[1] * iz2}};
        /* dSc = J^T GC J ; dJ = 2 GC J covc */
        double GJ[2][3], dSc[3][3], dJ[2][3];
        for (int a = 0; a < 2; ++a)
            for (int k = 0; k < 3; ++k) GJ[a][k] = GC[a][0] * J[0][k] + GC[a][1] * J[1][k];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) dSc[a][b] = J[0][a] * GJ[0][b] + J[1][a] * GJ[1][b];
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 3; ++b) {
                double acc = 0.0;
                for (int k = 0; k < 3; ++k) acc += GJ[a][k] * P.covc[k][b];
                dJ[a][b] = 2.0 * acc;
            }
        /* dS3 = Rcw^T dSc Rcw */
        double t1[3][3], dS3[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                double acc = 0.0;
                for (int k = 0; k < 3; ++k) acc += Rw[3 * k + a] * dSc[k][b];
                t1[a][b] = acc;
            }
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                double acc = 0.0;
                for (int k = 0; k < 3; ++k) acc += t1[a][k] * Rw[3 * k + b];
                dS3[a][b] = acc;
            }
        /* log_scale: 2 s2 diag(R^T dS3 R) */
        for (int a = 0; a < 3; ++a) {
            double acc = 0.0;
            for (int j = 0; j < 3; ++j)
                for (int k = 0; k < 3; ++k) acc += P.rot[j][a] * dS3[j][k] * P.rot[k][a];
            g_ls[3 * i + a] = 2.0 * P.s2[a] * acc;
        }
        /* dR = 2 dS3 (R diag(s2)) */
        double dR[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                double acc = 0.0;
                for (int k = 0; k < 3; ++k) acc += dS3[a][k] * (P.rot[k][b] * P.s2[b]);
                dR[a][b] = 2.0 * acc;
            }
        double gq[4];
        quat_grad(dR, P.qh, gq);
        double dot = P.qh[0] * gq[0] + P.qh[1] * gq[1] + P.qh[2] * gq[2] + P.qh[3] * gq[3];
        for (int k = 0; k < 4; ++k) g_rot[4 * i + k] = (gq[k] - P.qh[k] * dot) / P.qn;
        /* position through the mean projection and through J */
        double gt[3];
        gt[0] = (fx * iz) * gm0 - dJ[0][2] * fx * iz2;
        gt[1] = (fy * iz) * gm1 - dJ[1][2] * fy * iz2;
        gt[2] = -fx * P.t[0] * iz2 * gm0 - fy * P.t[1] * iz2 * gm1 - dJ[0][0] * fx * iz2 -
                dJ[1][1] * fy * iz2 + dJ[0][2] * 2 * fx * P.t[0] * iz2 * iz +
                dJ[1][2] * 2 * fy * P.t[1] * iz2 * iz;
        double gp[3];
        for (int b = 0; b < 3; ++b) gp[b] = gt[0] * Rw[b] + gt[1] * Rw[3 + b] + gt[2] * Rw[6 + b];
        /* colour: SH coefficients and the view direction */
        double coef[16] = {0};
        for (int k = 0; k < nbc; ++k) {
            for (int ch = 0; ch < 3; ++ch) g_sh[48 * i + 3 * k + ch] = bs[k] * grgb[ch];
            coef[k] = s[3 * k] * grgb[0] + s[3 * k + 1] * grgb[1] + s[3 * k + 2] * grgb[2];
        }
        double db[16][3];
        sh_basis_grad(d, sh_degree, db);
        double gdir[3] = {0, 0, 0};
        for (int dd = 0; dd < 3; ++dd)
            for (int k = 0; k < nbc; ++k) gdir[dd] += coef[k] * db[k][dd];
        double vd = d[0] * gdir[0] + d[1] * gdir[1] + d[2] * gdir[2];
        for (int b = 0; b < 3; ++b) g_pos[3 * i + b] = gp[b] + (gdir[b] - d[b] * vd) / vl;
        double a0 = gm0 * (cam[CAM_W] / 2), a1 = gm1 * (cam[CAM_H] / 2);
        pos2d_norm[i] = sqrt(a0 * a0 + a1 * a1);
    }
}

/* ------------------------------------------------------------- adam */
/* adam_step (optimizer.py:101-133) for one parameter group of `count`
 * values: moments, bias correction, per-element clip to +-lr, p -= step.
 * The caller passes the learning rate it resolved via AdamState.rate_for
 * (optimizer.py:63-76) and the post-increment step count t. */
void orc_adam_group(int64_t count, double *p, const double *g, double *m, double *v, double lr,
                    int64_t t, double b1, double b2, double eps) {
    double bc1 = 1.0 - pow(b1, (double)t);
    double bc2 = 1.0 - pow(b2, (double)t);
    for (int64_t i = 0; i < count; ++i) {
        m[i] = m[i] * b1;
        m[i] = m[i] + (1 - b1) * g[i];
        v[i] = v[i] * b2;
        v[i] = v[i] + (1 - b2) * g[i] * g[i];
        double step = lr * (m[i] / bc1) / (sqrt(v[i] / bc2) + eps);
        if (step < -lr) step = -lr;
        if (step > lr) step = lr;
        p[i] -= step;
    }
}

/* GaussianMap.normalize_rotations (core.py:225-229). Returns -1 on a zero norm. */
int orc_normalize_rotations(int64_t n, double *rot) {
    for (int64_t i = 0; i < n; ++i) {
        double *q = rot + 4 * i;
        double nn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        if (nn == 0.0) return -1;
        for (int k = 0; k < 4; ++k) q[k] /= nn;
    }
    return 0;
}

/* ------------------------------------------------------------ threads */
void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_get_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
