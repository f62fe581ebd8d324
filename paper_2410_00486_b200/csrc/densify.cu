// densify.cu -- K10: clone / split / prune and opacity reset as stream
// compaction.
//
// Restates densify_and_prune (densify.py:103-173) + resize_for_densify
// (optimizer.py:136-146):
//   candidates = grad2d_accum / max(obs,1) > grad_threshold  &  obs > 0
//   small      = candidates & max(exp(log_scale)) <= pct * extent   -> clone
//   large      = candidates & ~small                                -> split x2
//   keep_old   = ~large & logistic(logit) >= prune_opacity
// New entries (clones in index order, then split children in
// repeat(split_idx, 2) order) are filtered by 1/(1+exp(-logit)) >= prune
// (densify.py:158).  The masks are evaluated in FLOAT64 from the stored
// float32 values, so they are the same IEEE double operations the oracle
// performs on those values: bit-exact masks and
// indices.  Output order = survivors (original order), clones, children,
// obtained with order-preserving exclusive scans.
#include "common.cuh"

namespace ss {

cudaError_t launch_scan_u32(const uint32_t* in, int64_t n, uint32_t* out, int64_t* total,
                            void* ws, cudaStream_t s);
size_t scan_ws_bytes(int64_t n);

__device__ __forceinline__ double logistic_stable(double x) {
    // core.py:16-24
    if (x >= 0) return 1.0 / (1.0 + exp(-x));
    double e = exp(x);
    return e / (1.0 + e);
}

__global__ void densify_masks_kernel(int64_t n, const float* __restrict__ opl,
                                     const float* __restrict__ ls,
                                     const float* __restrict__ grad2d,
                                     const int32_t* __restrict__ obs, double thr, double prune,
                                     double limit, uint32_t* cK, uint32_t* cC, uint32_t* cL,
                                     uint32_t* cS, uint8_t* mask) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t ob = obs[i];
    double cnt = (double)(ob > 1 ? ob : 1);
    double mean_norm = (double)grad2d[i] / cnt;
    bool cand = (mean_norm > thr) && (ob > 0);
    double ms = fmax(fmax(exp((double)ls[3 * i]), exp((double)ls[3 * i + 1])),
                     exp((double)ls[3 * i + 2]));
    bool small = cand && (ms <= limit);
    bool large = cand && !small;
    double l = (double)opl[i];
    bool keep = !large && (logistic_stable(l) >= prune);
    bool fresh = (1.0 / (1.0 + exp(-l))) >= prune;
    cK[i] = keep;
    cC[i] = small && fresh;
    cL[i] = large;
    cS[i] = (large && fresh) ? 2u : 0u;
    mask[i] = (small ? 1 : 0) | (large ? 2 : 0) | (keep ? 4 : 0) | (fresh ? 8 : 0);
}

// counts: [kept, cloned(unfiltered), split(unfiltered), pruned, n_new]
__global__ void densify_counts_kernel(int64_t n, const int64_t* tot, const uint8_t* mask,
                                      int64_t* counts) {
    // tot: [nK, nC, nL, nS]
    __shared__ unsigned long long small_cnt, pruned_cnt;
    if (threadIdx.x == 0) small_cnt = pruned_cnt = 0;
    __syncthreads();
    unsigned long long a = 0, b = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        uint8_t m = mask[i];
        a += (m & 1) ? 1 : 0;
        b += (!(m & 4) && !(m & 2)) ? 1 : 0;
    }
    atomicAdd(&small_cnt, a);
    atomicAdd(&pruned_cnt, b);
    __syncthreads();
    if (threadIdx.x == 0) {
        counts[0] = tot[0];
        counts[1] = (int64_t)small_cnt;
        counts[2] = tot[2];
        counts[3] = (int64_t)pruned_cnt;
        counts[4] = tot[1] + tot[3];
    }
}

// Survivors: gather every plane (params, stats are reset, moments).
struct Planes {
    const float* in[24];
    float* out[24];
    int k[24];
    int count;
};

__global__ void densify_gather_kernel(int64_t n, const uint32_t* __restrict__ cK,
                                      const uint32_t* __restrict__ oK, Planes P,
                                      int64_t* survivors) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n || !cK[i]) return;
    int64_t d = oK[i];
    if (survivors) survivors[d] = i;
    for (int p = 0; p < P.count; ++p) {
        int k = P.k[p];
        for (int j = 0; j < k; ++j) P.out[p][d * k + j] = P.in[p][i * k + j];
    }
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

__device__ __forceinline__ float normal_from(uint64_t seed, uint32_t idx) {
    uint32_t a = hash32((uint32_t)seed ^ hash32(idx * 2u + 1u));
    uint32_t b = hash32((uint32_t)(seed >> 32) ^ hash32(idx * 2u + 2u) ^ 0x9e3779b9u);
    float u1 = ((a >> 8) + 1u) * (1.0f / 16777217.0f);
    float u2 = (b >> 8) * (1.0f / 16777216.0f);
    return sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
}

// New entries: clones at pos - clone_step * mean_g3d, split children at
// pos + R(q) (normal * exp(log_scale)) with log_scale - ln(shrink).
__global__ void densify_new_kernel(int64_t n, const uint8_t* __restrict__ mask,
                                   const uint32_t* __restrict__ oC,
                                   const uint32_t* __restrict__ oL,
                                   const uint32_t* __restrict__ oS, const int64_t* tot,
                                   const float* __restrict__ pos, const float* __restrict__ rot,
                                   const float* __restrict__ ls, const float* __restrict__ opl,
                                   const float* __restrict__ dc, const float* __restrict__ rest,
                                   const float* __restrict__ g3d, const int32_t* __restrict__ obs,
                                   const float* __restrict__ normals, uint64_t seed,
                                   double clone_step, double shrink_log, ss_map out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t m = mask[i];
    if (!(m & 8) || !(m & 3)) return;  // not fresh or not a candidate
    const int64_t nK = tot[0], nC = tot[1];
    auto copy_rest = [&](int64_t d) {
        for (int k = 0; k < 3; ++k) out.d_sh_dc[3 * d + k] = dc[3 * i + k];
        for (int k = 0; k < 45; ++k) out.d_sh_rest[45 * d + k] = rest[45 * i + k];
        out.d_opacity_logits[d] = opl[i];
        for (int k = 0; k < 4; ++k) out.d_rotations[4 * d + k] = rot[4 * i + k];
    };
    if (m & 1) {  // clone
        int64_t d = nK + oC[i];
        double cnt = (double)(obs[i] > 1 ? obs[i] : 1);
        for (int k = 0; k < 3; ++k) {
            out.d_positions[3 * d + k] =
                (float)((double)pos[3 * i + k] - clone_step * ((double)g3d[3 * i + k] / cnt));
            out.d_log_scales[3 * d + k] = ls[3 * i + k];
        }
        copy_rest(d);
    } else {  // split into two children
        double q[4] = {rot[4 * i], rot[4 * i + 1], rot[4 * i + 2], rot[4 * i + 3]};
        double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        for (int k = 0; k < 4; ++k) q[k] /= qn;
        double w = q[0], x = q[1], y = q[2], z = q[3];
        double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                       2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                       2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
        for (int c = 0; c < 2; ++c) {
            int64_t d = nK + nC + oS[i] + c;
            int64_t r = 2 * (int64_t)oL[i] + c;  // row in repeat(split_idx, 2) order
            double loc[3];
            for (int k = 0; k < 3; ++k) {
                double nv = normals ? (double)normals[3 * r + k]
                                    : (double)normal_from(seed, (uint32_t)(3 * r + k));
                loc[k] = nv * exp((double)ls[3 * i + k]);
            }
            for (int k = 0; k < 3; ++k) {
                out.d_positions[3 * d + k] = (float)((double)pos[3 * i + k] + R[3 * k] * loc[0] +
                                                     R[3 * k + 1] * loc[1] + R[3 * k + 2] * loc[2]);
                out.d_log_scales[3 * d + k] = (float)((double)ls[3 * i + k] - shrink_log);
            }
            copy_rest(d);
        }
    }
}

struct DensifyWs {
    uint32_t *cK, *cC, *cL, *cS, *oK, *oC, *oL, *oS;
    uint8_t* mask;
    int64_t* tot;  // 4
    void* scan_ws;
};

static DensifyWs densify_layout(int64_t n, void* base, size_t* bytes) {
    size_t off = 0;
    char* b = reinterpret_cast<char*>(base);
    auto take = [&](size_t sz) {
        off = (off + 255) & ~size_t(255);
        void* p = b ? b + off : nullptr;
        off += sz;
        return p;
    };
    DensifyWs w;
    size_t u = sizeof(uint32_t) * (size_t)(n > 0 ? n : 1);
    w.cK = (uint32_t*)take(u);
    w.cC = (uint32_t*)take(u);
    w.cL = (uint32_t*)take(u);
    w.cS = (uint32_t*)take(u);
    w.oK = (uint32_t*)take(u);
    w.oC = (uint32_t*)take(u);
    w.oL = (uint32_t*)take(u);
    w.oS = (uint32_t*)take(u);
    w.mask = (uint8_t*)take((size_t)(n > 0 ? n : 1));
    w.tot = (int64_t*)take(sizeof(int64_t) * 4);
    w.scan_ws = take(scan_ws_bytes(n));
    if (bytes) *bytes = off + 256;
    return w;
}

size_t densify_workspace_bytes(int64_t n) {
    size_t b;
    densify_layout(n, nullptr, &b);
    return b;
}

cudaError_t launch_densify_count(const ss_map* mp, float thr, float prune, double limit,
                                 void* ws, int64_t* d_counts, uint8_t* d_mask_out,
                                 cudaStream_t s) {
    DensifyWs w = densify_layout(mp->n, ws, nullptr);
    int64_t n = mp->n;
    cudaError_t e = cudaMemsetAsync(w.tot, 0, sizeof(int64_t) * 4, s);
    if (e != cudaSuccess) return e;
    if (n > 0) {
        densify_masks_kernel<<<div_up(n, 256), 256, 0, s>>>(
            n, mp->d_opacity_logits, mp->d_log_scales, mp->d_grad2d_accum, mp->d_obs_count,
            (double)thr, (double)prune, limit, w.cK, w.cC, w.cL, w.cS, w.mask);
        uint32_t* cs[4] = {w.cK, w.cC, w.cL, w.cS};
        uint32_t* os[4] = {w.oK, w.oC, w.oL, w.oS};
        for (int k = 0; k < 4; ++k) {
            e = launch_scan_u32(cs[k], n, os[k], w.tot + k, w.scan_ws, s);
            if (e != cudaSuccess) return e;
        }
    }
    densify_counts_kernel<<<1, 256, 0, s>>>(n, w.tot, w.mask, d_counts);
    if (d_mask_out && n > 0)
        cudaMemcpyAsync(d_mask_out, w.mask, (size_t)n, cudaMemcpyDeviceToDevice, s);
    return cudaGetLastError();
}

// planes: caller-provided list of extra per-Gaussian float planes (Adam
// moments) to gather for survivors; their new-entry tail is zeroed.
cudaError_t launch_densify_apply(const ss_map* mp, void* ws, const float* normals, uint64_t seed,
                                 float clone_step, float shrink_log, const ss_map* out,
                                 int n_planes, const float* const* pin, float* const* pout,
                                 const int* pk, int64_t n_new_host, int64_t* survivors,
                                 cudaStream_t s) {
    DensifyWs w = densify_layout(mp->n, ws, nullptr);
    int64_t n = mp->n;
    if (n == 0) return cudaSuccess;
    Planes P;
    int c = 0;
    auto add = [&](const float* a, float* b, int k) {
        P.in[c] = a;
        P.out[c] = b;
        P.k[c] = k;
        ++c;
    };
    add(mp->d_positions, out->d_positions, 3);
    add(mp->d_rotations, out->d_rotations, 4);
    add(mp->d_log_scales, out->d_log_scales, 3);
    add(mp->d_opacity_logits, out->d_opacity_logits, 1);
    add(mp->d_sh_dc, out->d_sh_dc, 3);
    add(mp->d_sh_rest, out->d_sh_rest, 45);
    for (int p = 0; p < n_planes && c < 24; ++p) add(pin[p], pout[p], pk[p]);
    P.count = c;
    densify_gather_kernel<<<div_up(n, 256), 256, 0, s>>>(n, w.cK, w.oK, P, survivors);
    densify_new_kernel<<<div_up(n, 256), 256, 0, s>>>(
        n, w.mask, w.oC, w.oL, w.oS, w.tot, mp->d_positions, mp->d_rotations, mp->d_log_scales,
        mp->d_opacity_logits, mp->d_sh_dc, mp->d_sh_rest, mp->d_grad3d_accum, mp->d_obs_count,
        normals, seed, (double)clone_step, (double)shrink_log, *out);
    (void)n_new_host;
    return cudaGetLastError();
}

// resize_for_densify (optimizer.py:136-146) for a moment set: per plane,
// out[i] = in[survivors[i]] for i < n_surv, zero rows after (n_new fresh
// primitives).  One launch for every plane (grid.y = plane).
struct ResizePlanes {
    const float* in[16];
    float* out[16];
    int32_t k[16];
};

__global__ void resize_moments_kernel(int64_t n_out, const int64_t* __restrict__ surv,
                                      int64_t n_surv, ResizePlanes P) {
    const int pl = blockIdx.y;
    const int k = P.k[pl];
    const int64_t nf = n_out * k;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nf;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e / k, c = e - row * k;
        P.out[pl][e] = row < n_surv ? P.in[pl][surv[row] * k + c] : 0.f;
    }
}

cudaError_t launch_resize_moments(int64_t n_out, const int64_t* surv, int64_t n_surv,
                                  int n_planes, const float* const* pin, float* const* pout,
                                  const int32_t* pk, cudaStream_t s) {
    if (n_planes == 0 || n_out == 0) return cudaSuccess;
    ResizePlanes P = {};
    int kmax = 1;
    for (int p = 0; p < n_planes; ++p) {
        P.in[p] = pin[p];
        P.out[p] = pout[p];
        P.k[p] = pk[p];
        kmax = pk[p] > kmax ? pk[p] : kmax;
    }
    const int64_t nf = n_out * kmax;
    const int blocks = (int)((nf + 255) / 256 < 4096 ? (nf + 255) / 256 : 4096);
    resize_moments_kernel<<<dim3(blocks, n_planes), 256, 0, s>>>(n_out, surv, n_surv, P);
    return cudaGetLastError();
}

}  // namespace ss
