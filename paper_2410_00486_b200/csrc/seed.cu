// seed.cu -- F3: geometry seeding, seed_from_points (densify.py:53-83).
//
// One isotropic primitive per point of an incoming keyframe cloud: scale =
// mean distance to the 3 nearest neighbours within the cloud (the k + 1 = 4
// nearest including the point itself, self dropped, as cKDTree.query(k=4)
// with dist[:, 1:]), floored at 1e-4; a lone point gets 1% of the scene
// extent; identity rotation, opacity 0.1, DC colour (c - 0.5) / SH_C0.
//
// The reference builds a k-d tree on the host.  Here: a uniform grid over
// the cloud's bounding box (~2 points per cell), a counting sort of the
// points by cell (histogram, scan, scatter), then one thread per point
// searching Chebyshev shells of cells r = 0, 1, 2, ... and keeping the 4
// smallest squared distances (float64, like cKDTree).  After shell r every
// point closer than r * h has been visited (cell(p + d) - cell(p) <= r per
// axis for |d| <= r h); the search stops once the 4th distance is <= (r-1) h
// (one cell of slack for the float cell index), so the result is the exact
// kNN.
#include "common.cuh"

namespace ss {

cudaError_t launch_scan_u32(const uint32_t* in, int64_t n, uint32_t* out, int64_t* total,
                            void* ws, cudaStream_t s);
size_t scan_ws_bytes(int64_t n);

constexpr float kSeedMinScale = 1e-4f;  // densify.py MIN_SEED_SCALE
constexpr float kSeedOpacity = 0.1f;    // densify.py INIT_OPACITY
constexpr double kSH_C0d = 0.28209479177387814;
constexpr int kSeedMaxGrid = 160;       // cells per axis

struct SeedGrid {
    float lo[3];
    float h;
    int g[3];
    int ncell;
};

__device__ __forceinline__ unsigned f2ord(float f) {  // order-preserving float -> uint
    const unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// bounding box (ordered-uint min / max) and the non-finite check
__global__ void seed_bbox_kernel(int64_t n, const float* __restrict__ p, unsigned* bb,
                                 int32_t* nonfinite) {
    unsigned mn[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, mx[3] = {0u, 0u, 0u};
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float v = p[3 * i + k];
            if (!isfinite(v)) {
                bad = true;
                continue;
            }
            const unsigned o = f2ord(v);
            mn[k] = min(mn[k], o);
            mx[k] = max(mx[k], o);
        }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            mn[k] = min(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], d));
            mx[k] = max(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], d));
        }
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            atomicMin(bb + k, mn[k]);
            atomicMax(bb + 3 + k, mx[k]);
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(nonfinite, 1);
}

// g cells along the longest axis (host-chosen: ~2 points per cell for a
// volume-filling cloud); the other axes get as many cells of the same size
__global__ void seed_grid_kernel(int g, const unsigned* bb, SeedGrid* gd) {
    float lo[3], ext = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = ord2f(bb[k]);
        ext = fmaxf(ext, ord2f(bb[3 + k]) - lo[k]);
    }
    const float h = ext > 0.f ? ext / (float)g * 1.0001f + 1e-30f : 1.f;
    SeedGrid s;
    int nc = 1;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        s.lo[k] = lo[k];
        s.g[k] = min(g, (int)((ord2f(bb[3 + k]) - lo[k]) / h) + 1);
        nc *= s.g[k];
    }
    s.h = h;
    s.ncell = nc;
    *gd = s;
}

__device__ __forceinline__ void seed_cell(const SeedGrid& g, float x, float y, float z, int c[3]) {
    const float v[3] = {x, y, z};
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = min(g.g[k] - 1, max(0, (int)((v[k] - g.lo[k]) / g.h)));
}

__global__ void seed_count_kernel(int64_t n, const float* __restrict__ p, const SeedGrid* gd,
                                  uint32_t* __restrict__ cell_of, uint32_t* __restrict__ count) {
    const SeedGrid g = *gd;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int c[3];
        seed_cell(g, p[3 * i], p[3 * i + 1], p[3 * i + 2], c);
        const uint32_t id = (uint32_t)((c[2] * g.g[1] + c[1]) * g.g[0] + c[0]);
        cell_of[i] = id;
        atomicAdd(count + id, 1u);
    }
}

__global__ void seed_scatter_kernel(int64_t n, const uint32_t* __restrict__ cell_of,
                                    const uint32_t* __restrict__ start, uint32_t* fill,
                                    uint32_t* __restrict__ sorted) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t c = cell_of[i];
        sorted[start[c] + atomicAdd(fill + c, 1u)] = (uint32_t)i;
    }
}

// 4 smallest squared distances (ascending) by insertion
__device__ __forceinline__ void keep4(double d, double b[4]) {
    if (d >= b[3]) return;
    b[3] = d;
#pragma unroll
    for (int k = 3; k > 0; --k)
        if (b[k] < b[k - 1]) {
            const double t = b[k];
            b[k] = b[k - 1];
            b[k - 1] = t;
        }
}

__global__ void seed_knn_kernel(int64_t n, const float* __restrict__ p,
                                const float* __restrict__ colors, const SeedGrid* gd,
                                const uint32_t* __restrict__ start,
                                const uint32_t* __restrict__ count,
                                const uint32_t* __restrict__ sorted, float scene_extent,
                                float* __restrict__ pos, float4* __restrict__ rot,
                                float* __restrict__ log_scale, float* __restrict__ opl,
                                float* __restrict__ sh_dc) {
    const SeedGrid g = *gd;
    const int kq = n - 1 < 3 ? (int)(n - 1) : 3;  // neighbours averaged
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x = p[3 * i], y = p[3 * i + 1], z = p[3 * i + 2];
        double mean_dist;
        if (n == 1) {
            mean_dist = 0.01 * (double)scene_extent;
        } else {
            int c[3];
            seed_cell(g, (float)x, (float)y, (float)z, c);
            double best[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
            const int rmax = max(g.g[0], max(g.g[1], g.g[2]));
            for (int r = 0; r <= rmax; ++r) {
                for (int dz = -r; dz <= r; ++dz) {
                    const int cz = c[2] + dz;
                    if (cz < 0 || cz >= g.g[2]) continue;
                    for (int dy = -r; dy <= r; ++dy) {
                        const int cy = c[1] + dy;
                        if (cy < 0 || cy >= g.g[1]) continue;
                        const bool face = abs(dz) == r || abs(dy) == r;
                        for (int dx = -r; dx <= r; dx += (face ? 1 : max(1, 2 * r))) {
                            const int cx = c[0] + dx;
                            if (cx < 0 || cx >= g.g[0]) continue;
                            const uint32_t cid = (uint32_t)((cz * g.g[1] + cy) * g.g[0] + cx);
                            const uint32_t s0 = start[cid], s1 = s0 + count[cid];
                            for (uint32_t q = s0; q < s1; ++q) {
                                const uint32_t j = sorted[q];
                                const double ex = (double)p[3 * j] - x;
                                const double ey = (double)p[3 * j + 1] - y;
                                const double ez = (double)p[3 * j + 2] - z;
                                keep4(ex * ex + ey * ey + ez * ez, best);
                            }
                        }
                    }
                }
                // exact once the (kq+1)-th distance is within the searched
                // radius; (r - 1) h leaves one cell of slack for the float
                // rounding of the cell index
                const double rad = (double)(r - 1) * (double)g.h;
                if (r >= 1 && best[kq] <= rad * rad) break;
            }
            double s = 0.0;
            for (int k = 1; k <= kq; ++k) s += sqrt(best[k]);
            mean_dist = s / (double)kq;
        }
        const float ls = (float)log(fmax(mean_dist, (double)kSeedMinScale));
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            pos[3 * i + k] = p[3 * i + k];
            log_scale[3 * i + k] = ls;
            sh_dc[3 * i + k] = (float)(((double)colors[3 * i + k] - 0.5) / kSH_C0d);
        }
        rot[i] = make_float4(1.f, 0.f, 0.f, 0.f);
        opl[i] = (float)log((double)kSeedOpacity / (1.0 - (double)kSeedOpacity));
    }
}

// ------------------------------------------------------------ workspace
struct SeedWs {
    unsigned* bb;      // 6
    SeedGrid* grid;    // 1
    uint32_t* count;   // max cells
    uint32_t* fill;    // max cells
    uint32_t* start;   // max cells
    uint32_t* cell_of; // n
    uint32_t* sorted;  // n
    int64_t* total;
    void* scan_ws;
    size_t bytes;
};

static int seed_grid_cells(int64_t n) {  // cells along the longest axis
    int g = (int)ceil(cbrt((double)n * 0.5));
    return g < 1 ? 1 : (g > kSeedMaxGrid ? kSeedMaxGrid : g);
}

static SeedWs seed_layout(int64_t n, void* base) {
    SeedWs w;
    size_t off = 0;
    auto take = [&](size_t b) {
        off = (off + 255) & ~size_t(255);
        void* p = base ? static_cast<char*>(base) + off : nullptr;
        off += b;
        return p;
    };
    const size_t g = (size_t)seed_grid_cells(n);
    const size_t maxc = g * g * g;
    w.bb = static_cast<unsigned*>(take(6 * sizeof(unsigned)));
    w.grid = static_cast<SeedGrid*>(take(sizeof(SeedGrid)));
    w.count = static_cast<uint32_t*>(take(maxc * 4));
    w.fill = static_cast<uint32_t*>(take(maxc * 4));
    w.start = static_cast<uint32_t*>(take(maxc * 4));
    w.cell_of = static_cast<uint32_t*>(take((size_t)(n > 0 ? n : 1) * 4));
    w.sorted = static_cast<uint32_t*>(take((size_t)(n > 0 ? n : 1) * 4));
    w.total = static_cast<int64_t*>(take(sizeof(int64_t)));
    w.scan_ws = take(scan_ws_bytes((int64_t)maxc));
    w.bytes = off + 256;
    return w;
}

size_t seed_workspace_bytes(int64_t n) { return seed_layout(n, nullptr).bytes; }

__global__ void seed_init_kernel(unsigned* bb, int32_t* nonfinite) {
    const int t = threadIdx.x;
    if (t < 3) bb[t] = 0xffffffffu;
    else if (t < 6) bb[t] = 0u;
    if (t == 0) *nonfinite = 0;
}

cudaError_t launch_seed(int64_t n, const float* pts, const float* colors, float scene_extent,
                        float* pos, float* rot, float* ls, float* opl, float* sh_dc,
                        int32_t* nonfinite, void* ws, size_t ws_bytes, cudaStream_t s) {
    SeedWs w = seed_layout(n, ws);
    if (w.bytes > ws_bytes) return cudaErrorInvalidValue;
    seed_init_kernel<<<1, 32, 0, s>>>(w.bb, nonfinite);
    if (n == 0) return cudaGetLastError();
    const int blocks = div_up(n, 256) < 1184 ? div_up(n, 256) : 1184;
    seed_bbox_kernel<<<blocks, 256, 0, s>>>(n, pts, w.bb, nonfinite);
    const int g = seed_grid_cells(n);
    seed_grid_kernel<<<1, 1, 0, s>>>(g, w.bb, w.grid);
    const size_t maxc = (size_t)g * g * g;
    cudaError_t e = cudaMemsetAsync(w.count, 0, maxc * 4, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(w.fill, 0, maxc * 4, s);
    if (e != cudaSuccess) return e;
    seed_count_kernel<<<blocks, 256, 0, s>>>(n, pts, w.grid, w.cell_of, w.count);
    e = launch_scan_u32(w.count, (int64_t)maxc, w.start, w.total, w.scan_ws, s);
    if (e != cudaSuccess) return e;
    seed_scatter_kernel<<<blocks, 256, 0, s>>>(n, w.cell_of, w.start, w.fill, w.sorted);
    seed_knn_kernel<<<div_up(n, 128), 128, 0, s>>>(
        n, pts, colors, w.grid, w.start, w.count, w.sorted, scene_extent, pos,
        reinterpret_cast<float4*>(rot), ls, opl, sh_dc);
    return cudaGetLastError();
}

}  // namespace ss
