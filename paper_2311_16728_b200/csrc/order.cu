// order.cu -- map layout: spatial (Morton) order of the Gaussians in HBM.
//
// Not a step of the method: Eq. 3 does not depend on where a Gaussian sits in memory (its index
// only breaks ties between equal depths, SPEC.md:348 (3)).  It is the map's layout: kernels that
// run one thread per Gaussian (A1, A9, A11, the bin scatter) and the raster backward's atomics
// into the per-(view, Gaussian) records all do better when Gaussians that land on the same
// tiles are neighbours in memory (culled warps are uniform, CTA-level tile aggregation sees few
// tiles, atomics and gathers hit the same L2 lines).  A map built by keyframe insertion
// is already roughly spatially grouped; the synthetic inputs are shuffled on
// purpose, so the mapping engine re-orders once at construction and after every densify.
//
// gs_spatial_order: perm[k] = index of the Gaussian placed at position k, by ascending 30-bit
// Morton code of its mean on a 1024^3 grid over the means' bounding box, ties by index (stable
// LSD radix sort, sort.cu).  gs_permute_columns: dst[r][k] = src[r][perm[k]].
#include <algorithm>

#include "gs_internal.cuh"

namespace gsk {

// order-preserving map of a float onto uint32 (for atomicMin / atomicMax on floats)
__device__ __forceinline__ uint32_t f2ord(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

// bbox[0..2] = min, bbox[3..5] = max of the means (ordered uint32), pre-set to (~0, 0)
__global__ void __launch_bounds__(256) k_bbox(const float *__restrict__ P, int64_t ld, int64_t n,
                                              uint32_t *__restrict__ bbox) {
    uint32_t lo[3] = {~0u, ~0u, ~0u}, hi[3] = {0u, 0u, 0u};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int a = 0; a < 3; a++) {
            const uint32_t o = f2ord(P[a * ld + i]);
            lo[a] = min(lo[a], o);
            hi[a] = max(hi[a], o);
        }
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
            lo[a] = min(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], s));
            hi[a] = max(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], s));
        }
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int a = 0; a < 3; a++) {
            atomicMin(&bbox[a], lo[a]);
            atomicMax(&bbox[3 + a], hi[a]);
        }
}

// spread the low 10 bits of x to bits 0, 3, 6, ...
__device__ __forceinline__ uint32_t spread3(uint32_t x) {
    x &= 0x3ffu;
    x = (x | (x << 16)) & 0x030000ffu;
    x = (x | (x << 8)) & 0x0300f00fu;
    x = (x | (x << 4)) & 0x030c30c3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}

// cell of coordinate x in [lo, hi]: min(1023, (int)((x - lo) * (1024 / (hi - lo)))), fp32 IEEE
// operations in this order (the GPU test recomputes it in numpy float32)
__device__ __forceinline__ uint32_t cell(float x, float lo, float scale) {
    const float t = __fmul_rn(__fsub_rn(x, lo), scale);
    return (uint32_t)min(1023, max(0, (int)t));
}

__global__ void __launch_bounds__(256) k_morton(const float *__restrict__ P, int64_t ld, int64_t n,
                                                const uint32_t *__restrict__ bbox, uint64_t *__restrict__ keys,
                                                uint32_t *__restrict__ vals, uint32_t *__restrict__ count) {
    float lo[3], sc[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        lo[a] = ord2f(bbox[a]);
        const float ext = __fsub_rn(ord2f(bbox[3 + a]), lo[a]);
        sc[a] = ext > 0.f ? __fdiv_rn(1024.0f, ext) : 0.f;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *count = (uint32_t)n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t code = spread3(cell(P[i], lo[0], sc[0])) | spread3(cell(P[ld + i], lo[1], sc[1])) << 1 |
                              spread3(cell(P[2 * ld + i], lo[2], sc[2])) << 2;
        keys[i] = code;
        vals[i] = (uint32_t)i;
    }
}

__global__ void __launch_bounds__(256) k_permute_columns(const float *__restrict__ src, float *__restrict__ dst,
                                                         int64_t ld, int64_t n, const uint32_t *__restrict__ perm) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int64_t r = blockIdx.y;
    dst[r * ld + k] = src[r * ld + perm[k]];
}

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct OrderTemp {
    size_t bbox, keys0, vals0, keys1, vals1, count, hdr, look, total;
    int64_t blocks;
};

static OrderTemp order_temp(int64_t n) {
    OrderTemp t;
    t.blocks = std::max<int64_t>((n + SORT_TILE - 1) / SORT_TILE, 1);
    const int64_t cap = t.blocks * SORT_TILE;
    size_t o = 0;
    auto take = [&](size_t b) {
        size_t r = o;
        o += al(b);
        return r;
    };
    t.bbox = take(6 * sizeof(uint32_t));
    t.keys0 = take((size_t)cap * sizeof(uint64_t));
    t.vals0 = take((size_t)cap * sizeof(uint32_t));
    t.keys1 = take((size_t)cap * sizeof(uint64_t));
    t.vals1 = take((size_t)cap * sizeof(uint32_t));
    t.count = take(sizeof(uint32_t));
    t.hdr = take(sizeof(WsHeader));
    t.look = take((size_t)SORT_MAX_PASSES * t.blocks * SORT_RADIX * sizeof(uint32_t));
    t.total = o;
    return t;
}

size_t spatial_order_temp_bytes(int64_t n) { return order_temp(n).total; }

cudaError_t launch_spatial_order(const float *P, int64_t ld, int64_t n, uint32_t *perm, void *temp,
                                 cudaStream_t s) {
    const OrderTemp t = order_temp(n);
    uint32_t *bbox = at<uint32_t>(temp, t.bbox);
    cudaMemsetAsync(bbox, 0xff, 3 * sizeof(uint32_t), s);
    cudaMemsetAsync(bbox + 3, 0, 3 * sizeof(uint32_t), s);
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    k_bbox<<<grid, 256, 0, s>>>(P, ld, n, bbox);
    uint64_t *k0 = at<uint64_t>(temp, t.keys0);
    uint32_t *v0 = at<uint32_t>(temp, t.vals0);
    k_morton<<<grid, 256, 0, s>>>(P, ld, n, bbox, k0, v0, at<uint32_t>(temp, t.count));
    cudaError_t e = launch_sort(k0, v0, at<uint64_t>(temp, t.keys1), at<uint32_t>(temp, t.vals1),
                                at<uint32_t>(temp, t.count), t.blocks * SORT_TILE, 30, at<WsHeader>(temp, t.hdr),
                                at<uint32_t>(temp, t.look), t.blocks, s);
    if (e != cudaSuccess) return e;
    // the sort leaves the result in the primary buffers (k_sort_fixup)
    return cudaMemcpyAsync(perm, v0, (size_t)n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
}

cudaError_t launch_permute_columns(const float *src, float *dst, int64_t ld, int rows, int64_t n,
                                   const uint32_t *perm, cudaStream_t s) {
    if (n == 0 || rows == 0) return cudaGetLastError();
    dim3 grid((unsigned)((n + 255) / 256), (unsigned)rows);
    k_permute_columns<<<grid, 256, 0, s>>>(src, dst, ld, n, perm);
    return cudaGetLastError();
}

}  // namespace gsk
