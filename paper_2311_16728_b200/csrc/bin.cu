// bin.cu -- A3-A5 binning by tile buckets (the default binning path).
//
// Same result as key duplication + a global stable sort of (tile << 32 | depth_bits) keys
// (SPEC.md:348 (2)-(3); R10/R11), computed as an MSD radix sort whose first digit is the whole
// tile id:
//   1. A1 counts the pairs of every (view, tile) with atomics while it projects (no key array);
//   2. an exclusive scan of the V*tiles counts gives each tile's range (and the total P);
//   3. k_bin_scatter writes each pair's (depth_bits << 32 | gaussian id) into its tile's bucket
//      (slot from a per-tile atomic cursor -- arbitrary order inside the bucket);
//   4. k_tile_sort sorts every bucket by (depth_bits, id) in shared memory (bitonic network,
//      padded to a power of two) -- (depth, id) is unique, so the order is exactly the stable
//      order of the global sort -- and writes the sorted values, the full keys and the range.
// Buckets longer than the shared-memory capacity (4096 pairs) are sorted with the same network
// in global memory (correct, slower; only for extreme tile lists).  Compared with the global LSD sort
// this reads/writes each pair ~3 times instead of 2 x (number of 8-bit digits) and replaces
// ~10 dependent launches per iteration by 3.
#include "gs_internal.cuh"

namespace gsk {

constexpr int TS_THREADS = 512;
constexpr int TS_SMEM_KEYS = 4096;  // 32 KB of u64 keys per CTA

// One thread per visible Gaussian (compacted list).  When the V*tiles table fits in shared
// memory, a CTA first counts its pairs per tile there, reserves each tile's sub-range with one
// global atomic per (CTA, tile) on the padded cursors, then hands out slots with shared-memory
// atomics -- so global atomic traffic is one per touched tile per CTA, not one per pair.
__global__ void __launch_bounds__(256) k_bin_scatter(const int4 *__restrict__ rect, const int32_t *__restrict__ radius,
                                                     const float *__restrict__ depth,
                                                     const uint32_t *__restrict__ vis_list,
                                                     const uint32_t *__restrict__ tile_start,
                                                     uint32_t *__restrict__ cursor, int64_t n, int V, int TX,
                                                     int tiles, int64_t cap, uint64_t *__restrict__ tmp,
                                                     WsHeader *hdr) {
    extern __shared__ uint32_t s_bins[];  // [0, VT): counts then running slot; [VT, 2 VT): base
    const int VT = V * tiles;
    const bool use_smem = VT <= SMEM_BINS;  // uniform (the launch passes 2*VT words of dynamic smem)
    if ((int64_t)hdr->P > cap) {  // capacity overflow: flag it, emit nothing
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&hdr->flags, 1u);
        return;
    }
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = t < hdr->vis_count;
    const uint32_t gi = live ? vis_list[t] : 0u;
    if (use_smem) {
        for (int b = threadIdx.x; b < VT; b += blockDim.x) s_bins[b] = 0;
        __syncthreads();
        if (live)
            for (int v = 0; v < V; v++) {
                const int64_t m = (int64_t)v * n + gi;
                if (radius[m] <= 0) continue;
                const int4 r = rect[m];
                for (int ty = r.y; ty < r.w; ty++)
                    for (int tx = r.x; tx < r.z; tx++) atomicAdd(&s_bins[v * tiles + ty * TX + tx], 1u);
            }
        __syncthreads();
        for (int b = threadIdx.x; b < VT; b += blockDim.x) {
            uint32_t c = s_bins[b];
            s_bins[VT + b] = c ? tile_start[b] + atomicAdd(&cursor[(size_t)b * CNT_STRIDE], c) : 0u;
            s_bins[b] = 0;
        }
        __syncthreads();
    }
    if (!live) return;
    for (int v = 0; v < V; v++) {
        const int64_t m = (int64_t)v * n + gi;
        if (radius[m] <= 0) continue;
        const int4 r = rect[m];
        const uint64_t key = (uint64_t)__float_as_uint(depth[m]) << 32 | gi;
        const uint32_t tb = (uint32_t)v * tiles;
        for (int ty = r.y; ty < r.w; ty++)
            for (int tx = r.x; tx < r.z; tx++) {
                const uint32_t gt = tb + ty * TX + tx;
                const uint32_t pos = use_smem ? s_bins[VT + gt] + atomicAdd(&s_bins[gt], 1u)
                                              : tile_start[gt] + atomicAdd(&cursor[(size_t)gt * CNT_STRIDE], 1u);
                tmp[pos] = key;
            }
    }
}

// Bitonic network over `len` (power of two) keys at `a`, CTA-wide: every stage is len/2
// compare-exchanges indexed by pair q (no idle lanes), separated by barriers.
__device__ __forceinline__ void bitonic(uint64_t *a, int len) {
    const int half = len >> 1;
    for (int k = 2; k <= len; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int q = threadIdx.x; q < half; q += blockDim.x) {
                const int i = ((q & ~(j - 1)) << 1) | (q & (j - 1));
                const int p = i + j;
                uint64_t x = a[i], y = a[p];
                const bool up = (i & k) == 0;
                if ((x > y) == up) {
                    a[i] = y;
                    a[p] = x;
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(TS_THREADS) k_tile_sort(const uint32_t *__restrict__ tile_start,
                                                          const uint32_t *__restrict__ tile_count, int64_t cap,
                                                          uint64_t *__restrict__ tmp, uint64_t *__restrict__ keys,
                                                          uint32_t *__restrict__ vals, uint2 *__restrict__ ranges,
                                                          uint64_t *__restrict__ big, const WsHeader *hdr) {
    __shared__ uint64_t sk[TS_SMEM_KEYS];
    const uint32_t gt = blockIdx.x;
    const bool ok = (int64_t)hdr->P <= cap;
    const uint32_t start = ok ? tile_start[gt] : 0u;
    const uint32_t len = ok ? tile_count[(size_t)gt * CNT_STRIDE] : 0u;
    // empty tiles keep the (0, 0) range of the other binning path and of the oracle
    if (threadIdx.x == 0) ranges[gt] = len ? make_uint2(start, start + len) : make_uint2(0u, 0u);
    if (len == 0) return;
    const uint64_t hi = (uint64_t)gt << 32;
    if (len <= TS_SMEM_KEYS) {
        int lp = 1;
        while (lp < (int)len) lp <<= 1;
        for (int i = threadIdx.x; i < lp; i += TS_THREADS) sk[i] = i < (int)len ? tmp[start + i] : ~0ull;
        __syncthreads();
        bitonic(sk, lp);
        for (int i = threadIdx.x; i < (int)len; i += TS_THREADS) {
            uint64_t k = sk[i];
            vals[start + i] = (uint32_t)k;
            keys[start + i] = hi | (k >> 32);
        }
    } else {
        // long bucket: the same network in global memory, on a padded copy in this bucket's own
        // region [2*start, 2*start + 2*len) of the overflow buffer (lp <= 2*len; disjoint per CTA)
        int lp = 1;
        while (lp < (int)len) lp <<= 1;
        uint64_t *g = big + 2 * (size_t)start;
        for (int i = threadIdx.x; i < lp; i += TS_THREADS) g[i] = i < (int)len ? tmp[start + i] : ~0ull;
        __threadfence_block();
        __syncthreads();
        bitonic(g, lp);
        for (int i = threadIdx.x; i < (int)len; i += TS_THREADS) {
            uint64_t k = g[i];
            vals[start + i] = (uint32_t)k;
            keys[start + i] = hi | (k >> 32);
        }
    }
}

cudaError_t launch_bin(const Layout &L, void *ws, cudaStream_t s) {
    const int64_t VT = (int64_t)L.V * L.tiles;
    cudaMemsetAsync(at<char>(ws, L.tile_cursor), 0, (size_t)VT * CNT_STRIDE * sizeof(uint32_t), s);
    const size_t smem = VT <= SMEM_BINS ? (size_t)2 * VT * sizeof(uint32_t) : 0;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_bin_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             2 * SMEM_BINS * (int)sizeof(uint32_t));
        attr = true;
    }
    if (L.n > 0)
        k_bin_scatter<<<(unsigned)((L.n + 255) / 256), 256, smem, s>>>(
            at<int4>(ws, L.rect), at<int32_t>(ws, L.radius), at<float>(ws, L.depth), at<uint32_t>(ws, L.vis_list),
            at<uint32_t>(ws, L.tile_start), at<uint32_t>(ws, L.tile_cursor), L.n, L.V, L.TX, L.tiles, L.cap,
            at<uint64_t>(ws, L.keys1), at<WsHeader>(ws, L.hdr));
    ProfScope prof("k_tile_sort", s);
    k_tile_sort<<<(unsigned)VT, TS_THREADS, 0, s>>>(at<uint32_t>(ws, L.tile_start), at<uint32_t>(ws, L.tile_count),
                                                    L.cap, at<uint64_t>(ws, L.keys1), at<uint64_t>(ws, L.keys0),
                                                    at<uint32_t>(ws, L.vals0), at<uint2>(ws, L.ranges),
                                                    at<uint64_t>(ws, L.bin_big), at<WsHeader>(ws, L.hdr));
    return cudaGetLastError();
}

}  // namespace gsk
