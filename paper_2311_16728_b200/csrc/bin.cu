// bin.cu -- A3-A5 binning by tile buckets (the default binning path).
//
// Same result as key duplication + a global stable sort of (tile << 32 | depth_bits) keys
// (SPEC.md:348 (2)-(3); R10/R11), computed as an MSD radix sort whose first digit is the whole
// tile id:
//   1. A1 counts the pairs of every (view, tile) with atomics while it projects (no key array);
//   2. an exclusive scan of the V*tiles counts gives each tile's range (and the total P);
//   3. k_bin_scatter writes each pair's (depth_bits << 32 | gaussian id) into its tile's bucket
//      (slot from a per-tile atomic cursor -- arbitrary order inside the bucket);
//   4. every bucket is sorted by (depth_bits, id) with a bitonic network padded to a power of
//      two -- (depth, id) is unique, so the order is exactly the stable order of the global
//      sort -- and the sorted values, the full keys and the range are written.  Buckets of up
//      to 256 pairs are sorted by a group of two warps (k_tile_sort_small), longer ones are
//      queued for k_tile_sort_big (a CTA of 16 warps, up to 4096 pairs; a longer list is sorted
//      as 4096-pair windows by separate CTAs, then merged by the CTA that finishes last).  Keys live
//      in registers; short exchange distances use shuffles, long ones shared memory.  The
//      sorted pairs' 48-byte raster records are gathered in the same pass (raster.cu).
// Compared with the global LSD sort this reads/writes each pair ~3 times instead of
// 2 x (number of 8-bit digits) and replaces ~10 dependent launches per iteration by 4.
#include <algorithm>

#include "gs_internal.cuh"


namespace gsk {


// One thread per visible Gaussian (compacted list).  When the V*tiles table fits in shared
// memory, a CTA first counts its pairs per tile there, reserves each tile's sub-range with one
// global atomic per (CTA, tile) on the padded cursors, then hands out slots with shared-memory
// atomics -- so global atomic traffic is one per touched tile per CTA, not one per pair.
constexpr int BIN_THREADS = 256;  // threads (visible Gaussians) per k_bin_scatter CTA

__global__ void __launch_bounds__(BIN_THREADS) k_bin_scatter(const int4 *__restrict__ rect, const int32_t *__restrict__ radius,
                                                     const float4 *__restrict__ rec0, const float4 *__restrict__ rec1,
                                                     const uint64_t *__restrict__ tmask,
                                                     const float *__restrict__ depth,
                                                     const uint32_t *__restrict__ vis_list,
                                                     const uint32_t *__restrict__ tile_start,
                                                     uint32_t *__restrict__ cursor, int64_t n, int V, int TX,
                                                     int tiles, int64_t cap, uint64_t *__restrict__ tmp,
                                                     WsHeader *hdr) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    extern __shared__ uint32_t s_bins[];  // [0, VT): counts then running slot; [VT, 2 VT): base
    const int VT = V * tiles;
    const bool use_smem = VT <= SMEM_BINS;  // uniform (the launch passes 2*VT words of dynamic smem)
    if ((int64_t)hdr->P > cap) {  // capacity overflow: flag it, emit nothing
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&hdr->flags, 1u);
        return;
    }
    // the grid covers all n Gaussians; CTAs past the compacted visible list have nothing to bin
    if (blockIdx.x * blockDim.x >= hdr->vis_count) return;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = t < hdr->vis_count;
    const uint32_t gi = live ? vis_list[t] : 0u;
    // every lane stays to the end: rects of > 64 tiles are binned by the whole warp
    // (warp_big_rects), the others by their own lane from the hit mask
    auto big_args = [&](int64_t m, bool big, float4 &g, float &C) {
        g = big ? rec0[m] : make_float4(0.f, 0.f, 0.f, 0.f);
        C = big ? rec1[m].x : 0.f;
    };
    if (use_smem) {
        for (int b = threadIdx.x; b < VT; b += blockDim.x) s_bins[b] = 0;
        __syncthreads();
        for (int v = 0; v < V; v++) {
            const int64_t m = (int64_t)v * n + gi;
            const bool vis = live && radius[m] > 0;
            const int4 r = vis ? rect[m] : make_int4(0, 0, 0, 0);
            const bool big = (r.z - r.x) * (r.w - r.y) > 64;
            if (vis && !big)
                for_each_binned_tile(r, tmask[m], rec0, rec1, m,
                                     [&](int tx, int ty) { atomicAdd(&s_bins[v * tiles + ty * TX + tx], 1u); });
            float4 g;
            float C;
            big_args(m, big, g, C);
            warp_big_rects(
                big, r, g.x, g.y, g.z, g.w, C, 0ull,
                [&](uint64_t, int tx, int ty) { atomicAdd(&s_bins[v * tiles + ty * TX + tx], 1u); },
                [](int, uint32_t) {});
        }
        __syncthreads();
        for (int b = threadIdx.x; b < VT; b += blockDim.x) {
            uint32_t c = s_bins[b];
            s_bins[VT + b] = c ? tile_start[b] + atomicAdd(&cursor[(size_t)b * CNT_STRIDE], c) : 0u;
            s_bins[b] = 0;
        }
        __syncthreads();
    }
    for (int v = 0; v < V; v++) {
        const int64_t m = (int64_t)v * n + gi;
        const bool vis = live && radius[m] > 0;
        const int4 r = vis ? rect[m] : make_int4(0, 0, 0, 0);
        const bool big = (r.z - r.x) * (r.w - r.y) > 64;
        const uint64_t key = vis ? (uint64_t)__float_as_uint(depth[m]) << 32 | gi : 0ull;
        const uint32_t tb = (uint32_t)v * tiles;
        auto emit = [&](uint64_t k, int tx, int ty) {
            const uint32_t gt = tb + ty * TX + tx;
            const uint32_t pos = use_smem ? s_bins[VT + gt] + atomicAdd(&s_bins[gt], 1u)
                                          : tile_start[gt] + atomicAdd(&cursor[(size_t)gt * CNT_STRIDE], 1u);
            tmp[pos] = k;
        };
        if (vis && !big) for_each_binned_tile(r, tmask[m], rec0, rec1, m, [&](int tx, int ty) { emit(key, tx, ty); });
        float4 g;
        float C;
        big_args(m, big, g, C);
        warp_big_rects(big, r, g.x, g.y, g.z, g.w, C, key, emit, [](int, uint32_t) {});
    }
}


// ---- group bitonic sort: a group of W warps holds lp = 32 E W keys in registers; key g (its
// bitonic index) = w * 32 E + e * 32 + lane (striped, so loads and stores coalesce).  Distances
// j < 32 are exchanged with shuffles, 32 <= j < 32 E inside the thread, j >= 32 E through shared
// memory with a group barrier per stage.  Pair direction: ascending iff (g & k) == 0.
// distances JMAX, JMAX / 2, ..., 1 of the merge step k (all static: no divergent-looking
// branches around the shuffles)
template <int E, int JMAX>
__device__ __forceinline__ void merge_regs(uint64_t (&x)[E], int lane, int gw, int k) {
#pragma unroll
    for (int j = JMAX; j >= 1; j >>= 1) {
        if (j >= 32) {
            const int ej = j >> 5;
#pragma unroll
            for (int e = 0; e < E; e++)
                if ((e & ej) == 0) {
                    const bool up = ((gw + e * 32 + lane) & k) == 0;
                    const uint64_t a = x[e], b = x[e | ej];
                    const bool sw = (a > b) == up;
                    x[e] = sw ? b : a;
                    x[e | ej] = sw ? a : b;
                }
        } else {
            const bool lower = (lane & j) == 0;
#pragma unroll
            for (int e = 0; e < E; e++) {
                const bool up = ((gw + e * 32 + lane) & k) == 0;
                const uint64_t a = x[e];
                const uint64_t b = __shfl_xor_sync(0xffffffffu, a, j);
                const bool take_min = lower == up;
                x[e] = take_min ? (a < b ? a : b) : (a < b ? b : a);
            }
        }
    }
}

// merge steps k = K, 2K, ..., 32 E (each entirely in registers)
template <int E, int K>
__device__ __forceinline__ void sort_regs(uint64_t (&x)[E], int lane, int gw) {
    merge_regs<E, K / 2>(x, lane, gw, K);
    if constexpr (K < 32 * E) sort_regs<E, 2 * K>(x, lane, gw);
}

__device__ __forceinline__ void group_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Sort the bucket tmp[start, start + len) (len <= 32 E W) with a group of W warps (group-local
// thread index gt_idx, named barrier bar_id; sk = 32 E W keys of shared memory) and write the
// sorted values and full keys (hi | depth bits).
struct RecSrc {  // per-(view, Gaussian) record sources for the fused pair-record gather
    const float4 *rec0, *rec1, *rec2;
    float4 *prec;
    int64_t vbase;  // view * n of the bucket's view
};

// One merge step k of the network on the window of LP = 32 E W keys held in registers (x, key
// (base + gw + e * 32 + lane)), for the distances j = min(k / 2, LP / 2) ... 1: j >= 32 E through
// shared memory (group barrier per stage), j < 32 E in registers.  base is the window's offset in
// the whole (padded) bucket; directions use the global index, so windows compose into one network.
template <int E, int W>
__device__ __forceinline__ void merge_window(uint64_t (&x)[E], uint64_t *sk, int gt_idx, int bar_id, int base, int k) {
    constexpr int LP = 32 * E * W, NTH = 32 * W;
    const int lane = gt_idx & 31;
    const int gw = (gt_idx >> 5) * 32 * E;
    if (k >= 64 * E) {
#pragma unroll
        for (int e = 0; e < E; e++) sk[gw + e * 32 + lane] = x[e];
        group_bar(bar_id, NTH);
        for (int j = min(k, LP) >> 1; j >= 32 * E; j >>= 1) {
            for (int q = gt_idx; q < LP / 2; q += NTH) {
                const int i = ((q & ~(j - 1)) << 1) | (q & (j - 1));
                const int p = i + j;
                const uint64_t a = sk[i], c = sk[p];
                if ((a > c) == (((base + i) & k) == 0)) {
                    sk[i] = c;
                    sk[p] = a;
                }
            }
            group_bar(bar_id, NTH);
        }
#pragma unroll
        for (int e = 0; e < E; e++) x[e] = sk[gw + e * 32 + lane];
        merge_regs<E, 16 * E>(x, lane, base + gw, k);
        group_bar(bar_id, NTH);  // sk is rewritten by the next step
    } else {
        merge_regs<E, 16 * E>(x, lane, base + gw, k);  // (only reached with k < 64 E from sort_window)
    }
}

// Sort the window (merge steps k = 2 .. LP) in place in registers.
template <int E, int W>
__device__ __forceinline__ void sort_window(uint64_t (&x)[E], uint64_t *sk, int gt_idx, int bar_id, int base) {
    constexpr int LP = 32 * E * W;
    const int lane = gt_idx & 31;
    const int gw = (gt_idx >> 5) * 32 * E;
    sort_regs<E, 2>(x, lane, base + gw);  // k = 2 .. 32 E
    for (int k = 64 * E; k <= LP; k <<= 1) merge_window<E, W>(x, sk, gt_idx, bar_id, base, k);
}

__device__ __forceinline__ void emit_pair(uint64_t k, uint32_t pos, uint64_t hi, uint64_t *keys, uint32_t *vals,
                                          const RecSrc &rs) {
    const uint32_t gi = (uint32_t)k;
    vals[pos] = gi;
    keys[pos] = hi | (k >> 32);
    write_pair_record(rs.prec, pos, rs.rec0, rs.rec1, rs.rec2, rs.vbase + gi, gi);
}

// Sort the bucket tmp[start, start + len) (len <= 32 E W) with a group of W warps (group-local
// thread index gt_idx, named barrier bar_id; sk = 32 E W keys of shared memory) and write the
// sorted values, full keys (hi | depth bits) and pair records.
template <int E, int W>
__device__ __forceinline__ void group_sort(const uint64_t *__restrict__ tmp, uint32_t start, uint32_t len,
                                           uint64_t hi, uint64_t *__restrict__ keys, uint32_t *__restrict__ vals,
                                           uint64_t *sk, int gt_idx, int bar_id, const RecSrc &rs) {
    const int lane = gt_idx & 31;
    const int gw = (gt_idx >> 5) * 32 * E;
    uint64_t x[E];
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint32_t g = gw + e * 32 + lane;
        x[e] = g < len ? tmp[start + g] : ~0ull;
    }
    sort_window<E, W>(x, sk, gt_idx, bar_id, 0);
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint32_t g = gw + e * 32 + lane;
        if (g < len) emit_pair(x[e], start + g, hi, keys, vals, rs);
    }
}

constexpr int SG_WARPS = 2;   // warps of the small-bucket CTA (<= 256 pairs)
constexpr int BG_WARPS = 16;   // warps of the long-bucket CTA (<= 4096 pairs)
constexpr int BG_MAX = 4096;    // longest bucket sorted in one register / shared-memory window

// Pass 1: one 2-warp CTA per (view, tile) (tile = blockIdx.x, so every branch below is provably
// uniform and the shuffles need no warp re-convergence).  Writes the range; sorts buckets of
// <= 256 pairs; queues longer buckets for pass 2.
__global__ void __launch_bounds__(SG_WARPS * 32) k_tile_sort_small(
    const uint32_t *__restrict__ tile_start, const uint32_t *__restrict__ tile_count, int64_t cap,
    const uint64_t *__restrict__ tmp, uint64_t *__restrict__ keys, uint32_t *__restrict__ vals,
    uint2 *__restrict__ ranges, uint2 *__restrict__ big_items, WsHeader *hdr, RecSrc rs, int64_t n, int tiles) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    __shared__ uint64_t sk[256];
    const int gt = blockIdx.x;
    rs.vbase = (int64_t)(gt / tiles) * n;
    const bool ok = (int64_t)hdr->P <= cap;
    const uint32_t start = ok ? tile_start[gt] : 0u;
    const uint32_t len = ok ? tile_count[(size_t)gt * CNT_STRIDE] : 0u;
    // empty tiles keep the (0, 0) range of the other binning path and of the oracle
    if (threadIdx.x == 0) ranges[gt] = len ? make_uint2(start, start + len) : make_uint2(0u, 0u);
    const uint64_t hi = (uint64_t)gt << 32;
    if (len == 0) return;
    if (len <= 64) group_sort<1, SG_WARPS>(tmp, start, len, hi, keys, vals, sk, threadIdx.x, 1, rs);
    else if (len <= 128) group_sort<2, SG_WARPS>(tmp, start, len, hi, keys, vals, sk, threadIdx.x, 1, rs);
    else if (len <= 256) group_sort<4, SG_WARPS>(tmp, start, len, hi, keys, vals, sk, threadIdx.x, 1, rs);
    else if (threadIdx.x == 0) {  // one work item per BG_MAX-pair window of the bucket
        const uint32_t nwin = (len + BG_MAX - 1) / BG_MAX;
        const uint32_t b = atomicAdd(&hdr->n_big, nwin);
        for (uint32_t w = 0; w < nwin; w++) big_items[b + w] = make_uint2((uint32_t)gt, w);
    }
}

// Merge of the sorted runs [0, r), [r, 2r), ... of src (length len) into dst, pairwise, by the
// whole CTA: each thread takes a contiguous slice of the merged output of a pair and finds where
// it starts in the two runs by binary search on the diagonal (merge path; keys are unique, so
// the split is exact), then merges its slice sequentially.
__device__ void merge_pairs(const uint64_t *__restrict__ src, uint64_t *__restrict__ dst, uint32_t len, uint32_t r,
                            int tid, int nth) {
    for (uint32_t lo = 0; lo < len; lo += 2 * r) {
        const uint32_t la = min(r, len - lo), lb = min(r, len - lo - la);
        const uint64_t *a = src + lo, *b = a + la;
        const uint32_t tot = la + lb, per = (tot + nth - 1) / nth;
        const uint32_t d0 = min(tot, (uint32_t)tid * per), d1 = min(tot, d0 + per);
        if (d0 < d1) {
            // smallest i with a[i] > b[d0 - i - 1] (i elements of a precede output d0)
            uint32_t ilo = d0 > lb ? d0 - lb : 0u, ihi = min(d0, la);
            while (ilo < ihi) {
                const uint32_t i = (ilo + ihi) / 2;
                if (a[i] < b[d0 - i - 1]) ilo = i + 1; else ihi = i;
            }
            uint32_t i = ilo, j = d0 - ilo;
            for (uint32_t d = d0; d < d1; d++) {
                const bool ta = j >= lb || (i < la && a[i] < b[j]);
                dst[lo + d] = ta ? a[i++] : b[j++];
            }
        }
    }
}

// Pass 2: one CTA of 16 warps per queued work item (grid-stride): buckets of up to 4096 pairs
// are sorted in registers and shared memory and emitted; a longer bucket is one item per
// 4096-pair window -- each window sorted by its own CTA into the bucket's scratch region (so the
// windows of one long tile list sort in parallel), and the CTA that finishes the bucket's last
// window (per-bucket counter: slot 1 of the tile's padded cursor line, zeroed with the cursors)
// merges the sorted windows pairwise (merge path) and emits the pairs.
__global__ void __launch_bounds__(BG_WARPS * 32) k_tile_sort_big(
    const uint32_t *__restrict__ tile_start, const uint32_t *__restrict__ tile_count, const uint64_t *__restrict__ tmp,
    uint64_t *__restrict__ keys, uint32_t *__restrict__ vals, const uint2 *__restrict__ big_items,
    uint64_t *__restrict__ big, uint32_t *__restrict__ done, const WsHeader *hdr, RecSrc rs, int64_t n, int tiles) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    constexpr int W = BG_WARPS, NTH = 32 * BG_WARPS;
    __shared__ __align__(16) uint64_t sk[BG_MAX];
    __shared__ bool s_last;
    const uint32_t nb = hdr->n_big;
    for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const uint2 item = big_items[b];
        const uint32_t gt = item.x, w = item.y;
        const uint32_t start = tile_start[gt];
        const uint32_t len = tile_count[(size_t)gt * CNT_STRIDE];
        const uint64_t hi = (uint64_t)gt << 32;
        rs.vbase = (int64_t)(gt / tiles) * n;
        if (len <= 512) group_sort<1, W>(tmp, start, len, hi, keys, vals, sk, threadIdx.x, 1, rs);
        else if (len <= 1024) group_sort<2, W>(tmp, start, len, hi, keys, vals, sk, threadIdx.x, 1, rs);
        else if (len <= 2048) group_sort<4, W>(tmp, start, len, hi, keys, vals, sk, threadIdx.x, 1, rs);
        else if (len <= BG_MAX) group_sort<8, W>(tmp, start, len, hi, keys, vals, sk, threadIdx.x, 1, rs);
        else {
            // window w, sorted into the bucket's scratch region [2 start, 2 start + 2 len): runs
            // in the first half, the merge ping-pongs with the second
            uint64_t *A = big + 2 * (size_t)start, *B = A + len;
            const uint32_t w0 = w * BG_MAX, wlen = min((uint32_t)BG_MAX, len - w0);
            constexpr int E = 8;
            const int lane = threadIdx.x & 31, gw = (threadIdx.x >> 5) * 32 * E;
            uint64_t x[E];
#pragma unroll
            for (int e = 0; e < E; e++) {
                const uint32_t g = gw + e * 32 + lane;
                x[e] = g < wlen ? tmp[start + w0 + g] : ~0ull;
            }
            sort_window<E, W>(x, sk, threadIdx.x, 1, 0);
#pragma unroll
            for (int e = 0; e < E; e++) {
                const uint32_t g = gw + e * 32 + lane;
                if (g < wlen) A[w0 + g] = x[e];
            }
            __threadfence();
            __syncthreads();
            const uint32_t nwin = (len + BG_MAX - 1) / BG_MAX;
            if (threadIdx.x == 0) s_last = atomicAdd(&done[(size_t)gt * CNT_STRIDE + 1], 1u) == nwin - 1;
            __syncthreads();
            if (s_last) {
                __threadfence();
                uint64_t *src = A, *dst = B;
                for (uint32_t r = BG_MAX; r < len; r *= 2) {
                    merge_pairs(src, dst, len, r, threadIdx.x, NTH);
                    __threadfence_block();
                    __syncthreads();
                    uint64_t *t = src;
                    src = dst;
                    dst = t;
                }
                for (uint32_t i = threadIdx.x; i < len; i += NTH) emit_pair(src[i], start + i, hi, keys, vals, rs);
            }
        }
        __syncthreads();
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
    if (L.n > 0) {
        ProfScope prof_scatter("k_bin_scatter", s);
        launch_pdl(k_bin_scatter, (unsigned)((L.n + BIN_THREADS - 1) / BIN_THREADS), BIN_THREADS, smem, s, 
            at<int4>(ws, L.rect), at<int32_t>(ws, L.radius), at<float4>(ws, L.rec0), at<float4>(ws, L.rec1),
            at<uint64_t>(ws, L.tile_mask), at<float>(ws, L.depth), at<uint32_t>(ws, L.vis_list),
            at<uint32_t>(ws, L.tile_start), at<uint32_t>(ws, L.tile_cursor), L.n, L.V, L.TX, L.tiles, L.cap,
            at<uint64_t>(ws, L.keys1), at<WsHeader>(ws, L.hdr));
    }
    ProfScope prof("k_tile_sort", s);
    const RecSrc rs{at<float4>(ws, L.rec0), at<float4>(ws, L.rec1), at<float4>(ws, L.rec2), at<float4>(ws, L.prec), 0};
    launch_pdl(k_tile_sort_small, (unsigned)VT, SG_WARPS * 32, 0, s,
               at<uint32_t>(ws, L.tile_start), at<uint32_t>(ws, L.tile_count), L.cap, at<uint64_t>(ws, L.keys1),
               at<uint64_t>(ws, L.keys0), at<uint32_t>(ws, L.vals0), at<uint2>(ws, L.ranges),
               at<uint2>(ws, L.big_tiles), at<WsHeader>(ws, L.hdr), rs, L.n, L.tiles);
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    // 16-warp CTAs: up to 4 resident per SM
    // one CTA per queued item where possible (items: buckets of <= 4096 pairs, windows of longer ones)
    launch_pdl(k_tile_sort_big, (unsigned)std::min<int64_t>(VT + L.cap / BG_MAX + 1, 4 * sms), BG_WARPS * 32, 0, s,
               at<uint32_t>(ws, L.tile_start), at<uint32_t>(ws, L.tile_count), at<uint64_t>(ws, L.keys1),
               at<uint64_t>(ws, L.keys0), at<uint32_t>(ws, L.vals0), at<uint2>(ws, L.big_tiles),
               at<uint64_t>(ws, L.bin_big), at<uint32_t>(ws, L.tile_cursor), at<WsHeader>(ws, L.hdr), rs, L.n,
               L.tiles);
    return cudaGetLastError();
}

}  // namespace gsk
