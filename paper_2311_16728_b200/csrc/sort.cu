// sort.cu -- A2 (exclusive scan of tiles touched), A3 (key duplication), A4 (stable LSD
// radix sort of (key, value) pairs) and A5 (tile ranges).
//
// SPEC.md:348 (2) "bin survivors into 16x16-pixel tiles", (3) "per tile, sort contributors
// by ascending depth (ties by primitive id)"; R10/R11: key = (view*tiles + tile) << 32 |
// float_bits(depth) (depth > znear > 0, so the bits order like the values), emitted per
// Gaussian in index order and per tile row-major; a stable sort therefore orders equal keys
// by Gaussian index.  Everything runs without a host sync: the pair count P stays on the
// device, grids are sized by capacity and CTAs beyond P exit.
//
// The sort is a hand-written onesweep-style LSD radix sort (Adinets & Merrill 2022): one
// upfront histogram of every digit, then one kernel per 8-bit digit that ranks a 4096-pair
// tile with warp-level match/popc (stable), resolves its global digit offsets with a
// decoupled look-back over the preceding CTAs, stages the tile in shared memory in sorted
// order and writes it out coalesced.  Passes whose digit is constant over all keys are
// skipped on the device (the source/destination of each pass is chosen by the histogram
// kernel), which removes the constant high bits of depth.
#include "gs_internal.cuh"

namespace gsk {

// ------------------------------------------------------------------------------------ scan
constexpr uint64_t SCAN_FLAG_A = 1ull << 62;  // aggregate available
constexpr uint64_t SCAN_FLAG_P = 2ull << 62;  // inclusive prefix available
constexpr uint64_t SCAN_VAL = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t *p) {
    return *reinterpret_cast<const volatile uint64_t *>(p);
}
__device__ __forceinline__ void st_volatile_u64(uint64_t *p, uint64_t v) {
    *reinterpret_cast<volatile uint64_t *>(p) = v;
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t *p) {
    return *reinterpret_cast<const volatile uint32_t *>(p);
}
__device__ __forceinline__ void st_volatile_u32(uint32_t *p, uint32_t v) {
    *reinterpret_cast<volatile uint32_t *>(p) = v;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan(const uint32_t *__restrict__ in, uint32_t *__restrict__ out,
                                                       int64_t M, uint64_t *flags, WsHeader *hdr, int stride) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    __shared__ uint32_t s_bid;
    __shared__ uint32_t s_warp[SCAN_THREADS / 32];
    __shared__ uint64_t s_prefix;
    int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_bid = atomicAdd(&hdr->scan_ctr, 1u);
    __syncthreads();
    int64_t bid = s_bid;
    int64_t base = bid * SCAN_TILE + (int64_t)tid * SCAN_ITEMS;
    uint32_t v[SCAN_ITEMS];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        int64_t idx = base + k;
        v[k] = idx < M ? in[idx * stride] : 0u;
        sum += v[k];
    }
    // block exclusive scan of per-thread sums
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < SCAN_THREADS / 32 ? s_warp[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < SCAN_THREADS / 32) s_warp[lane] = wi - w;  // exclusive warp offsets
        uint32_t agg = __shfl_sync(0xffffffffu, wi, SCAN_THREADS / 32 - 1);
        if (lane == 0) {
            // decoupled look-back (single thread; predecessors are already running)
            uint64_t excl = 0;
            if (bid == 0) {
                st_volatile_u64(&flags[0], SCAN_FLAG_P | (uint64_t)agg);
            } else {
                st_volatile_u64(&flags[bid], SCAN_FLAG_A | (uint64_t)agg);
                int64_t look = bid - 1;
                while (look >= 0) {
                    uint64_t f = ld_volatile_u64(&flags[look]);
                    if ((f >> 62) == 0) continue;
                    excl += f & SCAN_VAL;
                    if (f & SCAN_FLAG_P) break;
                    look--;
                }
                st_volatile_u64(&flags[bid], SCAN_FLAG_P | (excl + agg));
            }
            s_prefix = excl;
            if ((bid + 1) * SCAN_TILE >= M) hdr->P = (uint32_t)(excl + agg);  // last CTA: total pairs
        }
    }
    __syncthreads();
    uint32_t run = (uint32_t)s_prefix + s_warp[warp] + (incl - sum);
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        int64_t idx = base + k;
        if (idx < M) out[idx] = run;
        run += v[k];
    }
}

cudaError_t launch_scan_u32(const uint32_t *in, uint32_t *out, int64_t count, uint64_t *flags, WsHeader *hdr,
                            cudaStream_t s, int in_stride) {
    if (count == 0) return cudaGetLastError();
    launch_pdl(k_scan, (unsigned)((count + SCAN_TILE - 1) / SCAN_TILE), SCAN_THREADS, 0, s, in, out, count, flags, hdr,
                                                                                    in_stride);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ duplicate
__global__ void __launch_bounds__(256) k_duplicate(const int4 *__restrict__ rect, const uint32_t *__restrict__ off,
                                                   const uint32_t *__restrict__ tt, const float4 *__restrict__ rec0,
                                                   const float4 *__restrict__ rec1, const uint64_t *__restrict__ tmask,
                                                   const float *__restrict__ depth,
                                                   int64_t n, int64_t M, int TX, int tiles, int64_t cap,
                                                   uint64_t *__restrict__ keys, uint32_t *__restrict__ vals,
                                                   WsHeader *hdr) {
    int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= M) return;
    if ((int64_t)hdr->P > cap) {  // capacity overflow: flag it, emit nothing
        if (m == 0) atomicOr(&hdr->flags, 1u);
        return;
    }
    uint32_t cnt = tt[m];
    if (cnt == 0) return;
    int64_t o = off[m];
    int64_t view = m / n;
    uint32_t gi = (uint32_t)(m - view * n);
    int4 r = rect[m];
    uint32_t bits = __float_as_uint(depth[m]);
    uint64_t tbase = (uint64_t)view * tiles;
    for_each_binned_tile(r, tmask[m], rec0, rec1, m, [&](int tx, int ty) {  // R10'
        keys[o] = ((tbase + (uint64_t)(ty * TX + tx)) << 32) | bits;
        vals[o] = gi;
        o++;
    });
}

cudaError_t launch_duplicate(const Layout &L, void *ws, cudaStream_t s) {
    if (L.M == 0) return cudaGetLastError();
    k_duplicate<<<(L.M + 255) / 256, 256, 0, s>>>(
        at<int4>(ws, L.rect), at<uint32_t>(ws, L.offsets), at<uint32_t>(ws, L.tiles_touched), at<float4>(ws, L.rec0),
        at<float4>(ws, L.rec1), at<uint64_t>(ws, L.tile_mask), at<float>(ws, L.depth),
        L.n, L.M, L.TX, L.tiles, L.cap, at<uint64_t>(ws, L.keys0), at<uint32_t>(ws, L.vals0), at<WsHeader>(ws, L.hdr));
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ radix sort
// Pair count seen by the sort / ranges / raster: 0 after a capacity overflow (the outputs of
// that call are invalid and flagged; nothing reads or writes beyond the buffers).
__device__ __forceinline__ uint32_t count_of(const uint32_t *count, int64_t cap) {
    uint32_t c = *count;
    return c > cap ? 0u : c;
}

// One pass over all keys: histogram of every digit; the last CTA scans them and decides which
// passes are trivial (a digit shared by every key) and the buffer each pass reads.
__global__ void __launch_bounds__(256) k_sort_hist(const uint64_t *__restrict__ keys, const uint32_t *count,
                                                   int64_t cap, int passes, WsHeader *hdr) {
    __shared__ uint32_t s_h[SORT_MAX_PASSES][SORT_RADIX];
    __shared__ bool s_last;
    for (int k = threadIdx.x; k < SORT_MAX_PASSES * SORT_RADIX; k += blockDim.x) (&s_h[0][0])[k] = 0;
    __syncthreads();
    uint32_t P = count_of(count, cap);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = keys[i];
        for (int p = 0; p < passes; p++) atomicAdd(&s_h[p][(k >> (p * SORT_BITS)) & (SORT_RADIX - 1)], 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < passes * SORT_RADIX; k += blockDim.x) {
        uint32_t c = (&s_h[0][0])[k];
        if (c) atomicAdd(&(&hdr->sort_hist[0][0])[k], c);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&hdr->hist_ctr, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // last CTA: exclusive scan of each pass histogram (warp p handles pass p)
    __shared__ int s_triv[SORT_MAX_PASSES];
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < passes) {
        volatile uint32_t *h = hdr->sort_hist[warp];
        uint32_t run = 0;
        bool trivial = false;
        for (int c = 0; c < SORT_RADIX; c += 32) {
            uint32_t x = h[c + lane];
            trivial |= __any_sync(0xffffffffu, x == P);
            uint32_t incl = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            hdr->sort_start[warp][c + lane] = run + incl - x;
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) s_triv[warp] = trivial || P == 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int sel = 0;
        for (int p = 0; p < passes; p++) {
            hdr->sort_sel[p] = sel;
            hdr->sort_ctr[p] = s_triv[p] ? 0xFFFFFFFFu : 0u;  // 0xFFFFFFFF marks a skipped pass
            if (!s_triv[p]) sel ^= 1;
        }
        hdr->sort_sel[passes] = sel;
    }
}

constexpr uint32_t LB_FLAG_A = 1u << 30;
constexpr uint32_t LB_FLAG_P = 2u << 30;
constexpr uint32_t LB_VAL = (1u << 30) - 1;

struct SortSmem {
    uint32_t whist[SORT_THREADS / 32][SORT_RADIX];  // per-warp digit counts -> exclusive warp offsets
    uint32_t local_start[SORT_RADIX];              // digit start inside the tile
    uint32_t global_start[SORT_RADIX];             // digit start in the output
    uint64_t keys[SORT_TILE];
    uint32_t vals[SORT_TILE];
    uint32_t bid;
};

__global__ void __launch_bounds__(SORT_THREADS) k_sort_pass(uint64_t *k0, uint32_t *v0, uint64_t *k1, uint32_t *v1,
                                                            const uint32_t *count, int64_t cap, int pass,
                                                            WsHeader *hdr, uint32_t *lookback, int64_t nblk) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem &S = *reinterpret_cast<SortSmem *>(smem_raw);
    int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t ctr_word = ld_volatile_u32(&hdr->sort_ctr[pass]);
    if (ctr_word == 0xFFFFFFFFu) return;  // trivial pass: skipped on the device
    if (tid == 0) S.bid = atomicAdd(&hdr->sort_ctr[pass], 1u);
    for (int k = tid; k < (SORT_THREADS / 32) * SORT_RADIX; k += SORT_THREADS) (&S.whist[0][0])[k] = 0;
    __syncthreads();
    const uint32_t P = count_of(count, cap);
    const int64_t bid = S.bid;
    const int64_t base = bid * SORT_TILE;
    if (base >= P) return;
    const int sel = hdr->sort_sel[pass];
    const uint64_t *sk = sel ? k1 : k0;
    const uint32_t *sv = sel ? v1 : v0;
    uint64_t *dk = sel ? k0 : k1;
    uint32_t *dv = sel ? v0 : v1;
    const int shift = pass * SORT_BITS;
    const int tile_n = (int)(((int64_t)P - base) < SORT_TILE ? ((int64_t)P - base) : SORT_TILE);
    // warp-striped load: warp w owns [w*32*ITEMS, (w+1)*32*ITEMS) of the tile
    uint64_t key[SORT_ITEMS];
    uint32_t val[SORT_ITEMS];
    uint32_t dig[SORT_ITEMS];
    uint32_t rank[SORT_ITEMS];
    const int wbase = warp * 32 * SORT_ITEMS;
#pragma unroll
    for (int j = 0; j < SORT_ITEMS; j++) {
        int li = wbase + j * 32 + lane;
        bool ok = li < tile_n;
        key[j] = ok ? sk[base + li] : 0ull;
        val[j] = ok ? sv[base + li] : 0u;
        dig[j] = ok ? (uint32_t)((key[j] >> shift) & (SORT_RADIX - 1)) : 0x100u;
    }
    // stable warp ranking: items are visited in tile order (j outer, lane inner)
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < SORT_ITEMS; j++) {
        uint32_t d = dig[j];
        uint32_t peers = __match_any_sync(0xffffffffu, d);
        int leader = __ffs(peers) - 1;
        uint32_t before = 0;
        if (lane == leader && d < SORT_RADIX) {
            before = S.whist[warp][d];
            S.whist[warp][d] = before + __popc(peers);
        }
        before = __shfl_sync(0xffffffffu, before, leader);
        rank[j] = before + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();
    // per digit (thread d): warp counts -> exclusive warp offsets; tile total
    uint32_t total = 0;
    {
        int d = tid;  // SORT_THREADS == SORT_RADIX
#pragma unroll
        for (int w = 0; w < SORT_THREADS / 32; w++) {
            uint32_t c = S.whist[w][d];
            S.whist[w][d] = total;
            total += c;
        }
        // publish the tile aggregate for the look-back
        uint32_t *lb = lookback + (size_t)pass * nblk * SORT_RADIX;
        if (bid == 0) {
            st_volatile_u32(&lb[d], LB_FLAG_P | total);
        } else {
            st_volatile_u32(&lb[(size_t)bid * SORT_RADIX + d], LB_FLAG_A | total);
        }
        // exclusive scan of totals over digits (block scan) -> local_start
        uint32_t incl = total;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        __shared__ uint32_t s_wsum[SORT_THREADS / 32];
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        uint32_t woff = 0;
        for (int w = 0; w < warp; w++) woff += s_wsum[w];
        S.local_start[d] = woff + incl - total;
        // decoupled look-back over preceding tiles for digit d
        uint32_t excl = 0;
        if (bid > 0) {
            int64_t look = bid - 1;
            while (true) {
                uint32_t f = ld_volatile_u32(&lb[(size_t)look * SORT_RADIX + d]);
                if ((f >> 30) == 0) continue;
                excl += f & LB_VAL;
                if (f & LB_FLAG_P) break;
                look--;
            }
            st_volatile_u32(&lb[(size_t)bid * SORT_RADIX + d], LB_FLAG_P | (excl + total));
        }
        S.global_start[d] = hdr->sort_start[pass][d] + excl;
    }
    __syncthreads();
    // scatter into shared memory in tile-sorted order
#pragma unroll
    for (int j = 0; j < SORT_ITEMS; j++) {
        uint32_t d = dig[j];
        if (d < SORT_RADIX) {
            uint32_t pos = S.local_start[d] + S.whist[warp][d] + rank[j];
            S.keys[pos] = key[j];
            S.vals[pos] = val[j];
        }
    }
    __syncthreads();
    // coalesced write-out
    for (int li = tid; li < tile_n; li += SORT_THREADS) {
        uint64_t k = S.keys[li];
        uint32_t d = (uint32_t)((k >> shift) & (SORT_RADIX - 1));
        uint32_t gpos = S.global_start[d] + (uint32_t)li - S.local_start[d];
        dk[gpos] = k;
        dv[gpos] = S.vals[li];
    }
}

// Copy the result back to the primary buffers if the number of executed passes was odd.
__global__ void k_sort_fixup(uint64_t *k0, uint32_t *v0, const uint64_t *k1, const uint32_t *v1,
                             const uint32_t *count, int64_t cap, const WsHeader *hdr, int passes) {
    if (hdr->sort_sel[passes] == 0) return;
    uint32_t P = count_of(count, cap);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        k0[i] = k1[i];
        v0[i] = v1[i];
    }
}

int sort_passes(int key_bits) { return (key_bits + SORT_BITS - 1) / SORT_BITS; }

int hi_bits_for(int64_t count) {
    int b = 0;
    while ((1ll << b) < count) b++;
    return b;
}

static int g_num_sms = 0;
static int num_sms() {
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

cudaError_t launch_sort(uint64_t *k0, uint32_t *v0, uint64_t *k1, uint32_t *v1, const uint32_t *count, int64_t cap,
                        int key_bits, WsHeader *hdr, uint32_t *lookback, int64_t sort_blocks, cudaStream_t s) {
    int passes = sort_passes(key_bits);
    if (passes > SORT_MAX_PASSES || cap == 0) return cudaGetLastError();
    // reset the sort section of the header (counters, histograms)
    cudaMemsetAsync(&hdr->hist_ctr, 0,
                    offsetof(WsHeader, sort_start) - offsetof(WsHeader, hist_ctr), s);
    cudaMemsetAsync(lookback, 0, (size_t)passes * sort_blocks * SORT_RADIX * sizeof(uint32_t), s);
    int hist_blocks = (int)std::min<int64_t>(2 * num_sms(), (cap + 255) / 256);
    if (hist_blocks < 1) hist_blocks = 1;
    k_sort_hist<<<hist_blocks, 256, 0, s>>>(k0, count, cap, passes, hdr);
    size_t smem = sizeof(SortSmem);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_sort_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set = true;
    }
    ProfScope prof("k_sort_pass", s);
    for (int p = 0; p < passes; p++)
        k_sort_pass<<<sort_blocks, SORT_THREADS, smem, s>>>(k0, v0, k1, v1, count, cap, p, hdr, lookback, sort_blocks);
    k_sort_fixup<<<std::max(1, num_sms() * 4), 256, 0, s>>>(k0, v0, k1, v1, count, cap, hdr, passes);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ ranges
__global__ void __launch_bounds__(256) k_ranges(const uint64_t *__restrict__ keys, const uint32_t *count, int64_t cap,
                                                uint2 *__restrict__ ranges) {
    uint32_t P = count_of(count, cap);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t t = (uint32_t)(keys[i] >> 32);
        if (i == 0 || (uint32_t)(keys[i - 1] >> 32) != t) ranges[t].x = (uint32_t)i;
        if (i == P - 1 || (uint32_t)(keys[i + 1] >> 32) != t) ranges[t].y = (uint32_t)(i + 1);
    }
}

cudaError_t launch_ranges(const Layout &L, void *ws, cudaStream_t s) {
    cudaMemsetAsync(at<char>(ws, L.ranges), 0, (size_t)L.V * L.tiles * sizeof(uint2), s);
    int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(num_sms() * 8, (L.cap + 255) / 256));
    k_ranges<<<blocks, 256, 0, s>>>(at<uint64_t>(ws, L.keys0), &at<WsHeader>(ws, L.hdr)->P, L.cap,
                                    at<uint2>(ws, L.ranges));
    return cudaGetLastError();
}

}  // namespace gsk
