// raster.cu -- A6 (per-tile front-to-back alpha compositing, Eq. 3) and A8 (its backward).
//
// Eq. 3 with the reading prod_{j<i}(1 - alpha_j) (R1), evaluated per
// pixel over the depth-sorted list of its tile (SPEC.md:348 (4)): power = -1/2 d^T Q d with
// d = pixel - mean2d (fp32 recipe order, bit-exact to the oracle), cut at power < -4.5
// (Mahalanobis^2 > 9, R9) or power > 0; alpha = min(0.99, sigma e^power) (R7); skip alpha
// < 1/255; stop the pixel when T (1 - alpha) < 1e-4 (R8).
//
// Data movement: after binning, k_gather_pairs writes one 48-byte record per (tile, Gaussian)
// pair in sorted order -- (u, v, A, B), (C, sigma, r, g), (b, id, -, q_limit) -- so a tile's
// list is one contiguous range.  The raster kernels stream it into shared memory with TMA
// bulk copies (cp.async.bulk + mbarrier complete_tx), double-buffered: the copy of batch b+1
// is in flight while batch b is composited, and no thread waits on dependent gathers.
//
// Layout: one thread per pixel; each warp owns an 8x4 pixel block (2 x 4 blocks per 16x16
// tile); a CTA holds 8 warps (a whole tile) or, at pyramid levels with fewer lists than
// 2 x SMs, one warp (eight CTAs per tile) so that every SM gets work.  For every batch
// of 256 records each warp builds, in parallel over the batch (one record per lane, ballot +
// popc), the ordered list of Gaussians that can reach its block: the exact minimum of d^T Q d
// over the block is compared with the Gaussian's limit min(9, 2 ln(255 sigma)) (3-sigma
// cutoff or alpha >= 1/255), padded so the test is conservative.  The sequential per-pixel
// loop only visits that list -- no pixel result changes.  A CTA leaves as soon as all of its
// pixels have stopped.
//
// The backward replays each pixel's list back to front: dL/dc, dL/dalpha
// = T_k sum_c g_c (c_k - acc), dL/dsigma, dL/dpower -> dL/dmean2d, dL/dconic.  A warp owns an
// 8x8 block as four 4x4 quadrants of eight lanes (two pixels per lane); each quadrant culls
// and walks its own list, and the nine per-pixel gradients of its Gaussian are summed over its
// eight lanes with a transposing butterfly (10 shuffles) and added to the per-(view, Gaussian)
// record with one scalar red.global.add per lane.
#include "gs_internal.cuh"

namespace gsk {

#define FMA __fmaf_rn
#define MUL __fmul_rn
#define SUB __fsub_rn

constexpr float ALPHA_MAX = 0.99f;
constexpr float ALPHA_MIN = 1.0f / 255.0f;
constexpr float T_STOP = 1e-4f;
constexpr float POWER_CUT = -4.5f;
constexpr int BATCH = 256;  // records per staged batch (list indices fit in a byte)
// backward: per-lane atomics instead of the group reductions when no quadrant group has more
// than this many contributing lanes (measured: chunked 3, 5, 7; tile-serial 2, 3, 6, 8)
constexpr int FEW_CHUNK = 5;
constexpr int FEW_TILEQ = 3;

// power = -1/2 (A dx^2 + C dy^2) - B dx dy in the recipe's op order.  The pair records carry
// the conic pre-scaled, (hA, nB, hC) = (-A/2, -B, -C/2) (write_pair_record): scaling by -1/2 is
// exact and commutes with rounding, so fma(hC dy, dy, (hA dx) dx) is the recipe's -0.5 qf bit
// for bit and nB dx its -(B dx) -- the same power, one multiplication fewer per pixel and entry.
__device__ __forceinline__ float pixel_power(float px, float py, const float4 g0, float hC, float &dx, float &dy) {
    dx = SUB(px, g0.x);
    dy = SUB(py, g0.y);
    const float hq = FMA(MUL(hC, dy), dy, MUL(MUL(g0.z, dx), dx));
    return FMA(MUL(g0.w, dx), dy, hq);
}

// e^power with the SFU: ex2.approx.ftz(power * log2 e).  Forward and backward evaluate alpha
// with this same sequence, so their skip / stop decisions agree bit for bit.
__device__ __forceinline__ float fast_exp(float power) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(power * 1.4426950408889634f));
    return y;
}

// Conservative warp-level skip: minimum of d^T Q d over the warp's pixel block (centres
// [x0, x0 + 7] x [y0, y0 + 3]) exceeds the Gaussian's limit.  Exact box-ellipse minimum:
// 0 if the mean is inside, else the smallest of the four clamped edge minima.  The padding
// (1e-3 relative + 1e-3 absolute) absorbs the rounding of the per-pixel fp32 power, so a
// culled Gaussian can never pass the per-pixel tests.
__device__ __forceinline__ bool block_misses(const float4 g0, const float4 g1, float qlim, float x0, float y0,
                                             float h = 3.f, float w = 7.f) {
    if (qlim < 0.f) return true;
    const float A = -2.f * g0.z, B = -g0.w, C = -2.f * g1.x;  // the record's pre-scaled conic (exact)
    const float ax = x0 - g0.x, bx = x0 + w - g0.x, ay = y0 - g0.y, by = y0 + h - g0.y;
    if (ax <= 0.f && bx >= 0.f && ay <= 0.f && by >= 0.f) return false;
    float best = 3.4e38f;
    // edges x = X: f = A X^2 + 2 B X y + C y^2, y* = -B X / C clamped to [ay, by].  The
    // minimiser may be approximate (SFU reciprocals): f is evaluated exactly at a feasible
    // point, and a point off the true minimiser by a relative 1e-7 raises f by O(1e-14),
    // far inside the padding
    float rC, rA;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rC) : "f"(C));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rA) : "f"(A));
    const float nBC = -B * rC, nBA = -B * rA;
#pragma unroll
    for (int e = 0; e < 2; e++) {
        float X = e ? bx : ax;
        float y = fminf(fmaxf(nBC * X, ay), by);
        best = fminf(best, A * X * X + 2.f * B * X * y + C * y * y);
        float Y = e ? by : ay;
        float x = fminf(fmaxf(nBA * Y, ax), bx);
        best = fminf(best, A * x * x + 2.f * B * x * Y + C * Y * Y);
    }
    return best > qlim * 1.001f + 1e-3f;
}

// ---------------------------------------------------------------- per-pair records (gather)
// rec[pos] = (u, v, -A/2, -B) | (-C/2, sigma, r, g) | (b, id bits, 0, q_limit(sigma)), pos < P.
__global__ void __launch_bounds__(256) k_gather_pairs(const uint32_t *__restrict__ vals,
                                                      const uint64_t *__restrict__ keys,
                                                      const float4 *__restrict__ rec0,
                                                      const float4 *__restrict__ rec1,
                                                      const float4 *__restrict__ rec2, int64_t n, int tiles,
                                                      const uint32_t *count, int64_t cap,
                                                      float4 *__restrict__ prec) {
    uint32_t P = *count;
    if (P > cap) P = 0;  // overflow: nothing valid to gather
    for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < P;
         pos += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t gi = vals[pos];
        const int64_t view = (int64_t)(keys[pos] >> 32) / tiles;
        write_pair_record(prec, pos, rec0, rec1, rec2, view * n + gi, gi);
    }
}

// ---------------------------------------------------------------- TMA bulk copy + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
}
// one elected thread: expect `bytes` on the barrier and start the global -> shared bulk copy
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

struct RasterSmem {
    // double-buffered batch of pair records (2 x 12 KB) + one sentinel record per buffer at
    // index BATCH (never written by the bulk copies): the forward pads its groups with it
    float4 rec[2][(BATCH + 1) * 3];
    uint64_t bar[2];
};
// the sentinel: far away (power -> -inf: cut), sigma 0 (alpha 0), q_limit -1
__device__ __forceinline__ void init_sentinel(RasterSmem &S, int tid) {
    if (tid < 2) {
        S.rec[tid][3 * BATCH] = make_float4(-1e6f, -1e6f, 1.f, 0.f);
        S.rec[tid][3 * BATCH + 1] = make_float4(1.f, 0.f, 0.f, 0.f);
        S.rec[tid][3 * BATCH + 2] = make_float4(0.f, 0.f, 0.f, -1.f);
    }
}

// CTA = WARPS warps of one 16x16 tile: blockIdx.x = tile_x * (8 / WARPS) + sub-tile.
template <int WARPS>
__device__ __forceinline__ void warp_block(int bxi, int &tile_x, int &wx0, int &wy0, int &lx, int &ly) {
    constexpr int SUB = 8 / WARPS;
    const int sub = bxi % SUB;
    tile_x = bxi / SUB;
    const int wg = sub * WARPS + (threadIdx.x >> 5);  // warp block index 0..7 within the tile
    const int lane = threadIdx.x & 31;
    wx0 = (wg & 1) * 8;
    wy0 = (wg >> 1) * 4;
    lx = wx0 + (lane & 7);
    ly = wy0 + (lane >> 3);
}

// Per-pixel outputs of the forward: colour (+ T_final bg), T, last position, composited count;
// with CHUNKED the reverse pass turning the per-chunk records into (T after the chunk,
// normalised colour behind it) for the chunked backward.
template <bool CHUNKED, bool STATS = true>
__device__ __forceinline__ void fwd_finish(int view, int px, int py, int W, int H, float T, float c0, float c1,
                                           float c2, uint32_t last, uint32_t composited, float bg0, float bg1,
                                           float bg2, float *out_rgb, float *out_T, float *T_keep,
                                           uint32_t *ncontrib, uint32_t *ncomp, size_t chunk_base_tile, int lpix,
                                           float4 *chunk_bwd) {
    const int64_t HW = (int64_t)H * W;
    const int64_t pix = (int64_t)py * W + px;
    float *o = out_rgb + (int64_t)view * 3 * HW + pix;
    o[0] = c0 + T * bg0;
    o[HW] = c1 + T * bg1;
    o[2 * HW] = c2 + T * bg2;
    if (out_T) out_T[(int64_t)view * HW + pix] = T;
    T_keep[(int64_t)view * HW + pix] = T;
    ncontrib[(int64_t)view * HW + pix] = last;
    if (STATS) ncomp[(int64_t)view * HW + pix] = composited;
    if (CHUNKED && last > 0) {
        // reverse pass over the chunks up to the last composited one: normalised colour behind
        // each chunk, acc_end(k) = behind(k) / T_after(k), behind(k) = sum of the later chunks'
        // colour + T_final bg (positive terms only -- no cancellation); eight chunks per round,
        // their loads issued together before any store
        float e0 = T * bg0, e1 = T * bg1, e2 = T * bg2;
        float4 *col = chunk_bwd + chunk_base_tile * TILE_PIX + lpix;
        for (int k = (int)((last - 1) / CHUNK); k >= 0; k -= 8) {
            float4 e[8];
#pragma unroll
            for (int u = 0; u < 8; u++)
                if (k - u >= 0) e[u] = col[(size_t)(k - u) * TILE_PIX];
#pragma unroll
            for (int u = 0; u < 8; u++)
                if (k - u >= 0) {
                    const float inv = 1.0f / e[u].x;
                    col[(size_t)(k - u) * TILE_PIX] = make_float4(e[u].x, e0 * inv, e1 * inv, e2 * inv);
                    e0 += e[u].y;
                    e1 += e[u].z;
                    e2 += e[u].w;
                }
        }
    }
}

// STATS: also count the composited entries per pixel (n_composited, a diagnostic output:
// gs_set_render_stats) -- off on the hot path, where it costs 2 of ~33 instructions per entry
template <int WARPS, bool CHUNKED, bool STATS>
__global__ void __launch_bounds__(WARPS * 32) k_raster_fwd(const uint2 *__restrict__ ranges,
                                                           const float4 *__restrict__ prec, int W, int H, int TX,
                                                           int tiles, float bg0, float bg1, float bg2,
                                                           float *__restrict__ out_rgb, float *__restrict__ out_T,
                                                           float *__restrict__ T_keep, uint32_t *__restrict__ ncontrib,
                                                           uint32_t *__restrict__ ncomp,
                                                           const uint32_t *__restrict__ chunk_base,
                                                           float4 *__restrict__ chunk_bwd,
                                                           const uint32_t *__restrict__ order) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    constexpr int NT = WARPS * 32;
    __shared__ __align__(128) RasterSmem S;
    constexpr int SEG = CHUNKED ? CHUNK : BATCH;  // list segment = unit of chunk recording
    constexpr int NSEG = BATCH / SEG;
    constexpr int FG = 8;                       // list entries evaluated together in phase 2
    constexpr int SEGP = SEG + FG;              // segment stride: FG padding entries after each list
    __shared__ __align__(16) int wl[WARPS][NSEG * SEGP];  // segment s's selection at [s * SEGP, ...)
    __shared__ int segn[WARPS][NSEG];
    // tiles in longest-list-first order (shorter lists end the kernel: less tail); without an
    // order blockIdx decides
    int view = blockIdx.z, tile_y = blockIdx.y, bxi = blockIdx.x;
    if (order) {
        constexpr int SUB = 8 / WARPS;  // CTAs per tile
        const int64_t lin = ((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        const uint32_t gt = order[lin / SUB];
        view = gt / tiles;
        tile_y = (gt % tiles) / TX;
        bxi = (int)((gt % tiles) % TX) * SUB + (int)(lin % SUB);
    }
    int tile_x, bx0, by0, lx, ly;
    warp_block<WARPS>(bxi, tile_x, bx0, by0, lx, ly);
    const int tile = tile_y * TX + tile_x;
    const int tid = threadIdx.x;
    const int px = tile_x * TILE + lx;
    const int py = tile_y * TILE + ly;
    const float wx0 = (float)(tile_x * TILE + bx0);
    const float wy0 = (float)(tile_y * TILE + by0);
    const bool inside = px < W && py < H;
    const uint2 range = ranges[(int64_t)view * tiles + tile];
    const int todo_all = (int)(range.y - range.x);
    const float fx = (float)px, fy = (float)py;
    float T = 1.0f, c0 = 0.f, c1 = 0.f, c2 = 0.f;
    uint32_t last = 0, composited = 0;
    bool done = !inside;
    const int warp = tid >> 5, lane = tid & 31;
    const unsigned lt = (1u << lane) - 1u;
    const float4 *src = prec + 3 * (size_t)range.x;
    init_sentinel(S, tid);
    if (tid == 0) {
        mbar_init(&S.bar[0]);
        mbar_init(&S.bar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (todo_all > 0) bulk_load(S.rec[0], src, (uint32_t)min(BATCH, todo_all) * 48u, &S.bar[0]);
    }
    __syncthreads();
    uint32_t phases = 0u;                  // bit b = parity to wait for on buffer b
    int inflight = todo_all > 0 ? 0 : -1;  // buffer with an unconsumed copy (-1: none)
    for (int b0 = 0, it = 0; b0 < todo_all; b0 += BATCH, it++) {
        const int buf = it & 1;
        if (__syncthreads_count(done) == NT) break;
        const int cnt = min(BATCH, todo_all - b0);
        if (tid == 0 && b0 + BATCH < todo_all) {  // prefetch the next batch into the other buffer
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_load(S.rec[buf ^ 1], src + 3 * (size_t)(b0 + BATCH),
                      (uint32_t)min(BATCH, todo_all - b0 - BATCH) * 48u, &S.bar[buf ^ 1]);
        }
        mbar_wait(&S.bar[buf], (phases >> buf) & 1u);
        phases ^= 1u << buf;
        inflight = b0 + BATCH < todo_all ? (buf ^ 1) : -1;
        const float4 *r = S.rec[buf];
        // phase 1 (parallel over the batch): per SEG-entry segment, the ordered list of the
        // Gaussians that can reach this warp's 8x4 block
        int nsel = 0;
        for (int k = 0; k < cnt; k += 32) {
            const int seg = k / SEG;
            if (k % SEG == 0) nsel = 0;
            int j = k + lane;
            bool hit = j < cnt && !block_misses(r[3 * j], r[3 * j + 1], r[3 * j + 2].w, wx0, wy0);
            unsigned b = __ballot_sync(0xffffffffu, hit);
            if (hit) wl[warp][seg * SEGP + nsel + __popc(b & lt)] = j;
            nsel += __popc(b);
            if (k + 32 >= cnt || (k + 32) % SEG == 0) {  // segment complete: its count, and FG
                if (lane == 0) segn[warp][seg] = nsel;   // padding entries (the sentinel record:
                if (lane < FG) wl[warp][seg * SEGP + nsel + lane] = BATCH;  // never composited)
            }
        }
        __syncwarp();
        const int nseg = (cnt + SEG - 1) / SEG;
        for (int sg = 0; sg < nseg; sg++) {
            const bool active_in_seg = !done;    // this segment is a chunk the pixel reaches
            if (__all_sync(0xffffffffu, done)) break;
            float d0 = 0.f, d1 = 0.f, d2 = 0.f;  // colour composited in this segment
            const int ns = segn[warp][sg];
            const int *wls = &wl[warp][sg * SEGP];
            // phase 2 (sequential per pixel): composite the warp's list front to back, FG entries
            // at a time: their alphas (record loads, power, SFU exp) are independent and computed
            // first, then the compositing recurrence (T, C) runs over them branch-free -- the
            // latency of the independent part overlaps across the group
            for (int t = 0; t < ns; t += FG) {
                if (__all_sync(0xffffffffu, done)) break;
                const int4 ja = *reinterpret_cast<const int4 *>(&wls[t]);
                const int4 jb = *reinterpret_cast<const int4 *>(&wls[t + 4]);
                const int jj[FG] = {ja.x, ja.y, ja.z, ja.w, jb.x, jb.y, jb.z, jb.w};
                float al[FG], cr[FG], cg[FG], cb[FG];
                bool ok[FG];
#pragma unroll
                for (int k = 0; k < FG; k++) {
                    const int j = jj[k];  // past the list end: the sentinel (cut, alpha 0)
                    const float4 g0 = r[3 * j], g1 = r[3 * j + 1];
                    float dx, dy;
                    const float p = pixel_power(fx, fy, g0, g1.x, dx, dy);
                    al[k] = fminf(ALPHA_MAX, g1.y * fast_exp(p));
                    ok[k] = !(p > 0.0f || p < POWER_CUT) && al[k] >= ALPHA_MIN;
                    cr[k] = g1.z;
                    cg[k] = g1.w;
                    cb[k] = r[3 * j + 2].x;
                }
#pragma unroll
                for (int k = 0; k < FG; k++) {
                    const float test_T = __fmaf_rn(-T, al[k], T);  // T (1 - alpha) as one fma
                    const bool live = ok[k] && !done;
                    const bool stop = live && test_T < T_STOP;
                    const bool take = live && !(test_T < T_STOP);
                    done = done || stop;
                    const float w = take ? al[k] * T : 0.f;
                    d0 += cr[k] * w;
                    d1 += cg[k] * w;
                    d2 += cb[k] * w;
                    T = take ? test_T : T;
                    if constexpr (STATS) composited += take ? 1u : 0u;
                    if (take) last = (uint32_t)(b0 + jj[k] + 1);
                }
            }
            c0 += d0;
            c1 += d1;
            c2 += d2;
            // chunked backward (few tiles): record (T after this chunk, colour it composited)
            if (CHUNKED && inside && active_in_seg)
                chunk_bwd[((size_t)chunk_base[view * tiles + tile] + it * NSEG + sg) * TILE_PIX + ly * TILE + lx] =
                    make_float4(T, d0, d1, d2);
        }
    }
    // never leave with a bulk copy still writing into this CTA's shared memory
    if (inflight >= 0 && tid == 0) mbar_wait(&S.bar[inflight], (phases >> inflight) & 1u);
    if (inside)
        fwd_finish<CHUNKED, STATS>(view, px, py, W, H, T, c0, c1, c2, last, composited, bg0, bg1, bg2, out_rgb, out_T, T_keep,
                            ncontrib, ncomp, CHUNKED ? chunk_base[view * tiles + tile] : 0, ly * TILE + lx,
                            chunk_bwd);
}

// ================================================================ chunked backward (few tiles)
// At pyramid levels with few tiles (V * tiles < CHUNK_MAX_TILES) each warp of the tile-serial
// backward would walk a long list alone.  The forward (same kernel, CHUNKED instance) records,
// for every CHUNK-entry chunk of a tile list that a pixel reaches, the transmittance after the
// chunk and the colour composited in it; its epilogue turns these into the normalised colour
// behind each chunk (suffix sums of positive terms + T_final bg, no cancellation).  The backward
// then gives every chunk its own CTA (the whole tile, two pixels per lane), which replays that
// chunk back to front from (T after the chunk, colour behind it) -- the chunks run in parallel
// instead of one after the other, and the longest dependent chain is CHUNK entries.

// exclusive scan over the 1024 threads of a CTA (s_warp: 33 words of shared memory)
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t *s_warp, uint32_t &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    __syncthreads();  // s_warp may still be read by a previous call
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = s_warp[lane];
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += u;
        }
        s_warp[lane] = wi - w;
        if (lane == 31) s_warp[32] = wi;
    }
    __syncthreads();
    total = s_warp[32];
    return s_warp[warp] + incl - v;
}

// Backward schedule of the chunked path: chunks ordered by their position j in the tile list
// (first chunks first: most pixels are still active there, so the longest replays start
// first), positions >= 255 in one class.  Without per-chunk atomics: the tiles sorted by chunk
// count, descending (q(t): one shared atomic per tile for ties), make "the tiles with more
// than j chunks" a prefix of that order for every j, so chunk (t, j) goes to
// P_j + q(t) with P_j = sum_{j' < j} #{tiles with > j' chunks}.  chunk_base[] must be written
// (and visible to the CTA) before the call; nch(i) = chunks of list i; 1024 threads.
template <class NCH>
__device__ __forceinline__ void chunk_order_schedule(NCH nch, int VT, const uint32_t *__restrict__ chunk_base,
                                                     uint32_t *__restrict__ chunk_order, int64_t max_chunks,
                                                     uint32_t *s_warp, uint32_t *H /* [258] shared */) {
    const int t = threadIdx.x;
    if (t < 258) H[t] = 0;
    __syncthreads();
    for (int i = t; i < VT; i += 1024) {
        const uint32_t c = nch(i);
        atomicAdd(&H[min(c, 256u)], 1u);
        if (c > 255) atomicAdd(&H[257], c - 255);  // size of the j >= 255 class
    }
    __syncthreads();
    // S[v] = #tiles with min(nch, 256) > v (suffix sums): thread t holds bin 256 - t
    uint32_t dummy;
    const uint32_t hv = t <= 256 ? H[256 - t] : 0u;
    const uint32_t suf = block_exclusive_scan(hv, s_warp, dummy);  // sum over bins > 256 - t
    __syncthreads();
    uint32_t *S = H;  // reuse: S[v] for v = 0..256, class-255 size kept in H[257]
    const uint32_t big = H[257];
    __syncthreads();
    if (t <= 256) S[256 - t] = suf;
    __syncthreads();
    // P_j = sum_{j' < j} S[j'] for j = 0..255; class 255 holds the S[255] tiles' chunks >= 255
    const uint32_t m = t < 255 ? S[t] : (t == 255 ? big : 0u);
    const uint32_t Pj = block_exclusive_scan(m, s_warp, dummy);
    __shared__ uint32_t P[256], q_cur[257], c255;
    if (t < 256) P[t] = Pj;
    if (t <= 256) q_cur[t] = S[t];  // tiles with more chunks than v come first
    if (t == 0) c255 = 0;
    __syncthreads();
    for (int i = t; i < VT; i += 1024) {
        const uint32_t c = nch(i), base = chunk_base[i];
        const uint32_t q = atomicAdd(&q_cur[min(c, 256u)], 1u);  // position in the descending order
        const uint32_t jmax = min(c, 255u);
        for (uint32_t j = 0; j < jmax; j++) {
            const uint32_t pos = P[j] + q;
            if (pos < max_chunks && base + j < max_chunks) chunk_order[pos] = base + j;
        }
        for (uint32_t j = 255; j < c; j++) {
            const uint32_t pos = P[255] + atomicAdd(&c255, 1u);
            if (pos < max_chunks && base + j < max_chunks) chunk_order[pos] = base + j;
        }
    }
}

__global__ void __launch_bounds__(1024) k_chunk_index(const uint2 *__restrict__ ranges, int VT,
                                                      uint32_t *__restrict__ chunk_base,
                                                      uint32_t *__restrict__ chunk_tile,
                                                      uint32_t *__restrict__ chunk_order, WsHeader *hdr,
                                                      int64_t max_chunks) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    __shared__ uint32_t s_warp[33];
    __shared__ uint32_t H[258];
    const int t = threadIdx.x;
    const int per = (VT + 1023) / 1024;  // consecutive lists per thread for the tile-order scan
    const int i0 = t * per, i1 = min(VT, i0 + per);
    auto nch = [&](int i) { const uint2 r = ranges[i]; return (r.y - r.x + CHUNK - 1) / CHUNK; };
    uint32_t nsum = 0;
    for (int i = i0; i < i1; i++) nsum += nch(i);
    uint32_t total;
    uint32_t cb = block_exclusive_scan(nsum, s_warp, total);
    if (t == 0) hdr->nchunks = (uint32_t)min((int64_t)total, max_chunks);
    for (int i = i0; i < i1; i++) {
        chunk_base[i] = cb;
        cb += nch(i);
    }
    __syncthreads();
    for (int i = t; i < VT; i += 1024) {
        const uint32_t c = nch(i), base = chunk_base[i];
        for (uint32_t k = 0; k < c; k++)
            if (base + k < max_chunks) chunk_tile[base + k] = (uint32_t)i;
    }
    chunk_order_schedule(nch, VT, chunk_base, chunk_order, max_chunks, s_warp, H);
}

// ================================================================ two-pixel packed backward
// A warp owns an 8x8 block, every lane two pixels, evaluated with Blackwell's packed fp32x2
// instructions (FFMA2 / FMUL2 / FADD2, IEEE round-to-nearest per element, so the power and
// alpha of each pixel are the same bits as the scalar forward).  Per-pixel validity is folded
// into masked alphas instead of branches.
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Per-lane state of the lane's two pixels in the back-to-front replay.
struct Pix2 {
    float2 T, acc0, acc1, acc2, g0, g1, g2;  // T after the entry, colour behind, dL/dpixel
    uint32_t lastA, lastB;                   // 1-based list position of the last composited
};

// ---- quadrant groups: the warp's 8x8 block as four 4x4 quadrants, eight lanes each (lane
// 8q + i: quadrant q, pixels (i & 3, i >> 2) and (i & 3, (i >> 2) + 2) inside it).  Every group
// walks its own list -- the Gaussians that reach its 4x4 quadrant -- so a warp step advances
// four entries (one per group) and the walk is the longest of the four quadrant lists instead
// of the 8x8 block's list.  Replica-like map, mean over the warps without the stop at the
// last contributor: 283 vs 639 entries at level 2, 114 vs 224 at level 1, 62 vs 100 at level 0.

// Sums of nine values over the eight lanes of a group: the eight of a[] with a transposing
// butterfly at offsets 4, 2, 1 (lane i of the group ends with the total of value i), the ninth
// (b, total in every lane) summed alongside: 4 + 2 + 1 + 3 = 10 shuffles.
__device__ __forceinline__ float group_sum9_transposed(float a[8], float &b, int lane) {
    const bool b2 = lane & 4, b1 = lane & 2, b0 = lane & 1;
    float h[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const float send = b2 ? a[k] : a[k + 4];
        const float keep = b2 ? a[k + 4] : a[k];
        h[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    b += __shfl_xor_sync(0xffffffffu, b, 4);
    float q[2];
#pragma unroll
    for (int k = 0; k < 2; k++) {
        const float send = b1 ? h[k] : h[k + 2];
        const float keep = b1 ? h[k + 2] : h[k];
        q[k] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    b += __shfl_xor_sync(0xffffffffu, b, 2);
    const float send = b0 ? q[0] : q[1];
    const float r = (b0 ? q[1] : q[0]) + __shfl_xor_sync(0xffffffffu, send, 1);
    b += __shfl_xor_sync(0xffffffffu, b, 1);
    return r;
}

// One warp step of the quadrant-group replay: every group its own entry j (the sentinel past
// its list's end, 1-based list position `position`): recover T before it, dL/dalpha =
// T sum_c g_c (c - acc), then the gradient moments S(a), S(b), S(a dx), S(a dy), S(b dy) with
// a = dL/dpower dx, b = dL/dpower dy, dL/dsigma and dL/dcolour, summed over the group and
// added to its Gaussian's per-view record.  FEW (warp-uniform): if no group has more than FEW
// contributing lanes, those lanes add their own values.
template <int FEW>
__device__ __forceinline__ void bwdq_entry(Pix2 &P, const float4 *r, int j, uint32_t position, float fx,
                                           float2 fy2, int lane, float *g2dv) {
    const float4 g0 = r[3 * j], g1 = r[3 * j + 1];
    const float dx = SUB(fx, g0.x);
    const float2 dy2 = __fadd2_rn(fy2, f2(-g0.y));
    const float hAdxdx = MUL(MUL(g0.z, dx), dx);
    const float2 hq2 = __ffma2_rn(__fmul2_rn(f2(g1.x), dy2), dy2, f2(hAdxdx));
    const float2 p2 = __ffma2_rn(f2(MUL(g0.w, dx)), dy2, hq2);
    const float2 e2 = make_float2(fast_exp(p2.x), fast_exp(p2.y));
    const float2 araw = __fmul2_rn(f2(g1.y), e2);
    const float aA = fminf(ALPHA_MAX, araw.x), aB = fminf(ALPHA_MAX, araw.y);
    const bool vA = position <= P.lastA && !(p2.x > 0.0f || p2.x < POWER_CUT) && aA >= ALPHA_MIN;
    const bool vB = position <= P.lastB && !(p2.y > 0.0f || p2.y < POWER_CUT) && aB >= ALPHA_MIN;
    const unsigned bal = __ballot_sync(0xffffffffu, vA || vB);
    if (bal == 0u) return;
    const float2 al = make_float2(vA ? aA : 0.f, vB ? aB : 0.f);
    const float2 ua = make_float2(vA && !(araw.x > ALPHA_MAX) ? aA : 0.f, vB && !(araw.y > ALPHA_MAX) ? aB : 0.f);
    const float2 ue = make_float2(ua.x != 0.f ? e2.x : 0.f, ua.y != 0.f ? e2.y : 0.f);
    P.T = __fmul2_rn(P.T, make_float2(rcp_approx(1.0f - al.x), rcp_approx(1.0f - al.y)));
    const float2 w2 = __fmul2_rn(al, P.T);
    const float2 d0 = __fadd2_rn(f2(g1.z), make_float2(-P.acc0.x, -P.acc0.y));
    const float2 d1 = __fadd2_rn(f2(g1.w), make_float2(-P.acc1.x, -P.acc1.y));
    const float2 d2 = __fadd2_rn(f2(r[3 * j + 2].x), make_float2(-P.acc2.x, -P.acc2.y));
    const float2 dLda = __fmul2_rn(P.T, __ffma2_rn(P.g2, d2, __ffma2_rn(P.g1, d1, __fmul2_rn(P.g0, d0))));
    P.acc0 = __ffma2_rn(al, d0, P.acc0);
    P.acc1 = __ffma2_rn(al, d1, P.acc1);
    P.acc2 = __ffma2_rn(al, d2, P.acc2);
    const float2 dr = __fmul2_rn(P.g0, w2), dg = __fmul2_rn(P.g1, w2), db = __fmul2_rn(P.g2, w2);
    const float2 dsig = __fmul2_rn(ue, dLda);
    const float2 dp = __fmul2_rn(ua, dLda);
    const float2 a2 = __fmul2_rn(dp, f2(dx));
    const float2 b2 = __fmul2_rn(dp, dy2);
    const float2 qa = __fmul2_rn(a2, f2(dx));
    const float2 qb = __fmul2_rn(a2, dy2);
    const float2 qc = __fmul2_rn(b2, dy2);
    float vals8[8] = {a2.x + a2.y, b2.x + b2.y, qa.x + qa.y, qb.x + qb.y,
                      qc.x + qc.y, dsig.x + dsig.y, dr.x + dr.y, dg.x + dg.y};
    float v9 = db.x + db.y;
    const uint32_t gi = __float_as_uint(r[3 * j + 2].y);
    float *dst = g2dv + 12 * gi;
    const int gsh = lane & 24;  // this lane's group: ballot bits [gsh, gsh + 8)
    if (FEW > 0) {
        const bool few = __popc(bal & 0xffu) <= FEW && __popc(bal & 0xff00u) <= FEW &&
                         __popc(bal & 0xff0000u) <= FEW && __popc(bal & 0xff000000u) <= FEW;
        if (few) {
            if (vA || vB) {
#pragma unroll
                for (int k = 0; k < 8; k++) atomicAdd(dst + k, vals8[k]);
                atomicAdd(dst + 8, v9);
            }
            return;
        }
    }
    const float mine = group_sum9_transposed(vals8, v9, lane);
    if ((bal >> gsh) & 0xffu) {  // the group has a contribution (its entry is not the sentinel)
        const int i = lane & 7;
        atomicAdd(dst + i, mine);
        if (i == 0) atomicAdd(dst + 8, v9);
    }
}

// Chunked backward (levels with few tiles): one CTA (4 warps, 8x8 blocks) per chunk; the
// chunk's records are loaded once for the whole tile and culled as in k_raster_bwdq.
__global__ void __launch_bounds__(128) k_raster_bwdq_chunk(const uint2 *__restrict__ ranges,
                                                           const float4 *__restrict__ prec,
                                                           const uint32_t *__restrict__ chunk_base,
                                                           const uint32_t *__restrict__ chunk_tile,
                                                           const WsHeader *__restrict__ hdr, int64_t n, int W,
                                                           int H, int TX, int tiles,
                                                           const float *__restrict__ dL_drgb,
                                                           const uint32_t *__restrict__ ncontrib,
                                                           const float4 *__restrict__ chunk_bwd,
                                                           float4 *__restrict__ g2d,
                                                           const uint32_t *__restrict__ chunk_order) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    __shared__ __align__(128) float4 rec[(CHUNK + 1) * 3];  // + the sentinel at index CHUNK
    __shared__ uint64_t bar;
    __shared__ uint8_t wl[4][4][CHUNK];
    __shared__ uint8_t wl8[4][CHUNK];
    if ((int)blockIdx.x >= (int)hdr->nchunks) return;
    const int c = chunk_order[blockIdx.x];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane >> 3, gl = lane & 7;
    const uint32_t gt = chunk_tile[c];
    const int view = gt / tiles, tl = gt % tiles;
    const int tx = tl % TX, ty = tl / TX;
    const int qx = (warp & 1) * 8 + (q & 1) * 4, qy = (warp >> 1) * 8 + (q >> 1) * 4;  // quadrant origin
    const int lx = qx + (gl & 3), lyA = qy + (gl >> 2), lyB = lyA + 2;
    const int px = tx * TILE + lx, pyA = ty * TILE + lyA, pyB = ty * TILE + lyB;
    const uint2 range = ranges[gt];
    const int b0 = (int)(c - chunk_base[gt]) * CHUNK;
    const int cnt = min(CHUNK, (int)(range.y - range.x) - b0);
    const int64_t HW = (int64_t)H * W;
    Pix2 P;
    P.T = f2(1.f);
    P.acc0 = P.acc1 = P.acc2 = P.g0 = P.g1 = P.g2 = f2(0.f);
    P.lastA = P.lastB = 0;
    const float *gbase = dL_drgb + (int64_t)view * 3 * HW;
    const float4 *cb = chunk_bwd + (size_t)c * TILE_PIX;
    if (px < W && pyA < H) {
        const int64_t pix = (int64_t)pyA * W + px;
        const uint32_t last = ncontrib[(int64_t)view * HW + pix];
        if ((uint32_t)b0 < last) {  // this chunk holds composited entries of the pixel
            const float4 e = cb[lyA * TILE + lx];
            P.lastA = last;
            P.T.x = e.x;
            P.acc0.x = e.y;
            P.acc1.x = e.z;
            P.acc2.x = e.w;
            P.g0.x = gbase[pix];
            P.g1.x = gbase[HW + pix];
            P.g2.x = gbase[2 * HW + pix];
        }
    }
    if (px < W && pyB < H) {
        const int64_t pix = (int64_t)pyB * W + px;
        const uint32_t last = ncontrib[(int64_t)view * HW + pix];
        if ((uint32_t)b0 < last) {
            const float4 e = cb[lyB * TILE + lx];
            P.lastB = last;
            P.T.y = e.x;
            P.acc0.y = e.y;
            P.acc1.y = e.z;
            P.acc2.y = e.w;
            P.g0.y = gbase[pix];
            P.g1.y = gbase[HW + pix];
            P.g2.y = gbase[2 * HW + pix];
        }
    }
    uint32_t glast = max(P.lastA, P.lastB);  // the group's last composited position
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) glast = max(glast, __shfl_xor_sync(0xffffffffu, glast, o));
    uint32_t wlast = glast;
#pragma unroll
    for (int o = 16; o > 4; o >>= 1) wlast = max(wlast, __shfl_xor_sync(0xffffffffu, wlast, o));
    if (tid == 0) {
        mbar_init(&bar);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 3)  // the sentinel: far away (cut), sigma 0, id 0
        rec[3 * CHUNK + tid] = tid == 0 ? make_float4(-1e6f, -1e6f, 1.f, 0.f)
                                        : (tid == 1 ? make_float4(1.f, 0.f, 0.f, 0.f) : make_float4(0.f, 0.f, 0.f, -1.f));
    if (__syncthreads_or(wlast != 0) == 0) return;  // no pixel of the tile reaches this chunk
    if (tid == 0) bulk_load(rec, prec + 3 * ((size_t)range.x + b0), (uint32_t)cnt * 48u, &bar);
    if (wlast == 0) return;  // warp-uniform; the copy is waited on by the warps that use it
    mbar_wait(&bar, 0u);
    // per group: the entries (back to front) that can reach its 4x4 quadrant -- the warp's
    // 8x8 block culled first (one entry per lane), then each group tests the survivors
    const float fqx = (float)(tx * TILE + qx), fqy = (float)(ty * TILE + qy);
    const unsigned lt = (1u << gl) - 1u;
    int nsel = 0;
    int n8 = 0;
    {
        const float wx0 = (float)(tx * TILE + (warp & 1) * 8), wy0 = (float)(ty * TILE + (warp >> 1) * 8);
        const unsigned lt32 = (1u << lane) - 1u;
        for (int k = 0; k < cnt; k += 32) {
            const int jj = k + lane;
            const int idx = cnt - 1 - jj;
            const bool hit = jj < cnt && (uint32_t)(b0 + idx + 1) <= wlast &&
                             !block_misses(rec[3 * idx], rec[3 * idx + 1], rec[3 * idx + 2].w, wx0, wy0, 7.f, 7.f);
            const unsigned b = __ballot_sync(0xffffffffu, hit);
            if (hit) wl8[warp][n8 + __popc(b & lt32)] = (uint8_t)idx;
            n8 += __popc(b);
        }
        __syncwarp();
    }
    for (int k = 0; k < n8; k += 8) {
        const int e = k + gl;
        const int idx = e < n8 ? wl8[warp][e] : 0;
        const bool hit = e < n8 && (uint32_t)(b0 + idx + 1) <= glast &&
                         !block_misses(rec[3 * idx], rec[3 * idx + 1], rec[3 * idx + 2].w, fqx, fqy, 3.f, 3.f);
        const unsigned gb = (__ballot_sync(0xffffffffu, hit) >> (lane & 24)) & 0xffu;
        if (hit) wl[warp][q][nsel + __popc(gb & lt)] = (uint8_t)idx;
        nsel += __popc(gb);
    }
    __syncwarp();
    int nmax = nsel;
#pragma unroll
    for (int o = 16; o > 4; o >>= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
    const float fx = (float)px;
    const float2 fy2 = make_float2((float)pyA, (float)pyB);
    float *g2dv = reinterpret_cast<float *>(g2d + 3 * (int64_t)view * n);
    for (int t = 0; t < nmax; t++) {
        const int j = t < nsel ? wl[warp][q][t] : CHUNK;
        bwdq_entry<FEW_CHUNK>(P, rec, j, (uint32_t)(b0 + j + 1), fx, fy2, lane, g2dv);
    }
}

// Tile-serial backward (levels with many tiles): one CTA (4 warps) per 16x16 tile, TMA
// double-buffered record batches from the end of the list; the warp culls each batch against
// its 8x8 block, each eight-lane group the survivors against its 4x4 quadrant, and every group
// walks its own list.
__global__ void __launch_bounds__(128) k_raster_bwdq(const uint2 *__restrict__ ranges,
                                                     const float4 *__restrict__ prec, int64_t n, int W, int H,
                                                     int TX, int tiles, float bg0, float bg1, float bg2,
                                                     const float *__restrict__ dL_drgb,
                                                     const float *__restrict__ T_keep,
                                                     const uint32_t *__restrict__ ncontrib,
                                                     float4 *__restrict__ g2d, const uint32_t *__restrict__ order) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    __shared__ __align__(128) RasterSmem S;
    __shared__ uint8_t wl[4][4][BATCH];
    __shared__ uint8_t wl8[4][BATCH];
    __shared__ uint32_t s_maxlast;
    int view = blockIdx.z, ty = blockIdx.y, tx = blockIdx.x;
    if (order) {
        const uint32_t gt = order[((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x];
        view = gt / tiles;
        ty = (gt % tiles) / TX;
        tx = (gt % tiles) % TX;
    }
    const int tile = ty * TX + tx;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane >> 3, gl = lane & 7;
    const int qx = (warp & 1) * 8 + (q & 1) * 4, qy = (warp >> 1) * 8 + (q >> 1) * 4;  // quadrant origin
    const int px = tx * TILE + qx + (gl & 3);
    const int pyA = ty * TILE + qy + (gl >> 2), pyB = pyA + 2;
    const bool inA = px < W && pyA < H, inB = px < W && pyB < H;
    const uint2 range = ranges[(int64_t)view * tiles + tile];
    const float fx = (float)px;
    const float2 fy2 = make_float2((float)pyA, (float)pyB);
    float *g2dv = reinterpret_cast<float *>(g2d + 3 * (int64_t)view * n);
    const int64_t HW = (int64_t)H * W;
    const int64_t pixA = (int64_t)pyA * W + px, pixB = (int64_t)pyB * W + px;
    Pix2 P;
    P.T = f2(1.f);
    P.g0 = P.g1 = P.g2 = f2(0.f);
    P.lastA = P.lastB = 0;
    const float *gbase = dL_drgb + (int64_t)view * 3 * HW;
    if (inA) {
        P.T.x = T_keep[(int64_t)view * HW + pixA];
        P.lastA = ncontrib[(int64_t)view * HW + pixA];
        P.g0.x = gbase[pixA];
        P.g1.x = gbase[HW + pixA];
        P.g2.x = gbase[2 * HW + pixA];
    }
    if (inB) {
        P.T.y = T_keep[(int64_t)view * HW + pixB];
        P.lastB = ncontrib[(int64_t)view * HW + pixB];
        P.g0.y = gbase[pixB];
        P.g1.y = gbase[HW + pixB];
        P.g2.y = gbase[2 * HW + pixB];
    }
    init_sentinel(S, tid);
    if (tid == 0) {
        s_maxlast = 0;
        mbar_init(&S.bar[0]);
        mbar_init(&S.bar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t glast = max(P.lastA, P.lastB);  // the group's last composited position
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) glast = max(glast, __shfl_xor_sync(0xffffffffu, glast, o));
    uint32_t wlast = glast;
#pragma unroll
    for (int o = 16; o > 4; o >>= 1) wlast = max(wlast, __shfl_xor_sync(0xffffffffu, wlast, o));
    if (lane == 0) atomicMax(&s_maxlast, wlast);
    __syncthreads();
    const int todo_all = (int)s_maxlast;
    const float4 *src = prec + 3 * (size_t)range.x;
    if (tid == 0 && todo_all > 0) {
        int cnt0 = min(BATCH, todo_all);
        bulk_load(S.rec[0], src + 3 * (size_t)(todo_all - cnt0), (uint32_t)cnt0 * 48u, &S.bar[0]);
    }
    uint32_t phases = 0u;
    P.acc0 = f2(bg0);
    P.acc1 = f2(bg1);
    P.acc2 = f2(bg2);
    const unsigned lt = (1u << gl) - 1u;
    const float fqx = (float)(tx * TILE + qx), fqy = (float)(ty * TILE + qy);
    for (int b_end = todo_all, it = 0; b_end > 0; b_end -= BATCH, it++) {
        const int buf = it & 1;
        const int cnt = min(BATCH, b_end);
        const int b_start = b_end - cnt;
        __syncthreads();
        if (tid == 0 && b_start > 0) {
            int cn = min(BATCH, b_start);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_load(S.rec[buf ^ 1], src + 3 * (size_t)(b_start - cn), (uint32_t)cn * 48u, &S.bar[buf ^ 1]);
        }
        mbar_wait(&S.bar[buf], (phases >> buf) & 1u);
        phases ^= 1u << buf;
        const float4 *r = S.rec[buf];
        int nsel = 0;
        if ((uint32_t)b_start < wlast) {
            int n8 = 0;
            {
                const float wx0 = (float)(tx * TILE + (warp & 1) * 8), wy0 = (float)(ty * TILE + (warp >> 1) * 8);
                const unsigned lt32 = (1u << lane) - 1u;
                for (int k = 0; k < cnt; k += 32) {
                    const int jj = k + lane;
                    const int idx = cnt - 1 - jj;
                    const bool hit = jj < cnt && (uint32_t)(b_start + idx + 1) <= wlast &&
                                     !block_misses(r[3 * idx], r[3 * idx + 1], r[3 * idx + 2].w, wx0, wy0, 7.f, 7.f);
                    const unsigned b = __ballot_sync(0xffffffffu, hit);
                    if (hit) wl8[warp][n8 + __popc(b & lt32)] = (uint8_t)idx;
                    n8 += __popc(b);
                }
                __syncwarp();
            }
            for (int k = 0; k < n8; k += 8) {
                const int e = k + gl;
                const int idx = e < n8 ? wl8[warp][e] : 0;
                const bool hit = e < n8 && (uint32_t)(b_start + idx + 1) <= glast &&
                                 !block_misses(r[3 * idx], r[3 * idx + 1], r[3 * idx + 2].w, fqx, fqy, 3.f, 3.f);
                const unsigned gb = (__ballot_sync(0xffffffffu, hit) >> (lane & 24)) & 0xffu;
                if (hit) wl[warp][q][nsel + __popc(gb & lt)] = (uint8_t)idx;
                nsel += __popc(gb);
            }
        }
        __syncwarp();
        int nmax = nsel;
#pragma unroll
        for (int o = 16; o > 4; o >>= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
        for (int t = 0; t < nmax; t++) {
            const int j = t < nsel ? wl[warp][q][t] : BATCH;
            bwdq_entry<FEW_TILEQ>(P, r, j, (uint32_t)(b_start + j + 1), fx, fy2, lane, g2dv);
        }
    }
}

// (view, tile) indices ordered by decreasing list length (bucketed by length / 8): launched in
// this order the long tiles start first and the short ones fill the end of the kernel.
__global__ void __launch_bounds__(1024) k_tile_order(const uint2 *__restrict__ ranges, int VT,
                                                     uint32_t *__restrict__ order) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    __shared__ uint32_t hist[256];
    const int tid = threadIdx.x;
    if (tid < 256) hist[tid] = 0;
    __syncthreads();
    for (int t = tid; t < VT; t += blockDim.x) {
        const uint2 r = ranges[t];
        atomicAdd(&hist[255 - min(255u, (r.y - r.x) >> 3)], 1u);
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the 256 bucket counts by one warp
        uint32_t v[8], s = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            v[k] = hist[tid * 8 + k];
            s += v[k];
        }
        uint32_t incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (tid >= o) incl += u;
        }
        uint32_t run = incl - s;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            hist[tid * 8 + k] = run;
            run += v[k];
        }
    }
    __syncthreads();
    for (int t = tid; t < VT; t += blockDim.x) {
        const uint2 r = ranges[t];
        order[atomicAdd(&hist[255 - min(255u, (r.y - r.x) >> 3)], 1u)] = (uint32_t)t;
    }
}

// ---------------------------------------------------------------- A2 + raster schedule, fused
// Bucket binning with V * tiles <= 8192: one CTA scans the per-(view, tile) pair counts into the
// tile starts and the pair total P (A2), and from the same counts builds the raster schedule --
// the chunk tables and first-chunk-first order of the chunked path (levels with few tiles) or the
// longest-list-first tile order -- so neither needs a launch of its own.
constexpr int TSCAN_ITEMS = 8;  // counts per thread (1024 threads: up to 8192 tiles)

__global__ void __launch_bounds__(1024) k_tile_scan(const uint32_t *__restrict__ counts, int VT, int64_t cap,
                                                    uint32_t *__restrict__ tile_start, WsHeader *hdr, int chunked,
                                                    uint32_t *__restrict__ chunk_base, uint32_t *__restrict__ chunk_tile,
                                                    uint32_t *__restrict__ chunk_order, int64_t max_chunks,
                                                    uint32_t *__restrict__ tile_order) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    __shared__ uint32_t s_warp[33];
    __shared__ uint32_t hist[258];
    const int t = threadIdx.x;
    uint32_t c[TSCAN_ITEMS], sum = 0;
#pragma unroll
    for (int k = 0; k < TSCAN_ITEMS; k++) {
        const int i = t * TSCAN_ITEMS + k;
        c[k] = i < VT ? counts[(size_t)i * CNT_STRIDE] : 0u;
        sum += c[k];
    }
    uint32_t P;
    uint32_t run = block_exclusive_scan(sum, s_warp, P);
#pragma unroll
    for (int k = 0; k < TSCAN_ITEMS; k++) {
        const int i = t * TSCAN_ITEMS + k;
        if (i < VT) tile_start[i] = run;
        run += c[k];
    }
    if (t == 0) hdr->P = P;
    const bool ok = (int64_t)P <= cap;  // overflow: nothing is binned, nothing to schedule
    if (t < 256) hist[t] = 0;
    __syncthreads();
    if (chunked) {
        // chunk bases in tile order from the contiguous per-thread items (c[] = list lengths) ...
        uint32_t nsum = 0;
#pragma unroll
        for (int k = 0; k < TSCAN_ITEMS; k++) nsum += ok ? (c[k] + CHUNK - 1) / CHUNK : 0u;
        uint32_t total;
        uint32_t cb = block_exclusive_scan(nsum, s_warp, total);
        if (t == 0) hdr->nchunks = (uint32_t)min((int64_t)total, max_chunks);
#pragma unroll
        for (int k = 0; k < TSCAN_ITEMS; k++) {
            const int i = t * TSCAN_ITEMS + k;
            if (i < VT) chunk_base[i] = cb;
            cb += ok ? (c[k] + CHUNK - 1) / CHUNK : 0u;
        }
        __syncthreads();
        // ... then chunk -> tile and the backward's chunk order, tiles strided over the threads
        auto nch = [&](int i) { return ok ? (counts[(size_t)i * CNT_STRIDE] + CHUNK - 1) / CHUNK : 0u; };
        for (int i = t; i < VT; i += 1024) {
            const uint32_t c = nch(i), base = chunk_base[i];
            for (uint32_t j = 0; j < c; j++)
                if (base + j < max_chunks) chunk_tile[base + j] = (uint32_t)i;
        }
        chunk_order_schedule(nch, VT, chunk_base, chunk_order, max_chunks, s_warp, hist);
    } else {  // longest list first: bucket by length / 8, descending
#pragma unroll
        for (int k = 0; k < TSCAN_ITEMS; k++)
            if (t * TSCAN_ITEMS + k < VT) atomicAdd(&hist[255 - min(255u, c[k] >> 3)], 1u);
        __syncthreads();
        const uint32_t hv = t < 256 ? hist[t] : 0u;
        uint32_t dummy;
        const uint32_t hb = block_exclusive_scan(hv, s_warp, dummy);
        if (t < 256) hist[t] = hb;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < TSCAN_ITEMS; k++) {
            const int i = t * TSCAN_ITEMS + k;
            if (i < VT) tile_order[atomicAdd(&hist[255 - min(255u, c[k] >> 3)], 1u)] = (uint32_t)i;
        }
    }
}

bool fused_tile_schedule(const Layout &L) { return (int64_t)L.V * L.tiles <= 1024 * TSCAN_ITEMS; }

cudaError_t launch_tile_scan(const Layout &L, void *ws, cudaStream_t s) {
    ProfScope prof("k_tile_scan", s);
    launch_pdl(k_tile_scan, 1, 1024, 0, s, at<uint32_t>(ws, L.tile_count), L.V * L.tiles, L.cap,
               at<uint32_t>(ws, L.tile_start), at<WsHeader>(ws, L.hdr), L.max_chunks > 0 ? 1 : 0,
               at<uint32_t>(ws, L.chunk_base), at<uint32_t>(ws, L.chunk_tile), at<uint32_t>(ws, L.chunk_order),
               L.max_chunks, at<uint32_t>(ws, L.tile_order));
    return cudaGetLastError();
}

// Warps per CTA: 8 (one CTA per tile) when the grid fills the GPU, else one (eight CTAs per
// tile) at pyramid levels with few tiles so that every SM gets work.  Measured (round 2):
// one-warp instead of two-warp CTAs for 148..295 lists (Replica level 2), 1.587 -> 1.582 ms.
static int raster_warps(const Layout &L) {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    const int64_t t = (int64_t)L.V * L.tiles;
    return t >= 2 * sms ? 8 : 1;
}

cudaError_t launch_gather_pairs(const Layout &L, void *ws, cudaStream_t s) {
    if (L.cap == 0) return cudaGetLastError();
    const int blocks = (int)std::min<int64_t>((L.cap + 255) / 256, 148 * 16);
    k_gather_pairs<<<blocks, 256, 0, s>>>(at<uint32_t>(ws, L.vals0), at<uint64_t>(ws, L.keys0), at<float4>(ws, L.rec0),
                                          at<float4>(ws, L.rec1), at<float4>(ws, L.rec2), L.n, L.tiles,
                                          &at<WsHeader>(ws, L.hdr)->P, L.cap, at<float4>(ws, L.prec));
    return cudaGetLastError();
}

static int g_render_stats = 0;
void set_render_stats(int on) { g_render_stats = on; }
int render_stats() { return g_render_stats; }

template <int WARPS>
static void fwd_launch(const Layout &L, void *ws, const float bg[3], float *out_rgb, float *out_T,
                       const uint32_t *cbase, float4 *cbwd, const uint32_t *order, cudaStream_t s) {
    dim3 grid(L.TX * (8 / WARPS), L.TY, L.V);
    auto kern = render_stats() ? (cbwd ? k_raster_fwd<WARPS, true, true> : k_raster_fwd<WARPS, false, true>)
                               : (cbwd ? k_raster_fwd<WARPS, true, false> : k_raster_fwd<WARPS, false, false>);
    launch_pdl(kern, grid, WARPS * 32, 0, s, at<uint2>(ws, L.ranges), at<float4>(ws, L.prec), L.W, L.H, L.TX, L.tiles, bg[0],
                                     bg[1], bg[2], out_rgb, out_T, at<float>(ws, L.Tfinal),
                                     at<uint32_t>(ws, L.ncontrib), at<uint32_t>(ws, L.ncomp), cbase, cbwd, order);
}


cudaError_t launch_raster_fwd(const Layout &L, void *ws, const float bg[3], float *out_rgb, float *out_T,
                              cudaStream_t s, bool scheduled) {
    ProfScope prof("k_raster_fwd", s);
    uint32_t *cbase = nullptr;
    float4 *cbwd = nullptr;
    if (L.max_chunks > 0) {  // few tiles: record per-chunk state for the chunk-parallel backward
        if (!scheduled)
            launch_pdl(k_chunk_index, 1, 1024, 0, s, at<uint2>(ws, L.ranges), L.V * L.tiles,
                   at<uint32_t>(ws, L.chunk_base), at<uint32_t>(ws, L.chunk_tile), at<uint32_t>(ws, L.chunk_order),
                   at<WsHeader>(ws, L.hdr), L.max_chunks);
        cbase = at<uint32_t>(ws, L.chunk_base);
        cbwd = at<float4>(ws, L.chunk_bwd);
    }
    // many tiles: longest tile lists first, for this forward and the backward (the chunked levels
    // order their backward chunks in k_chunk_index instead)
    const uint32_t *order = nullptr;
    if (L.max_chunks == 0) {
        if (!scheduled)
            launch_pdl(k_tile_order, 1, 1024, 0, s, at<uint2>(ws, L.ranges), L.V * L.tiles,
                       at<uint32_t>(ws, L.tile_order));
        order = at<uint32_t>(ws, L.tile_order);
    }
    switch (raster_warps(L)) {
        case 8: fwd_launch<8>(L, ws, bg, out_rgb, out_T, cbase, cbwd, order, s); break;
        default: fwd_launch<1>(L, ws, bg, out_rgb, out_T, cbase, cbwd, order, s); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_raster_bwd(const Layout &L, void *ws, const float bg[3], const float *dL_drgb, cudaStream_t s) {
    ProfScope prof("k_raster_bwd", s);
    if (L.max_chunks > 0) {  // chunked path (few tiles): every chunk replayed independently
        launch_pdl(k_raster_bwdq_chunk, (unsigned)L.max_chunks, 128, 0, s, 
            at<uint2>(ws, L.ranges), at<float4>(ws, L.prec), at<uint32_t>(ws, L.chunk_base),
            at<uint32_t>(ws, L.chunk_tile), at<WsHeader>(ws, L.hdr), L.n, L.W, L.H, L.TX, L.tiles, dL_drgb,
            at<uint32_t>(ws, L.ncontrib), at<float4>(ws, L.chunk_bwd), at<float4>(ws, L.grad2d),
            at<uint32_t>(ws, L.chunk_order));
        return cudaGetLastError();
    }
    // many tiles: two pixels per lane, packed fp32x2
    dim3 grid(L.TX, L.TY, L.V);
    launch_pdl(k_raster_bwdq, grid, 128, 0, s, at<uint2>(ws, L.ranges), at<float4>(ws, L.prec), L.n, L.W, L.H, L.TX,
                                       L.tiles, bg[0], bg[1], bg[2], dL_drgb, at<float>(ws, L.Tfinal),
                                       at<uint32_t>(ws, L.ncontrib), at<float4>(ws, L.grad2d), at<uint32_t>(ws, L.tile_order));
    return cudaGetLastError();
}

}  // namespace gsk
