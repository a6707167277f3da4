// gs_internal.cuh -- shared declarations of the libgs.so kernels (CUDA path only; the CPU
// oracle in oracle/ shares nothing with this tree).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gs.h"

namespace gsk {

constexpr int TILE = GS_TILE;               // 16x16 pixel tiles
constexpr int BLOCK_PIX = TILE * TILE;      // one thread per pixel in the raster kernels

// radix sort: 8-bit digits, one decoupled-look-back ("onesweep") pass per digit
constexpr int SORT_BITS = 8;
constexpr int SORT_RADIX = 1 << SORT_BITS;
constexpr int SORT_THREADS = 256;
constexpr int SORT_ITEMS = 16;
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;  // 4096 pairs per CTA
constexpr int SORT_MAX_PASSES = 8;

// bucket binning: per-(view, tile) counters are padded to 256 B (one L2 slice each) and
// aggregated in shared memory when the table fits
constexpr int CNT_STRIDE = 64;         // u32 words between two counters
constexpr int SMEM_BINS = 6144;         // max V*tiles aggregated in shared memory

// decoupled-look-back exclusive scan of tiles_touched
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

struct CamBatch {
    gs_camera c[GS_MAX_VIEWS];
};

// Device-side header at the start of every workspace.
struct WsHeader {
    uint32_t flags;        // bit 0: pair capacity overflow
    uint32_t P;            // total pairs of the last preprocess (may exceed capacity)
    uint32_t scan_ctr;     // dynamic CTA index of the scan
    uint32_t vis_count;    // Gaussians visible in at least one view (compacted list length)
    uint32_t n_big;        // tiles whose list is too long for the one-warp sort (bin.cu)
    uint32_t hist_ctr;     // last-CTA detection of the sort histogram
    uint32_t sort_ctr[SORT_MAX_PASSES];
    int32_t sort_sel[SORT_MAX_PASSES + 1];  // source buffer of each pass (0 = primary)
    uint32_t sort_hist[SORT_MAX_PASSES][SORT_RADIX];
    uint32_t sort_start[SORT_MAX_PASSES][SORT_RADIX];
    uint32_t nchunks;      // list chunks of the chunked raster path (raster.cu)
};

// Chunk-parallel raster backward for levels with few tiles or long lists: every CHUNK-entry
// chunk of a tile list is replayed by its own CTA from state the forward recorded (raster.cu).
constexpr int CHUNK = 128;             // list entries per chunk of the chunked raster path
constexpr int TILE_PIX = 256;          // pixels per 16x16 tile (per-chunk record stride)
// Chunk-parallel raster (raster.cu) below CHUNK_MAX_TILES (view, tile) lists -- the coarse GP
// levels, where few tiles with long lists would leave the tile-serial kernels with a long tail --
// and, up to CHUNK_LONG_MAX_TILES lists (the one-CTA tile scan builds the chunk tables), for
// levels whose pair capacity allows CHUNK_LONG_MEAN pairs per list (the multi-view coarse levels).
// Measured (graph replay, round 2): 600 -> 1000 takes Replica level 1 (836 lists) onto it,
// 1.787 -> 1.728 ms per step; chunking Replica level 0 (3225 lists, 212 pairs on average) is
// slower (1.837 vs 1.764 ms): there the tile kernels fill the GPU and the chunk records cost more
// than the tail.  With the quadrant-group backward, 128-entry chunks (64 before) and the
// long-list rule (EuRoC level 2: 1536 lists of 1813 pairs on average): Replica 1.617 -> 1.588 ms,
// EuRoC 6.65 -> 6.33 ms; 512 pairs per list (EuRoC level 1 too) 6.46 ms, 2048 as 1024.
constexpr int CHUNK_MAX_TILES = 1000;
constexpr int64_t CHUNK_LONG_MAX_TILES = 8192;
constexpr int64_t CHUNK_LONG_MEAN = 1024;
__host__ __device__ inline bool use_chunked(int64_t view_tiles, int64_t cap) {
    return view_tiles < CHUNK_MAX_TILES || (view_tiles <= CHUNK_LONG_MAX_TILES && cap >= CHUNK_LONG_MEAN * view_tiles);
}

// Byte offsets of every buffer inside a render workspace (pure function of n, V, W, H, cap).
struct Layout {
    int64_t n, M, cap;  // M = V * n
    int V, W, H, TX, TY, tiles;
    int64_t scan_blocks, sort_blocks;
    size_t hdr, rec0, rec1, rec2, depth, radius, rect, tiles_touched, offsets, grad2d, scan_flags, vis_list;
    size_t slot, scratch;  // per-Gaussian list index (~0u = invisible); per-list-entry gradients [59][n]
    size_t tile_count, tile_start, tile_cursor, bin_big, big_tiles;  // bucket binning (bin.cu)
    size_t tile_mask;   // per (view, Gaussian): rect tiles the ellipse reaches (rects <= 64 tiles)
    size_t tile_order;  // (view, tile) indices, longest list first (raster.cu)
    size_t prec;  // per-pair 48-byte records in sorted order (raster.cu)
    int64_t max_chunks;  // chunked raster path (0 if unused)
    size_t chunk_base, chunk_tile, chunk_bwd, chunk_order;
    size_t keys0, keys1, vals0, vals1, sort_look, ranges, ncontrib, ncomp, Tfinal, total;
};

Layout make_layout(int64_t n, int V, int W, int H, int64_t cap);
// largest layout (capacity) fitting in ws_bytes; returns false if even cap = 0 does not fit
bool layout_for_bytes(int64_t n, int V, int W, int H, size_t ws_bytes, Layout *out);

// ---- Programmatic dependent launch (PDL): kernels of the per-iteration chain are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's CTAs are scheduled while its
// predecessor drains.  Every such kernel calls pdl_wait() before touching global memory (it
// returns once the predecessor grid has completed and its writes are visible -- so completion
// stays transitive along the chain) and pdl_trigger() to let its own successor be scheduled.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();  // api.cu: on unless the environment sets GS_PDL=0 (A/B measurements)

// Eager launches only: measured on B200, PDL shortens the eager mapping step by ~7 % but slows
// the replay of a captured CUDA graph (whose launches are already pipelined) by ~2 %, so launches
// recorded into a graph stay plain.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap);
    if (!pdl_enabled() || cap != cudaStreamCaptureStatusNone) {
        kernel<<<grid, block, smem, s>>>(static_cast<KArgs>(args)...);
        return cudaGetLastError();
    }
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

template <typename T>
__host__ __device__ inline T *at(void *ws, size_t off) {
    return reinterpret_cast<T *>(reinterpret_cast<char *>(ws) + off);
}

// Exact ellipse-tile test (R10'): can the 3-sigma ellipse d^T Q d <= 9 reach a pixel
// centre of tile (tx, ty)?  Box minimum of the quadratic form over the tile's pixel centres (mean
// inside -> 0, else the four clamped edge minima) against 9.01; fp32 IEEE operations in the same
// fixed order as the oracle, so both sides bin exactly the same pairs.
// rA = 1/A, rC = 1/C (IEEE, computed once per Gaussian by the caller: ellipse_recips)
__device__ __forceinline__ void ellipse_recips(float A, float C, float &rA, float &rC) {
    rA = __fdiv_rn(1.0f, A);
    rC = __fdiv_rn(1.0f, C);
}
__device__ __forceinline__ bool tile_hits_ellipse(float u, float v, float A, float B, float C, float rA, float rC,
                                                  int tx, int ty) {
    const float ax = __fsub_rn((float)(tx * TILE), u), bx = __fsub_rn((float)(tx * TILE + TILE - 1), u);
    const float ay = __fsub_rn((float)(ty * TILE), v), by = __fsub_rn((float)(ty * TILE + TILE - 1), v);
    if (ax <= 0.f && bx >= 0.f && ay <= 0.f && by >= 0.f) return true;
    const float B2 = __fmul_rn(2.f, B);
    float best = __int_as_float(0x7f800000);
#pragma unroll
    for (int e = 0; e < 2; e++) {
        const float X = e ? bx : ax;
        const float y = fminf(fmaxf(__fmul_rn(-__fmul_rn(B, X), rC), ay), by);
        best = fminf(best, __fmaf_rn(__fmul_rn(C, y), y, __fmaf_rn(__fmul_rn(B2, X), y, __fmul_rn(__fmul_rn(A, X), X))));
        const float Y = e ? by : ay;
        const float x = fminf(fmaxf(__fmul_rn(-__fmul_rn(B, Y), rA), ax), bx);
        best = fminf(best, __fmaf_rn(__fmul_rn(C, Y), Y, __fmaf_rn(__fmul_rn(B2, x), Y, __fmul_rn(__fmul_rn(A, x), x))));
    }
    return best <= 9.01f;
}

// Visit the binned tiles of rect r (row-major order), f(tx, ty): from the hit mask for rects of
// <= 64 tiles, else by re-running the ellipse test (the bucket binning hands those rects to
// warp_big_rects instead; the radix path's k_duplicate still walks them here).
template <typename F>
__device__ __forceinline__ void for_each_binned_tile(const int4 r, uint64_t mask, const float4 *__restrict__ rec0,
                                                     const float4 *__restrict__ rec1, int64_t m, F f) {
    const int rw = r.z - r.x;
    if (rw * (r.w - r.y) <= 64) {
        const uint64_t row_bits = rw >= 64 ? ~0ull : (1ull << rw) - 1;
        for (int ty = r.y; mask; ty++, mask >>= rw) {  // row by row: no division
            uint64_t m = mask & row_bits;
            while (m) {
                const int bit = __ffsll((long long)m) - 1;
                m &= m - 1;
                f(r.x + bit, ty);
            }
            if (rw >= 64) break;
        }
    } else {  // large rect (rare): the test again, from the records
        const float4 g = rec0[m];
        const float C = rec1[m].x;
        float rA, rC;
        ellipse_recips(g.z, C, rA, rC);
        for (int ty = r.y; ty < r.w; ty++)
            for (int tx = r.x; tx < r.z; tx++)
                if (tile_hits_ellipse(g.x, g.y, g.z, g.w, C, rA, rC, tx, ty)) f(tx, ty);
    }
}

// Rects of more than 64 tiles (no hit mask; a few large footprints near the camera, up to
// ~1000 tiles) are binned by the whole warp instead of their own thread, which would otherwise
// walk them serially and hold its CTA (and the kernel's tail) for the entire rect.  For every
// lane with `big` set, in lane order, the 32 lanes test tiles k = lane, lane + 32, ... of its
// rect (row-major index k) with the same exact test and call f(owner's payload, tx, ty) per hit;
// done(owner_lane, hits) is then called on every lane with the rect's total hit count.
// All 32 lanes must call it (converged).  Visit order differs from the row-major one: callers
// only count or fill buckets whose order the tile sorts fix.
template <typename F, typename G>
__device__ __forceinline__ void warp_big_rects(bool big, int4 r, float u, float v, float A, float B, float C,
                                               uint64_t payload, F f, G done) {
    unsigned bm = __ballot_sync(0xffffffffu, big);
    const int lane = threadIdx.x & 31;
    while (bm) {
        const int src = __ffs(bm) - 1;
        bm &= bm - 1;
        const int x0 = __shfl_sync(0xffffffffu, r.x, src), y0 = __shfl_sync(0xffffffffu, r.y, src);
        const int rw = __shfl_sync(0xffffffffu, r.z, src) - x0;
        const int area = rw * (__shfl_sync(0xffffffffu, r.w, src) - y0);
        const float uu = __shfl_sync(0xffffffffu, u, src), vv = __shfl_sync(0xffffffffu, v, src);
        const float AA = __shfl_sync(0xffffffffu, A, src), BB = __shfl_sync(0xffffffffu, B, src);
        const float CC = __shfl_sync(0xffffffffu, C, src);
        const uint64_t pl = __shfl_sync(0xffffffffu, payload, src);
        float rA, rC;
        ellipse_recips(AA, CC, rA, rC);
        uint32_t hits = 0;
        for (int k = lane; k < area; k += 32) {
            const int ty = y0 + k / rw, tx = x0 + k % rw;
            if (tile_hits_ellipse(uu, vv, AA, BB, CC, rA, rC, tx, ty)) {
                hits++;
                f(pl, tx, ty);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, o);
        done(src, hits);
    }
}

// Largest d^T Q d at which a Gaussian can still be composited: the 3-sigma cutoff (R9) or the
// alpha >= 1/255 skip, alpha <= sigma e^(-q/2) (R7), whichever is tighter (-1: never composited).
__device__ __forceinline__ float q_limit(float sigma) {
    if (sigma * 255.0f < 1.0f) return -1.0f;
    return fminf(9.0f, 2.0f * __logf(255.0f * sigma));
}

// 48-byte per-pair record consumed by the raster kernels (raster.cu), the conic pre-scaled for
// the power (exact: pixel_power): (u, v, -A/2, -B) | (-C/2, sigma, r, g) | (b, Gaussian id
// bits, 0, q_limit(sigma))
__device__ __forceinline__ void write_pair_record(float4 *__restrict__ prec, int64_t pos,
                                                  const float4 *__restrict__ rec0, const float4 *__restrict__ rec1,
                                                  const float4 *__restrict__ rec2, int64_t m, uint32_t gi) {
    const float4 r0 = rec0[m], r1 = rec1[m];
    prec[3 * pos] = make_float4(r0.x, r0.y, -0.5f * r0.z, -r0.w);
    prec[3 * pos + 1] = make_float4(-0.5f * r1.x, r1.y, r1.z, r1.w);
    prec[3 * pos + 2] = make_float4(rec2[m].x, __uint_as_float(gi), 0.f, q_limit(r1.y));
}

int sort_passes(int key_bits);

// Live per-kernel timing for the benchmark (gs_profile_kernel / gs_profile_read): events are
// recorded on the launching stream around the launches of one named kernel only.
void prof_mark(const char *kernel, cudaStream_t s, bool begin);
struct ProfScope {
    const char *k;
    cudaStream_t s;
    ProfScope(const char *kernel, cudaStream_t st) : k(kernel), s(st) { prof_mark(k, s, true); }
    ~ProfScope() { prof_mark(k, s, false); }
};
int hi_bits_for(int64_t count);

// ---- launchers (each returns cudaGetLastError()) ----
cudaError_t launch_preprocess(const gs_params &p, const CamBatch &cams, int V, const Layout &L, void *ws,
                              bool count_tiles, cudaStream_t s);
// exclusive scan of `count` u32 (decoupled look-back); writes the total to hdr->P
// ---- A11 arithmetic shared by the Adam kernels (pyramid_adam.cu) and the fused reduce + Adam +
// broadcast over peer memory (comm.cu): one definition, so both give the same bits.
struct AdamArgs {
    float lr[6];      // per class; in Adam mode already divided by (1 - beta1^t)
    float b1, b2, eps;
    float rs_bc2;     // 1 / sqrt(1 - beta2^t)
    int sgd, zero;
    const int64_t *step_dev;  // non-null: t read on the device; lr[] hold the raw rates
};

// device-step mode: bias corrections from t = *step_dev, once per CTA
__device__ __forceinline__ void adam_device_step(AdamArgs &a) {
    if (!a.step_dev || a.sgd) return;
    __shared__ float s_lr[6], s_rs;
    if (threadIdx.x == 0) {
        const double t = (double)*a.step_dev;
        const double bc1 = 1.0 - pow((double)a.b1, t), bc2 = 1.0 - pow((double)a.b2, t);
        for (int k = 0; k < 6; k++) s_lr[k] = (float)((double)a.lr[k] / bc1);
        s_rs = (float)(1.0 / sqrt(bc2));
    }
    __syncthreads();
    for (int k = 0; k < 6; k++) a.lr[k] = s_lr[k];
    a.rs_bc2 = s_rs;
}

__device__ __forceinline__ int row_class(int row) {
    return row < 3 ? 0 : row < 7 ? 1 : row < 10 ? 2 : row == 10 ? 3 : row < 14 ? 4 : 5;
}

// p -= lr m_hat / (sqrt(v_hat) + eps) with m_hat = m / bc1, v_hat = v / bc2, rewritten as
// p -= (lr / bc1) m / (sqrt(v) / sqrt(bc2) + eps); sqrt and the division use the SFU
// approximations (rel. error ~1e-7, inside the 1e-6 parity contract), which keeps the kernel
// at the HBM roofline instead of the IEEE div/sqrt instruction sequences.
__device__ __forceinline__ void adam1(float &p, float &g, float &m, float &v, float lr, const AdamArgs &a) {
    if (a.sgd) {
        p = p - lr * g;
    } else {
        m = a.b1 * m + (1.f - a.b1) * g;
        v = a.b2 * v + (1.f - a.b2) * g * g;
        float sq = v > 0.f ? v * rsqrtf(v) : 0.f;
        p = p - __fdividef(lr * m, sq * a.rs_bc2 + a.eps);
    }
    if (a.zero) g = 0.f;
}

AdamArgs adam_args(const gs_adam_hparams &hp, int64_t step, int zero, const int64_t *step_dev = nullptr);

// fused A10 + A11 over peer memory (comm.cu)
void comm_shard(int64_t total, int rank, int world, int64_t *e0, int64_t *e1);
cudaError_t launch_peer_barrier(uint32_t *const *flags, int rank, int world, uint32_t *epoch_dev, int64_t *step_dev,
                                cudaStream_t s);
cudaError_t launch_reduce_adam_bcast(const gs_params &p, float *const *param_peers, float *const *grad_peers,
                                     float *p_mc, float *g_mc, float *m, float *v, const gs_adam_hparams &hp,
                                     int64_t step, const int64_t *step_dev, int rank, int world, cudaStream_t s);

cudaError_t launch_scan_u32(const uint32_t *in, uint32_t *out, int64_t count, uint64_t *flags, WsHeader *hdr,
                            cudaStream_t s, int in_stride = 1);
// binning mode: 0 = tile buckets + in-tile sort (bin.cu), 1 = global onesweep LSD radix sort
int binning_mode();
cudaError_t launch_bin(const Layout &L, void *ws, cudaStream_t s);
cudaError_t launch_duplicate(const Layout &L, void *ws, cudaStream_t s);
// generic pair sort on the primary buffers of a workspace (or debug buffers)
size_t spatial_order_temp_bytes(int64_t n);  // order.cu
cudaError_t launch_spatial_order(const float *P, int64_t ld, int64_t n, uint32_t *perm, void *temp, cudaStream_t s);
cudaError_t launch_permute_columns(const float *src, float *dst, int64_t ld, int rows, int64_t n,
                                   const uint32_t *perm, cudaStream_t s);
cudaError_t launch_sort(uint64_t *k0, uint32_t *v0, uint64_t *k1, uint32_t *v1, const uint32_t *count,
                        int64_t cap, int key_bits, WsHeader *hdr, uint32_t *lookback, int64_t sort_blocks,
                        cudaStream_t s);
cudaError_t launch_ranges(const Layout &L, void *ws, cudaStream_t s);
cudaError_t launch_gather_pairs(const Layout &L, void *ws, cudaStream_t s);
// scheduled: the tile scan (launch_tile_scan) already built the chunk tables / tile order
cudaError_t launch_raster_fwd(const Layout &L, void *ws, const float bg[3], float *out_rgb, float *out_T,
                              cudaStream_t s, bool scheduled = false);
// A2 for the bucket binning fused with the raster schedule (one CTA; V * tiles <= 8192)
bool fused_tile_schedule(const Layout &L);
// diagnostic per-pixel composited counts in the forward (off on the hot path)
void set_render_stats(int on);
int render_stats();
cudaError_t launch_tile_scan(const Layout &L, void *ws, cudaStream_t s);
cudaError_t launch_raster_bwd(const Layout &L, void *ws, const float bg[3], const float *dL_drgb, cudaStream_t s);
// A9 into the compacted scratch (one row per parameter, one column per visible Gaussian)
cudaError_t launch_preprocess_bwd(const gs_params &p, const CamBatch &cams, int V, const Layout &L, void *ws,
                                  float *grad2d_norm, cudaStream_t s, int64_t *step_inc = nullptr);
// grads += scratch gathered back to the parameter layout (dense, coalesced)
cudaError_t launch_grad_accumulate(const gs_params &p, const Layout &L, void *ws, float *grads, cudaStream_t s);
// fused A11: Adam over all Gaussians with the gradient gathered from the scratch (0 if invisible)
cudaError_t launch_adam_fused(const gs_params &p, const Layout &L, void *ws, float *m, float *v,
                              const gs_adam_hparams &hp, int64_t step, const int64_t *step_dev, cudaStream_t s);
// densify and prune (densify.cu)
size_t densify_temp_bytes(int64_t n);
cudaError_t launch_densify_stats(const int32_t *radius, int64_t n, int V, float *vis_count, int32_t *max_radius,
                                 cudaStream_t s);
cudaError_t launch_densify_plan(const gs_params &p, const float *grad_accum, const float *vis_count,
                                const int32_t *max_radius, float grad_thr, float big, float logit_thr,
                                int32_t max_screen, void *temp, cudaStream_t s);
void densify_totals(const void *temp, int64_t n, uint32_t tot[3]);
cudaError_t launch_densify_tags(int64_t n, const void *temp, const uint8_t *tin, uint8_t *tout, cudaStream_t s);
cudaError_t launch_densify_apply(const gs_params &p, const float *m, const float *v, const float *z, const void *temp,
                                 const gs_params &out, float *out_m, float *out_v, cudaStream_t s);
// geometry-based densification (densify.cu)
cudaError_t launch_geometry_densify(const gs_camera &cam, const float *uv, const int32_t *active, const float *kp_depth,
                                    const float *depth_map, const float *image, int nk, int mode, float rho,
                                    const gs_params &out, int32_t *src, int32_t *count, cudaStream_t s);
cudaError_t launch_loss(const float *render, const float *gt, int V, int H, int W, float lambda, float *loss,
                        float *dL, void *ws, cudaStream_t s);
size_t loss_ws_bytes(int V, int H, int W);
cudaError_t launch_pyramid(const float *img, int N, int C, int H, int W, int levels, float *out, cudaStream_t s);
cudaError_t launch_adam(const gs_params &p, float *g, float *m, float *v, const gs_adam_hparams &hp, int64_t step,
                        int64_t g0, int64_t g1, int zero, cudaStream_t s, int row_begin = 0, int row_end = -1,
                        int64_t *step_dev = nullptr);
cudaError_t launch_exp_scale(const float *s, float *out, int64_t n, cudaStream_t st);

}  // namespace gsk
