// api.cu -- the extern "C" boundary of libgs.so (declared and documented in include/gs.h).
// Argument validation, workspace layout, the forward/backward state token and kernel
// sequencing live here; all arithmetic of the path runs in the kernels of this directory.
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <cmath>
#include <cstdlib>

#include "gs_internal.cuh"

namespace gsk {

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

Layout make_layout(int64_t n, int V, int W, int H, int64_t cap) {
    Layout L;
    std::memset(&L, 0, sizeof(L));
    L.n = n;
    L.V = V;
    L.W = W;
    L.H = H;
    L.M = (int64_t)V * n;
    L.TX = (W + TILE - 1) / TILE;
    L.TY = (H + TILE - 1) / TILE;
    L.tiles = L.TX * L.TY;
    L.cap = ((cap + SORT_TILE - 1) / SORT_TILE) * SORT_TILE;
    L.scan_blocks = (std::max<int64_t>(L.M, (int64_t)V * L.tiles) + SCAN_TILE - 1) / SCAN_TILE;
    L.sort_blocks = L.cap / SORT_TILE;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t r = o;
        o += al(bytes);
        return r;
    };
    const size_t M = (size_t)L.M;
    L.hdr = take(sizeof(WsHeader));
    L.rec0 = take(M * sizeof(float4));
    L.rec1 = take(M * sizeof(float4));
    L.rec2 = take(M * sizeof(float4));
    L.depth = take(M * sizeof(float));
    L.radius = take(M * sizeof(int32_t));
    L.rect = take(M * sizeof(int4));
    L.tiles_touched = take(M * sizeof(uint32_t));
    L.tile_mask = take(M * sizeof(uint64_t));
    L.offsets = take(M * sizeof(uint32_t));
    L.grad2d = take(M * 3 * sizeof(float4));
    L.scan_flags = take((size_t)std::max<int64_t>(L.scan_blocks, 1) * sizeof(uint64_t));
    L.vis_list = take((size_t)std::max<int64_t>(n, 1) * sizeof(uint32_t));
    L.slot = take((size_t)std::max<int64_t>(n, 1) * sizeof(uint32_t));
    L.scratch = take((size_t)59 * std::max<int64_t>(n, 1) * sizeof(float));
    L.ranges = take((size_t)V * L.tiles * sizeof(uint2));
    L.ncontrib = take((size_t)V * W * H * sizeof(uint32_t));
    L.ncomp = take((size_t)V * W * H * sizeof(uint32_t));
    L.Tfinal = take((size_t)V * W * H * sizeof(float));
    L.keys0 = take((size_t)L.cap * sizeof(uint64_t));
    L.keys1 = take((size_t)L.cap * sizeof(uint64_t));
    L.vals0 = take((size_t)L.cap * sizeof(uint32_t));
    L.vals1 = take((size_t)L.cap * sizeof(uint32_t));
    L.tile_count = take((size_t)V * L.tiles * CNT_STRIDE * sizeof(uint32_t));
    L.tile_start = take((size_t)V * L.tiles * sizeof(uint32_t));
    L.tile_cursor = take((size_t)V * L.tiles * CNT_STRIDE * sizeof(uint32_t));
    L.bin_big = take((size_t)2 * L.cap * sizeof(uint64_t));
    L.big_tiles = take(((size_t)V * L.tiles + (size_t)L.cap / 4096 + 1) * sizeof(uint2));  // (tile, window) items
    L.tile_order = take((size_t)V * L.tiles * sizeof(uint32_t));
    L.prec = take((size_t)3 * L.cap * sizeof(float4));
    L.max_chunks = use_chunked((int64_t)V * L.tiles, L.cap) ? L.cap / CHUNK + (int64_t)V * L.tiles : 0;
    L.chunk_base = take((size_t)V * L.tiles * sizeof(uint32_t));
    L.chunk_tile = take((size_t)std::max<int64_t>(L.max_chunks, 1) * sizeof(uint32_t));
    L.chunk_order = take((size_t)std::max<int64_t>(L.max_chunks, 1) * sizeof(uint32_t));
    L.chunk_bwd = take((size_t)L.max_chunks * TILE_PIX * sizeof(float4));
    L.sort_look = take((size_t)SORT_MAX_PASSES * std::max<int64_t>(L.sort_blocks, 1) * SORT_RADIX * sizeof(uint32_t));
    L.total = o;
    return L;
}

bool layout_for_bytes(int64_t n, int V, int W, int H, size_t ws_bytes, Layout *out) {
    Layout L0 = make_layout(n, V, W, H, 0);
    if (L0.total > ws_bytes) return false;
    // largest capacity (in SORT_TILE units) whose layout fits: binary search; every pair costs at
    // least 24 bytes, which bounds the search
    int64_t lo = 0, hi = (int64_t)((ws_bytes - L0.total) / ((size_t)SORT_TILE * 24)) + 1;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) / 2;
        if (make_layout(n, V, W, H, mid * SORT_TILE).total <= ws_bytes) lo = mid;
        else hi = mid - 1;
    }
    *out = make_layout(n, V, W, H, lo * SORT_TILE);
    return true;
}

// ---- forward/backward state token (SPEC.md:355-359 StaleRenderState) ----
struct Token {
    const float *data;
    int64_t n, ld;
    int32_t D, V;
    uint64_t cam_hash;
    int stage;  // 1 = preprocessed, 2 = rendered, 3 = parameters stepped in place
    int mode;   // binning mode of the preprocess
};
static std::mutex g_mu;
static std::unordered_map<const void *, Token> g_tokens;

static uint64_t hash_cams(const gs_camera *c, int V) {
    uint64_t h = 1469598103934665603ull;
    const unsigned char *p = reinterpret_cast<const unsigned char *>(c);
    for (size_t k = 0; k < sizeof(gs_camera) * (size_t)V; k++) h = (h ^ p[k]) * 1099511628211ull;
    return h;
}
static int g_binning_mode_decl();
static Token make_token(const gs_params *p, const gs_camera *c, int V, int stage) {
    return Token{p->data, p->n, p->ld, p->sh_degree, V, hash_cams(c, V), stage, g_binning_mode_decl()};
}
static bool same(const Token &a, const Token &b) {
    return a.data == b.data && a.n == b.n && a.ld == b.ld && a.D == b.D && a.V == b.V && a.cam_hash == b.cam_hash;
}

static gs_status check_params(const gs_params *p) {
    if (!p || p->n < 0 || (p->n > 0 && !p->data)) return GS_ERR_INVALID_ARG;
    if (p->sh_degree < 0 || p->sh_degree > 3) return GS_ERR_INVALID_ARG;
    if (p->ld < p->n || p->ld % 4 != 0) return GS_ERR_SHAPE;
    if (p->n >= (int64_t)1 << 31) return GS_ERR_NOT_SUPPORTED;
    return GS_OK;
}

static gs_status check_views(const gs_camera *cams, int V, CamBatch *cb) {
    if (!cams || V <= 0) return GS_ERR_INVALID_ARG;
    if (V > GS_MAX_VIEWS) return GS_ERR_NOT_SUPPORTED;
    for (int v = 0; v < V; v++) {
        if (cams[v].width <= 0 || cams[v].height <= 0) return GS_ERR_INVALID_ARG;
        if (cams[v].width != cams[0].width || cams[v].height != cams[0].height) return GS_ERR_SHAPE;
        cb->c[v] = cams[v];
    }
    return GS_OK;
}

static gs_status cuda_status(cudaError_t e) { return e == cudaSuccess ? GS_OK : GS_ERR_CUDA; }

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("GS_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

static int g_binning_mode = 0;
int binning_mode() { return g_binning_mode; }
static int g_binning_mode_decl() { return g_binning_mode; }
// binning mode recorded by the preprocess of this workspace
static int it_mode(const void *ws) {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_tokens.find(ws);
    return it == g_tokens.end() ? g_binning_mode : it->second.mode;
}

// ---- live kernel timing ----
struct Prof {
    std::mutex mu;
    std::string name;
    bool on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    size_t used = 0;
};
static Prof g_prof;

void prof_mark(const char *kernel, cudaStream_t s, bool begin) {
    if (!g_prof.on) return;
    std::lock_guard<std::mutex> g(g_prof.mu);
    if (!g_prof.on || g_prof.name != kernel) return;
    if (begin) {
        if (g_prof.used == g_prof.ev.size()) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            g_prof.ev.push_back({a, b});
        }
        cudaEventRecord(g_prof.ev[g_prof.used].first, s);
    } else {
        cudaEventRecord(g_prof.ev[g_prof.used].second, s);
        g_prof.used++;
    }
}

}  // namespace gsk

using namespace gsk;

extern "C" {

int32_t gs_param_rows(int32_t sh_degree) { return 11 + 3 * (sh_degree + 1) * (sh_degree + 1); }

int64_t gs_param_ld(int64_t n) { return ((n + 63) / 64) * 64; }

gs_status gs_workspace_size(int64_t n, int32_t n_views, int32_t width, int32_t height, int64_t pair_capacity,
                            size_t *bytes) {
    if (!bytes || n < 0 || n_views <= 0 || width <= 0 || height <= 0 || pair_capacity < 0) return GS_ERR_INVALID_ARG;
    if (n_views > GS_MAX_VIEWS) return GS_ERR_NOT_SUPPORTED;
    if (pair_capacity >= ((int64_t)1 << 30)) return GS_ERR_NOT_SUPPORTED;
    *bytes = make_layout(n, n_views, width, height, pair_capacity).total;
    return GS_OK;
}

gs_status gs_preprocess(const gs_params *params, const gs_camera *cams, int32_t n_views, void *ws, size_t ws_bytes,
                        gs_stream_t stream) {
    gs_status st = check_params(params);
    if (st) return st;
    static thread_local CamBatch cb;
    if ((st = check_views(cams, n_views, &cb))) return st;
    if (!ws) return GS_ERR_INVALID_ARG;
    Layout L;
    if (!layout_for_bytes(params->n, n_views, cams[0].width, cams[0].height, ws_bytes, &L)) return GS_ERR_SHAPE;
    cudaStream_t s = (cudaStream_t)stream;
    WsHeader *hdr = at<WsHeader>(ws, L.hdr);
    cudaMemsetAsync(hdr, 0, offsetof(WsHeader, hist_ctr), s);  // flags, P, scan counter, visible count, n_big
    cudaMemsetAsync(at<char>(ws, L.scan_flags), 0, (size_t)std::max<int64_t>(L.scan_blocks, 1) * 8, s);
    const bool buckets = binning_mode() == 0;
    if (buckets)
        cudaMemsetAsync(at<char>(ws, L.tile_count), 0, (size_t)n_views * L.tiles * CNT_STRIDE * sizeof(uint32_t), s);
    cudaError_t e = launch_preprocess(*params, cb, n_views, L, ws, buckets, s);
    if (e == cudaSuccess) {
        if (buckets && fused_tile_schedule(L))  // tile starts + raster schedule, one CTA
            e = launch_tile_scan(L, ws, s);
        else if (buckets)  // tile ranges straight from the per-tile counts
            e = launch_scan_u32(at<uint32_t>(ws, L.tile_count), at<uint32_t>(ws, L.tile_start),
                                (int64_t)n_views * L.tiles, at<uint64_t>(ws, L.scan_flags), hdr, s, CNT_STRIDE);
        else  // pair offsets of every (view, Gaussian) for key duplication
            e = launch_scan_u32(at<uint32_t>(ws, L.tiles_touched), at<uint32_t>(ws, L.offsets), L.M,
                                at<uint64_t>(ws, L.scan_flags), hdr, s);
    }
    if (e != cudaSuccess) return GS_ERR_CUDA;
    std::lock_guard<std::mutex> g(g_mu);
    g_tokens[ws] = make_token(params, cams, n_views, 1);
    return GS_OK;
}

gs_status gs_render_forward(const gs_params *params, const gs_camera *cams, int32_t n_views, void *ws,
                            size_t ws_bytes, const float bg[3], float *out_rgb, float *out_T, gs_stream_t stream) {
    gs_status st = check_params(params);
    if (st) return st;
    static thread_local CamBatch cb;
    if ((st = check_views(cams, n_views, &cb))) return st;
    if (!ws || !bg || !out_rgb) return GS_ERR_INVALID_ARG;
    Layout L;
    if (!layout_for_bytes(params->n, n_views, cams[0].width, cams[0].height, ws_bytes, &L)) return GS_ERR_SHAPE;
    {
        std::lock_guard<std::mutex> g(g_mu);
        auto it = g_tokens.find(ws);
        if (it == g_tokens.end() || !same(it->second, make_token(params, cams, n_views, 1)))
            return GS_ERR_STALE_STATE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    WsHeader *hdr = at<WsHeader>(ws, L.hdr);
    cudaError_t e;
    if (it_mode(ws) == 0) {
        e = launch_bin(L, ws, s);
    } else {
        int key_bits = 32 + std::max(1, hi_bits_for((int64_t)n_views * L.tiles));
        e = launch_duplicate(L, ws, s);
        if (e == cudaSuccess)
            e = launch_sort(at<uint64_t>(ws, L.keys0), at<uint32_t>(ws, L.vals0), at<uint64_t>(ws, L.keys1),
                            at<uint32_t>(ws, L.vals1), &hdr->P, L.cap, key_bits, hdr,
                            at<uint32_t>(ws, L.sort_look), L.sort_blocks, s);
        if (e == cudaSuccess) e = launch_ranges(L, ws, s);
        if (e == cudaSuccess) e = launch_gather_pairs(L, ws, s);  // bucket sort gathers itself
    }
    if (e == cudaSuccess) e = launch_raster_fwd(L, ws, bg, out_rgb, out_T, s, it_mode(ws) == 0 && fused_tile_schedule(L));
    if (e != cudaSuccess) return GS_ERR_CUDA;
    std::lock_guard<std::mutex> g(g_mu);
    g_tokens[ws] = make_token(params, cams, n_views, 2);
    return GS_OK;
}

gs_status gs_loss_workspace_size(int32_t V, int32_t H, int32_t W, size_t *bytes) {
    if (!bytes || V <= 0 || H <= 0 || W <= 0) return GS_ERR_INVALID_ARG;
    *bytes = loss_ws_bytes(V, H, W);
    return GS_OK;
}

gs_status gs_photometric_loss(const float *render, const float *gt, int32_t V, int32_t H, int32_t W, float lambda,
                              float *loss, float *dL_drender, void *ws, size_t ws_bytes, gs_stream_t stream) {
    if (!render || !gt || !loss || !ws || V <= 0 || H <= 0 || W <= 0) return GS_ERR_INVALID_ARG;
    if (!(lambda >= 0.f && lambda <= 1.f)) return GS_ERR_INVALID_ARG;
    if (ws_bytes < loss_ws_bytes(V, H, W)) return GS_ERR_SHAPE;
    return cuda_status(launch_loss(render, gt, V, H, W, lambda, loss, dL_drender, ws, (cudaStream_t)stream));
}

gs_status gs_render_backward(const gs_params *params, const gs_camera *cams, int32_t n_views, void *ws,
                             size_t ws_bytes, const float bg[3], const float *dL_drgb, float *grads,
                             float *grad2d_norm_accum, gs_stream_t stream) {
    gs_status st = check_params(params);
    if (st) return st;
    static thread_local CamBatch cb;
    if ((st = check_views(cams, n_views, &cb))) return st;
    if (!ws || !bg || !dL_drgb || !grads) return GS_ERR_INVALID_ARG;
    Layout L;
    if (!layout_for_bytes(params->n, n_views, cams[0].width, cams[0].height, ws_bytes, &L)) return GS_ERR_SHAPE;
    {
        std::lock_guard<std::mutex> g(g_mu);
        auto it = g_tokens.find(ws);
        if (it == g_tokens.end() || it->second.stage != 2 || !same(it->second, make_token(params, cams, n_views, 2)))
            return GS_ERR_STALE_STATE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = launch_raster_bwd(L, ws, bg, dL_drgb, s);
    if (e == cudaSuccess) e = launch_preprocess_bwd(*params, cb, n_views, L, ws, grad2d_norm_accum, s);
    if (e == cudaSuccess) e = launch_grad_accumulate(*params, L, ws, grads, s);
    return cuda_status(e);
}

gs_status gs_render_backward_adam(gs_params *params, const gs_camera *cams, int32_t n_views, void *ws,
                                  size_t ws_bytes, const float bg[3], const float *dL_drgb, float *m, float *v,
                                  const gs_adam_hparams *hp, int64_t step, int64_t *step_dev,
                                  float *grad2d_norm_accum, gs_stream_t stream) {
    gs_status st = check_params(params);
    if (st) return st;
    static thread_local CamBatch cb;
    if ((st = check_views(cams, n_views, &cb))) return st;
    if (!ws || !bg || !dL_drgb || !hp || step < 0 || (step == 0 && !step_dev)) return GS_ERR_INVALID_ARG;
    if (!hp->sgd_mode && (!m || !v)) return GS_ERR_INVALID_ARG;
    Layout L;
    if (!layout_for_bytes(params->n, n_views, cams[0].width, cams[0].height, ws_bytes, &L)) return GS_ERR_SHAPE;
    {
        std::lock_guard<std::mutex> g(g_mu);
        auto it = g_tokens.find(ws);
        if (it == g_tokens.end() || it->second.stage != 2 || !same(it->second, make_token(params, cams, n_views, 2)))
            return GS_ERR_STALE_STATE;
        // the parameters change in place: any further backward on this forward state is stale
        it->second.stage = 3;
    }
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = launch_raster_bwd(L, ws, bg, dL_drgb, s);
    if (e == cudaSuccess)
        e = launch_preprocess_bwd(*params, cb, n_views, L, ws, grad2d_norm_accum, s, step == 0 ? step_dev : nullptr);
    if (e == cudaSuccess) e = launch_adam_fused(*params, L, ws, m, v, *hp, step, step == 0 ? step_dev : nullptr, s);
    return cuda_status(e);
}

gs_status gs_pyramid(const float *img, int32_t n_images, int32_t C, int32_t H, int32_t W, int32_t n_levels, float *out,
                     gs_stream_t stream) {
    if (!img || n_images <= 0 || C <= 0 || H <= 0 || W <= 0 || n_levels < 0) return GS_ERR_INVALID_ARG;
    if (n_levels > 0 && (int64_t)std::min(H, W) <= ((int64_t)1 << n_levels)) return GS_ERR_SHAPE;
    if (n_levels == 0) return GS_OK;
    if (!out) return GS_ERR_INVALID_ARG;
    return cuda_status(launch_pyramid(img, n_images, C, H, W, n_levels, out, (cudaStream_t)stream));
}

gs_status gs_adam_step(gs_params *params, float *grads, float *m, float *v, const gs_adam_hparams *hp, int64_t step,
                       int64_t g_begin, int64_t g_end, int32_t zero_grads, gs_stream_t stream) {
    gs_status st = check_params(params);
    if (st) return st;
    if (!grads || !hp || step < 1 || g_begin < 0 || g_end > params->n || g_begin > g_end) return GS_ERR_INVALID_ARG;
    if (!hp->sgd_mode && (!m || !v)) return GS_ERR_INVALID_ARG;
    if (g_begin == g_end) return GS_OK;
    return cuda_status(launch_adam(*params, grads, m, v, *hp, step, g_begin, g_end, zero_grads, (cudaStream_t)stream));
}

gs_status gs_adam_step_rows(gs_params *params, float *grads, float *m_rows, float *v_rows, const gs_adam_hparams *hp,
                            int64_t step, int32_t row_begin, int32_t row_end, int32_t zero_grads,
                            gs_stream_t stream) {
    gs_status st = check_params(params);
    if (st) return st;
    const int32_t K = gs_param_rows(params->sh_degree);
    if (!grads || !hp || step < 1 || row_begin < 0 || row_end > K || row_begin > row_end) return GS_ERR_INVALID_ARG;
    if (!hp->sgd_mode && (!m_rows || !v_rows)) return GS_ERR_INVALID_ARG;
    if (row_begin == row_end || params->n == 0) return GS_OK;
    return cuda_status(launch_adam(*params, grads, m_rows, v_rows, *hp, step, 0, params->n, zero_grads,
                                   (cudaStream_t)stream, row_begin, row_end));
}

gs_status gs_adam_step_rows_dev(gs_params *params, float *grads, float *m_rows, float *v_rows,
                                const gs_adam_hparams *hp, int64_t *step_dev, int32_t row_begin, int32_t row_end,
                                int32_t zero_grads, gs_stream_t stream) {
    gs_status st = check_params(params);
    if (st) return st;
    const int32_t K = gs_param_rows(params->sh_degree);
    if (!grads || !hp || !step_dev || row_begin < 0 || row_end > K || row_begin > row_end) return GS_ERR_INVALID_ARG;
    if (!hp->sgd_mode && (!m_rows || !v_rows)) return GS_ERR_INVALID_ARG;
    if (row_begin == row_end || params->n == 0) return GS_OK;
    return cuda_status(launch_adam(*params, grads, m_rows, v_rows, *hp, 1, 0, params->n, zero_grads,
                                   (cudaStream_t)stream, row_begin, row_end, step_dev));
}

gs_status gs_densify_temp_size(int64_t n, size_t *bytes) {
    if (!bytes || n < 0) return GS_ERR_INVALID_ARG;
    *bytes = densify_temp_bytes(n);
    return GS_OK;
}

gs_status gs_densify_stats(const gs_params *params, const gs_camera *cams, int32_t n_views, const void *ws,
                           size_t ws_bytes, float *vis_count, int32_t *max_radius, gs_stream_t stream) {
    gs_status st = check_params(params);
    if (st) return st;
    static thread_local CamBatch cb;
    if ((st = check_views(cams, n_views, &cb))) return st;
    if (!ws || (params->n > 0 && (!vis_count || !max_radius))) return GS_ERR_INVALID_ARG;
    Layout L;
    if (!layout_for_bytes(params->n, n_views, cams[0].width, cams[0].height, ws_bytes, &L)) return GS_ERR_SHAPE;
    {
        std::lock_guard<std::mutex> g(g_mu);
        auto it = g_tokens.find(ws);
        if (it == g_tokens.end() || it->second.stage < 1 || it->second.stage > 2 ||
            !same(it->second, make_token(params, cams, n_views, 1)))
            return GS_ERR_STALE_STATE;
    }
    return cuda_status(launch_densify_stats(at<int32_t>(const_cast<void *>(ws), L.radius), params->n, n_views,
                                            vis_count, max_radius, (cudaStream_t)stream));
}

gs_status gs_densify_plan(const gs_params *params, const float *grad_accum, const float *vis_count,
                          const int32_t *max_radius, const gs_densify_cfg *cfg, void *temp, size_t temp_bytes,
                          int64_t counts[4], gs_stream_t stream) {
    gs_status st = check_params(params);
    if (st) return st;
    if (!cfg || !counts || !temp || (params->n > 0 && (!grad_accum || !vis_count || !max_radius)))
        return GS_ERR_INVALID_ARG;
    if (!(cfg->opacity_threshold > 0.f && cfg->opacity_threshold < 1.f)) return GS_ERR_INVALID_ARG;
    if (temp_bytes < densify_temp_bytes(params->n)) return GS_ERR_SHAPE;
    cudaStream_t s = (cudaStream_t)stream;
    const float logit_thr =
        (float)std::log((double)cfg->opacity_threshold / (1.0 - (double)cfg->opacity_threshold));
    const float big = cfg->percent_dense * cfg->scene_extent;
    cudaError_t e = launch_densify_plan(*params, grad_accum, vis_count, max_radius, cfg->grad_threshold, big,
                                        logit_thr, cfg->max_screen_px, temp, s);
    if (e != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) return GS_ERR_CUDA;
    uint32_t tot[3] = {0, 0, 0};
    if (params->n > 0) densify_totals(temp, params->n, tot);
    counts[0] = tot[1];
    counts[1] = tot[2];
    counts[2] = params->n - (int64_t)tot[0] - (int64_t)tot[2];
    counts[3] = (int64_t)tot[0] + tot[1] + 2 * (int64_t)tot[2];
    return cuda_status(cudaGetLastError());
}

gs_status gs_densify_apply(const gs_params *params, const float *m, const float *v, const float *z, const void *temp,
                           size_t temp_bytes, gs_params *out, float *out_m, float *out_v, gs_stream_t stream) {
    gs_status st = check_params(params);
    if (st) return st;
    if ((st = check_params(out))) return st;
    if (!temp || (params->n > 0 && !z) || out->sh_degree != params->sh_degree) return GS_ERR_INVALID_ARG;
    if ((m == nullptr) != (out_m == nullptr) || (v == nullptr) != (out_v == nullptr) || (m == nullptr) != (v == nullptr))
        return GS_ERR_INVALID_ARG;
    if (temp_bytes < densify_temp_bytes(params->n)) return GS_ERR_SHAPE;
    return cuda_status(launch_densify_apply(*params, m, v, z, temp, *out, out_m, out_v, (cudaStream_t)stream));
}

gs_status gs_densify_tags(int64_t n, const void *temp, size_t temp_bytes, const uint8_t *tags_in, uint8_t *tags_out,
                          gs_stream_t stream) {
    if (n < 0 || !temp || (n > 0 && (!tags_in || !tags_out))) return GS_ERR_INVALID_ARG;
    if (temp_bytes < densify_temp_bytes(n)) return GS_ERR_SHAPE;
    return cuda_status(launch_densify_tags(n, temp, tags_in, tags_out, (cudaStream_t)stream));
}

gs_status gs_geometry_densify(const gs_camera *cam, const float *uv, const int32_t *active, const float *kp_depth,
                              const float *depth_map, const float *image, int32_t n_keypoints, int32_t mode, float rho,
                              gs_params *out, int32_t *src, int32_t *count, gs_stream_t stream) {
    if (!cam || n_keypoints < 0 || !count || (mode != 0 && mode != 1)) return GS_ERR_INVALID_ARG;
    gs_status st = check_params(out);
    if (st) return st;
    if (cam->width <= 0 || cam->height <= 0 || !(cam->fx > 0.f) || !(cam->fy > 0.f)) return GS_ERR_INVALID_ARG;
    if (n_keypoints > 0 && (!uv || !active || !image || !src || (mode == 1 && !depth_map) ||
                            (mode == 0 && !kp_depth) || !(rho > 0.f)))
        return GS_ERR_INVALID_ARG;
    if (out->n < n_keypoints || out->sh_degree < 0) return GS_ERR_SHAPE;
    return cuda_status(launch_geometry_densify(*cam, uv, active, kp_depth, depth_map, image, n_keypoints, mode, rho,
                                               *out, src, count, (cudaStream_t)stream));
}

gs_status gs_query_status(const void *ws, size_t ws_bytes, gs_stream_t stream, int32_t *flags, int64_t *pairs) {
    if (!ws || !flags || ws_bytes < sizeof(WsHeader)) return GS_ERR_INVALID_ARG;
    WsHeader h;
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return GS_ERR_CUDA;
    if (cudaMemcpy(&h, ws, sizeof(uint32_t) * 2, cudaMemcpyDeviceToHost) != cudaSuccess) return GS_ERR_CUDA;
    *flags = (int32_t)h.flags;
    if (pairs) *pairs = h.P;
    return (h.flags & 1u) ? GS_ERR_CAPACITY : GS_OK;
}

gs_status gs_comm_shard(int64_t n, int32_t sh_degree, int32_t rank, int32_t world, int64_t *e_begin, int64_t *e_end) {
    if (!e_begin || !e_end || n < 0 || sh_degree < 0 || sh_degree > 3 || world < 1 || world > 8 || rank < 0 ||
        rank >= world)
        return GS_ERR_INVALID_ARG;
    comm_shard((int64_t)gs_param_rows(sh_degree) * gs_param_ld(n), rank, world, e_begin, e_end);
    return GS_OK;
}

gs_status gs_peer_barrier(uint32_t *const *flag_peers, int32_t rank, int32_t world, uint32_t *epoch,
                          int64_t *step_dev, gs_stream_t stream) {
    if (!flag_peers || !epoch || world < 1 || world > 8 || rank < 0 || rank >= world) return GS_ERR_INVALID_ARG;
    for (int q = 0; q < world; q++)
        if (!flag_peers[q]) return GS_ERR_INVALID_ARG;
    return cuda_status(launch_peer_barrier(flag_peers, rank, world, epoch, step_dev, (cudaStream_t)stream));
}

gs_status gs_reduce_adam_bcast(const gs_params *params, float *const *param_peers, float *const *grad_peers,
                               float *param_mc, float *grad_mc, float *m_shard, float *v_shard,
                               const gs_adam_hparams *hp, int64_t step, const int64_t *step_dev, int32_t rank,
                               int32_t world, gs_stream_t stream) {
    gs_status st = check_params(params);
    if (st) return st;
    if (!hp || !param_peers || !grad_peers || world < 1 || world > 8 || rank < 0 || rank >= world) return GS_ERR_INVALID_ARG;
    if (!step_dev && step < 1) return GS_ERR_INVALID_ARG;
    if (!hp->sgd_mode && (!m_shard || !v_shard)) return GS_ERR_INVALID_ARG;
    if ((param_mc == nullptr) != (grad_mc == nullptr)) return GS_ERR_INVALID_ARG;
    for (int q = 0; q < world; q++)
        if (!param_peers[q] || !grad_peers[q]) return GS_ERR_INVALID_ARG;
    if (param_peers[rank] != params->data) return GS_ERR_INVALID_ARG;
    if (params->ld % 4) return GS_ERR_SHAPE;
    return cuda_status(launch_reduce_adam_bcast(*params, param_peers, grad_peers, param_mc, grad_mc, m_shard, v_shard,
                                                *hp, step, step_dev, rank, world, (cudaStream_t)stream));
}

gs_status gs_status_async(const void *ws, size_t ws_bytes, int32_t *dst, gs_stream_t stream) {
    if (!ws || !dst || ws_bytes < sizeof(WsHeader)) return GS_ERR_INVALID_ARG;
    // WsHeader starts with {flags, P}: one async 8-byte copy (a memcpy node when captured)
    if (cudaMemcpyAsync(dst, ws, sizeof(uint32_t) * 2, cudaMemcpyDefault, (cudaStream_t)stream) != cudaSuccess)
        return GS_ERR_CUDA;
    return GS_OK;
}

gs_status gs_workspace_release(const void *ws) {
    if (!ws) return GS_ERR_INVALID_ARG;
    g_tokens.erase(ws);
    return GS_OK;
}

const char *gs_status_str(gs_status s) {
    switch (s) {
        case GS_OK: return "ok";
        case GS_ERR_INVALID_ARG: return "invalid argument";
        case GS_ERR_SHAPE: return "shape mismatch / too many levels / workspace too small";
        case GS_ERR_CAPACITY: return "tile-pair capacity exceeded";
        case GS_ERR_STALE_STATE: return "stale render state (backward without matching forward)";
        case GS_ERR_CUDA: return "CUDA error";
        case GS_ERR_NOT_SUPPORTED: return "not supported";
    }
    return "unknown status";
}

gs_status gs_spatial_order_temp_size(int64_t n, size_t *bytes) {
    if (!bytes || n < 0) return GS_ERR_INVALID_ARG;
    if (n >= ((int64_t)1 << 30)) return GS_ERR_NOT_SUPPORTED;
    *bytes = spatial_order_temp_bytes(n);
    return GS_OK;
}

gs_status gs_spatial_order(const gs_params *params, uint32_t *perm, void *temp, size_t temp_bytes,
                           gs_stream_t stream) {
    gs_status st = check_params(params);
    if (st) return st;
    size_t need = 0;
    if ((st = gs_spatial_order_temp_size(params->n, &need))) return st;
    if (!perm || !temp) return GS_ERR_INVALID_ARG;
    if (temp_bytes < need) return GS_ERR_SHAPE;
    if (params->n == 0) return GS_OK;
    return cuda_status(launch_spatial_order(params->data, params->ld, params->n, perm, temp, (cudaStream_t)stream));
}

gs_status gs_permute_columns(const float *src, float *dst, int64_t ld, int32_t rows, int64_t n, const uint32_t *perm,
                             gs_stream_t stream) {
    if (n < 0 || rows < 0 || ld < n) return GS_ERR_INVALID_ARG;
    if (n > 0 && rows > 0 && (!src || !dst || !perm || src == dst)) return GS_ERR_INVALID_ARG;
    return cuda_status(launch_permute_columns(src, dst, ld, rows, n, perm, (cudaStream_t)stream));
}

gs_status gs_sort_temp_size(int64_t n, int32_t key_bits, size_t *bytes) {
    if (!bytes || n < 0 || key_bits <= 0 || key_bits > 64) return GS_ERR_INVALID_ARG;
    if (n >= ((int64_t)1 << 30)) return GS_ERR_NOT_SUPPORTED;
    int64_t blocks = (n + SORT_TILE - 1) / SORT_TILE;
    *bytes = al(sizeof(WsHeader)) + al(sizeof(uint32_t)) +
             al((size_t)SORT_MAX_PASSES * std::max<int64_t>(blocks, 1) * SORT_RADIX * sizeof(uint32_t));
    return GS_OK;
}

gs_status gs_debug_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *keys_alt, uint32_t *vals_alt, int64_t n,
                              int32_t key_bits, void *temp, size_t temp_bytes, gs_stream_t stream) {
    size_t need = 0;
    gs_status st = gs_sort_temp_size(n, key_bits, &need);
    if (st) return st;
    if (!keys || !vals || !keys_alt || !vals_alt || !temp) return GS_ERR_INVALID_ARG;
    if (temp_bytes < need) return GS_ERR_SHAPE;
    if (n == 0) return GS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    int64_t blocks = (n + SORT_TILE - 1) / SORT_TILE;
    WsHeader *hdr = at<WsHeader>(temp, 0);
    uint32_t *count = at<uint32_t>(temp, al(sizeof(WsHeader)));
    uint32_t *look = at<uint32_t>(temp, al(sizeof(WsHeader)) + al(sizeof(uint32_t)));
    uint32_t nn = (uint32_t)n;
    // count lives in device memory like the workspace pair count (captured as a memset node)
    cudaMemsetAsync(count, 0, sizeof(uint32_t), s);
    cudaMemcpyAsync(count, &nn, sizeof(uint32_t), cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);  // &nn is a stack variable
    return cuda_status(launch_sort(keys, vals, keys_alt, vals_alt, count, blocks * SORT_TILE, key_bits, hdr, look,
                                   blocks, s));
}

gs_status gs_debug_workspace_view(void *ws, size_t ws_bytes, int64_t n, int32_t n_views, int32_t width,
                                  int32_t height, gs_ws_view *out) {
    if (!ws || !out || n < 0 || n_views <= 0 || width <= 0 || height <= 0) return GS_ERR_INVALID_ARG;
    Layout L;
    if (!layout_for_bytes(n, n_views, width, height, ws_bytes, &L)) return GS_ERR_SHAPE;
    out->rec0 = at<const float>(ws, L.rec0);
    out->rec1 = at<const float>(ws, L.rec1);
    out->rec2 = at<const float>(ws, L.rec2);
    out->depth = at<const float>(ws, L.depth);
    out->radius = at<const int32_t>(ws, L.radius);
    out->rect = at<const int32_t>(ws, L.rect);
    out->tiles_touched = at<const uint32_t>(ws, L.tiles_touched);
    out->offsets = at<const uint32_t>(ws, L.offsets);
    out->keys = at<const uint64_t>(ws, L.keys0);
    out->vals = at<const uint32_t>(ws, L.vals0);
    out->ranges = at<const uint32_t>(ws, L.ranges);
    out->n_contrib = at<const uint32_t>(ws, L.ncontrib);
    out->n_composited = at<const uint32_t>(ws, L.ncomp);
    out->capacity = L.cap;
    return GS_OK;
}

gs_status gs_set_binning(int32_t mode) {
    if (mode != 0 && mode != 1) return GS_ERR_INVALID_ARG;
    g_binning_mode = mode;
    return GS_OK;
}

gs_status gs_profile_kernel(const char *kernel) {
    std::lock_guard<std::mutex> g(g_prof.mu);
    g_prof.on = kernel != nullptr;
    g_prof.name = kernel ? kernel : "";
    g_prof.used = 0;
    return GS_OK;
}

gs_status gs_profile_read(double *total_ms, int64_t *launches) {
    if (!total_ms || !launches) return GS_ERR_INVALID_ARG;
    std::lock_guard<std::mutex> g(g_prof.mu);
    double t = 0;
    for (size_t k = 0; k < g_prof.used; k++) {
        float ms = 0;
        if (cudaEventSynchronize(g_prof.ev[k].second) != cudaSuccess) return GS_ERR_CUDA;
        if (cudaEventElapsedTime(&ms, g_prof.ev[k].first, g_prof.ev[k].second) != cudaSuccess) return GS_ERR_CUDA;
        t += ms;
    }
    *total_ms = t;
    *launches = (int64_t)g_prof.used;
    g_prof.used = 0;
    return GS_OK;
}

gs_status gs_set_render_stats(int32_t on) {
    set_render_stats(on ? 1 : 0);
    return GS_OK;
}

gs_status gs_debug_exp_scale(const float *s, float *out, int64_t n, gs_stream_t stream) {
    if (!s || !out || n < 0) return GS_ERR_INVALID_ARG;
    return cuda_status(launch_exp_scale(s, out, n, (cudaStream_t)stream));
}

}  // extern "C"
