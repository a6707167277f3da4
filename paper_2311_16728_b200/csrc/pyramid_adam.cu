// pyramid_adam.cu -- A0 (Gaussian pyramid level) and A11 (fused optimiser step).
//
// A0: "constructed by repeatedly applying Gaussian smoothing and downsampling";
// R18: [1,4,6,4,1]/16 horizontally then vertically, reflect-101 border, keep even rows and
// columns, ceil-halved size.  One thread per output pixel; the 5x5 input neighbourhood is
// read through L1 (the whole image pyramid of a keyframe is a few MB).
//
// A11: PAPER.md:568 (fixed learning rate) with R20: bias-corrected Adam, per-class learning
// rate, dense over all Gaussians of the range.  Streaming kernel over the K x ld parameter
// rows with 16-byte vector loads/stores; the gradient is zeroed in the same pass when asked
// (the next iteration accumulates into it), so p, g, m, v are each touched once.
#include "gs_internal.cuh"

namespace gsk {

__device__ __forceinline__ int refl101(int i, int n) {
    if (n == 1) return 0;
    while (i < 0 || i >= n) {
        if (i < 0) i = -i;
        if (i >= n) i = 2 * (n - 1) - i;
    }
    return i;
}

__global__ void k_pyr_down(const float *__restrict__ in, int planes, int H, int W, float *__restrict__ out) {
    const int Ho = (H + 1) / 2, Wo = (W + 1) / 2;
    int64_t total = (int64_t)planes * Ho * Wo;
    const float k[5] = {1.f / 16, 4.f / 16, 6.f / 16, 4.f / 16, 1.f / 16};
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
        int x = (int)(o % Wo);
        int y = (int)((o / Wo) % Ho);
        int64_t p = o / ((int64_t)Ho * Wo);
        const float *src = in + p * (int64_t)H * W;
        int cx[5];
#pragma unroll
        for (int j = 0; j < 5; j++) cx[j] = refl101(2 * x + j - 2, W);
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const float *row = src + (int64_t)refl101(2 * y + i - 2, H) * W;
            float hsum = 0.f;
#pragma unroll
            for (int j = 0; j < 5; j++) hsum += k[j] * __ldg(row + cx[j]);
            acc += k[i] * hsum;
        }
        out[o] = acc;
    }
}

cudaError_t launch_pyramid(const float *img, int N, int C, int H, int W, int levels, float *out, cudaStream_t s) {
    const float *src = img;
    float *dst = out;
    int h = H, w = W;
    for (int l = 0; l < levels; l++) {
        int ho = (h + 1) / 2, wo = (w + 1) / 2;
        int64_t total = (int64_t)N * C * ho * wo;
        int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
        k_pyr_down<<<std::max(blocks, 1), 256, 0, s>>>(src, N * C, h, w, dst);
        src = dst;
        dst += total;
        h = ho;
        w = wo;
    }
    return cudaGetLastError();
}

constexpr int ADAM_THREADS = 256;
constexpr int ADAM_UNROLL = 2;

// grid (ceil(ld/4 / (256*2)), rows): the parameter class (learning rate) is uniform per CTA row;
// P, G, Mm, Vv point at the first row of the range, row0 is its parameter row (class lookup)
__global__ void __launch_bounds__(ADAM_THREADS) k_adam(float *__restrict__ P, float *__restrict__ G,
                                                       float *__restrict__ Mm, float *__restrict__ Vv, int64_t ld,
                                                       int64_t g0, int64_t g1, int row0, AdamArgs a) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    adam_device_step(a);  // device-step mode only
    const int row = blockIdx.y;
    const float lr = a.lr[row_class(row0 + row)];
    const int64_t per_row = ld / 4;
    const int64_t rbase = (int64_t)row * per_row;
    float4 *P4 = reinterpret_cast<float4 *>(P) + rbase, *G4 = reinterpret_cast<float4 *>(G) + rbase;
    float4 *M4 = reinterpret_cast<float4 *>(Mm) + rbase, *V4 = reinterpret_cast<float4 *>(Vv) + rbase;
    int64_t q[ADAM_UNROLL];
    float4 p[ADAM_UNROLL], g[ADAM_UNROLL], m[ADAM_UNROLL], v[ADAM_UNROLL];
    bool live[ADAM_UNROLL];
#pragma unroll
    for (int u = 0; u < ADAM_UNROLL; u++) {
        q[u] = ((int64_t)blockIdx.x * ADAM_UNROLL + u) * ADAM_THREADS + threadIdx.x;
        int64_t col = q[u] * 4;
        live[u] = q[u] < per_row && col + 3 >= g0 && col < g1;
        if (live[u]) {
            p[u] = P4[q[u]];
            g[u] = G4[q[u]];
            if (!a.sgd) {
                m[u] = M4[q[u]];
                v[u] = V4[q[u]];
            } else {
                m[u] = v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }
#pragma unroll
    for (int u = 0; u < ADAM_UNROLL; u++) {
        if (!live[u]) continue;
        int64_t col = q[u] * 4;
        float *pp = &p[u].x, *gg = &g[u].x, *mm = &m[u].x, *vv = &v[u].x;
        if (col >= g0 && col + 3 < g1) {
#pragma unroll
            for (int k = 0; k < 4; k++) adam1(pp[k], gg[k], mm[k], vv[k], lr, a);
        } else {
            for (int k = 0; k < 4; k++)
                if (col + k >= g0 && col + k < g1) adam1(pp[k], gg[k], mm[k], vv[k], lr, a);
        }
        P4[q[u]] = p[u];
        if (a.zero) G4[q[u]] = g[u];
        if (!a.sgd) {
            M4[q[u]] = m[u];
            V4[q[u]] = v[u];
        }
    }
}

// ---- dense column kernels over the compacted backward scratch ---------------------------
// thread = 4 consecutive Gaussians (one float4 of every row); grid.y splits the rows
constexpr int COL_THREADS = 256;
constexpr int ROW_GROUPS = 8;

__device__ __forceinline__ bool load_slots(const uint32_t *slot, int64_t i0, int64_t n, uint32_t sl[4]) {
    bool any = false;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        sl[k] = i0 + k < n ? slot[i0 + k] : 0xFFFFFFFFu;
        any |= sl[k] != 0xFFFFFFFFu;
    }
    return any;
}

__global__ void __launch_bounds__(COL_THREADS) k_grad_accumulate(float *__restrict__ G, int64_t ld, int64_t n,
                                                                 int rows, const uint32_t *__restrict__ slot,
                                                                 const float *__restrict__ S) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    const int64_t c4 = (int64_t)blockIdx.x * COL_THREADS + threadIdx.x;
    const int64_t i0 = c4 * 4;
    if (i0 >= n) return;
    uint32_t sl[4];
    if (!load_slots(slot, i0, n, sl)) return;
    const int rpg = (rows + gridDim.y - 1) / gridDim.y;
    const int r0 = blockIdx.y * rpg, r1 = min(rows, r0 + rpg);
    for (int row = r0; row < r1; row++) {
        float4 *gp = reinterpret_cast<float4 *>(G + (int64_t)row * ld) + c4;
        float4 g = *gp;
        const float *Sr = S + (int64_t)row * n;
        if (sl[0] != 0xFFFFFFFFu) g.x += Sr[sl[0]];
        if (sl[1] != 0xFFFFFFFFu) g.y += Sr[sl[1]];
        if (sl[2] != 0xFFFFFFFFu) g.z += Sr[sl[2]];
        if (sl[3] != 0xFFFFFFFFu) g.w += Sr[sl[3]];
        *gp = g;
    }
}

__global__ void __launch_bounds__(COL_THREADS) k_adam_fused(float *__restrict__ P, float *__restrict__ Mm,
                                                            float *__restrict__ Vv, int64_t ld, int64_t n, int rows,
                                                            const uint32_t *__restrict__ slot,
                                                            const float *__restrict__ S, AdamArgs a) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    adam_device_step(a);
    const int64_t c4 = (int64_t)blockIdx.x * COL_THREADS + threadIdx.x;
    const int64_t i0 = c4 * 4;
    if (i0 >= n) return;
    uint32_t sl[4];
    load_slots(slot, i0, n, sl);
    const int rpg = (rows + gridDim.y - 1) / gridDim.y;
    const int r0 = blockIdx.y * rpg, r1 = min(rows, r0 + rpg);
#pragma unroll 2
    for (int row = r0; row < r1; row++) {
        const float lr = a.lr[row_class(row)];
        const int64_t q = (int64_t)row * (ld / 4) + c4;
        // m and v are streamed (evict-first loads and stores), so the updated parameters -- read
        // again by the next iteration's projection -- tend to stay in L2
        float4 p = reinterpret_cast<float4 *>(P)[q];
        float4 m = a.sgd ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldcs(reinterpret_cast<float4 *>(Mm) + q);
        float4 v = a.sgd ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldcs(reinterpret_cast<float4 *>(Vv) + q);
        const float *Sr = S + (int64_t)row * n;
        float g[4];
#pragma unroll
        for (int k = 0; k < 4; k++) g[k] = sl[k] != 0xFFFFFFFFu ? __ldcs(Sr + sl[k]) : 0.f;
        float *pp = &p.x, *mm = &m.x, *vv = &v.x;
#pragma unroll
        for (int k = 0; k < 4; k++)
            if (i0 + k < n) adam1(pp[k], g[k], mm[k], vv[k], lr, a);
        reinterpret_cast<float4 *>(P)[q] = p;
        if (!a.sgd) {
            __stcs(reinterpret_cast<float4 *>(Mm) + q, m);
            __stcs(reinterpret_cast<float4 *>(Vv) + q, v);
        }
    }
}

cudaError_t launch_grad_accumulate(const gs_params &p, const Layout &L, void *ws, float *grads, cudaStream_t s) {
    int64_t cols4 = (p.n + 3) / 4;
    if (cols4 == 0) return cudaGetLastError();
    dim3 grid((unsigned)((cols4 + COL_THREADS - 1) / COL_THREADS), ROW_GROUPS);
    launch_pdl(k_grad_accumulate, grid, COL_THREADS, 0, s, grads, p.ld, p.n, gs_param_rows(p.sh_degree),
                                                   at<uint32_t>(ws, L.slot), at<float>(ws, L.scratch));
    return cudaGetLastError();
}

AdamArgs adam_args(const gs_adam_hparams &hp, int64_t step, int zero, const int64_t *step_dev) {
    AdamArgs a;
    a.step_dev = step_dev;
    if (step_dev) step = 1;  // placeholder; the kernel derives the corrections from *step_dev
    double bc1 = 1.0 - std::pow((double)hp.beta1, (double)step);
    double bc2 = 1.0 - std::pow((double)hp.beta2, (double)step);
    for (int k = 0; k < 6; k++) a.lr[k] = (hp.sgd_mode || step_dev) ? hp.lr[k] : (float)((double)hp.lr[k] / bc1);
    a.b1 = hp.beta1;
    a.b2 = hp.beta2;
    a.eps = hp.eps;
    a.rs_bc2 = (float)(1.0 / std::sqrt(bc2));
    a.sgd = hp.sgd_mode;
    a.zero = zero;
    return a;
}

cudaError_t launch_adam_fused(const gs_params &p, const Layout &L, void *ws, float *m, float *v,
                              const gs_adam_hparams &hp, int64_t step, const int64_t *step_dev, cudaStream_t s) {
    AdamArgs a = adam_args(hp, step, 0, step_dev);
    int64_t cols4 = (p.n + 3) / 4;
    if (cols4 == 0) return cudaGetLastError();
    dim3 grid((unsigned)((cols4 + COL_THREADS - 1) / COL_THREADS), ROW_GROUPS);
    ProfScope prof("k_adam_fused", s);
    launch_pdl(k_adam_fused, grid, COL_THREADS, 0, s, p.data, m, v, p.ld, p.n, gs_param_rows(p.sh_degree),
                                              at<uint32_t>(ws, L.slot), at<float>(ws, L.scratch), a);
    return cudaGetLastError();
}

__global__ void k_step_inc(int64_t *step_dev) { *step_dev += 1; }

cudaError_t launch_adam(const gs_params &p, float *g, float *m, float *v, const gs_adam_hparams &hp, int64_t step,
                        int64_t g0, int64_t g1, int zero, cudaStream_t s, int row_begin, int row_end,
                        int64_t *step_dev) {
    if (step_dev) {  // device-step mode: take step *step_dev + 1 and count it (graph replay)
        k_step_inc<<<1, 1, 0, s>>>(step_dev);
        step = 1;
    }
    AdamArgs a = adam_args(hp, step, zero, step_dev);
    if (row_end < 0) row_end = gs_param_rows(p.sh_degree);
    const int rows = row_end - row_begin;
    int64_t per_row = p.ld / 4;
    dim3 grid((unsigned)((per_row + ADAM_THREADS * ADAM_UNROLL - 1) / (ADAM_THREADS * ADAM_UNROLL)), rows);
    ProfScope prof("k_adam", s);
    const int64_t off = (int64_t)row_begin * p.ld;
    if (per_row > 0 && rows > 0) launch_pdl(k_adam, grid, ADAM_THREADS, 0, s, p.data + off, g + off, m, v, p.ld, g0, g1, row_begin, a);
    return cudaGetLastError();
}

}  // namespace gsk
