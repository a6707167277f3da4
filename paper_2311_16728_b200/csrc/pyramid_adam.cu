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

struct AdamArgs {
    float lr[6];
    float b1, b2, eps, bc1, bc2;
    int sgd, zero;
};

__device__ __forceinline__ int row_class(int row) {
    return row < 3 ? 0 : row < 7 ? 1 : row < 10 ? 2 : row == 10 ? 3 : row < 14 ? 4 : 5;
}

__device__ __forceinline__ void adam1(float &p, float &g, float &m, float &v, float lr, const AdamArgs &a) {
    if (a.sgd) {
        p = p - lr * g;
    } else {
        m = a.b1 * m + (1.f - a.b1) * g;
        v = a.b2 * v + (1.f - a.b2) * g * g;
        float mh = m / a.bc1, vh = v / a.bc2;
        p = p - lr * mh / (sqrtf(vh) + a.eps);
    }
    if (a.zero) g = 0.f;
}

__global__ void __launch_bounds__(256) k_adam(float *__restrict__ P, float *__restrict__ G, float *__restrict__ Mm,
                                              float *__restrict__ Vv, int rows, int64_t ld, int64_t g0, int64_t g1,
                                              AdamArgs a) {
    const int64_t per_row = ld / 4;
    const int64_t total = (int64_t)rows * per_row;
    float4 *P4 = reinterpret_cast<float4 *>(P), *G4 = reinterpret_cast<float4 *>(G);
    float4 *M4 = reinterpret_cast<float4 *>(Mm), *V4 = reinterpret_cast<float4 *>(Vv);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        int row = (int)(q / per_row);
        int64_t col = (q - row * per_row) * 4;
        if (col + 3 < g0 || col >= g1) continue;
        float lr = a.lr[row_class(row)];
        float4 p = P4[q], g = G4[q], m = a.sgd ? make_float4(0, 0, 0, 0) : M4[q],
               v = a.sgd ? make_float4(0, 0, 0, 0) : V4[q];
        bool full = col >= g0 && col + 3 < g1;
        if (full) {
            adam1(p.x, g.x, m.x, v.x, lr, a);
            adam1(p.y, g.y, m.y, v.y, lr, a);
            adam1(p.z, g.z, m.z, v.z, lr, a);
            adam1(p.w, g.w, m.w, v.w, lr, a);
        } else {
            float *pp = &p.x, *gg = &g.x, *mm = &m.x, *vv = &v.x;
            for (int k = 0; k < 4; k++)
                if (col + k >= g0 && col + k < g1) adam1(pp[k], gg[k], mm[k], vv[k], lr, a);
        }
        P4[q] = p;
        if (a.zero) G4[q] = g;
        if (!a.sgd) {
            M4[q] = m;
            V4[q] = v;
        }
    }
}

static int g_sms = 0;

cudaError_t launch_adam(const gs_params &p, float *g, float *m, float *v, const gs_adam_hparams &hp, int64_t step,
                        int64_t g0, int64_t g1, int zero, cudaStream_t s) {
    if (g_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_sms <= 0) g_sms = 148;
    }
    AdamArgs a;
    for (int k = 0; k < 6; k++) a.lr[k] = hp.lr[k];
    a.b1 = hp.beta1;
    a.b2 = hp.beta2;
    a.eps = hp.eps;
    a.bc1 = (float)(1.0 - std::pow((double)hp.beta1, (double)step));
    a.bc2 = (float)(1.0 - std::pow((double)hp.beta2, (double)step));
    a.sgd = hp.sgd_mode;
    a.zero = zero;
    int rows = gs_param_rows(p.sh_degree);
    int64_t total = (int64_t)rows * (p.ld / 4);
    int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)g_sms * 8);
    if (blocks > 0) k_adam<<<blocks, 256, 0, s>>>(p.data, g, m, v, rows, p.ld, g0, g1, a);
    return cudaGetLastError();
}

}  // namespace gsk
