// loss.cu -- A7: photometric loss of Eq. 4 and its gradient.
//
// L_v = (1 - lambda) mean|x - y| + lambda (1 - mean SSIM(x, y)) per view, lambda = 0.2
// (PAPER.md:568).  SSIM per channel with an 11x11 Gaussian window (sigma 1.5), C1 = 0.01^2,
// C2 = 0.03^2, zero-padded 'same' (R17).  The window is separable, so each
// 16x16 output tile loads a 26x26 halo of x and y into shared memory and runs a horizontal
// then a vertical 11-tap pass over the five moment maps (x, y, x^2, y^2, xy).  The gradient
// is the windowed-correlation form: dSSIM/dx_p = (w * A)_p + 2 x_p (w * B)_p + y_p (w * C)_p
// with A = dS/dmu_x, B = dS/dE[x^2], C = dS/dE[xy] per pixel, so a second kernel applies
// the same separable window to the three partial maps.  Loss sums are reduced per CTA; the
// first CTA of each view in the gradient kernel (or a one-CTA-per-view kernel when no gradient
// is requested) sums that view's partials in a fixed order (deterministic) and writes the loss.
#include <cmath>

#include "gs_internal.cuh"

namespace gsk {

constexpr int LT = 16;          // output tile
constexpr int HALO = 5;         // 11-tap window radius
constexpr int LS = LT + 2 * HALO;  // 26
constexpr int LSP = 48;         // padded row stride: the two half-warps of a row pass read
                                // disjoint bank halves (48 = 16 mod 32)

struct Win {
    float g[11];
};

static Win make_window() {
    Win w;
    double s = 0, v[11];
    for (int i = 0; i < 11; i++) {
        v[i] = std::exp(-((i - 5) * (i - 5)) / (2.0 * 1.5 * 1.5));
        s += v[i];
    }
    for (int i = 0; i < 11; i++) w.g[i] = (float)(v[i] / s);
    return w;
}

constexpr float SS_C1 = 0.01f * 0.01f;
constexpr float SS_C2 = 0.03f * 0.03f;

// grid: (ceil(W/16), ceil(H/16), V*3); partial maps dA, dB, dC [V][3][H][W];
// block partial sums part[(v*3 + c) * nbt + bt][2] = (sum |x-y|, sum SSIM)
__global__ void __launch_bounds__(LT *LT) k_ssim_fwd(const float *__restrict__ X, const float *__restrict__ Y, int H,
                                                     int W, Win win, float *__restrict__ dA, float *__restrict__ dB,
                                                     float *__restrict__ dC, float2 *__restrict__ part) {
    __shared__ float sx[LS][LSP], sy[LS][LSP];
    __shared__ float h[5][LS][LT];
    __shared__ float red[2][LT * LT / 32];
    const int plane = blockIdx.z;  // v*3 + c
    const int64_t HW = (int64_t)H * W;
    const float *x = X + plane * HW, *y = Y + plane * HW;
    const int x0 = blockIdx.x * LT - HALO, y0 = blockIdx.y * LT - HALO;
    const int tid = threadIdx.x;
    for (int k = tid; k < LS * LS; k += LT * LT) {
        int r = k / LS, c = k % LS;
        int gy = y0 + r, gx = x0 + c;
        bool ok = gy >= 0 && gy < H && gx >= 0 && gx < W;
        sx[r][c] = ok ? x[(int64_t)gy * W + gx] : 0.f;
        sy[r][c] = ok ? y[(int64_t)gy * W + gx] : 0.f;
    }
    __syncthreads();
    // horizontal pass over all LS rows, LT output columns
    for (int k = tid; k < LS * LT; k += LT * LT) {
        int r = k / LT, c = k % LT;
        float a = 0, b = 0, aa = 0, bb = 0, ab = 0;
#pragma unroll
        for (int j = 0; j < 11; j++) {
            float xv = sx[r][c + j], yv = sy[r][c + j], w = win.g[j];
            a += w * xv;
            b += w * yv;
            aa += w * xv * xv;
            bb += w * yv * yv;
            ab += w * xv * yv;
        }
        h[0][r][c] = a; h[1][r][c] = b; h[2][r][c] = aa; h[3][r][c] = bb; h[4][r][c] = ab;
    }
    __syncthreads();
    const int r = tid / LT, c = tid % LT;
    const int gy = blockIdx.y * LT + r, gx = blockIdx.x * LT + c;
    float mx = 0, my = 0, exx = 0, eyy = 0, exy = 0;
#pragma unroll
    for (int i = 0; i < 11; i++) {
        float w = win.g[i];
        mx += w * h[0][r + i][c];
        my += w * h[1][r + i][c];
        exx += w * h[2][r + i][c];
        eyy += w * h[3][r + i][c];
        exy += w * h[4][r + i][c];
    }
    float l1 = 0.f, S = 0.f;
    if (gy < H && gx < W) {
        float sxx = exx - mx * mx, syy = eyy - my * my, sxy = exy - mx * my;
        float a1 = 2.f * mx * my + SS_C1, a2 = 2.f * sxy + SS_C2;
        float b1 = mx * mx + my * my + SS_C1, b2 = sxx + syy + SS_C2;
        float ib = 1.f / (b1 * b2);
        S = a1 * a2 * ib;
        float dS_dmx = 2.f * my * a2 * ib - S * 2.f * mx / b1;
        float dS_dsxx = -S / b2;
        float dS_dsxy = 2.f * a1 * ib;
        int64_t o = plane * HW + (int64_t)gy * W + gx;
        dA[o] = dS_dmx + dS_dsxx * (-2.f * mx) + dS_dsxy * (-my);
        dB[o] = dS_dsxx;
        dC[o] = dS_dsxy;
        l1 = fabsf(sx[r + HALO][c + HALO] - sy[r + HALO][c + HALO]);
    }
    // block reduction (fixed order)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        S += __shfl_xor_sync(0xffffffffu, S, o);
    }
    if ((tid & 31) == 0) {
        red[0][tid >> 5] = l1;
        red[1][tid >> 5] = S;
    }
    __syncthreads();
    if (tid == 0) {
        float a = 0, b = 0;
        for (int k = 0; k < LT * LT / 32; k++) {
            a += red[0][k];
            b += red[1][k];
        }
        int nbt = gridDim.x * gridDim.y;
        part[(int64_t)plane * nbt + blockIdx.y * gridDim.x + blockIdx.x] = make_float2(a, b);
    }
}

// Fixed-order sum of the 3 * nbt partials of view v with one CTA of 256 threads (deterministic).
__device__ __forceinline__ void finalize_view(const float2 *__restrict__ part, int v, int nbt, float lambda,
                                              float invN, float *loss) {
    __shared__ double sa[8], sb[8];
    double a = 0, b = 0;
    for (int k = threadIdx.x; k < 3 * nbt; k += blockDim.x) {
        const float2 p = part[(int64_t)v * 3 * nbt + k];
        a += p.x;
        b += p.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sa[threadIdx.x >> 5] = a;
        sb[threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double ta = 0, tb = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            ta += sa[w];
            tb += sb[w];
        }
        loss[v] = (float)((1.0 - lambda) * ta * invN + lambda * (1.0 - tb * invN));
    }
}

// loss only (no gradient requested): one CTA per view
__global__ void __launch_bounds__(256) k_loss_final(const float2 *__restrict__ part, int nbt, float lambda, float invN,
                                                    float *loss) {
    finalize_view(part, blockIdx.x, nbt, lambda, invN, loss);
}

__global__ void __launch_bounds__(LT *LT) k_ssim_bwd(const float *__restrict__ X, const float *__restrict__ Y, int H,
                                                     int W, Win win, float lambda, float invN,
                                                     const float *__restrict__ dA, const float *__restrict__ dB,
                                                     const float *__restrict__ dC, float *__restrict__ dL,
                                                     const float2 *__restrict__ part, float *__restrict__ loss) {
    __shared__ float s[3][LS][LSP];
    __shared__ float h[3][LS][LT];
    const int plane = blockIdx.z;
    const int64_t HW = (int64_t)H * W;
    const int x0 = blockIdx.x * LT - HALO, y0 = blockIdx.y * LT - HALO;
    const int tid = threadIdx.x;
    for (int k = tid; k < LS * LS; k += LT * LT) {
        int r = k / LS, c = k % LS;
        int gy = y0 + r, gx = x0 + c;
        bool ok = gy >= 0 && gy < H && gx >= 0 && gx < W;
        int64_t o = plane * HW + (int64_t)gy * W + gx;
        s[0][r][c] = ok ? dA[o] : 0.f;
        s[1][r][c] = ok ? dB[o] : 0.f;
        s[2][r][c] = ok ? dC[o] : 0.f;
    }
    __syncthreads();
    for (int k = tid; k < LS * LT; k += LT * LT) {
        int r = k / LT, c = k % LT;
        float a = 0, b = 0, cc = 0;
#pragma unroll
        for (int j = 0; j < 11; j++) {
            float w = win.g[j];
            a += w * s[0][r][c + j];
            b += w * s[1][r][c + j];
            cc += w * s[2][r][c + j];
        }
        h[0][r][c] = a; h[1][r][c] = b; h[2][r][c] = cc;
    }
    __syncthreads();
    const int r = tid / LT, c = tid % LT;
    const int gy = blockIdx.y * LT + r, gx = blockIdx.x * LT + c;
    // the first CTA of each view also reduces that view's loss partials (written by k_ssim_fwd)
    if (blockIdx.x == 0 && blockIdx.y == 0 && plane % 3 == 0)
        finalize_view(part, plane / 3, gridDim.x * gridDim.y, lambda, invN, loss);
    if (gy >= H || gx >= W) return;
    float sa = 0, sb = 0, sc = 0;
#pragma unroll
    for (int i = 0; i < 11; i++) {
        float w = win.g[i];
        sa += w * h[0][r + i][c];
        sb += w * h[1][r + i][c];
        sc += w * h[2][r + i][c];
    }
    int64_t o = plane * HW + (int64_t)gy * W + gx;
    float xv = X[o], yv = Y[o];
    float dssim = sa + 2.f * xv * sb + yv * sc;
    float d = xv - yv;
    float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
    dL[o] = (1.f - lambda) * sgn * invN - lambda * dssim * invN;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t loss_ws_bytes(int V, int H, int W) {
    size_t plane = (size_t)V * 3 * H * W * sizeof(float);
    size_t nbt = (size_t)((W + LT - 1) / LT) * ((H + LT - 1) / LT);
    return 3 * align256(plane) + align256((size_t)V * 3 * nbt * sizeof(float2));
}

cudaError_t launch_loss(const float *render, const float *gt, int V, int H, int W, float lambda, float *loss, float *dL,
                        void *ws, cudaStream_t s) {
    static const Win win = make_window();
    size_t plane = align256((size_t)V * 3 * H * W * sizeof(float));
    float *dA = at<float>(ws, 0), *dB = at<float>(ws, plane), *dC = at<float>(ws, 2 * plane);
    float2 *part = at<float2>(ws, 3 * plane);
    dim3 grid((W + LT - 1) / LT, (H + LT - 1) / LT, V * 3);
    const int nbt = grid.x * grid.y;
    float invN = (float)(1.0 / (3.0 * H * W));
    k_ssim_fwd<<<grid, LT * LT, 0, s>>>(render, gt, H, W, win, dA, dB, dC, part);
    if (dL)
        k_ssim_bwd<<<grid, LT * LT, 0, s>>>(render, gt, H, W, win, lambda, invN, dA, dB, dC, dL, part, loss);
    else
        k_loss_final<<<V, 256, 0, s>>>(part, nbt, lambda, invN, loss);
    return cudaGetLastError();
}

}  // namespace gsk
