// loss.cu -- A7: photometric loss of Eq. 4 and its gradient.
//
// L_v = (1 - lambda) mean|x - y| + lambda (1 - mean SSIM(x, y)) per view, lambda = 0.2
// (PAPER.md:568).  SSIM per channel with an 11x11 Gaussian window (sigma 1.5), C1 = 0.01^2,
// C2 = 0.03^2, zero-padded 'same' (R17).  The window is separable, so each
// 32x32 output tile loads a 42x42 halo of x and y into shared memory and runs a horizontal
// then a vertical 11-tap pass over the five moment maps (x, y, x^2, y^2, xy).  The gradient
// is the windowed-correlation form: dSSIM/dx_p = (w * A)_p + 2 x_p (w * B)_p + y_p (w * C)_p
// with A = dS/dmu_x, B = dS/dE[x^2], C = dS/dE[xy] per pixel, so a second kernel applies
// the same separable window to the three partial maps.  Both passes accumulate two maps at a
// time with Blackwell's packed fp32x2 FFMA2 (x and y, x^2 and y^2; A and B).  Loss sums are reduced per CTA; the
// first CTA of each view in the gradient kernel (or a one-CTA-per-view kernel when no gradient
// is requested) sums that view's partials in a fixed order (deterministic) and writes the loss.
#include <cmath>

#include "gs_internal.cuh"

namespace gsk {

constexpr int TW = 32, TH = 32;  // output tile (columns x rows)
constexpr int HALO = 5;           // 11-tap window radius
constexpr int SW = TW + 2 * HALO, SH = TH + 2 * HALO;  // 42 x 42 input patch
constexpr int SWP = SW + 1;       // padded row stride
constexpr int NT = 256;           // threads per CTA
constexpr int HC = 4;             // horizontal pass: consecutive output columns per thread
constexpr int VR = 4;             // vertical pass: consecutive output rows per thread

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

// Load the (TH + 10) x (TW + 10) patches of M maps around the tile into smem (zero outside the
// image).  Warp w takes patch rows w, w + 8, ...; lanes cover the 42 columns in two steps (no
// index division).  All global loads are issued before the first shared store.
template <int M>
__device__ __forceinline__ void load_patches(float (*dst)[SH][SWP], const float *const (&src)[M], int H, int W,
                                             int x0, int y0) {
    constexpr int NW = NT / 32, RPW = (SH + NW - 1) / NW;  // rows per warp
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float v[M][RPW][2];
#pragma unroll
    for (int i = 0; i < RPW; i++) {
        const int r = warp + i * NW;
        const int gy = y0 + r;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int c = lane + 32 * h;
            const int gx = x0 + c;
            const bool ok = r < SH && c < SW && gy >= 0 && gy < H && gx >= 0 && gx < W;
#pragma unroll
            for (int m = 0; m < M; m++) v[m][i][h] = ok ? __ldg(src[m] + (int64_t)gy * W + gx) : 0.f;
        }
    }
#pragma unroll
    for (int i = 0; i < RPW; i++) {
        const int r = warp + i * NW;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int c = lane + 32 * h;
            if (r < SH && c < SW)
#pragma unroll
                for (int m = 0; m < M; m++) dst[m][r][c] = v[m][i][h];
        }
    }
}

// grid: (ceil(W/TW), ceil(H/TH), V*3); partial maps dA, dB, dC [V][3][H][W];
// block partial sums part[(v*3 + c) * nbt + bt] = (sum |x-y|, sum SSIM).
// Register blocking: the horizontal pass gives each thread HC adjacent outputs of one row (the
// 10 + HC inputs are loaded once), the vertical pass VR adjacent outputs of one column.
__global__ void __launch_bounds__(NT) k_ssim_fwd(const float *__restrict__ X, const float *__restrict__ Y, int H,
                                                 int W, Win win, float *__restrict__ dA, float *__restrict__ dB,
                                                 float *__restrict__ dC, float2 *__restrict__ part) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    __shared__ float sxy[2][SH][SWP];
    // horizontal-pass results: (x, y) and (x^2, y^2) as float2 pairs, xy alone -- the passes run
    // on packed fp32x2 FFMA2 (per-element fused multiply-add, the same rounding as the scalar FFMA)
    __shared__ float2 hm2[2][SH][TW + 1];
    __shared__ float hm1[SH][TW + 1];
    float (*sx)[SWP] = sxy[0];
    float (*sy)[SWP] = sxy[1];
    __shared__ float red[2][NT / 32];
    const int plane = blockIdx.z;  // v*3 + c
    const int64_t HW = (int64_t)H * W;
    const int tid = threadIdx.x;
    const float *const srcs[2] = {X + plane * HW, Y + plane * HW};
    load_patches<2>(sxy, srcs, H, W, blockIdx.x * TW - HALO, blockIdx.y * TH - HALO);
    __syncthreads();
    // horizontal pass: SH rows x TW columns of the five moment maps (x, y, x^2, y^2, xy)
    for (int it = tid; it < SH * (TW / HC); it += NT) {
        const int r = it / (TW / HC), c0 = (it % (TW / HC)) * HC;
        float2 m1[HC], m2[HC];  // (x, y), (x^2, y^2)
        float mxy[HC];
#pragma unroll
        for (int o = 0; o < HC; o++) {
            m1[o] = m2[o] = make_float2(0.f, 0.f);
            mxy[o] = 0.f;
        }
#pragma unroll
        for (int j = 0; j < 10 + HC; j++) {
            const float2 v = make_float2(sx[r][c0 + j], sy[r][c0 + j]);
            const float2 vv = __fmul2_rn(v, v);
            const float xy = v.x * v.y;
#pragma unroll
            for (int o = 0; o < HC; o++) {
                const int t = j - o;  // tap index of input j for output o
                if (t >= 0 && t < 11) {
                    const float w = win.g[t];
                    const float2 w2 = make_float2(w, w);
                    m1[o] = __ffma2_rn(w2, v, m1[o]);
                    m2[o] = __ffma2_rn(w2, vv, m2[o]);
                    mxy[o] = __fmaf_rn(w, xy, mxy[o]);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < HC; o++) {
            hm2[0][r][c0 + o] = m1[o];
            hm2[1][r][c0 + o] = m2[o];
            hm1[r][c0 + o] = mxy[o];
        }
    }
    __syncthreads();
    // vertical pass: column c, rows r0 .. r0 + VR - 1
    const int c = tid % TW, r0 = (tid / TW) * VR;
    float2 v1[VR], v2[VR];
    float vxy[VR];
#pragma unroll
    for (int o = 0; o < VR; o++) {
        v1[o] = v2[o] = make_float2(0.f, 0.f);
        vxy[o] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 10 + VR; j++) {
        const float2 p1 = hm2[0][r0 + j][c], p2 = hm2[1][r0 + j][c];
        const float pxy = hm1[r0 + j][c];
#pragma unroll
        for (int o = 0; o < VR; o++) {
            const int t = j - o;
            if (t >= 0 && t < 11) {
                const float w = win.g[t];
                const float2 w2 = make_float2(w, w);
                v1[o] = __ffma2_rn(w2, p1, v1[o]);
                v2[o] = __ffma2_rn(w2, p2, v2[o]);
                vxy[o] = __fmaf_rn(w, pxy, vxy[o]);
            }
        }
    }
    float mom[5][VR];
#pragma unroll
    for (int o = 0; o < VR; o++) {
        mom[0][o] = v1[o].x;
        mom[1][o] = v1[o].y;
        mom[2][o] = v2[o].x;
        mom[3][o] = v2[o].y;
        mom[4][o] = vxy[o];
    }
    float l1 = 0.f, S_sum = 0.f;
    const int gx = blockIdx.x * TW + c;
#pragma unroll
    for (int o = 0; o < VR; o++) {
        const int gy = blockIdx.y * TH + r0 + o;
        if (gy < H && gx < W) {
            const float mx = mom[0][o], my = mom[1][o];
            const float sxx = mom[2][o] - mx * mx, syy = mom[3][o] - my * my, sxy = mom[4][o] - mx * my;
            const float a1 = 2.f * mx * my + SS_C1, a2 = 2.f * sxy + SS_C2;
            const float b1 = mx * mx + my * my + SS_C1, b2 = sxx + syy + SS_C2;
            // SFU reciprocals (rel. error ~1e-7; b1, b2 >= C1, C2 > 0)
            const float ib = __fdividef(1.f, b1 * b2);
            const float S = a1 * a2 * ib;
            const float dS_dmx = 2.f * my * a2 * ib - __fdividef(S * 2.f * mx, b1);
            const float dS_dsxx = -__fdividef(S, b2);
            const float dS_dsxy = 2.f * a1 * ib;
            const int64_t o_ = plane * HW + (int64_t)gy * W + gx;
            dA[o_] = dS_dmx + dS_dsxx * (-2.f * mx) + dS_dsxy * (-my);
            dB[o_] = dS_dsxx;
            dC[o_] = dS_dsxy;
            S_sum += S;
            l1 += fabsf(sx[r0 + o + HALO][c + HALO] - sy[r0 + o + HALO][c + HALO]);
        }
    }
    // block reduction (fixed order)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        S_sum += __shfl_xor_sync(0xffffffffu, S_sum, o);
    }
    if ((tid & 31) == 0) {
        red[0][tid >> 5] = l1;
        red[1][tid >> 5] = S_sum;
    }
    __syncthreads();
    if (tid == 0) {
        float a = 0, b = 0;
        for (int k = 0; k < NT / 32; k++) {
            a += red[0][k];
            b += red[1][k];
        }
        const int nbt = gridDim.x * gridDim.y;
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
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    finalize_view(part, blockIdx.x, nbt, lambda, invN, loss);
}

__global__ void __launch_bounds__(NT) k_ssim_bwd(const float *__restrict__ X, const float *__restrict__ Y, int H,
                                                 int W, Win win, float lambda, float invN,
                                                 const float *__restrict__ dA, const float *__restrict__ dB,
                                                 const float *__restrict__ dC, float *__restrict__ dL,
                                                 const float2 *__restrict__ part, float *__restrict__ loss) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    __shared__ float s[3][SH][SWP];
    __shared__ float2 hm2[SH][TW + 1];  // (A, B) pairs for packed FFMA2; C alone
    __shared__ float hm1[SH][TW + 1];
    const int plane = blockIdx.z;
    const int64_t HW = (int64_t)H * W;
    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TW - HALO, y0 = blockIdx.y * TH - HALO;
    // this thread's output pixels: column c, rows r0 .. r0 + VR - 1 (x, y prefetched now)
    const int c = tid % TW, r0 = (tid / TW) * VR;
    const int gx = blockIdx.x * TW + c;
    float xv[VR], yv[VR];
#pragma unroll
    for (int o = 0; o < VR; o++) {
        const int gy = blockIdx.y * TH + r0 + o;
        const bool ok = gx < W && gy < H;
        xv[o] = ok ? __ldg(X + plane * HW + (int64_t)gy * W + gx) : 0.f;
        yv[o] = ok ? __ldg(Y + plane * HW + (int64_t)gy * W + gx) : 0.f;
    }
    const float *const srcs[3] = {dA + plane * HW, dB + plane * HW, dC + plane * HW};
    load_patches<3>(s, srcs, H, W, x0, y0);
    __syncthreads();
    for (int it = tid; it < SH * (TW / HC); it += NT) {
        const int r = it / (TW / HC), c0 = (it % (TW / HC)) * HC;
        float2 ab[HC];
        float cc[HC];
#pragma unroll
        for (int o = 0; o < HC; o++) {
            ab[o] = make_float2(0.f, 0.f);
            cc[o] = 0.f;
        }
#pragma unroll
        for (int j = 0; j < 10 + HC; j++) {
            const float2 v = make_float2(s[0][r][c0 + j], s[1][r][c0 + j]);
            const float vc = s[2][r][c0 + j];
#pragma unroll
            for (int o = 0; o < HC; o++) {
                const int t = j - o;
                if (t >= 0 && t < 11) {
                    const float w = win.g[t];
                    ab[o] = __ffma2_rn(make_float2(w, w), v, ab[o]);
                    cc[o] = __fmaf_rn(w, vc, cc[o]);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < HC; o++) {
            hm2[r][c0 + o] = ab[o];
            hm1[r][c0 + o] = cc[o];
        }
    }
    __syncthreads();
    // the first CTA of each view also reduces that view's loss partials (written by k_ssim_fwd)
    if (blockIdx.x == 0 && blockIdx.y == 0 && plane % 3 == 0)
        finalize_view(part, plane / 3, gridDim.x * gridDim.y, lambda, invN, loss);
    float2 vab[VR];
    float vc[VR];
#pragma unroll
    for (int o = 0; o < VR; o++) {
        vab[o] = make_float2(0.f, 0.f);
        vc[o] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 10 + VR; j++) {
        const float2 p = hm2[r0 + j][c];
        const float pc = hm1[r0 + j][c];
#pragma unroll
        for (int o = 0; o < VR; o++) {
            const int t = j - o;
            if (t >= 0 && t < 11) {
                const float w = win.g[t];
                vab[o] = __ffma2_rn(make_float2(w, w), p, vab[o]);
                vc[o] = __fmaf_rn(w, pc, vc[o]);
            }
        }
    }
    float acc[3][VR];
#pragma unroll
    for (int o = 0; o < VR; o++) {
        acc[0][o] = vab[o].x;
        acc[1][o] = vab[o].y;
        acc[2][o] = vc[o];
    }
    if (gx >= W) return;
#pragma unroll
    for (int o = 0; o < VR; o++) {
        const int gy = blockIdx.y * TH + r0 + o;
        if (gy >= H) break;
        const int64_t o_ = plane * HW + (int64_t)gy * W + gx;
        const float dssim = acc[0][o] + 2.f * xv[o] * acc[1][o] + yv[o] * acc[2][o];
        const float d = xv[o] - yv[o];
        const float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
        dL[o_] = (1.f - lambda) * sgn * invN - lambda * dssim * invN;
    }
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t loss_ws_bytes(int V, int H, int W) {
    size_t plane = (size_t)V * 3 * H * W * sizeof(float);
    size_t nbt = (size_t)((W + TW - 1) / TW) * ((H + TH - 1) / TH);
    return 3 * align256(plane) + align256((size_t)V * 3 * nbt * sizeof(float2));
}

cudaError_t launch_loss(const float *render, const float *gt, int V, int H, int W, float lambda, float *loss, float *dL,
                        void *ws, cudaStream_t s) {
    static const Win win = make_window();
    size_t plane = align256((size_t)V * 3 * H * W * sizeof(float));
    float *dA = at<float>(ws, 0), *dB = at<float>(ws, plane), *dC = at<float>(ws, 2 * plane);
    float2 *part = at<float2>(ws, 3 * plane);
    dim3 grid((W + TW - 1) / TW, (H + TH - 1) / TH, V * 3);
    const int nbt = grid.x * grid.y;
    float invN = (float)(1.0 / (3.0 * H * W));
    ProfScope prof("k_ssim", s);
    launch_pdl(k_ssim_fwd, grid, NT, 0, s, render, gt, H, W, win, dA, dB, dC, part);
    if (dL)
        launch_pdl(k_ssim_bwd, grid, NT, 0, s, render, gt, H, W, win, lambda, invN, dA, dB, dC, dL, part, loss);
    else
        launch_pdl(k_loss_final, V, 256, 0, s, part, nbt, lambda, invN, loss);
    return cudaGetLastError();
}

}  // namespace gsk
