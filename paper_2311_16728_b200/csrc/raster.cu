// raster.cu -- A6 (per-tile front-to-back alpha compositing, Eq. 3) and A8 (its backward).
//
// Eq. 3 with the reading prod_{j<i}(1 - alpha_j) (R1), evaluated per
// pixel over the depth-sorted list of its tile (SPEC.md:348 (4)): power = -1/2 d^T Q d with
// d = pixel - mean2d (fp32 recipe order, bit-exact to the oracle), cut at power < -4.5
// (Mahalanobis^2 > 9, R9) or power > 0; alpha = min(0.99, sigma e^power) (R7); skip alpha
// < 1/255; stop the pixel when T (1 - alpha) < 1e-4 (R8).
//
// Layout: one 256-thread CTA per (view, 16x16 tile), one thread per pixel; each warp owns an
// 8x4 pixel block (2 x 4 blocks per tile).  Gaussian records are staged in shared memory in
// batches of 256; each warp then builds, in parallel over the batch (one Gaussian per lane,
// ballot + popc), the ordered list of Gaussians that can reach its block: the exact minimum of
// d^T Q d over the block is compared with the Gaussian's limit min(9, 2 ln(255 sigma)) (3-sigma
// cutoff or alpha >= 1/255), padded so the test is conservative.  The sequential per-pixel
// loop then only visits that list -- no pixel result changes.  The CTA leaves as soon as every
// pixel of the tile has stopped.
//
// The backward replays each pixel's list back to front: dL/dc, dL/dalpha
// = T_k sum_c g_c (c_k - acc), dL/dsigma, dL/dpower -> dL/dmean2d, dL/dconic.  The nine
// per-pixel gradients of a Gaussian are summed over the warp with a transposing butterfly
// (9 + 5 shuffles instead of 45) and added to the per-(view, Gaussian) record by nine lanes
// with one scalar red.global.add each.
#include "gs_internal.cuh"

namespace gsk {

#define FMA __fmaf_rn
#define MUL __fmul_rn
#define SUB __fsub_rn

constexpr float ALPHA_MAX = 0.99f;
constexpr float ALPHA_MIN = 1.0f / 255.0f;
constexpr float T_STOP = 1e-4f;
constexpr float POWER_CUT = -4.5f;

// power = -1/2 (A dx^2 + C dy^2) - B dx dy in the recipe's op order
__device__ __forceinline__ float pixel_power(float px, float py, const float4 g0, float C, float &dx, float &dy) {
    dx = SUB(px, g0.x);
    dy = SUB(py, g0.y);
    float qf = FMA(MUL(C, dy), dy, MUL(MUL(g0.z, dx), dx));
    return FMA(-MUL(g0.w, dx), dy, MUL(-0.5f, qf));
}

// e^power with the SFU: ex2.approx.ftz(power * log2 e).  Forward and backward evaluate alpha
// with this same sequence, so their skip / stop decisions agree bit for bit.
__device__ __forceinline__ float fast_exp(float power) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(power * 1.4426950408889634f));
    return y;
}

// Largest d^T Q d at which a Gaussian can still be composited: the 3-sigma cutoff (R9) or the
// alpha >= 1/255 skip, alpha <= sigma e^(-q/2) (R7), whichever is tighter (-1: never composited).
__device__ __forceinline__ float q_limit(float sigma) {
    if (sigma * 255.0f < 1.0f) return -1.0f;
    return fminf(9.0f, 2.0f * __logf(255.0f * sigma));
}

// Conservative warp-level skip: minimum of d^T Q d over the warp's pixel block (centres
// [x0, x0 + 7] x [y0, y0 + 3]) exceeds the Gaussian's limit.  Exact box-ellipse minimum:
// 0 if the mean is inside, else the smallest of the four clamped edge minima.  The padding
// (1e-3 relative + 1e-3 absolute) absorbs the rounding of the per-pixel fp32 power, so a
// culled Gaussian can never pass the per-pixel tests.
__device__ __forceinline__ bool block_misses(const float4 g0, const float4 g1, float qlim, float x0, float y0) {
    if (qlim < 0.f) return true;
    const float A = g0.z, B = g0.w, C = g1.x;
    const float ax = x0 - g0.x, bx = x0 + 7.f - g0.x, ay = y0 - g0.y, by = y0 + 3.f - g0.y;
    if (ax <= 0.f && bx >= 0.f && ay <= 0.f && by >= 0.f) return false;
    float best = 3.4e38f;
    // edges x = X: f = A X^2 + 2 B X y + C y^2, y* = -B X / C clamped to [ay, by]
#pragma unroll
    for (int e = 0; e < 2; e++) {
        float X = e ? bx : ax;
        float y = fminf(fmaxf(-B * X / C, ay), by);
        best = fminf(best, A * X * X + 2.f * B * X * y + C * y * y);
        float Y = e ? by : ay;
        float x = fminf(fmaxf(-B * Y / A, ax), bx);
        best = fminf(best, A * x * x + 2.f * B * x * Y + C * Y * Y);
    }
    return best > qlim * 1.001f + 1e-3f;
}

// thread -> pixel: warp w covers the 8x4 block (w & 1, w >> 1) of the tile
__device__ __forceinline__ void pixel_of(int tid, int &lx, int &ly) {
    int w = tid >> 5, l = tid & 31;
    lx = (w & 1) * 8 + (l & 7);
    ly = (w >> 1) * 4 + (l >> 3);
}

__global__ void __launch_bounds__(BLOCK_PIX) k_raster_fwd(const uint2 *__restrict__ ranges,
                                                          const uint32_t *__restrict__ vals,
                                                          const float4 *__restrict__ rec0,
                                                          const float4 *__restrict__ rec1,
                                                          const float4 *__restrict__ rec2, int64_t n, int W, int H,
                                                          int TX, int tiles, float bg0, float bg1, float bg2,
                                                          float *__restrict__ out_rgb, float *__restrict__ out_T,
                                                          float *__restrict__ T_keep, uint32_t *__restrict__ ncontrib,
                                                          uint32_t *__restrict__ ncomp) {
    __shared__ float4 s0[BLOCK_PIX];
    __shared__ float4 s1[BLOCK_PIX];
    __shared__ float4 s2[BLOCK_PIX];
    __shared__ uint8_t wl[BLOCK_PIX / 32][BLOCK_PIX];
    const int view = blockIdx.z;
    const int tile = blockIdx.y * TX + blockIdx.x;
    const int tid = threadIdx.x;
    int lx, ly;
    pixel_of(tid, lx, ly);
    const int px = blockIdx.x * TILE + lx;
    const int py = blockIdx.y * TILE + ly;
    const float wx0 = (float)(blockIdx.x * TILE + ((tid >> 5) & 1) * 8);
    const float wy0 = (float)(blockIdx.y * TILE + (tid >> 6) * 4);
    const bool inside = px < W && py < H;
    const uint2 range = ranges[(int64_t)view * tiles + tile];
    const int todo_all = (int)(range.y - range.x);
    const float fx = (float)px, fy = (float)py;
    const int64_t vbase = (int64_t)view * n;
    float T = 1.0f, c0 = 0.f, c1 = 0.f, c2 = 0.f;
    uint32_t last = 0, composited = 0;
    bool done = !inside;
    const int warp = tid >> 5, lane = tid & 31;
    const unsigned lt = (1u << lane) - 1u;
    for (int b0 = 0; b0 < todo_all; b0 += BLOCK_PIX) {
        if (__syncthreads_count(done) == BLOCK_PIX) break;
        int idx = b0 + tid;
        if (idx < todo_all) {
            int64_t m = vbase + vals[range.x + idx];
            float4 r1 = rec1[m], r2 = rec2[m];
            r2.w = q_limit(r1.y);
            s0[tid] = rec0[m];
            s1[tid] = r1;
            s2[tid] = r2;
        }
        __syncthreads();
        const int cnt = min(BLOCK_PIX, todo_all - b0);
        // phase 1 (parallel over the batch): ordered list of the Gaussians whose padded
        // 3-sigma box meets this warp's 8x4 block
        int nsel = 0;
        for (int k = 0; k < cnt; k += 32) {
            int j = k + lane;
            bool hit = j < cnt && !block_misses(s0[j], s1[j], s2[j].w, wx0, wy0);
            unsigned b = __ballot_sync(0xffffffffu, hit);
            if (hit) wl[warp][nsel + __popc(b & lt)] = (uint8_t)j;
            nsel += __popc(b);
        }
        __syncwarp();
        // phase 2 (sequential per pixel): composite the warp's list front to back
        for (int t = 0; t < nsel; t++) {
            if (__all_sync(0xffffffffu, done)) break;
            const int j = wl[warp][t];
            float4 g0 = s0[j];
            float4 g1 = s1[j];
            float4 g2 = s2[j];
            float dx, dy;
            float power = pixel_power(fx, fy, g0, g1.x, dx, dy);
            if (done || power > 0.0f || power < POWER_CUT) continue;
            float alpha = fminf(ALPHA_MAX, g1.y * fast_exp(power));
            if (alpha < ALPHA_MIN) continue;
            float test_T = T * (1.0f - alpha);
            if (test_T < T_STOP) {
                done = true;
                continue;
            }
            float w = alpha * T;
            c0 += g1.z * w;
            c1 += g1.w * w;
            c2 += g2.x * w;
            T = test_T;
            composited++;
            last = (uint32_t)(b0 + j + 1);  // 1-based list position of the last composited
        }
    }
    if (inside) {
        int64_t HW = (int64_t)H * W;
        int64_t pix = (int64_t)py * W + px;
        float *o = out_rgb + (int64_t)view * 3 * HW + pix;
        o[0] = c0 + T * bg0;
        o[HW] = c1 + T * bg1;
        o[2 * HW] = c2 + T * bg2;
        if (out_T) out_T[(int64_t)view * HW + pix] = T;
        T_keep[(int64_t)view * HW + pix] = T;
        ncontrib[(int64_t)view * HW + pix] = last;
        ncomp[(int64_t)view * HW + pix] = composited;
    }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Warp sum of eight values with a transposing butterfly: at offsets 16, 8, 4 every lane keeps
// half of its values and receives the partner's other half (4 + 2 + 1 shuffles), then two
// plain xor steps finish the sum.  Lane l ends with the total of value index
// ((l >> 4) & 1) * 4 + ((l >> 3) & 1) * 2 + ((l >> 2) & 1); 9 shuffles instead of 40.
__device__ __forceinline__ float warp_sum8_transposed(float a[8], int lane) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
    float h[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        float send = b4 ? a[k] : a[k + 4];
        float keep = b4 ? a[k + 4] : a[k];
        h[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    float q[2];
#pragma unroll
    for (int k = 0; k < 2; k++) {
        float send = b3 ? h[k] : h[k + 2];
        float keep = b3 ? h[k + 2] : h[k];
        q[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    float send = b2 ? q[0] : q[1];
    float r = (b2 ? q[1] : q[0]) + __shfl_xor_sync(0xffffffffu, send, 4);
    r += __shfl_xor_sync(0xffffffffu, r, 2);
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    return r;
}

__global__ void __launch_bounds__(BLOCK_PIX) k_raster_bwd(const uint2 *__restrict__ ranges,
                                                          const uint32_t *__restrict__ vals,
                                                          const float4 *__restrict__ rec0,
                                                          const float4 *__restrict__ rec1,
                                                          const float4 *__restrict__ rec2, int64_t n, int W, int H,
                                                          int TX, int tiles, float bg0, float bg1, float bg2,
                                                          const float *__restrict__ dL_drgb,
                                                          const float *__restrict__ T_keep,
                                                          const uint32_t *__restrict__ ncontrib,
                                                          float4 *__restrict__ g2d) {
    __shared__ float4 s0[BLOCK_PIX];
    __shared__ float4 s1[BLOCK_PIX];
    __shared__ float4 s2[BLOCK_PIX];
    __shared__ uint32_t sid[BLOCK_PIX];
    __shared__ uint8_t wl[BLOCK_PIX / 32][BLOCK_PIX];
    __shared__ uint32_t s_maxlast;
    const int view = blockIdx.z;
    const int tile = blockIdx.y * TX + blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31;
    int lx, ly;
    pixel_of(tid, lx, ly);
    const int px = blockIdx.x * TILE + lx;
    const int py = blockIdx.y * TILE + ly;
    const float wx0 = (float)(blockIdx.x * TILE + ((tid >> 5) & 1) * 8);
    const float wy0 = (float)(blockIdx.y * TILE + (tid >> 6) * 4);
    const bool inside = px < W && py < H;
    const uint2 range = ranges[(int64_t)view * tiles + tile];
    const float fx = (float)px, fy = (float)py;
    const int64_t vbase = (int64_t)view * n;
    const int64_t HW = (int64_t)H * W;
    const int64_t pix = (int64_t)py * W + px;
    float T = 1.f, g_0 = 0.f, g_1 = 0.f, g_2 = 0.f;
    uint32_t last = 0;
    if (inside) {
        T = T_keep[(int64_t)view * HW + pix];
        last = ncontrib[(int64_t)view * HW + pix];
        const float *g = dL_drgb + (int64_t)view * 3 * HW + pix;
        g_0 = g[0];
        g_1 = g[HW];
        g_2 = g[2 * HW];
    }
    if (tid == 0) s_maxlast = 0;
    __syncthreads();
    // the warp's own furthest composited position bounds its work; the CTA's bounds the batches
    uint32_t wlast = last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wlast = max(wlast, __shfl_xor_sync(0xffffffffu, wlast, o));
    if (lane == 0) atomicMax(&s_maxlast, wlast);
    __syncthreads();
    const int todo_all = (int)s_maxlast;
    float acc0 = bg0, acc1 = bg1, acc2 = bg2;
    // process positions todo_all .. 1 (1-based within the tile range), batches from the back
    for (int b_end = todo_all; b_end > 0; b_end -= BLOCK_PIX) {
        int b_start = max(0, b_end - BLOCK_PIX);
        int cnt = b_end - b_start;
        __syncthreads();
        if (tid < cnt) {
            int pos = b_end - 1 - tid;  // s[tid] holds 0-based position b_end-1-tid (back to front)
            uint32_t gi = vals[range.x + pos];
            int64_t m = vbase + gi;
            sid[tid] = gi;
            float4 r1 = rec1[m], r2 = rec2[m];
            r2.w = q_limit(r1.y);
            s0[tid] = rec0[m];
            s1[tid] = r1;
            s2[tid] = r2;
        }
        __syncthreads();
        // phase 1: ordered (back to front) list of the batch entries this warp must replay --
        // at or before its furthest composited position and with a box meeting its block
        const int warp = tid >> 5;
        const unsigned lt = (1u << lane) - 1u;
        const int j0 = (uint32_t)b_end > wlast ? (int)((uint32_t)b_end - wlast) : 0;
        int nsel = 0;
        for (int k = 0; k < cnt; k += 32) {
            int j = k + lane;
            bool hit = j < cnt && j >= j0 && !block_misses(s0[j], s1[j], s2[j].w, wx0, wy0);
            unsigned b = __ballot_sync(0xffffffffu, hit);
            if (hit) wl[warp][nsel + __popc(b & lt)] = (uint8_t)j;
            nsel += __popc(b);
        }
        __syncwarp();
        for (int t = 0; t < nsel; t++) {
            const int j = wl[warp][t];
            const uint32_t position = (uint32_t)(b_end - j);  // 1-based position in the tile list
            float4 g0 = s0[j];
            float4 g2 = s2[j];
            float4 g1 = s1[j];
            float dLdu = 0.f, dLdv = 0.f, dLdA = 0.f, dLdB = 0.f, dLdC = 0.f, dLdsig = 0.f;
            float dLdr = 0.f, dLdg = 0.f, dLdb = 0.f;
            bool contrib = false;
            if (position <= last) {
                float dx, dy;
                float power = pixel_power(fx, fy, g0, g1.x, dx, dy);
                if (!(power > 0.0f || power < POWER_CUT)) {
                    float e = fast_exp(power);
                    float a_raw = g1.y * e;
                    float alpha = fminf(ALPHA_MAX, a_raw);
                    if (alpha >= ALPHA_MIN) {
                        contrib = true;
                        T = __fdividef(T, 1.0f - alpha);  // transmittance before this Gaussian
                        float w = alpha * T;
                        dLdr = g_0 * w;
                        dLdg = g_1 * w;
                        dLdb = g_2 * w;
                        float cr = g1.z, cg = g1.w, cb = g2.x;
                        float dLda = T * (g_0 * (cr - acc0) + g_1 * (cg - acc1) + g_2 * (cb - acc2));
                        acc0 = alpha * cr + (1.f - alpha) * acc0;
                        acc1 = alpha * cg + (1.f - alpha) * acc1;
                        acc2 = alpha * cb + (1.f - alpha) * acc2;
                        if (!(a_raw > ALPHA_MAX)) {
                            dLdsig = e * dLda;
                            float dLdp = alpha * dLda;
                            float A = g0.z, B = g0.w, C = g1.x;
                            dLdu = dLdp * (A * dx + B * dy);
                            dLdv = dLdp * (C * dy + B * dx);
                            dLdA = -0.5f * dx * dx * dLdp;
                            dLdB = -dx * dy * dLdp;
                            dLdC = -0.5f * dy * dy * dLdp;
                        }
                    }
                }
            }
            if (__any_sync(0xffffffffu, contrib)) {
                // per-(view, Gaussian) record: [u, v, A, B | C, sigma, r, g | b, -, -, -]
                float vals8[8] = {dLdu, dLdv, dLdA, dLdB, dLdC, dLdsig, dLdr, dLdg};
                float mine = warp_sum8_transposed(vals8, lane);
                float bsum = warp_sum(dLdb);
                float *dst = reinterpret_cast<float *>(g2d + 3 * (vbase + sid[j]));
                if ((lane & 3) == 0)
                    atomicAdd(dst + ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1), mine);
                if (lane == 1) atomicAdd(dst + 8, bsum);
            }
        }
    }
}

cudaError_t launch_raster_fwd(const Layout &L, void *ws, const float bg[3], float *out_rgb, float *out_T,
                              cudaStream_t s) {
    dim3 grid(L.TX, L.TY, L.V);
    ProfScope prof("k_raster_fwd", s);
    k_raster_fwd<<<grid, BLOCK_PIX, 0, s>>>(at<uint2>(ws, L.ranges), at<uint32_t>(ws, L.vals0), at<float4>(ws, L.rec0),
                                            at<float4>(ws, L.rec1), at<float4>(ws, L.rec2), L.n, L.W, L.H, L.TX,
                                            L.tiles, bg[0], bg[1], bg[2], out_rgb, out_T, at<float>(ws, L.Tfinal),
                                            at<uint32_t>(ws, L.ncontrib), at<uint32_t>(ws, L.ncomp));
    return cudaGetLastError();
}

cudaError_t launch_raster_bwd(const Layout &L, void *ws, const float bg[3], const float *dL_drgb, cudaStream_t s) {
    dim3 grid(L.TX, L.TY, L.V);
    ProfScope prof("k_raster_bwd", s);
    k_raster_bwd<<<grid, BLOCK_PIX, 0, s>>>(at<uint2>(ws, L.ranges), at<uint32_t>(ws, L.vals0), at<float4>(ws, L.rec0),
                                            at<float4>(ws, L.rec1), at<float4>(ws, L.rec2), L.n, L.W, L.H, L.TX,
                                            L.tiles, bg[0], bg[1], bg[2], dL_drgb, at<float>(ws, L.Tfinal),
                                            at<uint32_t>(ws, L.ncontrib), at<float4>(ws, L.grad2d));
    return cudaGetLastError();
}

}  // namespace gsk
