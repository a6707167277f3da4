// densify.cu -- SURVEY §8(f) f1: adaptive density control, densify and prune (
// PAPER.md:229 "splitting or cloning hyper primitives with large loss gradients similar to
// [kerbl2023]").  Readings R27-R30 in DESIGN.md.
//
//   k_densify_stats     after a forward: per Gaussian, number of views it is visible in (+=) and
//                       the largest pixel radius (max=) -- with the backward's ||dL/dmean2d||
//                       sums (R24) these are the statistics of the densify interval;
//   k_densify_classify  keep / clone / split / prune per Gaussian, decided with fp32 IEEE
//                       operations (the oracle takes the same decisions bit for bit), and the
//                       three flags whose exclusive scans (k_scan) place every output;
//   k_densify_apply     writes the new map: kept and cloned originals in index order (bitwise
//                       copies with their Adam moments), then the clones, then two children per
//                       split parent; new Gaussians at P + R(q) diag(e^s) z with zero moments,
//                       split children with log s - ln 1.6.
#include <cmath>

#include "gs_internal.cuh"

namespace gsk {

__global__ void __launch_bounds__(256) k_densify_stats(const int32_t *__restrict__ radius, int64_t n, int V,
                                                       float *__restrict__ vis_count, int32_t *__restrict__ max_radius) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int cnt = 0, mr = 0;
    for (int v = 0; v < V; v++) {
        const int32_t r = radius[(int64_t)v * n + i];
        if (r > 0) {
            cnt++;
            mr = max(mr, r);
        }
    }
    if (cnt) {
        vis_count[i] += (float)cnt;
        max_radius[i] = max(max_radius[i], mr);
    }
}

struct DensifyTemp {  // offsets inside the caller's temp buffer
    size_t hdr[3], flags[3], cls, flag[3], off[3], total;
};

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

static DensifyTemp densify_temp(int64_t n) {
    DensifyTemp t;
    size_t o = 0;
    const int64_t blocks = std::max<int64_t>((n + SCAN_TILE - 1) / SCAN_TILE, 1);
    for (int k = 0; k < 3; k++) {
        t.hdr[k] = o;
        o += al256(sizeof(WsHeader));
        t.flags[k] = o;
        o += al256((size_t)blocks * sizeof(uint64_t));
    }
    t.cls = o;
    o += al256((size_t)std::max<int64_t>(n, 1));
    for (int k = 0; k < 3; k++) {
        t.flag[k] = o;
        o += al256((size_t)std::max<int64_t>(n, 1) * sizeof(uint32_t));
        t.off[k] = o;
        o += al256((size_t)std::max<int64_t>(n, 1) * sizeof(uint32_t));
    }
    t.total = o;
    return t;
}

size_t densify_temp_bytes(int64_t n) { return densify_temp(n).total; }

__global__ void __launch_bounds__(256) k_densify_classify(const float *__restrict__ P, int64_t n, int64_t ld,
                                                          const float *__restrict__ grad_accum,
                                                          const float *__restrict__ vis_count,
                                                          const int32_t *__restrict__ max_radius, float grad_thr,
                                                          float big, float logit_thr, int32_t max_screen,
                                                          uint8_t *__restrict__ cls, uint32_t *__restrict__ f_keep,
                                                          uint32_t *__restrict__ f_clone,
                                                          uint32_t *__restrict__ f_split) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float vc = vis_count[i];
    const float mean = vc > 0.f ? __fdiv_rn(grad_accum[i], vc) : 0.f;
    const bool high = mean >= grad_thr;
    float maxs = 0.f;
#pragma unroll
    for (int j = 0; j < 3; j++) maxs = fmaxf(maxs, (float)exp((double)P[(7 + j) * ld + i]));
    const bool large = maxs > big;
    const bool prune = P[10 * ld + i] < logit_thr || max_radius[i] > max_screen;
    const uint8_t c = prune ? 3 : (high && !large) ? 1 : (high && large) ? 2 : 0;
    cls[i] = c;
    f_keep[i] = c <= 1;
    f_clone[i] = c == 1;
    f_split[i] = c == 2;
}

// fp32 rotation of a raw quaternion (normalised) applied to diag(e^s) z
__device__ __forceinline__ void gauss_offset(const float q[4], const float e[3], const float z[3], float o[3]) {
    const float in = rsqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    const float w = q[0] * in, x = q[1] * in, y = q[2] * in, zq = q[3] * in;
    const float R[9] = {1.f - 2.f * (y * y + zq * zq), 2.f * (x * y - w * zq), 2.f * (x * zq + w * y),
                        2.f * (x * y + w * zq), 1.f - 2.f * (x * x + zq * zq), 2.f * (y * zq - w * x),
                        2.f * (x * zq - w * y), 2.f * (y * zq + w * x), 1.f - 2.f * (x * x + y * y)};
    const float d[3] = {e[0] * z[0], e[1] * z[1], e[2] * z[2]};
#pragma unroll
    for (int a = 0; a < 3; a++) o[a] = R[3 * a] * d[0] + R[3 * a + 1] * d[1] + R[3 * a + 2] * d[2];
}

__global__ void __launch_bounds__(256) k_densify_apply(const float *__restrict__ P, const float *__restrict__ M,
                                                       const float *__restrict__ Vv, int64_t n, int64_t ld, int K,
                                                       const float *__restrict__ zs, const uint8_t *__restrict__ cls,
                                                       const uint32_t *__restrict__ o_keep,
                                                       const uint32_t *__restrict__ o_clone,
                                                       const uint32_t *__restrict__ o_split, const WsHeader *h_keep,
                                                       const WsHeader *h_clone, float *__restrict__ Q,
                                                       float *__restrict__ QM, float *__restrict__ QV, int64_t ldo) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t c = cls[i];
    if (c == 3) return;
    const int64_t n_keep = h_keep->P, n_clone = h_clone->P;
    if (c <= 1) {  // the original itself, moments included
        const int64_t d = o_keep[i];
        for (int r = 0; r < K; r++) {
            Q[r * ldo + d] = P[r * ld + i];
            if (QM) {
                QM[r * ldo + d] = M[r * ld + i];
                QV[r * ldo + d] = Vv[r * ld + i];
            }
        }
        if (c == 0) return;
    }
    const float q[4] = {P[3 * ld + i], P[4 * ld + i], P[5 * ld + i], P[6 * ld + i]};
    const float e[3] = {(float)exp((double)P[7 * ld + i]), (float)exp((double)P[8 * ld + i]),
                        (float)exp((double)P[9 * ld + i])};
    const int nchild = c == 1 ? 1 : 2;
    const int64_t d0 = c == 1 ? n_keep + o_clone[i] : n_keep + n_clone + 2 * (int64_t)o_split[i];
    for (int k = 0; k < nchild; k++) {
        const int64_t d = d0 + k;
        float o[3];
        gauss_offset(q, e, zs + (i * 2 + k) * 3, o);
        for (int r = 0; r < K; r++) {
            float val = P[r * ld + i];
            if (r < 3) val += o[r];
            else if (c == 2 && r >= 7 && r < 10) val -= 0.470003629245735553650937031148f;  // ln 1.6
            Q[r * ldo + d] = val;
            if (QM) {
                QM[r * ldo + d] = 0.f;
                QV[r * ldo + d] = 0.f;
            }
        }
    }
}

cudaError_t launch_densify_stats(const int32_t *radius, int64_t n, int V, float *vis_count, int32_t *max_radius,
                                 cudaStream_t s) {
    if (n > 0) k_densify_stats<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(radius, n, V, vis_count, max_radius);
    return cudaGetLastError();
}

cudaError_t launch_densify_plan(const gs_params &p, const float *grad_accum, const float *vis_count,
                                const int32_t *max_radius, float grad_thr, float big, float logit_thr,
                                int32_t max_screen, void *temp, cudaStream_t s) {
    const DensifyTemp t = densify_temp(p.n);
    for (int k = 0; k < 3; k++) cudaMemsetAsync(at<char>(temp, t.hdr[k]), 0, sizeof(WsHeader), s);
    const int64_t blocks = std::max<int64_t>((p.n + SCAN_TILE - 1) / SCAN_TILE, 1);
    for (int k = 0; k < 3; k++) cudaMemsetAsync(at<char>(temp, t.flags[k]), 0, (size_t)blocks * sizeof(uint64_t), s);
    if (p.n == 0) return cudaGetLastError();
    k_densify_classify<<<(unsigned)((p.n + 255) / 256), 256, 0, s>>>(
        p.data, p.n, p.ld, grad_accum, vis_count, max_radius, grad_thr, big, logit_thr, max_screen,
        at<uint8_t>(temp, t.cls), at<uint32_t>(temp, t.flag[0]), at<uint32_t>(temp, t.flag[1]),
        at<uint32_t>(temp, t.flag[2]));
    for (int k = 0; k < 3; k++) {
        cudaError_t e = launch_scan_u32(at<uint32_t>(temp, t.flag[k]), at<uint32_t>(temp, t.off[k]), p.n,
                                        at<uint64_t>(temp, t.flags[k]), at<WsHeader>(temp, t.hdr[k]), s);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

void densify_totals(const void *temp, int64_t n, uint32_t tot[3]) {
    const DensifyTemp t = densify_temp(n);
    for (int k = 0; k < 3; k++) {
        WsHeader h;
        cudaMemcpy(&h, at<char>(const_cast<void *>(temp), t.hdr[k]), sizeof(WsHeader), cudaMemcpyDeviceToHost);
        tot[k] = h.P;
    }
}

// per-Gaussian byte tags through the planned densification: a kept or cloned original keeps its
// tag, its clone and split children inherit it
__global__ void __launch_bounds__(256) k_densify_tags(const uint8_t *__restrict__ cls, int64_t n,
                                                      const uint32_t *__restrict__ o_keep,
                                                      const uint32_t *__restrict__ o_clone,
                                                      const uint32_t *__restrict__ o_split, const WsHeader *h_keep,
                                                      const WsHeader *h_clone, const uint8_t *__restrict__ tin,
                                                      uint8_t *__restrict__ tout) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t c = cls[i], tag = tin[i];
    const int64_t n_keep = h_keep->P, n_clone = h_clone->P;
    if (c <= 1) tout[o_keep[i]] = tag;
    if (c == 1) tout[n_keep + o_clone[i]] = tag;
    if (c == 2) tout[n_keep + n_clone + 2 * (int64_t)o_split[i]] = tout[n_keep + n_clone + 2 * (int64_t)o_split[i] + 1] = tag;
}

cudaError_t launch_densify_tags(int64_t n, const void *temp, const uint8_t *tin, uint8_t *tout, cudaStream_t s) {
    const DensifyTemp t = densify_temp(n);
    if (n == 0) return cudaGetLastError();
    void *tp = const_cast<void *>(temp);
    k_densify_tags<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
        at<uint8_t>(tp, t.cls), n, at<uint32_t>(tp, t.off[0]), at<uint32_t>(tp, t.off[1]), at<uint32_t>(tp, t.off[2]),
        at<WsHeader>(tp, t.hdr[0]), at<WsHeader>(tp, t.hdr[1]), tin, tout);
    return cudaGetLastError();
}

cudaError_t launch_densify_apply(const gs_params &p, const float *m, const float *v, const float *z, const void *temp,
                                 const gs_params &out, float *out_m, float *out_v, cudaStream_t s) {
    const DensifyTemp t = densify_temp(p.n);
    if (p.n == 0) return cudaGetLastError();
    void *tp = const_cast<void *>(temp);
    k_densify_apply<<<(unsigned)((p.n + 255) / 256), 256, 0, s>>>(
        p.data, m, v, p.n, p.ld, gs_param_rows(p.sh_degree), z, at<uint8_t>(tp, t.cls), at<uint32_t>(tp, t.off[0]),
        at<uint32_t>(tp, t.off[1]), at<uint32_t>(tp, t.off[2]), at<WsHeader>(tp, t.hdr[0]),
        at<WsHeader>(tp, t.hdr[1]), out.data, out_m, out_v, out.ld);
    return cudaGetLastError();
}

}  // namespace gsk

namespace gsk {

// ---------------------------------------------------------------- f2: geometry-based densification
// SPEC.md:473-481 with the create_map_points initialisation;
// readings R31-R33 in DESIGN.md.  One CTA walks the keypoints in chunks of 1024, in order: a thread
// per keypoint decides (inactive, pixel inside the image, depth from the depth map or from the
// K = 4 nearest active keypoints within rho, inverse-distance weighted), a block scan of the
// decisions gives each new primitive its row (keypoint order), and the thread writes it.
constexpr int GD_THREADS = 1024;

__global__ void __launch_bounds__(GD_THREADS) k_geometry_densify(const gs_camera cam, const float2 *__restrict__ uv,
                                                                 const int32_t *__restrict__ active,
                                                                 const float *__restrict__ kp_depth,
                                                                 const float *__restrict__ depth_map,
                                                                 const float *__restrict__ image, int nk, int mode,
                                                                 float rho, int K, float *__restrict__ out,
                                                                 int64_t ldo, int32_t *__restrict__ src,
                                                                 int32_t *__restrict__ count) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_base;
    const int W = cam.width, H = cam.height;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    for (int c0 = 0; c0 < nk; c0 += GD_THREADS) {
        const int k = c0 + threadIdx.x;
        bool ok = k < nk && !active[k];
        float u = 0.f, v = 0.f;
        int px = 0, py = 0;
        double d = 0.0;
        if (ok) {
            const float2 p = uv[k];
            u = p.x;
            v = p.y;
            px = __float2int_rn(u);
            py = __float2int_rn(v);
            ok = px >= 0 && px < W && py >= 0 && py < H;
        }
        if (ok && mode == 1) {
            d = depth_map[(int64_t)py * W + px];
            ok = d > 0.0;
        } else if (ok) {
            // K = 4 nearest active keypoints within rho (fp32 squared distances, ties by index)
            int best[4];
            float bd[4];
            int nb = 0;
            const float r2 = __fmul_rn(rho, rho);
            for (int j = 0; j < nk; j++) {
                if (!active[j]) continue;
                const float2 q = uv[j];
                const float dx = __fsub_rn(q.x, u), dy = __fsub_rn(q.y, v);
                const float d2 = __fmaf_rn(dx, dx, __fmul_rn(dy, dy));
                if (!(d2 <= r2)) continue;
                int pos = nb;
                while (pos > 0 && d2 < bd[pos - 1]) pos--;
                if (pos >= 4) continue;
                for (int t = (nb < 4 ? nb : 3); t > pos; t--) {
                    bd[t] = bd[t - 1];
                    best[t] = best[t - 1];
                }
                bd[pos] = d2;
                best[pos] = j;
                if (nb < 4) nb++;
            }
            ok = nb > 0;
            if (ok) {
                double sw = 0.0, swd = 0.0, zsum = 0.0;
                int nz = 0;
                for (int t = 0; t < nb; t++) {
                    if (bd[t] == 0.f) {
                        zsum += kp_depth[best[t]];
                        nz++;
                    }
                    const double w = 1.0 / sqrt((double)bd[t]);
                    sw += w;
                    swd += w * kp_depth[best[t]];
                }
                d = nz ? zsum / nz : swd / sw;
            }
        }
        // block-wide exclusive scan of the decisions -> rows in keypoint order
        const unsigned b = __ballot_sync(0xffffffffu, ok);
        if (lane == 0) s_warp[warp] = __popc(b);
        __syncthreads();
        if (warp == 0) {
            const uint32_t w = s_warp[lane];
            uint32_t incl = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += x;
            }
            s_warp[lane] = incl - w;
        }
        __syncthreads();
        const uint32_t row = s_base + s_warp[warp] + __popc(b & ((1u << lane) - 1u));
        if (ok) {
            const double xc[3] = {d * ((double)u - cam.cx) / cam.fx, d * ((double)v - cam.cy) / cam.fy, d};
            for (int a = 0; a < 3; a++) {  // P = R^T (p_c - t)
                double s = 0.0;
                for (int bb = 0; bb < 3; bb++) s += (double)cam.R[3 * bb + a] * (xc[bb] - (double)cam.t[bb]);
                out[a * ldo + row] = (float)s;
            }
            out[3 * ldo + row] = 1.f;
            out[4 * ldo + row] = out[5 * ldo + row] = out[6 * ldo + row] = 0.f;
            const float ls = (float)log(d / cam.fx);
            out[7 * ldo + row] = out[8 * ldo + row] = out[9 * ldo + row] = ls;
            out[10 * ldo + row] = (float)log(0.1 / 0.9);
            for (int ch = 0; ch < 3; ch++)
                out[(11 + ch) * ldo + row] =
                    (float)(((double)image[(int64_t)ch * H * W + (int64_t)py * W + px] - 0.5) / 0.28209479177387814);
            for (int r = 14; r < K; r++) out[r * ldo + row] = 0.f;
            src[row] = k;
        }
        __syncthreads();
        if (threadIdx.x == GD_THREADS - 1) s_base = row + (ok ? 1u : 0u);
        __syncthreads();
    }
    if (threadIdx.x == 0) *count = (int32_t)s_base;
}

cudaError_t launch_geometry_densify(const gs_camera &cam, const float *uv, const int32_t *active, const float *kp_depth,
                                    const float *depth_map, const float *image, int nk, int mode, float rho,
                                    const gs_params &out, int32_t *src, int32_t *count, cudaStream_t s) {
    k_geometry_densify<<<1, GD_THREADS, 0, s>>>(cam, reinterpret_cast<const float2 *>(uv), active, kp_depth, depth_map,
                                                image, nk, mode, rho, gs_param_rows(out.sh_degree), out.data, out.ld,
                                                src, count);
    return cudaGetLastError();
}

}  // namespace gsk
