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
