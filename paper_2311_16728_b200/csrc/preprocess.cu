// preprocess.cu -- A1 (projection, EWA covariance, SH colour) and A9 (its backward).
//
// A1 follows PAPER.md:178 (alpha_i = sigma_i * G(R, t, P_i, r_i, s_i), G = 3DGS EWA
// splatting) and SPEC.md:315-343; the decision quantities (culling, depth, mean2d, conic,
// radius, tile rect) follow the fp32 decision recipe of DESIGN.md exactly -- IEEE ops with
// explicit __fmaf_rn / __fmul_rn / __fadd_rn / __fdiv_rn / __fsqrt_rn so that nvcc cannot
// contract or approximate them -- which makes tile binning and sort order bit-exact to the
// CPU oracle.  One thread per Gaussian loops over the views of the batch, so the 4K bytes of
// parameters per Gaussian are read from HBM once per call (K1).
//
// A9 is the chain rule of SPEC.md:358 from the per-(view, Gaussian) 2D gradients that the
// raster backward accumulated to dL/d{P, q, log s, logit sigma, SH}, summed over the views
// (R22) and added to the caller's gradient buffer.
#include "gs_internal.cuh"


namespace gsk {

#define FMA __fmaf_rn
#define MUL __fmul_rn
#define ADD __fadd_rn
#define SUB __fsub_rn
#define DIV __fdiv_rn
#define SQRT __fsqrt_rn

__device__ __forceinline__ float dot3(float a0, float a1, float a2, float b0, float b1, float b2) {
    return FMA(a2, b2, FMA(a1, b1, MUL(a0, b0)));
}

// Real SH basis to degree D (sign convention of the cited renderer).
// Constants: sqrt(1/4pi), sqrt(3/4pi), sqrt(15/4pi), 1/4 sqrt(5/pi), 1/4 sqrt(15/pi),
// 1/4 sqrt(35/2pi), 1/2 sqrt(105/pi), 1/4 sqrt(21/2pi), 1/4 sqrt(7/pi), 1/4 sqrt(105/pi).
#define SH_C0 0.28209479177387814f
#define SH_C1 0.4886025119029199f
#define SH_C2A 1.0925484305920792f
#define SH_C2B 0.31539156525252005f
#define SH_C2C 0.5462742152960396f
#define SH_C3A 0.5900435899266435f
#define SH_C3B 2.890611442640554f
#define SH_C3C 0.4570457994644658f
#define SH_C3D 0.3731763325901154f
#define SH_C3E 1.445305721320277f

template <int D>
__device__ __forceinline__ void sh_basis(float x, float y, float z, float Y[16]) {
    Y[0] = SH_C0;
    if (D >= 1) {
        Y[1] = -SH_C1 * y;
        Y[2] = SH_C1 * z;
        Y[3] = -SH_C1 * x;
    }
    if (D >= 2) {
        float xx = x * x, yy = y * y, zz = z * z;
        Y[4] = SH_C2A * x * y;
        Y[5] = -SH_C2A * y * z;
        Y[6] = SH_C2B * (2.f * zz - xx - yy);
        Y[7] = -SH_C2A * x * z;
        Y[8] = SH_C2C * (xx - yy);
        if (D >= 3) {
            Y[9] = -SH_C3A * y * (3.f * xx - yy);
            Y[10] = SH_C3B * x * y * z;
            Y[11] = -SH_C3C * y * (4.f * zz - xx - yy);
            Y[12] = SH_C3D * z * (2.f * zz - 3.f * xx - 3.f * yy);
            Y[13] = -SH_C3C * x * (4.f * zz - xx - yy);
            Y[14] = SH_C3E * z * (xx - yy);
            Y[15] = -SH_C3A * x * (xx - 3.f * yy);
        }
    }
}

// d(sum_l c_l Y_l)/d(x,y,z) for coefficient vector c (one colour channel)
template <int D>
__device__ __forceinline__ void sh_grad_dir(float x, float y, float z, const float c[16], float g[3]) {
    g[0] = g[1] = g[2] = 0.f;
    if (D >= 1) {
        g[0] += -SH_C1 * c[3];
        g[1] += -SH_C1 * c[1];
        g[2] += SH_C1 * c[2];
    }
    if (D >= 2) {
        g[0] += SH_C2A * y * c[4] - SH_C2A * z * c[7] - 2.f * SH_C2B * x * c[6] + 2.f * SH_C2C * x * c[8];
        g[1] += SH_C2A * x * c[4] - SH_C2A * z * c[5] - 2.f * SH_C2B * y * c[6] - 2.f * SH_C2C * y * c[8];
        g[2] += -SH_C2A * y * c[5] + 4.f * SH_C2B * z * c[6] - SH_C2A * x * c[7];
        if (D >= 3) {
            float xx = x * x, yy = y * y, zz = z * z;
            g[0] += -SH_C3A * 6.f * x * y * c[9] + SH_C3B * y * z * c[10] + SH_C3C * 2.f * x * y * c[11] -
                    SH_C3D * 6.f * x * z * c[12] - SH_C3C * (4.f * zz - 3.f * xx - yy) * c[13] +
                    SH_C3E * 2.f * x * z * c[14] - SH_C3A * (3.f * xx - 3.f * yy) * c[15];
            g[1] += -SH_C3A * (3.f * xx - 3.f * yy) * c[9] + SH_C3B * x * z * c[10] -
                    SH_C3C * (4.f * zz - xx - 3.f * yy) * c[11] - SH_C3D * 6.f * y * z * c[12] +
                    SH_C3C * 2.f * x * y * c[13] - SH_C3E * 2.f * y * z * c[14] + SH_C3A * 6.f * x * y * c[15];
            g[2] += SH_C3B * x * y * c[10] - SH_C3C * 8.f * y * z * c[11] +
                    SH_C3D * (6.f * zz - 3.f * xx - 3.f * yy) * c[12] - SH_C3C * 8.f * x * z * c[13] +
                    SH_C3E * (xx - yy) * c[14];
        }
    }
}

// View-independent part of the recipe: normalised quaternion, R(q), e^s, Sigma3.
struct Cov3 {
    bool ok;
    float qn[4], inv_norm;
    float Rq[9], e[3], M[9];
    float S00, S01, S02, S11, S12, S22;
};

__device__ __forceinline__ Cov3 cov3_recipe(float q0, float q1, float q2, float q3, float s0, float s1, float s2) {
    Cov3 c;
    float d4 = FMA(q3, q3, FMA(q2, q2, FMA(q1, q1, MUL(q0, q0))));
    c.ok = d4 != 0.0f;
    float inv = DIV(1.0f, SQRT(d4));
    c.inv_norm = inv;
    float w = MUL(q0, inv), x = MUL(q1, inv), y = MUL(q2, inv), z = MUL(q3, inv);
    c.qn[0] = w; c.qn[1] = x; c.qn[2] = y; c.qn[3] = z;
    c.Rq[0] = SUB(1.0f, MUL(2.0f, FMA(y, y, MUL(z, z))));
    c.Rq[1] = MUL(2.0f, FMA(x, y, -MUL(w, z)));
    c.Rq[2] = MUL(2.0f, FMA(x, z, MUL(w, y)));
    c.Rq[3] = MUL(2.0f, FMA(x, y, MUL(w, z)));
    c.Rq[4] = SUB(1.0f, MUL(2.0f, FMA(x, x, MUL(z, z))));
    c.Rq[5] = MUL(2.0f, FMA(y, z, -MUL(w, x)));
    c.Rq[6] = MUL(2.0f, FMA(x, z, -MUL(w, y)));
    c.Rq[7] = MUL(2.0f, FMA(y, z, MUL(w, x)));
    c.Rq[8] = SUB(1.0f, MUL(2.0f, FMA(x, x, MUL(y, y))));
    c.e[0] = (float)exp((double)s0);  // recipe: (float)exp((double)s)
    c.e[1] = (float)exp((double)s1);
    c.e[2] = (float)exp((double)s2);
#pragma unroll
    for (int r = 0; r < 3; r++)
#pragma unroll
        for (int k = 0; k < 3; k++) c.M[3 * r + k] = MUL(c.Rq[3 * r + k], c.e[k]);
    const float *M = c.M;
    c.S00 = dot3(M[0], M[1], M[2], M[0], M[1], M[2]);
    c.S01 = dot3(M[0], M[1], M[2], M[3], M[4], M[5]);
    c.S02 = dot3(M[0], M[1], M[2], M[6], M[7], M[8]);
    c.S11 = dot3(M[3], M[4], M[5], M[3], M[4], M[5]);
    c.S12 = dot3(M[3], M[4], M[5], M[6], M[7], M[8]);
    c.S22 = dot3(M[6], M[7], M[8], M[6], M[7], M[8]);
    return c;
}

// Per-view part of the recipe.
struct Proj {
    bool ok;
    float pc[3], z, tx, ty, txc, tyc;
    bool clx, cly;
    float T0[3], T1[3];
    float a, b, c, det, A, B, C, u, v;
    int r, x0, y0, x1, y1;
};

__device__ __forceinline__ Proj project_recipe(const gs_camera &cam, float px, float py, float pz, const Cov3 &cv,
                                               int TX, int TY) {
    Proj p;
    p.ok = false;
    const float *R = cam.R;
    p.pc[0] = ADD(dot3(R[0], R[1], R[2], px, py, pz), cam.t[0]);
    p.pc[1] = ADD(dot3(R[3], R[4], R[5], px, py, pz), cam.t[1]);
    p.pc[2] = ADD(dot3(R[6], R[7], R[8], px, py, pz), cam.t[2]);
    float z = p.pc[2];
    p.z = z;
    if (!(z > cam.znear) || !cv.ok) return p;
    float tx = DIV(p.pc[0], z), ty = DIV(p.pc[1], z);
    p.tx = tx; p.ty = ty;
    p.txc = fminf(fmaxf(tx, -cam.lim_x), cam.lim_x);
    p.tyc = fminf(fmaxf(ty, -cam.lim_y), cam.lim_y);
    p.clx = (tx < -cam.lim_x) || (tx > cam.lim_x);
    p.cly = (ty < -cam.lim_y) || (ty > cam.lim_y);
    float J00 = DIV(cam.fx, z), J02 = DIV(-MUL(cam.fx, p.txc), z);
    float J11 = DIV(cam.fy, z), J12 = DIV(-MUL(cam.fy, p.tyc), z);
#pragma unroll
    for (int j = 0; j < 3; j++) {
        p.T0[j] = FMA(J02, R[6 + j], MUL(J00, R[j]));
        p.T1[j] = FMA(J12, R[6 + j], MUL(J11, R[3 + j]));
    }
    // U = T Sigma3 (column j of Sigma3 = (S0j, S1j, S2j))
    float U00 = dot3(p.T0[0], p.T0[1], p.T0[2], cv.S00, cv.S01, cv.S02);
    float U01 = dot3(p.T0[0], p.T0[1], p.T0[2], cv.S01, cv.S11, cv.S12);
    float U02 = dot3(p.T0[0], p.T0[1], p.T0[2], cv.S02, cv.S12, cv.S22);
    float U10 = dot3(p.T1[0], p.T1[1], p.T1[2], cv.S00, cv.S01, cv.S02);
    float U11 = dot3(p.T1[0], p.T1[1], p.T1[2], cv.S01, cv.S11, cv.S12);
    float U12 = dot3(p.T1[0], p.T1[1], p.T1[2], cv.S02, cv.S12, cv.S22);
    float a = ADD(dot3(U00, U01, U02, p.T0[0], p.T0[1], p.T0[2]), 0.3f);
    float b = dot3(U00, U01, U02, p.T1[0], p.T1[1], p.T1[2]);
    float c = ADD(dot3(U10, U11, U12, p.T1[0], p.T1[1], p.T1[2]), 0.3f);
    p.a = a; p.b = b; p.c = c;
    float det = FMA(-b, b, MUL(a, c));
    p.det = det;
    if (!(det > 0.0f)) return p;
    float idet = DIV(1.0f, det);
    p.A = MUL(c, idet); p.B = MUL(-b, idet); p.C = MUL(a, idet);
    float mid = MUL(0.5f, ADD(a, c));
    float lam = ADD(mid, SQRT(fmaxf(0.0f, FMA(mid, mid, -det))));
    p.r = (int)ceilf(MUL(3.0f, SQRT(lam)));
    p.u = FMA(cam.fx, tx, cam.cx);
    p.v = FMA(cam.fy, ty, cam.cy);
    float rf = (float)p.r, fTX = (float)TX, fTY = (float)TY;
    p.x0 = (int)fminf(fmaxf(floorf(MUL(SUB(p.u, rf), 0.0625f)), 0.0f), fTX);
    p.x1 = (int)fminf(fmaxf(ADD(floorf(MUL(ADD(p.u, rf), 0.0625f)), 1.0f), 0.0f), fTX);
    p.y0 = (int)fminf(fmaxf(floorf(MUL(SUB(p.v, rf), 0.0625f)), 0.0f), fTY);
    p.y1 = (int)fminf(fmaxf(ADD(floorf(MUL(ADD(p.v, rf), 0.0625f)), 1.0f), 0.0f), fTY);
    p.ok = (p.x1 - p.x0) * (p.y1 - p.y0) != 0;
    return p;
}

__device__ __forceinline__ void cam_centre(const gs_camera &cam, float C[3]) {
#pragma unroll
    for (int k = 0; k < 3; k++) C[k] = -(cam.R[k] * cam.t[0] + cam.R[3 + k] * cam.t[1] + cam.R[6 + k] * cam.t[2]);
}

// SH colour of a Gaussian at (px, py, pz) seen from cam: c = max(0, sum_l SH_l Y_l(dir) + 0.5),
// dir = normalize(P - C_cam) (R6); shc = its 3 NC coefficients, [l][channel]
template <int D>
__device__ __forceinline__ void sh_colour(const gs_camera &cam, float px, float py, float pz, const float *shc,
                                          float rgb[3]) {
    constexpr int NC = (D + 1) * (D + 1);
    float Cc[3];
    cam_centre(cam, Cc);
    float dx = px - Cc[0], dy = py - Cc[1], dz = pz - Cc[2];
    float inv = rsqrtf(dx * dx + dy * dy + dz * dz);
    float Y[16];
    sh_basis<D>(dx * inv, dy * inv, dz * inv, Y);
#pragma unroll
    for (int ch = 0; ch < 3; ch++) {
        float acc = 0.5f;
#pragma unroll
        for (int l = 0; l < NC; l++) acc += shc[3 * l + ch] * Y[l];
        rgb[ch] = fmaxf(acc, 0.0f);
    }
}

template <int D, bool SPLIT>
__device__ __forceinline__ void preprocess_one(const float *__restrict__ P, int64_t n, int64_t ld,
                                               const CamBatch &cams, int V, const Layout &L, char *ws,
                                               bool count_tiles, bool smem_cnt, uint32_t *s_cnt, int64_t i) {
    constexpr int NC = (D + 1) * (D + 1);
    // SPLIT (one or two views): two phases, the geometry of every view first (rows 0..10), then
    // -- only for a Gaussian visible in some view -- its 3 NC SH coefficients and the colour of
    // its visible views, so the SH registers are never live together with the projection's
    // (79 instead of 123 registers at D = 3: more warps in flight for this latency-bound kernel).
    // Otherwise one phase with every load issued before the projection chain: with many views
    // the records outgrow L2 and the split's two half-record writes per (view, Gaussian) cost
    // more than the occupancy gains (A1).
    uint64_t vis_views = 0;
    float shc[SPLIT ? 1 : 3 * NC];
    if constexpr (!SPLIT) {
#pragma unroll
        for (int k = 0; k < 3 * NC; k++) shc[k] = P[(11 + k) * ld + i];
    }
    float px = P[i], py = P[ld + i], pz = P[2 * ld + i];
    Cov3 cv = cov3_recipe(P[3 * ld + i], P[4 * ld + i], P[5 * ld + i], P[6 * ld + i], P[7 * ld + i], P[8 * ld + i],
                          P[9 * ld + i]);
    float op = P[10 * ld + i];
    float sigma = 1.0f / (1.0f + expf(-op));
    float4 *rec0 = at<float4>(ws, L.rec0);
    float4 *rec1 = at<float4>(ws, L.rec1);
    float4 *rec2 = at<float4>(ws, L.rec2);
    float *depth = at<float>(ws, L.depth);
    int32_t *radius = at<int32_t>(ws, L.radius);
    int4 *rect = at<int4>(ws, L.rect);
    uint32_t *tt = at<uint32_t>(ws, L.tiles_touched);
    float4 *g2d = at<float4>(ws, L.grad2d);
    bool any_vis = false;
    for (int v = 0; v < V; v++) {
        const gs_camera &cam = cams.c[v];
        int64_t m = (int64_t)v * n + i;
        Proj p = project_recipe(cam, px, py, pz, cv, L.TX, L.TY);
        if (!p.ok) {
            radius[m] = 0;
            tt[m] = 0;
            continue;
        }
        any_vis = true;
        vis_views |= 1ull << v;
        rec0[m] = make_float4(p.u, p.v, p.A, p.B);
        // padded exact 3-sigma extents of the ellipse d^T Q d <= 9 (Q^-1 = Sigma2' = [[a, b], [b, c]]):
        // used by the raster kernels for a conservative warp-level skip test
        const float ea = 3.0f * sqrtf(p.a) * 1.0001f + 1e-3f, ec = 3.0f * sqrtf(p.c) * 1.0001f + 1e-3f;
        if constexpr (SPLIT) {  // rec1.zw, rec2.x: the colour, phase 2
            reinterpret_cast<float2 *>(rec1 + m)[0] = make_float2(p.C, sigma);
            reinterpret_cast<float *>(rec2 + m)[1] = ea;
            reinterpret_cast<float2 *>(rec2 + m)[1] = make_float2(ec, 0.f);
        } else {
            float rgb[3];
            sh_colour<D>(cam, px, py, pz, shc, rgb);
            rec1[m] = make_float4(p.C, sigma, rgb[0], rgb[1]);
            rec2[m] = make_float4(rgb[2], ea, ec, 0.f);
        }
        depth[m] = p.z;
        radius[m] = p.r;
        rect[m] = make_int4(p.x0, p.y0, p.x1, p.y1);
        // pairs: the tiles of the rect the 3-sigma ellipse can reach (R10'); with the bucket
        // binning also the per-(view, tile) pair counts (bin.cu)
        // (rects of <= 64 tiles keep the hit mask for the key emission, bit = row-major rect index)
        uint32_t hits = 0;
        uint64_t mask = 0;
        const int tb = v * L.tiles;
        const int rw = p.x1 - p.x0;
        uint32_t *tc = at<uint32_t>(ws, L.tile_count);
        float rA, rC;
        ellipse_recips(p.A, p.C, rA, rC);
        for (int ty = p.y0; ty < p.y1; ty++)
            for (int tx = p.x0; tx < p.x1; tx++) {
                if (!tile_hits_ellipse(p.u, p.v, p.A, p.B, p.C, rA, rC, tx, ty)) continue;
                hits++;
                const int bit = (ty - p.y0) * rw + (tx - p.x0);
                if (bit < 64) mask |= 1ull << bit;
                if (count_tiles) {
                    const int b = tb + ty * L.TX + tx;
                    if (smem_cnt) atomicAdd(&s_cnt[b], 1u);
                    else atomicAdd(&tc[(size_t)b * CNT_STRIDE], 1u);
                }
            }
        tt[m] = hits;
        at<uint64_t>(ws, L.tile_mask)[m] = mask;
        float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
        g2d[3 * m] = zero;
        g2d[3 * m + 1] = zero;
        g2d[3 * m + 2] = zero;
    }
    // phase 2 (SPLIT): the SH colour of the visible views
    if (SPLIT && vis_views) {
        float sh2[3 * NC];
#pragma unroll
        for (int k = 0; k < 3 * NC; k++) sh2[k] = P[(11 + k) * ld + i];
        do {
            const int v = __ffsll((long long)vis_views) - 1;
            vis_views &= vis_views - 1;
            const int64_t m = (int64_t)v * n + i;
            float rgb[3];
            sh_colour<D>(cams.c[v], px, py, pz, sh2, rgb);
            reinterpret_cast<float2 *>(rec1 + m)[1] = make_float2(rgb[0], rgb[1]);
            reinterpret_cast<float *>(rec2 + m)[0] = rgb[2];
        } while (vis_views);
    }
    // compacted list of Gaussians visible in some view (warp-aggregated append) so that the
    // backward chain runs on full warps of visible Gaussians only
    unsigned active = __activemask();
    unsigned mask = __ballot_sync(active, any_vis);
    uint32_t slot = 0xFFFFFFFFu;
    if (mask) {
        int lane = threadIdx.x & 31;
        int leader = __ffs(mask) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(&at<WsHeader>(ws, L.hdr)->vis_count, (uint32_t)__popc(mask));
        base = __shfl_sync(active, base, leader);
        if (any_vis) {
            slot = base + __popc(mask & ((1u << lane) - 1u));
            at<uint32_t>(ws, L.vis_list)[slot] = (uint32_t)i;
        }
    }
    at<uint32_t>(ws, L.slot)[i] = slot;
}

template <int D, bool SPLIT>
__global__ void __launch_bounds__(256) k_preprocess(const float *__restrict__ P, int64_t n, int64_t ld,
                                                    const CamBatch cams, int V, Layout L, char *ws,
                                                    bool count_tiles) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    __shared__ uint32_t s_cnt[SMEM_BINS];
    const int VT = V * L.tiles;
    const bool smem_cnt = count_tiles && VT <= SMEM_BINS;  // uniform
    if (smem_cnt) {
        for (int b = threadIdx.x; b < VT; b += blockDim.x) s_cnt[b] = 0;
        __syncthreads();
    }
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) preprocess_one<D, SPLIT>(P, n, ld, cams, V, L, ws, count_tiles, smem_cnt, s_cnt, i);
    if (smem_cnt) {  // one global add per (CTA, tile) into the padded counters
        __syncthreads();
        uint32_t *tc = at<uint32_t>(ws, L.tile_count);
        for (int b = threadIdx.x; b < VT; b += blockDim.x) {
            uint32_t c = s_cnt[b];
            if (c) atomicAdd(&tc[(size_t)b * CNT_STRIDE], c);
        }
    }
}


// ---------------------------------------------------------------------------------------------
// A9: chain rule from the per-(view, Gaussian) 2D gradients (u, v, A, B, C, sigma, r, g, b) to
// the parameters, in fp32.
// One thread per visible Gaussian (compacted list entry t): the chain of all views is summed
// and written to column t of the scratch (row r = parameter row r), coalesced across the warp.
template <int D>
__global__ void __launch_bounds__(128) k_preprocess_bwd(const float *__restrict__ P, int64_t n, int64_t ld,
                                                        const CamBatch cams, int V, Layout L, char *ws,
                                                        float *__restrict__ gnorm, int64_t *step_inc) {
    pdl_wait();  // PDL: the predecessor grid has completed (gs_internal.cuh)
    pdl_trigger();
    constexpr int NC = (D + 1) * (D + 1);
    if (step_inc && blockIdx.x == 0 && threadIdx.x == 0) *step_inc += 1;  // device step for the fused Adam
    const uint32_t nvis = at<WsHeader>(ws, L.hdr)->vis_count;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nvis) return;
    const int64_t i = at<const uint32_t>(ws, L.vis_list)[t];
    const int32_t *radius = at<const int32_t>(ws, L.radius);
    float4 *g2d = at<float4>(ws, L.grad2d);
    float *S = at<float>(ws, L.scratch);  // [row][n], column t
    // loads whose values are needed only late, issued up front (the kernel is latency-bound)
    const float gnorm_old = gnorm ? gnorm[i] : 0.f;
    // rendered views 0..63 (bit v: radius > 0), one pass of independent loads; views >= 64 test
    // the radius again
    uint64_t vm = 0;
#pragma unroll 8
    for (int v = 0; v < min(V, 64); v++) vm |= (uint64_t)(radius[(int64_t)v * n + i] > 0) << v;
#define RENDERED(v, m) ((v) < 64 ? ((vm >> (v)) & 1ull) != 0 : radius[m] > 0)
    float px = P[i], py = P[ld + i], pz = P[2 * ld + i];
    Cov3 cv = cov3_recipe(P[3 * ld + i], P[4 * ld + i], P[5 * ld + i], P[6 * ld + i], P[7 * ld + i], P[8 * ld + i],
                          P[9 * ld + i]);
    float op = P[10 * ld + i];
    float sig = 1.0f / (1.0f + expf(-op));
    float gP[3] = {0.f, 0.f, 0.f}, gR[9], gs[3] = {0.f, 0.f, 0.f}, gop = 0.f;
#pragma unroll
    for (int k = 0; k < 9; k++) gR[k] = 0.f;
    float norm_acc = 0.f;
    const float S3[9] = {cv.S00, cv.S01, cv.S02, cv.S01, cv.S11, cv.S12, cv.S02, cv.S12, cv.S22};
    float GS3a[9];  // dL/dSigma3 summed over the views
#pragma unroll
    for (int k = 0; k < 9; k++) GS3a[k] = 0.f;
    // ---- geometry: conic -> Sigma2 -> (Sigma3, J) -> (q, s), mean2d -> P
    for (int v = 0; v < V; v++) {
        int64_t m = (int64_t)v * n + i;
        if (!RENDERED(v, m)) continue;
        const gs_camera &cam = cams.c[v];
        Proj p = project_recipe(cam, px, py, pz, cv, L.TX, L.TY);
        float4 ga = g2d[3 * m], gb = g2d[3 * m + 1];
        // the raster backward accumulated moments over pixels: S(a), S(b), S(a dx), S(a dy),
        // S(b dy) with a = dL/dpower dx, b = dL/dpower dy (d = pixel - mean2d); with the conic
        // (A, B, C) of this view: dL/du = A S(a) + B S(b), dL/dv = B S(a) + C S(b),
        // dL/dA = -S(a dx)/2, dL/dB = -S(a dy), dL/dC = -S(b dy)/2
        float A = p.A, B = p.B, C = p.C;
        float gu = A * ga.x + B * ga.y, gv = B * ga.x + C * ga.y;
        float gA = -0.5f * ga.z, gB = -ga.w, gC = -0.5f * gb.x;
        gop += gb.y;
        norm_acc += sqrtf(gu * gu + gv * gv);
        // conic Q = Sigma2'^-1 : dL/dSigma2 = -Q G Q, G = [[gA, gB/2], [gB/2, gC]]
        float hB = 0.5f * gB;
        float QG00 = A * gA + B * hB, QG01 = A * hB + B * gC;
        float QG10 = B * gA + C * hB, QG11 = B * hB + C * gC;
        float H00 = -(QG00 * A + QG01 * B);
        float H01 = -(QG00 * B + QG01 * C);
        float H11 = -(QG10 * B + QG11 * C);
        // HT = H T (2x3), T rows T0, T1
        float HT0[3], HT1[3];
#pragma unroll
        for (int c = 0; c < 3; c++) {
            HT0[c] = H00 * p.T0[c] + H01 * p.T1[c];
            HT1[c] = H01 * p.T0[c] + H11 * p.T1[c];
        }
        // dL/dSigma3 = T^T H T (symmetric)
        float GS3[9];
#pragma unroll
        for (int r = 0; r < 3; r++)
#pragma unroll
            for (int c = 0; c < 3; c++) GS3[3 * r + c] = p.T0[r] * HT0[c] + p.T1[r] * HT1[c];
        // dL/dT = 2 H T Sigma3
        float GT0[3], GT1[3];
#pragma unroll
        for (int c = 0; c < 3; c++) {
            GT0[c] = 2.f * (HT0[0] * S3[c] + HT0[1] * S3[3 + c] + HT0[2] * S3[6 + c]);
            GT1[c] = 2.f * (HT1[0] * S3[c] + HT1[1] * S3[3 + c] + HT1[2] * S3[6 + c]);
        }
        // dL/dJ = dL/dT W^T (W = camera R); only J00, J02, J11, J12 vary
        const float *W = cam.R;
        float GJ00 = GT0[0] * W[0] + GT0[1] * W[1] + GT0[2] * W[2];
        float GJ02 = GT0[0] * W[6] + GT0[1] * W[7] + GT0[2] * W[8];
        float GJ11 = GT1[0] * W[3] + GT1[1] * W[4] + GT1[2] * W[5];
        float GJ12 = GT1[0] * W[6] + GT1[1] * W[7] + GT1[2] * W[8];
        float z = p.z, x = p.pc[0], y = p.pc[1], fx = cam.fx, fy = cam.fy;
        float iz = 1.f / z, iz2 = iz * iz;
        float gpc0 = 0.f, gpc1 = 0.f, gpc2 = 0.f;
        gpc2 += -fx * iz2 * GJ00 - fy * iz2 * GJ11;
        if (!p.clx) {
            gpc0 += -fx * iz2 * GJ02;
            gpc2 += 2.f * fx * x * iz2 * iz * GJ02;
        } else {
            gpc2 += fx * p.txc * iz2 * GJ02;
        }
        if (!p.cly) {
            gpc1 += -fy * iz2 * GJ12;
            gpc2 += 2.f * fy * y * iz2 * iz * GJ12;
        } else {
            gpc2 += fy * p.tyc * iz2 * GJ12;
        }
        // mean2d u = fx x/z + cx
        gpc0 += gu * fx * iz;
        gpc1 += gv * fy * iz;
        gpc2 += -(gu * fx * x + gv * fy * y) * iz2;
        // p_c = W P + t
#pragma unroll
        for (int k = 0; k < 3; k++) gP[k] += W[k] * gpc0 + W[3 + k] * gpc1 + W[6 + k] * gpc2;
        // dL/dSigma3 is of the world-frame covariance: summed over the views, then taken
        // through Sigma3 = M M^T once after the loop (linear in it)
#pragma unroll
        for (int k = 0; k < 9; k++) GS3a[k] += GS3[k];
    }
    {
        const float *GS3 = GS3a;
        // Sigma3 = M M^T: dL/dM = 2 GS3 M ; M = Rq diag(e)
#pragma unroll
        for (int r = 0; r < 3; r++)
#pragma unroll
            for (int j = 0; j < 3; j++) {
                float gm = 2.f * (GS3[3 * r] * cv.M[j] + GS3[3 * r + 1] * cv.M[3 + j] + GS3[3 * r + 2] * cv.M[6 + j]);
                gs[j] += gm * cv.Rq[3 * r + j] * cv.e[j];  // d/dlog s = e d/de
                gR[3 * r + j] += gm * cv.e[j];
            }
    }
    // ---- SH colour, one channel at a time: c = max(0, sum_l SH_l Y_l(dir) + 0.5) (R6)
#pragma unroll 1
    for (int ch = 0; ch < 3; ch++) {
        float c[16], acc_sh[16];
#pragma unroll
        for (int l = 0; l < NC; l++) {
            c[l] = P[(11 + 3 * l + ch) * ld + i];
            acc_sh[l] = 0.f;
        }
        for (int v = 0; v < V; v++) {
            int64_t m = (int64_t)v * n + i;
            if (!RENDERED(v, m)) continue;
            const float *gcol4 = reinterpret_cast<const float *>(g2d + 3 * m);
            float gcol = gcol4[6 + ch];  // record [.. | C, sigma, r, g | b ..]
            float Cc[3];
            cam_centre(cams.c[v], Cc);
            float dx = px - Cc[0], dy = py - Cc[1], dz = pz - Cc[2];
            float nd = sqrtf(dx * dx + dy * dy + dz * dz), ind = 1.f / nd;
            float dir[3] = {dx * ind, dy * ind, dz * ind};
            float Y[16];
            sh_basis<D>(dir[0], dir[1], dir[2], Y);
            float a = 0.5f;
#pragma unroll
            for (int l = 0; l < NC; l++) a += c[l] * Y[l];
            if (a < 0.f) continue;  // clamped channel: zero gradient
#pragma unroll
            for (int l = 0; l < NC; l++) acc_sh[l] += Y[l] * gcol;
            if (D > 0) {
                float gd[3];
                sh_grad_dir<D>(dir[0], dir[1], dir[2], c, gd);
                float dd = dir[0] * gd[0] + dir[1] * gd[1] + dir[2] * gd[2];
#pragma unroll
                for (int k = 0; k < 3; k++) gP[k] += gcol * (gd[k] - dir[k] * dd) * ind;
            }
        }
#pragma unroll
        for (int l = 0; l < NC; l++) S[(11 + 3 * l + ch) * n + t] = acc_sh[l];
    }
    // consumed: reset the 2D records so a repeated backward on the same forward starts from 0
    for (int v = 0; v < V; v++) {
        int64_t m = (int64_t)v * n + i;
        if (RENDERED(v, m)) g2d[3 * m] = g2d[3 * m + 1] = g2d[3 * m + 2] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
#undef RENDERED
    // quaternion: dL/dq_hat from dL/dRq, then through the normalisation
    float w_ = cv.qn[0], qx = cv.qn[1], qy = cv.qn[2], qz = cv.qn[3];
    const float *g = gR;
    float gq0 = 2.f * (-qz * g[1] + qy * g[2] + qz * g[3] - qx * g[5] - qy * g[6] + qx * g[7]);
    float gq1 = 2.f * (qy * g[1] + qz * g[2] + qy * g[3] - 2.f * qx * g[4] - w_ * g[5] + qz * g[6] + w_ * g[7] -
                       2.f * qx * g[8]);
    float gq2 = 2.f * (-2.f * qy * g[0] + qx * g[1] + w_ * g[2] + qx * g[3] + qz * g[5] - w_ * g[6] + qz * g[7] -
                       2.f * qy * g[8]);
    float gq3 = 2.f * (-2.f * qz * g[0] - w_ * g[1] + qx * g[2] + w_ * g[3] - 2.f * qz * g[4] + qy * g[5] + qx * g[6] +
                       qy * g[7]);
    float dotg = w_ * gq0 + qx * gq1 + qy * gq2 + qz * gq3;
    float in = cv.inv_norm;
    S[0 * n + t] = gP[0];
    S[1 * n + t] = gP[1];
    S[2 * n + t] = gP[2];
    S[3 * n + t] = (gq0 - w_ * dotg) * in;
    S[4 * n + t] = (gq1 - qx * dotg) * in;
    S[5 * n + t] = (gq2 - qy * dotg) * in;
    S[6 * n + t] = (gq3 - qz * dotg) * in;
    S[7 * n + t] = gs[0];
    S[8 * n + t] = gs[1];
    S[9 * n + t] = gs[2];
    S[10 * n + t] = sig * (1.f - sig) * gop;
    if (gnorm) gnorm[i] = gnorm_old + norm_acc;
}

// the two-phase A1 (geometry, then SH colour) up to this many views per call (measured: TUM
// +2.6 %, EuRoC even, the 64-view stress step -1.6 %)
constexpr int SPLIT_MAX_VIEWS = 2;

template <int D>
static void launch_pre(bool split, int64_t blocks, cudaStream_t s, const gs_params &p, const CamBatch &cams, int V,
                       const Layout &L, void *ws, bool count_tiles) {
    if (split)
        launch_pdl(k_preprocess<D, true>, blocks, 256, 0, s, p.data, p.n, p.ld, cams, V, L, (char *)ws, count_tiles);
    else
        launch_pdl(k_preprocess<D, false>, blocks, 256, 0, s, p.data, p.n, p.ld, cams, V, L, (char *)ws, count_tiles);
}

cudaError_t launch_preprocess(const gs_params &p, const CamBatch &cams, int V, const Layout &L, void *ws,
                              bool count_tiles, cudaStream_t s) {
    int64_t blocks = (p.n + 255) / 256;
    if (blocks == 0) return cudaGetLastError();
    ProfScope prof("k_preprocess", s);
    switch (p.sh_degree) {
        case 0: launch_pre<0>(V <= SPLIT_MAX_VIEWS, blocks, s, p, cams, V, L, ws, count_tiles); break;
        case 1: launch_pre<1>(V <= SPLIT_MAX_VIEWS, blocks, s, p, cams, V, L, ws, count_tiles); break;
        case 2: launch_pre<2>(V <= SPLIT_MAX_VIEWS, blocks, s, p, cams, V, L, ws, count_tiles); break;
        default: launch_pre<3>(V <= SPLIT_MAX_VIEWS, blocks, s, p, cams, V, L, ws, count_tiles); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_preprocess_bwd(const gs_params &p, const CamBatch &cams, int V, const Layout &L, void *ws,
                                  float *grad2d_norm, cudaStream_t s, int64_t *step_inc) {
    int64_t blocks = (p.n + 127) / 128;  // grid sized for every Gaussian; threads past vis_count exit
    if (blocks == 0) return cudaGetLastError();
    char *w = (char *)ws;
    ProfScope prof("k_preprocess_bwd", s);
    switch (p.sh_degree) {
        case 0: launch_pdl(k_preprocess_bwd<0>, blocks, 128, 0, s, p.data, p.n, p.ld, cams, V, L, w, grad2d_norm, step_inc); break;
        case 1: launch_pdl(k_preprocess_bwd<1>, blocks, 128, 0, s, p.data, p.n, p.ld, cams, V, L, w, grad2d_norm, step_inc); break;
        case 2: launch_pdl(k_preprocess_bwd<2>, blocks, 128, 0, s, p.data, p.n, p.ld, cams, V, L, w, grad2d_norm, step_inc); break;
        default: launch_pdl(k_preprocess_bwd<3>, blocks, 128, 0, s, p.data, p.n, p.ld, cams, V, L, w, grad2d_norm, step_inc); break;
    }
    return cudaGetLastError();
}

__global__ void k_exp_scale(const float *s, float *out, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (float)exp((double)s[i]);
}

cudaError_t launch_exp_scale(const float *s, float *out, int64_t n, cudaStream_t st) {
    if (n > 0) k_exp_scale<<<(n + 255) / 256, 256, 0, st>>>(s, out, n);
    return cudaGetLastError();
}

}  // namespace gsk
