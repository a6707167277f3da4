/*
 * oracle.c -- CPU ORACLE for the Photo-SLAM photorealistic-mapping hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load, call or link this library.  It shares
 * no code, header, constant table or helper with the CUDA path
 * (paper_2311_16728_b200/csrc); neither side includes or imports the other.
 *
 * What it computes (citations are /root/reference lines; "SURVEY" = /root/repo/SURVEY.md
 * §8(c), whose readings R1..R26 are restated in DESIGN.md):
 *   - per-Gaussian projection ("alpha_i = sigma_i * G(R,t,P_i,r_i,s_i)",
 *     G = 3DGS EWA splatting), SH colour;
 *   - Eq. 3 as a PER-PIXEL brute force over every non-culled Gaussian in
 *     ascending (depth, index) order -- the plain definition the tile renderer reaches;
 *   - Eq. 4 loss (lambda = 0.2 PAPER.md:568) with its analytic gradient;
 *   - reverse-mode gradients of Eq. 3 through the projection to P, r, s, sigma, SH
 *     ("optimization ... by minimizing the photometric loss");
 *   - the Gaussian pyramid level ("Gaussian smoothing and downsampling");
 *   - the optimiser step (Adam with fixed per-class rates);
 *   - the tile binning reference (SPEC.md:348 steps (2)-(3)) for bit-exact comparison.
 *
 * Two modes share this source (SURVEY §8(c) "Two oracle modes"):
 *   ORC_FP64   every quantity in double (finite-difference pins, closed forms);
 *   ORC_RECIPE the decision quantities (cull, depth, mean2d, conic, radius, rect, power)
 *              follow the fp32 decision recipe of DESIGN.md §"fp32 decision recipe"
 *               with IEEE fp32 ops and explicit fmaf; alpha, T, colour,
 *              loss and gradients are then evaluated in double from those values.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math (see oracle/oracle.py).
 * parity unpinned: nothing -- every function has a pin in tests/test_oracle_*.py (the R15
 * clamped-tangent and R7 alpha-clamp branches in test_oracle_clamps.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define ORC_FP64 0
#define ORC_RECIPE 1
#define ORC_TILE 16

/* Camera: world->camera p_c = R P + t (row-major R), pixels centred at integers. */
typedef struct {
    float R[9];
    float t[3];
    float fx, fy, cx, cy;
    int32_t width, height;
    float znear, lim_x, lim_y;
} orc_camera;

typedef struct {
    int64_t n;
    int D;
    const float *means;      /* [n][3] */
    const float *quats;      /* [n][4] (w,x,y,z) raw */
    const float *log_scales; /* [n][3] */
    const float *opac;       /* [n] logits */
    const float *sh;         /* [n][(D+1)^2][3] */
} orc_scene;

typedef struct {
    int radius; /* 0 => culled */
    int rect[4];
    double depth, u, v, A, B, C;     /* value path (promoted fp32 in recipe mode) */
    float depth_f, u_f, v_f, A_f, B_f, C_f;
    double sigma, rgb[3];
    int clamped[3];
} orc_proj;

static int g_threads = 0;
void orc_set_threads(int n) { g_threads = n; }
int orc_get_threads(void) { return g_threads > 0 ? g_threads : omp_get_max_threads(); }

/* ------------------------------------------------------------------------------------ */
/* Real spherical harmonics to degree 3 (constants = textbook normalisations  */
/* sqrt(1/4pi), sqrt(3/4pi), sqrt(15/4pi), 1/4 sqrt(5/pi), 1/4 sqrt(15/pi),              */
/* 1/4 sqrt(35/2pi), 1/2 sqrt(105/pi), 1/4 sqrt(21/2pi), 1/4 sqrt(7/pi), 1/4 sqrt(105/pi)),*/
/* sign convention of the cited 3DGS renderer ("color converted from SH"). */
/* Y[l] for unit dir (x,y,z); dY[l][3] = partial derivatives treating x,y,z independent. */
static void sh_basis(int D, double x, double y, double z, double Y[16], double dY[16][3]) {
    const double pi = M_PI;
    const double c0 = sqrt(1.0 / (4.0 * pi));
    const double c1 = sqrt(3.0 / (4.0 * pi));
    const double c2a = sqrt(15.0 / (4.0 * pi));      /* xy, yz, xz */
    const double c2b = 0.25 * sqrt(5.0 / pi);       /* 2zz - xx - yy */
    const double c2c = 0.25 * sqrt(15.0 / pi);      /* xx - yy */
    const double c3a = 0.25 * sqrt(35.0 / (2.0 * pi));
    const double c3b = 0.5 * sqrt(105.0 / pi);
    const double c3c = 0.25 * sqrt(21.0 / (2.0 * pi));
    const double c3d = 0.25 * sqrt(7.0 / pi);
    const double c3e = 0.25 * sqrt(105.0 / pi);
    memset(Y, 0, 16 * sizeof(double));
    memset(dY, 0, 16 * 3 * sizeof(double));
    Y[0] = c0;
    if (D < 1) return;
    Y[1] = -c1 * y;  dY[1][1] = -c1;
    Y[2] = c1 * z;   dY[2][2] = c1;
    Y[3] = -c1 * x;  dY[3][0] = -c1;
    if (D < 2) return;
    double xx = x * x, yy = y * y, zz = z * z;
    Y[4] = c2a * x * y;                 dY[4][0] = c2a * y;  dY[4][1] = c2a * x;
    Y[5] = -c2a * y * z;                dY[5][1] = -c2a * z; dY[5][2] = -c2a * y;
    Y[6] = c2b * (2 * zz - xx - yy);    dY[6][0] = -2 * c2b * x; dY[6][1] = -2 * c2b * y; dY[6][2] = 4 * c2b * z;
    Y[7] = -c2a * x * z;                dY[7][0] = -c2a * z; dY[7][2] = -c2a * x;
    Y[8] = c2c * (xx - yy);             dY[8][0] = 2 * c2c * x; dY[8][1] = -2 * c2c * y;
    if (D < 3) return;
    Y[9] = -c3a * y * (3 * xx - yy);
    dY[9][0] = -c3a * 6 * x * y;        dY[9][1] = -c3a * (3 * xx - 3 * yy);
    Y[10] = c3b * x * y * z;
    dY[10][0] = c3b * y * z; dY[10][1] = c3b * x * z; dY[10][2] = c3b * x * y;
    Y[11] = -c3c * y * (4 * zz - xx - yy);
    dY[11][0] = -c3c * (-2 * x * y); dY[11][1] = -c3c * (4 * zz - xx - 3 * yy); dY[11][2] = -c3c * 8 * y * z;
    Y[12] = c3d * z * (2 * zz - 3 * xx - 3 * yy);
    dY[12][0] = c3d * (-6 * x * z); dY[12][1] = c3d * (-6 * y * z); dY[12][2] = c3d * (6 * zz - 3 * xx - 3 * yy);
    Y[13] = -c3c * x * (4 * zz - xx - yy);
    dY[13][0] = -c3c * (4 * zz - 3 * xx - yy); dY[13][1] = -c3c * (-2 * x * y); dY[13][2] = -c3c * 8 * x * z;
    Y[14] = c3e * z * (xx - yy);
    dY[14][0] = c3e * 2 * x * z; dY[14][1] = -c3e * 2 * y * z; dY[14][2] = c3e * (xx - yy);
    Y[15] = -c3a * x * (xx - 3 * yy);
    dY[15][0] = -c3a * (3 * xx - 3 * yy); dY[15][1] = -c3a * (-6 * x * y);
}

/* The basis with every monomial taken in absolute value, at nonnegative (xa, ya, za): the
   magnitude a finite-precision evaluation of Y_l / dY_l at a direction whose components are
   at most (xa, ya, za) in size rounds (rounding allowance only, see orc_backward's mag). */
static void sh_basis_abs(int D, double x, double y, double z, double Y[16], double dY[16][3]) {
    const double pi = M_PI;
    const double c0 = sqrt(1.0 / (4.0 * pi)), c1 = sqrt(3.0 / (4.0 * pi)), c2a = sqrt(15.0 / (4.0 * pi));
    const double c2b = 0.25 * sqrt(5.0 / pi), c2c = 0.25 * sqrt(15.0 / pi), c3a = 0.25 * sqrt(35.0 / (2.0 * pi));
    const double c3b = 0.5 * sqrt(105.0 / pi), c3c = 0.25 * sqrt(21.0 / (2.0 * pi)), c3d = 0.25 * sqrt(7.0 / pi);
    const double c3e = 0.25 * sqrt(105.0 / pi);
    memset(Y, 0, 16 * sizeof(double));
    memset(dY, 0, 16 * 3 * sizeof(double));
    Y[0] = c0;
    if (D < 1) return;
    Y[1] = c1 * y;  dY[1][1] = c1;
    Y[2] = c1 * z;  dY[2][2] = c1;
    Y[3] = c1 * x;  dY[3][0] = c1;
    if (D < 2) return;
    double xx = x * x, yy = y * y, zz = z * z;
    Y[4] = c2a * x * y;               dY[4][0] = c2a * y;  dY[4][1] = c2a * x;
    Y[5] = c2a * y * z;               dY[5][1] = c2a * z;  dY[5][2] = c2a * y;
    Y[6] = c2b * (2 * zz + xx + yy);  dY[6][0] = 2 * c2b * x; dY[6][1] = 2 * c2b * y; dY[6][2] = 4 * c2b * z;
    Y[7] = c2a * x * z;               dY[7][0] = c2a * z;  dY[7][2] = c2a * x;
    Y[8] = c2c * (xx + yy);           dY[8][0] = 2 * c2c * x; dY[8][1] = 2 * c2c * y;
    if (D < 3) return;
    Y[9] = c3a * y * (3 * xx + yy);   dY[9][0] = c3a * 6 * x * y; dY[9][1] = c3a * (3 * xx + 3 * yy);
    Y[10] = c3b * x * y * z;          dY[10][0] = c3b * y * z; dY[10][1] = c3b * x * z; dY[10][2] = c3b * x * y;
    Y[11] = c3c * y * (4 * zz + xx + yy);
    dY[11][0] = c3c * 2 * x * y; dY[11][1] = c3c * (4 * zz + xx + 3 * yy); dY[11][2] = c3c * 8 * y * z;
    Y[12] = c3d * z * (2 * zz + 3 * xx + 3 * yy);
    dY[12][0] = c3d * 6 * x * z; dY[12][1] = c3d * 6 * y * z; dY[12][2] = c3d * (6 * zz + 3 * xx + 3 * yy);
    Y[13] = c3c * x * (4 * zz + xx + yy);
    dY[13][0] = c3c * (4 * zz + 3 * xx + yy); dY[13][1] = c3c * 2 * x * y; dY[13][2] = c3c * 8 * x * z;
    Y[14] = c3e * z * (xx + yy);      dY[14][0] = c3e * 2 * x * z; dY[14][1] = c3e * 2 * y * z; dY[14][2] = c3e * (xx + yy);
    Y[15] = c3a * x * (xx + 3 * yy);  dY[15][0] = c3a * (3 * xx + 3 * yy); dY[15][1] = c3a * 6 * x * y;
}

/* exported for the orthonormality pin */
void orc_sh_basis(int D, int64_t n, const double *dirs, double *Y_out, double *dY_out) {
    for (int64_t i = 0; i < n; i++) {
        double Y[16], dY[16][3];
        sh_basis(D, dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2], Y, dY);
        memcpy(Y_out + 16 * i, Y, sizeof(Y));
        if (dY_out) memcpy(dY_out + 48 * i, dY, sizeof(dY));
    }
}

/* Colour c = max(0, sum_l SH_l Y_l(dir) + 0.5), dir = normalize(P - C_cam), C_cam = -R^T t
   (SPEC.md:338).  Double precision in both modes (value path). */
static void eval_colour(const orc_scene *s, int64_t i, const orc_camera *cam, double rgb[3], int clamped[3]) {
    double Cc[3];
    for (int k = 0; k < 3; k++)
        Cc[k] = -((double)cam->R[0 * 3 + k] * cam->t[0] + (double)cam->R[1 * 3 + k] * cam->t[1] +
                  (double)cam->R[2 * 3 + k] * cam->t[2]);
    double d[3] = {s->means[3 * i] - Cc[0], s->means[3 * i + 1] - Cc[1], s->means[3 * i + 2] - Cc[2]};
    double nd = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    double Y[16], dY[16][3];
    sh_basis(s->D, d[0] / nd, d[1] / nd, d[2] / nd, Y, dY);
    int K = (s->D + 1) * (s->D + 1);
    for (int ch = 0; ch < 3; ch++) {
        double acc = 0.5;
        for (int l = 0; l < K; l++) acc += (double)s->sh[(i * K + l) * 3 + ch] * Y[l];
        clamped[ch] = acc < 0.0;
        rgb[ch] = acc < 0.0 ? 0.0 : acc;
    }
}

static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

/* Rotation matrix of a unit quaternion (w,x,y,z) -- standard formula (SPEC.md:321 build_cov3d). */
static void quat_to_rot(const double q[4], double Rq[9]) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    Rq[0] = 1 - 2 * (y * y + z * z); Rq[1] = 2 * (x * y - w * z);     Rq[2] = 2 * (x * z + w * y);
    Rq[3] = 2 * (x * y + w * z);     Rq[4] = 1 - 2 * (x * x + z * z); Rq[5] = 2 * (y * z - w * x);
    Rq[6] = 2 * (x * z - w * y);     Rq[7] = 2 * (y * z + w * x);     Rq[8] = 1 - 2 * (x * x + y * y);
}

/* ---------------------------- fp64 projection ------------------------------------- */
/* Sigma3 = R S S^T R^T; Sigma2 = J W Sigma3 W^T J^T + 0.3 I (SPEC.md:328,
   SURVEY R13); conic = Sigma2^-1; r = ceil(3 sqrt(lambda_max)); culling
   (z <= znear, |q| = 0, det <= 0, empty tile rect). */
typedef struct {
    double pc[3], z, tx, ty, txc, ty_c;
    int clx, cly; /* tan clamp active */
    double qn[4], qnorm, Rq[9], sc[3], M[9], S3[9];
    double J[6], T[6], S2[3]; /* S2 = (a,b,c) incl. floor */
} orc_fwd64;

static int fwd64(const orc_scene *s, int64_t i, const orc_camera *cam, orc_fwd64 *f) {
    const float *P = s->means + 3 * i;
    for (int r = 0; r < 3; r++)
        f->pc[r] = (double)cam->R[3 * r] * P[0] + (double)cam->R[3 * r + 1] * P[1] +
                   (double)cam->R[3 * r + 2] * P[2] + (double)cam->t[r];
    f->z = f->pc[2];
    const float *q = s->quats + 4 * i;
    double qq = (double)q[0] * q[0] + (double)q[1] * q[1] + (double)q[2] * q[2] + (double)q[3] * q[3];
    f->qnorm = sqrt(qq);
    if (!(f->z > cam->znear) || qq == 0.0) return 0;
    for (int k = 0; k < 4; k++) f->qn[k] = q[k] / f->qnorm;
    quat_to_rot(f->qn, f->Rq);
    for (int k = 0; k < 3; k++) f->sc[k] = exp((double)s->log_scales[3 * i + k]);
    for (int r = 0; r < 3; r++)
        for (int c = 0; c < 3; c++) f->M[3 * r + c] = f->Rq[3 * r + c] * f->sc[c];
    for (int r = 0; r < 3; r++)
        for (int c = 0; c < 3; c++)
            f->S3[3 * r + c] = f->M[3 * r] * f->M[3 * c] + f->M[3 * r + 1] * f->M[3 * c + 1] +
                               f->M[3 * r + 2] * f->M[3 * c + 2];
    double z = f->z;
    f->tx = f->pc[0] / z;
    f->ty = f->pc[1] / z;
    double lx = cam->lim_x, ly = cam->lim_y;
    f->clx = (f->tx < -lx) || (f->tx > lx);
    f->cly = (f->ty < -ly) || (f->ty > ly);
    f->txc = f->tx < -lx ? -lx : (f->tx > lx ? lx : f->tx);
    f->ty_c = f->ty < -ly ? -ly : (f->ty > ly ? ly : f->ty);
    double fx = cam->fx, fy = cam->fy;
    /* J = d(pi)/d(p_c) with the clamped tangent */
    f->J[0] = fx / z; f->J[1] = 0; f->J[2] = -fx * f->txc / z;
    f->J[3] = 0; f->J[4] = fy / z; f->J[5] = -fy * f->ty_c / z;
    /* T = J W, W = camera rotation */
    for (int r = 0; r < 2; r++)
        for (int c = 0; c < 3; c++)
            f->T[3 * r + c] = f->J[3 * r] * cam->R[c] + f->J[3 * r + 1] * cam->R[3 + c] +
                              f->J[3 * r + 2] * cam->R[6 + c];
    double U[6];
    for (int r = 0; r < 2; r++)
        for (int c = 0; c < 3; c++)
            U[3 * r + c] = f->T[3 * r] * f->S3[c] + f->T[3 * r + 1] * f->S3[3 + c] + f->T[3 * r + 2] * f->S3[6 + c];
    f->S2[0] = U[0] * f->T[0] + U[1] * f->T[1] + U[2] * f->T[2] + 0.3;
    f->S2[1] = U[0] * f->T[3] + U[1] * f->T[4] + U[2] * f->T[5];
    f->S2[2] = U[3] * f->T[3] + U[4] * f->T[4] + U[5] * f->T[5] + 0.3;
    return 1;
}

/* exported for pins: Sigma3 (row-major 3x3) and Sigma2 incl. the 0.3 floor (a, b, c) */
int orc_debug_cov(const float *mean, const float *quat, const float *log_scale, const orc_camera *cam,
                  double *S3, double *S2) {
    float op = 0.0f, sh[3] = {0, 0, 0};
    orc_scene s = {1, 0, mean, quat, log_scale, &op, sh};
    orc_fwd64 f;
    if (!fwd64(&s, 0, cam, &f)) return 0;
    memcpy(S3, f.S3, sizeof(f.S3));
    memcpy(S2, f.S2, sizeof(f.S2));
    return 1;
}

static void tiles_of(const orc_camera *cam, double u, double v, int r, int rect[4]) {
    int TX = (cam->width + ORC_TILE - 1) / ORC_TILE, TY = (cam->height + ORC_TILE - 1) / ORC_TILE;
    double x0 = floor((u - r) / ORC_TILE), x1 = floor((u + r) / ORC_TILE) + 1;
    double y0 = floor((v - r) / ORC_TILE), y1 = floor((v + r) / ORC_TILE) + 1;
    x0 = x0 < 0 ? 0 : (x0 > TX ? TX : x0); x1 = x1 < 0 ? 0 : (x1 > TX ? TX : x1);
    y0 = y0 < 0 ? 0 : (y0 > TY ? TY : y0); y1 = y1 < 0 ? 0 : (y1 > TY ? TY : y1);
    rect[0] = (int)x0; rect[1] = (int)y0; rect[2] = (int)x1; rect[3] = (int)y1;
}

static void project_fp64(const orc_scene *s, int64_t i, const orc_camera *cam, orc_proj *o) {
    memset(o, 0, sizeof(*o));
    orc_fwd64 f;
    if (!fwd64(s, i, cam, &f)) return;
    double a = f.S2[0], b = f.S2[1], c = f.S2[2];
    double det = a * c - b * b;
    if (!(det > 0)) return;
    double mid = 0.5 * (a + c);
    double disc = mid * mid - det;
    double lam = mid + sqrt(disc > 0 ? disc : 0);
    int r = (int)ceil(3.0 * sqrt(lam));
    double u = cam->fx * f.tx + cam->cx, v = cam->fy * f.ty + cam->cy;
    int rect[4];
    tiles_of(cam, u, v, r, rect);
    if ((rect[2] - rect[0]) * (rect[3] - rect[1]) == 0) return;
    o->radius = r;
    memcpy(o->rect, rect, sizeof(rect));
    o->depth = f.z; o->u = u; o->v = v;
    o->A = c / det; o->B = -b / det; o->C = a / det;
    o->sigma = sigmoid(s->opac[i]);
    eval_colour(s, i, cam, o->rgb, o->clamped);
}

/* ---------------------------- fp32 decision recipe -------------------------------- */
/* DESIGN.md "fp32 decision recipe".  IEEE fp32, no contraction, fmaf   */
/* where the recipe says fma.  Every line below is one line of the recipe.             */
static float dot3f(const float a[3], const float b[3]) { return fmaf(a[2], b[2], fmaf(a[1], b[1], a[0] * b[0])); }

static void project_recipe(const orc_scene *s, int64_t i, const orc_camera *cam, orc_proj *o) {
    memset(o, 0, sizeof(*o));
    const float *P = s->means + 3 * i;
    float pc[3];
    for (int r = 0; r < 3; r++) pc[r] = dot3f(cam->R + 3 * r, P) + cam->t[r];
    float z = pc[2];
    if (!(z > cam->znear)) return;
    const float *q = s->quats + 4 * i;
    float d4 = fmaf(q[3], q[3], fmaf(q[2], q[2], fmaf(q[1], q[1], q[0] * q[0])));
    if (d4 == 0.0f) return;
    float inv = 1.0f / sqrtf(d4);
    float w = q[0] * inv, x = q[1] * inv, y = q[2] * inv, zq = q[3] * inv;
    float Rq[9];
    Rq[0] = 1.0f - 2.0f * fmaf(y, y, zq * zq);
    Rq[1] = 2.0f * fmaf(x, y, -(w * zq));
    Rq[2] = 2.0f * fmaf(x, zq, w * y);
    Rq[3] = 2.0f * fmaf(x, y, w * zq);
    Rq[4] = 1.0f - 2.0f * fmaf(x, x, zq * zq);
    Rq[5] = 2.0f * fmaf(y, zq, -(w * x));
    Rq[6] = 2.0f * fmaf(x, zq, -(w * y));
    Rq[7] = 2.0f * fmaf(y, zq, w * x);
    Rq[8] = 1.0f - 2.0f * fmaf(x, x, y * y);
    float e[3];
    for (int k = 0; k < 3; k++) e[k] = (float)exp((double)s->log_scales[3 * i + k]);
    float M[9], S3[9];
    for (int r = 0; r < 3; r++)
        for (int c = 0; c < 3; c++) M[3 * r + c] = Rq[3 * r + c] * e[c];
    for (int r = 0; r < 3; r++)
        for (int c = 0; c < 3; c++) S3[3 * r + c] = dot3f(M + 3 * r, M + 3 * c);
    float tx = pc[0] / z, ty = pc[1] / z;
    float txc = fminf(fmaxf(tx, -cam->lim_x), cam->lim_x);
    float tyc = fminf(fmaxf(ty, -cam->lim_y), cam->lim_y);
    float J00 = cam->fx / z, J02 = -(cam->fx * txc) / z;
    float J11 = cam->fy / z, J12 = -(cam->fy * tyc) / z;
    const float *W = cam->R;
    float T0[3], T1[3];
    for (int j = 0; j < 3; j++) {
        T0[j] = fmaf(J02, W[6 + j], J00 * W[j]);
        T1[j] = fmaf(J12, W[6 + j], J11 * W[3 + j]);
    }
    float U0[3], U1[3];
    for (int j = 0; j < 3; j++) {
        float col[3] = {S3[j], S3[3 + j], S3[6 + j]};
        U0[j] = dot3f(T0, col);
        U1[j] = dot3f(T1, col);
    }
    float a = dot3f(U0, T0) + 0.3f;
    float b = dot3f(U0, T1);
    float c = dot3f(U1, T1) + 0.3f;
    float det = fmaf(-b, b, a * c);
    if (!(det > 0.0f)) return;
    float idet = 1.0f / det;
    float A = c * idet, B = -b * idet, C = a * idet;
    float mid = 0.5f * (a + c);
    float lam = mid + sqrtf(fmaxf(0.0f, fmaf(mid, mid, -det)));
    int r = (int)ceilf(3.0f * sqrtf(lam));
    float u = fmaf(cam->fx, tx, cam->cx), v = fmaf(cam->fy, ty, cam->cy);
    float TX = (float)((cam->width + ORC_TILE - 1) / ORC_TILE), TY = (float)((cam->height + ORC_TILE - 1) / ORC_TILE);
    float rf = (float)r;
    float fx0 = fminf(fmaxf(floorf((u - rf) * 0.0625f), 0.0f), TX);
    float fx1 = fminf(fmaxf(floorf((u + rf) * 0.0625f) + 1.0f, 0.0f), TX);
    float fy0 = fminf(fmaxf(floorf((v - rf) * 0.0625f), 0.0f), TY);
    float fy1 = fminf(fmaxf(floorf((v + rf) * 0.0625f) + 1.0f, 0.0f), TY);
    int rect[4] = {(int)fx0, (int)fy0, (int)fx1, (int)fy1};
    if ((rect[2] - rect[0]) * (rect[3] - rect[1]) == 0) return;
    o->radius = r;
    memcpy(o->rect, rect, sizeof(rect));
    o->depth_f = z; o->u_f = u; o->v_f = v; o->A_f = A; o->B_f = B; o->C_f = C;
    o->depth = z; o->u = u; o->v = v; o->A = A; o->B = B; o->C = C;
    o->sigma = sigmoid(s->opac[i]);
    eval_colour(s, i, cam, o->rgb, o->clamped);
}

static void project_one(int mode, const orc_scene *s, int64_t i, const orc_camera *cam, orc_proj *o) {
    if (mode == ORC_RECIPE) project_recipe(s, i, cam, o);
    else project_fp64(s, i, cam, o);
}

static orc_proj *project_all(int mode, const orc_scene *s, const orc_camera *cam) {
    orc_proj *pr = (orc_proj *)malloc(sizeof(orc_proj) * (s->n > 0 ? s->n : 1));
#pragma omp parallel for schedule(static) num_threads(orc_get_threads())
    for (int64_t i = 0; i < s->n; i++) project_one(mode, s, i, cam, pr + i);
    return pr;
}

/* Exported: per-Gaussian projection for pins and parity. */
void orc_project(int mode, int64_t n, int D, const float *means, const float *quats, const float *log_scales,
                 const float *opac, const float *sh, const orc_camera *cam, int32_t *radius, int32_t *rect,
                 double *depth, double *mean2d, double *conic, double *rgb, double *sigma, uint32_t *depth_bits,
                 float *mean2d_f, float *conic_f) {
    orc_scene s = {n, D, means, quats, log_scales, opac, sh};
    orc_proj *pr = project_all(mode, &s, cam);
    for (int64_t i = 0; i < n; i++) {
        orc_proj *o = pr + i;
        radius[i] = o->radius;
        for (int k = 0; k < 4; k++) rect[4 * i + k] = o->rect[k];
        depth[i] = o->depth;
        mean2d[2 * i] = o->u; mean2d[2 * i + 1] = o->v;
        conic[3 * i] = o->A; conic[3 * i + 1] = o->B; conic[3 * i + 2] = o->C;
        for (int k = 0; k < 3; k++) rgb[3 * i + k] = o->rgb[k];
        sigma[i] = o->sigma;
        uint32_t bits; memcpy(&bits, &o->depth_f, 4); depth_bits[i] = bits;
        mean2d_f[2 * i] = o->u_f; mean2d_f[2 * i + 1] = o->v_f;
        conic_f[3 * i] = o->A_f; conic_f[3 * i + 1] = o->B_f; conic_f[3 * i + 2] = o->C_f;
    }
    free(pr);
}

/* exp of a log-scale exactly as the recipe states: (float)exp((double)s) */
void orc_exp_scale_f32(int64_t n, const float *s, float *out) {
#pragma omp parallel for schedule(static) num_threads(orc_get_threads())
    for (int64_t i = 0; i < n; i++) out[i] = (float)exp((double)s[i]);
}

/* ---------------------------- binning reference ----------------------------------- */
/* SPEC.md:348 (2) "bin survivors into 16x16-pixel tiles", (3) "sort contributors by     */
/* ascending depth (ties by primitive id)"; key = (view*tiles + tile)<<32 */
/* | float_bits(depth), value = Gaussian index, stable in emission order (index, then    */
/* tiles row-major).  A sort on (key, value) is that stable sort.                        */
typedef struct { uint64_t key; uint32_t val; } orc_pair;
static int cmp_pair(const void *pa, const void *pb) {
    const orc_pair *a = (const orc_pair *)pa, *b = (const orc_pair *)pb;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return a->val < b->val ? -1 : (a->val > b->val);
}

/* Returns the pair count; if keys != NULL fills sorted keys/vals and ranges[V*tiles][2]. */
/* Exact ellipse-tile test (SURVEY §8(f) f3 "exact ellipse-tile binning", R10'): can the
   3-sigma ellipse d^T Q d <= 9 (R9) reach a pixel centre of tile (tx, ty)?  Minimum of the
   quadratic form over the tile's box of pixel centres [16 tx, 16 tx + 15] x [16 ty, 16 ty + 15]:
   0 if the mean is inside, else the smallest of the four edge minima (y* = -B X / C clamped),
   compared with 9.01 (0.1 % margin over the per-pixel cutoff, so a tile holding a pixel the
   Gaussian can reach is never dropped).  fp32 IEEE operations in a fixed order (explicit fmaf,
   -ffp-contract=off): the GPU takes the same decision bit for bit. */
static int tile_hits_ellipse(float u, float v, float A, float B, float C, int tx, int ty) {
    const float ax = (float)(tx * ORC_TILE) - u, bx = (float)(tx * ORC_TILE + ORC_TILE - 1) - u;
    const float ay = (float)(ty * ORC_TILE) - v, by = (float)(ty * ORC_TILE + ORC_TILE - 1) - v;
    if (ax <= 0.f && bx >= 0.f && ay <= 0.f && by >= 0.f) return 1;
    const float rA = 1.0f / A, rC = 1.0f / C;  /* the edge minimisers y* = -B X / C via 1/C */
    float best = INFINITY;
    for (int e = 0; e < 2; e++) {
        const float X = e ? bx : ax;
        const float y = fminf(fmaxf(-(B * X) * rC, ay), by);
        const float fx_ = fmaf(C * y, y, fmaf((2.f * B) * X, y, (A * X) * X));
        best = fminf(best, fx_);
        const float Y = e ? by : ay;
        const float x = fminf(fmaxf(-(B * Y) * rA, ax), bx);
        const float fy_ = fmaf(C * Y, Y, fmaf((2.f * B) * x, Y, (A * x) * x));
        best = fminf(best, fy_);
    }
    return best <= 9.01f;
}

static int64_t tiles_of_gaussian(const orc_proj *o) {
    int64_t c = 0;
    for (int ty = o->rect[1]; ty < o->rect[3]; ty++)
        for (int tx = o->rect[0]; tx < o->rect[2]; tx++)
            c += tile_hits_ellipse(o->u_f, o->v_f, o->A_f, o->B_f, o->C_f, tx, ty);
    return c;
}

int64_t orc_bin(int64_t n, int D, const float *means, const float *quats, const float *log_scales,
                const float *opac, const float *sh, int V, const orc_camera *cams, uint64_t *keys,
                uint32_t *vals, uint32_t *ranges, int32_t *tiles_touched) {
    orc_scene s = {n, D, means, quats, log_scales, opac, sh};
    int TXv = (cams[0].width + ORC_TILE - 1) / ORC_TILE, TYv = (cams[0].height + ORC_TILE - 1) / ORC_TILE;
    int64_t tiles = (int64_t)TXv * TYv;
    int64_t P = 0;
    orc_proj **prs = (orc_proj **)malloc(sizeof(orc_proj *) * V);
    for (int v = 0; v < V; v++) {
        prs[v] = project_all(ORC_RECIPE, &s, cams + v);
        for (int64_t i = 0; i < n; i++) {
            orc_proj *o = prs[v] + i;
            int64_t tt = o->radius > 0 ? tiles_of_gaussian(o) : 0;
            if (tiles_touched) tiles_touched[(int64_t)v * n + i] = (int32_t)tt;
            P += tt;
        }
    }
    if (keys) {
        orc_pair *pairs = (orc_pair *)malloc(sizeof(orc_pair) * (P > 0 ? P : 1));
        int64_t k = 0;
        for (int v = 0; v < V; v++)
            for (int64_t i = 0; i < n; i++) {
                orc_proj *o = prs[v] + i;
                if (o->radius == 0) continue;
                uint32_t bits; memcpy(&bits, &o->depth_f, 4);
                for (int ty = o->rect[1]; ty < o->rect[3]; ty++)
                    for (int tx = o->rect[0]; tx < o->rect[2]; tx++) {
                        if (!tile_hits_ellipse(o->u_f, o->v_f, o->A_f, o->B_f, o->C_f, tx, ty)) continue;
                        uint64_t gt = (uint64_t)v * tiles + (uint64_t)ty * TXv + tx;
                        pairs[k].key = (gt << 32) | bits;
                        pairs[k].val = (uint32_t)i;
                        k++;
                    }
            }
        qsort(pairs, P, sizeof(orc_pair), cmp_pair);
        memset(ranges, 0, sizeof(uint32_t) * 2 * tiles * V);
        for (int64_t j = 0; j < P; j++) {
            keys[j] = pairs[j].key;
            vals[j] = pairs[j].val;
            uint64_t gt = pairs[j].key >> 32;
            if (j == 0 || (pairs[j - 1].key >> 32) != gt) ranges[2 * gt] = (uint32_t)j;
            if (j == P - 1 || (pairs[j + 1].key >> 32) != gt) ranges[2 * gt + 1] = (uint32_t)(j + 1);
        }
        free(pairs);
    }
    for (int v = 0; v < V; v++) free(prs[v]);
    free(prs);
    return P;
}

/* ---------------------------- per-pixel compositing ------------------------------- */
/* Global (depth, index) order of the visible Gaussians of one view (SPEC.md:348 (3)).  */
static const orc_proj *g_sort_pr;
static int g_sort_mode;
static int cmp_depth(const void *pa, const void *pb) {
    int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
    const orc_proj *A = g_sort_pr + a, *B = g_sort_pr + b;
    if (g_sort_mode == ORC_RECIPE) {
        uint32_t ba, bb; memcpy(&ba, &A->depth_f, 4); memcpy(&bb, &B->depth_f, 4);
        if (ba != bb) return ba < bb ? -1 : 1;
    } else if (A->depth != B->depth) return A->depth < B->depth ? -1 : 1;
    return a < b ? -1 : (a > b);
}
static int64_t depth_order(int mode, const orc_proj *pr, int64_t n, int64_t *order) {
    int64_t m = 0;
    for (int64_t i = 0; i < n; i++)
        if (pr[i].radius > 0) order[m++] = i;
    g_sort_pr = pr; g_sort_mode = mode;
    qsort(order, m, sizeof(int64_t), cmp_depth);
    return m;
}

/* power = -1/2 d^T Q d, d = pixel - mean2d, Q = conic (SPEC.md:348 (4)).
   Recipe: dx = x-u; qf = fma(C dy, dy, (A dx) dx); power = fma(-(B dx), dy, -0.5 qf). */
static double pixel_power(int mode, const orc_proj *g, int px, int py, double *dx, double *dy) {
    if (mode == ORC_RECIPE) {
        float fdx = (float)px - g->u_f, fdy = (float)py - g->v_f;
        float qf = fmaf(g->C_f * fdy, fdy, (g->A_f * fdx) * fdx);
        float p = fmaf(-(g->B_f * fdx), fdy, -0.5f * qf);
        *dx = fdx; *dy = fdy;
        return (double)p;
    }
    *dx = px - g->u; *dy = py - g->v;
    return -0.5 * (g->A * *dx * *dx + g->C * *dy * *dy) - g->B * *dx * *dy;
}

#define ORC_ALPHA_MAX 0.99
#define ORC_ALPHA_MIN (1.0 / 255.0)
#define ORC_T_STOP 1e-4
#define ORC_CUTOFF (-4.5) /* Mahalanobis^2 <= 9 */

typedef struct { int64_t k; double alpha, ep, T, dx, dy; int clamped; } orc_contrib;

/* Front-to-back compositing of one pixel (Eq. 3 with prod_{j<i}(1-alpha_j), SURVEY R1;
   skip alpha < 1/255, stop when T(1-alpha) < 1e-4, bg composited). Returns
   the number of composited Gaussians; fills the list if list != NULL.  *flag is set if a
   decision lies inside the ambiguity band of the parity contract. */
static int composite_pixel(int mode, const orc_proj *pr, const int64_t *order, int64_t m, int px, int py,
                           const double bg[3], double out_rgb[3], double *out_T, int64_t *last_id, int *flag,
                           orc_contrib *list, int list_cap) {
    double T = 1.0, C[3] = {0, 0, 0};
    int nc = 0;
    *last_id = -1;
    *flag = 0;
    for (int64_t j = 0; j < m; j++) {
        const orc_proj *g = pr + order[j];
        double dx, dy;
        double p = pixel_power(mode, g, px, py, &dx, &dy);
        if (p > 0.0 || p < ORC_CUTOFF) continue;
        double ep = exp(p);
        double a = g->sigma * ep;
        int clamped = 0;
        if (mode == ORC_RECIPE && fabs(a - ORC_ALPHA_MAX) <= 1e-6) *flag = 1;
        if (a > ORC_ALPHA_MAX) { a = ORC_ALPHA_MAX; clamped = 1; }
        if (mode == ORC_RECIPE && fabs(255.0 * a - 1.0) <= 4e-6) *flag = 1;
        if (a < ORC_ALPHA_MIN) continue;
        double test = T * (1.0 - a);
        if (mode == ORC_RECIPE && fabs(test - ORC_T_STOP) <= 1e-8) *flag = 1;
        if (test < ORC_T_STOP) break;
        if (list && nc < list_cap) {
            list[nc].k = order[j]; list[nc].alpha = a; list[nc].ep = ep; list[nc].T = T;
            list[nc].dx = dx; list[nc].dy = dy; list[nc].clamped = clamped;
        }
        for (int ch = 0; ch < 3; ch++) C[ch] += g->rgb[ch] * a * T;
        T = test;
        nc++;
        *last_id = order[j];
    }
    for (int ch = 0; ch < 3; ch++) out_rgb[ch] = C[ch] + T * bg[ch];
    *out_T = T;
    return nc;
}

/* Render a list of pixels (view, y, x) of V views.  Outputs per listed pixel. */
void orc_render(int mode, int64_t n, int D, const float *means, const float *quats, const float *log_scales,
                const float *opac, const float *sh, int V, const orc_camera *cams, const double *bg,
                int64_t npix, const int32_t *pix, double *out_rgb, double *out_T, int32_t *out_ncomp,
                int64_t *out_last, int32_t *out_flag) {
    orc_scene s = {n, D, means, quats, log_scales, opac, sh};
    for (int v = 0; v < V; v++) {
        orc_proj *pr = project_all(mode, &s, cams + v);
        int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
        int64_t m = depth_order(mode, pr, n, order);
#pragma omp parallel for schedule(dynamic, 64) num_threads(orc_get_threads())
        for (int64_t q = 0; q < npix; q++) {
            if (pix[3 * q] != v) continue;
            int flag;
            out_ncomp[q] = composite_pixel(mode, pr, order, m, pix[3 * q + 2], pix[3 * q + 1], bg,
                                           out_rgb + 3 * q, out_T + q, out_last + q, &flag, NULL, 0);
            out_flag[q] = flag;
        }
        free(order);
        free(pr);
    }
}

/* ---------------------------- analytic backward ----------------------------------- */
/* Per-(view, Gaussian) gradient of the 2D quantities: u, v, A, B, C, sigma, r, g, b.   */
enum { G_U, G_V, G_A, G_B, G_C, G_SIG, G_R, G_G, G_BL, G_N };

/* Chain from 2D gradients of one view to the 3D parameters:
   conic -> Sigma2 -> (Sigma3, T=JW) -> (q, s) and p_c -> P; SH; sigmoid. Adds into g*. */
static void chain_to_3d(const orc_scene *s, int64_t i, const orc_camera *cam, const double g2[G_N],
                        const int clamped[3], double *gm, double *gq, double *gs, double *go, double *gsh) {
    orc_fwd64 f;
    if (!fwd64(s, i, cam, &f)) return;
    double a = f.S2[0], b = f.S2[1], c = f.S2[2];
    double det = a * c - b * b;
    double Q[4] = {c / det, -b / det, -b / det, a / det};
    /* dL/dQ as a symmetric matrix (B appears twice in Q) */
    double G[4] = {g2[G_A], 0.5 * g2[G_B], 0.5 * g2[G_B], g2[G_C]};
    /* H = -Q G Q : dL/dSigma2 (entry-wise, symmetric) */
    double QG[4] = {Q[0] * G[0] + Q[1] * G[2], Q[0] * G[1] + Q[1] * G[3],
                    Q[2] * G[0] + Q[3] * G[2], Q[2] * G[1] + Q[3] * G[3]};
    double H[4] = {-(QG[0] * Q[0] + QG[1] * Q[2]), -(QG[0] * Q[1] + QG[1] * Q[3]),
                   -(QG[2] * Q[0] + QG[3] * Q[2]), -(QG[2] * Q[1] + QG[3] * Q[3])};
    /* Sigma2 = T Sigma3 T^T: dL/dSigma3 = T^T H T; dL/dT = 2 H T Sigma3 */
    const double *T = f.T;
    double GS3[9];
    for (int r = 0; r < 3; r++)
        for (int cc = 0; cc < 3; cc++) {
            double acc = 0;
            for (int p = 0; p < 2; p++)
                for (int q2 = 0; q2 < 2; q2++) acc += T[3 * p + r] * H[2 * p + q2] * T[3 * q2 + cc];
            GS3[3 * r + cc] = acc;
        }
    double HT[6];
    for (int p = 0; p < 2; p++)
        for (int cc = 0; cc < 3; cc++) HT[3 * p + cc] = H[2 * p] * T[cc] + H[2 * p + 1] * T[3 + cc];
    double GT[6];
    for (int p = 0; p < 2; p++)
        for (int cc = 0; cc < 3; cc++)
            GT[3 * p + cc] = 2.0 * (HT[3 * p] * f.S3[cc] + HT[3 * p + 1] * f.S3[3 + cc] + HT[3 * p + 2] * f.S3[6 + cc]);
    /* T = J W: dL/dJ = dL/dT W^T */
    double GJ[6];
    for (int p = 0; p < 2; p++)
        for (int k = 0; k < 3; k++)
            GJ[3 * p + k] = GT[3 * p] * cam->R[3 * k] + GT[3 * p + 1] * cam->R[3 * k + 1] + GT[3 * p + 2] * cam->R[3 * k + 2];
    double fx = cam->fx, fy = cam->fy, z = f.z, x = f.pc[0], y = f.pc[1];
    double gpc[3] = {0, 0, 0};
    /* J00 = fx/z, J02 = -fx txc/z, J11 = fy/z, J12 = -fy tyc/z, txc = clamp(x/z) */
    gpc[2] += GJ[0] * (-fx / (z * z)) + GJ[4] * (-fy / (z * z));
    if (!f.clx) { gpc[0] += GJ[2] * (-fx / (z * z)); gpc[2] += GJ[2] * (2.0 * fx * x / (z * z * z)); }
    else gpc[2] += GJ[2] * (fx * f.txc / (z * z));
    if (!f.cly) { gpc[1] += GJ[5] * (-fy / (z * z)); gpc[2] += GJ[5] * (2.0 * fy * y / (z * z * z)); }
    else gpc[2] += GJ[5] * (fy * f.ty_c / (z * z));
    /* mean2d: u = fx x/z + cx, v = fy y/z + cy */
    gpc[0] += g2[G_U] * fx / z;
    gpc[1] += g2[G_V] * fy / z;
    gpc[2] += g2[G_U] * (-fx * x / (z * z)) + g2[G_V] * (-fy * y / (z * z));
    /* p_c = W P + t: dL/dP = W^T dL/dp_c */
    for (int k = 0; k < 3; k++)
        gm[k] += cam->R[k] * gpc[0] + cam->R[3 + k] * gpc[1] + cam->R[6 + k] * gpc[2];
    /* Sigma3 = M M^T, M = Rq diag(s): dL/dM = 2 GS3 M */
    double GM[9];
    for (int r = 0; r < 3; r++)
        for (int cc = 0; cc < 3; cc++)
            GM[3 * r + cc] = 2.0 * (GS3[3 * r] * f.M[cc] + GS3[3 * r + 1] * f.M[3 + cc] + GS3[3 * r + 2] * f.M[6 + cc]);
    double GR[9];
    for (int j = 0; j < 3; j++) {
        double gsj = 0;
        for (int r = 0; r < 3; r++) { gsj += GM[3 * r + j] * f.Rq[3 * r + j]; GR[3 * r + j] = GM[3 * r + j] * f.sc[j]; }
        gs[j] += gsj * f.sc[j]; /* d/dlog s = s d/ds */
    }
    double w = f.qn[0], qx = f.qn[1], qy = f.qn[2], qz = f.qn[3];
    double gqn[4];
    gqn[0] = 2 * (-qz * GR[1] + qy * GR[2] + qz * GR[3] - qx * GR[5] - qy * GR[6] + qx * GR[7]);
    gqn[1] = 2 * (qy * GR[1] + qz * GR[2] + qy * GR[3] - 2 * qx * GR[4] - w * GR[5] + qz * GR[6] + w * GR[7] - 2 * qx * GR[8]);
    gqn[2] = 2 * (-2 * qy * GR[0] + qx * GR[1] + w * GR[2] + qx * GR[3] + qz * GR[5] - w * GR[6] + qz * GR[7] - 2 * qy * GR[8]);
    gqn[3] = 2 * (-2 * qz * GR[0] - w * GR[1] + qx * GR[2] + w * GR[3] - 2 * qz * GR[4] + qy * GR[5] + qx * GR[6] + qy * GR[7]);
    /* q_hat = q/|q|: dL/dq = (g - q_hat (q_hat . g)) / |q| */
    double dotg = w * gqn[0] + qx * gqn[1] + qy * gqn[2] + qz * gqn[3];
    for (int k = 0; k < 4; k++) gq[k] += (gqn[k] - f.qn[k] * dotg) / f.qnorm;
    /* opacity: sigma = sigmoid(logit) */
    double sg = sigmoid(s->opac[i]);
    go[0] += sg * (1 - sg) * g2[G_SIG];
    /* SH colour: c = max(0, sum SH Y(dir) + 0.5), dir = (P - C)/|P - C| */
    double Cc[3];
    for (int k = 0; k < 3; k++)
        Cc[k] = -((double)cam->R[k] * cam->t[0] + (double)cam->R[3 + k] * cam->t[1] + (double)cam->R[6 + k] * cam->t[2]);
    double d[3] = {s->means[3 * i] - Cc[0], s->means[3 * i + 1] - Cc[1], s->means[3 * i + 2] - Cc[2]};
    double nd = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    double dir[3] = {d[0] / nd, d[1] / nd, d[2] / nd};
    double Y[16], dY[16][3];
    sh_basis(s->D, dir[0], dir[1], dir[2], Y, dY);
    int K = (s->D + 1) * (s->D + 1);
    double gdir[3] = {0, 0, 0};
    const double gc[3] = {g2[G_R], g2[G_G], g2[G_BL]};
    for (int ch = 0; ch < 3; ch++) {
        if (clamped[ch]) continue;
        for (int l = 0; l < K; l++) {
            gsh[l * 3 + ch] += Y[l] * gc[ch];
            double shv = s->sh[(i * K + l) * 3 + ch];
            for (int k = 0; k < 3; k++) gdir[k] += gc[ch] * shv * dY[l][k];
        }
    }
    double dd = dir[0] * gdir[0] + dir[1] * gdir[1] + dir[2] * gdir[2];
    for (int k = 0; k < 3; k++) gm[k] += (gdir[k] - dir[k] * dd) / nd;
}

/* Backward of sum over views of <dL/dI_v, I_v> for listed pixels.  dL_drgb[npix][3].
   Outputs (zeroed here, fp64, per-class AoS): gm[n][3], gq[n][4], gs[n][3], go[n], gsh[n][K][3];
   grad2d_norm[n] = sum over views of ||dL/dmean2d_v|| if non-NULL.
   flag_gauss[n] (optional): 1 if the Gaussian was evaluated at a band-flagged pixel.
   mag (optional, [n][3+4+3+1+3K] in that class order): the conditioning of each gradient
   element -- for every 2-D quantity k (u, v, A, B, C, sigma, r, g, b) the sum over pixels of
   the absolute values of the per-pixel terms that make up its gradient, S_k (each product split
   into its addends: dL/dalpha from |g||c| + |g||acc|, dL/du from |A dx| + |B dy|, ...; every
   term weighted by its pixel's transmittance conditioning kappa = 1 + sum_j alpha_j/(1-alpha_j)
   over the composited layers), carried
   to the parameters by chain_to_3d_abs (the chain with |coefficients| and |intermediates|).  An
   evaluation in precision eps (any summation order, any association of the chain) is within a
   small multiple of eps * mag of the exact value; the GPU parity tests use it as their rounding
   allowance.  Not the method: a bound on what rounding can do to it. */
static void chain_to_3d_abs(const orc_scene *s, int64_t i, const orc_camera *cam, const double S[G_N],
                            const int clamped[3], double *gm, double *gq, double *gs, double *go, double *gsh) {
    /* chain_to_3d with every coefficient and every intermediate replaced by its absolute value
       (sums of |products|; a subtraction becomes an addition): applied to the nonnegative S it
       bounds, step by step, the magnitudes a finite-precision evaluation of the chain rounds. */
    orc_fwd64 f;
    if (!fwd64(s, i, cam, &f)) return;
    double a = f.S2[0], b = f.S2[1], c = f.S2[2];
    double det = a * c - b * b;
    double Q[4] = {fabs(c / det), fabs(b / det), fabs(b / det), fabs(a / det)};
    double G[4] = {S[G_A], 0.5 * S[G_B], 0.5 * S[G_B], S[G_C]};
    double QG[4] = {Q[0] * G[0] + Q[1] * G[2], Q[0] * G[1] + Q[1] * G[3],
                    Q[2] * G[0] + Q[3] * G[2], Q[2] * G[1] + Q[3] * G[3]};
    double H[4] = {QG[0] * Q[0] + QG[1] * Q[2], QG[0] * Q[1] + QG[1] * Q[3],
                   QG[2] * Q[0] + QG[3] * Q[2], QG[2] * Q[1] + QG[3] * Q[3]};
    double T[6];
    for (int k = 0; k < 6; k++) T[k] = fabs(f.T[k]);
    double GS3[9];
    for (int r = 0; r < 3; r++)
        for (int cc = 0; cc < 3; cc++) {
            double acc = 0;
            for (int p = 0; p < 2; p++)
                for (int q2 = 0; q2 < 2; q2++) acc += T[3 * p + r] * H[2 * p + q2] * T[3 * q2 + cc];
            GS3[3 * r + cc] = acc;
        }
    double HT[6];
    for (int p = 0; p < 2; p++)
        for (int cc = 0; cc < 3; cc++) HT[3 * p + cc] = H[2 * p] * T[cc] + H[2 * p + 1] * T[3 + cc];
    double GT[6];
    for (int p = 0; p < 2; p++)
        for (int cc = 0; cc < 3; cc++)
            GT[3 * p + cc] = 2.0 * (HT[3 * p] * fabs(f.S3[cc]) + HT[3 * p + 1] * fabs(f.S3[3 + cc]) +
                                    HT[3 * p + 2] * fabs(f.S3[6 + cc]));
    double GJ[6];
    for (int p = 0; p < 2; p++)
        for (int k = 0; k < 3; k++)
            GJ[3 * p + k] = GT[3 * p] * fabs(cam->R[3 * k]) + GT[3 * p + 1] * fabs(cam->R[3 * k + 1]) +
                            GT[3 * p + 2] * fabs(cam->R[3 * k + 2]);
    double fx = cam->fx, fy = cam->fy, z = f.z, x = fabs(f.pc[0]), y = fabs(f.pc[1]);
    double gpc[3] = {0, 0, 0};
    gpc[2] += GJ[0] * (fx / (z * z)) + GJ[4] * (fy / (z * z));
    if (!f.clx) { gpc[0] += GJ[2] * (fx / (z * z)); gpc[2] += GJ[2] * (2.0 * fx * x / (z * z * z)); }
    else gpc[2] += GJ[2] * (fx * fabs(f.txc) / (z * z));
    if (!f.cly) { gpc[1] += GJ[5] * (fy / (z * z)); gpc[2] += GJ[5] * (2.0 * fy * y / (z * z * z)); }
    else gpc[2] += GJ[5] * (fy * fabs(f.ty_c) / (z * z));
    gpc[0] += S[G_U] * fx / z;
    gpc[1] += S[G_V] * fy / z;
    gpc[2] += S[G_U] * (fx * x / (z * z)) + S[G_V] * (fy * y / (z * z));
    for (int k = 0; k < 3; k++)
        gm[k] += fabs(cam->R[k]) * gpc[0] + fabs(cam->R[3 + k]) * gpc[1] + fabs(cam->R[6 + k]) * gpc[2];
    double M[9];
    for (int k = 0; k < 9; k++) M[k] = fabs(f.M[k]);
    double GM[9];
    for (int r = 0; r < 3; r++)
        for (int cc = 0; cc < 3; cc++)
            GM[3 * r + cc] = 2.0 * (GS3[3 * r] * M[cc] + GS3[3 * r + 1] * M[3 + cc] + GS3[3 * r + 2] * M[6 + cc]);
    double GR[9];
    for (int j = 0; j < 3; j++) {
        double gsj = 0;
        for (int r = 0; r < 3; r++) { gsj += GM[3 * r + j] * fabs(f.Rq[3 * r + j]); GR[3 * r + j] = GM[3 * r + j] * f.sc[j]; }
        gs[j] += gsj * f.sc[j];
    }
    double w = fabs(f.qn[0]), qx = fabs(f.qn[1]), qy = fabs(f.qn[2]), qz = fabs(f.qn[3]);
    double gqn[4];
    gqn[0] = 2 * (qz * GR[1] + qy * GR[2] + qz * GR[3] + qx * GR[5] + qy * GR[6] + qx * GR[7]);
    gqn[1] = 2 * (qy * GR[1] + qz * GR[2] + qy * GR[3] + 2 * qx * GR[4] + w * GR[5] + qz * GR[6] + w * GR[7] + 2 * qx * GR[8]);
    gqn[2] = 2 * (2 * qy * GR[0] + qx * GR[1] + w * GR[2] + qx * GR[3] + qz * GR[5] + w * GR[6] + qz * GR[7] + 2 * qy * GR[8]);
    gqn[3] = 2 * (2 * qz * GR[0] + w * GR[1] + qx * GR[2] + w * GR[3] + 2 * qz * GR[4] + qy * GR[5] + qx * GR[6] + qy * GR[7]);
    double dotg = w * gqn[0] + qx * gqn[1] + qy * gqn[2] + qz * gqn[3];
    for (int k = 0; k < 4; k++) gq[k] += (gqn[k] + fabs(f.qn[k]) * dotg) / f.qnorm;
    double sg = sigmoid(s->opac[i]);
    go[0] += sg * (1 - sg) * S[G_SIG];
    double Cc[3];
    for (int k = 0; k < 3; k++)
        Cc[k] = -((double)cam->R[k] * cam->t[0] + (double)cam->R[3 + k] * cam->t[1] + (double)cam->R[6 + k] * cam->t[2]);
    double d[3] = {s->means[3 * i] - Cc[0], s->means[3 * i + 1] - Cc[1], s->means[3 * i + 2] - Cc[2]};
    double nd = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    double dir[3] = {d[0] / nd, d[1] / nd, d[2] / nd};
    /* a direction component is the rounded difference P_k - C_k: its size for the allowance is
       (|P_k| + |C_k|) / |d|, not |dir_k| (a component near 0 carries an absolute error) */
    double da[3];
    for (int k = 0; k < 3; k++) da[k] = (fabs((double)s->means[3 * i + k]) + fabs(Cc[k])) / nd;
    double Y[16], dY[16][3];
    sh_basis_abs(s->D, da[0], da[1], da[2], Y, dY);
    int K = (s->D + 1) * (s->D + 1);
    double gdir[3] = {0, 0, 0};
    const double gc[3] = {S[G_R], S[G_G], S[G_BL]};
    for (int ch = 0; ch < 3; ch++) {
        if (clamped[ch]) continue;
        for (int l = 0; l < K; l++) {
            gsh[l * 3 + ch] += Y[l] * gc[ch];
            double shv = fabs(s->sh[(i * K + l) * 3 + ch]);
            for (int k = 0; k < 3; k++) gdir[k] += gc[ch] * shv * dY[l][k];
        }
    }
    double dd = fabs(dir[0]) * gdir[0] + fabs(dir[1]) * gdir[1] + fabs(dir[2]) * gdir[2];
    for (int k = 0; k < 3; k++) gm[k] += (gdir[k] + fabs(dir[k]) * dd) / nd;
}

void orc_backward(int mode, int64_t n, int D, const float *means, const float *quats, const float *log_scales,
                  const float *opac, const float *sh, int V, const orc_camera *cams, const double *bg,
                  int64_t npix, const int32_t *pix, const double *dL_drgb, double *gm, double *gq, double *gs,
                  double *go, double *gsh, double *grad2d_norm, int32_t *flag_gauss, double *mag) {
    orc_scene s = {n, D, means, quats, log_scales, opac, sh};
    int K = (D + 1) * (D + 1);
    int P = 11 + 3 * K;
    memset(gm, 0, sizeof(double) * 3 * n); memset(gq, 0, sizeof(double) * 4 * n);
    memset(gs, 0, sizeof(double) * 3 * n); memset(go, 0, sizeof(double) * n);
    memset(gsh, 0, sizeof(double) * 3 * K * n);
    if (grad2d_norm) memset(grad2d_norm, 0, sizeof(double) * n);
    if (flag_gauss) memset(flag_gauss, 0, sizeof(int32_t) * n);
    if (mag) memset(mag, 0, sizeof(double) * P * n);
    int nth = orc_get_threads();
    for (int v = 0; v < V; v++) {
        orc_proj *pr = project_all(mode, &s, cams + v);
        int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
        int64_t m = depth_order(mode, pr, n, order);
        int64_t *slot = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
        for (int64_t i = 0; i < n; i++) slot[i] = -1;
        for (int64_t j = 0; j < m; j++) slot[order[j]] = j;
        double *g2 = (double *)calloc((size_t)nth * (m > 0 ? m : 1) * G_N, sizeof(double));
        double *s2 = mag ? (double *)calloc((size_t)nth * (m > 0 ? m : 1) * G_N, sizeof(double)) : NULL;
#pragma omp parallel num_threads(nth)
        {
            int tid = omp_get_thread_num();
            double *mine = g2 + (size_t)tid * (m > 0 ? m : 1) * G_N;
            double *mine_s = s2 ? s2 + (size_t)tid * (m > 0 ? m : 1) * G_N : NULL;
            int cap = 4096;
            orc_contrib *list = (orc_contrib *)malloc(sizeof(orc_contrib) * cap);
#pragma omp for schedule(dynamic, 16)
            for (int64_t q = 0; q < npix; q++) {
                if (pix[3 * q] != v) continue;
                int px = pix[3 * q + 2], py = pix[3 * q + 1];
                double rgb[3], Tf; int64_t last; int flag;
                int nc = composite_pixel(mode, pr, order, m, px, py, bg, rgb, &Tf, &last, &flag, list, cap);
                while (nc > cap) {
                    cap *= 2;
                    list = (orc_contrib *)realloc(list, sizeof(orc_contrib) * cap);
                    nc = composite_pixel(mode, pr, order, m, px, py, bg, rgb, &Tf, &last, &flag, list, cap);
                }
                const double *gpix = dL_drgb + 3 * q;
                if (flag && flag_gauss) {
                    /* every Gaussian evaluated at this pixel is marked (exclusion set) */
                    for (int64_t j = 0; j < m; j++) {
                        double dx, dy;
                        double p = pixel_power(mode, pr + order[j], px, py, &dx, &dy);
                        if (!(p > 0.0 || p < ORC_CUTOFF)) {
#pragma omp atomic write
                            flag_gauss[order[j]] = 1;
                        }
                    }
                }
                double acc[3] = {bg[0], bg[1], bg[2]};
                /* transmittance conditioning of this pixel (rounding allowance only): a relative
                   error delta in every alpha_j moves each T_k by up to sum_j alpha_j/(1-alpha_j)
                   delta relative -- d log T / d alpha_j = -1/(1-alpha_j) */
                double kappa = 1.0;
                if (mine_s)
                    for (int c = 0; c < nc; c++) kappa += list[c].alpha / (1.0 - list[c].alpha);
                for (int c = nc - 1; c >= 0; c--) {
                    const orc_contrib *e = list + c;
                    const orc_proj *g = pr + e->k;
                    double *G = mine + slot[e->k] * G_N;
                    double dLda = 0, dLda_mag = 0;
                    for (int ch = 0; ch < 3; ch++) {
                        G[G_R + ch] += gpix[ch] * e->alpha * e->T;
                        dLda += gpix[ch] * (g->rgb[ch] - acc[ch]);
                        dLda_mag += fabs(gpix[ch]) * (fabs(g->rgb[ch]) + fabs(acc[ch]));
                        acc[ch] = e->alpha * g->rgb[ch] + (1.0 - e->alpha) * acc[ch];
                    }
                    dLda *= e->T;
                    dLda_mag *= e->T * kappa;
                    double *S = mine_s ? mine_s + slot[e->k] * G_N : NULL;
                    if (S)
                        for (int ch = 0; ch < 3; ch++) S[G_R + ch] += fabs(gpix[ch] * e->alpha * e->T) * kappa;
                    if (e->clamped) continue; /* alpha = 0.99 constant */
                    G[G_SIG] += e->ep * dLda;
                    double dLdp = e->alpha * dLda;
                    double dx = e->dx, dy = e->dy;
                    G[G_U] += dLdp * (g->A * dx + g->B * dy);
                    G[G_V] += dLdp * (g->C * dy + g->B * dx);
                    G[G_A] += dLdp * (-0.5 * dx * dx);
                    G[G_B] += dLdp * (-dx * dy);
                    G[G_C] += dLdp * (-0.5 * dy * dy);
                    if (S) {
                        double pm = e->alpha * dLda_mag;
                        S[G_SIG] += e->ep * dLda_mag;
                        S[G_U] += pm * (fabs(g->A * dx) + fabs(g->B * dy));
                        S[G_V] += pm * (fabs(g->C * dy) + fabs(g->B * dx));
                        S[G_A] += pm * 0.5 * dx * dx;
                        S[G_B] += pm * fabs(dx * dy);
                        S[G_C] += pm * 0.5 * dy * dy;
                    }
                }
            }
            free(list);
        }
        /* reduce thread buffers in fixed order, then chain each Gaussian to 3D */
#pragma omp parallel for schedule(static) num_threads(nth)
        for (int64_t j = 0; j < m; j++) {
            double tot[G_N] = {0};
            for (int t = 0; t < nth; t++)
                for (int k = 0; k < G_N; k++) tot[k] += g2[((size_t)t * m + j) * G_N + k];
            int64_t i = order[j];
            chain_to_3d(&s, i, cams + v, tot, pr[i].clamped, gm + 3 * i, gq + 4 * i, gs + 3 * i, go + i,
                        gsh + (size_t)3 * K * i);
            if (grad2d_norm) grad2d_norm[i] += sqrt(tot[G_U] * tot[G_U] + tot[G_V] * tot[G_V]);
            if (mag) {
                double S[G_N] = {0};
                for (int t = 0; t < nth; t++)
                    for (int k = 0; k < G_N; k++) S[k] += s2[((size_t)t * m + j) * G_N + k];
                double *mg = mag + (size_t)P * i;
                chain_to_3d_abs(&s, i, cams + v, S, pr[i].clamped, mg, mg + 3, mg + 7, mg + 10, mg + 11);
            }
        }
        free(g2); free(s2); free(slot); free(order); free(pr);
    }
}

/* ---------------------------- loss (Eq. 4) ---------------------------------------- */
/* L = (1-lambda) mean|I_r - I_gt| + lambda (1 - mean SSIM), SSIM with
   an 11x11 Gaussian window sigma = 1.5, C1 = 0.01^2, C2 = 0.03^2, per channel, zero-padded
   'same'.  L1 subgradient at 0 is 0.
   Written as the plain definition: 2D windowed sums with w(i,j) = g(i) g(j).            */
#define ORC_WIN 11
static void ssim_window(double w[ORC_WIN]) {
    double s = 0;
    for (int i = 0; i < ORC_WIN; i++) { w[i] = exp(-((i - 5) * (i - 5)) / (2.0 * 1.5 * 1.5)); s += w[i]; }
    for (int i = 0; i < ORC_WIN; i++) w[i] /= s;
}

/* images [3][H][W]; loss and SSIM mean returned; dL [3][H][W] if non-NULL */
void orc_loss(const double *r, const double *gt, int H, int W, double lambda, double *loss, double *ssim_mean,
              double *dL, double *ssim_map) {
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
    double g[ORC_WIN];
    ssim_window(g);
    int64_t HW = (int64_t)H * W, N = 3 * HW;
    double *dA = (double *)calloc(N, sizeof(double)), *dB = (double *)calloc(N, sizeof(double)),
           *dC = (double *)calloc(N, sizeof(double));
    double l1 = 0, ssum = 0;
    for (int ch = 0; ch < 3; ch++) {
        const double *x = r + ch * HW, *y = gt + ch * HW;
#pragma omp parallel for schedule(static) reduction(+ : l1, ssum) num_threads(orc_get_threads())
        for (int py = 0; py < H; py++)
            for (int px = 0; px < W; px++) {
                double mx = 0, my = 0, exx = 0, eyy = 0, exy = 0;
                for (int i = 0; i < ORC_WIN; i++) {
                    int qy = py + i - 5;
                    if (qy < 0 || qy >= H) continue;
                    for (int j = 0; j < ORC_WIN; j++) {
                        int qx = px + j - 5;
                        if (qx < 0 || qx >= W) continue;
                        double wij = g[i] * g[j];
                        double xv = x[(int64_t)qy * W + qx], yv = y[(int64_t)qy * W + qx];
                        mx += wij * xv; my += wij * yv;
                        exx += wij * xv * xv; eyy += wij * yv * yv; exy += wij * xv * yv;
                    }
                }
                double sxx = exx - mx * mx, syy = eyy - my * my, sxy = exy - mx * my;
                double a1 = 2 * mx * my + C1, a2 = 2 * sxy + C2;
                double b1 = mx * mx + my * my + C1, b2 = sxx + syy + C2;
                double S = (a1 * a2) / (b1 * b2);
                ssum += S;
                if (ssim_map) ssim_map[ch * HW + (int64_t)py * W + px] = S;
                double d = x[(int64_t)py * W + px] - y[(int64_t)py * W + px];
                l1 += fabs(d);
                /* partials of S w.r.t. mu_x, sigma_x^2, sigma_xy, then w.r.t. raw moments */
                double dS_dmx = 2 * my * a2 / (b1 * b2) - S * 2 * mx / b1;
                double dS_dsxx = -S / b2;
                double dS_dsxy = 2 * a1 / (b1 * b2);
                int64_t o = ch * HW + (int64_t)py * W + px;
                dA[o] = dS_dmx + dS_dsxx * (-2 * mx) + dS_dsxy * (-my); /* d/d mu_x at fixed E */
                dB[o] = dS_dsxx;                                        /* d/d E[x^2] */
                dC[o] = dS_dsxy;                                        /* d/d E[xy]  */
            }
    }
    double ms = ssum / N;
    *loss = (1 - lambda) * l1 / N + lambda * (1 - ms);
    if (ssim_mean) *ssim_mean = ms;
    if (dL) {
        for (int ch = 0; ch < 3; ch++) {
            const double *x = r + ch * HW, *y = gt + ch * HW;
#pragma omp parallel for schedule(static) num_threads(orc_get_threads())
            for (int py = 0; py < H; py++)
                for (int px = 0; px < W; px++) {
                    double sa = 0, sb = 0, sc = 0;
                    for (int i = 0; i < ORC_WIN; i++) {
                        int qy = py + i - 5;
                        if (qy < 0 || qy >= H) continue;
                        for (int j = 0; j < ORC_WIN; j++) {
                            int qx = px + j - 5;
                            if (qx < 0 || qx >= W) continue;
                            double wij = g[i] * g[j];
                            int64_t o = ch * HW + (int64_t)qy * W + qx;
                            sa += wij * dA[o]; sb += wij * dB[o]; sc += wij * dC[o];
                        }
                    }
                    int64_t o = ch * HW + (int64_t)py * W + px;
                    double xv = x[(int64_t)py * W + px], yv = y[(int64_t)py * W + px];
                    double dssim = sa + 2 * xv * sb + yv * sc;
                    double d = xv - yv;
                    double sgn = d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0);
                    dL[o] = (1 - lambda) * sgn / N - lambda * dssim / N;
                }
        }
    }
    free(dA); free(dB); free(dC);
}

/* ---------------------------- Gaussian pyramid ------------------------------------ */
/* One level: blur with the 5-tap binomial [1,4,6,4,1]/16 in both directions with a      */
/* reflect-101 border, keep even rows/columns, output ceil(H/2) x ceil(W/2)              */
/* ("Gaussian smoothing and downsampling").       */
static int refl101(int i, int n) {
    if (n == 1) return 0;
    while (i < 0 || i >= n) {
        if (i < 0) i = -i;
        if (i >= n) i = 2 * (n - 1) - i;
    }
    return i;
}
void orc_pyramid_level(const double *in, int C, int H, int W, double *out) {
    const double k[5] = {1 / 16.0, 4 / 16.0, 6 / 16.0, 4 / 16.0, 1 / 16.0};
    int Ho = (H + 1) / 2, Wo = (W + 1) / 2;
    for (int c = 0; c < C; c++)
        for (int y = 0; y < Ho; y++)
            for (int x = 0; x < Wo; x++) {
                double acc = 0;
                for (int i = 0; i < 5; i++)
                    for (int j = 0; j < 5; j++)
                        acc += k[i] * k[j] * in[((int64_t)c * H + refl101(2 * y + i - 2, H)) * W + refl101(2 * x + j - 2, W)];
                out[((int64_t)c * Ho + y) * Wo + x] = acc;
            }
}

/* ---------------------------- optimiser step -------------------------------------- */
/* PAPER.md:568 "Stochastic Gradient Descent ... fixed learning rate"; Adam,
   bias-corrected, fixed lr per class; sgd_mode: p -= lr g.  Arrays of length cnt, all
   with the same lr (the caller splits by class).  step is 1-based. */
void orc_adam(int64_t cnt, double *p, const double *g, double *m, double *v, double lr, double beta1,
              double beta2, double eps, int64_t step, int sgd_mode) {
    double bc1 = 1.0 - pow(beta1, (double)step), bc2 = 1.0 - pow(beta2, (double)step);
    for (int64_t i = 0; i < cnt; i++) {
        if (sgd_mode) { p[i] -= lr * g[i]; continue; }
        m[i] = beta1 * m[i] + (1 - beta1) * g[i];
        v[i] = beta2 * v[i] + (1 - beta2) * g[i] * g[i];
        double mh = m[i] / bc1, vh = v[i] / bc2;
        p[i] -= lr * mh / (sqrt(vh) + eps);
    }
}

/* ---------------------------- densify and prune ------------------- */
/* SPEC.md:463-471 densify_and_prune ("splitting or cloning hyper primitives with
   large loss gradients similar to [kerbl2023]"), with DESIGN.md readings R27-R30:
   per Gaussian i (record rec[i][K] = P xyz | q wxyz | log s | logit | SH, the parameter rows of
   one Gaussian), statistics grad_accum[i] = sum of ||dL/dmean2d|| (pixels) over the visible
   (iteration, view) pairs, vis_count[i] = their number, max_radius[i] = the largest pixel radius;
   decisions in fp32 (the same IEEE operations as the GPU):
     mean  = vis_count > 0 ? grad_accum / vis_count : 0;   high = mean >= grad_thr
     large = max_j (float)exp((double)log s_j) > percent_dense * extent
     prune = logit < (float)log(op_thr / (1 - op_thr))  or  max_radius > max_screen
   class: prune -> 3 (removed); else high && !large -> 1 (clone); high && large -> 2 (split);
   else 0 (keep).  New map (row order): the kept and cloned originals in index order (bitwise
   copies), then one clone per clone parent (parent order), then two children per split parent
   (parent order, child 0 then 1).  A clone is the parent with P + R(q) diag(e^s) z[i][0]; split
   child c has P + R(q) diag(e^s) z[i][c] and log s - ln 1.6 (scale / 1.6); every other field
   (quaternion, opacity, SH) is copied.  New Gaussians get m = v = 0, originals keep theirs.
   z: [n][2][3] standard-normal samples (an input: the randomness the method draws).
   counts[4] = (clone, split, prune, n_new).  out_* may be NULL (counts only); otherwise they
   hold n_new records (double). */
void orc_densify(int64_t n, int K, const float *rec, const float *m, const float *v, const float *grad_accum,
                 const float *vis_count, const int32_t *max_radius, const float *z, float grad_thr,
                 float percent_dense, float extent, float op_thr, int32_t max_screen, int8_t *cls,
                 int64_t counts[4], double *out_rec, double *out_m, double *out_v) {
    const float logit_thr = (float)log((double)op_thr / (1.0 - (double)op_thr));
    const float big = percent_dense * extent;
    int64_t nc = 0, ns = 0, np_ = 0;
    for (int64_t i = 0; i < n; i++) {
        const float *r = rec + i * K;
        const float mean = vis_count[i] > 0.f ? grad_accum[i] / vis_count[i] : 0.f;
        const int high = mean >= grad_thr;
        float maxs = 0.f;
        for (int j = 0; j < 3; j++) {
            const float e = (float)exp((double)r[7 + j]);
            if (e > maxs) maxs = e;
        }
        const int large = maxs > big;
        const int prune = r[10] < logit_thr || max_radius[i] > max_screen;
        cls[i] = prune ? 3 : (high && !large) ? 1 : (high && large) ? 2 : 0;
        nc += cls[i] == 1;
        ns += cls[i] == 2;
        np_ += cls[i] == 3;
    }
    counts[0] = nc;
    counts[1] = ns;
    counts[2] = np_;
    counts[3] = n - np_ + nc + ns;
    if (!out_rec) return;
    int64_t o = 0;
    for (int64_t i = 0; i < n; i++)  /* kept and cloned originals */
        if (cls[i] == 0 || cls[i] == 1) {
            for (int k = 0; k < K; k++) {
                out_rec[o * K + k] = rec[i * K + k];
                out_m[o * K + k] = m[i * K + k];
                out_v[o * K + k] = v[i * K + k];
            }
            o++;
        }
    for (int pass = 1; pass <= 2; pass++)  /* clones, then split children */
        for (int64_t i = 0; i < n; i++) {
            if (cls[i] != pass) continue;
            const float *r = rec + i * K;
            double q[4] = {r[3], r[4], r[5], r[6]}, Rq[9];
            const double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
            for (int j = 0; j < 4; j++) q[j] = qn > 0.0 ? q[j] / qn : (j == 0);
            quat_to_rot(q, Rq);
            double e[3];
            for (int j = 0; j < 3; j++) e[j] = exp((double)r[7 + j]);
            for (int c = 0; c < pass; c++) {
                const float *zz = z + (i * 2 + c) * 3;
                for (int k = 0; k < K; k++) {
                    out_rec[o * K + k] = r[k];
                    out_m[o * K + k] = 0.0;
                    out_v[o * K + k] = 0.0;
                }
                for (int a = 0; a < 3; a++) {
                    double d = 0.0;
                    for (int j = 0; j < 3; j++) d += Rq[3 * a + j] * e[j] * zz[j];
                    out_rec[o * K + a] = (double)r[a] + d;
                }
                if (pass == 2)
                    for (int j = 0; j < 3; j++) out_rec[o * K + 7 + j] = (double)r[7 + j] - log(1.6);
                o++;
            }
        }
}

/* ---------------------------- geometry-based densification -------- */
/* SPEC.md:473-481 geometry_densify ("actively create additional temporary hyper
   primitives based on the inactive 2D feature points"), initialisation as create_map_points
   (SPEC.md:261), with DESIGN.md readings R31-R33.  Keypoint k at pixel (u, v); active[k] != 0 if
   it observes a map primitive (its camera-space depth kp_depth[k]).  For every INACTIVE keypoint,
   in index order:
     RGB-D (mode 1): d = depth_map[round(v)][round(u)] (nearest pixel); skipped if d <= 0;
     mono (mode 0): among active keypoints with squared pixel distance <= rho^2 (fp32:
       fmaf(dx, dx, dy * dy)), the K = 4 nearest (ties: lower index) -> d = sum(w_i d_i) / sum(w_i)
       with w_i = 1 / dist_i (an exactly coincident neighbour: the mean of the coincident depths);
       skipped if none.
   New primitive: P = R^T (d ((u - cx) / fx, (v - cy) / fy, 1) - t); q = (1, 0, 0, 0);
   log s = log(d / fx) on all three axes; logit = logit(0.1); SH DC c = (pixel colour - 0.5) / C0
   with the nearest pixel's colour (so the degree-0 colour equals the pixel), higher SH 0.
   out_rec [count][K] (K = 11 + 3(D+1)^2, NULL: count only); src[count] = keypoint index.
   Returns count. */
int64_t orc_geometry_densify(const orc_camera *cam, int64_t nk, const float *uv, const int32_t *active,
                             const float *kp_depth, const float *depth_map, const float *image, int mode, int D,
                             float rho, double *out_rec, int32_t *src) {
    const int K = 11 + 3 * (D + 1) * (D + 1);
    const int W = cam->width, H = cam->height;
    const double C0 = 0.28209479177387814;
    int64_t cnt = 0;
    for (int64_t k = 0; k < nk; k++) {
        if (active[k]) continue;
        const float u = uv[2 * k], v = uv[2 * k + 1];
        const int px = (int)lrintf(u), py = (int)lrintf(v);
        if (px < 0 || px >= W || py < 0 || py >= H) continue;
        double d = 0.0;
        if (mode == 1) {
            d = depth_map[(int64_t)py * W + px];
            if (!(d > 0.0)) continue;
        } else {
            int best[4];
            float bd[4];
            int nb = 0;
            const float r2 = rho * rho;
            for (int64_t j = 0; j < nk; j++) {
                if (!active[j]) continue;
                const float dx = uv[2 * j] - u, dy = uv[2 * j + 1] - v;
                const float d2 = fmaf(dx, dx, dy * dy);
                if (!(d2 <= r2)) continue;
                /* insert into the sorted top-4 (strictly smaller distance moves ahead; equal
                   distances keep index order because j ascends) */
                int pos = nb;
                while (pos > 0 && d2 < bd[pos - 1]) pos--;
                if (pos >= 4) continue;
                for (int q = (nb < 4 ? nb : 3); q > pos; q--) {
                    bd[q] = bd[q - 1];
                    best[q] = best[q - 1];
                }
                bd[pos] = d2;
                best[pos] = (int)j;
                if (nb < 4) nb++;
            }
            if (nb == 0) continue;
            double sw = 0.0, swd = 0.0, zsum = 0.0;
            int nz = 0;
            for (int q = 0; q < nb; q++) {
                if (bd[q] == 0.f) {
                    zsum += kp_depth[best[q]];
                    nz++;
                }
                const double w = 1.0 / sqrt((double)bd[q]);
                sw += w;
                swd += w * kp_depth[best[q]];
            }
            d = nz ? zsum / nz : swd / sw;
        }
        if (out_rec) {
            double *o = out_rec + cnt * K;
            for (int q = 0; q < K; q++) o[q] = 0.0;
            const double xc[3] = {d * ((double)u - cam->cx) / cam->fx, d * ((double)v - cam->cy) / cam->fy, d};
            for (int a = 0; a < 3; a++) { /* P = R^T (p_c - t) */
                double s = 0.0;
                for (int b = 0; b < 3; b++) s += (double)cam->R[3 * b + a] * (xc[b] - (double)cam->t[b]);
                o[a] = s;
            }
            o[3] = 1.0;
            for (int a = 0; a < 3; a++) o[7 + a] = log(d / cam->fx);
            o[10] = log(0.1 / 0.9);
            for (int ch = 0; ch < 3; ch++)
                o[11 + ch] = ((double)image[(int64_t)ch * H * W + (int64_t)py * W + px] - 0.5) / C0;
            src[cnt] = (int32_t)k;
        }
        cnt++;
    }
    return cnt;
}
