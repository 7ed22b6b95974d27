/* TEST INFRASTRUCTURE ONLY — CPU oracle for the 3-D front end.
 *
 * The reference is a 2-D analog of 3DGS and has NO 3-D code, tests or vectors (SURVEY.md §8a
 * A3b): this front end is required by BASELINE.json's north_star item (1)
 * ("EWA projection to 2D covariance, SH-degree-3 colour evaluation, radius/tile-rect culling").
 * It restates the published 3DGS algorithm (Kerbl et al., SIGGRAPH 2023, §4 and its public
 * rasterizer's preprocess/backward): camera transform, perspective mean, EWA covariance
 * Σ2 = J W Σ3 Wᵀ Jᵀ with the 1.3·tan(fov) clamp of the Jacobian, Σ3 = R S Sᵀ Rᵀ from a
 * normalised quaternion and log-scales, SH degree 3 colour + 0.5 clamped at 0, sigmoid opacity.
 * Everything after the 2-D record — low-pass bump (dilation.hpp:67-80), inverse, 3σ extents
 * (rasterizer.cpp:23-46), tile grid, blending and its backward — is the reference's own 2-D path
 * (or_render_prepared / or_backward_prepared, restated from rasterizer.cpp and pinned against it).
 *
 * PARITY UNPINNED at the reference: no reference code exists for this row. The restatement is
 * pinned instead by (a) known-answer values from the formulas (tests/test_oracle3d.py) and
 * (b) central finite differences of or3d_project in FP64 against or3d_chain, the same check the
 * reference's own FP64 instantiation exists for.
 *
 * Arithmetic: FP64 throughout; the 2-D records are rounded to float for the blend.
 *
 * Parameter layout per Gaussian (59 floats, SoA [59][n] for the model functions):
 *   0-2 mean (world)   3-6 quaternion (w, x, y, z; normalised in the forward)
 *   7-9 log-scales      10 raw opacity      11 + 3k + c: SH coefficient k (0..15) of channel c
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "tgs_oracle.h"

static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* Real SH basis up to degree 3 at a unit direction and its partial derivatives (treating x, y,
 * z as independent; the normalisation is chained separately). */
void or3d_sh_basis(double x, double y, double z, double* b /*16*/, double* db /*16x3*/) {
    const double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    double d[16][3];
    memset(d, 0, sizeof(d));
    b[0] = SH_C0;
    b[1] = -SH_C1 * y;  d[1][1] = -SH_C1;
    b[2] = SH_C1 * z;   d[2][2] = SH_C1;
    b[3] = -SH_C1 * x;  d[3][0] = -SH_C1;
    b[4] = SH_C2[0] * xy;               d[4][0] = SH_C2[0] * y;  d[4][1] = SH_C2[0] * x;
    b[5] = SH_C2[1] * yz;               d[5][1] = SH_C2[1] * z;  d[5][2] = SH_C2[1] * y;
    b[6] = SH_C2[2] * (2 * zz - xx - yy);
    d[6][0] = -2 * SH_C2[2] * x; d[6][1] = -2 * SH_C2[2] * y; d[6][2] = 4 * SH_C2[2] * z;
    b[7] = SH_C2[3] * xz;               d[7][0] = SH_C2[3] * z;  d[7][2] = SH_C2[3] * x;
    b[8] = SH_C2[4] * (xx - yy);        d[8][0] = 2 * SH_C2[4] * x; d[8][1] = -2 * SH_C2[4] * y;
    b[9] = SH_C3[0] * y * (3 * xx - yy);
    d[9][0] = 6 * SH_C3[0] * xy; d[9][1] = SH_C3[0] * (3 * xx - 3 * yy);
    b[10] = SH_C3[1] * xy * z;
    d[10][0] = SH_C3[1] * yz; d[10][1] = SH_C3[1] * xz; d[10][2] = SH_C3[1] * xy;
    b[11] = SH_C3[2] * y * (4 * zz - xx - yy);
    d[11][0] = -2 * SH_C3[2] * xy; d[11][1] = SH_C3[2] * (4 * zz - xx - 3 * yy);
    d[11][2] = 8 * SH_C3[2] * yz;
    b[12] = SH_C3[3] * z * (2 * zz - 3 * xx - 3 * yy);
    d[12][0] = -6 * SH_C3[3] * xz; d[12][1] = -6 * SH_C3[3] * yz;
    d[12][2] = SH_C3[3] * (6 * zz - 3 * xx - 3 * yy);
    b[13] = SH_C3[4] * x * (4 * zz - xx - yy);
    d[13][0] = SH_C3[4] * (4 * zz - 3 * xx - yy); d[13][1] = -2 * SH_C3[4] * xy;
    d[13][2] = 8 * SH_C3[4] * xz;
    b[14] = SH_C3[5] * z * (xx - yy);
    d[14][0] = 2 * SH_C3[5] * xz; d[14][1] = -2 * SH_C3[5] * yz; d[14][2] = SH_C3[5] * (xx - yy);
    b[15] = SH_C3[6] * x * (xx - 3 * yy);
    d[15][0] = SH_C3[6] * (3 * xx - 3 * yy); d[15][1] = -6 * SH_C3[6] * xy;
    if (db) memcpy(db, d, sizeof(d));
}

/* Everything the forward computes for one Gaussian (kept for the chain rule). */
typedef struct {
    double tc[3], iz, cxz, cyz;
    int clx, cly;
    double J00, J02, J11, J12, T[2][3];
    double qn[4], qnorm, Rq[3][3], s[3], M[3][3], S3[3][3];
    double s00, s01, s11;
    double alpha;
    double dir[3], dlen, b[16], db[16][3], raw[3];
} fwd3d_t;

/* Returns 1 visible, 0 culled (camera depth <= znear), -1 invalid (non-finite, zero quaternion). */
static int forward_one(const double* th, const or_camera* cam, double bump, fwd3d_t* f) {
    for (int k = 0; k < OR3D_PARAMS; ++k)
        if (!isfinite(th[k])) return -1;
    const double* R = cam->R;
    for (int i = 0; i < 3; ++i)
        f->tc[i] = R[3 * i] * th[0] + R[3 * i + 1] * th[1] + R[3 * i + 2] * th[2] + cam->t[i];
    if (!(f->tc[2] > cam->znear)) return 0;
    const double tz = f->tc[2];
    f->iz = 1.0 / tz;
    const double limx = 1.3 * 0.5 * (double)cam->W / cam->fx;
    const double limy = 1.3 * 0.5 * (double)cam->H / cam->fy;
    const double rx = f->tc[0] * f->iz, ry = f->tc[1] * f->iz;
    f->clx = rx < -limx || rx > limx;
    f->cly = ry < -limy || ry > limy;
    f->cxz = rx < -limx ? -limx : (rx > limx ? limx : rx);
    f->cyz = ry < -limy ? -limy : (ry > limy ? limy : ry);
    f->J00 = cam->fx * f->iz;
    f->J02 = -cam->fx * f->cxz * f->iz;
    f->J11 = cam->fy * f->iz;
    f->J12 = -cam->fy * f->cyz * f->iz;
    for (int j = 0; j < 3; ++j) {
        f->T[0][j] = f->J00 * R[j] + f->J02 * R[6 + j];
        f->T[1][j] = f->J11 * R[3 + j] + f->J12 * R[6 + j];
    }
    /* Σ3 = (Rq S)(Rq S)ᵀ */
    const double qw = th[3], qx = th[4], qy = th[5], qz = th[6];
    f->qnorm = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    if (!(f->qnorm > 0)) return -1;
    const double r = qw / f->qnorm, x = qx / f->qnorm, y = qy / f->qnorm, z = qz / f->qnorm;
    f->qn[0] = r; f->qn[1] = x; f->qn[2] = y; f->qn[3] = z;
    double (*Q)[3] = f->Rq;
    Q[0][0] = 1 - 2 * (y * y + z * z); Q[0][1] = 2 * (x * y - r * z); Q[0][2] = 2 * (x * z + r * y);
    Q[1][0] = 2 * (x * y + r * z); Q[1][1] = 1 - 2 * (x * x + z * z); Q[1][2] = 2 * (y * z - r * x);
    Q[2][0] = 2 * (x * z - r * y); Q[2][1] = 2 * (y * z + r * x); Q[2][2] = 1 - 2 * (x * x + y * y);
    for (int j = 0; j < 3; ++j) f->s[j] = exp(th[7 + j]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) f->M[i][j] = Q[i][j] * f->s[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            f->S3[i][j] = f->M[i][0] * f->M[j][0] + f->M[i][1] * f->M[j][1] + f->M[i][2] * f->M[j][2];
    /* Σ2 = T Σ3 Tᵀ, plus the low-pass bump (dilation.hpp:73-80) */
    double U[2][3];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            U[i][j] = f->T[i][0] * f->S3[0][j] + f->T[i][1] * f->S3[1][j] + f->T[i][2] * f->S3[2][j];
    f->s00 = U[0][0] * f->T[0][0] + U[0][1] * f->T[0][1] + U[0][2] * f->T[0][2] + bump;
    f->s01 = U[0][0] * f->T[1][0] + U[0][1] * f->T[1][1] + U[0][2] * f->T[1][2];
    f->s11 = U[1][0] * f->T[1][0] + U[1][1] * f->T[1][1] + U[1][2] * f->T[1][2] + bump;
    f->alpha = 1.0 / (1.0 + exp(-th[10]));
    /* view direction from the camera centre C = -Rᵀ t */
    double C[3];
    for (int j = 0; j < 3; ++j) C[j] = -(R[j] * cam->t[0] + R[3 + j] * cam->t[1] + R[6 + j] * cam->t[2]);
    double d[3] = {th[0] - C[0], th[1] - C[1], th[2] - C[2]};
    f->dlen = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    for (int j = 0; j < 3; ++j) f->dir[j] = d[j] / f->dlen;
    or3d_sh_basis(f->dir[0], f->dir[1], f->dir[2], f->b, &f->db[0][0]);
    for (int c = 0; c < 3; ++c) {
        double acc = 0.5;
        for (int k = 0; k < 16; ++k) acc += f->b[k] * th[11 + 3 * k + c];
        f->raw[c] = acc;
    }
    return 1;
}

int or3d_project(const double* theta, const or_camera* cam, double bump, double* out) {
    fwd3d_t f;
    const int v = forward_one(theta, cam, bump, &f);
    if (v != 1) return v;
    out[0] = cam->fx * f.tc[0] * f.iz + cam->cx;
    out[1] = cam->fy * f.tc[1] * f.iz + cam->cy;
    out[2] = f.s00; out[3] = f.s01; out[4] = f.s11;
    out[5] = f.alpha;
    for (int c = 0; c < 3; ++c) out[6 + c] = f.raw[c] > 0 ? f.raw[c] : 0.0;
    out[9] = f.tc[2];
    out[10] = 3.0 * sqrt(f.s00);
    out[11] = 3.0 * sqrt(f.s11);
    return 1;
}

void or3d_chain(const double* th, const or_camera* cam, double bump, const double* g, double* grad) {
    fwd3d_t f;
    memset(grad, 0, sizeof(double) * OR3D_PARAMS);
    if (forward_one(th, cam, bump, &f) != 1) return;
    const double* R = cam->R;
    const double gu = g[0], gv = g[1], m00 = g[2], m01 = g[3], m11 = g[4];
    /* colour: clamp at 0 passes the gradient where the raw value is >= 0 */
    double dcol[3], ddir[3] = {0, 0, 0};
    for (int c = 0; c < 3; ++c) dcol[c] = f.raw[c] < 0 ? 0.0 : g[6 + c];
    for (int k = 0; k < 16; ++k) {
        double wk = 0;
        for (int c = 0; c < 3; ++c) {
            grad[11 + 3 * k + c] = f.b[k] * dcol[c];
            wk += dcol[c] * th[11 + 3 * k + c];
        }
        for (int j = 0; j < 3; ++j) ddir[j] += wk * f.db[k][j];
    }
    const double dd = ddir[0] * f.dir[0] + ddir[1] * f.dir[1] + ddir[2] * f.dir[2];
    double dmu[3];
    for (int j = 0; j < 3; ++j) dmu[j] = (ddir[j] - f.dir[j] * dd) / f.dlen;
    /* opacity */
    grad[10] = g[5] * f.alpha * (1.0 - f.alpha);
    /* mean projection */
    const double fx = cam->fx, fy = cam->fy, iz = f.iz, iz2 = iz * iz;
    double dt[3];
    dt[0] = gu * fx * iz;
    dt[1] = gv * fy * iz;
    dt[2] = -(gu * fx * f.tc[0] + gv * fy * f.tc[1]) * iz2;
    /* covariance: G = [[m00, m01], [m01, m11]] = dL/dΣ2 (symmetric convention of the 2-D sums) */
    const double G[2][2] = {{m00, m01}, {m01, m11}};
    double GT[2][3], dS3[3][3], dT[2][3];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) GT[i][j] = G[i][0] * f.T[0][j] + G[i][1] * f.T[1][j];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) dS3[a][b] = f.T[0][a] * GT[0][b] + f.T[1][a] * GT[1][b];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            dT[i][j] = 2.0 * (GT[i][0] * f.S3[0][j] + GT[i][1] * f.S3[1][j] + GT[i][2] * f.S3[2][j]);
    /* T = J W: dJ = dT Wᵀ (only the four non-zero entries of J depend on the mean) */
    const double dJ00 = dT[0][0] * R[0] + dT[0][1] * R[1] + dT[0][2] * R[2];
    const double dJ02 = dT[0][0] * R[6] + dT[0][1] * R[7] + dT[0][2] * R[8];
    const double dJ11 = dT[1][0] * R[3] + dT[1][1] * R[4] + dT[1][2] * R[5];
    const double dJ12 = dT[1][0] * R[6] + dT[1][1] * R[7] + dT[1][2] * R[8];
    dt[2] += -fx * iz2 * dJ00 - fy * iz2 * dJ11;
    /* J02 = -fx cxz / tz: unclamped cxz = tx / tz, clamped cxz constant */
    if (f.clx) {
        dt[2] += dJ02 * fx * f.cxz * iz2;
    } else {
        dt[0] += dJ02 * (-fx * iz2);
        dt[2] += dJ02 * 2.0 * fx * f.cxz * iz2;
    }
    if (f.cly) {
        dt[2] += dJ12 * fy * f.cyz * iz2;
    } else {
        dt[1] += dJ12 * (-fy * iz2);
        dt[2] += dJ12 * 2.0 * fy * f.cyz * iz2;
    }
    for (int j = 0; j < 3; ++j) grad[j] = R[j] * dt[0] + R[3 + j] * dt[1] + R[6 + j] * dt[2] + dmu[j];
    /* Σ3 = M Mᵀ: dM = 2 dΣ3 M; M = Rq diag(s) */
    double dM[3][3], dR[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            dM[i][j] = 2.0 * (dS3[i][0] * f.M[0][j] + dS3[i][1] * f.M[1][j] + dS3[i][2] * f.M[2][j]);
    for (int j = 0; j < 3; ++j) {
        double ds = 0;
        for (int i = 0; i < 3; ++i) {
            dR[i][j] = dM[i][j] * f.s[j];
            ds += dM[i][j] * f.Rq[i][j];
        }
        grad[7 + j] = ds * f.s[j];
    }
    const double r = f.qn[0], x = f.qn[1], y = f.qn[2], z = f.qn[3];
    double dq[4];
    dq[0] = 2 * (-z * dR[0][1] + y * dR[0][2] + z * dR[1][0] - x * dR[1][2] - y * dR[2][0] + x * dR[2][1]);
    dq[1] = 2 * (y * dR[0][1] + z * dR[0][2] + y * dR[1][0] - 2 * x * dR[1][1] - r * dR[1][2] +
                 z * dR[2][0] + r * dR[2][1] - 2 * x * dR[2][2]);
    dq[2] = 2 * (-2 * y * dR[0][0] + x * dR[0][1] + r * dR[0][2] + x * dR[1][0] + z * dR[1][2] -
                 r * dR[2][0] + z * dR[2][1] - 2 * y * dR[2][2]);
    dq[3] = 2 * (-2 * z * dR[0][0] - r * dR[0][1] + x * dR[0][2] + r * dR[1][0] - 2 * z * dR[1][1] +
                 y * dR[1][2] + x * dR[2][0] + y * dR[2][1]);
    const double qd = r * dq[0] + x * dq[1] + y * dq[2] + z * dq[3];
    for (int k = 0; k < 4; ++k) grad[3 + k] = (dq[k] - f.qn[k] * qd) / f.qnorm;
}

/* ---------------------------------------------------------------- whole model */
static const float* g_depth3d;
static int cmp_depth3d(const void* a, const void* b) {
    const uint32_t i = *(const uint32_t*)a, j = *(const uint32_t*)b;
    const float di = g_depth3d[i], dj = g_depth3d[j];
    if (di != dj) return di < dj ? -1 : 1;
    return i < j ? -1 : (i > j ? 1 : 0);
}

static void gather_theta(const float* params, int64_t n, int64_t i, double* th) {
    for (int k = 0; k < OR3D_PARAMS; ++k) th[k] = (double)params[(size_t)k * (size_t)n + (size_t)i];
}

/* Records of the visible Gaussians in blend order (ascending float depth, ties by row), orig =
 * row. Returns 0, or 1 for an invalid Gaussian (the GPU's TGSX_EINVAL). */
int or3d_prepare(const float* params, int64_t n, const or_camera* cam, int lowpass_p,
                 or_prepared* out, float* depth_out, int64_t* out_visible) {
    if (lowpass_p < 1) return 1;
    const double bump = 0.3 + 0.5 * (double)(lowpass_p - 1);
    const size_t nn = (size_t)(n ? n : 1);
    float* rec = (float*)malloc(sizeof(float) * 12 * nn);
    float* depth = (float*)malloc(sizeof(float) * nn);
    uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * nn);
    int64_t nv = 0;
    int rc = 0;
    for (int64_t i = 0; i < n; ++i) {
        double th[OR3D_PARAMS], o[12];
        gather_theta(params, n, i, th);
        const int v = or3d_project(th, cam, bump, o);
        if (v < 0) { rc = 1; break; }
        if (v == 0) continue;
        const double det = o[2] * o[4] - o[3] * o[3];
        if (!(det > 0)) { rc = 2; break; }
        float* r = rec + 12 * (size_t)i;
        r[0] = (float)o[0]; r[1] = (float)o[1];
        r[2] = (float)(o[4] / det); r[3] = (float)(-o[3] / det); r[4] = (float)(o[2] / det);
        r[5] = (float)o[5]; r[6] = (float)o[6]; r[7] = (float)o[7]; r[8] = (float)o[8];
        r[9] = (float)o[10]; r[10] = (float)o[11];
        depth[i] = (float)o[9];
        order[nv++] = (uint32_t)i;
    }
    if (rc == 0) {
        g_depth3d = depth;
        qsort(order, (size_t)nv, sizeof(uint32_t), cmp_depth3d);
        for (int64_t k = 0; k < nv; ++k) {
            const float* r = rec + 12 * (size_t)order[k];
            out->mx[k] = r[0]; out->my[k] = r[1];
            out->i00[k] = r[2]; out->i01[k] = r[3]; out->i11[k] = r[4];
            out->alpha[k] = r[5];
            out->c0[k] = r[6]; out->c1[k] = r[7]; out->c2[k] = r[8];
            out->rx[k] = r[9]; out->ry[k] = r[10];
            out->orig[k] = order[k];
            if (depth_out) depth_out[k] = depth[order[k]];
        }
        *out_visible = nv;
    }
    free(rec); free(depth); free(order);
    return rc;
}

typedef struct {
    or_prepared sp;
    float* buf;
    uint32_t* orig;
    int64_t nv;
} prep3d_t;

static int prep3d(const float* params, int64_t n, const or_camera* cam, int lowpass_p, prep3d_t* p) {
    const size_t nn = (size_t)(n ? n : 1);
    p->buf = (float*)malloc(sizeof(float) * 11 * nn);
    p->orig = (uint32_t*)malloc(sizeof(uint32_t) * nn);
    float* b = p->buf;
    or_prepared* sp = &p->sp;
    sp->mx = b; sp->my = b + nn; sp->i00 = b + 2 * nn; sp->i01 = b + 3 * nn;
    sp->i11 = b + 4 * nn; sp->alpha = b + 5 * nn; sp->c0 = b + 6 * nn; sp->c1 = b + 7 * nn;
    sp->c2 = b + 8 * nn; sp->rx = b + 9 * nn; sp->ry = b + 10 * nn; sp->orig = p->orig;
    return or3d_prepare(params, n, cam, lowpass_p, sp, NULL, &p->nv);
}

int or3d_render(const float* params, int64_t n, const or_camera* cam, int p, int ox, int oy,
                const float* bg, int lowpass_p, float* out_rgb, float* out_T, uint64_t* out_ops,
                uint64_t* out_evals) {
    prep3d_t pp;
    int rc = prep3d(params, n, cam, lowpass_p > 0 ? lowpass_p : p, &pp);
    if (rc == 0)
        rc = or_render_prepared(&pp.sp, pp.nv, p, ox, oy, cam->W, cam->H, bg, out_rgb, out_T,
                                out_ops, out_evals);
    free(pp.buf); free(pp.orig);
    return rc;
}

/* grads [59][n] (row order, zero for unseen Gaussians); screen [10][n] row order (may be NULL
 * members). The chain rule is evaluated in FP64 on the FP32 screen sums. */
int or3d_backward(const float* params, int64_t n, const or_camera* cam, int p, int ox, int oy,
                  const float* bg, const float* dLdC, int lowpass_p, float* grads,
                  or_screen_grads* screen) {
    const int lp = lowpass_p > 0 ? lowpass_p : p;
    prep3d_t pp;
    int rc = prep3d(params, n, cam, lp, &pp);
    if (rc) { free(pp.buf); free(pp.orig); return rc; }
    const size_t nn = (size_t)(n ? n : 1);
    float* acc = (float*)calloc(10 * nn, sizeof(float));
    uint8_t* touched = (uint8_t*)calloc(nn, 1);
    or_screen_grads sg = {acc, acc + nn, acc + 2 * nn, acc + 3 * nn, acc + 4 * nn, acc + 5 * nn,
                          acc + 6 * nn, acc + 7 * nn, acc + 8 * nn, acc + 9 * nn, touched};
    rc = or_backward_prepared(&pp.sp, pp.nv, n, p, ox, oy, cam->W, cam->H, bg, dLdC, &sg);
    const double bump = 0.3 + 0.5 * (double)(lp - 1);
    for (int64_t i = 0; rc == 0 && i < n; ++i) {
        double th[OR3D_PARAMS], g[9], gr[OR3D_PARAMS];
        for (int q = 0; q < 9; ++q) g[q] = (double)acc[(size_t)q * nn + (size_t)i];
        if (touched[i]) {
            gather_theta(params, n, i, th);
            or3d_chain(th, cam, bump, g, gr);
        } else {
            memset(gr, 0, sizeof(gr));
        }
        for (int k = 0; k < OR3D_PARAMS; ++k) grads[(size_t)k * (size_t)n + (size_t)i] = (float)gr[k];
    }
    if (screen) {
        float* dst[10] = {screen->gmx, screen->gmy, screen->gs00, screen->gs01, screen->gs11,
                          screen->galpha, screen->gc0, screen->gc1, screen->gc2, screen->maxw};
        for (int q = 0; q < 10; ++q)
            if (dst[q]) memcpy(dst[q], acc + (size_t)q * nn, sizeof(float) * (size_t)n);
        if (screen->touched) memcpy(screen->touched, touched, (size_t)n);
    }
    free(acc); free(touched); free(pp.buf); free(pp.orig);
    return rc;
}

/* Adam for the 3-D parameters: the 2-D update (or_adam_step) with the 3DGS
 * per-group learning rates; raw opacity clamped to [-12, 12] (gaussian.hpp:105-116). FP32 with
 * the same operation order as the GPU kernel (bit-exact given equal gradients). */
void or3d_adam_config(or3d_adam_cfg* c, int64_t step, int64_t total_steps, double extent) {
    c->beta1 = 0.9f;
    c->beta2 = 0.999f;
    c->eps = 1e-15f;
    const double frac = total_steps > 0 ? (double)step / (double)total_steps : 0.0;
    c->lr_pos = (float)(1.6e-4 * extent * pow(0.01, frac));
    c->lr_rot = 1e-3f;
    c->lr_scale = 5e-3f;
    c->lr_opacity = 5e-2f;
    c->lr_dc = 2.5e-3f;
    c->lr_rest = 2.5e-3f / 20.0f;
    c->bc1 = (float)(1.0 - pow(0.9, (double)step));
    c->bc2 = (float)(1.0 - pow(0.999, (double)step));
    c->raw_cap = 12.0f;
}

float or3d_lr(const or3d_adam_cfg* c, int k) {
    if (k < 3) return c->lr_pos;
    if (k < 7) return c->lr_rot;
    if (k < 10) return c->lr_scale;
    if (k == 10) return c->lr_opacity;
    if (k < 14) return c->lr_dc;
    return c->lr_rest;
}

void or3d_adam_step(float* params, const float* grads, float* m, float* v, int64_t n,
                    const or3d_adam_cfg* c) {
    const float omb1 = 1.0f - c->beta1, omb2 = 1.0f - c->beta2;
    for (int k = 0; k < OR3D_PARAMS; ++k) {
        const float lr = or3d_lr(c, k);
        for (int64_t i = 0; i < n; ++i) {
            const size_t o = (size_t)k * (size_t)n + (size_t)i;
            const float g = grads[o];
            const float mm = c->beta1 * m[o] + omb1 * g;
            const float vv = c->beta2 * v[o] + (omb2 * g) * g;
            m[o] = mm;
            v[o] = vv;
            const float mh = mm / c->bc1;
            const float vh = vv / c->bc2;
            float th = params[o] - (lr * mh) / (sqrtf(vh) + c->eps);
            if (k == 10) th = th < -c->raw_cap ? -c->raw_cap : (c->raw_cap < th ? c->raw_cap : th);
            params[o] = th;
        }
    }
}

/* ---------------------------------------------------------------- 3-D densification
 * The 2-D densify event (tgs_oracle.c or_densify_event) restated on the 3-D
 * parameters, the specification the GPU's tgsx_densify3d (csrc/densify3d.cu) is checked
 * against. No reference code exists for it (the reference densifier is 2-D and missing):
 *   coin (one draw) -> select: accum = visit - visit_evt > 0, visit > tau_v, activate(raw
 *   opacity) >= mask floor, averaged position norm > tau_pos or (coin and averaged colour norm >
 *   tau_color) -> cap to budget - n (top-k by averaged position norm, ties by lower index) ->
 *   spawn in parent-index order, 3 draws per child: radius cbrt(u1), z = 1 - 2 u2, phi = 2 pi
 *   u3 -> a point uniform in the unit ball, mapped through R(q) diag(exp(log-scales)) (the
 *   parent's 1-sigma ellipsoid; double arithmetic, rounded to float at the end); log-scales -
 *   ln 2 (float), quaternion and SH copied, raw opacity = inverse_activate(0.1), id = next_id++,
 *   tau_v = tau_v_init, zero statistics and moments -> prune activate(raw opacity) < prune
 *   floor, order-preserving over every array -> reset (sums zero, visit_evt = visit). */
static const float* g3_key;
static int cmp3_desc_key(const void* a, const void* b) {
    const int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
    if (g3_key[i] != g3_key[j]) return g3_key[i] > g3_key[j] ? -1 : 1;
    return i < j ? -1 : (i > j ? 1 : 0);
}

static void or3d_copy_row(or3d_model* s, int64_t dst, int64_t src) {
    const int64_t cap = s->cap;
    for (int k = 0; k < OR3D_PARAMS; ++k) {
        s->params[k * cap + dst] = s->params[k * cap + src];
        s->m1[k * cap + dst] = s->m1[k * cap + src];
        s->m2[k * cap + dst] = s->m2[k * cap + src];
    }
    s->pos_acc[dst] = s->pos_acc[src];
    s->col_acc[dst] = s->col_acc[src];
    s->visit[dst] = s->visit[src];
    s->visit_evt[dst] = s->visit_evt[src];
    s->visit_aud[dst] = s->visit_aud[src];
    s->id[dst] = s->id[src];
    s->tau_v[dst] = s->tau_v[src];
}

int64_t or3d_densify_event(or3d_model* s, const or_densify_cfg* c, int64_t budget, or_pcg32* rng,
                           int64_t* out_spawned, int64_t* out_pruned, int64_t* out_candidates,
                           int* out_coin) {
    const int64_t cap = s->cap, n0 = s->n;
    const int coin = or_pcg32_uniform(rng) < (double)c->color_branch_prob;
    uint8_t* cand = (uint8_t*)calloc((size_t)(n0 ? n0 : 1), 1);
    float* key = (float*)calloc((size_t)(n0 ? n0 : 1), sizeof(float));
    int64_t nc = 0;
    for (int64_t i = 0; i < n0; ++i) {
        const int32_t cnt = s->visit[i] - s->visit_evt[i];
        if (cnt > 0 && (double)s->visit[i] > s->tau_v[i] &&
            or_activatef(s->params[10 * cap + i]) >= c->opacity_mask_floor) {
            const float cf = (float)cnt;
            const float ap = s->pos_acc[i] / cf, ac = s->col_acc[i] / cf;
            key[i] = ap;
            cand[i] = (ap > c->tau_pos) || (coin && ac > c->tau_color);
            nc += cand[i];
        }
    }
    int64_t remaining = budget - n0;
    if (remaining < 0) remaining = 0;
    if (nc > remaining) {
        int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)nc);
        int64_t w = 0;
        for (int64_t i = 0; i < n0; ++i)
            if (cand[i]) idx[w++] = i;
        g3_key = key;
        qsort(idx, (size_t)nc, sizeof(int64_t), cmp3_desc_key);
        for (int64_t i = remaining; i < nc; ++i) cand[idx[i]] = 0;
        free(idx);
    }
    const double two_pi = 6.28318530717958647692;
    const float ln2 = 0.693147180559945309f;
    int64_t w = n0;
    for (int64_t i = 0; i < n0; ++i) {
        if (!cand[i] || w >= cap) continue;
        const double u1 = or_pcg32_uniform(rng), u2 = or_pcg32_uniform(rng), u3 = or_pcg32_uniform(rng);
        const double rad = cbrt(u1), z = 1.0 - 2.0 * u2;
        const double rxy = sqrt(fmax(0.0, 1.0 - z * z)), ph = two_pi * u3;
        const double e[3] = {rad * rxy * cos(ph), rad * rxy * sin(ph), rad * z};
        const double qw = s->params[3 * cap + i], qx = s->params[4 * cap + i], qy = s->params[5 * cap + i],
                     qz = s->params[6 * cap + i];
        const double qn = sqrt((qw * qw + qx * qx) + (qy * qy + qz * qz));
        const double r = qw / qn, x = qx / qn, y = qy / qn, zq = qz / qn;
        const double Q[3][3] = {{1 - 2 * (y * y + zq * zq), 2 * (x * y - r * zq), 2 * (x * zq + r * y)},
                                {2 * (x * y + r * zq), 1 - 2 * (x * x + zq * zq), 2 * (y * zq - r * x)},
                                {2 * (x * zq - r * y), 2 * (y * zq + r * x), 1 - 2 * (x * x + y * y)}};
        double d[3];
        for (int k = 0; k < 3; ++k) d[k] = exp((double)s->params[(7 + k) * cap + i]) * e[k];
        for (int k = 0; k < 3; ++k) {
            const double o = Q[k][0] * d[0] + Q[k][1] * d[1] + Q[k][2] * d[2];
            s->params[k * cap + w] = (float)((double)s->params[k * cap + i] + o);
        }
        for (int k = 3; k < 7; ++k) s->params[k * cap + w] = s->params[k * cap + i];
        for (int k = 7; k < 10; ++k) s->params[k * cap + w] = s->params[k * cap + i] - ln2;
        s->params[10 * cap + w] = c->child_raw_opacity;
        for (int k = 11; k < OR3D_PARAMS; ++k) s->params[k * cap + w] = s->params[k * cap + i];
        for (int k = 0; k < OR3D_PARAMS; ++k) s->m1[k * cap + w] = s->m2[k * cap + w] = 0.f;
        s->pos_acc[w] = s->col_acc[w] = 0.f;
        s->visit[w] = s->visit_evt[w] = s->visit_aud[w] = 0;
        s->id[w] = s->next_id++;
        s->tau_v[w] = c->tau_v_init;
        ++w;
    }
    free(cand);
    free(key);
    const int64_t spawned = w - n0;
    s->n = w;
    int64_t kept = 0;
    for (int64_t r = 0; r < s->n; ++r) {
        if (or_activatef(s->params[10 * cap + r]) < c->opacity_prune_floor) continue;
        if (kept != r) or3d_copy_row(s, kept, r);
        ++kept;
    }
    const int64_t pruned = s->n - kept;
    s->n = kept;
    for (int64_t i = 0; i < s->n; ++i) {
        s->pos_acc[i] = 0.f;
        s->col_acc[i] = 0.f;
        s->visit_evt[i] = s->visit[i];
    }
    if (out_spawned) *out_spawned = spawned;
    if (out_pruned) *out_pruned = pruned;
    if (out_candidates) *out_candidates = nc;
    if (out_coin) *out_coin = coin;
    return s->n;
}

/* update_visit_thresholds SPEC.md:349-357 on the visits since the last audit. */
void or3d_visit_audit(or3d_model* s) {
    for (int64_t i = 0; i < s->n; ++i) {
        if (s->visit[i] - s->visit_aud[i] < 5) {
            const double t = s->tau_v[i] * 0.5;
            s->tau_v[i] = t < 1.0 ? 1.0 : t;
        }
        s->visit_aud[i] = s->visit[i];
    }
}
