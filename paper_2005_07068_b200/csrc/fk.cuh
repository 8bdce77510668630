// fk.cuh — forward kinematics on one warp (fp64) -> 38 fp32 primitive records,
// conservative screen boxes, the union box and kc(h).
//
// Follows DESIGN §2 (frames, chain, dimensions) for Eq. (1)-(3) and the
// primitive geometry of P:L82; kc per P:L130 with reading AMB-7.  Runs inside k_eval
// (warp 0 of every CTA) so the records never leave shared memory.
#pragma once
#include "common.cuh"

namespace hp {

struct FkScratch {
  double h[kNdof];
  double sn[kNdof], cs[kNdof];
  double RW[3][3];
  double J[5][4][3];        // joint centres, camera frame
  double Rs[5][3][3][3];    // segment frames R_W R_k^H (k = 1..3), camera frame
  int bad;                  // non-finite pose
  int nearf[kNprim];        // primitive lies entirely beyond z_near
};

// Exact records (common.cuh EXACT layout): only the near-plane path reads them.
struct __align__(16) FkExact {
  float rec[kNprim][kRec];
};

struct __align__(16) FkOut {
  float rec[kNprim][kRec];  // FAST layout (common.cuh)
  int4 box[kNprim];  // x0, y0, x1, y1 inclusive; x0 > x1 = empty
  int4 ubox;
  double kc;
  int near_ok;  // every primitive lies entirely beyond z_near (fast min-depth path)
};

__device__ __forceinline__ void mat3_mul(const double a[3][3], const double b[3][3],
                                         double o[3][3]) {
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) o[i][j] = a[i][0] * b[0][j] + a[i][1] * b[1][j] + a[i][2] * b[2][j];
}

// Bounds of the body {c + E q : |q| <= 1}, A = E E^T, on the image: the tangent planes
// through the camera centre containing an image axis satisfy
// (cz^2 - Azz) u^2 - 2 (ca cz - Aaz) u + (ca^2 - Aaa) = 0.  Evaluated in fp32 (the boxes only
// need to be conservative; finish_box adds a rounding margin) with the discriminant expanded so the
// ca^2 cz^2 terms cancel analytically:
//   disc = Aaa cz^2 + Azz ca^2 - 2 Aaz ca cz + Aaz^2 - Aaa Azz.
// Accumulates into [u0,u1]x[v0,v1] (normalised image coordinates); returns 0 behind the
// camera, 2 if the body straddles z = 0.
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_approx_fk(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ int gen_bounds(const float c[3], const float A[3][3], float& u0,
                                          float& u1, float& v0, float& v1, float& zmin) {
  const float zext = sqrt_approx(fmaxf(A[2][2], 0.f));
  zmin = fminf(zmin, c[2] - zext);
  if (c[2] + zext <= 0.f) return 0;
  if (c[2] - zext <= 0.f) return 2;
  // approximate rcp / sqrt: ~1e-7 relative, far inside finish_box's margin
  const float qa = fmaf(c[2], c[2], -A[2][2]), inv = rcp_approx_fk(qa);
#pragma unroll
  for (int ax = 0; ax < 2; ax++) {
    const float ca = c[ax], Aaa = A[ax][ax], Aaz = A[ax][2], Azz = A[2][2];
    const float qb = fmaf(ca, c[2], -Aaz);
    const float disc = Aaa * c[2] * c[2] + Azz * ca * ca - 2.f * Aaz * ca * c[2] + Aaz * Aaz -
                       Aaa * Azz;
    const float sq = sqrt_approx(fmaxf(disc, 0.f));
    const float lo = (qb - sq) * inv, hi = (qb + sq) * inv;
    if (ax == 0) {
      u0 = fminf(u0, lo);
      u1 = fmaxf(u1, hi);
    } else {
      v0 = fminf(v0, lo);
      v1 = fmaxf(v1, hi);
    }
  }
  return 1;
}

// A = R diag(s^2) R^T with R given by its columns.
__device__ __forceinline__ void shape_from_axes(const float col[3][3], const float s[3],
                                                float A[3][3]) {
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++)
      A[i][j] = col[0][i] * col[0][j] * s[0] * s[0] + col[1][i] * col[1][j] * s[1] * s[1] +
                col[2][i] * col[2][j] * s[2] * s[2];
}

// Disc of radius r centred at c with unit normal a: A = r^2 (I - a a^T).
__device__ __forceinline__ void disc_shape(const float a[3], float r, float A[3][3]) {
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) A[i][j] = r * r * ((i == j ? 1.f : 0.f) - a[i] * a[j]);
}

__device__ __forceinline__ int4 finish_box(int st_any, int full, float u0, float u1, float v0,
                                           float v1, const CamParams& cam) {
  int4 b = make_int4(1, 1, 0, 0);  // empty
  if (!st_any) return b;
  if (full) return make_int4(0, 0, cam.W - 1, cam.H - 1);
  // pixel i is a candidate iff its centre i + 0.5 lies within the bounds.  The bounds are
  // the exact silhouette's (tangent planes), so the margin only has to absorb the fp32 /
  // approximate-MUFU rounding of u, v (~1e-6 relative, i.e. ~1e-3 px at f = 575): 2e-5
  // relative plus 0.01 px.  (A whole-pixel margin made 13 % more tile-primitive tests.)
  const float mu = 2e-5f * (fmaxf(fabsf(u0), fabsf(u1)) + 1.f) * cam.fx + 0.01f;
  const float mv = 2e-5f * (fmaxf(fabsf(v0), fabsf(v1)) + 1.f) * cam.fy + 0.01f;
  float x0 = ceilf(fmaf(cam.fx, u0, cam.cx) - 0.5f - mu);
  float x1 = floorf(fmaf(cam.fx, u1, cam.cx) - 0.5f + mu);
  float y0 = ceilf(fmaf(cam.fy, v0, cam.cy) - 0.5f - mv);
  float y1 = floorf(fmaf(cam.fy, v1, cam.cy) - 0.5f + mv);
  x0 = fmaxf(x0, 0.f);
  y0 = fmaxf(y0, 0.f);
  x1 = fminf(x1, (float)(cam.W - 1));
  y1 = fminf(y1, (float)(cam.H - 1));
  if (!(x0 <= x1 && y0 <= y1)) return b;
  return make_int4((int)x0, (int)y0, (int)x1, (int)y1);
}

// Bounds of a primitive from up to two generator bodies.
__device__ __forceinline__ int4 prim_box(int ng, const float c[2][3], const float A[2][3][3],
                                         const CamParams& cam, float& zmin) {
  float u0 = 3e38f, u1 = -3e38f, v0 = 3e38f, v1 = -3e38f;
  int any = 0, full = 0;
  zmin = 3e38f;
  for (int g = 0; g < ng; g++) {
    const int st = gen_bounds(c[g], A[g], u0, u1, v0, v1, zmin);
    if (st) any = 1;
    if (st == 2) full = 1;
  }
  return finish_box(any, full, u0, u1, v0, v1, cam);
}

// Tile-list cull shape of a cone (k_fk_batch): a point p with |p - c| <= r projects within
// R = f r |c| / (c_z (c_z - r)) px of the projection P(c) (f = max(f_x, f_y); the image-plane
// offset is M (p - c) / (c_z (c_z + (p - c)_z)) with M = [[c_z, 0, -c_x], [0, c_z, -c_y]],
// whose largest singular value is |c|).  A cone — the convex hull of its two end discs —
// therefore lies in the 2-D capsule of radius max(R_0, R_1) around the segment
// P(J_0) P(J_1), and a tile whose rectangle projects on the segment's normal farther than R
// from it (separating axis) is skipped.  Stored per cone: (n_x, n_y, n . P(J_0), R); R = inf
// (no refinement) within 1 mm of the camera plane.  Margins: 1e-4 relative + 0.02 px for
// the fp32 / approximate-MUFU rounding of P (~1e-6 relative).
constexpr int kNcone = kCyl - kCone0;
__device__ __forceinline__ float proj_radius(const float c[3], float r, float f) {
  if (!(c[2] - r > 1.f)) return __int_as_float(0x7f800000);
  const float R = f * r * sqrt_approx(fmaf(c[0], c[0], fmaf(c[1], c[1], c[2] * c[2]))) *
                  rcp_approx_fk(c[2] * (c[2] - r));
  return fmaf(R, 1.0001f, 0.02f);
}
__device__ __forceinline__ float4 cone_capsule(const float J0[3], const float J1[3], float r0,
                                               float r1, const CamParams& cam) {
  const float f = fmaxf(cam.fx, cam.fy);
  const float R = fmaxf(proj_radius(J0, r0, f), proj_radius(J1, r1, f));
  const float i0 = rcp_approx_fk(J0[2]), i1 = rcp_approx_fk(J1[2]);
  const float p0x = fmaf(cam.fx, J0[0] * i0, cam.cx), p0y = fmaf(cam.fy, J0[1] * i0, cam.cy);
  const float ex = fmaf(cam.fx, J1[0] * i1, cam.cx) - p0x;
  const float ey = fmaf(cam.fy, J1[1] * i1, cam.cy) - p0y;
  const float L = sqrt_approx(fmaf(ex, ex, ey * ey));
  if (L > 1e-3f) {
    const float iL = rcp_approx_fk(L);
    return make_float4(-ey * iL, ex * iL, (ex * p0y - ey * p0x) * iL, R);
  }
  return make_float4(1.f, 0.f, p0x, R + L);  // degenerate axis: a disc of radius R + L
}

__device__ __forceinline__ void put3(float* r, int off, const double v[3]) {
  r[off + 0] = (float)v[0];
  r[off + 1] = (float)v[1];
  r[off + 2] = (float)v[2];
}

// FAST record of a primitive (common.cuh "FAST record layout"): local origin cen, rows of
// M, Q = diag(q), g = (0, 0, g2), h; fp64 throughout, fp32 coefficients out.  The expansion
// point is the projection of cen, rounded to fp32 first so the coefficients belong to the
// point the kernel subtracts.  axial: cones / cylinder (the axial row of M and the half
// length hl).
__device__ __forceinline__ void write_fast_quadric(float* rec, const double cen[3], const double M[3][3],
                                   double q2, double g2, double h, bool axial,
                                   double ihl) {
  double cl[3];
  for (int a = 0; a < 3; a++) cl[a] = M[a][0] * cen[0] + M[a][1] * cen[1] + M[a][2] * cen[2];
  float xp = 0.f, yp = 0.f;  // any fp32 point will do (the coefficients are computed for it)
  if (cen[2] > 1e-3) {
    const float iz = __frcp_rn((float)cen[2]);
    xp = (float)cen[0] * iz;
    yp = (float)cen[1] * iz;
  }
  const double dp[3] = {(double)xp, (double)yp, 1.0};
  double m0[3], m1[3], dl[3];
  for (int a = 0; a < 3; a++) {
    m0[a] = M[a][0];
    m1[a] = M[a][1];
    dl[a] = M[a][0] * dp[0] + M[a][1] * dp[1] + M[a][2];
  }
  auto QX = [&](const double u[3], const double v[3]) {  // Q = diag(1, 1, q2)
    return u[0] * v[0] + u[1] * v[1] + q2 * u[2] * v[2];
  };
  const double A[6] = {QX(dl, dl), 2.0 * QX(m0, dl), 2.0 * QX(m1, dl),
                       QX(m0, m0), 2.0 * QX(m0, m1), QX(m1, m1)};
  const double b0 = QX(dl, cl) - g2 * dl[2], bx = QX(m0, cl) - g2 * m0[2],
               by = QX(m1, cl) - g2 * m1[2];
  const double c0 = QX(cl, cl) - 2.0 * g2 * cl[2] + h;
  const double D[6] = {b0 * b0 - c0 * A[0],       2.0 * b0 * bx - c0 * A[1],
                       2.0 * b0 * by - c0 * A[2], bx * bx - c0 * A[3],
                       2.0 * bx * by - c0 * A[4], by * by - c0 * A[5]};
  const double ic0 = 1.0 / c0;
  rec[kFxp] = xp;
  rec[kFyp] = yp;
  for (int i = 0; i < 6; i++) rec[kFd + i] = (float)D[i];
  rec[kFb + 0] = (float)(b0 * ic0);
  rec[kFb + 1] = (float)(bx * ic0);
  rec[kFb + 2] = (float)(by * ic0);
  rec[kFic0] = (float)ic0;
  if (axial) {
    const double ih = ihl;  // 1 / the half length (host fp64)
    rec[kFlz + 0] = (float)(M[2][0] * ih);
    rec[kFlz + 1] = (float)(M[2][1] * ih);
    rec[kFlz + 2] = (float)(M[2][2] * ih);
    rec[kFnclz] = (float)(-cl[2] * ih);
  } else {
    for (int i = kFlz; i <= kFnclz; i++) rec[i] = 0.f;
  }
  for (int i = kFnclz + 1; i < kRec; i++) rec[i] = 0.f;  // unused: deterministic records
}

// Build record + box of device primitive j (see common.cuh for the order).
// EXACT-layout record + box of device primitive j (see common.cuh for the order); shape
// (may be null): a cone's tile-list capsule (cone_capsule).  fk_team converts the record
// to the FAST layout afterwards (to_fast).
__device__ void build_prim(int j, const FkScratch& s, const DimsD& dm,
                                        const CamParams& cam, float* rec, int4& box,
                                        float& zmin, float4* shape = nullptr) {
#pragma unroll
  for (int i = 0; i < kRec; i++) rec[i] = 0.f;
  float gc[2][3], gA[2][3][3];
  int ng = 0;
  if (j < kCone0) {  // sphere at joint (f, k)
    int f = j >> 2, k = j & 3;
    double r = dm.rad[f][k];
    const double* c = s.J[f][k];
    put3(rec, kC, c);
    rec[kR2] = (float)(r * r);
    for (int i = 0; i < 3; i++) gc[0][i] = (float)c[i];
    for (int a = 0; a < 3; a++)
      for (int b = 0; b < 3; b++) gA[0][a][b] = (a == b) ? (float)(r * r) : 0.f;
    ng = 1;
  } else if (j < kCyl) {  // truncated cone J_k -> J_{k+1}
    int f, k;
    if (j < 32) {
      f = 1 + (j - kCone0) / 3;
      k = (j - kCone0) % 3;
    } else {
      f = 0;
      k = j - 32 + 1;
    }
    const double* J0 = s.J[f][k];
    const double* J1 = s.J[f][k + 1];
    double L = dm.len[f][k], r0 = dm.rad[f][k], r1 = dm.rad[f][k + 1];
    // segment frame columns: e1 = col0, axis = -col1 (the segment runs along -y_k), e2 = col2
    double e1[3], e2[3], ax[3], m[3];
    for (int i = 0; i < 3; i++) {
      e1[i] = s.Rs[f][k][i][0];
      ax[i] = -s.Rs[f][k][i][1];
      e2[i] = s.Rs[f][k][i][2];
      m[i] = 0.5 * (J0[i] + J1[i]);
    }
    put3(rec, kC, m);
    double rows[3][3] = {{e1[0], e1[1], e1[2]}, {e2[0], e2[1], e2[2]}, {ax[0], ax[1], ax[2]}};
    for (int a = 0; a < 3; a++) {
      put3(rec, kM + 3 * a, rows[a]);
      rec[kCl + a] = (float)(rows[a][0] * m[0] + rows[a][1] * m[1] + rows[a][2] * m[2]);
    }
    rec[kRm] = (float)(0.5 * (r0 + r1));
    rec[kK] = (float)dm.cone_k[f][k];
    rec[kHl] = (float)(0.5 * L);
    float axf[3] = {(float)ax[0], (float)ax[1], (float)ax[2]};
    for (int i = 0; i < 3; i++) {
      gc[0][i] = (float)J0[i];
      gc[1][i] = (float)J1[i];
    }
    if (shape) *shape = cone_capsule(gc[0], gc[1], (float)r0, (float)r1, cam);
    disc_shape(axf, (float)r0, gA[0]);
    disc_shape(axf, (float)r1, gA[1]);
    ng = 2;
  } else if (j == kCyl) {  // palm: elliptic cylinder y_H in [-len, 0]
    double cx[3], cy[3], cz[3], m[3];
    for (int i = 0; i < 3; i++) {
      cx[i] = s.RW[i][0];
      cy[i] = s.RW[i][1];
      cz[i] = s.RW[i][2];
      m[i] = s.h[i] - 0.5 * dm.palm_len * cy[i];
    }
    put3(rec, kC, m);
    double rows[3][3];
    const double iw = dm.inv_sd[1][0], it = dm.inv_sd[1][2];  // 1 / semi-axes (host)
    for (int i = 0; i < 3; i++) {
      rows[0][i] = cx[i] * iw;
      rows[1][i] = cz[i] * it;
      rows[2][i] = cy[i];
    }
    for (int a = 0; a < 3; a++) {
      put3(rec, kM + 3 * a, rows[a]);
      rec[kCl + a] = (float)(rows[a][0] * m[0] + rows[a][1] * m[1] + rows[a][2] * m[2]);
    }
    rec[kRm] = 1.f;
    rec[kK] = 0.f;
    rec[kHl] = (float)(0.5 * dm.palm_len);
    float cols[3][3], sd[3] = {(float)dm.palm_half_w, 0.f, (float)dm.palm_half_t};
    for (int i = 0; i < 3; i++) {
      cols[0][i] = (float)cx[i];
      cols[1][i] = (float)cy[i];
      cols[2][i] = (float)cz[i];
    }
    for (int e = 0; e < 2; e++) {
      double yc = e == 0 ? 0.0 : -dm.palm_len;
      for (int i = 0; i < 3; i++) gc[e][i] = (float)(s.h[i] + yc * cy[i]);
      shape_from_axes(cols, sd, gA[e]);
    }
    ng = 2;
  } else {  // ellipsoids: thumb proximal (35), palm caps (36, 37)
    double c[3], cols[3][3], sd[3];
    if (j == kEll0) {
      for (int i = 0; i < 3; i++) c[i] = 0.5 * (s.J[0][0][i] + s.J[0][1][i]);
      for (int a = 0; a < 3; a++)
        for (int i = 0; i < 3; i++) cols[a][i] = s.Rs[0][0][i][a];
      sd[0] = dm.th_x;
      sd[1] = 0.5 * dm.len[0][0];
      sd[2] = dm.th_z;
    } else {
      double yc = j == kEll0 + 1 ? 0.0 : -dm.palm_len;
      for (int i = 0; i < 3; i++) c[i] = s.h[i] + yc * s.RW[i][1];
      for (int a = 0; a < 3; a++)
        for (int i = 0; i < 3; i++) cols[a][i] = s.RW[i][a];
      sd[0] = dm.palm_half_w;
      sd[1] = dm.cap_half;
      sd[2] = dm.palm_half_t;
    }
    put3(rec, kC, c);
    for (int a = 0; a < 3; a++) {
      const double is = dm.inv_sd[j == kEll0 ? 0 : 1][a];  // 1 / sd[a] (host)
      double row[3] = {cols[a][0] * is, cols[a][1] * is, cols[a][2] * is};
      put3(rec, kM + 3 * a, row);
      rec[kCl + a] = (float)(row[0] * c[0] + row[1] * c[1] + row[2] * c[2]);
    }
    float colf[3][3], sdf[3] = {(float)sd[0], (float)sd[1], (float)sd[2]};
    for (int a = 0; a < 3; a++)
      for (int i = 0; i < 3; i++) colf[a][i] = (float)cols[a][i];
    for (int i = 0; i < 3; i++) gc[0][i] = (float)c[i];
    shape_from_axes(colf, sdf, gA[0]);
    ng = 1;
  }
  box = prim_box(ng, gc, gA, cam, zmin);
}

// FAST record of primitive j straight from the fp64 FK geometry (the same frames build_prim
// uses), independent of the EXACT record and the box, so a team can build both in
// parallel.
// The sphere at joint (f, k) = primitive j < kCone0: |p - c|^2 - r^2 with M = I, Q = I —
// its own call, so the constants fold (the general builder's runtime M = I would cost a full
// quadric expansion); the same values as build_fast's sphere branch.
__device__ __forceinline__ void build_fast_sphere(int j, const FkScratch& s, const DimsD& dm,
                                                  float* rec) {
  const int f = j >> 2, k = j & 3;
  const double r = dm.rad[f][k];
  double c[3], M[3][3];
  for (int i = 0; i < 3; i++) {
    c[i] = s.J[f][k][i];
    for (int a = 0; a < 3; a++) M[a][i] = a == i ? 1.0 : 0.0;
  }
  write_fast_quadric(rec, c, M, 1.0, 0.0, -r * r, false, 0.0);
}

__device__ __forceinline__ void build_fast(int j, const FkScratch& s, const DimsD& dm,
                                           float* rec) {
  // the kinds differ only in the quadric's frame and coefficients: one write_fast_quadric
  // call after the branches, so a warp holding several kinds runs its arithmetic once
  double c[3], M[3][3], q2, g2, h, ihl;  // Q = diag(1, 1, q2)
  bool axial;
  if (j < kCone0) {  // sphere at joint (f, k): |p - c|^2 - r^2, M = I
    const int f = j >> 2, k = j & 3;
    const double r = dm.rad[f][k];
    for (int i = 0; i < 3; i++) {
      c[i] = s.J[f][k][i];
      for (int a = 0; a < 3; a++) M[a][i] = a == i ? 1.0 : 0.0;
    }
    q2 = 1.0;
    g2 = 0.0;
    h = -r * r;
    axial = false;
    ihl = 0.0;
  } else if (j < kCyl) {  // truncated cone J_k -> J_{k+1}: rows e1, e2, axis; midpoint origin
    int f, k;
    if (j < 32) {
      f = 1 + (j - kCone0) / 3;
      k = (j - kCone0) % 3;
    } else {
      f = 0;
      k = j - 32 + 1;
    }
    for (int i = 0; i < 3; i++) {
      M[0][i] = s.Rs[f][k][i][0];
      M[1][i] = s.Rs[f][k][i][2];
      M[2][i] = -s.Rs[f][k][i][1];
      c[i] = 0.5 * (s.J[f][k][i] + s.J[f][k + 1][i]);
    }
    // x^2 + y^2 - (r_m + k z)^2: Q = diag(1, 1, -k^2), g = (0, 0, -r_m k), h = -r_m^2
    const double rm = 0.5 * (dm.rad[f][k] + dm.rad[f][k + 1]), kk = dm.cone_k[f][k];
    q2 = -kk * kk;
    g2 = -rm * kk;
    h = -rm * rm;
    axial = true;
    ihl = dm.inv_hl[f][k];
  } else if (j == kCyl) {  // palm: (x/a)^2 + (z/b)^2 - 1, axial y_H in [-len, 0]
    const double iw = dm.inv_sd[1][0], it = dm.inv_sd[1][2];  // 1 / semi-axes (host)
    for (int i = 0; i < 3; i++) {
      M[0][i] = s.RW[i][0] * iw;
      M[1][i] = s.RW[i][2] * it;
      M[2][i] = s.RW[i][1];
      c[i] = s.h[i] - 0.5 * dm.palm_len * s.RW[i][1];
    }
    q2 = 0.0;
    g2 = 0.0;
    h = -1.0;
    axial = true;
    ihl = dm.inv_hl_palm;
  } else {  // ellipsoids: |l|^2 - 1 with rows = axes / semi-axes (dm.inv_sd)
    if (j == kEll0) {
      for (int i = 0; i < 3; i++) c[i] = 0.5 * (s.J[0][0][i] + s.J[0][1][i]);
      for (int a = 0; a < 3; a++)
        for (int i = 0; i < 3; i++) M[a][i] = s.Rs[0][0][i][a];
    } else {
      const double yc = j == kEll0 + 1 ? 0.0 : -dm.palm_len;
      for (int i = 0; i < 3; i++) c[i] = s.h[i] + yc * s.RW[i][1];
      for (int a = 0; a < 3; a++)
        for (int i = 0; i < 3; i++) M[a][i] = s.RW[i][a];
    }
    for (int a = 0; a < 3; a++) {
      const double is = dm.inv_sd[j == kEll0 ? 0 : 1][a];  // 1 / sd[a] (host)
      for (int i = 0; i < 3; i++) M[a][i] *= is;
    }
    q2 = 1.0;
    g2 = 0.0;
    h = -1.0;
    axial = false;
    ihl = 0.0;
  }
  write_fast_quadric(rec, c, M, q2, g2, h, axial, ihl);
}

#if HP_FK_PROF
__device__ unsigned long long g_fkprof[16];
__shared__ unsigned long long s_fkprof[16];  // staged in shared memory (see fit.cuh)
#define FKPROF(i) \
  if (blockIdx.x == 7 && threadIdx.x == 0) s_fkprof[i] = clock64();
#else
#define FKPROF(i)
#endif
// One warp: the union box of the 38 primitive boxes, the near-plane flag and kc(h) (P:L130,
// AMB-7) of the pose in s / out.
__device__ __forceinline__ void fk_finish_warp(const FkScratch& s, FkOut& out, double kc_rest) {
  const int lane = threadIdx.x & 31;
  // ---- warp 0: union box, near-plane flag, kc ----
  // (the solid is the convex hull of its generators, so zmin bounds its nearest point; the
  // 1e-3 relative slack covers the fp32 evaluation)
  int near_ok = 1;
  int4 u = make_int4(1 << 30, 1 << 30, -1, -1);
  for (int j = lane; j < kNprim; j += 32) {
    near_ok &= s.nearf[j];
    const int4 b = out.box[j];
    if (b.x <= b.z) {
      u.x = min(u.x, b.x);
      u.y = min(u.y, b.y);
      u.z = max(u.z, b.z);
      u.w = max(u.w, b.w);
    }
  }
  FKPROF(5)
  near_ok = __all_sync(0xffffffffu, near_ok);
  u.x = __reduce_min_sync(0xffffffffu, u.x);  // redux.sync: one instruction per bound
  u.y = __reduce_min_sync(0xffffffffu, u.y);
  u.z = __reduce_max_sync(0xffffffffu, u.z);
  u.w = __reduce_max_sync(0xffffffffu, u.w);
  FKPROF(6)
  if (lane == 0) {
    if (s.bad || u.z < u.x) u = make_int4(1, 1, 0, 0);
    out.ubox = u;
    out.near_ok = near_ok && !s.bad;
    // kc(h) = sum over (index,middle), (middle,ring), (ring,little) of -min(phi, 0)
    double kc = 0.0;
    for (int f = 1; f <= 3; f++) {
      double phi = s.h[6 + 4 * f + 1] - s.h[6 + 4 * (f + 1) + 1] + kc_rest;
      kc += -fmin(phi, 0.0);
    }
    out.kc = s.bad ? __longlong_as_double(0x7ff8000000000000ll) : kc;
  }
  __syncwarp();
}

// Phase B of FK for finger f (sincos of the pose already in s.sn / s.cs): R_W, the chain of
// finger f in the camera frame (sparse column updates: B <- B Rz(MPz) touches columns 0, 1,
// B <- B Rx(t) columns 1, 2; the segment runs along -B[:,1]), its joints and segment
// frames.  f = 0 also stores R_W and the non-finite flag.
__device__ __forceinline__ void fk_finger_chain(FkScratch& s, const DimsD& dm, int f, int bad) {
    // R_W = Rz(th_z) Ry(th_y) Rx(th_x)  (AMB-10), written out
    const double cx = s.cs[3], sx = s.sn[3], cy = s.cs[4], sy = s.sn[4], cz = s.cs[5],
                 sz = s.sn[5];
    const double r0[3] = {cy, sy * sx, sy * cx}, r1[3] = {0.0, cx, -sx},
                 r2[3] = {-sy, cy * sx, cy * cx};  // rows of Ry Rx
    double RW[3][3];
    for (int j = 0; j < 3; j++) {
      RW[0][j] = cz * r0[j] - sz * r1[j];
      RW[1][j] = sz * r0[j] + cz * r1[j];
      RW[2][j] = r2[j];
    }
    if (f == 0) {
      for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) s.RW[i][j] = RW[i][j];
      s.bad = bad;
    }
    // B = R_W R_f0 (camera-frame base frame of the finger)
    double B[3][3];
    if (f == 0) mat3_mul(RW, dm.RT0, B);
    else
      for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) B[i][j] = RW[i][j];
    const int o = 6 + 4 * f;  // (MPx, MPz, PIP, DIP), Eq. (1)
    {                         // B <- B Rz(MPz)
      const double c = s.cs[o + 1], sn = s.sn[o + 1];
      for (int i = 0; i < 3; i++) {
        const double b0 = B[i][0], b1 = B[i][1];
        B[i][0] = c * b0 + sn * b1;
        B[i][1] = c * b1 - sn * b0;
      }
    }
    double J[3];
    for (int i = 0; i < 3; i++)
      J[i] = s.h[i] + RW[i][0] * dm.base[f][0] + RW[i][1] * dm.base[f][1] +
             RW[i][2] * dm.base[f][2];
    for (int i = 0; i < 3; i++) s.J[f][0][i] = J[i];
    for (int k = 0; k < 3; k++) {  // B <- B Rx(MPx | PIP | DIP); J += B (0, -L, 0)
      const int ai = k == 0 ? o : o + 1 + k;
      const double c = s.cs[ai], sn = s.sn[ai];
      for (int i = 0; i < 3; i++) {
        const double b1 = B[i][1], b2 = B[i][2];
        B[i][1] = c * b1 + sn * b2;
        B[i][2] = c * b2 - sn * b1;
      }
      const double L = dm.len[f][k];
      for (int i = 0; i < 3; i++) {
        J[i] -= L * B[i][1];
        s.J[f][k + 1][i] = J[i];
      }
      for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) s.Rs[f][k][i][j] = B[i][j];
    }
  }

// FK on a team of 1, 4 or 5 warps (warp 0 = the team leader).  pose: 26 values (float or
// double).  Writes `out`; `s` keeps the fp64 joints for the debug hook.
//   phase A (warp 0): load the pose, sincos of the 23 angles (one per lane, fp64)
//   phase B (warp 0, lanes 0..4): the finger chains directly in the camera frame with
//           sparse column updates: B <- B Rz(MPz) touches columns 0, 1, B <- B Rx(t)
//           columns 1, 2 (the segment runs along -B[:,1])
//   phase C: the 38 FAST records + fp32 screen boxes, one kind of work per warp (TEAM 4 / 5,
//           below), then on warp 0 the union box, the near-plane flag and kc(h)
// xrec (may be null): also keep the EXACT records (the near-plane path's) — TEAM >= 2
// when given, TEAM 1 (the debug hook) only for a pose that is not near_ok.
// shp (may be null): the cones' tile-list capsules [kNcone] (cone_capsule).
// out.rec holds the FAST records on return.
template <typename PoseT, int TEAM>
__device__ void fk_team(const PoseT* pose, const DimsD& dm, const CamParams& cam,
                        double kc_rest, FkScratch& s, FkOut& out, FkExact* xrec = nullptr,
                        float4* shp = nullptr) {
  FKPROF(0)
  static_assert(TEAM == 1 || TEAM == 4 || TEAM == 5,
                "FK teams of 1, 4 or 5 warps (warps 0..TEAM-1 of the CTA)");
  const int lane = threadIdx.x & 31, w = TEAM >= 2 ? (int)(threadIdx.x >> 5) : 0;
  if (w == 0) {
    if (lane < kNdof) {
      const double v = (double)pose[lane];
      s.h[lane] = v;
      if (lane >= 3) sincos(v, &s.sn[lane], &s.cs[lane]);
    }
    __syncwarp();
    FKPROF(1)
    int bad = 0;
    if (lane < kNdof) bad = !isfinite(s.h[lane]);
    bad = __any_sync(0xffffffffu, bad);
    if (lane < 5) fk_finger_chain(s, dm, lane, bad);
    __syncwarp();
    if (TEAM >= 2) asm volatile("bar.arrive 2, %0;" ::"n"(32 * TEAM) : "memory");
  } else if (TEAM >= 2) {
    asm volatile("bar.sync 2, %0;" ::"n"(32 * TEAM) : "memory");
  }
  FKPROF(2)
  // ---- phase C: records + boxes ----
  if (TEAM >= 2) {
    // TEAM 4: warp 0 the 20 spheres' boxes (+ EXACT records into xrec when it is given),
    // warp 1 the 14 cones', warp 2 the cylinder's + 3 ellipsoids', warp 3 the 18 FAST
    // quadric records straight from the frames, and warp 2's idle lanes the 20 spheres'
    // FAST records, all in parallel (no warp builds two records per lane)
    // TEAM 5: the spheres' FAST records on warp 4 instead (warp 2: the boxes only)
    if (w == 3) {
      if (lane < kNprim - kCone0) build_fast(kCone0 + lane, s, dm, out.rec[kCone0 + lane]);
    } else if (w == 4) {
      if (lane < kCone0) build_fast_sphere(lane, s, dm, out.rec[lane]);
    } else if (TEAM == 4 && w == 2 && lane >= kNprim - kCyl) {
      const int j = lane - (kNprim - kCyl);  // lanes 4..23: spheres 0..19
      if (j < kCone0) build_fast_sphere(j, s, dm, out.rec[j]);
    } else {
      const int j0 = w == 0 ? 0 : (w == 1 ? kCone0 : kCyl);
      const int j1 = w == 0 ? kCone0 : (w == 1 ? kCyl : kNprim);
      const int j = j0 + lane;
      if (j < j1) {
        float zmin;
        if (xrec) {
          build_prim(j, s, dm, cam, xrec->rec[j], out.box[j], zmin, nullptr);
        } else {  // no EXACT records wanted: dead stores to a local array (removed)
          float xl[kRec];
          build_prim(j, s, dm, cam, xl, out.box[j], zmin, nullptr);
        }
        s.nearf[j] = zmin > cam.znear * 1.001f;
      }
    }
    if (w != 0) {
      asm volatile("bar.arrive 1, %0;" ::"n"(32 * TEAM) : "memory");
      return;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * TEAM) : "memory");
  } else {
    // 38 records on 32 lanes: lanes 0..9 build two spheres each (the cheapest records),
    // lanes 10..27 one cone / cylinder / ellipsoid each, so no lane builds a sphere AND an
    // expensive record (the critical path of j = lane, lane + 32)
    static_assert(kCone0 == 20 && kNprim == 38, "lane map assumes 20 spheres + 18 others");
    const int nj = lane < 10 ? 2 : (lane < 28 ? 1 : 0);
    for (int k = 0; k < nj; k++) {
      const int j = lane < 10 ? 2 * lane + k : lane + 10;
      float zmin;
      build_prim(j, s, dm, cam, out.rec[j], out.box[j], zmin,
                 shp && j >= kCone0 && j < kCyl ? shp + (j - kCone0) : nullptr);
      s.nearf[j] = zmin > cam.znear * 1.001f;
    }
    __syncwarp();
    if (xrec) {  // a pose that may cross z_near keeps its EXACT records (global memory)
      int nok = 1;
      for (int j = lane; j < kNprim; j += 32) nok &= s.nearf[j];
      if (!__all_sync(0xffffffffu, nok))
        for (int i = lane; i < kNprim * kRec / 4; i += 32)
          reinterpret_cast<float4*>(xrec->rec)[i] =
              reinterpret_cast<const float4*>(out.rec)[i];
    }
    if (lane < kNprim - kCone0) build_fast(kCone0 + lane, s, dm, out.rec[kCone0 + lane]);
    if (lane < kCone0) build_fast_sphere(lane, s, dm, out.rec[lane]);  // (EXACT copied above)
    __syncwarp();
  }
  FKPROF(3)
  fk_finish_warp(s, out, kc_rest);
  FKPROF(4)
#if HP_FK_PROF
  if (blockIdx.x == 7 && threadIdx.x == 0)
    for (int q = 0; q < 16; q++) g_fkprof[q] = s_fkprof[q];
#endif
}

template <typename PoseT>
__device__ __forceinline__ void fk_warp(const PoseT* pose, const DimsD& dm, const CamParams& cam,
                                        double kc_rest, FkScratch& s, FkOut& out,
                                        FkExact* xrec = nullptr) {
  fk_team<PoseT, 1>(pose, dm, cam, kc_rest, s, out, xrec);
}

}  // namespace hp
