/*
 * oracle.c — plain fp64 CPU oracle for arXiv 2005.07068 (see oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY: never linked into or called by the product path.
 * Compile: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared -pthread oracle.c -lm
 * (-ffp-contract=off: the PSO arithmetic must round after every operation).
 *
 * Every function cites the passage it follows: P:Lnn = /root/reference/PAPER.md line nn;
 * DESIGN §n = /root/repo/DESIGN.md section n (the readings of silent/garbled points).
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ------------------------------------------------------------------------------------ */
/* Defaults                                                                             */
/* ------------------------------------------------------------------------------------ */

/* DESIGN §2 "Dimensions" table (P:L82 gives no numbers; AMB-9). */
void or_default_dims(or_dims* d) {
  static const double base[5][3] = {
      {30, -10, -8}, {27, -88, 0}, {9, -92, 0}, {-9, -89, 0}, {-26, -83, 0}};
  static const double len[5][3] = {
      {45, 32, 27}, {45, 27, 22}, {48, 30, 24}, {45, 28, 23}, {36, 21, 20}};
  static const double rad[5][4] = {{11, 10, 8.5, 7.5},
                                   {9, 8, 7, 6},
                                   {9.5, 8.5, 7.5, 6.5},
                                   {9, 8, 7, 6},
                                   {8, 7, 6.5, 5.5}};
  d->palm_half_w = 45;
  d->palm_half_t = 15;
  d->palm_len = 80;
  d->palm_cap_half_len = 10;
  memcpy(d->base, base, sizeof base);
  memcpy(d->seg_len, len, sizeof len);
  memcpy(d->radius, rad, sizeof rad);
  d->thumb_ell_x = 12;
  d->thumb_ell_z = 10;
  d->thumb_yaw_deg = 40;
  d->thumb_pitch_deg = 90;
}

/* d_m = 1 cm, d_M = 4 cm, lambda = 20, lambda_k = 10; depth_scale and rho are
 * readings AMB-2 and AMB-7. */
void or_default_cost(or_cost_params* p) {
  p->d_m = 10.0;
  p->d_M = 40.0;
  p->lambda = 20.0;
  p->lambda_k = 10.0;
  p->depth_scale = 0.1;
  p->kc_rest = 0.0;
  p->clamp_at_dm = 0;
}

/* P:L148-150 (64 particles, 30 generations, c1 2.8, c2 1.3), P:L152 (every 3, half). */
void or_default_pso(or_pso_params* p) {
  p->seed = 0;
  p->particles = 64;
  p->generations = 30;
  p->mutation_period = 3;
  p->per_dim_r = 0;
  p->c1 = 2.8;
  p->c2 = 1.3;
  p->mutation_fraction = 0.5;
  p->stop_threshold = -INFINITY;
  p->mutation_after_eval = 0;
}

/* AMB-12: fx = fy = 525, (cx, cy) = (320, 240) at 640x480, scaled with the width. */
void or_camera_for(int32_t width, int32_t height, or_camera* cam) {
  double scale = (double)width / 640.0;
  cam->width = width;
  cam->height = height;
  cam->fx = 525.0 * scale;
  cam->fy = 525.0 * scale;
  cam->cx = 0.5 * (double)width;
  cam->cy = 0.5 * (double)height;
  cam->z_near = 300.0;
  cam->z_far = 2000.0;
}

static double deg2rad(double deg) { return deg * (M_PI / 180.0); }

/* Tables 1-2 in flattening order: x,y,z mm; angles rad. */
void or_bounds(double lo[26], double hi[26]) {
  static const double wlo[6] = {-900, -680, 500, -30, -70, -35};
  static const double whi[6] = {900, 680, 1500, 120, 75, 20};
  static const double flo[5][4] = {
      {0, -15, 0, -15}, {0, -15, 0, 0}, {0, -10, 0, 0}, {0, -30, 0, 0}, {0, -45, 0, 0}};
  static const double fhi[5][4] = {
      {90, 60, 50, 70}, {90, 15, 100, 60}, {90, 10, 100, 60}, {90, 0, 100, 60}, {90, 0, 100, 60}};
  for (int i = 0; i < 3; i++) {
    lo[i] = wlo[i];
    hi[i] = whi[i];
  }
  for (int i = 3; i < 6; i++) {
    lo[i] = deg2rad(wlo[i]);
    hi[i] = deg2rad(whi[i]);
  }
  for (int f = 0; f < 5; f++)
    for (int j = 0; j < 4; j++) {
      lo[6 + 4 * f + j] = deg2rad(flo[f][j]);
      hi[6 + 4 * f + j] = deg2rad(fhi[f][j]);
    }
}

/* ------------------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al. 2011; DESIGN §4 RNG layout)                              */
/* ------------------------------------------------------------------------------------ */

void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; round++) {
    if (round > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* 53-bit uniform in [0, 1) from two words. */
double or_u01(uint32_t w0, uint32_t w1) {
  return ((double)(w0 >> 5) * 67108864.0 + (double)(w1 >> 6)) * (1.0 / 9007199254740992.0);
}

/* ------------------------------------------------------------------------------------ */
/* Small linear algebra                                                                  */
/* ------------------------------------------------------------------------------------ */

typedef double mat3[3][3];

static void rot_x(double a, mat3 m) {
  double c = cos(a), s = sin(a);
  mat3 r = {{1, 0, 0}, {0, c, -s}, {0, s, c}};
  memcpy(m, r, sizeof r);
}
static void rot_y(double a, mat3 m) {
  double c = cos(a), s = sin(a);
  mat3 r = {{c, 0, s}, {0, 1, 0}, {-s, 0, c}};
  memcpy(m, r, sizeof r);
}
static void rot_z(double a, mat3 m) {
  double c = cos(a), s = sin(a);
  mat3 r = {{c, -s, 0}, {s, c, 0}, {0, 0, 1}};
  memcpy(m, r, sizeof r);
}
static void matmul(const mat3 a, const mat3 b, mat3 out) {
  mat3 t;
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) t[i][j] = a[i][0] * b[0][j] + a[i][1] * b[1][j] + a[i][2] * b[2][j];
  memcpy(out, t, sizeof t);
}
static void matvec(const mat3 a, const double v[3], double out[3]) {
  double t[3];
  for (int i = 0; i < 3; i++) t[i] = a[i][0] * v[0] + a[i][1] * v[1] + a[i][2] * v[2];
  out[0] = t[0];
  out[1] = t[1];
  out[2] = t[2];
}
static double dot3(const double a[3], const double b[3]) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

/* ------------------------------------------------------------------------------------ */
/* Forward kinematics (Eq. 1-3; P:L82 geometry; DESIGN §2 frames)                */
/* ------------------------------------------------------------------------------------ */

/* p_cam = t + R_W p_H with R_W = Rz(th_z) Ry(th_y) Rx(th_x)  (AMB-10).
 * Finger f: R1 = R_f0 Rz(MPz) Rx(MPx), R2 = R1 Rx(PIP), R3 = R2 Rx(DIP);
 * J_{k+1} = J_k + R_{k+1} (0, -L_{k+1}, 0); R_f0 = I, thumb R_T0 = Rz(40deg) Ry(90deg). */
void or_fk(const double h[26], const or_dims* d, or_prim prims[38], double joints[5][4][3]) {
  mat3 Rx, Ry, Rz, RW, tmp;
  rot_x(h[3], Rx);
  rot_y(h[4], Ry);
  rot_z(h[5], Rz);
  matmul(Ry, Rx, tmp);
  matmul(Rz, tmp, RW);
  const double t[3] = {h[0], h[1], h[2]};
  int np = 0;

  /* Palm: elliptic cylinder y_H in [-len, 0] capped by two ellipsoids. */
  {
    or_prim* p = &prims[np++];
    p->kind = OR_CYLINDER;
    memcpy(p->c, t, sizeof t);
    memcpy(p->R, RW, sizeof(mat3));
    p->s[0] = d->palm_half_w;
    p->s[1] = d->palm_len;
    p->s[2] = d->palm_half_t;
    for (int e = 0; e < 2; e++) {
      double yH[3] = {0, e == 0 ? 0.0 : -d->palm_len, 0}, off[3];
      or_prim* q = &prims[np++];
      q->kind = OR_ELLIPSOID;
      matvec(RW, yH, off);
      for (int i = 0; i < 3; i++) q->c[i] = t[i] + off[i];
      memcpy(q->R, RW, sizeof(mat3));
      q->s[0] = d->palm_half_w;
      q->s[1] = d->palm_cap_half_len;
      q->s[2] = d->palm_half_t;
    }
  }

  for (int f = 0; f < 5; f++) {
    const double* a = &h[6 + 4 * f]; /* (MPx, MPz, PIP, DIP), Eq. (1) */
    mat3 R0, Rk[3], A, B;
    if (f == 0) {
      rot_z(deg2rad(d->thumb_yaw_deg), A);
      rot_y(deg2rad(d->thumb_pitch_deg), B);
      matmul(A, B, R0);
    } else {
      mat3 I = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
      memcpy(R0, I, sizeof I);
    }
    rot_z(a[1], A);
    rot_x(a[0], B);
    matmul(R0, A, tmp);
    matmul(tmp, B, Rk[0]);
    rot_x(a[2], A);
    matmul(Rk[0], A, Rk[1]);
    rot_x(a[3], A);
    matmul(Rk[1], A, Rk[2]);

    double JH[4][3];
    memcpy(JH[0], d->base[f], sizeof(double) * 3);
    for (int k = 0; k < 3; k++) {
      double seg[3] = {0, -d->seg_len[f][k], 0}, off[3];
      matvec(Rk[k], seg, off);
      for (int i = 0; i < 3; i++) JH[k + 1][i] = JH[k][i] + off[i];
    }
    double J[4][3];
    for (int k = 0; k < 4; k++) {
      double off[3];
      matvec(RW, JH[k], off);
      for (int i = 0; i < 3; i++) J[k][i] = t[i] + off[i];
      if (joints) memcpy(joints[f][k], J[k], sizeof(double) * 3);
    }
    for (int k = 0; k < 4; k++) {
      or_prim* s = &prims[np++];
      memset(s, 0, sizeof *s);
      s->kind = OR_SPHERE;
      memcpy(s->c, J[k], sizeof(double) * 3);
      s->s[0] = d->radius[f][k];
      if (k == 3) break;
      or_prim* g = &prims[np++];
      memset(g, 0, sizeof *g);
      if (f == 0 && k == 0) {
        /* Thumb: "the largest segment is an ellipsoid instead of a cone". */
        g->kind = OR_ELLIPSOID;
        for (int i = 0; i < 3; i++) g->c[i] = 0.5 * (J[0][i] + J[1][i]);
        matmul(RW, Rk[0], g->R);
        g->s[0] = d->thumb_ell_x;
        g->s[1] = 0.5 * d->seg_len[0][0];
        g->s[2] = d->thumb_ell_z;
      } else {
        /* Truncated cone J_k -> J_{k+1}, end radii = the joint sphere radii. */
        g->kind = OR_CONE;
        memcpy(g->c, J[k], sizeof(double) * 3);
        double L = d->seg_len[f][k];
        double ax[3];
        for (int i = 0; i < 3; i++) ax[i] = (J[k + 1][i] - J[k][i]) / L;
        for (int i = 0; i < 3; i++) g->R[i][1] = ax[i];
        g->s[0] = d->radius[f][k];
        g->s[1] = d->radius[f][k + 1];
        g->s[2] = L;
      }
    }
  }
}

/* kc(h) = sum_{p in Q} -min(phi(p,h), 0), Q = the 3 adjacent non-thumb pairs;
 * phi = MPz(radial finger) - MPz(ulnar finger) + rho (AMB-7, rad AMB-8). */
double or_kc(const double h[26], double rho) {
  double kc = 0.0;
  for (int f = 1; f <= 3; f++) {
    double phi = h[6 + 4 * f + 1] - h[6 + 4 * (f + 1) + 1] + rho;
    kc += -fmin(phi, 0.0);
  }
  return kc;
}

/* ------------------------------------------------------------------------------------ */
/* Ray casting (P:L114 r_d(h, C); S:L166 nearest analytic intersection)                   */
/* ------------------------------------------------------------------------------------ */

void or_ray(const or_camera* cam, double u, double v, double dir[3]) {
  dir[0] = (u - cam->cx) / cam->fx;
  dir[1] = (v - cam->cy) / cam->fy;
  dir[2] = 1.0;
}

/* Real roots of A t^2 + 2 B t + C = 0 (A may be 0); returns the count, sorted. */
static int quad_roots(double A, double B, double C, double r[2]) {
  if (A == 0.0) {
    if (B == 0.0) return 0;
    r[0] = -C / (2.0 * B);
    return 1;
  }
  double disc = B * B - A * C;
  if (disc < 0.0) return 0;
  double sq = sqrt(disc);
  double t1 = (-B - sq) / A, t2 = (-B + sq) / A;
  r[0] = fmin(t1, t2);
  r[1] = fmax(t1, t2);
  return 2;
}

static void consider(double t, double* best) {
  if (t > 0.0 && t < *best) *best = t;
}

/* Smallest t > 0 at which the ray t*dir meets the closed surface of the solid. */
double or_first_hit(const or_prim* p, const double d[3]) {
  double best = INFINITY, r[2];
  int n;
  switch (p->kind) {
    case OR_SPHERE: { /* |t d - c|^2 = r^2 */
      double A = dot3(d, d), B = -dot3(d, p->c), C = dot3(p->c, p->c) - p->s[0] * p->s[0];
      n = quad_roots(A, B, C, r);
      for (int i = 0; i < n; i++) consider(r[i], &best);
      break;
    }
    case OR_ELLIPSOID: { /* q = S^-1 R^T (t d - c), |q|^2 = 1 */
      double q0[3], qd[3];
      for (int j = 0; j < 3; j++) {
        double col[3] = {p->R[0][j], p->R[1][j], p->R[2][j]};
        qd[j] = dot3(col, d) / p->s[j];
        q0[j] = -dot3(col, p->c) / p->s[j];
      }
      n = quad_roots(dot3(qd, qd), dot3(q0, qd), dot3(q0, q0) - 1.0, r);
      for (int i = 0; i < n; i++) consider(r[i], &best);
      break;
    }
    case OR_CONE: { /* lateral surface in z in [0, L] plus the two end discs */
      double a[3] = {p->R[0][1], p->R[1][1], p->R[2][1]};
      double r0 = p->s[0], r1 = p->s[1], L = p->s[2], k = (r1 - r0) / L;
      double dd = dot3(d, d), de = dot3(d, p->c), ee = dot3(p->c, p->c);
      double da = dot3(d, a), ea = dot3(p->c, a);
      double m = r0 - k * ea, nn = k * da;
      double A = dd - da * da - nn * nn;
      double B = -de + da * ea - m * nn;
      double C = ee - ea * ea - m * m;
      n = quad_roots(A, B, C, r);
      for (int i = 0; i < n; i++) {
        double z = r[i] * da - ea;
        if (z >= 0.0 && z <= L) consider(r[i], &best);
      }
      if (da != 0.0) {
        for (int e = 0; e < 2; e++) {
          double zc = e == 0 ? 0.0 : L, rc = e == 0 ? r0 : r1;
          double t = (ea + zc) / da;
          double w[3] = {t * d[0] - p->c[0], t * d[1] - p->c[1], t * d[2] - p->c[2]};
          double rad2 = dot3(w, w) - zc * zc;
          if (rad2 <= rc * rc) consider(t, &best);
        }
      }
      break;
    }
    case OR_CYLINDER: { /* local (x,y,z) = R^T (t d - c): x^2/a^2 + z^2/b^2 = 1, y in [-len,0] */
      double g[3], hh[3];
      for (int j = 0; j < 3; j++) {
        double col[3] = {p->R[0][j], p->R[1][j], p->R[2][j]};
        g[j] = dot3(col, d);
        hh[j] = dot3(col, p->c);
      }
      double a = p->s[0], len = p->s[1], b = p->s[2];
      double A = (g[0] / a) * (g[0] / a) + (g[2] / b) * (g[2] / b);
      double B = -((g[0] / a) * (hh[0] / a) + (g[2] / b) * (hh[2] / b));
      double C = (hh[0] / a) * (hh[0] / a) + (hh[2] / b) * (hh[2] / b) - 1.0;
      n = quad_roots(A, B, C, r);
      for (int i = 0; i < n; i++) {
        double y = r[i] * g[1] - hh[1];
        if (y >= -len && y <= 0.0) consider(r[i], &best);
      }
      if (g[1] != 0.0) {
        for (int e = 0; e < 2; e++) {
          double yc = e == 0 ? 0.0 : -len;
          double t = (hh[1] + yc) / g[1];
          double x = t * g[0] - hh[0], z = t * g[2] - hh[2];
          if ((x / a) * (x / a) + (z / b) * (z / b) <= 1.0) consider(t, &best);
        }
      }
      break;
    }
  }
  return best;
}

/* Exact screen-space bounds of an ellipsoid-like body {c + E q : |q| <= 1} with
 * A = E E^T, from the tangent planes through the camera centre containing the image
 * axis: (cz^2 - Azz) u^2 - 2 (cx cz - Axz) u + (cx^2 - Axx) = 0.
 * Returns 0 = fully behind, 1 = bounds valid, 2 = straddles the camera plane. */
static int ellipsoid_bounds(const double c[3], const mat3 A, double ub[2], double vb[2]) {
  double zext = sqrt(fmax(A[2][2], 0.0));
  if (c[2] + zext <= 0.0) return 0;
  if (c[2] - zext <= 0.0) return 2;
  for (int ax = 0; ax < 2; ax++) {
    double qa = c[2] * c[2] - A[2][2];
    double qb = c[ax] * c[2] - A[ax][2];
    double qc = c[ax] * c[ax] - A[ax][ax];
    double disc = fmax(qb * qb - qa * qc, 0.0);
    double lo = (qb - sqrt(disc)) / qa, hi = (qb + sqrt(disc)) / qa;
    double* out = ax == 0 ? ub : vb;
    out[0] = lo;
    out[1] = hi;
  }
  return 1;
}

/* A = R diag(s^2) R^T */
static void shape_matrix(const mat3 R, const double s[3], mat3 A) {
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) {
      double acc = 0;
      for (int k = 0; k < 3; k++) acc += R[i][k] * s[k] * s[k] * R[j][k];
      A[i][j] = acc;
    }
}

/* Bounds of the primitive as a list of ellipsoid-like generators: the solid is the
 * convex hull of the generators, and x/z, y/z are quasi-linear, so the union of the
 * generators' bounds is the exact bound of the solid. */
static int prim_generators(const or_prim* p, double cs[2][3], mat3 As[2]) {
  switch (p->kind) {
    case OR_SPHERE: {
      double s[3] = {p->s[0], p->s[0], p->s[0]};
      mat3 I = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
      memcpy(cs[0], p->c, sizeof(double) * 3);
      shape_matrix(I, s, As[0]);
      return 1;
    }
    case OR_ELLIPSOID:
      memcpy(cs[0], p->c, sizeof(double) * 3);
      shape_matrix(p->R, p->s, As[0]);
      return 1;
    case OR_CONE: { /* the two end discs: A = r^2 (I - a a^T) */
      double a[3] = {p->R[0][1], p->R[1][1], p->R[2][1]};
      for (int e = 0; e < 2; e++) {
        double rr = e == 0 ? p->s[0] : p->s[1], zc = e == 0 ? 0.0 : p->s[2];
        for (int i = 0; i < 3; i++) cs[e][i] = p->c[i] + zc * a[i];
        for (int i = 0; i < 3; i++)
          for (int j = 0; j < 3; j++) As[e][i][j] = rr * rr * ((i == j ? 1.0 : 0.0) - a[i] * a[j]);
      }
      return 2;
    }
    case OR_CYLINDER: { /* the two end discs, semi-axes (a, 0, b) in the local frame */
      double s[3] = {p->s[0], 0.0, p->s[2]};
      for (int e = 0; e < 2; e++) {
        double yc = e == 0 ? 0.0 : -p->s[1];
        for (int i = 0; i < 3; i++) cs[e][i] = p->c[i] + yc * p->R[i][1];
        shape_matrix(p->R, s, As[e]);
      }
      return 2;
    }
  }
  return 0;
}

/* Conservative inclusive pixel box of the primitive: pixel i may be hit only if its
 * centre i + 0.5 lies inside the projected bounds; `margin` extra pixels absorb rounding. */
int32_t or_prim_box(const or_prim* p, const or_camera* cam, int32_t margin, int32_t box[4]) {
  double cs[2][3];
  mat3 As[2];
  int ng = prim_generators(p, cs, As);
  double u0 = INFINITY, u1 = -INFINITY, v0 = INFINITY, v1 = -INFINITY;
  int full = 0, any = 0;
  for (int g = 0; g < ng; g++) {
    double ub[2], vb[2];
    int st = ellipsoid_bounds(cs[g], As[g], ub, vb);
    if (st == 0) continue;
    any = 1;
    if (st == 2) {
      full = 1;
      continue;
    }
    u0 = fmin(u0, ub[0]);
    u1 = fmax(u1, ub[1]);
    v0 = fmin(v0, vb[0]);
    v1 = fmax(v1, vb[1]);
  }
  if (!any) return 0;
  double x0, x1, y0, y1;
  if (full) {
    x0 = 0;
    y0 = 0;
    x1 = cam->width - 1;
    y1 = cam->height - 1;
  } else {
    x0 = ceil(cam->fx * u0 + cam->cx - 0.5) - margin;
    x1 = floor(cam->fx * u1 + cam->cx - 0.5) + margin;
    y0 = ceil(cam->fy * v0 + cam->cy - 0.5) - margin;
    y1 = floor(cam->fy * v1 + cam->cy - 0.5) + margin;
    x0 = fmax(x0, 0);
    y0 = fmax(y0, 0);
    x1 = fmin(x1, cam->width - 1);
    y1 = fmin(y1, cam->height - 1);
  }
  if (x0 > x1 || y0 > y1) return 0;
  box[0] = (int32_t)x0;
  box[1] = (int32_t)y0;
  box[2] = (int32_t)x1;
  box[3] = (int32_t)y1;
  return 1;
}

/* r_d(pixel) = min over primitives of the first hit within [z_near, z_far] (AMB-27),
 * stored as the nearest fp32 value (the paper's depth images are fp32); 0 = none. */
static float pixel_depth(const or_prim* prims, int nprim, const uint8_t* use, const or_camera* cam,
                         double u, double v) {
  double dir[3], best = INFINITY;
  or_ray(cam, u, v, dir);
  for (int j = 0; j < nprim; j++) {
    if (use && !use[j]) continue;
    double t = or_first_hit(&prims[j], dir);
    if (t >= cam->z_near && t <= cam->z_far && t < best) best = t;
  }
  return isinf(best) ? 0.0f : (float)best;
}

void or_render_prims(const or_prim* prims, int32_t nprim, const or_camera* cam, int32_t culled,
                     float* depth) {
  int32_t W = cam->width, H = cam->height;
  int32_t(*boxes)[4] = malloc(sizeof(int32_t[4]) * (nprim > 0 ? nprim : 1));
  uint8_t* valid = malloc(nprim > 0 ? nprim : 1);
  uint8_t* use = malloc(nprim > 0 ? nprim : 1);
  for (int j = 0; j < nprim; j++) valid[j] = culled ? or_prim_box(&prims[j], cam, 1, boxes[j]) : 1;
  for (int32_t v = 0; v < H; v++)
    for (int32_t u = 0; u < W; u++) {
      for (int j = 0; j < nprim; j++)
        use[j] = !culled || (valid[j] && u >= boxes[j][0] && u <= boxes[j][2] && v >= boxes[j][1] &&
                             v <= boxes[j][3]);
      depth[(int64_t)v * W + u] = pixel_depth(prims, nprim, use, cam, u + 0.5, v + 0.5);
    }
  free(boxes);
  free(valid);
  free(use);
}

void or_render(const double h[26], const or_dims* d, const or_camera* cam, int32_t culled,
               float* depth) {
  or_prim prims[OR_NPRIM];
  or_fk(h, d, prims, NULL);
  or_render_prims(prims, OR_NPRIM, cam, culled, depth);
}

/* Edge pixels (DESIGN §6 tolerances): the hit status or the depth changes when the pixel's
 * ray moves by +-delta px along x or y, or the r_m decision |o_d - r_d| < d_m is
 * within rm_tol of its threshold.  Only these pixels may be decided differently by an fp32
 * renderer. */
void or_edge_mask_prims(const or_prim* prims, int32_t nprim, const or_camera* cam, double delta,
                        double depth_tol, const float* obs_depth, double d_m, double rm_tol,
                        uint8_t* edge) {
  int32_t W = cam->width, H = cam->height;
  static const double off[4][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}};
  for (int32_t v = 0; v < H; v++)
    for (int32_t u = 0; u < W; u++) {
      float z = pixel_depth(prims, nprim, NULL, cam, u + 0.5, v + 0.5);
      uint8_t e = 0;
      for (int k = 0; k < 4 && !e; k++) {
        float zk = pixel_depth(prims, nprim, NULL, cam, u + 0.5 + delta * off[k][0],
                               v + 0.5 + delta * off[k][1]);
        if ((zk > 0) != (z > 0)) e = 1;
        else if (z > 0 && fabs((double)zk - (double)z) > depth_tol) e = 1;
      }
      if (!e && obs_depth && z > 0) {
        double od = obs_depth[(int64_t)v * W + u];
        if (od > 0 && fabs(fabs(od - (double)z) - d_m) < rm_tol) e = 1;
      }
      edge[(int64_t)v * W + u] = e;
    }
}

void or_edge_mask(const double h[26], const or_dims* d, const or_camera* cam, double delta,
                  double depth_tol, const float* obs_depth, double d_m, double rm_tol,
                  uint8_t* edge) {
  or_prim prims[OR_NPRIM];
  or_fk(h, d, prims, NULL);
  or_edge_mask_prims(prims, OR_NPRIM, cam, delta, depth_tol, obs_depth, d_m, rm_tol, edge);
}

/* ------------------------------------------------------------------------------------ */
/* Eq. (4)-(5)                                                              */
/* ------------------------------------------------------------------------------------ */

/* r_m = [r_d > 0] and ([o_d undefined] or [|o_d - r_d| < d_m])     (AMB-4, AMB-5)
 * numerator over pixels with both depths defined, clamped at d_M   (AMB-1, AMB-3)      */
void or_score(const float* obs_depth, const uint8_t* obs_mask, const float* r_d, int64_t npx,
              const or_cost_params* cp, or_sums* out) {
  double clampv = cp->clamp_at_dm ? cp->d_m : cp->d_M;
  memset(out, 0, sizeof *out);
  for (int64_t i = 0; i < npx; i++) {
    double od = obs_depth[i], rd = r_d[i];
    int os = obs_mask[i] != 0;
    int rd_def = rd > 0.0, od_def = od > 0.0;
    int rm = rd_def && (!od_def || fabs(od - rd) < cp->d_m);
    out->s_o += os;
    out->s_rm += rm;
    out->s_or += (os || rm);
    out->s_and += (os && rm);
    if (rd_def && od_def) {
      out->n_both += 1;
      out->num += fmin(fabs(od - rd), clampv);
    }
  }
}

/* D = depth_scale * num / S_or + lambda (1 - 2 S_and / (S_and + S_or)); D = 0 if S_or = 0
 * (AMB-6); E = D + lambda_k kc (Eq. 5). */
double or_cost_from_sums(const or_sums* s, const or_cost_params* cp, double kc, double* D_out) {
  double D = 0.0;
  if (s->s_or > 0) {
    double sor = (double)s->s_or, sand = (double)s->s_and;
    D = cp->depth_scale * s->num / sor + cp->lambda * (1.0 - 2.0 * sand / (sand + sor));
  }
  if (D_out) *D_out = D;
  return D + cp->lambda_k * kc;
}

typedef struct {
  const double* poses;
  int32_t n, stride, start;
  const float* od;
  const uint8_t* os;
  const or_camera* cam;
  const or_dims* d;
  const or_cost_params* cp;
  int32_t culled;
  double* costs;
  or_sums* sums;
  double *kc, *D;
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* j = arg;
  int64_t npx = (int64_t)j->cam->width * j->cam->height;
  float* rd = malloc(sizeof(float) * (size_t)npx);
  for (int32_t i = j->start; i < j->n; i += j->stride) {
    const double* h = &j->poses[(int64_t)i * OR_NDOF];
    or_render(h, j->d, j->cam, j->culled, rd);
    or_sums s;
    or_score(j->od, j->os, rd, npx, j->cp, &s);
    double kc = or_kc(h, j->cp->kc_rest), D;
    j->costs[i] = or_cost_from_sums(&s, j->cp, kc, &D);
    if (j->sums) j->sums[i] = s;
    if (j->kc) j->kc[i] = kc;
    if (j->D) j->D[i] = D;
  }
  free(rd);
  return NULL;
}

static int32_t resolve_threads(int32_t threads) {
  if (threads > 0) return threads;
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int32_t)n : 1;
}

void or_eval_batch(const double* poses, int32_t n, const float* obs_depth, const uint8_t* obs_mask,
                   const or_camera* cam, const or_dims* d, const or_cost_params* cp, int32_t culled,
                   int32_t threads, double* costs, or_sums* sums, double* kc, double* D) {
  int32_t T = resolve_threads(threads);
  if (T > n) T = n > 0 ? n : 1;
  pthread_t* tid = malloc(sizeof(pthread_t) * T);
  batch_job* jobs = malloc(sizeof(batch_job) * T);
  for (int32_t t = 0; t < T; t++) {
    batch_job j = {poses, n, T, t, obs_depth, obs_mask, cam, d, cp, culled, costs, sums, kc, D};
    jobs[t] = j;
    if (T == 1) batch_worker(&jobs[t]);
    else pthread_create(&tid[t], NULL, batch_worker, &jobs[t]);
  }
  if (T > 1)
    for (int32_t t = 0; t < T; t++) pthread_join(tid[t], NULL);
  free(tid);
  free(jobs);
}

/* ------------------------------------------------------------------------------------ */
/* Algorithmic work: sum_prims |box_prim| F_kind + |box_union| F_px.           */
/* The per-kind constants are the FLOP counts of the frozen formulas in DESIGN §5.       */
/* ------------------------------------------------------------------------------------ */

#define F_SPHERE 20.0
#define F_ELLIPSOID 48.0
#define F_CONE 56.0
#define F_PX 15.0

double or_walg(const double h[26], const or_dims* d, const or_camera* cam, int64_t* tests_out,
               int64_t* union_px_out) {
  or_prim prims[OR_NPRIM];
  or_fk(h, d, prims, NULL);
  double w = 0.0;
  int64_t tests = 0;
  int32_t ub[4] = {cam->width, cam->height, -1, -1};
  for (int j = 0; j < OR_NPRIM; j++) {
    int32_t b[4];
    if (!or_prim_box(&prims[j], cam, 0, b)) continue;
    int64_t area = (int64_t)(b[2] - b[0] + 1) * (b[3] - b[1] + 1);
    double F = prims[j].kind == OR_SPHERE ? F_SPHERE
               : prims[j].kind == OR_ELLIPSOID ? F_ELLIPSOID
                                               : F_CONE; /* cone and cylinder share a formula */
    w += (double)area * F;
    tests += area;
    if (b[0] < ub[0]) ub[0] = b[0];
    if (b[1] < ub[1]) ub[1] = b[1];
    if (b[2] > ub[2]) ub[2] = b[2];
    if (b[3] > ub[3]) ub[3] = b[3];
  }
  int64_t upx = ub[2] >= ub[0] ? (int64_t)(ub[2] - ub[0] + 1) * (ub[3] - ub[1] + 1) : 0;
  w += (double)upx * F_PX;
  if (tests_out) *tests_out = tests;
  if (union_px_out) *union_px_out = upx;
  return w;
}

/* ------------------------------------------------------------------------------------ */
/* PSO (Eq. 6-7; readings AMB-15..22)                               */
/* ------------------------------------------------------------------------------------ */

/* w = 2 / |2 - psi - sqrt(psi^2 - 4 psi)|, psi = c1 + c2. */
double or_constriction(double c1, double c2) {
  double psi = c1 + c2;
  if (!(psi > 4.0)) return NAN;
  return 2.0 / fabs(2.0 - psi - sqrt(psi * psi - 4.0 * psi));
}

static void draw4(uint64_t seed, uint32_t i, uint32_t d, uint32_t k, uint32_t tag, uint32_t out[4]) {
  uint32_t ctr[4] = {i, d, k, tag};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  or_philox4x32_10(ctr, key, out);
}

static double sanitize(double e) { return isnan(e) ? INFINITY : e; }

int32_t or_pso_run(int32_t D, const double* lo, const double* hi, const double* init_lo,
                   const double* init_hi, int32_t mut_lo, int32_t mut_hi, const or_pso_params* pp,
                   or_batch_fn f, void* user, double* best_x, double* best_cost, double* trace,
                   int32_t* gens_run, double* X_out, double* V_out, double* P_out, double* Pcost_out) {
  int32_t N = pp->particles, K = pp->generations;
  double w = or_constriction(pp->c1, pp->c2);
  if (D < 1 || N < 1 || K < 1 || isnan(w) || pp->mutation_period < 0 ||
      !(pp->mutation_fraction >= 0.0 && pp->mutation_fraction <= 1.0) || mut_lo < 0 ||
      mut_hi > D || mut_lo > mut_hi)
    return -1;
  for (int d = 0; d < D; d++)
    if (!(lo[d] <= hi[d]) || !(init_lo[d] <= init_hi[d])) return -1;
  int32_t nmut = (int32_t)floor((double)N * pp->mutation_fraction);

  double* X = calloc((size_t)N * D, sizeof(double));
  double* V = calloc((size_t)N * D, sizeof(double));
  double* P = calloc((size_t)N * D, sizeof(double));
  double* G = calloc((size_t)D, sizeof(double));
  double* Pc = calloc((size_t)N, sizeof(double));
  double* E = calloc((size_t)N, sizeof(double));
  uint8_t* mark = calloc((size_t)N, 1);

  /* Generation 0: uniform positions in the init box, zero velocity. */
  for (int32_t i = 0; i < N; i++)
    for (int32_t d = 0; d < D; d++) {
      uint32_t r[4];
      draw4(pp->seed, (uint32_t)i, (uint32_t)d, 0, 0, r);
      double u = or_u01(r[0], r[1]);
      X[(int64_t)i * D + d] = init_lo[d] + u * (init_hi[d] - init_lo[d]);
    }
  f(X, N, D, E, user);
  for (int32_t i = 0; i < N; i++) {
    Pc[i] = sanitize(E[i]);
    memcpy(&P[(int64_t)i * D], &X[(int64_t)i * D], sizeof(double) * D);
  }
  int32_t g = 0;
  for (int32_t i = 1; i < N; i++)
    if (Pc[i] < Pc[g]) g = i;
  memcpy(G, &P[(int64_t)g * D], sizeof(double) * D);
  trace[0] = Pc[g];
  int32_t ran = 1;
  int stop = pp->stop_threshold > -INFINITY && Pc[g] < pp->stop_threshold;

  for (int32_t k = 1; k < K && !stop; k++) {
    /* mutation marks: the worst floor(N*frac) by Pcost, ties -> higher index worse (AMB-17);
     * in SPEC's order they are drawn after this generation's bookkeeping instead (below) */
    int do_mut = pp->mutation_period > 0 && k % pp->mutation_period == 0 && nmut > 0;
    for (int32_t i = 0; i < N; i++) {
      mark[i] = 0;
      if (!do_mut || pp->mutation_after_eval) continue;
      int32_t rank = 0;
      for (int32_t j = 0; j < N; j++)
        if (Pc[j] < Pc[i] || (Pc[j] == Pc[i] && j < i)) rank++;
      mark[i] = rank >= N - nmut;
    }
    for (int32_t i = 0; i < N; i++) {
      uint32_t r[4];
      double r1 = 0, r2 = 0;
      for (int32_t d = 0; d < D; d++) {
        if (d == 0 || pp->per_dim_r) {
          draw4(pp->seed, (uint32_t)i, pp->per_dim_r ? (uint32_t)d : 0u, (uint32_t)k, 1, r);
          r1 = or_u01(r[0], r[1]);
          r2 = or_u01(r[2], r[3]);
        }
        int64_t id = (int64_t)i * D + d;
        /* Eq. (6): v = w (v + c1 r1 (P - x) + c2 r2 (G - x)); Eq. (7): x = x + v */
        double a = pp->c1 * r1, b = P[id] - X[id], t1 = a * b, t2 = V[id] + t1;
        double c = pp->c2 * r2, e = G[d] - X[id], t3 = c * e, t4 = t2 + t3;
        double v = w * t4, x = X[id] + v;
        if (x < lo[d]) { /* AMB-16: clamp and zero that velocity component */
          x = lo[d];
          v = 0.0;
        } else if (x > hi[d]) {
          x = hi[d];
          v = 0.0;
        }
        X[id] = x;
        V[id] = v;
      }
      if (mark[i]) /* re-seed the finger dims uniformly in bounds */
        for (int32_t d = mut_lo; d < mut_hi; d++) {
          draw4(pp->seed, (uint32_t)i, (uint32_t)d, (uint32_t)k, 2, r);
          double u = or_u01(r[0], r[1]);
          int64_t id = (int64_t)i * D + d;
          X[id] = lo[d] + u * (hi[d] - lo[d]);
          V[id] = 0.0;
        }
    }
    f(X, N, D, E, user);
    for (int32_t i = 0; i < N; i++) {
      double e = sanitize(E[i]);
      if (e < Pc[i]) { /* strict improvement (AMB-22) */
        Pc[i] = e;
        memcpy(&P[(int64_t)i * D], &X[(int64_t)i * D], sizeof(double) * D);
      }
    }
    g = 0;
    for (int32_t i = 1; i < N; i++)
      if (Pc[i] < Pc[g]) g = i;
    memcpy(G, &P[(int64_t)g * D], sizeof(double) * D);
    trace[k] = Pc[g];
    ran = k + 1;
    stop = pp->stop_threshold > -INFINITY && Pc[g] < pp->stop_threshold;
    /* SPEC's order: mutate after the evaluation, ranked by the updated Pcost; the
     * next generation's update moves the re-drawn particles before they are evaluated.  Only
     * when another generation follows (a mutation after the last evaluation is never seen). */
    if (do_mut && pp->mutation_after_eval && k + 1 < K && !stop)
      for (int32_t i = 0; i < N; i++) {
        int32_t rank = 0;
        for (int32_t j = 0; j < N; j++)
          if (Pc[j] < Pc[i] || (Pc[j] == Pc[i] && j < i)) rank++;
        if (rank < N - nmut) continue;
        for (int32_t d = mut_lo; d < mut_hi; d++) {
          uint32_t r[4];
          draw4(pp->seed, (uint32_t)i, (uint32_t)d, (uint32_t)k, 2, r);
          double u = or_u01(r[0], r[1]);
          int64_t id = (int64_t)i * D + d;
          X[id] = lo[d] + u * (hi[d] - lo[d]);
          V[id] = 0.0;
        }
      }
  }
  for (int32_t k = ran; k < K; k++) trace[k] = trace[ran - 1];
  memcpy(best_x, G, sizeof(double) * D);
  *best_cost = Pc[g];
  if (gens_run) *gens_run = ran;
  if (X_out) memcpy(X_out, X, sizeof(double) * N * D);
  if (V_out) memcpy(V_out, V, sizeof(double) * N * D);
  if (P_out) memcpy(P_out, P, sizeof(double) * N * D);
  if (Pcost_out) memcpy(Pcost_out, Pc, sizeof(double) * N);
  free(X);
  free(V);
  free(P);
  free(G);
  free(Pc);
  free(E);
  free(mark);
  return 0;
}

typedef struct {
  const double* centre;
} sphere_ctx;

static void sphere_batch(const double* X, int32_t n, int32_t D, double* costs, void* user) {
  const sphere_ctx* s = user;
  for (int32_t i = 0; i < n; i++) {
    double acc = 0.0;
    for (int32_t d = 0; d < D; d++) {
      double t = X[(int64_t)i * D + d] - s->centre[d];
      acc = acc + t * t;
    }
    costs[i] = acc;
  }
}

int32_t or_pso_sphere(int32_t D, const double* lo, const double* hi, const double* init_lo,
                      const double* init_hi, int32_t mut_lo, int32_t mut_hi, const double* centre,
                      const or_pso_params* pp, double* best_x, double* best_cost, double* trace,
                      int32_t* gens_run, double* X_out, double* V_out, double* P_out,
                      double* Pcost_out) {
  sphere_ctx s = {centre};
  return or_pso_run(D, lo, hi, init_lo, init_hi, mut_lo, mut_hi, pp, sphere_batch, &s, best_x,
                    best_cost, trace, gens_run, X_out, V_out, P_out, Pcost_out);
}

typedef struct {
  const float* od;
  const uint8_t* os;
  const or_camera* cam;
  const or_dims* d;
  const or_cost_params* cp;
  int32_t culled, threads;
} hand_ctx;

static void hand_batch(const double* X, int32_t n, int32_t D, double* costs, void* user) {
  (void)D;
  const hand_ctx* c = user;
  or_eval_batch(X, n, c->od, c->os, c->cam, c->d, c->cp, c->culled, c->threads, costs, NULL, NULL,
                NULL);
}

int32_t or_pso_fit_hand(const float* obs_depth, const uint8_t* obs_mask, const or_camera* cam,
                        const or_dims* d, const or_cost_params* cp, const or_pso_params* pp,
                        const double* init_center, const double* init_radius, int32_t culled,
                        int32_t threads, double* best_x, double* best_cost, double* trace,
                        int32_t* gens_run, double* X_out, double* V_out, double* P_out,
                        double* Pcost_out) {
  double lo[26], hi[26], ilo[26], ihi[26];
  or_bounds(lo, hi);
  for (int i = 0; i < 26; i++) {
    ilo[i] = lo[i];
    ihi[i] = hi[i];
    if (init_center && init_radius) { /* centre +- radius intersected with the bounds */
      ilo[i] = fmax(lo[i], init_center[i] - init_radius[i]);
      ihi[i] = fmin(hi[i], init_center[i] + init_radius[i]);
    }
  }
  hand_ctx c = {obs_depth, obs_mask, cam, d, cp, culled, threads};
  return or_pso_run(26, lo, hi, ilo, ihi, 6, 26, pp, hand_batch, &c, best_x, best_cost, trace,
                    gens_run, X_out, V_out, P_out, Pcost_out);
}

/* ---- observation front end (row f3; definitions in oracle.h, DESIGN.md AMB-33..36) */
void or_segment(const uint16_t* depth_u16, const uint8_t* skin, int64_t npx,
                const or_segment_params* sp, float* o_d, uint8_t* o_s, int32_t band_out[2]) {
  int64_t lo = sp->lo, hi = sp->hi;
  if (sp->mode == 1) {
    int64_t m = -1;  /* nearest candidate depth */
    for (int64_t i = 0; i < npx; i++) {
      int64_t d = depth_u16[i];
      int cand = d > 0 && (skin == NULL || skin[i] != 0);
      if (cand && (m < 0 || d < m)) m = d;
    }
    if (m < 0) {
      lo = 1;
      hi = 0;  /* empty band */
    } else {
      lo = m;
      hi = m + sp->width;
    }
  }
  for (int64_t i = 0; i < npx; i++) {
    int64_t d = depth_u16[i];
    int valid = d > 0;
    int in_band = valid && lo <= d && d <= hi;
    int s = skin ? (skin[i] != 0 && (!valid || in_band)) : in_band;
    o_s[i] = (uint8_t)s;
    if (sp->keep_background) o_d[i] = valid ? (float)d : 0.0f;
    else o_d[i] = in_band ? (float)d : 0.0f;
  }
  if (band_out) {
    band_out[0] = (int32_t)lo;
    band_out[1] = (int32_t)hi;
  }
}
