// tile.cuh — the per-pixel analytic ray casting (packed fp32x2), the warp tile / warp block (TMA observation load, cull masks, min depth, scoring) and the cost finalisation shared by the renderers
// Part of the single translation unit kernels.cu (included after the observation kernels;
// shares its macros and helpers).
#pragma once

namespace hp {

// ---------------------------------------------------------------------------------------
// Per-primitive analytic first hit for the 4 pixels of a lane (DESIGN §5 formulas).
// Pixel ray d = (dx, dy_j, 1); t_c = (d.c)/|d|^2 re-centres the quadratic at the closest
// approach to the primitive's local origin, so its coefficients are O(primitive size)
// and fp32 does not cancel (a camera-origin quadratic has |c|^2 ~ 1e6 mm^2 against
// r^2 ~ 1e2).  Depth = t (d_z = 1).
// ---------------------------------------------------------------------------------------
// Pixel pairs use Blackwell's packed fp32 instructions (FFMA2 / FMUL2 / FADD2: two lanes
// of fp32 per instruction, PTX .f32x2): the lane's pixels q = (0,1) and (2,3) are processed
// as pairs, halving the issued FP instructions of the hot loop.  Scalars broadcast into a
// pair fold into the instruction's .F32 operand modifier (no extra moves).
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ f2 bc(float v) { return pk(v, v); }
__device__ __forceinline__ void unpk(f2 v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

struct Lane4 {
  float dx;                           // shared by the lane's pixels (one column)
  f2 dy[kPxPerLane / 2];              // pairs of rows
  f2 idd[kPxPerLane / 2];             // 1 / |d|^2 per pixel, paired
  float zb[kPxPerLane];               // min depth so far
};

// Single-MUFU approximations (flush-to-zero: denormals never occur in these quantities).
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float sqrt_approx_t(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// sqrt of both halves (NaN where negative): one MUFU.SQRT each (no x * rsqrt(x) multiply)
__device__ __forceinline__ f2 sqrt2(f2 x) {
  float a, b;
  unpk(x, a, b);
  return pk(sqrt_approx_t(a), sqrt_approx_t(b));
}
// -1/x of both halves (the negation folds into the MUFU operand)
__device__ __forceinline__ f2 nrcp2(f2 x) {
  float a, b;
  unpk(x, a, b);
  return pk(rcp_approx(-a), rcp_approx(-b));
}

// Branch-free min-depth update.  zb starts just above z_far, so z < zb also enforces
// z <= z_far; a NaN z (no real root / axial range miss) never wins.
// CHK = false when FK proved every primitive lies beyond z_near (the common case): then
// a plain fminf suffices (fminf ignores a NaN operand, and zb starts above z_far).
template <bool CHK>
__device__ __forceinline__ void keep(float z, float& zb, float znear) {
  if (CHK) zb = (z >= znear) & (z < zb) ? z : zb;
  else zb = fminf(zb, z);
}
template <bool CHK>
__device__ __forceinline__ void keep2(f2 z, float& zb0, float& zb1, float znear) {
  float a, b;
  unpk(z, a, b);
  keep<CHK>(a, zb0, znear);
  keep<CHK>(b, zb1, znear);
}

template <bool CHK>
__device__ __forceinline__ void isect_sphere(const float* __restrict__ r, Lane4& L, float znear) {
  const float4 q = *reinterpret_cast<const float4*>(r);  // c, r^2
  const float bx = fmaf(L.dx, q.x, q.z);
#pragma unroll
  for (int j = 0; j < kPxPerLane / 2; j++) {
    const f2 dy = L.dy[j], idd = L.idd[j];
    const f2 tc = mul2(fma2(dy, bc(q.y), bc(bx)), idd);
    const f2 ox = fma2(tc, bc(L.dx), bc(-q.x)), oy = fma2(tc, dy, bc(-q.y));
    const f2 oz = add2(tc, bc(-q.z));
    // m = -disc / |d|^2 with disc = r^2 - |o|^2;  z = t_c - sqrt(-m) = t_c + m rsqrt(-m)
    // (NaN when disc < 0: no hit)
    const f2 m = mul2(fma2(ox, ox, fma2(oy, oy, fma2(oz, oz, bc(-q.w)))), idd);
    float m0, m1;
    unpk(m, m0, m1);
    if (CHK) {
      // exact solid semantics near the camera (DESIGN §2 render definition): the smallest
      // t > 0 on the surface — the exit root when the camera is inside the sphere
      const f2 h = mul2(m, pk(rsqrt_approx(-m0), rsqrt_approx(-m1)));  // -sqrt(-m)
      float t10, t11, t20, t21;
      unpk(add2(tc, h), t10, t11);
      unpk(sub2(tc, h), t20, t21);
      keep<true>(t10 > 0.f ? t10 : t20, L.zb[2 * j], znear);
      keep<true>(t11 > 0.f ? t11 : t21, L.zb[2 * j + 1], znear);
    } else {
      keep2<false>(fma2(m, pk(rsqrt_approx(-m0), rsqrt_approx(-m1)), tc), L.zb[2 * j],
                   L.zb[2 * j + 1], znear);
    }
  }
}

template <bool CHK>
__device__ __forceinline__ void isect_ellipsoid(const float* __restrict__ r, Lane4& L,
                                                float znear) {
  const float4 r0 = *reinterpret_cast<const float4*>(r + 0);   // c, -
  const float4 r1 = *reinterpret_cast<const float4*>(r + 4);   // M00 M01 M02 M10
  const float4 r2 = *reinterpret_cast<const float4*>(r + 8);   // M11 M12 M20 M21
  const float4 r3 = *reinterpret_cast<const float4*>(r + 12);  // M22 cl0 cl1 cl2
  // d_l = M (dx, dy, 1): the dx part is shared by the lane's pixels
  const float px = fmaf(r1.x, L.dx, r1.z), py = fmaf(r1.w, L.dx, r2.y),
              pz = fmaf(r2.z, L.dx, r3.x);
  const float bx = fmaf(L.dx, r0.x, r0.z);
#pragma unroll
  for (int j = 0; j < kPxPerLane / 2; j++) {
    const f2 dy = L.dy[j];
    const f2 tc = mul2(fma2(dy, bc(r0.y), bc(bx)), L.idd[j]);
    const f2 lx = fma2(bc(r1.y), dy, bc(px)), ly = fma2(bc(r2.x), dy, bc(py)),
             lz = fma2(bc(r2.w), dy, bc(pz));
    const f2 ox = fma2(tc, lx, bc(-r3.y)), oy = fma2(tc, ly, bc(-r3.z)),
             oz = fma2(tc, lz, bc(-r3.w));
    const f2 A = fma2(lx, lx, fma2(ly, ly, mul2(lz, lz)));
    const f2 B = fma2(ox, lx, fma2(oy, ly, mul2(oz, lz)));
    const f2 C = fma2(ox, ox, fma2(oy, oy, fma2(oz, oz, bc(-1.f))));
    const f2 disc = sub2(mul2(B, B), mul2(A, C));
    // A > 0: the smaller root; only the absolute error of s matters (z = t_c + s), so the
    // plain form is accurate to ~1e-6 mm here
    if (CHK) {  // smallest t > 0: the far root when the camera is inside
      const f2 sq = sqrt2(disc), ia = nrcp2(A);
      float t10, t11, t20, t21;
      unpk(add2(tc, mul2(add2(B, sq), ia)), t10, t11);
      unpk(add2(tc, mul2(sub2(B, sq), ia)), t20, t21);
      keep<true>(t10 > 0.f ? t10 : t20, L.zb[2 * j], znear);
      keep<true>(t11 > 0.f ? t11 : t21, L.zb[2 * j + 1], znear);
    } else {
      const f2 s = mul2(add2(B, sqrt2(disc)), nrcp2(A));
      keep2<false>(add2(tc, s), L.zb[2 * j], L.zb[2 * j + 1], znear);
    }
  }
}

// Cone (and the elliptic cylinder with k = 0 in scaled coordinates):
// x^2 + y^2 - (r_m + k z)^2 = 0 with |z| <= half length.  Only the ENTERING root
// s = (-B - sqrt(disc)) / A is needed, for A > 0 (interior [s_lo, s_hi]) and for A < 0 (ray
// inside the double cone's opening, interior (-inf, s_lo] U [s_hi, inf)) alike: if it is
// outside the axial range the ray can only enter the finite solid through a cap disc, and
// every cap disc is the equator of a joint sphere / cap ellipsoid that is hit first
// (DESIGN §2), so the min over primitives is unchanged.
template <bool CHK>
__device__ __forceinline__ void isect_cone(const float* __restrict__ r, Lane4& L, float znear) {
  const float4 r0 = *reinterpret_cast<const float4*>(r + 0);
  const float4 r1 = *reinterpret_cast<const float4*>(r + 4);
  const float4 r2 = *reinterpret_cast<const float4*>(r + 8);
  const float4 r3 = *reinterpret_cast<const float4*>(r + 12);
  const float4 r4 = *reinterpret_cast<const float4*>(r + 16);  // rm, k, hl, -
  const float px = fmaf(r1.x, L.dx, r1.z), py = fmaf(r1.w, L.dx, r2.y),
              pz = fmaf(r2.z, L.dx, r3.x);
  const float bx = fmaf(L.dx, r0.x, r0.z);
  const float rm = r4.x, k = r4.y, hl = r4.z;
#pragma unroll
  for (int j = 0; j < kPxPerLane / 2; j++) {
    const f2 dy = L.dy[j];
    const f2 tc = mul2(fma2(dy, bc(r0.y), bc(bx)), L.idd[j]);
    const f2 lx = fma2(bc(r1.y), dy, bc(px)), ly = fma2(bc(r2.x), dy, bc(py)),
             lz = fma2(bc(r2.w), dy, bc(pz));
    const f2 ox = fma2(tc, lx, bc(-r3.y)), oy = fma2(tc, ly, bc(-r3.z)),
             oz = fma2(tc, lz, bc(-r3.w));
    const f2 g = fma2(bc(k), oz, bc(rm)), kd = mul2(bc(k), lz);
    const f2 A = fma2(lx, lx, fma2(ly, ly, sub2(bc(0.f), mul2(kd, kd))));
    const f2 B = fma2(ox, lx, fma2(oy, ly, sub2(bc(0.f), mul2(kd, g))));
    const f2 C = fma2(ox, ox, fma2(oy, oy, sub2(bc(0.f), mul2(g, g))));
    const f2 disc = sub2(mul2(B, B), mul2(A, C));
    if (CHK) {
      // Exact solid near the camera: with the near plane cutting a joint sphere, the caps
      // are no longer covered, so take the smallest t > 0 over both lateral roots in the
      // axial range and both cap discs (as the oracle's or_first_hit does).
      float a_[2], b_[2], dsc[2], tcv[2], lxv[2], lyv[2], lzv[2], oxv[2], oyv[2], ozv[2];
      unpk(A, a_[0], a_[1]);
      unpk(B, b_[0], b_[1]);
      unpk(disc, dsc[0], dsc[1]);
      unpk(tc, tcv[0], tcv[1]);
      unpk(lx, lxv[0], lxv[1]);
      unpk(ly, lyv[0], lyv[1]);
      unpk(lz, lzv[0], lzv[1]);
      unpk(ox, oxv[0], oxv[1]);
      unpk(oy, oyv[0], oyv[1]);
      unpk(oz, ozv[0], ozv[1]);
#pragma unroll
      for (int e = 0; e < 2; e++) {
        float best = __int_as_float(0x7f800000);
        const float sq = sqrtf(dsc[e]), ia = 1.f / a_[e];  // NaN roots when disc < 0
        const float sr[2] = {-(b_[e] + sq) * ia, (sq - b_[e]) * ia};
#pragma unroll
        for (int i = 0; i < 2; i++) {
          const float t = tcv[e] + sr[i];
          if (fabsf(fmaf(sr[i], lzv[e], ozv[e])) <= hl && t > 0.f) best = fminf(best, t);
        }
#pragma unroll
        for (int c = 0; c < 2; c++) {
          const float zc = c == 0 ? -hl : hl, rc = fmaf(k, zc, rm);
          const float sc = (zc - ozv[e]) / lzv[e];
          const float x = fmaf(sc, lxv[e], oxv[e]), y = fmaf(sc, lyv[e], oyv[e]);
          const float t = tcv[e] + sc;
          if (fmaf(x, x, y * y) <= rc * rc && t > 0.f) best = fminf(best, t);
        }
        keep<true>(best, L.zb[2 * j + e], znear);
      }
    } else {
      const f2 s = mul2(add2(B, sqrt2(disc)), nrcp2(A));  // NaN when disc < 0
      float za0, za1, z0, z1;
      unpk(fma2(s, lz, oz), za0, za1);
      unpk(add2(tc, s), z0, z1);
      const float nan = __int_as_float(0x7fc00000);
      keep<false>(fabsf(za0) <= hl ? z0 : nan, L.zb[2 * j], znear);
      keep<false>(fabsf(za1) <= hl ? z1 : nan, L.zb[2 * j + 1], znear);
    }
  }
}

// 1/x of both halves (one MUFU.RCP each)
__device__ __forceinline__ f2 rcp2(f2 x) {
  float a, b;
  unpk(x, a, b);
  return pk(rcp_approx(a), rcp_approx(b));
}

// ---------------------------------------------------------------------------------------
// Fast path, every primitive kind: the inverse-depth polynomial form (common.cuh FAST record
// layout).  Per lane (one column x): x' = x - xp and the y-Horner coefficients of D, b's
// affine part (b pre-scaled by 1 / c0), for cones the axial line's x part; per pixel pair:
// y' = y - yp, D by Horner, the inverse depth s = sqrt(D) / c0 + b / c0 of the entering
// root t = (b - sqrt(D)) / a (the same root: s = 1 / t), and the running MAXIMUM of s —
// 6 packed fp32x2 instructions and 2 MUFU for a sphere / ellipsoid pair, 8 + 2 FSETP for a
// cone, against 14-17 and 4 MUFU for the depth form (no per-pixel 1 / a, no 1 / |d|^2).  The
// depth is 1 / s once per pixel after all primitives.  For a < 0 (a ray inside a cone's
// opening) the root is the larger one, the entering one of the infinite solid; whenever it
// lies outside the axial range the ray enters the finite solid through a cap disc, which is
// the equator of a joint sphere / cap ellipsoid hit first, so the max over
// primitives is unchanged.  NaN (no real root) never wins; neither does a negative s (a
// root behind the camera) nor one outside the axial range.
// ---------------------------------------------------------------------------------------
struct QuadLane {
  float yp, d02, by, ic0, ed0, ed1, eb0;
  float lzy, lzl, nclz;  // axial (cones / cylinder), scaled by 1 / hl
};
template <bool AXIAL>
__device__ __forceinline__ QuadLane quad_lane(uint32_t r, float dx) {  // r: record address
  const float4 r0 = lds_f4_nv(r + 0);   // xp yp d00 d10
  const float4 r1 = lds_f4_nv(r + 16);  // d01 d20 d11 d02
  const float4 r2 = lds_f4_nv(r + 32);  // b0 bx by ic0 (b / c0)
  QuadLane q;
  if (AXIAL) {
    const float4 r3 = lds_f4_nv(r + 48);  // lzx lzy lz1 nclz (/ hl)
    q.lzy = r3.y;
    q.lzl = fmaf(r3.x, dx, r3.z);
    q.nclz = r3.w;
  }
  const float xq = dx - r0.x;
  q.yp = r0.y;
  q.d02 = r1.w;
  q.by = r2.z;
  q.ic0 = r2.w;
  q.ed0 = fmaf(fmaf(r1.y, xq, r0.w), xq, r0.z);
  q.ed1 = fmaf(r1.z, xq, r1.x);
  q.eb0 = fmaf(r2.y, xq, r2.x);
  return q;
}
// One pixel pair (rows dy): the inverse depth of the entering root, kept if larger.
template <bool AXIAL>
__device__ __forceinline__ void quad_pair(const QuadLane& q, f2 dy, float& sb0, float& sb1) {
  const f2 yq = sub2(dy, bc(q.yp));
  const f2 D = fma2(fma2(bc(q.d02), yq, bc(q.ed1)), yq, bc(q.ed0));
  const f2 B = fma2(bc(q.by), yq, bc(q.eb0));
  const f2 s = fma2(sqrt2(D), bc(q.ic0), B);  // NaN when D < 0: no hit
  float s0, s1;
  unpk(s, s0, s1);
  if (AXIAL) {
    // axial coordinate within [-hl, hl]: |s (-cl_z / hl) + (axis . d) / hl| <= s (false for
    // NaN and for s < 0); a predicated max, no select
    const f2 xv = fma2(bc(q.nclz), s, fma2(bc(q.lzy), dy, bc(q.lzl)));
    float x0, x1;
    unpk(xv, x0, x1);
    if (fabsf(x0) <= s0) sb0 = fmaxf(sb0, s0);
    if (fabsf(x1) <= s1) sb1 = fmaxf(sb1, s1);
  } else {
    sb0 = fmaxf(sb0, s0);
    sb1 = fmaxf(sb1, s1);
  }
}
// Depth of the nearest hit from the largest inverse depth: 1 / s (0 -> +inf: no hit).
__device__ __forceinline__ float depth_of(float sb) { return rcp_approx(sb); }

// ---------------------------------------------------------------------------------------
// One warp tile: TMA the observation tile, cull, ray-cast, min-depth, score.
// ---------------------------------------------------------------------------------------
struct TileSums {
  unsigned int rm = 0, both = 0, and_ = 0;
  unsigned long long num = 0;
};

// Tile geometry of a particle: the union box's x0 rounded down to 4 px, because a TMA box
// must start 16-byte aligned in global memory (an unaligned start faults on sm_100a).
struct TileGrid {
  int x0 = 0, y0 = 0, tx = 0, ntiles = 0;
  unsigned int magic = 0u;  // floor(2^32 / tx): t / tx = umulhi(t, magic) + {0, 1}
  TileGrid() = default;
  // need_origin = false: only the tile counts (origin() is not called; skips the division)
  __device__ __forceinline__ explicit TileGrid(int4 ub, bool need_origin = true) {
    x0 = ub.x & ~3;
    y0 = ub.y;
    const int bw = ub.z - x0 + 1, bh = ub.w - y0 + 1;
    tx = bw > 0 ? (bw + kTileW - 1) / kTileW : 0;
    const int ty = bh > 0 ? (bh + kTileH - 1) / kTileH : 0;
    ntiles = tx * ty;
    magic = need_origin && tx > 1 ? 0xFFFFFFFFu / (unsigned)tx : 0u;
  }
  __device__ __forceinline__ void origin(int t, int& X0, int& Y0) const {
    int qy = tx > 1 ? (int)__umulhi((unsigned)t, magic) : t;
    int qx = t - qy * tx;
    if (qx >= tx) {  // the estimate is low by at most one
      qy++;
      qx -= tx;
    }
    X0 = x0 + qx * kTileW;
    Y0 = y0 + qy * kTileH;
  }
};

// Cull the 38 conservative boxes against the tile [X0, X0+16) x [Y0, Y0+8): two ballots,
// split into 32-bit masks per kind (spheres = prims 0..19, cones + cylinder = 20..34,
// ellipsoids = 35..37).  Warp-collective.
__device__ __forceinline__ uint3 cull_tile(const FkOut& fo, int X0, int Y0) {
  const int lane = threadIdx.x & 31;
  const int4 b = fo.box[lane];
  const bool ov = b.x <= X0 + kTileW - 1 && b.z >= X0 && b.y <= Y0 + kTileH - 1 && b.w >= Y0;
  bool ov2 = false;
  if (lane < kNprim - 32) {
    const int4 c = fo.box[32 + lane];
    ov2 = c.x <= X0 + kTileW - 1 && c.z >= X0 && c.y <= Y0 + kTileH - 1 && c.w >= Y0;
  }
  const unsigned int lo = __ballot_sync(0xffffffffu, ov), hi = __ballot_sync(0xffffffffu, ov2);
  return make_uint3(lo & 0xFFFFFu, (lo >> 20) | ((hi & 0x7u) << 12), hi >> 3);
}

// Scoring of a lane's NPX pixels (rows rowb + 2 q of its column col in the observation
// tile, ROWS rows of 16 words): r_m, o_s AND r_m, the clamped |o_d - r_d| numerator and
// (BOTH) the both-defined count (AMB-1, -3, -4, -5).  Skipped for tiles where
// nothing rendered.
template <int NPX, bool BOTH>
__device__ __forceinline__ void score_lane(const EvalArgs& a, const float* zb, uint32_t obs_ls,
                                           TileSums& acc) {
  const float zfar = a.cam.zfar;
  const float d_m = a.cost.d_m, clampv = a.cost.clampv;
  const float qscale = a.cost.qscale, qmagic = a.cost.qmagic;
  bool any = false;
#pragma unroll
  for (int q = 0; q < NPX; q++) any |= zb[q] <= zfar;
  if (__any_sync(0xffffffffu, any)) {  // nothing rendered in this tile: nothing to score
    // numerator: round(min(|dd|, clamp) 2^qbits) from the bits of an fp32 magic-number
    // FFMA (exact: the value lies in [2^23, 2^24], ulp 1) minus the magic's bits: no
    // float-to-int conversion on the XU; every count is a predicated add
    const unsigned int magic_bits = __float_as_uint(qmagic);
    unsigned int num = 0u, both = 0u;
#pragma unroll
    for (int q = 0; q < NPX; q++) {
      const uint32_t w = lds_u32(obs_ls + 4u * (2 * q) * kTileW);
      // diff = | |o| - z |: o_d undefined is stored as NaN (kObsUndef), so diff is NaN
      // exactly there; bit 31 (o_s) is the float's sign, dropped by the absolute value.
      // hit = z <= z_far (off-image pixels have NaN rays and never hit, k_ray_table).
      // r_m = hit AND (diff < d_m OR o_d undefined) (AMB-4, AMB-5): "ltu" is
      // true for NaN.  o_s AND r_m adds bit 31 of w.  Both depths defined: hit AND diff
      // is a number; the numerator adds the bits of the magic-number FFMA minus the
      // magic's (predicated adds only: no selects, no float-to-int conversion).
      // r_m and o_s AND r_m in one packed counter (one PRMT + one predicated add): the
      // increment is 1 + (o_s ? 0xFFFF0000 : 0) — o_s's sign bit replicated into the high
      // half — so the counter holds r_m - (o_s AND r_m) 2^16 (unpack_counts)
      asm("{\n\t"
          ".reg .pred ph, pr, pb;\n\t"
          ".reg .f32 d, c;\n\t"
          ".reg .b32 t;\n\t"
          "mov.b32 d, %3;\n\t"
          "abs.f32 d, d;\n\t"
          "sub.f32 d, d, %4;\n\t"
          "abs.f32 d, d;\n\t"
          "setp.le.f32 ph, %4, %5;\n\t"
          "setp.ltu.and.f32 pr, d, %6, ph;\n\t"
          "prmt.b32 t, %3, 1, 0xBB54;\n\t"
          "@pr add.u32 %0, %0, t;\n\t"
          "setp.num.and.f32 pb, d, d, ph;\n\t"
          "@pb add.u32 %1, %1, 1;\n\t"
          "min.f32 c, d, %7;\n\t"
          "fma.rn.f32 c, c, %8, %9;\n\t"
          "mov.b32 t, c;\n\t"
          "sub.u32 t, t, %10;\n\t"
          "@pb add.u32 %2, %2, t;\n\t"
          "}"
          : "+r"(acc.rm), "+r"(both), "+r"(num)
          : "r"(w), "f"(zb[q]), "f"(zfar), "f"(d_m), "f"(clampv), "f"(qscale), "f"(qmagic),
            "r"(magic_bits));
    }
    if (BOTH) acc.both += both;
    acc.num += num;
  }
}

// One warp tile of 16 x 8 pixels (k_eval, the near-plane pass, the depth hooks): TMA the
// observation tile, ray-cast the culled primitives, min depth, score.  Lane: column
// lane & 15, rows lane >> 4 + {0, 2, 4, 6}.
// CHK = false: the FAST records of fo (the hot path); CHK = true: exact solid semantics
// near the camera from the EXACT records xr (instantiated only out of line, tiles_near).
// BOTH: count the both-defined pixels (only the hp_eval_sums test hook reports them).
// TMA: the observation-tile load, a.use_tma at run time (-1) or fixed at compile time (1).
template <int MODE, bool CHK, bool BOTH = true, int TMA = -1>
__device__ __forceinline__ void do_tile(const EvalArgs& a, const CUtensorMap* tmap,
                                        const FkOut& fo, const FkExact* xr, int X0, int Y0,
                                        uint3 km, uint32_t obs_s, uint32_t bar_s,
                                        uint32_t& phase, uint32_t dx_s, uint32_t dy_s,
                                        TileSums& acc, int yoff = 0) {
  const int lane = threadIdx.x & 31;
  const int col = lane & 15, rowb = lane >> 4;
  const float znear = a.cam.znear, zfar = a.cam.zfar;
  const float zinit = __uint_as_float(__float_as_uint(zfar) + 1u);  // next float above z_far
  const int use_tma = TMA >= 0 ? TMA : a.use_tma;
  if (MODE == kModeCost && use_tma) {
    // no proxy fence needed: the warp's reads of the previous tile in this buffer were
    // consumed before the __syncwarp that ended it (WAR across proxies is ordered)
    // rows past this frame's bottom come from the next frame (or TMA zero fill): they are
    // off-image, their rays are NaN and they are never scored
    HP_CHECK(yoff >= 0 && Y0 < a.cam.H);
    tma_load_2d_elect_s(obs_s, use_tma == 2 ? a.tmap_g : tmap, X0, Y0 + yoff, bar_s,
                        kTileW * kTileH * 4);
  }
  const unsigned int msph = km.x, mcone = km.y, mell = km.z;
  Lane4 L;
  const int x = X0 + col;
  HP_CHECK(X0 >= 0 && x < ray_dx_len(a.cam.W) && Y0 >= 0 && Y0 + rowb < a.cam.H + kRayPad);
  HP_CHECK((X0 & 3) == 0);  // TMA boxes start 16-byte aligned
  // the ray table by shared address: dx_s = &dx[lane's column], dy_s = &dy4[lane's row]
  L.dx = __uint_as_float(lds_u32(dx_s + 4u * X0));
  const float4 dy4 = lds_f4(dy_s + 16u * Y0);  // rows y, y+2, y+4, y+6
  const float dyv[4] = {dy4.x, dy4.y, dy4.z, dy4.w};
#pragma unroll
  for (int q = 0; q < kPxPerLane; q += 2) {
    const float dy0 = dyv[q], dy1 = dyv[q + 1];
    L.dy[q / 2] = pk(dy0, dy1);
    if (CHK) {  // the exact path's depth form needs 1 / |d|^2; the fast path none
      const float ddx = fmaf(L.dx, L.dx, 1.f);
      L.idd[q / 2] = pk(rcp_approx(fmaf(dy0, dy0, ddx)), rcp_approx(fmaf(dy1, dy1, ddx)));
    }
    L.zb[q] = CHK ? zinit : 0.f;  // fast path: the largest inverse depth so far
    L.zb[q + 1] = CHK ? zinit : 0.f;
  }
  if (CHK) {
    // exact solid semantics (both roots, cone caps, [z_near, z_far]) from the EXACT records
    for (unsigned int m = msph; m; m &= m - 1) isect_sphere<true>(xr->rec[__ffs(m) - 1], L, znear);
    for (unsigned int m = mcone; m; m &= m - 1)
      isect_cone<true>(xr->rec[kCone0 + __ffs(m) - 1], L, znear);
    for (unsigned int m = mell; m; m &= m - 1)
      isect_ellipsoid<true>(xr->rec[kEll0 + __ffs(m) - 1], L, znear);
  } else {
    for (unsigned int m = msph; m; m &= m - 1) {
      const QuadLane Q = quad_lane<false>(smem_u32(fo.rec[__ffs(m) - 1]), L.dx);
      quad_pair<false>(Q, L.dy[0], L.zb[0], L.zb[1]);
      quad_pair<false>(Q, L.dy[1], L.zb[2], L.zb[3]);
    }
    for (unsigned int m = mcone; m; m &= m - 1) {  // cones and the palm cylinder
      const QuadLane Q = quad_lane<true>(smem_u32(fo.rec[kCone0 + __ffs(m) - 1]), L.dx);
      quad_pair<true>(Q, L.dy[0], L.zb[0], L.zb[1]);
      quad_pair<true>(Q, L.dy[1], L.zb[2], L.zb[3]);
    }
    for (unsigned int m = mell; m; m &= m - 1) {
      const QuadLane Q = quad_lane<false>(smem_u32(fo.rec[kEll0 + __ffs(m) - 1]), L.dx);
      quad_pair<false>(Q, L.dy[0], L.zb[0], L.zb[1]);
      quad_pair<false>(Q, L.dy[1], L.zb[2], L.zb[3]);
    }
#pragma unroll
    for (int q = 0; q < kPxPerLane; q++) L.zb[q] = depth_of(L.zb[q]);
  }

  if (MODE == kModeDepth) {
#pragma unroll
    for (int q = 0; q < kPxPerLane; q++) {
      const int y = Y0 + rowb + 2 * q;
      if (x < a.cam.W && y < a.cam.H)
        a.depth_out[(size_t)y * a.cam.W + x] = L.zb[q] <= zfar ? L.zb[q] : 0.f;
    }
  } else {
    if (use_tma) {
      mbar_wait_s(bar_s, phase);
      phase ^= 1u;
    } else {
#pragma unroll
      for (int q = 0; q < kPxPerLane; q++) {
        const int y = Y0 + rowb + 2 * q;
        sts_u32(obs_s + 4u * ((rowb + 2 * q) * kTileW + col),
                (x < a.cam.W && y < a.cam.H) ? a.obs[(size_t)(y + yoff) * a.obs_pitch + x] : 0u);
      }
      __syncwarp();
    }
    score_lane<kPxPerLane, BOTH>(a, L.zb, obs_s + 4u * (rowb * kTileW + col), acc);
  }
  __syncwarp();
}

// A block-list entry (32 bytes): the block origin and its primitive masks already split
// the way the renderer's loops take them — per kind, the primitives in both 16 x 8 halves,
// in the top half only and in the bottom half only — so the loops start without decoding.
//   a = (X0 | Y0 << 16, spheres both, spheres top only, spheres bottom only)
//   b = (cones both, cones top only, cones bottom only, ellipsoids both | top << 8 |
//        bottom << 16)
// (spheres = prims 0..19, cones + the palm cylinder = 20..34, ellipsoids = 35..37)
struct BlockEnt {
  uint4 a, b;
};
__device__ __forceinline__ BlockEnt make_block_ent(int X0, int Y0, uint3 top, uint3 bot) {
  const unsigned s2 = top.x & bot.x, c2 = top.y & bot.y, e2 = top.z & bot.z;
  BlockEnt e;
  e.a = make_uint4((unsigned)X0 | ((unsigned)Y0 << 16), s2, top.x ^ s2, bot.x ^ s2);
  e.b = make_uint4(c2, top.y ^ c2, bot.y ^ c2, e2 | ((top.z ^ e2) << 8) | ((bot.z ^ e2) << 16));
  return e;
}
// The 38-bit half-block mask (lo: prims 0..31, hi: 32..37) split by kind.
__device__ __forceinline__ uint3 split_kinds(uint2 m) {
  return make_uint3(m.x & 0xFFFFFu, (m.x >> 20) | ((m.y & 7u) << 12), m.y >> 3);
}

// The batch renderer's warp BLOCK: 16 x 16 pixels = two 16 x 8 tiles with their own cull
// masks (the over-test of 16 x 8 tiles) sharing one tile fetch, one 1 KB TMA observation
// load, the ray set-up and each primitive's per-lane set-up.  Lane: column lane & 15,
// rows lane >> 4 + {0, 2, ..., 14}; pairs 0, 1 are the top tile, 2, 3 the bottom.
// rec_s: shared address of the particle's FAST records; obs_s: the warp's observation
// buffer, obs_ls: this lane's first pixel in it (column lane & 15, row lane >> 4).
template <bool SUMS, bool RG = false>
__device__ __forceinline__ void do_block(const EvalArgs& a, const CUtensorMap* tmap,
                                         uint32_t rec_s, BlockEnt e, uint32_t obs_s,
                                         uint32_t obs_ls, uint32_t bar_s, uint32_t& phase,
                                         uint32_t dx_s, uint32_t dy_s, TileSums& acc, int yoff,
                                         const float* ray_x = nullptr,
                                         const float4* ray_y = nullptr) {
  const uint4 ent = e.a;
  const int X0 = (int)(ent.x & 0xFFFFu), Y0 = (int)(ent.x >> 16);
  HP_CHECK(yoff >= 0 && Y0 < a.cam.H && (X0 & 3) == 0);
  tma_load_2d_elect_s(obs_s, tmap, X0, Y0 + yoff, bar_s, kTileW * kBlockH * 4);
  // RG: the ray table through L1 (global), else the CTA's shared copy
  const float dx = RG ? __ldg(ray_x + X0) : __uint_as_float(lds_u32(dx_s + 4u * X0));
  const float4 ya = RG ? __ldg(ray_y + Y0) : lds_f4(dy_s + 16u * Y0);  // rows y .. y+6
  const float4 yb = RG ? __ldg(ray_y + Y0 + 8) : lds_f4(dy_s + 16u * (Y0 + 8));  // y+8 ..
  const f2 dy[4] = {pk(ya.x, ya.y), pk(ya.z, ya.w), pk(yb.x, yb.y), pk(yb.z, yb.w)};
  float zb[8];  // the largest inverse depth so far, then the depth
#pragma unroll
  for (int q = 0; q < 8; q++) zb[q] = 0.f;
  // masks per kind, split into primitives in both halves / the top only / the bottom only
  // (no per-primitive half tests in the loops)
  const unsigned int s2 = ent.y, s_t = ent.z, s_b = ent.w;
  const unsigned int c2 = e.b.x, c_t = e.b.y, c_b = e.b.z;
  const unsigned int e2 = e.b.w & 0xFFu, e_t = (e.b.w >> 8) & 0xFFu, e_b = e.b.w >> 16;
  for (unsigned int m = s2; m; m &= m - 1) {
    const QuadLane Q = quad_lane<false>(rec_s + 4u * kRec * (__ffs(m) - 1), dx);
#pragma unroll
    for (int k = 0; k < 4; k++) quad_pair<false>(Q, dy[k], zb[2 * k], zb[2 * k + 1]);
  }
  for (unsigned int m = s_t; m; m &= m - 1) {
    const QuadLane Q = quad_lane<false>(rec_s + 4u * kRec * (__ffs(m) - 1), dx);
#pragma unroll
    for (int k = 0; k < 2; k++) quad_pair<false>(Q, dy[k], zb[2 * k], zb[2 * k + 1]);
  }
  for (unsigned int m = s_b; m; m &= m - 1) {
    const QuadLane Q = quad_lane<false>(rec_s + 4u * kRec * (__ffs(m) - 1), dx);
#pragma unroll
    for (int k = 2; k < 4; k++) quad_pair<false>(Q, dy[k], zb[2 * k], zb[2 * k + 1]);
  }
  // cones and the palm cylinder
  for (unsigned int m = c2; m; m &= m - 1) {
    const QuadLane Q = quad_lane<true>(rec_s + 4u * kRec * (kCone0 + __ffs(m) - 1), dx);
#pragma unroll
    for (int k = 0; k < 4; k++) quad_pair<true>(Q, dy[k], zb[2 * k], zb[2 * k + 1]);
  }
  for (unsigned int m = c_t; m; m &= m - 1) {
    const QuadLane Q = quad_lane<true>(rec_s + 4u * kRec * (kCone0 + __ffs(m) - 1), dx);
#pragma unroll
    for (int k = 0; k < 2; k++) quad_pair<true>(Q, dy[k], zb[2 * k], zb[2 * k + 1]);
  }
  for (unsigned int m = c_b; m; m &= m - 1) {
    const QuadLane Q = quad_lane<true>(rec_s + 4u * kRec * (kCone0 + __ffs(m) - 1), dx);
#pragma unroll
    for (int k = 2; k < 4; k++) quad_pair<true>(Q, dy[k], zb[2 * k], zb[2 * k + 1]);
  }
  for (unsigned int m = e2; m; m &= m - 1) {
    const QuadLane Q = quad_lane<false>(rec_s + 4u * kRec * (kEll0 + __ffs(m) - 1), dx);
#pragma unroll
    for (int k = 0; k < 4; k++) quad_pair<false>(Q, dy[k], zb[2 * k], zb[2 * k + 1]);
  }
  for (unsigned int m = e_t; m; m &= m - 1) {
    const QuadLane Q = quad_lane<false>(rec_s + 4u * kRec * (kEll0 + __ffs(m) - 1), dx);
#pragma unroll
    for (int k = 0; k < 2; k++) quad_pair<false>(Q, dy[k], zb[2 * k], zb[2 * k + 1]);
  }
  for (unsigned int m = e_b; m; m &= m - 1) {
    const QuadLane Q = quad_lane<false>(rec_s + 4u * kRec * (kEll0 + __ffs(m) - 1), dx);
#pragma unroll
    for (int k = 2; k < 4; k++) quad_pair<false>(Q, dy[k], zb[2 * k], zb[2 * k + 1]);
  }
#pragma unroll
  for (int q = 0; q < 8; q++) zb[q] = depth_of(zb[q]);
  mbar_wait_s(bar_s, phase);
  phase ^= 1u;
#if HP_HALF_SCORE
  // each 16 x 8 half scored only if something was rendered in it
  score_lane<4, SUMS>(a, zb, obs_ls, acc);
  score_lane<4, SUMS>(a, zb + 4, obs_ls + 4u * 8 * kTileW, acc);
#else
  score_lane<8, SUMS>(a, zb, obs_ls, acc);
#endif
  __syncwarp();
}

// A warp's share of one particle's 16 x 8 tiles (k_eval, the near-plane pass): the union
// grid with per-tile box culling; the warps of a CTA take tiles through the shared counter
// *next.  xr: the EXACT records (read by the CHK instantiation only).
struct TileRun {
  TileSums acc;
  uint32_t phase;
};
template <int MODE, bool CHK, bool BOTH = true, int TMA = -1>
__device__ __forceinline__ TileRun tile_loop(const EvalArgs& a, const CUtensorMap* tmap,
                                             const FkOut& fo, const FkExact* xr, int first,
                                             int stride, int count, int* next, uint32_t obs_s,
                                             uint32_t bar_s, uint32_t phase, const float* s_dx,
                                             const float* s_dy, int yoff) {
  const int lane = threadIdx.x & 31;
  const TileGrid g(fo.ubox);
  TileRun r;
  r.phase = phase;
  // loop-invariant shared addresses in registers (see k_render_persist)
  obs_s = pin_u32(obs_s);
  bar_s = pin_u32(bar_s);
  const uint32_t dx_s = pin_u32(smem_u32(s_dx + (lane & 15)));
  const uint32_t dy_s = pin_u32(smem_u32(s_dy + 4 * (lane >> 4)));
  int j = 0;
  if (lane == 0) j = atomicAdd(next, 1);
  j = __shfl_sync(0xffffffffu, j, 0);
  while (j < count) {
    int jn = 0;
    if (lane == 0) jn = atomicAdd(next, 1);  // the next tile, fetched early
    int X0, Y0;
    g.origin(first + j * stride, X0, Y0);
    const uint3 km = cull_tile(fo, X0, Y0);
    if (km.x | km.y | km.z)  // no primitive box touches the tile: nothing to render or score
      do_tile<MODE, CHK, BOTH, TMA>(a, tmap, fo, xr, X0, Y0, km, obs_s, bar_s, r.phase, dx_s,
                                    dy_s, r.acc, yoff);
    j = __shfl_sync(0xffffffffu, jn, 0);
  }
  return r;
}

// Particles with a primitive that may cross z_near (rare: a hand within ~25 cm of the near
// plane) take the exact-solid path out of line, so its registers never weigh on the hot
// loop's allocation.  The kernels' EvalArgs are __grid_constant__: no copy for the reference.
template <int MODE>
__device__ __noinline__ TileRun tiles_near(const EvalArgs& a, const CUtensorMap* tmap,
                                           const FkOut& fo, const FkExact* xr, int first,
                                           int stride, int count, int* next, uint32_t obs_s,
                                           uint32_t bar_s, uint32_t phase, const float* s_dx,
                                           const float* s_dy, int yoff) {
  return tile_loop<MODE, true>(a, tmap, fo, xr, first, stride, count, next, obs_s, bar_s,
                               phase, s_dx, s_dy, yoff);
}

// NEARCODE = false (the speculative fit kernels): no near-plane code at all; a particle
// that would need it raises a_.near_seen and the host re-runs the fit with NEARCODE = true.
template <int MODE, bool NEARCODE = true>
__device__ __forceinline__ TileRun run_tiles(const EvalArgs& a, const CUtensorMap* tmap,
                                             const FkOut& fo, const FkExact* xr, int first,
                                             int stride, int count, int* next, uint32_t obs_s,
                                             uint32_t bar_s, uint32_t phase, const float* s_dx,
                                             const float* s_dy, int yoff) {
#if HP_NEAR_TEST
  return tile_loop<MODE, false>(a, tmap, fo, xr, first, stride, count, next, obs_s, bar_s,
                                phase, s_dx, s_dy, yoff);
#else
  if (!NEARCODE) {
    if (!fo.near_ok && threadIdx.x == 0 && a.near_seen) atomicOr(a.near_seen, 1);
    return tile_loop<MODE, false>(a, tmap, fo, xr, first, stride, count, next, obs_s, bar_s,
                                  phase, s_dx, s_dy, yoff);
  }
  if (fo.near_ok)
    return tile_loop<MODE, false>(a, tmap, fo, xr, first, stride, count, next, obs_s, bar_s,
                                  phase, s_dx, s_dy, yoff);
  return tiles_near<MODE>(a, tmap, fo, xr, first, stride, count, next, obs_s, bar_s, phase,
                          s_dx, s_dy, yoff);
#endif
}

// Sum of a 64-bit value over the warp by two 32-bit REDUX: the low 24 bits and the rest.
// Exact while every lane's value is < 2^51 (each part's 32-lane sum stays < 2^32): a lane's
// numerator is < 2^25 per block (8 pixels of <= 2^22) and a particle has < 2^17 tiles
// (the ray table limits the image to < 2^24 pixels).
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
  const unsigned int lo = __reduce_add_sync(0xffffffffu, (unsigned int)v & 0xFFFFFFu);
  const unsigned int hi = __reduce_add_sync(0xffffffffu, (unsigned int)(v >> 24));
  return ((unsigned long long)hi << 24) + lo;
}
// The lane's packed counter (score_lane: rm holds r_m - (o_s AND r_m) 2^16, both < 2^16
// per lane) split into the two counts; once per lane before warp_reduce.
__device__ __forceinline__ void unpack_counts(TileSums& s) {
  const unsigned int p = s.rm;
  s.rm = p & 0xFFFFu;
  s.and_ = (0u - (p >> 16)) & 0xFFFFu;
}
template <bool BOTH = true>
__device__ __forceinline__ void warp_reduce(TileSums& s) {
  s.rm = __reduce_add_sync(0xffffffffu, s.rm);
  s.and_ = __reduce_add_sync(0xffffffffu, s.and_);
  if (BOTH) s.both = __reduce_add_sync(0xffffffffu, s.both);
  s.num = warp_sum_u64(s.num);
}

// Eq. (4)-(5) in fp64 from the integer sums v = (sum r_m, sum o_s AND r_m, numerator in
// 2^-qbits mm, both-defined count)  (AMB-1, -2, -3, -6).
__device__ __forceinline__ double finalize_cost(const EvalArgs& a, int p,
                                                const unsigned long long v[4], double kc) {
  const long long s_rm = (long long)v[0], s_and = (long long)v[1];
  const long long s_or = (long long)a.S_o[frame_of(a, p)] + s_rm - s_and;
  double D = 0.0;
  if (s_or > 0) {
    // 2^-qbits exactly (qbits in [0, 20]): the same bits as ldexp, without its slow path
    const double num = (double)v[2] * __longlong_as_double((long long)(1023 - a.cost.qbits) << 52);
    const double sor = (double)s_or, sand = (double)s_and;
    D = a.cost.depth_scale * num / sor + a.cost.lambda * (1.0 - 2.0 * sand / (sand + sor));
  }
  const double E = D + a.cost.lambda_k * kc;
  if (a.costs32) a.costs32[p] = (float)E;
  if (a.costs64) a.costs64[p] = E;
  if (a.sums_out)  // the ABI reports the numerator in 2^-20 mm (qbits <= 20)
    for (int k = 0; k < 4; k++)
      a.sums_out[(size_t)p * 4 + k] = k == 2 ? v[k] << (20 - a.cost.qbits) : v[k];
  return E;
}


}  // namespace hp
