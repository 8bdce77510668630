// kernels.cu — the hot path of libhp on sm_100a.
//
//   k_pack_obs, k_band_min, k_ingest : observation O = (O_s, O_d) -> one u32 per pixel
//                (fp32 depth bits, undefined depth = a quiet NaN, bit 31 = o_s) and
//                S_o = sum o_s; k_band_min / k_ingest segment a Kinect-like u16 frame first
//                (rows A0, f3)
//   k_ray_table: per-column dx, per-lane-row dy4 (NaN off the image)
//   k_fk_batch : batch path, one warp per pose — FK in fp64 (rows A2), the record out by a
//                bulk TMA store, the pose's list of non-empty 16x8 tiles with per-kind cull
//                masks (row A3); near-plane poses are queued for the exact pass
//   k_render_persist<NEAR, SUMS> : batch path renderer, persistent, PDL after k_fk_batch —
//                records + tile lists pulled into shared memory by 1-D TMA bulk copies,
//                per tile a TMA load of the observation, analytic ray casting of the tile's
//                primitives in packed fp32x2 (FFMA2), min depth, scoring, integer sums,
//                Eq. (4)-(5) per pose (rows A4, A5).  NEAR = true:
//                the second, normally empty launch for the queued poses (exact solids)
//   k_eval     : one CTA per (pose, split): FK on a 3-warp team, tiles culled on the fly,
//                split sums in global integer atomics; with pso_on it is the fused PSO
//                generation (update before FK, finalisation and bookkeeping in the grid's
//                last CTA; rows A7, A8).  Also the depth-image hooks (MODE = kModeDepth)
//   k_fk_debug : the same FK for the hp_debug_fk test hook.
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "fk.cuh"
#if HP_GEN_PROF
__device__ unsigned long long g_genprof[64][8];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define GENPROF_MIN(i) \
  if (a.pso_on && threadIdx.x == 0 && a.pso_k < 64) atomicMin(&g_genprof[a.pso_k][i], gtime());
#define GENPROF_MAX(i) \
  if (a.pso_on && threadIdx.x == 0 && a.pso_k < 64) atomicMax(&g_genprof[a.pso_k][i], gtime());
#define GENPROF_SET(i) \
  if (a.pso_on && threadIdx.x == 0 && a.pso_k < 64) g_genprof[a.pso_k][i] = gtime();
extern "C" int hp_debug_gen_prof(unsigned long long* out, int reset) {
  if (reset) {
    static unsigned long long init[64][8];
    for (int k = 0; k < 64; k++) {
      init[k][0] = ~0ull;
      for (int i = 1; i < 8; i++) init[k][i] = 0;
    }
    return (int)cudaMemcpyToSymbol(g_genprof, init, sizeof(init));
  }
  return (int)cudaMemcpyFromSymbol(out, g_genprof, sizeof(g_genprof));
}
#else
#define GENPROF_MIN(i)
#define GENPROF_MAX(i)
#define GENPROF_SET(i)
#endif
#include "pso.cuh"

// resident warps per SM the register budgets are sized for: 64 registers, 4 CTAs x 8 warps
// per SM (the renderer has no spills; k_eval's cost path spills 8 bytes, harmless)
#ifndef HP_MINB_WARPS
#define HP_MINB_WARPS 32
#endif
#ifndef HP_MINB_WARPS_EVAL
#define HP_MINB_WARPS_EVAL 32
#endif

namespace hp {

// ---------------------------------------------------------------------------------------
// Observation packing
// ---------------------------------------------------------------------------------------
__global__ void k_pack_obs(const float* __restrict__ depth, const uint8_t* __restrict__ mask,
                           uint32_t* __restrict__ obs, int W, int H, int pitch,
                           unsigned long long* S_o) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long npx = (long long)W * H;
  unsigned int cnt = 0;
  if (i < npx) {
    const int y = (int)(i / W), x = (int)(i % W);
    const float d = depth[i];
    const uint32_t bits = (d > 0.f && isfinite(d)) ? __float_as_uint(d) : kObsUndef;
    const uint32_t s = mask[i] ? 1u : 0u;
    obs[(long long)y * pitch + x] = bits | (s << 31);
    cnt = s;
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(S_o, (unsigned long long)cnt);
}

// ---------------------------------------------------------------------------------------
// Row f3 observation front end ("skin colour detection and depth segmentation";
// DESIGN AMB-33..36).  Integer mm throughout, so every decision is exact.
//   valid = d > 0;  band = [lo, hi] (mode 0) or [m, m + width] with m the nearest valid
//   (skin) depth (mode 1; none: empty band);  in_band = valid && lo <= d <= hi;
//   o_s = skin ? skin && (!valid || in_band) : in_band;
//   o_d = keep_background ? (valid ? d : 0) : (in_band ? d : 0).
// ---------------------------------------------------------------------------------------
__global__ void k_band_min(const uint16_t* __restrict__ depth, const uint8_t* __restrict__ skin,
                           int npx, unsigned int* m) {
  unsigned int best = 0xFFFFFFFFu;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npx; i += gridDim.x * blockDim.x) {
    const unsigned int d = depth[i];
    if (d > 0u && (skin == nullptr || skin[i] != 0)) best = min(best, d);
  }
  best = __reduce_min_sync(0xffffffffu, best);
  if ((threadIdx.x & 31) == 0 && best != 0xFFFFFFFFu) atomicMin(m, best);
}

__global__ void k_ingest(const uint16_t* __restrict__ depth, const uint8_t* __restrict__ skin,
                         int W, int H, int pitch, const SegD seg, const unsigned int* m,
                         uint32_t* __restrict__ obs, unsigned long long* S_o) {
  long long lo = seg.lo, hi = seg.hi;
  if (seg.mode == 1) {
    const unsigned int mm = *m;
    if (mm == 0xFFFFFFFFu) {
      lo = 1;
      hi = 0;
    } else {
      lo = mm;
      hi = (long long)mm + seg.width;
    }
  }
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned int cnt = 0;
  if (i < (long long)W * H) {
    const long long d = depth[i];
    const bool valid = d > 0, in_band = valid && lo <= d && d <= hi;
    const bool s = skin ? (skin[i] != 0 && (!valid || in_band)) : in_band;
    const bool def = seg.keep_background ? valid : in_band;
    const uint32_t bits = def ? __float_as_uint((float)d) : kObsUndef;
    const int y = (int)(i / W), x = (int)(i % W);
    obs[(long long)y * pitch + x] = bits | ((uint32_t)s << 31);
    cnt = s;
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(S_o, (unsigned long long)cnt);
}

__global__ void k_fill_undef(uint32_t* __restrict__ obs, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) obs[i] = kObsUndef;
}

__global__ void k_unpack_obs(const uint32_t* __restrict__ obs, int W, int H, int pitch,
                             float* __restrict__ depth, uint8_t* __restrict__ mask) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)W * H) return;
  const uint32_t w = obs[(i / W) * pitch + i % W];
  if (depth) depth[i] = (w & 0x7fffffffu) == kObsUndef ? 0.f : __uint_as_float(w & 0x7fffffffu);
  if (mask) mask[i] = (uint8_t)(w >> 31);
}

// Per-column / per-row ray directions, correctly rounded:
// d = ((u + 0.5 - cx)/fx, (v + 0.5 - cy)/fy, 1)  (P:L114 camera C).
// Layout: dx[W + kRayPad] then dy[H + kRayPad] (the pad covers tiles overhanging the image).
__global__ void k_ray_table(const CamParams cam, float* ray) {
  const int nx = ray_dx_len(cam.W), ny = cam.H + kRayPad;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const float nan = __int_as_float(0x7fc00000);
  if (i < nx) {
    ray[i] = i < cam.W ? __fdiv_rn((float)i + 0.5f - cam.cx, cam.fx) : nan;
  } else if (i < nx + 4 * ny) {
    const int y = (i - nx) / 4 + 2 * ((i - nx) % 4);  // dy4[y].q = dy(y + 2 q)
    ray[i] = y < cam.H ? __fdiv_rn((float)y + 0.5f - cam.cy, cam.fy) : nan;
  }
}

cudaError_t launch_ray_table(const CamParams& cam, float* ray, cudaStream_t st) {
  const int n = ray_floats(cam.W, cam.H);
  k_ray_table<<<(n + 255) / 256, 256, 0, st>>>(cam, ray);
  return cudaGetLastError();
}

__global__ void k_depth_to_mask(const float* __restrict__ depth, uint8_t* __restrict__ mask,
                                int npx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < npx) mask[i] = depth[i] > 0.f ? 1 : 0;
}

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
// sqrt of both halves (NaN where negative) and 1/x of both halves
__device__ __forceinline__ f2 sqrt2(f2 x) {
  float a, b;
  unpk(x, a, b);
  return mul2(x, pk(rsqrt_approx(a), rsqrt_approx(b)));
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
  int x0, y0, tx, ntiles;
  unsigned int magic;  // floor(2^32 / tx): t / tx = umulhi(t, magic) + {0, 1}
  __device__ __forceinline__ explicit TileGrid(int4 ub) {
    x0 = ub.x & ~3;
    y0 = ub.y;
    const int bw = ub.z - x0 + 1, bh = ub.w - ub.y + 1;
    tx = bw > 0 ? (bw + kTileW - 1) / kTileW : 0;
    const int ty = bh > 0 ? (bh + kTileH - 1) / kTileH : 0;
    ntiles = tx * ty;
    magic = tx > 1 ? 0xFFFFFFFFu / (unsigned)tx : 0u;
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

// BOTH: count the both-defined pixels (only the hp_eval_sums test hook reports them; the
// cost needs just the r_m and o_s AND r_m counts and the numerator)
template <int MODE, bool CHK, bool BOTH = true>
__device__ __forceinline__ void do_tile(const EvalArgs& a, const CUtensorMap* tmap,
                                        const FkOut& fo, int X0, int Y0, uint3 km,
                                        uint32_t* obs_buf, uint64_t* bar, uint32_t& phase,
                                        const float* s_dx, const float* s_dy, TileSums& acc,
                                        int yoff = 0) {
  const int lane = threadIdx.x & 31;
  const int col = lane & 15, rowb = lane >> 4;
  const float znear = a.cam.znear, zfar = a.cam.zfar;
  const float zinit = __uint_as_float(__float_as_uint(zfar) + 1u);  // next float above z_far
  if (MODE == kModeCost && a.use_tma) {
    // no proxy fence needed: the warp's reads of the previous tile in this buffer were
    // consumed before the __syncwarp that ended it (WAR across proxies is ordered)
    // rows past this frame's bottom come from the next frame (or TMA zero fill): they are
    // off-image, their rays are NaN and they are never scored
    HP_CHECK(yoff >= 0 && Y0 < a.cam.H);
    tma_load_2d_elect(obs_buf, a.use_tma == 2 ? a.tmap_g : tmap, X0, Y0 + yoff, bar,
                      kTileW * kTileH * 4);
  }
  const unsigned int msph = km.x, mcone = km.y, mell = km.z;
  Lane4 L;
  const int x = X0 + col;
  HP_CHECK(X0 >= 0 && x < ray_dx_len(a.cam.W) && Y0 >= 0 && Y0 + rowb < a.cam.H + kRayPad);
  HP_CHECK((X0 & 3) == 0);  // TMA boxes start 16-byte aligned
  L.dx = s_dx[x];
  const float ddx = fmaf(L.dx, L.dx, 1.f);
  const float4 dy4 = reinterpret_cast<const float4*>(s_dy)[Y0 + rowb];  // rows y, y+2, y+4, y+6
  const float dyv[4] = {dy4.x, dy4.y, dy4.z, dy4.w};
#pragma unroll
  for (int q = 0; q < kPxPerLane; q += 2) {
    const float dy0 = dyv[q], dy1 = dyv[q + 1];
    L.dy[q / 2] = pk(dy0, dy1);
    L.idd[q / 2] = pk(rcp_approx(fmaf(dy0, dy0, ddx)), rcp_approx(fmaf(dy1, dy1, ddx)));
    L.zb[q] = zinit;
    L.zb[q + 1] = zinit;
  }
  // CHK = false (the hot path): FK proved every primitive lies beyond z_near; CHK = true:
  // exact solid semantics near the camera (instantiated only out of line, see tiles_near)
  for (unsigned int m = msph; m; m &= m - 1) isect_sphere<CHK>(fo.rec[__ffs(m) - 1], L, znear);
  for (unsigned int m = mcone; m; m &= m - 1)
    isect_cone<CHK>(fo.rec[kCone0 + __ffs(m) - 1], L, znear);
  for (unsigned int m = mell; m; m &= m - 1)
    isect_ellipsoid<CHK>(fo.rec[kEll0 + __ffs(m) - 1], L, znear);

  if (MODE == kModeDepth) {
#pragma unroll
    for (int q = 0; q < kPxPerLane; q++) {
      const int y = Y0 + rowb + 2 * q;
      if (x < a.cam.W && y < a.cam.H)
        a.depth_out[(size_t)y * a.cam.W + x] = L.zb[q] <= zfar ? L.zb[q] : 0.f;
    }
  } else {
    if (a.use_tma) {
      mbar_wait(bar, phase);
      phase ^= 1u;
    } else {
#pragma unroll
      for (int q = 0; q < kPxPerLane; q++) {
        const int y = Y0 + rowb + 2 * q;
        obs_buf[(rowb + 2 * q) * kTileW + col] =
            (x < a.cam.W && y < a.cam.H) ? a.obs[(size_t)(y + yoff) * a.obs_pitch + x] : 0u;
      }
      __syncwarp();
    }
    const float d_m = a.cost.d_m, clampv = a.cost.clampv;
    const float qscale = a.cost.qscale, qmagic = a.cost.qmagic;
    bool any = false;
#pragma unroll
    for (int q = 0; q < kPxPerLane; q++) any |= L.zb[q] <= zfar;
    if (__any_sync(0xffffffffu, any)) {  // nothing rendered in this tile: nothing to score
      // numerator: round(min(|dd|, clamp) 2^qbits) from the bits of an fp32 magic-number
      // FFMA (exact: the sum lies in [2^23, 2^24], ulp 1), summed mod 2^32 and un-biased
      // once (the true per-lane sum is < 4 * 2^22); no float-to-int conversion on the XU
      unsigned int num = 0u - (unsigned)kPxPerLane * __float_as_uint(qmagic);
#pragma unroll
      for (int q = 0; q < kPxPerLane; q++) {
        const uint32_t w = obs_buf[(rowb + 2 * q) * kTileW + col];
        // o_d undefined is stored as NaN (kObsUndef), so diff is NaN exactly there
        const float diff = fabsf(__uint_as_float(w & 0x7fffffffu) - L.zb[q]);
        // off-image pixels have NaN rays and never hit (k_ray_table)
        const bool hit = L.zb[q] <= zfar;
        // r_m = 1 where |r_d - o_d| < d_m or o_d undefined (AMB-4, AMB-5):
        // !(diff >= d_m) is true for NaN
        const unsigned int rm = hit & !(diff >= d_m);
        const bool both = hit & (diff == diff);
        acc.rm += rm;
        acc.and_ += rm & (w >> 31);
        if (BOTH) acc.both += both;
        num += __float_as_uint(fmaf(both ? fminf(diff, clampv) : 0.f, qscale, qmagic));
      }
      acc.num += num;
    }
  }
  __syncwarp();
}

// A warp's share of one particle's tiles.  Tiles come from the FK kernel's list
// (nlist >= 0) or, when there is none, from the union grid with per-tile culling; the
// warps of a CTA take them through the shared counter *next.
struct TileRun {
  TileSums acc;
  uint32_t phase;
};
template <int MODE, bool CHK>
__device__ __forceinline__ TileRun tile_loop(const EvalArgs& a, const CUtensorMap* tmap,
                                             const FkOut& fo, const uint4* list, int nlist,
                                             int first, int stride, int count, int* next,
                                             uint32_t* obs_buf, uint64_t* bar, uint32_t phase,
                                             const float* s_dx, const float* s_dy, int yoff) {
  const int lane = threadIdx.x & 31;
  const TileGrid g(fo.ubox);
  TileRun r;
  r.phase = phase;
  int j = 0;
  if (lane == 0) j = atomicAdd(next, 1);
  j = __shfl_sync(0xffffffffu, j, 0);
  while (j < count) {
    int jn = 0;
    if (lane == 0) jn = atomicAdd(next, 1);  // the next tile, fetched early
    int X0, Y0;
    uint3 km;
    if (nlist >= 0) {
      const uint4 it = list[j];
      X0 = (int)(it.x & 0xFFFFu);
      Y0 = (int)(it.x >> 16);
      km = make_uint3(it.y, it.z, it.w);
    } else {
      g.origin(first + j * stride, X0, Y0);
      km = cull_tile(fo, X0, Y0);
    }
    if (km.x | km.y | km.z)  // no primitive box touches the tile: nothing to render or score
      do_tile<MODE, CHK>(a, tmap, fo, X0, Y0, km, obs_buf, bar, r.phase, s_dx, s_dy, r.acc,
                         yoff);
    j = __shfl_sync(0xffffffffu, jn, 0);
  }
  return r;
}

// Particles with a primitive that may cross z_near (rare: a hand within ~25 cm of the near
// plane) take the exact-solid path out of line, so its registers never weigh on the hot
// loop's allocation.  The kernels' EvalArgs are __grid_constant__: no copy for the reference.
template <int MODE>
__device__ __noinline__ TileRun tiles_near(const EvalArgs& a, const CUtensorMap* tmap,
                                           const FkOut& fo, const uint4* list, int nlist,
                                           int first, int stride, int count, int* next,
                                           uint32_t* obs_buf, uint64_t* bar, uint32_t phase,
                                           const float* s_dx, const float* s_dy, int yoff) {
  return tile_loop<MODE, true>(a, tmap, fo, list, nlist, first, stride, count, next, obs_buf,
                               bar, phase, s_dx, s_dy, yoff);
}

// NEARCODE = false (the speculative fit kernels): no near-plane code at all; a particle
// that would need it raises a_.near_seen and the host re-runs the fit with NEARCODE = true.
template <int MODE, bool NEARCODE = true>
__device__ __forceinline__ TileRun run_tiles(const EvalArgs& a, const CUtensorMap* tmap,
                                             const FkOut& fo, const uint4* list, int nlist,
                                             int first, int stride, int count, int* next,
                                             uint32_t* obs_buf, uint64_t* bar, uint32_t phase,
                                             const float* s_dx, const float* s_dy, int yoff) {
#if HP_NEAR_TEST
  return tile_loop<MODE, false>(a, tmap, fo, list, nlist, first, stride, count, next,
                                obs_buf, bar, phase, s_dx, s_dy, yoff);
#else
  if (!NEARCODE) {
    if (!fo.near_ok && threadIdx.x == 0 && a.near_seen) atomicOr(a.near_seen, 1);
    return tile_loop<MODE, false>(a, tmap, fo, list, nlist, first, stride, count, next,
                                  obs_buf, bar, phase, s_dx, s_dy, yoff);
  }
  if (fo.near_ok)
    return tile_loop<MODE, false>(a, tmap, fo, list, nlist, first, stride, count, next,
                                  obs_buf, bar, phase, s_dx, s_dy, yoff);
  return tiles_near<MODE>(a, tmap, fo, list, nlist, first, stride, count, next, obs_buf, bar,
                          phase, s_dx, s_dy, yoff);
#endif
}

__device__ __forceinline__ void warp_reduce(TileSums& s) {
  s.rm = __reduce_add_sync(0xffffffffu, s.rm);
  s.and_ = __reduce_add_sync(0xffffffffu, s.and_);
  s.both = __reduce_add_sync(0xffffffffu, s.both);
#pragma unroll
  for (int off = 16; off; off >>= 1) s.num += __shfl_xor_sync(0xffffffffu, s.num, off);
}

// Eq. (4)-(5) in fp64 from the integer sums v = (sum r_m, sum o_s AND r_m, numerator in
// 2^-qbits mm, both-defined count)  (AMB-1, -2, -3, -6).
__device__ __forceinline__ double finalize_cost(const EvalArgs& a, int p,
                                                const unsigned long long v[4], double kc) {
  const long long s_rm = (long long)v[0], s_and = (long long)v[1];
  const long long s_or = (long long)a.S_o[frame_of(a, p)] + s_rm - s_and;
  double D = 0.0;
  if (s_or > 0) {
    const double num = ldexp((double)v[2], -a.cost.qbits);
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

// ---------------------------------------------------------------------------------------
// k_eval: one CTA per (particle, split).  Warp 0 runs FK into shared memory while the other
// warps stage the ray table; then all warps take tiles dynamically.  Used for small swarms
// (S > 1 splits per particle keep every SM busy) and for the depth-image hooks.
// ---------------------------------------------------------------------------------------
#ifndef HP_EVAL_FK_TEAM
#define HP_EVAL_FK_TEAM 3  // k_eval's FK team: warps 0..2 (one primitive kind per warp)
#endif
constexpr int kEvalFkTeam = HP_EVAL_FK_TEAM;
template <int NW, typename PoseT, int MODE, bool NEARCODE = true>
__global__ void __launch_bounds__(NW * 32, HP_MINB_WARPS_EVAL / NW)
    k_eval(const __grid_constant__ EvalArgs a, const __grid_constant__ CUtensorMap tmap) {
  __shared__ FkScratch s_fk;
  __shared__ __align__(16) FkOut s_out;
  __shared__ __align__(128) uint32_t s_obs[NW][kTileW * kTileH];
  __shared__ __align__(8) uint64_t s_bar[NW];
  __shared__ unsigned long long s_red[NW][4];
  __shared__ int s_next;
  extern __shared__ float s_ray[];  // dx per column [W + pad], dy per row [H + pad]

  if (a.pdl) {
    // programmatic dependent launch (PSO generations): let the next generation's CTAs be
    // scheduled now, then wait until the previous generation's results are visible
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  GENPROF_MIN(0)
  if (a.done && *a.done) return;  // PSO stop rule reached (grid-uniform)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = blockIdx.x / a.S, sidx = blockIdx.x % a.S;
  const float* s_dx = s_ray;
  const float* s_dy = s_ray + ray_dx_len(a.cam.W);

  if (warp < kEvalFkTeam) {
    // FK on warps 0..kEvalFkTeam-1 (the records of each primitive kind on their own warp)
    __shared__ double s_pose[32];
    if (a.pso_on && a.pso_k >= 1) {
      // fused PSO update (Eq. 6-7, row A8) of this particle; every CTA of the particle
      // computes the same bits, split 0 stores them (double-buffered X, V)
      if (warp == 0)
        pso_update_warp(a.pso, p, a.pso_k, a.x_in, a.v_in, a.x_out, a.v_out, sidx == 0, s_pose,
                        /*deferred=*/true);
      __syncwarp();
      fk_team<double, kEvalFkTeam>(s_pose, a.dims, a.cam, a.cost.kc_rest, s_fk, s_out);
    } else {
      const PoseT* pose = static_cast<const PoseT*>(a.poses) + (size_t)p * kNdof;
      fk_team<PoseT, kEvalFkTeam>(pose, a.dims, a.cam, a.cost.kc_rest, s_fk, s_out);
    }
  } else {
    // while the FK team runs: stage the per-column / per-row ray directions (k_ray_table)
    const int n4 = ray_floats(a.cam.W, a.cam.H) / 4;
    for (int i = threadIdx.x - 32 * kEvalFkTeam; i < n4; i += (NW - kEvalFkTeam) * 32)
      reinterpret_cast<float4*>(s_ray)[i] = __ldg(reinterpret_cast<const float4*>(a.ray) + i);
    if (MODE == kModeCost && warp == NW - 1 && lane == 0) {
      for (int w = 0; w < NW; w++) mbar_init(&s_bar[w], 1);  // count 1: the expect_tx arrival
      fence_mbar_init();
      if (a.use_tma == 1) prefetch_tmap(&tmap);
    }
    if (threadIdx.x == 32 * kEvalFkTeam) s_next = 0;
  }
  __syncthreads();

  GENPROF_MAX(1)
  const TileGrid g(s_out.ubox);
  // this CTA owns tiles sidx, sidx + S, ...; warps take them dynamically (load balance)
  const int nmine = g.ntiles > sidx ? (g.ntiles - sidx + a.S - 1) / a.S : 0;
  TileSums acc = run_tiles<MODE, NEARCODE>(a, &tmap, s_out, nullptr, -1, sidx, a.S, nmine,
                                           &s_next, s_obs[warp], &s_bar[warp], 0u, s_dx, s_dy,
                                           frame_of(a, p) * a.cam.H)
                     .acc;

  GENPROF_MAX(2)
  if (MODE != kModeCost) return;
  // ---- reduction: warp shuffles, one atomic per sum per CTA ----
  warp_reduce(acc);
  if (lane == 0) {
    s_red[warp][0] = acc.rm;
    s_red[warp][1] = acc.and_;
    s_red[warp][2] = acc.num;
    s_red[warp][3] = acc.both;
  }
  __syncthreads();
  unsigned long long* gacc = a.acc + (size_t)p * 4;
  if (a.pso_on) {
    // ---- fused PSO generation: the CTAs only add their sums; the grid's last CTA
    // finalises every particle (Eq. 4-5) and runs the bookkeeping (row A7), so no CTA
    // waits on a per-particle counter round trip ----
    __shared__ int s_lastcta;
    if (threadIdx.x == 0) {
      unsigned long long v[4] = {0, 0, 0, 0};
      for (int w = 0; w < NW; w++)
        for (int k = 0; k < 4; k++) v[k] += s_red[w][k];
      for (int k = 0; k < 4; k++)
        if (v[k]) atomicAdd(gacc + k, v[k]);
      if (sidx == 0) a.kc_g[p] = s_out.kc;
      // one acq_rel arrival: releases this CTA's sums, and the last CTA acquires everyone's
      unsigned prev;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                   : "=r"(prev) : "l"(a.gcount) : "memory");
      s_lastcta = prev == gridDim.x - 1;
      if (s_lastcta) *a.gcount = 0;
    }
    __syncthreads();
    if (!s_lastcta) return;
    GENPROF_SET(3)
    // one pass per particle: Eq. (4)-(5), pbest (strict <, NaN = +inf) and the argmin;
    // pbest / gbest positions are left to the next generation's update (deferred)
    const PsoDev& ps = a.pso;
    const int N = ps.N, k = a.pso_k;
    const double stop = ps.dyn->stop;
    // the ray table is dead now: its shared memory holds the pbest costs when they fit
    const bool in_smem = (size_t)N * sizeof(double) <=
                         (size_t)ray_floats(a.cam.W, a.cam.H) * sizeof(float);
    double* pcs = in_smem ? reinterpret_cast<double*>(s_ray) : ps.Pc;
    __syncthreads();  // every warp is past its last ray-table read
    double bv = INFINITY;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      unsigned long long v[4];
      for (int q = 0; q < 4; q++) {
        v[q] = __ldcg(a.acc + (size_t)i * 4 + q);
        a.acc[(size_t)i * 4 + q] = 0ull;  // zero for the next generation
      }
      const double pc_old = __ldcg(ps.Pc + i);
      double e = finalize_cost(a, i, v, __ldcg(a.kc_g + i));  // also stores costs64 = E
      if (isnan(e)) e = INFINITY;
      const bool imp = k == 0 || e < pc_old;
      const double pc = imp ? e : pc_old;
      if (imp) ps.Pc[i] = e;
      if (in_smem) pcs[i] = pc;
      ps.pimp[i] = imp;
      if (pc < bv) {  // i ascending per thread: the lowest index wins ties
        bv = pc;
        bi = i;
      }
    }
    pso_book_tail(ps, k, a.pso_k >= 1 ? a.x_out : ps.X, pcs, bv, bi, stop);
    GENPROF_SET(4)
    return;
  }
  if (threadIdx.x == 0) {
    unsigned long long v[4] = {0, 0, 0, 0};
    for (int w = 0; w < NW; w++)
      for (int k = 0; k < 4; k++) v[k] += s_red[w][k];
    int last = 1;
    if (a.S > 1) {
      for (int k = 0; k < 4; k++)
        if (v[k]) atomicAdd(gacc + k, v[k]);
      __threadfence();
      last = atomicAdd(a.counters + p, 1u) == (unsigned)(a.S - 1);
      if (last) {
        __threadfence();
        for (int k = 0; k < 4; k++) v[k] = atomicExch(gacc + k, 0ull);  // read + reset
        a.counters[p] = 0;
      }
    }
    if (last) finalize_cost(a, p, v, s_out.kc);
  }
}

__global__ void k_fk_debug(const double* pose, const DimsD dims, const CamParams cam,
                           float* rec, int* boxes, double* joints, double* kc) {
  __shared__ FkScratch s;
  __shared__ __align__(16) FkOut o;
  fk_warp<double>(pose, dims, cam, 0.0, s, o);
  for (int j = threadIdx.x; j < kNprim; j += 32) {
    if (rec)
      for (int i = 0; i < kRec; i++) rec[j * kRec + i] = o.rec[j][i];
    if (boxes) {
      boxes[j * 4 + 0] = o.box[j].x;
      boxes[j * 4 + 1] = o.box[j].y;
      boxes[j * 4 + 2] = o.box[j].z;
      boxes[j * 4 + 3] = o.box[j].w;
    }
  }
  if (joints)
    for (int i = threadIdx.x; i < 60; i += 32) joints[i] = (&s.J[0][0][0])[i];
  if (kc && threadIdx.x == 0) *kc = o.kc;
}

// ---------------------------------------------------------------------------------------
// Two-kernel batch path for large swarms.
//   k_fk_batch      : one warp per particle — FK (fp64) and the particle's non-empty tile
//                     list with cull masks, written to global memory (L2-resident).
//   k_render_persist: persistent CTAs, ALL warps render.  Per particle one thread pulls the
//                     FK record and tile list into shared memory with 1-D TMA bulk copies
//                     (double-buffered: particle i + 2 is fetched as soon as particle i is
//                     finished, while i + 1 renders), so no warp ever waits on FK latency.
// ---------------------------------------------------------------------------------------
// A tile (qx, qy) overlaps primitive j iff column qx's x-range and row qy's y-range both
// overlap box j — the same four compares as cull_tile — so the tile masks are the AND of
// per-column and per-row 38-bit masks (tx + ty sets of 38 tests instead of tx * ty).
constexpr int kMaxBand = 64;  // columns / rows of the per-warp band masks
__device__ __forceinline__ int build_tile_list(const FkOut& fo, uint4* out, uint2* s_cm,
                                               uint2* s_rm) {
  const int lane = threadIdx.x & 31;
  const TileGrid g(fo.ubox);
  if (g.ntiles > kMaxTiles || g.tx > kMaxBand) return -1;  // the renderer culls per tile
  const int ty = g.tx > 0 ? g.ntiles / g.tx : 0;
  if (ty > kMaxBand) return -1;
  for (int q = lane; q < g.tx + ty; q += 32) {
    const bool col = q < g.tx;
    const int lo = col ? g.x0 + q * kTileW : g.y0 + (q - g.tx) * kTileH;
    const int hi = lo + (col ? kTileW : kTileH) - 1;
    // box j as (lo, hi) pairs along this axis: ints 0, 2 (x) or 1, 3 (y) of fo.box[j]
    const int* bx = reinterpret_cast<const int*>(fo.box) + (col ? 0 : 1);
    unsigned int m0 = 0, m1 = 0;
#pragma unroll 8
    for (int jj = 0; jj < 32; jj++)
      m0 |= (unsigned)(bx[4 * jj] <= hi && bx[4 * jj + 2] >= lo) << jj;
#pragma unroll
    for (int jj = 32; jj < kNprim; jj++)
      m1 |= (unsigned)(bx[4 * jj] <= hi && bx[4 * jj + 2] >= lo) << (jj - 32);
    HP_CHECK(q < g.tx + ty && q < 2 * kMaxBand);
    if (col) s_cm[q] = make_uint2(m0, m1);
    else s_rm[q - g.tx] = make_uint2(m0, m1);
  }
  __syncwarp();
  int cnt = 0;
  for (int base = 0; base < g.ntiles; base += 32) {  // one tile per lane
    const int t = base + lane;
    unsigned int lo = 0, hi = 0;
    int X0 = 0, Y0 = 0;
    if (t < g.ntiles) {
      g.origin(t, X0, Y0);
      HP_CHECK((X0 - g.x0) / kTileW < kMaxBand && (Y0 - g.y0) / kTileH < kMaxBand);
      const uint2 c = s_cm[(X0 - g.x0) / kTileW], r = s_rm[(Y0 - g.y0) / kTileH];
      lo = c.x & r.x;
      hi = c.y & r.y;
    }
    const unsigned int m0 = lo & 0xFFFFFu, m1 = (lo >> 20) | ((hi & 0x7u) << 12), m2 = hi >> 3;
    const bool ne = (lo | hi) != 0;
    const unsigned int bal = __ballot_sync(0xffffffffu, ne);
    if (ne) {
      HP_CHECK(cnt + __popc(bal & ((1u << lane) - 1u)) < kMaxTiles);
      out[cnt + __popc(bal & ((1u << lane) - 1u))] =
          make_uint4((unsigned)X0 | ((unsigned)Y0 << 16), m0, m1, m2);
    }
    cnt += __popc(bal);
  }
  return cnt;
}

#ifndef HP_FK_PDL
#define HP_FK_PDL 1  // programmatic dependent launch of k_render_persist after k_fk_batch
#endif
#ifndef HP_FK_WARPS
#define HP_FK_WARPS 4  // particles (warps) per k_fk_batch CTA
#endif
constexpr int kFkWarps = HP_FK_WARPS;
template <typename PoseT>
__global__ void __launch_bounds__(kFkWarps * 32, 32 / kFkWarps)
    k_fk_batch(const EvalArgs a) {
  __shared__ FkScratch s_fk[kFkWarps];
  __shared__ __align__(16) FkOut s_out[kFkWarps];
  static_assert(sizeof(FkScratch) >= 2 * kMaxBand * sizeof(uint2), "band masks alias s_fk");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if HP_FK_PDL
  // the renderer (launched with programmatic stream serialisation) may start its prologue
  // on SMs this grid frees; it waits for this grid's completion before reading its output
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  const int p = blockIdx.x * kFkWarps + warp;  // one warp per particle
  if (p >= a.n) return;  // warp-uniform; only warp-local synchronisation below
  const PoseT* pose = static_cast<const PoseT*>(a.poses) + (size_t)p * kNdof;
  fk_team<PoseT, 1>(pose, a.dims, a.cam, a.cost.kc_rest, s_fk[warp], s_out[warp]);
  // the record leaves by one bulk copy while the warp builds the tile list: every lane
  // orders its record writes before the async proxy, then lane 0 issues the copy
  fence_proxy_async();
  __syncwarp();
  if (lane == 0)
    bulk_s2g(static_cast<FkOut*>(a.fk_g) + p, &s_out[warp], (uint32_t)sizeof(FkOut));
  FKPROF(4)
  uint2* band = reinterpret_cast<uint2*>(&s_fk[warp]);  // FK scratch is dead by now
  const int cnt = build_tile_list(s_out[warp], a.tiles_g + (size_t)p * kMaxTiles, band,
                                  band + kMaxBand);
  FKPROF(5)
  if (lane == 0) {
    int ntl = cnt;
    if (!s_out[warp].near_ok) {  // some primitive may cross z_near: the exact pass renders it
      const unsigned slot_ = atomicAdd(a.near_count, 1u);
      HP_CHECK(slot_ < (unsigned)a.n);
      a.near_list[slot_] = p;
      ntl = -2;
    }
    a.ntl_g[p] = ntl;
    bulk_wait_all();  // the record copy completes before the CTA's shared memory retires
  }
  FKPROF(6)
}

// NEAR = false: the batch renderer.  Particles whose FK found a primitive that may cross
// z_near were queued by k_fk_batch (ntl = -2) and are skipped here; NEAR = true renders
// exactly those (exact-solid path) in a second, normally empty launch, so the
// near-plane code never shares a register allocation with the hot loop.
template <int NW, bool NEAR, bool SUMS>
__global__ void __launch_bounds__(NW * 32, HP_MINB_WARPS / NW)
    k_render_persist(const __grid_constant__ EvalArgs a,
                     const __grid_constant__ CUtensorMap tmap) {
  __shared__ __align__(16) FkOut s_out[2];
  __shared__ __align__(16) uint4 s_tiles[2][NEAR ? 1 : kMaxTiles];
  __shared__ __align__(128) uint32_t s_obs[NW][kTileW * kTileH];
  __shared__ __align__(8) uint64_t s_bar[NW];
  __shared__ __align__(8) uint64_t s_full[2];
  __shared__ unsigned long long s_acc[2][4];
  __shared__ int s_next[2], s_done[2], s_pid[2], s_ntl[2];
  extern __shared__ float s_ray[];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* s_dx = s_ray;
  const float* s_dy = s_ray + ray_dx_len(a.cam.W);
  unsigned int* const counter = a.pcount + (NEAR ? 2 : 0);  // [taken, CTAs exited]
  // one thread: take the next particle and pull its FK record + tile list into slot b
  auto issue = [&](int b) {
    int p = a.n;
    if (NEAR) {
      const unsigned k = atomicAdd(counter, 1u);
      if (k < __ldcg(a.near_count)) p = __ldcg(a.near_list + k);
    } else {
      p = (int)atomicAdd(counter, 1u);
    }
    s_pid[b] = p;
    if (p < a.n) {
      const int ntl = NEAR ? -1 : __ldcg(a.ntl_g + p);  // NEAR: cull every tile
      s_ntl[b] = ntl;
      if (ntl == -2) {  // queued for the near-plane pass: nothing to fetch
        mbar_arrive(&s_full[b]);
        return;
      }
      const uint32_t lb = ntl > 0 ? (uint32_t)ntl * 16u : 0u;
      mbar_expect_tx(&s_full[b], (uint32_t)sizeof(FkOut) + lb);
      bulk_g2s(&s_out[b], static_cast<const FkOut*>(a.fk_g) + p, (uint32_t)sizeof(FkOut),
               &s_full[b]);
      if (lb) bulk_g2s(s_tiles[b], a.tiles_g + (size_t)p * kMaxTiles, lb, &s_full[b]);
    } else {
      mbar_arrive(&s_full[b]);  // terminator: complete the phase without data
    }
  };
#if HP_FK_PDL
  // the near-plane pass may start its prologue as this grid's CTAs retire
  if (!NEAR) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  if (NEAR) {  // usually nothing was queued: leave before any set-up work
    __shared__ int s_any;
    if (threadIdx.x == 0) {
#if HP_FK_PDL
      asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
      s_any = __ldcg(a.near_count) > 0u;
    }
    __syncthreads();
    if (!s_any) return;  // the same for every CTA: no counter to reset
  }
  if (threadIdx.x == 0) {
    for (int w = 0; w < NW; w++) mbar_init(&s_bar[w], 1);
    for (int b = 0; b < 2; b++) {
      mbar_init(&s_full[b], 1);
      s_next[b] = 0;
      s_done[b] = 0;
      for (int k = 0; k < 4; k++) s_acc[b][k] = 0;
    }
    fence_mbar_init();
    if (a.use_tma == 1) prefetch_tmap(&tmap);
#if HP_FK_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous grid is complete
#endif
    issue(0);
    issue(1);
  }
  {
    const int n4 = ray_floats(a.cam.W, a.cam.H) / 4;
    for (int i = threadIdx.x; i < n4; i += NW * 32)
      reinterpret_cast<float4*>(s_ray)[i] = __ldg(reinterpret_cast<const float4*>(a.ray) + i);
  }
  __syncthreads();

  uint32_t phase = 0;
  for (int i = 0;; i++) {
    const int b = i & 1;
    mbar_wait(&s_full[b], (i >> 1) & 1);
    const int p = s_pid[b];
    if (p >= a.n) break;
    const FkOut& fo = s_out[b];
    const int nlist = s_ntl[b];
    const int yoff = frame_of(a, p) * a.cam.H;
    TileSums acc;
    if (nlist != -2) {
      const TileGrid g(fo.ubox);
      const int nt = nlist >= 0 ? nlist : g.ntiles;
      int t = 0;
      if (lane == 0) t = atomicAdd(&s_next[b], 1);
      t = __shfl_sync(0xffffffffu, t, 0);
      while (t < nt) {
        int tn = 0;
        if (lane == 0) tn = atomicAdd(&s_next[b], 1);
        int X0, Y0;
        uint3 km;
        if (nlist >= 0) {
          HP_CHECK(t >= 0 && t < kMaxTiles);
          const uint4 it = s_tiles[b][t];
          X0 = (int)(it.x & 0xFFFFu);
          Y0 = (int)(it.x >> 16);
          km = make_uint3(it.y, it.z, it.w);
        } else {
          g.origin(t, X0, Y0);
          km = cull_tile(fo, X0, Y0);
        }
        if (km.x | km.y | km.z)
          do_tile<kModeCost, NEAR, SUMS>(a, &tmap, fo, X0, Y0, km, s_obs[warp], &s_bar[warp],
                                         phase, s_dx, s_dy, acc, yoff);
        t = __shfl_sync(0xffffffffu, tn, 0);
      }
    }
    warp_reduce(acc);
    if (lane == 0) {
      if (acc.rm) atomicAdd(&s_acc[b][0], (unsigned long long)acc.rm);
      if (acc.and_) atomicAdd(&s_acc[b][1], (unsigned long long)acc.and_);
      if (acc.num) atomicAdd(&s_acc[b][2], acc.num);
      if (acc.both) atomicAdd(&s_acc[b][3], (unsigned long long)acc.both);
      __threadfence_block();
      if (atomicAdd(&s_done[b], 1) == NW - 1) {  // last warp for this particle
        __threadfence_block();
        unsigned long long v[4];
        for (int k = 0; k < 4; k++) {
          v[k] = s_acc[b][k];
          s_acc[b][k] = 0;
        }
        if (nlist != -2) finalize_cost(a, p, v, fo.kc);  // queued ones: the near pass
        s_next[b] = 0;
        s_done[b] = 0;
        fence_proxy_async();  // every warp's generic reads of slot b precede the refill
        issue(b);             // particle i + 2 into the freed slot
      }
    }
    __syncwarp();
  }
  // the last CTA to leave resets the counters for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(counter + 1, 1u) == gridDim.x - 1) {
      counter[0] = 0;
      counter[1] = 0;
      if (NEAR) *a.near_count = 0;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------------------
#ifndef HP_NW
#define HP_NW 8
#endif
constexpr int kEvalWarps = HP_NW;
#ifndef HP_RENDER_NW
#define HP_RENDER_NW 16  // warps per k_render_persist CTA (2 CTAs per SM at 64 registers)
#endif
constexpr int kRenderWarps = HP_RENDER_NW;

// Prefer the maximum shared-memory carveout (the default 64 KB split would cap the
// persistent kernel, 37 KB of shared memory per CTA, at one CTA per SM).
// Prefer the maximum shared-memory carveout and allow dynamic shared memory (the ray
// table) beyond the default 48 KB for large images (hp_create caps it at kMaxRayBytes).
static void set_carveouts() {
  static bool done = false;
  if (done) return;
  done = true;
  const int pct = cudaSharedmemCarveoutMaxShared;
  auto cfg = [&](auto f) {
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxRayBytes);
  };
  cfg(k_render_persist<kRenderWarps, false, false>);
  cfg(k_render_persist<kRenderWarps, true, false>);
  cfg(k_render_persist<kRenderWarps, false, true>);
  cfg(k_render_persist<kRenderWarps, true, true>);
  cfg(k_eval<kEvalWarps, float, kModeCost>);
  cfg(k_eval<kEvalWarps, double, kModeCost>);
  cfg(k_eval<kEvalWarps, double, kModeCost, false>);
  cfg(k_eval<kEvalWarps, float, kModeDepth>);
  cfg(k_eval<kEvalWarps, double, kModeDepth>);
}

size_t fk_record_bytes() { return sizeof(FkOut); }

int eval_blocks_per_sm(const CamParams& cam) {
  set_carveouts();
  int nb = 0;
  const size_t dyn = (size_t)ray_floats(cam.W, cam.H) * sizeof(float);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &nb, k_eval<kEvalWarps, double, kModeCost>, kEvalWarps * 32, dyn) != cudaSuccess)
    return 0;
  return nb;
}

int persist_blocks_per_sm(const CamParams& cam) {
  set_carveouts();
  int nb = 0;
  const size_t dyn = (size_t)ray_floats(cam.W, cam.H) * sizeof(float);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb,
                                                    k_render_persist<kRenderWarps, false, false>,
                                                    kRenderWarps * 32, dyn) != cudaSuccess)
    return 0;
  return nb;
}

cudaError_t launch_pack_obs(const float* depth, const uint8_t* mask, uint32_t* obs, int W,
                            int H, int pitch_words, unsigned long long* S_o, cudaStream_t st) {
  const long long npx = (long long)W * H;
  const int threads = 256;
  const long long blocks = (npx + threads - 1) / threads;
  k_pack_obs<<<(unsigned)blocks, threads, 0, st>>>(depth, mask, obs, W, H, pitch_words, S_o);
  return cudaGetLastError();
}

cudaError_t launch_band_min(const uint16_t* depth, const uint8_t* skin, int npx, unsigned int* m,
                            cudaStream_t st) {
  const int threads = 256, blocks = std::min((npx + threads - 1) / threads, 1184);
  if (blocks > 0) k_band_min<<<blocks, threads, 0, st>>>(depth, skin, npx, m);
  return cudaGetLastError();
}

cudaError_t launch_ingest(const uint16_t* depth, const uint8_t* skin, int W, int H,
                          int pitch_words, const SegD& seg, const unsigned int* m, uint32_t* obs,
                          unsigned long long* S_o, cudaStream_t st) {
  const long long npx = (long long)W * H;
  k_ingest<<<(unsigned)((npx + 255) / 256), 256, 0, st>>>(depth, skin, W, H, pitch_words, seg,
                                                           m, obs, S_o);
  return cudaGetLastError();
}

cudaError_t launch_fill_undef(uint32_t* obs, long long words, cudaStream_t st) {
  if (words > 0) k_fill_undef<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(obs, words);
  return cudaGetLastError();
}

cudaError_t launch_unpack_obs(const uint32_t* obs, int W, int H, int pitch_words, float* depth,
                              uint8_t* mask, cudaStream_t st) {
  const long long npx = (long long)W * H;
  k_unpack_obs<<<(unsigned)((npx + 255) / 256), 256, 0, st>>>(obs, W, H, pitch_words, depth,
                                                               mask);
  return cudaGetLastError();
}

cudaError_t launch_depth_to_mask(const float* depth, uint8_t* mask, int npx, cudaStream_t st) {
  k_depth_to_mask<<<(npx + 255) / 256, 256, 0, st>>>(depth, mask, npx);
  return cudaGetLastError();
}

cudaError_t launch_eval(const EvalArgs& a, bool pose_double, int mode, const CUtensorMap* map,
                        cudaStream_t st, cudaEvent_t* tev) {
  const long long blocks = (long long)a.n * a.S;
  if (blocks == 0) return cudaSuccess;
  const bool two = mode == kModeCost && a.S == 1 && a.persist_grid > 0;
  if (tev) {
    cudaEventRecord(tev[0], st);
    if (!two) cudaEventRecord(tev[1], st);  // single-launch paths: empty first interval
  }
  const dim3 grid((unsigned)blocks), block(kEvalWarps * 32);
  const size_t dyn = (size_t)ray_floats(a.cam.W, a.cam.H) * sizeof(float);
  if (two) {
    const dim3 rblock(kRenderWarps * 32);
    const dim3 fgrid((unsigned)((a.n + kFkWarps - 1) / kFkWarps));
    if (pose_double) k_fk_batch<double><<<fgrid, kFkWarps * 32, 0, st>>>(a);
    else k_fk_batch<float><<<fgrid, kFkWarps * 32, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (tev) cudaEventRecord(tev[1], st);
    const dim3 pgrid((unsigned)(a.persist_grid < a.n ? a.persist_grid : a.n));
#if HP_FK_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = pgrid;
    cfg.blockDim = rblock;
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const bool sums = a.sums_out != nullptr;
    e = sums ? cudaLaunchKernelEx(&cfg, k_render_persist<kRenderWarps, false, true>, a, *map)
             : cudaLaunchKernelEx(&cfg, k_render_persist<kRenderWarps, false, false>, a, *map);
    if (e != cudaSuccess) return e;
    // the near-plane pass (exits at once when k_fk_batch queued nothing)
    cfg.gridDim = dim3((unsigned)(pgrid.x < 148u ? pgrid.x : 148u));
    e = sums ? cudaLaunchKernelEx(&cfg, k_render_persist<kRenderWarps, true, true>, a, *map)
             : cudaLaunchKernelEx(&cfg, k_render_persist<kRenderWarps, true, false>, a, *map);
    if (e != cudaSuccess) return e;
#else
    if (a.sums_out) {
      k_render_persist<kRenderWarps, false, true><<<pgrid, rblock, dyn, st>>>(a, *map);
      k_render_persist<kRenderWarps, true, true><<<dim3(pgrid.x < 148u ? pgrid.x : 148u), rblock,
                                                 dyn, st>>>(a, *map);
    } else {
      k_render_persist<kRenderWarps, false, false><<<pgrid, rblock, dyn, st>>>(a, *map);
      k_render_persist<kRenderWarps, true, false><<<dim3(pgrid.x < 148u ? pgrid.x : 148u), rblock,
                                                  dyn, st>>>(a, *map);
    }
#endif
    if (tev) cudaEventRecord(tev[2], st);
    return cudaGetLastError();
  } else if (mode == kModeCost && a.pdl && pose_double) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e =
        a.near_seen ? cudaLaunchKernelEx(&cfg, k_eval<kEvalWarps, double, kModeCost, false>, a,
                                         *map)
                    : cudaLaunchKernelEx(&cfg, k_eval<kEvalWarps, double, kModeCost>, a, *map);
    if (tev) cudaEventRecord(tev[2], st);
    return e;
  } else if (mode == kModeCost) {
    if (pose_double && a.near_seen)
      k_eval<kEvalWarps, double, kModeCost, false><<<grid, block, dyn, st>>>(a, *map);
    else if (pose_double)
      k_eval<kEvalWarps, double, kModeCost><<<grid, block, dyn, st>>>(a, *map);
    else
      k_eval<kEvalWarps, float, kModeCost><<<grid, block, dyn, st>>>(a, *map);
  } else {
    if (pose_double)
      k_eval<kEvalWarps, double, kModeDepth><<<grid, block, dyn, st>>>(a, *map);
    else
      k_eval<kEvalWarps, float, kModeDepth><<<grid, block, dyn, st>>>(a, *map);
  }
  if (tev) cudaEventRecord(tev[2], st);
  return cudaGetLastError();
}

#if HP_FK_PROF
extern "C" int hp_debug_fk_prof(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_fkprof, sizeof(g_fkprof));
}
#endif

cudaError_t launch_fk_debug(const double* pose_dev, const DimsD& dims, const CamParams& cam,
                            float* rec, int* boxes, double* joints, double* kc,
                            cudaStream_t st) {
  k_fk_debug<<<1, 32, 0, st>>>(pose_dev, dims, cam, rec, boxes, joints, kc);
  return cudaGetLastError();
}

}  // namespace hp
