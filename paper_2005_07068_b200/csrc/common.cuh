// common.cuh — device-side parameter blocks, record layout and PTX helpers for libhp.
//
// This is product code (CUDA for sm_100a).  It shares nothing with oracle/: both follow
// DESIGN.md §2 (frozen model) and §3 (readings) independently.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

namespace hp {

constexpr int kNdof = 26;
constexpr int kNprim = 38;
constexpr int kRec = 24;   // floats per primitive record (96 B)
#ifndef HP_PX
#define HP_PX 4
#endif
constexpr int kPxPerLane = HP_PX;       // pixels per lane (one column, every other row)
constexpr int kTileW = 16;              // warp tile: 16 x (2 * kPxPerLane) pixels
constexpr int kTileH = 2 * kPxPerLane;
#ifndef HP_MAX_TILES
#define HP_MAX_TILES 256
#endif
constexpr int kMaxTiles = HP_MAX_TILES;  // block-list capacity per particle (16 x 16 blocks)
constexpr int kBlockH = 2 * kTileH;     // the batch renderer's warp block: two 16 x 8 tiles
                                        // (top / bottom half, each with its own cull masks)
constexpr int kRayPad = 16;             // ray-table slack for tiles overhanging the image
static_assert(kPxPerLane == 4, "the row table packs a lane's 4 rows into one float4");
// Ray table (k_ray_table), staged in shared memory by the evaluation kernels:
//   dx[x]  for x in [0, ray_dx_len(W)): (x + 1/2 - c_x) / f_x, NaN for x >= W
//   dy4[y] for y in [0, H + kRayPad):   float4 (dy(y), dy(y+2), dy(y+4), dy(y+6)) — the
//          rows of a lane whose first row is y — with dy(y) = (y + 1/2 - c_y) / f_y, NaN
//          for y >= H.  A NaN ray never hits (every intersection is NaN), so pixels off
//          the image need no bounds test in the scoring loop.
__host__ __device__ constexpr int ray_dx_len(int W) { return (W + kRayPad + 3) & ~3; }
constexpr size_t kMaxRayBytes = 64 * 1024;  // dynamic shared memory the kernels may use
__host__ __device__ constexpr int ray_floats(int W, int H) {
  return ray_dx_len(W) + 4 * (H + kRayPad);
}

// Primitive order on the device (sorted by kind so a cull mask splits by bit range):
//   0..19  spheres   (finger f, joint k) -> 4 f + k
//   20..31 cones     fingers 1..4, segment k -> 20 + 3 (f - 1) + k
//   32, 33 cones     thumb segments 2, 3
//   34     palm elliptic cylinder (same code path as the cones, k = 0)
//   35     thumb proximal ellipsoid
//   36, 37 palm cap ellipsoids
constexpr int kSphere0 = 0, kCone0 = 20, kCyl = 34, kEll0 = 35;
constexpr uint64_t kSphereMask = (1ull << 20) - 1;
constexpr uint64_t kConeMask = ((1ull << 35) - 1) ^ kSphereMask;
constexpr uint64_t kEllMask = ((1ull << 38) - 1) ^ ((1ull << 35) - 1);

// EXACT record layout (the near-plane path, FkExact), camera frame, fp32:
//   [0..2]  c: local origin (sphere/ellipsoid centre, cone/cylinder axis midpoint)
//   [3]     r^2 (sphere)
//   [4..12] M row-major: camera offset -> local (ellipsoid: diag(1/s) R^T;
//           cone: rows e1, e2, axis; cylinder: x_H/a, z_H/b, y_H)
//   [13..15] c_l = M c
//   [16] r_mid  [17] slope k  [18] half length (cone / cylinder)
enum RecField { kC = 0, kR2 = 3, kM = 4, kCl = 13, kRm = 16, kK = 17, kHl = 18 };
// FAST record layout (FkOut.rec, the hot loops; DESIGN §9 "inverse-depth polynomial form"),
// the same for every kind (spheres, ellipsoids, cones, the palm cylinder): with local
// coordinates l = M (p - c), implicit F(l) = l'Q l + 2 g.l + h and the pixel ray p = t d,
// d = (x, y, 1), F = 0 reads a t^2 - 2 b t + c0 = 0 with
//   a = dl'Q dl, b = dl'Q cl - g.dl, c0 = cl'Q cl - 2 g.cl + h   (dl = M d, cl = M c).
// c0 = F(camera) does not depend on the pixel, so in the inverse depth s = 1 / t the same
// equation is c0 s^2 - 2 b s + a = 0 and the root t = (b - sqrt(D)) / a the renderer wants
// (the entering root) is s = (b + sqrt(D)) / c0, D = b^2 - a c0: no per-pixel division, and
// the nearest hit is the LARGEST s.  D is quadratic, b affine in (x, y); FK expands them in
// fp64 about the projected centre (xp, yp) and stores fp32 coefficients of x' = x - xp,
// y' = y - yp (all terms O(D) over the primitive's box: the fp32 Horner evaluation does not
// cancel), b pre-scaled by 1 / c0:
//   [0] xp [1] yp  [2..7] D: d00 d10 d01 d20 d11 d02  [8..10] b / c0: b0 bx by  [11] 1 / c0
//   cones / cylinder: [12..14] (axis row of M) / hl (raw x, y, 1 coefficients)
//   [15] -cl_z / hl — the axial coordinate at the hit is within [-hl, hl] iff
//   |s (-cl_z / hl) + (lzx x + lzy y + lz1) / hl| <= s.
enum FastField { kFxp = 0, kFyp = 1, kFd = 2, kFb = 8, kFic0 = 11, kFlz = 12, kFnclz = 15 };

struct CamParams {
  int W, H;
  float fx, fy, cx, cy, znear, zfar;
};

struct DimsD {
  double palm_half_w, palm_half_t, palm_len, cap_half;
  double base[5][3], len[5][3], rad[5][4];
  double th_x, th_z;
  double RT0[3][3];  // thumb base frame Rz(yaw) Ry(pitch), host fp64
  double cone_k[5][3];  // (r_{k+1} - r_k) / L_k, the cone slopes (host fp64)
  double inv_hl[5][3];  // 1 / (L_k / 2): the cones' inverse half lengths (host fp64)
  double inv_hl_palm;   // 1 / (palm_len / 2)
  double inv_sd[2][3];  // inverse semi-axes: [0] the thumb ellipsoid (th_x, L_00 / 2, th_z),
                        // [1] the palm caps / cylinder (palm_half_w, cap_half, palm_half_t)
};

struct CostD {
  float d_m, clampv;  // per-pixel fp32 compare / clamp
  // numerator fixed point: round(min(|dd|, clamp) * 2^qbits) with qbits = the largest
  // integer <= 20 with clamp * 2^qbits <= 2^22 (so fp32 magic-number rounding is exact)
  float qscale, qmagic;  // 2^qbits, 1.5 * 2^23
  int qbits;
  double lambda, lambda_k, depth_scale, kc_rest;
};

struct PsoDyn {  // per-fit values, read from device memory so a captured graph is reusable
  uint64_t seed;
  double c1, c2, w, stop;
};
struct PsoDev {
  int N, D, K, period, per_dim_r, nmut, mut_lo, mut_hi;
  int mut_after;  // AMB-17 order: 0 mutate after the update of generation k = period, ...;
                  // 1 SPEC's: after generation k's bookkeeping, before k + 1's update
  const PsoDyn* dyn;
  const double *lo, *hi, *ilo, *ihi;  // [D]
  double *X, *V, *P, *Pc, *E, *G, *Gc, *trace;
  int* mark;
  int* done;
  int* gens_run;
  int* pimp;  // [N] deferred pbest flags (fused generations)
  int* gsel;  // [2] deferred gbest: index, taken from X (fused generations)
};

enum EvalMode { kModeCost = 0, kModeDepth = 1 };

struct EvalArgs {
  const void* poses;          // [n][26] float or double
  int n, S;                   // poses, CTAs per pose
  CamParams cam;
  DimsD dims;
  CostD cost;
  const unsigned long long* S_o;  // [frames] sum o_s per observation frame
  int frame_n;                    // frame-batched scoring: pose p scores frame p / frame_n
                                  // (0: every pose scores frame 0)
  unsigned long long* acc;        // [n][4] accumulators (zero between launches)
  unsigned int* counters;         // [n] CTA arrival counters (zero between launches)
  float* costs32;                 // optional [n]
  double* costs64;                // optional [n]
  unsigned long long* sums_out;   // optional [n][4]
  float* depth_out;               // kModeDepth: [H][W]
  const int* done;                // optional PSO stop flag: skip work when *done
  const uint32_t* obs;            // packed observation (plain-load path)
  int obs_pitch;                  // words per row
  int use_tma;                    // 1: TMA tile loads (default), 0: plain loads
  const CUtensorMap* tmap_g;      // the same descriptor in global memory (use_tma = 2)
  const float* ray;               // k_ray_table output: dx[W + pad], dy[H + pad]
  unsigned int* pcount;           // [4] persistent kernels (batch pass, near-plane pass):
                                  // particle counter, CTA exit counter
  int persist_grid;               // > 0: batch path (k_fk_batch + k_render_persist) with
                                  // this many renderer CTAs
  // PSO generation mode (hp_pso_fit): fused update before FK, fused bookkeeping at the end
  int pso_on, pso_k;
  PsoDev pso;
  const double *x_in, *v_in;      // generation k-1 positions / velocities
  double *x_out, *v_out;          // generation k (evaluated)
  unsigned int* gcount;           // grid arrival counter (zero between launches)
  double* kc_g;                   // [n] kc(h) of each particle (fused generation epilogue)
  int* near_seen;                 // non-null: speculative fit kernel (no near-plane code);
                                  // set when a particle needed it
  int pdl;                        // launched with programmatic dependent launch
  int fk_wait;                    // renderer launched under k_fk_batch (PDL): its first poses
                                  // wait for their FK flags (0: k_fk_batch is complete)
  // two-kernel batch path: k_fk_batch writes each particle's FK output and tile list here,
  // k_render_persist bulk-copies them into shared memory
  void* fk_g;                     // FkOut [n] (16-byte aligned records)
  void* fkx_g;                    // FkExact [n]: exact records, written for near-plane poses
  uint4* tiles_g;                 // [n][kMaxTiles] 16x16 blocks, 32 bytes each (BlockEnt,
                                  // tile.cuh: the origin and the masks split per kind)
  int* ntl_g;                     // [n] tile-list length (-1: box too large, cull on the fly;
                                  // -2: queued for the near-plane pass)
  unsigned int* fk_ready;         // [n] k_fk_batch -> renderer readiness: the launch epoch once
                                  // pose p's record, list and ntl are published (st.release)
  unsigned int* fk_epoch;         // the batch launch's epoch (the renderer's last CTA advances it)
  int* near_list;                 // [n] particles whose primitives may cross z_near
  unsigned int* near_count;       // their number (reset by the near-plane pass)
  // persistent fit (k_fit): per-CTA sums [2][grid][4] and per-particle evaluated position +
  // kc [2][N][32], both double-buffered by generation parity; the grid-barrier counter
  unsigned long long* fit_part;
  double* fit_xpub;
  unsigned int* fit_bar;
};

// Debug builds (-DHP_DEBUG_CHECKS=1): device-side bounds checks that trap (the GPU test
// suite is run once against such a build; compute-sanitizer is not available on the pool).
#if HP_DEBUG_CHECKS
#define HP_CHECK(cond)                                                              \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      printf("HP_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__,   \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                          \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define HP_CHECK(cond) \
  do {                 \
  } while (0)
#endif

// Observation frame of pose p; frame f occupies rows [f H, (f + 1) H) of the packed buffer
__device__ __forceinline__ int frame_of(const EvalArgs& a, int p) {
  return a.frame_n ? p / a.frame_n : 0;
}

// --------------------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA (cp.async.bulk.tensor), sm_90+ / sm_100a
// --------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Shared-memory counter increment with acquire-release semantics at CTA scope: releases
// the caller's earlier shared-memory writes, acquires those of earlier incrementers.
__device__ __forceinline__ int atom_add_acq_rel_cta(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;"
               : "=r"(old)
               : "r"(smem_u32(p)), "r"(v)
               : "memory");
  return old;
}
__device__ __forceinline__ int ld_acquire_cta_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_s32(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// expect_tx without arriving (the phase still waits for the pending arrival)
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar_s, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar_s),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  mbar_wait_s(smem_u32(bar), phase);
}
// A shared-memory address the compiler must keep in a register (no rematerialisation).
__device__ __forceinline__ uint32_t pin_u32(uint32_t v) {
  asm volatile("" : "+r"(v));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
}
// Non-volatile shared loads (schedulable like plain loads) of data that does not change
// while it is read (FK records, block lists).
__device__ __forceinline__ float4 lds_f4_nv(uint32_t a) {
  float4 v;
  asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds_f2_nv(uint32_t a) {
  float2 v;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds_u4_nv(uint32_t a) {
  uint4 v;
  asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "r"(a));
  return v;
}
// Warp-collective: lane 0 adds 1 to the shared counter at address a; every lane gets the
// old value (no divergent branch around the atomic).
template <int INC = 1>
__device__ __forceinline__ int warp_fetch_add(uint32_t a) {
  int old = 0;
  asm volatile(
      "{\n.reg .pred p;\n.reg .u32 l;\n"
      "mov.u32 l, %%laneid;\n"
      "setp.eq.u32 p, l, 0;\n"
      "@p atom.shared.add.u32 %0, [%1], %2;\n}"
      : "+r"(old)
      : "r"(a), "n"(INC)
      : "memory");
  return __shfl_sync(0xffffffffu, old, 0);
}
__device__ __forceinline__ int warp_fetch_add1(uint32_t a) { return warp_fetch_add<1>(a); }
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// Waiting with a suspend-time hint: the warp sleeps in hardware instead of spinning on
// issue slots (used by the FK producer, which waits most of the time).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// Whole-warp call (uniform control flow, warp-uniform operands): one elected lane arms
// the mbarrier with `bytes` and issues the 2-D TMA tile load.  Keeping the issue in
// uniform control flow spares the compiler its lane-election loop around UTMALDG.
__device__ __forceinline__ void tma_load_2d_elect_s(uint32_t dst_s, const CUtensorMap* map,
                                                    int x, int y, uint32_t bar_s,
                                                    uint32_t bytes) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "elect.sync _|p, 0xffffffff;\n"
      "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%4], %5;\n"
      "@p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];\n"
      "}\n" ::"r"(dst_s),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar_s), "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_elect(void* dst, const CUtensorMap* map, int x,
                                                  int y, uint64_t* bar, uint32_t bytes) {
  tma_load_2d_elect_s(smem_u32(dst), map, x, y, smem_u32(bar), bytes);
}

// 1-D bulk copy global -> shared (TMA unit), completing `bytes` on the mbarrier.
// Addresses 16-byte aligned, size a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 1-D bulk copy shared -> global (async proxy; the writer threads fence_proxy_async first)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               ::"l"(reinterpret_cast<uint64_t>(dst)), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// --------------------------------------------------------------------------------------
// Launchers (kernels.cu)
// --------------------------------------------------------------------------------------
// Packed observation word: fp32 o_d bits (bit 31 = o_s); an undefined o_d is this quiet
// NaN, so |o_d - r_d| is NaN exactly where o_d is undefined (one compare in the scoring)
constexpr uint32_t kObsUndef = 0x7fc00000u;
cudaError_t launch_fill_undef(uint32_t* obs, long long words, cudaStream_t st);
cudaError_t launch_pack_obs(const float* depth, const uint8_t* mask, uint32_t* obs, int W,
                            int H, int pitch_words, unsigned long long* S_o, cudaStream_t st);
// Row f3 front end: Kinect u16 depth (+ optional skin image) -> segmented packed observation.
struct SegD {
  int mode, lo, hi, width, keep_background;
};
// band_min (mode 1 only; *m preset to 0xFFFFFFFF): nearest valid (skin) depth of the frame
cudaError_t launch_band_min(const uint16_t* depth, const uint8_t* skin, int npx, unsigned int* m,
                            cudaStream_t st);
cudaError_t launch_ingest(const uint16_t* depth, const uint8_t* skin, int W, int H,
                          int pitch_words, const SegD& seg, const unsigned int* m, uint32_t* obs,
                          unsigned long long* S_o, cudaStream_t st);
cudaError_t launch_unpack_obs(const uint32_t* obs, int W, int H, int pitch_words, float* depth,
                              uint8_t* mask, cudaStream_t st);
// tev (optional, 3 events): recorded before the first launch, between the two launches of
// the batch path, and after the last (hp_set_timing); null when timing is off
// map: 16 x 8 observation boxes (k_eval, the near-plane pass); map16: 16 x 16 (the batch
// renderer's blocks; null = map, only for paths that never take the batch renderer)
cudaError_t launch_eval(const EvalArgs& a, bool pose_double, int mode, const CUtensorMap* map,
                        cudaStream_t st, cudaEvent_t* tev = nullptr,
                        const CUtensorMap* map16 = nullptr);
// persistent fit (k_fit, fit.cuh): one cooperative launch of a.S * N CTAs; exact = the
// near-plane code compiled in.  fit_blocks_per_sm: resident k_fit CTAs per SM (0: unusable)
cudaError_t launch_fit(const EvalArgs& a, const CUtensorMap* map, bool exact, cudaStream_t st);
int fit_blocks_per_sm(const CamParams& cam, int N);
cudaError_t launch_fk_debug(const double* pose_dev, const DimsD& dims, const CamParams& cam,
                            float* rec, int* boxes, double* joints, double* kc,
                            cudaStream_t st);
cudaError_t launch_ray_table(const CamParams& cam, float* ray, cudaStream_t st);
cudaError_t launch_depth_to_mask(const float* depth, uint8_t* mask, int npx, cudaStream_t st);
int persist_blocks_per_sm(const CamParams& cam);
int eval_blocks_per_sm(const CamParams& cam);  // resident k_eval CTAs per SM
size_t fk_record_bytes();
size_t fk_exact_bytes();

// PSO (pso.cu)
cudaError_t launch_pso_init(const PsoDev& p, cudaStream_t st);
cudaError_t launch_pso_update(const PsoDev& p, int k, cudaStream_t st);
cudaError_t launch_pso_book(const PsoDev& p, int k, cudaStream_t st);
cudaError_t launch_sphere_eval(const PsoDev& p, const double* centre, cudaStream_t st);

}  // namespace hp
