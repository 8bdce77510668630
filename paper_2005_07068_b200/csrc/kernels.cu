// kernels.cu — the hot path of libhp on sm_100a, one translation unit:
//
//   this file  : k_pack_obs, k_band_min, k_ingest (observation O = (O_s, O_d) -> one u32 per
//                pixel: fp32 depth bits, undefined depth = a quiet NaN, bit 31 = o_s;
//                S_o = sum o_s; rows A0, f3), k_ray_table (per-column dx,
//                per-lane-row dy4, NaN off the image), and every launcher
//   tile.cuh   : per-pixel analytic ray casting in packed fp32x2, the warp tile (TMA
//                observation load, cull masks, min depth, scoring), cost finalisation
//   eval.cuh   : k_eval — one CTA per (pose, split): small swarms, the depth hooks and the
//                fused PSO generation (rows A2-A8)
//   batch.cuh  : k_fk_batch (FK + tile lists, one warp per pose) and the persistent
//                renderer k_render_persist<NEAR, SUMS> (rows A2-A5)
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

}  // namespace hp

#include "tile.cuh"
#include "eval.cuh"
#include "fit.cuh"
#include "batch.cuh"

namespace hp {

// ---------------------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------------------
#ifndef HP_NW
#define HP_NW 8
#endif
constexpr int kEvalWarps = HP_NW;
#ifndef HP_RENDER_NW
#define HP_RENDER_NW 8  // warps per k_render_persist CTA (4 CTAs per SM at 64 registers)
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
  auto cfg = [&](auto f, size_t extra = 0) {
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(kMaxRayBytes + extra));
  };
  const size_t tiles = (size_t)kSlots * kMaxTiles * sizeof(BlockEnt);  // the block lists
  cfg(k_render_persist<kRenderWarps, false, false>, tiles);
  cfg(k_render_persist<kRenderWarps, true, false>, tiles);
  cfg(k_render_persist<kRenderWarps, false, true>, tiles);
  cfg(k_render_persist<kRenderWarps, true, true>, tiles);
  cfg(k_eval<kEvalWarps, float, kModeCost>);
  cfg(k_eval<kEvalWarps, double, kModeCost>);
  cfg(k_eval<kEvalWarps, double, kModeCost, false>);
  cfg(k_eval<kEvalWarps, float, kModeDepth>);
  cfg(k_eval<kEvalWarps, double, kModeDepth>);
  cfg(k_fit<false>);
  cfg(k_fit<true>);
}

static size_t fit_dyn_bytes(const CamParams& cam, int N) {
  return (size_t)ray_floats(cam.W, cam.H) * sizeof(float) + (size_t)N * kNdof * sizeof(double);
}

int fit_blocks_per_sm(const CamParams& cam, int N) {
  set_carveouts();
  if (N > kFitMaxN) return 0;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fit<false>, kFitWarps * 32,
                                                    fit_dyn_bytes(cam, N)) != cudaSuccess)
    return 0;
  return nb;
}

cudaError_t launch_fit(const EvalArgs& a, const CUtensorMap* map, bool exact, cudaStream_t st) {
  set_carveouts();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.S * a.pso.N));
  cfg.blockDim = dim3(kFitWarps * 32);
  cfg.dynamicSmemBytes = fit_dyn_bytes(a.cam, a.pso.N);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the grid barrier
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return exact ? cudaLaunchKernelEx(&cfg, k_fit<true>, a, *map)
               : cudaLaunchKernelEx(&cfg, k_fit<false>, a, *map);
}

size_t fk_record_bytes() { return sizeof(FkOut); }
size_t fk_exact_bytes() { return sizeof(FkExact); }

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
  const size_t dyn = render_dyn_bytes(cam.W, cam.H);
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
                        cudaStream_t st, cudaEvent_t* tev, const CUtensorMap* map16) {
  if (!map16) map16 = map;
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
    const size_t rdyn = render_dyn_bytes(a.cam.W, a.cam.H),
                 ndyn = render_dyn_bytes(a.cam.W, a.cam.H, true);  // the near pass
#if HP_FK_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = pgrid;
    cfg.blockDim = rblock;
    cfg.dynamicSmemBytes = rdyn;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    // timing mode: the renderer alone, launched after k_fk_batch completed (no PDL, so its
    // first poses need no FK flags); otherwise it starts on the SMs k_fk_batch frees
    cfg.numAttrs = tev ? 0 : 1;
    EvalArgs ar = a;
    ar.fk_wait = tev ? 0 : 1;
    const bool sums = a.sums_out != nullptr;
    e = sums ? cudaLaunchKernelEx(&cfg, k_render_persist<kRenderWarps, false, true>, ar, *map16)
             : cudaLaunchKernelEx(&cfg, k_render_persist<kRenderWarps, false, false>, ar, *map16);
    cfg.numAttrs = 1;
    if (e != cudaSuccess) return e;
    if (tev) cudaEventRecord(tev[2], st);  // the renderer alone (timing mode only)
    // the near-plane pass (exits at once when k_fk_batch queued nothing)
    cfg.gridDim = dim3((unsigned)(pgrid.x < 148u ? pgrid.x : 148u));
    cfg.dynamicSmemBytes = ndyn;
#if HP_SKIP_NEAR_TEST  // A/B measurement only: what the (normally empty) near pass costs
    if (0)
#endif
    e = sums ? cudaLaunchKernelEx(&cfg, k_render_persist<kRenderWarps, true, true>, a, *map)
             : cudaLaunchKernelEx(&cfg, k_render_persist<kRenderWarps, true, false>, a, *map);
    if (e != cudaSuccess) return e;
#else
    if (a.sums_out) {
      k_render_persist<kRenderWarps, false, true><<<pgrid, rblock, rdyn, st>>>(a, *map16);
      if (tev) cudaEventRecord(tev[2], st);
      k_render_persist<kRenderWarps, true, true><<<dim3(pgrid.x < 148u ? pgrid.x : 148u), rblock,
                                                 ndyn, st>>>(a, *map);
    } else {
      k_render_persist<kRenderWarps, false, false><<<pgrid, rblock, rdyn, st>>>(a, *map16);
      if (tev) cudaEventRecord(tev[2], st);
      k_render_persist<kRenderWarps, true, false><<<dim3(pgrid.x < 148u ? pgrid.x : 148u), rblock,
                                                  ndyn, st>>>(a, *map);
    }
#endif
    if (tev) cudaEventRecord(tev[3], st);
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
    if (tev) {
      cudaEventRecord(tev[2], st);
      cudaEventRecord(tev[3], st);  // single-kernel path: empty last interval
    }
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
  if (tev) {
    cudaEventRecord(tev[2], st);
    cudaEventRecord(tev[3], st);  // single-kernel path: empty last interval
  }
  return cudaGetLastError();
}

#if HP_FKB_PROF
extern "C" int hp_debug_fkb_prof(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_fkbprof, sizeof(g_fkbprof));
}
extern "C" int hp_debug_fkb_cta(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_fkbcta, sizeof(g_fkbcta));
}
#endif
#if HP_TAIL_PROF
extern "C" int hp_debug_tail_prof(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_tailprof, sizeof(g_tailprof));
}
#endif
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
