// api.cu — the C ABI of include/hp.h: context, observation upload, TMA descriptor,
// evaluation entry points, the CUDA-graph PSO driver and the test hooks.
#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <condition_variable>
#include <map>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/hp.h"
#include "common.cuh"

using namespace hp;

namespace {

// ---- NCCL, loaded at run time (dlopen) so single-GPU use has no NCCL dependency ----
// ABI subset of nccl.h 2.28 (nvidia-nccl wheel): ncclComm_t is an opaque pointer, the
// unique id is 128 bytes, ncclSuccess = 0, ncclFloat32 = 7, ncclFloat64 = 8.
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { kNcclFloat32 = 7, kNcclFloat64 = 8 };
struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};
NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    const char* env = getenv("HP_NCCL_LIB");
    void* h = env ? dlopen(env, RTLD_NOW | RTLD_GLOBAL) : nullptr;
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
      api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
      api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
      api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
      api.errorString = (decltype(api.errorString))dlsym(h, "ncclGetErrorString");
      if (api.getUniqueId && api.commInitRank && api.commDestroy && api.allGather &&
          api.errorString)
        api.handle = h;
    }
  }
  return api.handle ? &api : nullptr;
}

thread_local std::string g_err = "";

#if HP_LOOPBACK_TEST
// DEBUG BUILDS ONLY (-DHP_LOOPBACK_TEST=1, never the product library): W contexts on ONE
// GPU, each driven by its own host thread, stand in for W ranks.  The in-place allgather is
// performed with device copies at exactly ncclAllGather's offsets (rank r's chunk at
// r * chunk); ordering is by CUDA events recorded before a host barrier and waited on
// after it, so no kernel ever waits on another rank's kernel.  This executes the rank > 0
// slice offsets, the padded last chunk and the sharded fit's update -> eval -> allgather ->
// bookkeeping sequence without a multi-GPU box; NCCL stays the only product transport.
struct LoopGroup {
  int world = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t phase = 0;
  std::vector<void*> buf;
  std::vector<cudaEvent_t> ready, read;
};
std::mutex g_loop_m;
std::map<std::string, LoopGroup*> g_loop;

// generation-counting barrier; false on timeout (a rank that failed never arrives)
bool loop_barrier(LoopGroup* g) {
  std::unique_lock<std::mutex> lk(g->m);
  const uint64_t ph = g->phase;
  if (++g->arrived == g->world) {
    g->arrived = 0;
    g->phase++;
    g->cv.notify_all();
    return true;
  }
  return g->cv.wait_for(lk, std::chrono::seconds(120), [&] { return g->phase != ph; });
}
#endif

struct Graph {
  cudaGraphExec_t exec = nullptr;
  int N = -1, D = -1, K = -1, period = -1, per_dim_r = -1, nmut = -1, mut_lo = -1, mut_hi = -1;
  int sphere = -1;
  int mut_after = -1;
  int world = -1;
  int exact = -1;  // 1: generation kernels with the near-plane code (after a speculative miss)
};

}  // namespace

struct hp_ctx {
  int device = 0, sm_count = 0;
  hp_intrinsics cam{};
  hp_hand_dims dims{};
  hp_cost_params cost{};
  int max_n = 0;
  CamParams camp{};
  DimsD dimsd{};
  CostD costd{};
  // observation
  uint32_t* obs = nullptr;
  int pitch_words = 0;
  unsigned long long* S_o = nullptr;
  CUtensorMap tmap{};    // 16 x 8 observation boxes (k_eval, the near-plane pass)
  CUtensorMap tmap16{};  // 16 x 16 (the batch renderer's warp blocks)
  float* up_depth = nullptr;  // staging for host uploads
  uint8_t* up_mask = nullptr;
  int frames = 1;      // observation frames currently set (hp_set_observations)
  int frames_cap = 1;  // frames the buffers above hold
  unsigned int* band_m = nullptr;  // [frames_cap] nearest-depth reduction (row f3)
  // evaluation workspace
  unsigned long long* acc = nullptr;
  unsigned int* counters = nullptr;
  float* poses32 = nullptr;
  float* costs32 = nullptr;
  float* h_poses = nullptr;  // pinned
  float* h_costs = nullptr;  // pinned
  double* scratch = nullptr; // 26 + 38*24 + ... device scratch for hooks
  // PSO
  double *X = nullptr, *V = nullptr, *P = nullptr, *Pc = nullptr, *E = nullptr;
  double *G = nullptr, *Gc = nullptr, *trace = nullptr, *bnd = nullptr, *centre = nullptr;
  int* mark = nullptr;
  int* pimp = nullptr;  // deferred pbest flags (fused generations)
  int* gsel = nullptr;  // deferred gbest (index, from X)
  int* flags = nullptr;  // [0] done, [1] gens_run, [2] near-plane particle seen (speculative fit)
  PsoDyn* dyn = nullptr;
  double* h_out = nullptr;  // pinned: G[64], Gc, trace[K], gens_run
  int trace_cap = 0;
  int last_N = 0, last_D = 0, last_gens = 0, last_fused = 0;
  int64_t last_fit_launches = 0;
  double *X2 = nullptr, *V2 = nullptr;  // second position / velocity buffers (fused fit)
  unsigned int* gcount = nullptr;       // grid arrival counter of the fused bookkeeping
  // persistent fit (k_fit): per-CTA sums, per-particle positions + kc, barrier counter
  unsigned long long* fit_part = nullptr;
  double* fit_xpub = nullptr;
  unsigned int* fit_bar = nullptr;
  int fit_persist = 1;  // HP_NO_FIT_PERSIST=1: the per-generation kernels instead
  int last_persist = 0;  // the last fit ran k_fit (final X, V in the first buffers)
  Graph graph;
  cudaStream_t st = nullptr;
  cudaEvent_t ev = nullptr;
  int64_t last_launches = 0;
  CUtensorMap* tmap_g = nullptr;
  float* ray = nullptr;  // per-column / per-row ray directions (k_ray_table)
  unsigned int* pcount = nullptr;  // persistent-kernel counters (zero between launches)
  int persist_grid = 0;            // CTAs of the persistent kernels (0 = never use them)
  void* fk_g = nullptr;            // FkOut [max_n]
  void* fkx_g = nullptr;           // FkExact [max_n] (near-plane poses only)
  uint4* tiles_g = nullptr;        // [max_n][kMaxTiles]
  int* ntl_g = nullptr;            // [max_n]
  unsigned int* fk_ready = nullptr;  // [max_n] batch FK readiness epochs
  unsigned int* fk_epoch = nullptr;  // the batch launch epoch
  int* near_list = nullptr;        // [max_n] near-plane pass queue
  double* kc_g = nullptr;          // [max_n] kc per particle (fused PSO generations)
  unsigned int* near_count = nullptr;
  int blocks_per_sm = 0;           // resident k_eval CTAs per SM
  // particle-sharded mode (hp_shard): rank r owns poses [r chunk, (r + 1) chunk)
  ncclComm_t comm = nullptr;
#if HP_LOOPBACK_TEST
  LoopGroup* loop = nullptr;
#endif
  int rank = 0, world = 1;
  float* gat32 = nullptr;    // [chunk * world] allgather buffer (hp_eval_costs)
  double* gat64 = nullptr;   // [chunk * world] allgather buffer (hp_pso_fit costs)
  int64_t gat_cap = 0;       // chunk capacity of the buffers
  int use_tma = 1;   // HP_NO_TMA=1 in the environment selects plain loads (A/B, debugging)
  int sync_debug = 0;  // HP_SYNC_DEBUG=1: synchronise after every launch
  int use_pdl = 1;     // programmatic dependent launch between PSO generations (HP_NO_PDL=1)
  int zero_copy = 1;   // host path: kernels access mapped pinned buffers (HP_NO_ZEROCOPY=1)
  cudaEvent_t tev[4] = {nullptr, nullptr, nullptr, nullptr};  // hp_set_timing: per launch
  int timing = 0;
  int timed = 0;  // the last hp_eval_costs / hp_eval_sums recorded tev
  std::string err;
};

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e__ = (call);                                                          \
    if (e__ != cudaSuccess) {                                                          \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e__);                  \
      return e__ == cudaErrorMemoryAllocation ? HP_ERR_OOM : HP_ERR_CUDA;              \
    }                                                                                  \
  } while (0)

#define ARG(cond, msg)                \
  do {                                \
    if (!(cond)) {                    \
      if (ctx) ctx->err = (msg);      \
      g_err = (msg);                  \
      return HP_ERR_INVALID_ARG;      \
    }                                 \
  } while (0)

static double deg2rad(double d) { return d * (M_PI / 180.0); }

// particle-sharded mode (NCCL, or the debug loopback group)
static inline bool sharded(const hp_ctx* ctx) {
#if HP_LOOPBACK_TEST
  if (ctx->loop) return true;
#endif
  return ctx->comm != nullptr;
}

extern "C" {

hp_status hp_default_dims(hp_hand_dims* d) {
  if (!d) return HP_ERR_INVALID_ARG;
  static const float base[5][3] = {{30, -10, -8}, {27, -88, 0}, {9, -92, 0}, {-9, -89, 0}, {-26, -83, 0}};
  static const float len[5][3] = {{45, 32, 27}, {45, 27, 22}, {48, 30, 24}, {45, 28, 23}, {36, 21, 20}};
  static const float rad[5][4] = {
      {11, 10, 8.5f, 7.5f}, {9, 8, 7, 6}, {9.5f, 8.5f, 7.5f, 6.5f}, {9, 8, 7, 6}, {8, 7, 6.5f, 5.5f}};
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
  return HP_OK;
}

hp_status hp_default_cost(hp_cost_params* c) {
  if (!c) return HP_ERR_INVALID_ARG;
  c->d_m = 10.0;  // 1 cm
  c->d_M = 40.0;  // 4 cm
  c->lambda = 20.0;
  c->lambda_k = 10.0;
  c->depth_scale = 0.1;
  c->kc_rest = 0.0;
  c->clamp_at_dm = 0;
  return HP_OK;
}

hp_status hp_default_pso(hp_pso_params* p) {
  if (!p) return HP_ERR_INVALID_ARG;
  p->seed = 0;
  p->particles = 64;
  p->generations = 30;
  p->mutation_period = 3;
  p->per_dim_r = 0;
  p->c1 = 2.8;
  p->c2 = 1.3;
  p->mutation_fraction = 0.5;
  p->stop_threshold = -INFINITY;
  p->init_center = nullptr;
  p->init_radius = nullptr;
  p->mutation_after_eval = 0;
  return HP_OK;
}

hp_status hp_default_intrinsics(int32_t w, int32_t h, hp_intrinsics* o) {
  if (!o || w < 1 || h < 1) return HP_ERR_INVALID_ARG;
  const float s = (float)w / 640.f;
  o->width = w;
  o->height = h;
  o->fx = 525.f * s;
  o->fy = 525.f * s;
  o->cx = 0.5f * (float)w;
  o->cy = 0.5f * (float)h;
  o->z_near_mm = 300.f;
  o->z_far_mm = 2000.f;
  return HP_OK;
}

hp_status hp_bounds(double lo[26], double hi[26]) {
  if (!lo || !hi) return HP_ERR_INVALID_ARG;
  // Tables 1-2
  static const double wl[6] = {-900, -680, 500, -30, -70, -35};
  static const double wh[6] = {900, 680, 1500, 120, 75, 20};
  static const double fl[5][4] = {{0, -15, 0, -15}, {0, -15, 0, 0}, {0, -10, 0, 0}, {0, -30, 0, 0}, {0, -45, 0, 0}};
  static const double fh[5][4] = {{90, 60, 50, 70}, {90, 15, 100, 60}, {90, 10, 100, 60}, {90, 0, 100, 60}, {90, 0, 100, 60}};
  for (int i = 0; i < 6; i++) {
    lo[i] = i < 3 ? wl[i] : deg2rad(wl[i]);
    hi[i] = i < 3 ? wh[i] : deg2rad(wh[i]);
  }
  for (int f = 0; f < 5; f++)
    for (int j = 0; j < 4; j++) {
      lo[6 + 4 * f + j] = deg2rad(fl[f][j]);
      hi[6 + 4 * f + j] = deg2rad(fh[f][j]);
    }
  return HP_OK;
}

const char* hp_last_error(const hp_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

int64_t hp_last_launch_count(const hp_ctx* ctx) { return ctx ? ctx->last_launches : -1; }

hp_status hp_set_timing(hp_ctx* ctx, int32_t on) {
  ARG(ctx, "hp_set_timing: NULL context");
  cudaSetDevice(ctx->device);
  if (on && !ctx->tev[0])
    for (auto& e : ctx->tev) CK(cudaEventCreate(&e));
  ctx->timing = on ? 1 : 0;
  ctx->timed = 0;
  return HP_OK;
}

hp_status hp_last_kernel_ms(hp_ctx* ctx, float ms[3]) {
  ARG(ctx && ms, "hp_last_kernel_ms: NULL argument");
  if (!ctx->timed) {
    ctx->err = "hp_last_kernel_ms: no timed evaluation (hp_set_timing(ctx, 1) first)";
    return HP_ERR_STATE;
  }
  cudaSetDevice(ctx->device);
  CK(cudaEventSynchronize(ctx->tev[3]));
  CK(cudaEventElapsedTime(&ms[0], ctx->tev[0], ctx->tev[1]));
  CK(cudaEventElapsedTime(&ms[1], ctx->tev[1], ctx->tev[2]));
  CK(cudaEventElapsedTime(&ms[2], ctx->tev[2], ctx->tev[3]));
  return HP_OK;
}

int32_t hp_splits_for(const hp_ctx* ctx, int64_t n) {
  if (!ctx || n <= 0) return 1;
  // as many CTAs per pose as fit in ONE wave of resident CTAs (a second partial wave
  // doubles the latency of a small swarm); each split strides over the pose's tiles
  const int64_t target = (int64_t)ctx->sm_count * (ctx->blocks_per_sm > 0 ? ctx->blocks_per_sm : 3);
  int64_t s = target / n;
  if (s < 1) s = 1;
  if (s > 32) s = 32;
  return (int32_t)s;
}

void hp_destroy(hp_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->comm && nccl_api()) nccl_api()->commDestroy(ctx->comm);
  if (ctx->gat32) cudaFree(ctx->gat32);
  if (ctx->gat64) cudaFree(ctx->gat64);
  if (ctx->graph.exec) cudaGraphExecDestroy(ctx->graph.exec);
  void* dev[] = {ctx->obs, ctx->S_o, ctx->band_m, ctx->up_depth, ctx->up_mask, ctx->acc,
                 ctx->counters,
                 ctx->poses32, ctx->costs32, ctx->scratch, ctx->X, ctx->V, ctx->P, ctx->Pc,
                 ctx->E, ctx->G, ctx->Gc, ctx->trace, ctx->bnd, ctx->centre, ctx->mark,
                 ctx->flags, ctx->dyn, ctx->tmap_g, ctx->ray, ctx->pcount, ctx->X2,
                 ctx->V2, ctx->gcount, ctx->fk_g, ctx->fkx_g, ctx->tiles_g, ctx->ntl_g, ctx->fk_ready,
                 ctx->fk_epoch, ctx->near_list,
                 ctx->near_count, ctx->kc_g, ctx->pimp, ctx->gsel, ctx->fit_part,
                 ctx->fit_xpub, ctx->fit_bar};
  for (void* p : dev)
    if (p) cudaFree(p);
  if (ctx->h_poses) cudaFreeHost(ctx->h_poses);
  if (ctx->h_costs) cudaFreeHost(ctx->h_costs);
  if (ctx->h_out) cudaFreeHost(ctx->h_out);
  if (ctx->ev) cudaEventDestroy(ctx->ev);
  for (auto e : ctx->tev)
    if (e) cudaEventDestroy(e);
  if (ctx->st) cudaStreamDestroy(ctx->st);
  delete ctx;
}

static hp_status make_tmap(hp_ctx* ctx) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) {
      ctx->err = "cuTensorMapEncodeTiled unavailable";
      return HP_ERR_CUDA;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  // frames stack vertically: frame f is rows [f H, (f + 1) H)
  cuuint64_t gdim[2] = {(cuuint64_t)ctx->cam.width,
                        (cuuint64_t)ctx->cam.height * (cuuint64_t)ctx->frames_cap};
  cuuint64_t gstride[1] = {(cuuint64_t)ctx->pitch_words * 4};
  cuuint32_t es[2] = {1, 1};
  for (int m = 0; m < 2; m++) {
    cuuint32_t box[2] = {(cuuint32_t)kTileW, (cuuint32_t)(m == 0 ? kTileH : kBlockH)};
    CUresult r = encode(m == 0 ? &ctx->tmap : &ctx->tmap16, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2,
                        ctx->obs, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      ctx->err = "cuTensorMapEncodeTiled failed: " + std::to_string((int)r);
      return HP_ERR_CUDA;
    }
  }
  return HP_OK;
}

hp_status hp_create(const hp_intrinsics* cam, const hp_hand_dims* dims, const hp_cost_params* cost,
                    int32_t max_particles, int32_t device, hp_ctx** out) {
  hp_ctx* ctx = nullptr;
  ARG(out && cam, "hp_create: NULL argument");
  *out = nullptr;
  ARG(cam->width >= 1 && cam->height >= 1, "hp_create: width/height < 1");
  ARG((size_t)ray_floats(cam->width, cam->height) * sizeof(float) <= kMaxRayBytes,
      "hp_create: image too large (width + 4 height must stay below ~16k: the per-column / "
      "per-row ray table lives in shared memory)");
  ARG(cam->fx > 0 && cam->fy > 0, "hp_create: fx/fy <= 0");
  ARG(cam->z_near_mm > 0 && cam->z_far_mm > cam->z_near_mm, "hp_create: need 0 < z_near < z_far");
  ARG(max_particles >= 1, "hp_create: max_particles < 1");
  ARG(!cost || (cost->d_m > 0 && cost->d_M > 0 && cost->d_m <= 512 && cost->d_M <= 512),
      "hp_create: need 0 < d_m, d_M <= 512 mm (32-bit per-tile fixed-point numerator)");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    g_err = "hp_create: no CUDA device";
    return HP_ERR_NO_DEVICE;
  }
  if (device < 0) cudaGetDevice(&device);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10 || prop.minor != 0) {
    g_err = "hp_create: libhp is built for sm_100a (B200); device is sm_" +
            std::to_string(prop.major) + std::to_string(prop.minor);
    return HP_ERR_NO_DEVICE;
  }
  ctx = new hp_ctx();
  ctx->device = device;
  ctx->sm_count = prop.multiProcessorCount;
  ctx->cam = *cam;
  if (dims) ctx->dims = *dims; else hp_default_dims(&ctx->dims);
  if (cost) ctx->cost = *cost; else hp_default_cost(&ctx->cost);
  ctx->max_n = max_particles;
  if (const char* e = getenv("HP_NO_TMA")) ctx->use_tma = atoi(e) ? 0 : 1;
  if (const char* e = getenv("HP_TMA_MODE")) ctx->use_tma = atoi(e);
  if (const char* e = getenv("HP_SYNC_DEBUG")) ctx->sync_debug = atoi(e);
  if (const char* e = getenv("HP_NO_PDL")) ctx->use_pdl = atoi(e) ? 0 : 1;
  hp_status st = HP_OK;
#define CKC(call)                                 \
  do {                                            \
    cudaError_t e__ = (call);                     \
    if (e__ != cudaSuccess) {                     \
      g_err = std::string(#call) + ": " + cudaGetErrorString(e__); \
      hp_destroy(ctx);                            \
      return e__ == cudaErrorMemoryAllocation ? HP_ERR_OOM : HP_ERR_CUDA; \
    }                                             \
  } while (0)
  CKC(cudaSetDevice(device));
  CKC(cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking));
  CKC(cudaEventCreateWithFlags(&ctx->ev, cudaEventDisableTiming));
  // device parameter blocks
  ctx->camp = CamParams{cam->width, cam->height, cam->fx, cam->fy, cam->cx, cam->cy,
                        cam->z_near_mm, cam->z_far_mm};
  const hp_hand_dims& d = ctx->dims;
  DimsD& dd = ctx->dimsd;
  dd.palm_half_w = d.palm_half_w;
  dd.palm_half_t = d.palm_half_t;
  dd.palm_len = d.palm_len;
  dd.cap_half = d.palm_cap_half_len;
  for (int f = 0; f < 5; f++) {
    for (int i = 0; i < 3; i++) {
      dd.base[f][i] = d.base[f][i];
      dd.len[f][i] = d.seg_len[f][i];
    }
    for (int i = 0; i < 4; i++) dd.rad[f][i] = d.radius[f][i];
    for (int i = 0; i < 3; i++) {
      dd.cone_k[f][i] = (dd.rad[f][i + 1] - dd.rad[f][i]) / dd.len[f][i];
      dd.inv_hl[f][i] = 1.0 / (0.5 * dd.len[f][i]);
    }
  }
  dd.inv_hl_palm = 1.0 / (0.5 * d.palm_len);
  dd.th_x = d.thumb_ell_x;
  dd.th_z = d.thumb_ell_z;
  {  // R_T0 = Rz(yaw) Ry(pitch)
    const double a = deg2rad(d.thumb_yaw_deg), b = deg2rad(d.thumb_pitch_deg);
    const double ca = cos(a), sa = sin(a), cb = cos(b), sb = sin(b);
    const double Rz[3][3] = {{ca, -sa, 0}, {sa, ca, 0}, {0, 0, 1}};
    const double Ry[3][3] = {{cb, 0, sb}, {0, 1, 0}, {-sb, 0, cb}};
    for (int i = 0; i < 3; i++)
      for (int j = 0; j < 3; j++)
        dd.RT0[i][j] = Rz[i][0] * Ry[0][j] + Rz[i][1] * Ry[1][j] + Rz[i][2] * Ry[2][j];
  }
  // inverse semi-axes (IEEE divisions here give the bits the kernels would compute)
  dd.inv_sd[0][0] = 1.0 / dd.th_x;
  dd.inv_sd[0][1] = 1.0 / (0.5 * dd.len[0][0]);
  dd.inv_sd[0][2] = 1.0 / dd.th_z;
  dd.inv_sd[1][0] = 1.0 / dd.palm_half_w;
  dd.inv_sd[1][1] = 1.0 / dd.cap_half;
  dd.inv_sd[1][2] = 1.0 / dd.palm_half_t;
  const hp_cost_params& c = ctx->cost;
  {
    CostD& cd = ctx->costd;
    cd.d_m = (float)c.d_m;
    cd.clampv = (float)(c.clamp_at_dm ? c.d_m : c.d_M);
    cd.lambda = c.lambda;
    cd.lambda_k = c.lambda_k;
    cd.depth_scale = c.depth_scale;
    cd.kc_rest = c.kc_rest;
    // numerator fixed point 2^-qbits mm: clamp * 2^qbits <= 2^22 (clamp <= 512 by the
    // validation above, so qbits >= 13: 1.2e-4 mm; 16 for the default 40 mm)
    int qb = 20;
    while (qb > 0 && std::ldexp((double)cd.clampv, qb) > 4194304.0) qb--;
    cd.qbits = qb;
    cd.qscale = std::ldexp(1.0f, qb);
    cd.qmagic = 12582912.0f;  // 1.5 * 2^23
  }
  // observation buffers
  const int W = cam->width, H = cam->height;
  ctx->pitch_words = (W + 3) & ~3;  // 16-byte row pitch for TMA
  CKC(cudaMalloc(&ctx->obs, (size_t)ctx->pitch_words * H * 4));
  CKC(launch_fill_undef(ctx->obs, (long long)ctx->pitch_words * H, ctx->st));
  CKC(cudaMalloc(&ctx->S_o, sizeof(unsigned long long)));
  CKC(cudaMemset(ctx->S_o, 0, sizeof(unsigned long long)));
  CKC(cudaMalloc(&ctx->band_m, sizeof(unsigned int)));
  CKC(cudaMalloc(&ctx->up_depth, (size_t)W * H * 4));
  CKC(cudaMalloc(&ctx->up_mask, (size_t)W * H));
  st = make_tmap(ctx);
  if (st != HP_OK) {
    g_err = ctx->err;
    hp_destroy(ctx);
    return st;
  }
  // ray table (common.cuh layout; a multiple of 4 floats for the float4 staging copy)
  CKC(cudaMalloc(&ctx->ray, (size_t)ray_floats(W, H) * sizeof(float)));
  CKC(launch_ray_table(ctx->camp, ctx->ray, ctx->st));
  CKC(cudaMalloc(&ctx->fk_g, (size_t)max_particles * fk_record_bytes()));
  CKC(cudaMalloc(&ctx->fkx_g, (size_t)max_particles * fk_exact_bytes()));
  CKC(cudaMalloc(&ctx->tiles_g, (size_t)max_particles * kMaxTiles * 2 * sizeof(uint4)));
  CKC(cudaMalloc(&ctx->ntl_g, (size_t)max_particles * sizeof(int)));
  CKC(cudaMalloc(&ctx->fk_ready, (size_t)max_particles * sizeof(unsigned int)));
  CKC(cudaMemset(ctx->fk_ready, 0, (size_t)max_particles * sizeof(unsigned int)));
  CKC(cudaMalloc(&ctx->fk_epoch, sizeof(unsigned int)));
  {
    const unsigned int one = 1;  // epoch 1: no flag holds it yet
    CKC(cudaMemcpy(ctx->fk_epoch, &one, sizeof(one), cudaMemcpyHostToDevice));
  }
  CKC(cudaMalloc(&ctx->pcount, 4 * sizeof(unsigned int)));
  CKC(cudaMemset(ctx->pcount, 0, 4 * sizeof(unsigned int)));
  CKC(cudaMalloc(&ctx->near_list, (size_t)max_particles * sizeof(int)));
  CKC(cudaMalloc(&ctx->kc_g, (size_t)max_particles * sizeof(double)));
  CKC(cudaMalloc(&ctx->near_count, sizeof(unsigned int)));
  CKC(cudaMemset(ctx->near_count, 0, sizeof(unsigned int)));
  ctx->blocks_per_sm = eval_blocks_per_sm(ctx->camp);
  ctx->persist_grid = ctx->sm_count * persist_blocks_per_sm(ctx->camp);
  if (const char* e = getenv("HP_NO_ZEROCOPY"))
    if (atoi(e)) ctx->zero_copy = 0;
  if (const char* e = getenv("HP_NO_PERSIST"))
    if (atoi(e)) ctx->persist_grid = 0;
  if (const char* e = getenv("HP_PERSIST_GRID"))  // A/B: the renderer's CTA count
    if (atoi(e) > 0) ctx->persist_grid = atoi(e);
  // the persistent renderer always loads observation tiles by TMA from its kernel-parameter
  // descriptor (compile time); the HP_NO_TMA / HP_TMA_MODE A/B switches use k_eval
  if (ctx->use_tma != 1) ctx->persist_grid = 0;
  CKC(cudaMalloc(&ctx->tmap_g, sizeof(CUtensorMap)));
  CKC(cudaMemcpy(ctx->tmap_g, &ctx->tmap, sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  // evaluation workspace
  const size_t N = (size_t)max_particles;
  CKC(cudaMalloc(&ctx->acc, N * 4 * sizeof(unsigned long long)));
  CKC(cudaMemset(ctx->acc, 0, N * 4 * sizeof(unsigned long long)));
  CKC(cudaMalloc(&ctx->counters, N * sizeof(unsigned int)));
  CKC(cudaMemset(ctx->counters, 0, N * sizeof(unsigned int)));
  CKC(cudaMalloc(&ctx->poses32, N * kNdof * sizeof(float)));
  CKC(cudaMalloc(&ctx->costs32, N * sizeof(float)));
  CKC(cudaMallocHost(&ctx->h_poses, N * kNdof * sizeof(float)));
  CKC(cudaMallocHost(&ctx->h_costs, N * sizeof(float)));
  CKC(cudaMalloc(&ctx->scratch, 4096 * sizeof(double)));
  // PSO state (D <= 64 for the generic hook, 26 for the hand)
  const size_t ND = N * 64;
  CKC(cudaMalloc(&ctx->X, ND * sizeof(double)));
  CKC(cudaMalloc(&ctx->V, ND * sizeof(double)));
  CKC(cudaMalloc(&ctx->X2, ND * sizeof(double)));
  CKC(cudaMalloc(&ctx->V2, ND * sizeof(double)));
  CKC(cudaMalloc(&ctx->gcount, sizeof(unsigned int)));
  CKC(cudaMemset(ctx->gcount, 0, sizeof(unsigned int)));
  CKC(cudaMalloc(&ctx->fit_part, (size_t)2 * ctx->sm_count * 4 * sizeof(unsigned long long)));
  CKC(cudaMalloc(&ctx->fit_xpub, (size_t)2 * ctx->sm_count * 32 * sizeof(double)));
  CKC(cudaMalloc(&ctx->fit_bar, sizeof(unsigned int)));
  if (const char* e = getenv("HP_NO_FIT_PERSIST"))
    if (atoi(e)) ctx->fit_persist = 0;
  CKC(cudaMalloc(&ctx->P, ND * sizeof(double)));
  CKC(cudaMalloc(&ctx->Pc, N * sizeof(double)));
  CKC(cudaMalloc(&ctx->E, N * sizeof(double)));
  CKC(cudaMalloc(&ctx->mark, N * sizeof(int)));
  CKC(cudaMalloc(&ctx->pimp, N * sizeof(int)));
  CKC(cudaMalloc(&ctx->gsel, 2 * sizeof(int)));
  CKC(cudaMalloc(&ctx->G, 64 * sizeof(double)));
  CKC(cudaMalloc(&ctx->Gc, sizeof(double)));
  CKC(cudaMalloc(&ctx->bnd, 4 * 64 * sizeof(double)));
  CKC(cudaMalloc(&ctx->centre, 64 * sizeof(double)));
  CKC(cudaMalloc(&ctx->flags, 4 * sizeof(int)));
  CKC(cudaMemset(ctx->flags, 0, 4 * sizeof(int)));
  CKC(cudaMalloc(&ctx->dyn, sizeof(PsoDyn)));
  ctx->trace_cap = 0;
  CKC(cudaDeviceSynchronize());
#undef CKC
  *out = ctx;
  return HP_OK;
}

// Grow the observation buffers to M frames: re-encode the tensor map and drop captured
// graphs (they hold the old map by value).
static hp_status ensure_frames(hp_ctx* ctx, int M) {
  if (M <= ctx->frames_cap) return HP_OK;
  const int W = ctx->cam.width, H = ctx->cam.height;
  CK(cudaDeviceSynchronize());
  cudaFree(ctx->obs);
  cudaFree(ctx->S_o);
  cudaFree(ctx->band_m);
  cudaFree(ctx->up_depth);
  cudaFree(ctx->up_mask);
  ctx->obs = nullptr;
  ctx->S_o = nullptr;
  ctx->band_m = nullptr;
  ctx->up_depth = nullptr;
  ctx->up_mask = nullptr;
  ctx->frames_cap = 0;
  const size_t px = (size_t)W * H * M;
  CK(cudaMalloc(&ctx->obs, (size_t)ctx->pitch_words * H * M * 4));
  CK(launch_fill_undef(ctx->obs, (long long)ctx->pitch_words * H * M, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  CK(cudaMalloc(&ctx->S_o, (size_t)M * sizeof(unsigned long long)));
  CK(cudaMemset(ctx->S_o, 0, (size_t)M * sizeof(unsigned long long)));
  CK(cudaMalloc(&ctx->band_m, (size_t)M * sizeof(unsigned int)));
  CK(cudaMalloc(&ctx->up_depth, px * 4));
  CK(cudaMalloc(&ctx->up_mask, px));
  ctx->frames_cap = M;
  hp_status st = make_tmap(ctx);
  if (st != HP_OK) return st;
  CK(cudaMemcpy(ctx->tmap_g, &ctx->tmap, sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  if (ctx->graph.exec) {
    cudaGraphExecDestroy(ctx->graph.exec);
    ctx->graph.exec = nullptr;
  }
  return HP_OK;
}

hp_status hp_set_observations(hp_ctx* ctx, const float* depth, const uint8_t* mask,
                              int32_t frames, int32_t on_device, void* stream) {
  ARG(ctx && depth && mask, "hp_set_observations: NULL argument");
  ARG(frames >= 1, "hp_set_observations: frames must be >= 1");
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  hp_status st = ensure_frames(ctx, frames);
  if (st != HP_OK) return st;
  const int W = ctx->cam.width, H = ctx->cam.height;
  const size_t npx = (size_t)W * H;
  const float* dd = depth;
  const uint8_t* dm = mask;
  if (!on_device) {
    CK(cudaMemcpyAsync(ctx->up_depth, depth, npx * frames * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->up_mask, mask, npx * frames, cudaMemcpyHostToDevice, s));
    dd = ctx->up_depth;
    dm = ctx->up_mask;
  }
  CK(cudaMemsetAsync(ctx->S_o, 0, (size_t)frames * sizeof(unsigned long long), s));
  for (int f = 0; f < frames; f++)
    CK(launch_pack_obs(dd + f * npx, dm + f * npx, ctx->obs + (size_t)f * H * ctx->pitch_words,
                       W, H, ctx->pitch_words, ctx->S_o + f, s));
  CK(cudaStreamSynchronize(s));
  ctx->frames = frames;
  return HP_OK;
}

hp_status hp_default_segment(hp_segment_params* out) {
  if (!out) return HP_ERR_INVALID_ARG;
  *out = hp_segment_params{1, 0, 0, 250, 0};  // nearest-object band, 25 cm deep (AMB-34)
  return HP_OK;
}

hp_status hp_set_observation_kinect(hp_ctx* ctx, const uint16_t* depth_mm, const uint8_t* skin,
                                    int32_t frames, const hp_segment_params* seg,
                                    int32_t on_device, int32_t* band_out, void* stream) {
  ARG(ctx && depth_mm, "hp_set_observation_kinect: NULL argument");
  ARG(frames >= 1, "hp_set_observation_kinect: frames must be >= 1");
  hp_segment_params sp;
  hp_default_segment(&sp);
  if (seg) sp = *seg;
  ARG((sp.mode == 0 || sp.mode == 1) && sp.width_mm >= 0,
      "hp_set_observation_kinect: mode must be 0 or 1 and width_mm >= 0");
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  hp_status st = ensure_frames(ctx, frames);
  if (st != HP_OK) return st;
  const int W = ctx->cam.width, H = ctx->cam.height;
  const size_t npx = (size_t)W * H;
  const uint16_t* dd = depth_mm;
  const uint8_t* sk = skin;
  if (!on_device) {  // staging: up_depth holds 4 bytes per pixel, u16 needs 2
    CK(cudaMemcpyAsync(ctx->up_depth, depth_mm, npx * frames * 2, cudaMemcpyHostToDevice, s));
    dd = reinterpret_cast<const uint16_t*>(ctx->up_depth);
    if (skin) {
      CK(cudaMemcpyAsync(ctx->up_mask, skin, npx * frames, cudaMemcpyHostToDevice, s));
      sk = ctx->up_mask;
    }
  }
  const SegD sd{sp.mode, sp.lo_mm, sp.hi_mm, sp.width_mm, sp.keep_background};
  CK(cudaMemsetAsync(ctx->S_o, 0, (size_t)frames * sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(ctx->band_m, 0xFF, (size_t)frames * sizeof(unsigned int), s));
  for (int f = 0; f < frames; f++) {
    const uint16_t* df = dd + f * npx;
    const uint8_t* sf = sk ? sk + f * npx : nullptr;
    if (sp.mode == 1) CK(launch_band_min(df, sf, (int)npx, ctx->band_m + f, s));
    CK(launch_ingest(df, sf, W, H, ctx->pitch_words, sd, ctx->band_m + f,
                     ctx->obs + (size_t)f * H * ctx->pitch_words, ctx->S_o + f, s));
  }
  if (band_out) {
    std::vector<unsigned int> m(frames);
    CK(cudaMemcpyAsync(m.data(), ctx->band_m, frames * sizeof(unsigned int),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int f = 0; f < frames; f++) {
      long long lo = sp.lo_mm, hi = sp.hi_mm;
      if (sp.mode == 1) {
        if (m[f] == 0xFFFFFFFFu) {
          lo = 1;
          hi = 0;
        } else {
          lo = m[f];
          hi = (long long)m[f] + sp.width_mm;
        }
      }
      band_out[2 * f] = (int32_t)lo;
      band_out[2 * f + 1] = (int32_t)std::min<long long>(hi, INT32_MAX);
    }
  }
  CK(cudaStreamSynchronize(s));
  ctx->frames = frames;
  return HP_OK;
}

hp_status hp_get_observation(hp_ctx* ctx, int32_t frame, float* depth_dev, uint8_t* mask_dev,
                             void* stream) {
  ARG(ctx, "hp_get_observation: NULL context");
  ARG(frame >= 0 && frame < ctx->frames, "hp_get_observation: frame out of range");
  cudaSetDevice(ctx->device);
  const int W = ctx->cam.width, H = ctx->cam.height;
  CK(launch_unpack_obs(ctx->obs + (size_t)frame * H * ctx->pitch_words, W, H, ctx->pitch_words,
                       depth_dev, mask_dev, (cudaStream_t)stream));
  return HP_OK;
}

hp_status hp_set_observation(hp_ctx* ctx, const float* depth, const uint8_t* mask,
                             int32_t on_device, void* stream) {
  ARG(ctx && depth && mask, "hp_set_observation: NULL argument");
  return hp_set_observations(ctx, depth, mask, 1, on_device, stream);
}

static EvalArgs base_args(hp_ctx* ctx) {
  EvalArgs a{};
  a.cam = ctx->camp;
  a.dims = ctx->dimsd;
  a.cost = ctx->costd;
  a.S_o = ctx->S_o;
  a.acc = ctx->acc;
  a.counters = ctx->counters;
  a.obs = ctx->obs;
  a.obs_pitch = ctx->pitch_words;
  a.use_tma = ctx->use_tma;
  a.tmap_g = ctx->tmap_g;
  a.ray = ctx->ray;
  a.pcount = ctx->pcount;
  a.persist_grid = ctx->persist_grid;
  a.fk_g = ctx->fk_g;
  a.fkx_g = ctx->fkx_g;
  a.tiles_g = ctx->tiles_g;
  a.ntl_g = ctx->ntl_g;
  a.fk_ready = ctx->fk_ready;
  a.fk_epoch = ctx->fk_epoch;
  a.near_list = ctx->near_list;
  a.near_count = ctx->near_count;
  a.fit_part = ctx->fit_part;
  a.fit_xpub = ctx->fit_xpub;
  a.fit_bar = ctx->fit_bar;
  return a;
}

static hp_status render_depth(hp_ctx* ctx, const void* pose, bool pose_double, float* depth,
                              cudaStream_t s) {
  const int W = ctx->cam.width, H = ctx->cam.height;
  CK(cudaMemsetAsync(depth, 0, (size_t)W * H * 4, s));
  EvalArgs a = base_args(ctx);
  a.poses = pose;
  a.n = 1;
  a.S = 64;
  a.depth_out = depth;
  CK(launch_eval(a, pose_double, kModeDepth, &ctx->tmap, s));
  return HP_OK;
}

hp_status hp_render_observation(hp_ctx* ctx, const double* h_ref, float* depth_dev,
                                uint8_t* mask_dev, void* stream) {
  ARG(ctx && h_ref && depth_dev, "hp_render_observation: NULL argument");
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(ctx->scratch, h_ref, kNdof * sizeof(double), cudaMemcpyHostToDevice, s));
  hp_status r = render_depth(ctx, ctx->scratch, true, depth_dev, s);
  if (r != HP_OK) return r;
  if (mask_dev) CK(launch_depth_to_mask(depth_dev, mask_dev, ctx->cam.width * ctx->cam.height, s));
  CK(cudaStreamSynchronize(s));  // h_ref staging is reused
  return HP_OK;
}

hp_status hp_debug_render(hp_ctx* ctx, const float* pose_dev, float* depth_dev, void* stream) {
  ARG(ctx && pose_dev && depth_dev, "hp_debug_render: NULL argument");
  cudaSetDevice(ctx->device);
  return render_depth(ctx, pose_dev, false, depth_dev, (cudaStream_t)stream);
}

static hp_status eval_common(hp_ctx* ctx, const void* poses, int64_t n, float* costs32,
                             double* costs64, uint64_t* sums, cudaStream_t s,
                             int64_t frame_n = 0, bool pose_double = false) {
  EvalArgs a = base_args(ctx);
  a.poses = poses;
  a.n = (int)n;
  a.frame_n = (int)frame_n;
  a.S = hp_splits_for(ctx, n);
  a.costs32 = costs32;
  a.costs64 = costs64;
  a.sums_out = reinterpret_cast<unsigned long long*>(sums);
  CK(launch_eval(a, pose_double, kModeCost, &ctx->tmap, s, ctx->timing ? ctx->tev : nullptr,
                 &ctx->tmap16));
  ctx->timed = ctx->timing;
  if (ctx->sync_debug) CK(cudaStreamSynchronize(s));
  // the batch path is three kernels (FK, the persistent renderer, its near-plane pass)
  ctx->last_launches = (a.S == 1 && a.persist_grid > 0) ? 3 : 1;
  return HP_OK;
}

static inline void shard_range(int64_t n, int rank, int world, int64_t* b, int64_t* e) {
  const int64_t chunk = (n + world - 1) / world;
  *b = std::min<int64_t>(n, (int64_t)rank * chunk);
  *e = std::min<int64_t>(n, *b + chunk);
}

// Sharded objective: this rank scores its slice of the N poses into its chunk of the
// allgather buffer; ncclAllGather (in place) gives every rank all N costs.
// In-place allgather of `chunk` elements per rank (rank r's at buf + r chunk): NCCL over
// NVLink / NVSwitch in the product; device copies between same-GPU contexts in the debug
// loopback build.
static hp_status allgather(hp_ctx* ctx, void* buf, int64_t chunk, int dtype, cudaStream_t s) {
  const size_t es = dtype == kNcclFloat64 ? 8 : 4;
#if HP_LOOPBACK_TEST
  if (LoopGroup* g = ctx->loop) {
    const int r = ctx->rank;
    g->buf[r] = buf;
    CK(cudaEventRecord(g->ready[r], s));
    if (!loop_barrier(g)) {
      ctx->err = "loopback allgather: barrier timeout";
      return HP_ERR_NCCL;
    }
    for (int j = 0; j < g->world; j++) {
      if (j == r) continue;
      CK(cudaStreamWaitEvent(s, g->ready[j], 0));
      CK(cudaMemcpyAsync(static_cast<char*>(buf) + (size_t)j * chunk * es,
                         static_cast<const char*>(g->buf[j]) + (size_t)j * chunk * es,
                         (size_t)chunk * es, cudaMemcpyDeviceToDevice, s));
    }
    CK(cudaEventRecord(g->read[r], s));
    if (!loop_barrier(g)) {
      ctx->err = "loopback allgather: barrier timeout";
      return HP_ERR_NCCL;
    }
    // a rank's next write to its own chunk is ordered after every peer's read of it
    for (int j = 0; j < g->world; j++)
      if (j != r) CK(cudaStreamWaitEvent(s, g->read[j], 0));
    return HP_OK;
  }
#endif
  char* mine = static_cast<char*>(buf) + (size_t)ctx->rank * chunk * es;
  const ncclResult_t nr = nccl_api()->allGather(mine, buf, (size_t)chunk, dtype, ctx->comm, s);
  if (nr != 0) {
    ctx->err = std::string("ncclAllGather: ") + nccl_api()->errorString(nr);
    return HP_ERR_NCCL;
  }
  return HP_OK;
}

// Sharded objective: this rank scores its slice of the N poses into its chunk of the
// allgather buffer; the in-place allgather gives every rank all N costs.  A rank whose own
// scoring fails still takes part in the collective (so its peers do not hang in it) and
// then reports the error.
static hp_status eval_sharded(hp_ctx* ctx, const float* poses, int64_t n, float* costs,
                              cudaStream_t s) {
  const int64_t chunk = (n + ctx->world - 1) / ctx->world;
  if (chunk > ctx->gat_cap) {
    ctx->err = "sharded eval: n exceeds max_particles * world";
    return HP_ERR_INVALID_ARG;
  }
  int64_t b, e;
  shard_range(n, ctx->rank, ctx->world, &b, &e);
  int64_t launches = 0;
  hp_status r = HP_OK;
  if (e > b) {
    r = eval_common(ctx, poses + b * kNdof, e - b, ctx->gat32 + ctx->rank * chunk, nullptr,
                    nullptr, s);
    launches = ctx->last_launches;
  }
  const std::string local_err = ctx->err;
  hp_status g = allgather(ctx, ctx->gat32, chunk, kNcclFloat32, s);
  if (r != HP_OK) {
    ctx->err = local_err;
    return r;
  }
  if (g != HP_OK) return g;
  CK(cudaMemcpyAsync(costs, ctx->gat32, (size_t)n * sizeof(float), cudaMemcpyDeviceToDevice, s));
  ctx->last_launches = launches;
  return HP_OK;
}

hp_status hp_eval_costs(hp_ctx* ctx, const float* poses, int64_t n, float* costs, void* stream) {
  ARG(ctx, "hp_eval_costs: NULL ctx");
  ARG(n >= 0 && n <= (int64_t)ctx->max_n * ctx->world,
      "hp_eval_costs: n < 0 or n > max_particles (x world when sharded)");
  if (n == 0) return HP_OK;
  ARG(poses && costs, "hp_eval_costs: NULL buffer");
  cudaSetDevice(ctx->device);
  if (sharded(ctx)) return eval_sharded(ctx, poses, n, costs, (cudaStream_t)stream);
  return eval_common(ctx, poses, n, costs, nullptr, nullptr, (cudaStream_t)stream);
}

hp_status hp_eval_costs_frames(hp_ctx* ctx, const float* poses, int32_t frames,
                               int64_t n_per_frame, float* costs, void* stream) {
  ARG(ctx, "hp_eval_costs_frames: NULL context");
  ARG(frames == ctx->frames, "hp_eval_costs_frames: frames differs from the frame count of "
                             "the current observation (hp_set_observations)");
  const int64_t total = n_per_frame * ctx->frames;
  ARG(n_per_frame >= 0 && total <= ctx->max_n,
      "hp_eval_costs_frames: n_per_frame * frames must be in [0, max_particles]");
  if (total == 0) return HP_OK;
  ARG(poses && costs, "hp_eval_costs_frames: NULL argument");
  cudaSetDevice(ctx->device);
  // frames are this rank's own: no collective even in sharded mode (frames shard by rank)
  return eval_common(ctx, poses, total, costs, nullptr, nullptr, (cudaStream_t)stream,
                     n_per_frame);
}

hp_status hp_eval_sums_frames(hp_ctx* ctx, const float* poses, int32_t frames,
                              int64_t n_per_frame, uint64_t* sums, double* costs64,
                              void* stream) {
  ARG(ctx, "hp_eval_sums_frames: NULL context");
  ARG(frames == ctx->frames, "hp_eval_sums_frames: frames differs from the frame count of "
                             "the current observation (hp_set_observations)");
  const int64_t total = n_per_frame * ctx->frames;
  ARG(n_per_frame >= 0 && total <= ctx->max_n,
      "hp_eval_sums_frames: n_per_frame * frames must be in [0, max_particles]");
  if (total == 0) return HP_OK;
  ARG(poses && sums, "hp_eval_sums_frames: NULL argument");
  cudaSetDevice(ctx->device);
  return eval_common(ctx, poses, total, nullptr, costs64, sums, (cudaStream_t)stream,
                     n_per_frame);
}

static bool is_pinned(const void* p, void** dev = nullptr) {
  cudaPointerAttributes at{};
  if (dev) *dev = nullptr;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();  // clear the sticky-free error of an unknown pointer
    return false;
  }
  if (at.type != cudaMemoryTypeHost) return false;
  if (dev) *dev = at.devicePointer;  // mapped page-locked memory: the kernels' address
  return true;
}

hp_status hp_eval_costs_host(hp_ctx* ctx, const float* poses, int64_t n, float* costs,
                             void* stream) {
  ARG(ctx, "hp_eval_costs_host: NULL ctx");
  ARG(n >= 0 && n <= (int64_t)ctx->max_n * ctx->world,
      "hp_eval_costs_host: n < 0 or n > max_particles (x world when sharded)");
  if (n == 0) return HP_OK;
  ARG(poses && costs, "hp_eval_costs_host: NULL buffer");
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (sharded(ctx)) {
    // sharded: upload only this rank's slice, score it, allgather, download all costs
    const int64_t chunk = (n + ctx->world - 1) / ctx->world;
    if (chunk > ctx->gat_cap) {
      ctx->err = "sharded eval: n exceeds max_particles * world";
      return HP_ERR_INVALID_ARG;
    }
    int64_t b, e;
    shard_range(n, ctx->rank, ctx->world, &b, &e);
    const size_t in_bytes = (size_t)(e - b) * kNdof * sizeof(float);
    const bool in_pinned = is_pinned(poses), out_pinned = is_pinned(costs);
    if (!in_pinned) memcpy(ctx->h_poses, poses + b * kNdof, in_bytes);
    hp_status r = HP_OK;
    if (e > b) {
      cudaError_t ce = cudaMemcpyAsync(ctx->poses32, in_pinned ? poses + b * kNdof : ctx->h_poses,
                                       in_bytes, cudaMemcpyHostToDevice, s);
      if (ce != cudaSuccess) {
        ctx->err = std::string("cudaMemcpyAsync: ") + cudaGetErrorString(ce);
        r = HP_ERR_CUDA;
      } else {
        r = eval_common(ctx, ctx->poses32, e - b, ctx->gat32 + ctx->rank * chunk, nullptr,
                        nullptr, s);
      }
    }
    const std::string local_err = ctx->err;
    hp_status g = allgather(ctx, ctx->gat32, chunk, kNcclFloat32, s);  // always take part
    if (r != HP_OK) {
      ctx->err = local_err;
      return r;
    }
    if (g != HP_OK) return g;
    CK(cudaMemcpyAsync(out_pinned ? costs : ctx->h_costs, ctx->gat32, (size_t)n * sizeof(float),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (!out_pinned) memcpy(costs, ctx->h_costs, (size_t)n * sizeof(float));
    return HP_OK;
  }
  // Page-locked caller buffers (cudaHostAlloc / cudaHostRegister / torch pin_memory) are
  // DMA'd directly; pageable ones go through the context's pinned staging buffers.
  // Mapped page-locked buffers are read / written by the kernels over the host link
  // (zero-copy: the FK kernel's pose loads are the host->device transfer, the cost
  // finalisation's stores the device->host one), unless HP_NO_ZEROCOPY=1.
  const size_t in_bytes = (size_t)n * kNdof * sizeof(float), out_bytes = (size_t)n * 4;
  void *in_dev = nullptr, *out_dev = nullptr;
  const bool in_pinned = is_pinned(poses, &in_dev), out_pinned = is_pinned(costs, &out_dev);
  if (!ctx->zero_copy) in_dev = out_dev = nullptr;
  const float* src = poses;
  if (!in_pinned) {
    memcpy(ctx->h_poses, poses, in_bytes);
    src = ctx->h_poses;
  }
  const float* dposes = static_cast<const float*>(in_dev);
  if (!dposes) {
    CK(cudaMemcpyAsync(ctx->poses32, src, in_bytes, cudaMemcpyHostToDevice, s));
    dposes = ctx->poses32;
  }
  float* dcosts = out_dev ? static_cast<float*>(out_dev) : ctx->costs32;
  hp_status r = eval_common(ctx, dposes, n, dcosts, nullptr, nullptr, s);
  if (r != HP_OK) return r;
  if (!out_dev)
    CK(cudaMemcpyAsync(out_pinned ? costs : ctx->h_costs, ctx->costs32, out_bytes,
                       cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (!out_pinned) memcpy(costs, ctx->h_costs, out_bytes);
  return HP_OK;
}

hp_status hp_eval_sums(hp_ctx* ctx, const float* poses, int64_t n, uint64_t* sums,
                       double* costs64, void* stream) {
  ARG(ctx, "hp_eval_sums: NULL ctx");
  ARG(n >= 0 && n <= ctx->max_n, "hp_eval_sums: n < 0 or n > max_particles");
  if (n == 0) return HP_OK;
  ARG(poses && sums, "hp_eval_sums: NULL buffer");
  cudaSetDevice(ctx->device);
  return eval_common(ctx, poses, n, nullptr, costs64, sums, (cudaStream_t)stream);
}

hp_status hp_eval_sums_f64(hp_ctx* ctx, const double* poses, int64_t n, uint64_t* sums,
                           double* costs64, void* stream) {
  ARG(ctx, "hp_eval_sums_f64: NULL ctx");
  ARG(n >= 0 && n <= ctx->max_n, "hp_eval_sums_f64: n < 0 or n > max_particles");
  if (n == 0) return HP_OK;
  ARG(poses && (sums || costs64), "hp_eval_sums_f64: NULL buffer");
  cudaSetDevice(ctx->device);
  return eval_common(ctx, poses, n, nullptr, costs64, sums, (cudaStream_t)stream, 0, true);
}

hp_status hp_debug_batch_fk(hp_ctx* ctx, int64_t p, float* records, int32_t* boxes) {
  ARG(ctx && p >= 0 && p < ctx->max_n, "hp_debug_batch_fk: bad argument");
  cudaSetDevice(ctx->device);
  CK(cudaStreamSynchronize(ctx->st));
  CK(cudaDeviceSynchronize());
  std::vector<char> buf(fk_record_bytes());
  CK(cudaMemcpy(buf.data(), static_cast<char*>(ctx->fk_g) + (size_t)p * fk_record_bytes(),
                buf.size(), cudaMemcpyDeviceToHost));
  if (records) memcpy(records, buf.data(), kNprim * kRec * sizeof(float));
  if (boxes) memcpy(boxes, buf.data() + kNprim * kRec * sizeof(float), kNprim * 16);
  return HP_OK;
}

hp_status hp_debug_fk(hp_ctx* ctx, const double* pose, float* records, int32_t* boxes,
                      double* joints, double* kc) {
  ARG(ctx && pose, "hp_debug_fk: NULL argument");
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->st;
  double* dpose = ctx->scratch;                              // 26
  float* drec = reinterpret_cast<float*>(ctx->scratch + 32); // 38*24 floats = 456 doubles
  int* dbox = reinterpret_cast<int*>(ctx->scratch + 32 + 456);  // 152 ints = 76 doubles
  double* djoint = ctx->scratch + 32 + 456 + 80;             // 60
  double* dkc = djoint + 64;
  CK(cudaMemcpyAsync(dpose, pose, kNdof * sizeof(double), cudaMemcpyHostToDevice, s));
  CK(launch_fk_debug(dpose, ctx->dimsd, ctx->camp, drec, dbox, djoint, dkc, s));
  if (records) CK(cudaMemcpyAsync(records, drec, kNprim * kRec * 4, cudaMemcpyDeviceToHost, s));
  if (boxes) CK(cudaMemcpyAsync(boxes, dbox, kNprim * 16, cudaMemcpyDeviceToHost, s));
  if (joints) CK(cudaMemcpyAsync(joints, djoint, 60 * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (kc) CK(cudaMemcpyAsync(kc, dkc, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return HP_OK;
}

// ---------------------------------------------------------------------------------------
// PSO driver
// ---------------------------------------------------------------------------------------
static hp_status validate_pso(hp_ctx* ctx, const hp_pso_params* p) {
  ARG(p, "pso: NULL params");
  ARG(p->particles >= 1 && p->particles <= ctx->max_n, "pso: particles < 1 or > max_particles");
  ARG(!sharded(ctx) || p->particles >= ctx->world, "pso: sharded fit needs particles >= world");
  ARG(p->generations >= 1, "pso: generations < 1");
  ARG(p->c1 + p->c2 > 4.0, "pso: c1 + c2 must exceed 4 (P:L150 constriction)");
  ARG(p->mutation_fraction >= 0.0 && p->mutation_fraction <= 1.0, "pso: mutation_fraction");
  ARG(p->mutation_period >= 0, "pso: mutation_period < 0");
  ARG(p->mutation_after_eval == 0 || p->mutation_after_eval == 1,
      "pso: mutation_after_eval must be 0 or 1");
  return HP_OK;
}

static PsoDev pso_dev(hp_ctx* ctx, int N, int D, const hp_pso_params* p, int mut_lo, int mut_hi) {
  PsoDev d{};
  d.N = N;
  d.D = D;
  d.K = p->generations;
  d.period = p->mutation_period;
  d.per_dim_r = p->per_dim_r ? 1 : 0;
  d.nmut = (int)floor((double)N * p->mutation_fraction);
  d.mut_lo = mut_lo;
  d.mut_hi = mut_hi;
  d.mut_after = p->mutation_after_eval;
  d.dyn = ctx->dyn;
  d.lo = ctx->bnd;
  d.hi = ctx->bnd + 64;
  d.ilo = ctx->bnd + 128;
  d.ihi = ctx->bnd + 192;
  d.X = ctx->X;
  d.V = ctx->V;
  d.P = ctx->P;
  d.Pc = ctx->Pc;
  d.E = ctx->E;
  d.G = ctx->G;
  d.Gc = ctx->Gc;
  d.trace = ctx->trace;
  d.mark = ctx->mark;
  d.pimp = ctx->pimp;
  d.gsel = ctx->gsel;
  d.done = ctx->flags;
  d.gens_run = ctx->flags + 1;
  return d;
}

// Enqueue the whole fit on `s` (captured into a graph by the caller).
static hp_status enqueue_fit(hp_ctx* ctx, const PsoDev& d, bool sphere, cudaStream_t s,
                             int64_t* launches, bool exact) {
  int64_t n = 0;
  CK(launch_pso_init(d, s));
  n++;
  if (sphere) {  // test objective: standalone update / evaluate / bookkeeping kernels
    CK(launch_sphere_eval(d, ctx->centre, s));
    CK(launch_pso_book(d, 0, s));
    n += 2;
    for (int k = 1; k < d.K; k++) {
      CK(launch_pso_update(d, k, s));
      CK(launch_sphere_eval(d, ctx->centre, s));
      CK(launch_pso_book(d, k, s));
      n += 3;
    }
  } else if (sharded(ctx)) {
    // sharded hand fit: every rank updates ALL particles (identical bits everywhere),
    // scores its slice, allgathers the costs, and runs the identical bookkeeping
    const int64_t chunk = (d.N + ctx->world - 1) / ctx->world;
    int64_t b, e;
    shard_range(d.N, ctx->rank, ctx->world, &b, &e);
    EvalArgs a = base_args(ctx);
    a.persist_grid = 0;
    a.n = (int)(e - b);
    a.S = hp_splits_for(ctx, e - b);
    a.poses = d.X + b * d.D;
    a.costs64 = ctx->gat64 + ctx->rank * chunk;
    a.done = d.done;
    for (int k = 0; k < d.K; k++) {
      if (k >= 1) {
        CK(launch_pso_update(d, k, s));
        n++;
      }
      if (e > b) {
        CK(launch_eval(a, true, kModeCost, &ctx->tmap, s));
        n++;
      }
      hp_status gr = allgather(ctx, ctx->gat64, chunk, kNcclFloat64, s);
      if (gr != HP_OK) return gr;
      CK(launch_pso_book(d, k, s));
      n++;
    }
  } else {
    // the hand: ONE kernel per generation — PSO update (k >= 1) fused before FK in every
    // CTA, bookkeeping fused into the grid's last CTA; X, V double-buffered by parity
    EvalArgs a = base_args(ctx);
    a.persist_grid = 0;
    a.n = d.N;
    a.S = hp_splits_for(ctx, d.N);
    a.costs64 = d.E;
    a.done = d.done;
    a.pso_on = 1;
    a.pso = d;
    a.gcount = ctx->gcount;
    a.kc_g = ctx->kc_g;
    // speculative: generation kernels without the near-plane code; a particle that needs it
    // sets flags[2] and run_fit repeats the fit with the exact kernels
    a.near_seen = exact ? nullptr : ctx->flags + 2;
    a.pdl = ctx->use_pdl;
    double* Xb[2] = {ctx->X, ctx->X2};
    double* Vb[2] = {ctx->V, ctx->V2};
    for (int k = 0; k < d.K; k++) {
      a.pso_k = k;
      a.poses = Xb[0];
      a.x_in = Xb[(k + 1) & 1];
      a.v_in = Vb[(k + 1) & 1];
      a.x_out = Xb[k & 1];
      a.v_out = Vb[k & 1];
      CK(launch_eval(a, true, kModeCost, &ctx->tmap, s));
      n++;
    }
  }
  *launches = n;
  return HP_OK;
}

// The persistent fit (k_fit) applies: the fused hand fit, unsharded, one CTA of 32 warps per
// SM resident, and N particles x S >= 1 splits within the SMs.  Returns the split count.
static int fit_persist_splits(hp_ctx* ctx, int N) {
  if (!ctx->fit_persist || ctx->use_tma != 1 || N < 1 || N > ctx->sm_count) return 0;
  if (fit_blocks_per_sm(ctx->camp, N) < 1) return 0;
  return ctx->sm_count / N;
}

static hp_status enqueue_fit_persist(hp_ctx* ctx, const PsoDev& d, int S, cudaStream_t s,
                                     bool exact) {
  EvalArgs a = base_args(ctx);
  a.persist_grid = 0;
  a.n = d.N;
  a.S = S;
  a.pso = d;
  a.near_seen = exact ? nullptr : ctx->flags + 2;
  CK(cudaMemsetAsync(ctx->fit_bar, 0, sizeof(unsigned int), s));
  CK(cudaMemsetAsync(ctx->flags, 0, 3 * sizeof(int), s));  // done, gens_run, near seen
  CK(launch_fit(a, &ctx->tmap, exact, s));
  return HP_OK;
}

static hp_status run_fit(hp_ctx* ctx, const hp_pso_params* p, int D, const double* lo,
                         const double* hi, const double* ilo, const double* ihi, int mut_lo,
                         int mut_hi, bool sphere, double* best, double* best_cost, double* trace,
                         int32_t* gens_run, cudaStream_t user) {
  const int N = p->particles, K = p->generations;
  cudaStream_t s = ctx->st;
  if (K > ctx->trace_cap) {
    if (ctx->trace) cudaFree(ctx->trace);
    if (ctx->h_out) cudaFreeHost(ctx->h_out);
    ctx->trace = nullptr;
    ctx->h_out = nullptr;
    CK(cudaMalloc(&ctx->trace, (size_t)K * sizeof(double)));
    CK(cudaMallocHost(&ctx->h_out, (size_t)(K + 72) * sizeof(double)));
    ctx->trace_cap = K;
    if (ctx->graph.exec) {
      cudaGraphExecDestroy(ctx->graph.exec);
      ctx->graph.exec = nullptr;
    }
  }
  // per-fit parameters into device memory (the captured graph reads them); pageable
  // source: cudaMemcpyAsync stages it before returning
  std::vector<double> hbv(256, 0.0);
  for (int i = 0; i < D; i++) {
    hbv[i] = lo[i];
    hbv[64 + i] = hi[i];
    hbv[128 + i] = ilo[i];
    hbv[192 + i] = ihi[i];
  }
  PsoDyn dyn{p->seed, p->c1, p->c2, 0.0, p->stop_threshold};
  {
    const double psi = p->c1 + p->c2;  // w = 2 / |2 - psi - sqrt(psi^2 - 4 psi)|
    dyn.w = 2.0 / fabs(2.0 - psi - sqrt(psi * psi - 4.0 * psi));
  }
  CK(cudaEventRecord(ctx->ev, user));
  CK(cudaStreamWaitEvent(s, ctx->ev, 0));
  CK(cudaMemcpyAsync(ctx->bnd, hbv.data(), 256 * sizeof(double), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(ctx->dyn, &dyn, sizeof dyn, cudaMemcpyHostToDevice, s));
  PsoDev d = pso_dev(ctx, N, D, p, mut_lo, mut_hi);
  if (sharded(ctx) && !sphere) {
    if ((N + ctx->world - 1) / ctx->world > ctx->gat_cap) {
      ctx->err = "sharded fit: particles exceed max_particles * world";
      return HP_ERR_INVALID_ARG;
    }
    d.E = ctx->gat64;  // costs arrive through the allgather
  }
  Graph& g = ctx->graph;
  // the fused hand fit runs speculatively without the near-plane code first (exact = 0);
  // only if some particle needed it is the whole fit repeated with the exact kernels
  // (same seed: the same trajectory, now exact).  Sphere / sharded fits never use it.
  const bool fused = !sphere && !sharded(ctx);
  double* ho = ctx->h_out;
  int64_t launches = 0, total_launches = 0;
  // the persistent fit: one cooperative kernel (speculative without the near-plane code);
  // should a particle need that code, the fit is repeated on the exact generation kernels
  const int fitS = fused && D == kNdof ? fit_persist_splits(ctx, N) : 0;
  ctx->last_persist = 0;
  if (fitS > 0) {
    hp_status r = enqueue_fit_persist(ctx, d, fitS, s, false);
    if (r != HP_OK) return r;
    CK(cudaMemcpyAsync(ho, ctx->G, D * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ho + 64, ctx->Gc, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ho + 65, ctx->flags + 1, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ho + 72, ctx->trace, K * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    total_launches = 1;
    int seen = 0;
    memcpy(&seen, reinterpret_cast<int*>(ho + 65) + 1, sizeof(int));
    ctx->last_persist = !seen;
  }
  for (int exact = fused ? 0 : 1; !ctx->last_persist; exact++) {
    if (fitS > 0 && !exact) continue;  // the speculative pass was the persistent one
    const bool same = g.exec && g.N == N && g.D == D && g.K == K && g.period == d.period &&
                      g.per_dim_r == d.per_dim_r && g.nmut == d.nmut &&
                      g.mut_lo == mut_lo && g.mut_hi == mut_hi && g.sphere == (int)sphere &&
                      g.mut_after == d.mut_after &&
                      g.world == ctx->world && g.exact == exact;
#if HP_LOOPBACK_TEST
    if (ctx->loop) {  // debug loopback ranks: eager launches (host barriers between them)
      hp_status r = enqueue_fit(ctx, d, sphere, s, &launches, exact != 0);
      if (r != HP_OK) return r;
    } else
#endif
    if (!same) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
      cudaGraph_t graph;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      hp_status r = enqueue_fit(ctx, d, sphere, s, &launches, exact != 0);
      cudaError_t ce = cudaStreamEndCapture(s, &graph);
      if (r != HP_OK) return r;
      CK(ce);
      CK(cudaGraphInstantiate(&g.exec, graph, 0));
      ctx->last_fit_launches = launches;
      cudaGraphDestroy(graph);
      g.N = N;
      g.D = D;
      g.K = K;
      g.period = d.period;
      g.per_dim_r = d.per_dim_r;
      g.nmut = d.nmut;
      g.mut_lo = mut_lo;
      g.mut_hi = mut_hi;
      g.sphere = sphere;
      g.mut_after = d.mut_after;
      g.world = ctx->world;
      g.exact = exact;
    } else {
      launches = ctx->last_fit_launches;
    }
    if (!exact) CK(cudaMemsetAsync(ctx->flags + 2, 0, sizeof(int), s));
#if HP_LOOPBACK_TEST
    if (!ctx->loop)
#endif
      CK(cudaGraphLaunch(g.exec, s));
    CK(cudaMemcpyAsync(ho, ctx->G, D * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ho + 64, ctx->Gc, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ho + 65, ctx->flags + 1, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ho + 72, ctx->trace, K * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    total_launches += launches;
    int seen = 0;
    memcpy(&seen, reinterpret_cast<int*>(ho + 65) + 1, sizeof(int));
    if (exact || !seen) break;
  }
  launches = total_launches;  // both passes when the speculative one had to be repeated
  ctx->last_launches = launches;
  ctx->last_N = N;
  ctx->last_D = D;
  memcpy(best, ho, D * sizeof(double));
  *best_cost = ho[64];
  int gr = 0;
  memcpy(&gr, ho + 65, sizeof(int));
  if (gens_run) *gens_run = gr;
  ctx->last_gens = gr;
  ctx->last_fused = !sphere && !sharded(ctx);
  if (trace) {
    for (int k = 0; k < K; k++) trace[k] = k < gr ? ho[72 + k] : ho[72 + gr - 1];
  }
  return HP_OK;
}

hp_status hp_pso_fit(hp_ctx* ctx, const hp_pso_params* p, double* best_pose, double* best_cost,
                     double* trace, int32_t* gens_run, void* stream) {
  ARG(ctx, "hp_pso_fit: NULL ctx");
  hp_status r = validate_pso(ctx, p);
  if (r != HP_OK) return r;
  ARG(best_pose && best_cost, "hp_pso_fit: NULL output");
  cudaSetDevice(ctx->device);
  double lo[26], hi[26], ilo[26], ihi[26];
  hp_bounds(lo, hi);
  for (int i = 0; i < 26; i++) {
    ilo[i] = lo[i];
    ihi[i] = hi[i];
    if (p->init_center && p->init_radius) {  // centre +- radius intersected with the bounds
      ilo[i] = fmax(lo[i], p->init_center[i] - p->init_radius[i]);
      ihi[i] = fmin(hi[i], p->init_center[i] + p->init_radius[i]);
    }
  }
  return run_fit(ctx, p, 26, lo, hi, ilo, ihi, 6, 26, false, best_pose, best_cost, trace,
                 gens_run, (cudaStream_t)stream);
}

hp_status hp_track(hp_ctx* ctx, const float* depth_seq, const uint8_t* mask_seq,
                   int32_t frames, int32_t on_device, const hp_pso_params* p,
                   const double* track_radius, double* poses_out, double* costs_out,
                   double* traces_out, void* stream) {
  ARG(ctx && depth_seq && mask_seq && p && track_radius && poses_out,
      "hp_track: NULL argument");
  ARG(frames >= 0, "hp_track: frames < 0");
  hp_status r = validate_pso(ctx, p);
  if (r != HP_OK) return r;
  const size_t npx = (size_t)ctx->cam.width * ctx->cam.height;
  hp_pso_params q = *p;
  double centre[26];
  for (int32_t f = 0; f < frames; f++) {
    r = hp_set_observation(ctx, depth_seq + f * npx, mask_seq + f * npx, on_device, stream);
    if (r != HP_OK) return r;
    q.seed = p->seed + (uint64_t)f;  // one independent Philox stream per frame
    if (f > 0) {  // warm start: the previous frame's best pose +- track_radius
      q.init_center = centre;
      q.init_radius = track_radius;
    }
    double cost;
    r = hp_pso_fit(ctx, &q, poses_out + 26 * (size_t)f, &cost,
                   traces_out ? traces_out + (size_t)f * p->generations : nullptr, nullptr,
                   stream);
    if (r != HP_OK) return r;
    if (costs_out) costs_out[f] = cost;
    memcpy(centre, poses_out + 26 * (size_t)f, sizeof centre);
  }
  return HP_OK;
}

hp_status hp_debug_pso_sphere(hp_ctx* ctx, int32_t D, const double* lo, const double* hi,
                              const double* init_lo, const double* init_hi, int32_t mut_lo,
                              int32_t mut_hi, const double* centre, const hp_pso_params* p,
                              double* best_x, double* best_cost, double* trace,
                              int32_t* gens_run, void* stream) {
  ARG(ctx, "hp_debug_pso_sphere: NULL ctx");
  hp_status r = validate_pso(ctx, p);
  if (r != HP_OK) return r;
  ARG(D >= 1 && D <= 64 && lo && hi && init_lo && init_hi && centre && best_x && best_cost,
      "hp_debug_pso_sphere: bad argument");
  ARG(mut_lo >= 0 && mut_lo <= mut_hi && mut_hi <= D, "hp_debug_pso_sphere: mutation dims");
  cudaSetDevice(ctx->device);
  CK(cudaMemcpyAsync(ctx->centre, centre, D * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  return run_fit(ctx, p, D, lo, hi, init_lo, init_hi, mut_lo, mut_hi, true, best_x, best_cost,
                 trace, gens_run, (cudaStream_t)stream);
}

hp_status hp_pso_state(hp_ctx* ctx, int32_t particles, int32_t D, double* X, double* V,
                       double* P, double* Pcost) {
  ARG(ctx, "hp_pso_state: NULL ctx");
  if (ctx->last_N == 0) {
    ctx->err = "hp_pso_state: no fit has run";
    return HP_ERR_STATE;
  }
  ARG(particles == ctx->last_N && D == ctx->last_D,
      "hp_pso_state: particles / D differ from the last fit's (the buffers' capacity)");
  cudaSetDevice(ctx->device);
  const size_t nd = (size_t)ctx->last_N * ctx->last_D * sizeof(double);
  // the fused hand fit double-buffers X, V: generation g lives in buffer g & 1
  const bool second = ctx->last_fused && !ctx->last_persist && ((ctx->last_gens - 1) & 1);
  if (X) CK(cudaMemcpy(X, second ? ctx->X2 : ctx->X, nd, cudaMemcpyDeviceToHost));
  if (V) CK(cudaMemcpy(V, second ? ctx->V2 : ctx->V, nd, cudaMemcpyDeviceToHost));
  if (P) CK(cudaMemcpy(P, ctx->P, nd, cudaMemcpyDeviceToHost));
  if (Pcost) CK(cudaMemcpy(Pcost, ctx->Pc, ctx->last_N * sizeof(double), cudaMemcpyDeviceToHost));
  return HP_OK;
}

hp_status hp_shard_range(int64_t n, int32_t rank, int32_t world, int64_t* begin, int64_t* end) {
  hp_ctx* ctx = nullptr;
  ARG(begin && end && n >= 0 && world >= 1 && rank >= 0 && rank < world,
      "hp_shard_range: bad argument");
  shard_range(n, rank, world, begin, end);
  return HP_OK;
}

hp_status hp_nccl_available(int32_t* available) {
  if (!available) return HP_ERR_INVALID_ARG;
  *available = nccl_api() != nullptr;
  return HP_OK;
}

hp_status hp_get_nccl_id(uint8_t* id) {
  hp_ctx* ctx = nullptr;
  ARG(id, "hp_get_nccl_id: NULL id");
  NcclApi* api = nccl_api();
  if (!api) {
    g_err = "hp_get_nccl_id: libnccl.so.2 not found (set HP_NCCL_LIB)";
    return HP_ERR_NCCL;
  }
  ncclUniqueId u;
  const ncclResult_t r = api->getUniqueId(&u);
  if (r != 0) {
    g_err = std::string("ncclGetUniqueId: ") + api->errorString(r);
    return HP_ERR_NCCL;
  }
  memcpy(id, u.internal, 128);
  return HP_OK;
}

static hp_status shard_buffers(hp_ctx* ctx, int rank, int world);

hp_status hp_shard(hp_ctx* ctx, const uint8_t* id, int32_t rank, int32_t world) {
  ARG(ctx && id, "hp_shard: NULL argument");
  ARG(world >= 1 && rank >= 0 && rank < world, "hp_shard: bad rank/world");
  if (sharded(ctx)) {
    ctx->err = "hp_shard: context is already sharded";
    return HP_ERR_STATE;
  }
  NcclApi* api = nccl_api();
  if (!api) {
    ctx->err = "hp_shard: libnccl.so.2 not found (set HP_NCCL_LIB)";
    return HP_ERR_NCCL;
  }
  cudaSetDevice(ctx->device);
  ncclUniqueId u;
  memcpy(u.internal, id, 128);
  const ncclResult_t r = api->commInitRank(&ctx->comm, world, u, rank);
  if (r != 0) {
    ctx->comm = nullptr;
    ctx->err = std::string("ncclCommInitRank: ") + api->errorString(r);
    return HP_ERR_NCCL;
  }
  return shard_buffers(ctx, rank, world);
}

#if HP_LOOPBACK_TEST
// Debug builds only (see LoopGroup): join loopback group `group` as rank/world.  Every
// member is a context on the same device, driven by its own host thread.
hp_status hp_shard_loopback(hp_ctx* ctx, const char* group, int32_t rank, int32_t world) {
  ARG(ctx && group, "hp_shard_loopback: NULL argument");
  ARG(world >= 1 && rank >= 0 && rank < world, "hp_shard_loopback: bad rank/world");
  if (sharded(ctx)) {
    ctx->err = "hp_shard_loopback: context is already sharded";
    return HP_ERR_STATE;
  }
  cudaSetDevice(ctx->device);
  LoopGroup* g;
  {
    std::lock_guard<std::mutex> lk(g_loop_m);
    LoopGroup*& slot = g_loop[group];
    if (!slot) {
      slot = new LoopGroup();
      slot->world = world;
      slot->buf.assign(world, nullptr);
      slot->ready.assign(world, nullptr);
      slot->read.assign(world, nullptr);
    }
    g = slot;
  }
  ARG(g->world == world, "hp_shard_loopback: world differs from the group's");
  CK(cudaEventCreateWithFlags(&g->ready[rank], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&g->read[rank], cudaEventDisableTiming));
  ctx->loop = g;
  return shard_buffers(ctx, rank, world);
}
#endif

static hp_status shard_buffers(hp_ctx* ctx, int rank, int world) {
  ctx->rank = rank;
  ctx->world = world;
  ctx->gat_cap = ctx->max_n;  // chunk <= max_particles
  const size_t cap = (size_t)ctx->gat_cap * world;
  CK(cudaMalloc(&ctx->gat32, cap * sizeof(float)));
  CK(cudaMalloc(&ctx->gat64, cap * sizeof(double)));
  // host staging for the full gathered cost vector of hp_eval_costs_host
  cudaFreeHost(ctx->h_costs);
  ctx->h_costs = nullptr;
  CK(cudaMallocHost(&ctx->h_costs, cap * sizeof(float)));
  if (ctx->graph.exec) {
    cudaGraphExecDestroy(ctx->graph.exec);
    ctx->graph.exec = nullptr;
  }
  return HP_OK;
}

}  // extern "C"
