/*
 * hp.h — C ABI of the B200-native swarm scorer for arXiv 2005.07068
 * ("Recognition of 26 Degrees of Freedom of Hands Using Model-based approach and
 * Depth-Color Images").  Library: paper_2005_07068_b200/libhp.so (sm_100a).
 *
 * Citations: P:Lnn = /root/reference/PAPER.md line nn; DESIGN §n = /root/repo/DESIGN.md.
 *
 * Conventions for every entry point
 *  - Every function returns hp_status; no exception or exit crosses the ABI.  On failure
 *    the message is available from hp_last_error(ctx) (thread-local global text when ctx
 *    is NULL or creation failed).
 *  - Units: mm for positions and depths, radians for angles, depth 0 = undefined.
 *  - Pose layout (Eq. (1)-(3); flattening order S:L122): 26 values
 *    [x_c, y_c, z_c, th_x, th_y, th_z, then thumb, index, middle, ring, little each
 *    (th_MP^x, th_MP^z, th_PIP, th_DIP)], row-major [N][26].
 *  - Streams: `stream` is a cudaStream_t (passed as void*; NULL = the legacy default
 *    stream).  Device-pointer calls are enqueued on it and return without synchronising
 *    unless stated otherwise.
 *  - Ownership: the context owns its device workspace (sized by max_particles at
 *    creation) and a copy of the observation.  Caller buffers are only read/written
 *    during the call (host pointers) or until the enqueued work completes (device
 *    pointers); the library never frees or retains them.
 *  - Threads: one host thread per context at a time; distinct contexts are independent.
 *  - There is no CPU fallback: without a usable sm_100 device hp_create fails.
 */
#ifndef HP_H
#define HP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HP_NDOF 26  /* Eq. (3): h = (q_i, q_c), 5 x 4 finger angles + 6 wrist DOF */
#define HP_NPRIM 38 /* 3 palm + 5 x (3 segments + 4 spheres) */
#define HP_REC_FLOATS 24

typedef struct hp_ctx hp_ctx;

typedef enum {
  HP_OK = 0,
  HP_ERR_INVALID_ARG = 1, /* null pointer, bad size, bad parameter (see each call) */
  HP_ERR_CUDA = 2,        /* a CUDA runtime / driver call failed                   */
  HP_ERR_OOM = 3,         /* device or pinned-host allocation failed               */
  HP_ERR_NCCL = 4,        /* NCCL failure in the sharded mode                      */
  HP_ERR_STATE = 5,       /* call not valid in the context's current state         */
  HP_ERR_NO_DEVICE = 6    /* no sm_100 device / library built for another arch     */
} hp_status;

/* Camera C ("focal length and viewing direction"): pinhole, pixel (u, v) casts the
 * ray d = ((u + 0.5 - cx)/fx, (v + 0.5 - cy)/fy, 1); depth = camera z.  The per-pixel
 * arithmetic is fp32.  Errors: width/height < 1, fx/fy <= 0, !(0 < z_near < z_far). */
typedef struct {
  int32_t width, height;
  float fx, fy, cx, cy;
  float z_near_mm, z_far_mm;
} hp_intrinsics;

/* Hand model dimensions ("measured from a real hand"; values DESIGN §2). */
typedef struct {
  float palm_half_w, palm_half_t, palm_len, palm_cap_half_len;
  float base[5][3];    /* MCP centres in the hand frame H             */
  float seg_len[5][3]; /* L1, L2, L3                                  */
  float radius[5][4];  /* joint spheres MCP, PIP, DIP, tip            */
  float thumb_ell_x, thumb_ell_z;       /* thumb proximal ellipsoid cross semi-axes */
  float thumb_yaw_deg, thumb_pitch_deg; /* R_T0 = Rz(yaw) Ry(pitch)                 */
} hp_hand_dims;

/* Eq. (4)-(5) constants and readings. */
typedef struct {
  double d_m;         /* r_m threshold, mm (10)                           */
  double d_M;         /* numerator clamp, mm (40) — AMB-1                 */
  double lambda;      /* area weight (20)                                 */
  double lambda_k;    /* collision weight (10)                            */
  double depth_scale; /* mm -> cm (0.1) — AMB-2                           */
  double kc_rest;     /* rho in phi = MPz(radial) - MPz(ulnar) + rho (0)  */
  int32_t clamp_at_dm;/* 1 = literal Eq. (4) clamp at d_m                 */
} hp_cost_params;

/* PSO (Eq. (6)-(7)); DESIGN §4. */
typedef struct {
  uint64_t seed;
  int32_t particles;       /* >= 1 and <= max_particles (paper: 64)   */
  int32_t generations;     /* >= 1 (paper: 30)                        */
  int32_t mutation_period; /* >= 0, 0 = off (paper: 3)                */
  int32_t per_dim_r;       /* 0: scalar r1, r2 per particle (AMB-15)          */
  double c1, c2;           /* c1 + c2 > 4 (paper: 2.8, 1.3)           */
  double mutation_fraction;/* [0, 1] (paper: 0.5)                             */
  double stop_threshold;   /* stop when G's cost < this; -INFINITY = off      */
  const double* init_center; /* host [26] or NULL: init box = centre +- radius  */
  const double* init_radius; /* host [26] or NULL   intersected with Tables 1-2 */
  /* Mutation order (P:L152 is silent; DESIGN.md AMB-17): 0 (default) = the worst particles
   * are re-drawn right after the Eq. (6)-(7) update of generations k = period, 2 period, ...
   * and evaluated as drawn; 1 = SPEC's order: re-drawn after generation k's
   * evaluation and bookkeeping, so generation k + 1's update moves them before they are
   * evaluated.  Errors: any other value. */
  int32_t mutation_after_eval;
} hp_pso_params;

/* Fill with the defaults of DESIGN §2 / P:L130 / P:L148-152.  Errors: NULL. */
hp_status hp_default_dims(hp_hand_dims* out);
hp_status hp_default_cost(hp_cost_params* out);
hp_status hp_default_pso(hp_pso_params* out);
/* AMB-12 Kinect-like intrinsics for a width x height frame (fx = 525 * width / 640). */
hp_status hp_default_intrinsics(int32_t width, int32_t height, hp_intrinsics* out);
/* Tables 1-2 in pose units (rad, mm), host arrays of 26. */
hp_status hp_bounds(double lo[26], double hi[26]);

/* Create a context on `device` (the current CUDA device if < 0) with a workspace for up
 * to max_particles poses per call.  dims/cost may be NULL (defaults).  The observation
 * starts empty (all undefined); set it with hp_set_observation.
 * Reading of the north star's hp_create(observation, intrinsics, model dims): creation and
 * the observation are two calls here, so one context (its device workspace, ray table and
 * captured fit graph) serves a whole frame sequence — hp_set_observation replaces the
 * frame in place (row f1 tracking, row f3 ingestion) without re-creating anything;
 * hp_create followed by hp_set_observation is the north star's call.
 * Errors: INVALID_ARG (NULL out/cam, bad intrinsics, max_particles < 1, an image whose
 * ray table (width + 4 height + 80 floats) exceeds 64 KB of shared memory), NO_DEVICE, OOM. */
hp_status hp_create(const hp_intrinsics* cam, const hp_hand_dims* dims,
                    const hp_cost_params* cost, int32_t max_particles, int32_t device,
                    hp_ctx** out);

/* Observation O = (O_s, O_d): depth [H][W] fp32 mm (0, negative or non-finite =
 * undefined) and skin mask [H][W] u8 (nonzero = hand).  Both host (on_device = 0) or both
 * device (on_device = 1) pointers, row-major, no padding.  The context copies and packs
 * them into one u32 per pixel and computes S_o = sum o_s (DESIGN §1 row A0); the caller
 * may free its buffers when the call returns (the call synchronises `stream`).
 * Errors: INVALID_ARG (NULL ctx/depth/mask), CUDA. */
hp_status hp_set_observation(hp_ctx* ctx, const float* depth_mm, const uint8_t* mask,
                             int32_t on_device, void* stream);

/* Frame-batched observations (M frames x N particles per call, the
 * per-particle parallelism of P:L162 extended over a batch of observations): depth
 * [frames][H][W] fp32 and mask [frames][H][W] u8, same conventions as hp_set_observation,
 * which is this call with frames = 1.  Replaces the current observation(s); buffers grow
 * on demand (growing synchronises the device and rebuilds the cached fit graph).  Plain
 * hp_eval_costs / hp_pso_fit / hp_track score frame 0.
 * Errors: INVALID_ARG (NULL pointers, frames < 1), OOM, CUDA. */
hp_status hp_set_observations(hp_ctx* ctx, const float* depth_mm, const uint8_t* mask,
                              int32_t frames, int32_t on_device, void* stream);

/* Kinect-like observation front end.  P:L92: "skin colour detection
 * and depth segmentation extract the hand region ... O = (O_s, O_d)".  Readings DESIGN.md
 * AMB-33..36: with valid = d > 0 and band = [lo_mm, hi_mm] (mode 0) or [m, m + width_mm]
 * (mode 1, m = the nearest valid depth among skin pixels, or among all pixels without a skin
 * image; no candidate = empty band), in_band = valid && lo <= d <= hi:
 *   O_s = skin ? skin && (!valid || in_band) : in_band
 *   O_d = keep_background ? (valid ? d : 0) : (in_band ? d : 0)
 * Integer mm limits, inclusive: bit-exact with the oracle's or_segment. */
typedef struct {
  int32_t mode;            /* 0 fixed band, 1 nearest-object band (default) */
  int32_t lo_mm, hi_mm;    /* mode 0 */
  int32_t width_mm;        /* mode 1 (default 250) */
  int32_t keep_background; /* 1: O_d keeps every valid depth (default 0) */
} hp_segment_params;
hp_status hp_default_segment(hp_segment_params* out);
/* depth_mm [frames][H][W] u16 (Kinect mm, 0 = no reading), skin [frames][H][W] u8 or NULL,
 * host (on_device = 0) or device pointers; seg NULL = defaults.  Segments, packs and sets
 * `frames` observation frames (as hp_set_observations).  band_out (host [frames][2], may be
 * NULL) receives each frame's band.  Synchronises `stream`.
 * Errors: INVALID_ARG (NULL ctx/depth, frames < 1, mode not 0/1, width_mm < 0), OOM, CUDA. */
hp_status hp_set_observation_kinect(hp_ctx* ctx, const uint16_t* depth_mm, const uint8_t* skin,
                                    int32_t frames, const hp_segment_params* seg,
                                    int32_t on_device, int32_t* band_out, void* stream);
/* Unpack observation frame `frame` into device buffers depth [H][W] fp32 (0 = undefined) and
 * mask [H][W] u8 (either may be NULL).  Async.  Errors: INVALID_ARG (frame out of range). */
hp_status hp_get_observation(hp_ctx* ctx, int32_t frame, float* depth_dev, uint8_t* mask_dev,
                             void* stream);

/* Simulation protocol: render pose h_ref (host fp64 [26]) with this context's
 * camera and model into depth_dev [H][W] fp32 (0 = no hit) and mask_dev [H][W] u8
 * (silhouette), both device buffers (mask_dev may be NULL).  Async on `stream`. */
hp_status hp_render_observation(hp_ctx* ctx, const double* h_ref, float* depth_dev,
                                uint8_t* mask_dev, void* stream);

/* Objective E(h, O) = D(O, h, C) + lambda_k kc(h) (Eq. (4)-(5)) of n poses.
 * poses_dev: device fp32 [n][26]; costs_dev: device fp32 [n].  Poses are scored as given
 * (no clamping); non-finite poses give NaN.  n = 0 is a no-op.  Async on `stream`.
 * Errors: INVALID_ARG (NULL ctx/pointers with n > 0, n < 0 or n > max_particles). */
hp_status hp_eval_costs(hp_ctx* ctx, const float* poses_dev, int64_t n, float* costs_dev,
                        void* stream);

/* Frame-batched objective: poses_dev [frames][n_per_frame][26] fp32, pose i of block f
 * scored against observation frame f (hp_set_observations); costs_dev [frames][n_per_frame]
 * fp32.  `frames` states the caller's buffer layout and must equal the frame count of the
 * current observation.  Bitwise equal to scoring each block with hp_eval_costs against that
 * frame alone.  Local to this context even when sharded (frames shard across ranks with no
 * collective).  n_per_frame = 0 is a no-op.  Async on `stream`.
 * Errors: INVALID_ARG (frames != the observation's frame count, n_per_frame < 0,
 * frames * n_per_frame > max_particles, NULL). */
hp_status hp_eval_costs_frames(hp_ctx* ctx, const float* poses_dev, int32_t frames,
                               int64_t n_per_frame, float* costs_dev, void* stream);
/* Its test hook: the sums and fp64 costs of hp_eval_sums, frame-batched. */
hp_status hp_eval_sums_frames(hp_ctx* ctx, const float* poses_dev, int32_t frames,
                              int64_t n_per_frame, uint64_t* sums_dev, double* costs64_dev,
                              void* stream);

/* Same with HOST buffers: moves poses in, scores, moves costs out, then synchronises
 * `stream` (the end-to-end path a host application calls).  Mapped page-locked buffers
 * (cudaHostAlloc / torch pin_memory under unified addressing) are accessed by the kernels
 * directly — the FK kernel loads the poses and the cost finalisation stores the costs over
 * the host link, no separate copies (HP_NO_ZEROCOPY=1 in the environment: DMA copies
 * instead); other page-locked buffers are DMA'd directly; pageable ones are staged through
 * the context's pinned buffers (one extra host memcpy each way). */
hp_status hp_eval_costs_host(hp_ctx* ctx, const float* poses_host, int64_t n,
                             float* costs_host, void* stream);

/* Per-pose integer sums behind Eq. (4) (test hook, async): sums_dev [n][4] u64 =
 * (sum r_m, sum (o_s AND r_m), sum over both-defined pixels of rint(min(|o_d - r_d|,
 * clamp) * 2^q) * 2^(20 - q), number of both-defined pixels), i.e. the numerator in
 * 2^-20 mm units quantised per pixel to 2^-q mm, q = the largest integer <= 20 with
 * clamp * 2^q <= 2^22 (16 for the default 40 mm clamp); costs64_dev [n] fp64 may be NULL. */
hp_status hp_eval_sums(hp_ctx* ctx, const float* poses_dev, int64_t n, uint64_t* sums_dev,
                       double* costs64_dev, void* stream);
/* The same for fp64 poses (device [n][26], the precision of the PSO state):
 * exactly the scoring a fit's generation applies to its particles, so a host PSO fed these
 * costs retraces hp_pso_fit (the "PSO-step parity" check of DESIGN §6).  sums_dev or
 * costs64_dev may be NULL (not both).  Async.  Errors: as hp_eval_sums. */
hp_status hp_eval_sums_f64(hp_ctx* ctx, const double* poses_dev, int64_t n,
                           uint64_t* sums_dev, double* costs64_dev, void* stream);

/* Full PSO fit on the GPU: init, K generations of update +
 * mutation + evaluation + bookkeeping captured in one CUDA graph, one device->host copy at
 * the end.  Synchronous.  Outputs (host): best_pose [26] (G), best_cost (its E), trace
 * [generations] (G's cost after each generation; entries after an early stop repeat the
 * last value, may be NULL), gens_run (may be NULL).
 * Errors: INVALID_ARG (particles < 1 or > max_particles, generations < 1, c1 + c2 <= 4,
 * mutation_fraction outside [0, 1], mutation_period < 0, NULL outputs), CUDA. */
hp_status hp_pso_fit(hp_ctx* ctx, const hp_pso_params* params, double* best_pose,
                     double* best_cost, double* trace, int32_t* gens_run, void* stream);

/* Temporal tracking over a frame sequence (SPEC S:L568-576 warm
 * start): frame f's observation (depth_seq / mask_seq [frames][H][W], host or device as
 * on_device says) is fitted with hp_pso_fit, seed = params->seed + f; frame 0 uses the
 * params' init box, frame f > 0 the box previous best pose +- track_radius[26] (host)
 * intersected with Tables 1-2.  Outputs (host): poses_out [frames][26], costs_out
 * [frames] and traces_out [frames][generations] (both may be NULL).  Synchronous.
 * Errors: as hp_set_observation and hp_pso_fit. */
hp_status hp_track(hp_ctx* ctx, const float* depth_seq, const uint8_t* mask_seq,
                   int32_t frames, int32_t on_device, const hp_pso_params* params,
                   const double* track_radius, double* poses_out, double* costs_out,
                   double* traces_out, void* stream);

/* Final swarm state of the last hp_pso_fit / hp_debug_pso_sphere (host, synchronous):
 * X, V, P [particles][D] and Pcost [particles]; any pointer may be NULL.  particles and D
 * state the buffers' capacity and must equal the last fit's.
 * Errors: STATE (no fit has run), INVALID_ARG (particles / D differ). */
hp_status hp_pso_state(hp_ctx* ctx, int32_t particles, int32_t D, double* X, double* V,
                       double* P, double* Pcost);

/* ---- test hooks ------------------------------------------------------------------- */
/* FK of one host fp64 pose on the device (the same device function hp_eval_costs runs):
 * records [38][24] fp32 (layout DESIGN §9), boxes [38][4] int32 (x0, y0, x1, y1 inclusive,
 * x0 > x1 = empty), joints [5][4][3] fp64 camera-frame joint centres, kc (fp64).  Any
 * output may be NULL.  Synchronous. */
hp_status hp_debug_fk(hp_ctx* ctx, const double* pose, float* records, int32_t* boxes,
                      double* joints, double* kc);
/* The FK output record k_fk_batch left for pose p of the last batch-path evaluation
 * (records [38][24] FAST layout, boxes [38][4]), host buffers, synchronous: the batch path's
 * FK against hp_debug_fk's. */
hp_status hp_debug_batch_fk(hp_ctx* ctx, int64_t p, float* records, int32_t* boxes);
/* Depth image [H][W] fp32 (device) of the pose pose_dev (device fp32 [26]) produced by
 * the same tile/culling/intersection code as hp_eval_costs.  Async. */
hp_status hp_debug_render(hp_ctx* ctx, const float* pose_dev, float* depth_dev, void* stream);
/* The PSO of hp_pso_fit on f(x) = sum_d (x_d - centre_d)^2 (fp64, left to right, no FMA)
 * over D <= 64 dims with bounds lo/hi, init box, mutation dims [mut_lo, mut_hi); host
 * arrays.  Same outputs as hp_pso_fit.  Synchronous. */
hp_status hp_debug_pso_sphere(hp_ctx* ctx, int32_t D, const double* lo, const double* hi,
                              const double* init_lo, const double* init_hi, int32_t mut_lo,
                              int32_t mut_hi, const double* centre, const hp_pso_params* params,
                              double* best_x, double* best_cost, double* trace,
                              int32_t* gens_run, void* stream);

/* ---- particle-sharded multi-GPU mode (one process per GPU) -------------
 * Only the particles shard: the observation is replicated, rank r scores poses
 * [r*ceil(N/W), min(N, (r+1)*ceil(N/W))) and NCCL allgathers the costs (over NVLink /
 * NVSwitch), so every rank holds all N costs.  In hp_pso_fit every rank then runs the
 * identical update of all particles and the identical bookkeeping, so G is known
 * everywhere without a broadcast and the result is bitwise independent of W (integer
 * pixel sums, fp64 swarm state).  NCCL is loaded at run time (libnccl.so.2, or the path in
 * HP_NCCL_LIB); single-GPU use never needs it. */
/* The slice of n poses owned by `rank` of `world` (host-only, no GPU needed). */
hp_status hp_shard_range(int64_t n, int32_t rank, int32_t world, int64_t* begin, int64_t* end);
/* 1 if libnccl.so.2 could be loaded. */
hp_status hp_nccl_available(int32_t* available);
/* A fresh NCCL unique id (128 bytes) on rank 0; broadcast it to the other ranks (the
 * Python binding uses torch.distributed).  Errors: NCCL. */
hp_status hp_get_nccl_id(uint8_t* id);
/* Collective: every rank calls it with the same id.  Afterwards hp_eval_costs takes the
 * FULL batch (n <= max_particles * world), scores this rank's slice and returns all n
 * costs on every rank; hp_pso_fit runs sharded (particles >= world).  If a rank's own
 * scoring fails it still takes part in the allgather (its peers do not hang) and then
 * returns the error.  Errors: INVALID_ARG, STATE (already sharded), NCCL, OOM.
 * Reading of the north star's hp_create_sharded: sharding is a call on an existing
 * context (hp_create + hp_shard), so the same context type serves both modes and the
 * unique-id exchange (torch.distributed in the binding) stays outside the library. */
hp_status hp_shard(hp_ctx* ctx, const uint8_t* id, int32_t rank, int32_t world);
/* DEBUG BUILDS ONLY (compiled with -DHP_LOOPBACK_TEST=1; the product library does not
 * export it): join an in-process loopback group of `world` contexts on ONE device, each
 * driven by its own host thread, instead of an NCCL communicator.  The allgather is done
 * with device copies at NCCL's offsets, ordered by events and a host barrier, so the
 * sharded code paths (rank > 0 slices, the padded last chunk, the sharded fit) can be
 * executed on a single-GPU box.  Errors: INVALID_ARG, STATE. */
hp_status hp_shard_loopback(hp_ctx* ctx, const char* group, int32_t rank, int32_t world);

/* Number of kernel launches the last hp_eval_costs / hp_pso_fit enqueued (bench).  A hand
 * fit first runs generation kernels without the near-plane code; if a particle needed it
 * the fit is repeated with the exact kernels and both passes are counted. */
int64_t hp_last_launch_count(const hp_ctx* ctx);
/* Per-launch device timing of the evaluation (bench.py's roofline leg).
   hp_set_timing(ctx, 1) makes every later hp_eval_costs / hp_eval_costs_host / hp_eval_sums
   record four CUDA events on the stream the kernels run on: before the first launch,
   between the launches of the batch path (k_fk_batch | k_render_persist | its near-plane
   pass), after the last. hp_last_kernel_ms waits for the last event and returns ms[0] =
   first launch (k_fk_batch; 0 on single-launch paths), ms[1] = the renderer / fused kernel
   alone, ms[2] = the near-plane pass (0 on single-launch paths).  HP_ERR_STATE if no timed
   evaluation was enqueued since timing was switched on.  Timing adds event records between
   the launches and launches the renderer after k_fk_batch has completed (no programmatic
   dependent launch, so its first poses skip the per-pose FK ready flags): ms[1] is the
   renderer alone, and the FK / render overlap of the untimed path is lost; leave it off
   outside measurement. */
hp_status hp_set_timing(hp_ctx* ctx, int32_t on);
hp_status hp_last_kernel_ms(hp_ctx* ctx, float ms[3]);

/* Split factor S (CTAs per particle) used for n poses. */
int32_t hp_splits_for(const hp_ctx* ctx, int64_t n);

const char* hp_last_error(const hp_ctx* ctx);
void hp_destroy(hp_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
