/*
 * oracle.h — the CPU oracle for the hand-pose swarm scorer of arXiv 2005.07068.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2005_07068_b200/,
 * include/, the CUDA library) may include, link, import or execute anything under
 * oracle/.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may call it.  It shares no code, header, table or constant
 * generator with the CUDA path; both implement DESIGN.md §2 ("frozen model") and
 * §3 ("readings") independently.
 *
 * Plain, slow, obviously correct: fp64 throughout, brute force over every pixel x
 * every primitive (an optional culled mode skips primitives whose conservative
 * screen box excludes the pixel and must be bitwise identical), no blocking, no
 * fusion.  Citations: P:Lnn = /root/reference/PAPER.md line nn (section, equation).
 *
 * Parity status (see DESIGN.md §6 for the pins that fix each function):
 *   or_philox4x32_10 ........ pinned (Random123 known-answer vectors)
 *   or_fk .................... pinned (closed-form joint positions, invariants)
 *   or_first_hit / or_render . pinned (analytic sphere depths, disk area, brute force)
 *   or_score / or_cost ....... pinned (worked 2x2 example, invariants, self-match 0)
 *   or_kc .................... pinned (closed-form pair examples)
 *   or_pso_run ............... pinned (w closed form, fixed point, sphere convergence; Eq. 6
 *                              coefficient / r1-r2 assignment by a hand-derived 2-particle
 *                              trajectory and the c2 = 0 / c1 = 0 limits; both mutation orders)
 *   or_edge_mask ............. pinned (the analytic silhouette / depth / r_m rings of an
 *                              on-axis sphere)
 *   or_pso_fit_hand .......... parity unpinned: the paper prints no trajectory (Figs. 6-9 absent)
 *   or_segment ............... pinned (recovers a rendered hand in front of a background
 *                              plane exactly; dropout / skin / empty-frame special cases)
 */
#ifndef HP_ORACLE_H
#define HP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_NDOF 26
#define OR_NPRIM 38

enum { OR_SPHERE = 0, OR_ELLIPSOID = 1, OR_CONE = 2, OR_CYLINDER = 3 };

/* Pinhole camera C: pixel (u,v) casts the ray d = ((u+0.5-cx)/fx, (v+0.5-cy)/fy, 1). */
typedef struct {
  int32_t width, height;
  double fx, fy, cx, cy;
  double z_near, z_far; /* mm; per-primitive hits outside [z_near, z_far] are discarded */
} or_camera;

/* Hand dimensions ("measured from a real hand", no numbers: DESIGN.md §2 table). */
typedef struct {
  double palm_half_w;      /* elliptic cylinder semi-axis along x_H (45)   */
  double palm_half_t;      /* elliptic cylinder semi-axis along z_H (15)   */
  double palm_len;         /* cylinder spans y_H in [-palm_len, 0] (80)    */
  double palm_cap_half_len;/* cap ellipsoid semi-axis along y_H (10)       */
  double base[5][3];       /* MCP joint centres in hand frame H            */
  double seg_len[5][3];    /* L1, L2, L3                                   */
  double radius[5][4];     /* joint sphere radii MCP, PIP, DIP, tip        */
  double thumb_ell_x;      /* thumb proximal ellipsoid semi-axis, local x (12) */
  double thumb_ell_z;      /* thumb proximal ellipsoid semi-axis, local z (10) */
  double thumb_yaw_deg;    /* R_T0 = Rz(yaw) Ry(pitch): 40, 90            */
  double thumb_pitch_deg;
} or_dims;

/* Eq. (4)/(5) constants and the readings of DESIGN.md §3. */
typedef struct {
  double d_m;          /* r_m match threshold, mm (10)                 */
  double d_M;          /* numerator clamp, mm (40)                     */
  double lambda;       /* area weight (20)                             */
  double lambda_k;     /* collision weight (10)                        */
  double depth_scale;  /* mm -> cm (0.1)                               */
  double kc_rest;      /* rho in phi = MPz(radial) - MPz(ulnar) + rho, rad (0) */
  int32_t clamp_at_dm; /* 1: literal Eq. (4) clamp at d_m instead of d_M */
} or_cost_params;

/* One placed primitive, camera frame, mm.
 *  SPHERE:    c = centre, s[0] = radius.
 *  ELLIPSOID: c = centre, R columns = local axes, s = semi-axes (local x, y, z).
 *  CONE:      c = centre of the proximal end disc (J_k), R column 1 = unit axis towards
 *             J_{k+1}, s = (r0, r1, L); the solid is {p : z=(p-c).a in [0,L],
 *             |p-c-z a| <= r0 + (r1-r0) z/L}, caps included.
 *  CYLINDER:  c = centre of the y_H = 0 end, R = hand frame axes, s = (a, len, b); the
 *             solid is {x^2/a^2 + z^2/b^2 <= 1, y in [-len, 0]} in local coordinates. */
typedef struct {
  int32_t kind;
  double c[3];
  double R[3][3]; /* R[row][col]; column j is local axis j in camera coordinates */
  double s[3];
} or_prim;

typedef struct {
  int64_t s_o;    /* sum o_s                         */
  int64_t s_or;   /* sum (o_s OR r_m)                */
  int64_t s_and;  /* sum (o_s AND r_m)               */
  int64_t s_rm;   /* sum r_m                         */
  int64_t n_both; /* pixels with r_d > 0 and o_d > 0 */
  double num;     /* sum over n_both pixels of min(|o_d - r_d|, clamp), mm */
} or_sums;

typedef struct {
  uint64_t seed;
  int32_t particles, generations, mutation_period, per_dim_r;
  double c1, c2, mutation_fraction;
  double stop_threshold; /* -INFINITY = off */
  /* AMB-17 (P:L152 is silent on the order): 0 = mutate after the Eq. 6-7 update and before
   * the evaluation of generations k = period, 2 period, ... (mutated poses are evaluated as
   * drawn); 1 = SPEC's order: mutate after generation k's evaluation and
   * bookkeeping, so the next update moves the mutated particles before they are evaluated. */
  int32_t mutation_after_eval;
} or_pso_params;

/* Batch objective: costs[i] = f(X[i*D .. i*D+D-1]); NaN is treated as +inf by the PSO. */
typedef void (*or_batch_fn)(const double* X, int32_t n, int32_t D, double* costs, void* user);

/* ---- defaults ---- */
void or_default_dims(or_dims* d);
void or_default_cost(or_cost_params* p);
void or_default_pso(or_pso_params* p);
void or_camera_for(int32_t width, int32_t height, or_camera* cam); /* fx=525*W/640 ... */
void or_bounds(double lo[26], double hi[26]);                      /* Tables 1-2, rad / mm */

/* ---- RNG ---- */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double or_u01(uint32_t w0, uint32_t w1);

/* ---- kinematics (Eq. 1-3) ---- */
void or_fk(const double h[26], const or_dims* d, or_prim prims[38], double joints[5][4][3]);
double or_kc(const double h[26], double rho);

/* ---- rendering ---- */
double or_first_hit(const or_prim* p, const double dir[3]); /* smallest t>0 on the solid, or +inf */
void or_ray(const or_camera* cam, double u, double v, double dir[3]);
/* depth: H*W fp32, 0 = no hit.  culled = 1 skips primitives outside their conservative box. */
void or_render_prims(const or_prim* prims, int32_t nprim, const or_camera* cam, int32_t culled, float* depth);
void or_render(const double h[26], const or_dims* d, const or_camera* cam, int32_t culled, float* depth);
/* edge mask: 1 where hit status or depth (> depth_tol mm) changes when the ray moves by
 * +-delta px in u or v, or where ||o_d - r_d| - d_m| < rm_tol (obs_depth may be NULL). */
void or_edge_mask_prims(const or_prim* prims, int32_t nprim, const or_camera* cam, double delta,
                        double depth_tol, const float* obs_depth, double d_m, double rm_tol,
                        uint8_t* edge);
void or_edge_mask(const double h[26], const or_dims* d, const or_camera* cam, double delta,
                  double depth_tol, const float* obs_depth, double d_m, double rm_tol, uint8_t* edge);
/* conservative pixel box [x0,x1]x[y0,y1] of one primitive (inclusive), margin in px;
 * returns 0 if empty. */
int32_t or_prim_box(const or_prim* p, const or_camera* cam, int32_t margin, int32_t box[4]);

/* ---- observation front end ("skin colour detection and depth
 * segmentation extract the hand region of the colour and depth images; the result of this
 * preprocessing is O = (O_s, O_d)").  DESIGN.md §3 AMB-33..36 fix the reading:
 *   valid    = d > 0                       (Kinect: 0 = no reading)
 *   band     = [lo, hi] (mode 0) or [m, m + width], m = min d over valid pixels that are
 *              skin (or all valid pixels without a skin image): the hand is the nearest
 *              object (mode 1; no candidate: empty band)
 *   in_band  = valid and lo <= d <= hi
 *   O_s      = skin ? skin and (not valid or in_band) : in_band
 *   O_d      = keep_background ? (valid ? d : 0) : (in_band ? d : 0)
 * All band limits are integer mm, so every decision is exact in any precision. */
typedef struct {
  int32_t mode;            /* 0 fixed band, 1 nearest-object band */
  int32_t lo, hi, width;   /* mm */
  int32_t keep_background; /* 1: O_d keeps all valid depth (o_d defined where o_s = 0, AMB-30) */
} or_segment_params;
/* depth_u16 [npx] mm, skin [npx] u8 or NULL -> o_d [npx] fp32 mm, o_s [npx] u8 0/1;
 * band_out (may be NULL) receives the band used {lo, hi} (mode 1 without candidates: {1, 0}). */
void or_segment(const uint16_t* depth_u16, const uint8_t* skin, int64_t npx,
                const or_segment_params* sp, float* o_d, uint8_t* o_s, int32_t band_out[2]);

/* ---- cost (Eq. 4-5) ---- */
void or_score(const float* obs_depth, const uint8_t* obs_mask, const float* r_d, int64_t npx,
              const or_cost_params* cp, or_sums* out);
double or_cost_from_sums(const or_sums* s, const or_cost_params* cp, double kc, double* D_out);
/* full objective for a batch of n poses; sums/kc/D may be NULL. threads<=0: all cores. */
void or_eval_batch(const double* poses, int32_t n, const float* obs_depth, const uint8_t* obs_mask,
                   const or_camera* cam, const or_dims* d, const or_cost_params* cp, int32_t culled,
                   int32_t threads, double* costs, or_sums* sums, double* kc, double* D);

/* ---- algorithmic work: FLOPs the method must do for one pose ---- */
double or_walg(const double h[26], const or_dims* d, const or_camera* cam, int64_t* tests_out,
               int64_t* union_px_out);

/* ---- PSO (Eq. 6-7) ---- */
double or_constriction(double c1, double c2); /* NaN if c1+c2 <= 4 */
/* Generic bounded PSO with mutation of dims [mut_lo, mut_hi).  Returns 0 on success,
 * -1 on invalid parameters.  trace has `generations` entries (entries after an early
 * stop repeat the last value); X_out/V_out/P_out (N*D) and Pcost_out (N) may be NULL. */
int32_t or_pso_run(int32_t D, const double* lo, const double* hi, const double* init_lo,
                   const double* init_hi, int32_t mut_lo, int32_t mut_hi, const or_pso_params* pp,
                   or_batch_fn f, void* user, double* best_x, double* best_cost, double* trace,
                   int32_t* gens_run, double* X_out, double* V_out, double* P_out, double* Pcost_out);
/* Sphere objective f(x) = sum_d (x_d - centre_d)^2 evaluated left to right, no FMA. */
int32_t or_pso_sphere(int32_t D, const double* lo, const double* hi, const double* init_lo,
                      const double* init_hi, int32_t mut_lo, int32_t mut_hi, const double* centre,
                      const or_pso_params* pp, double* best_x, double* best_cost, double* trace,
                      int32_t* gens_run, double* X_out, double* V_out, double* P_out, double* Pcost_out);
/* The paper's fit: D = 26, Table 1-2 bounds, mutation dims 6..25.
 * init_center/init_radius (26 each) may be NULL: the full Table 1-2 box. */
int32_t or_pso_fit_hand(const float* obs_depth, const uint8_t* obs_mask, const or_camera* cam,
                        const or_dims* d, const or_cost_params* cp, const or_pso_params* pp,
                        const double* init_center, const double* init_radius, int32_t culled,
                        int32_t threads, double* best_x, double* best_cost, double* trace,
                        int32_t* gens_run, double* X_out, double* V_out, double* P_out,
                        double* Pcost_out);

#ifdef __cplusplus
}
#endif
#endif
