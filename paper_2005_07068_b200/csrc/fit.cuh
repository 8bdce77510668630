// fit.cuh — k_fit: a whole PSO hand fit (rows A2-A9) in ONE persistent cooperative kernel
// Part of the single translation unit kernels.cu (included after eval.cuh; shares its
// macros and helpers).
#pragma once

namespace hp {

// ---------------------------------------------------------------------------------------
// k_fit (DESIGN §9 "persistent fit"): the generation loop of P:L138-152 runs inside one
// cooperative launch of S x N CTAs (S splits per particle, one CTA of 32 warps per SM).
// Every CTA keeps its particle's swarm state (x, v, pbest) and the swarm-wide pbest costs
// and gbest in shared memory; per generation:
//   1. warp 0: Eq. (6)-(7) update of the CTA's particle (k >= 1; every split computes the
//      same bits), warps 0-4: FK of that pose into shared memory (fk_team)
//   2. all warps: the split's share of the particle's 16 x 8 tiles (run_tiles)
//   3. the CTA's integer sums (and, split 0, the evaluated position and kc) to global
//      memory, double-buffered by generation parity; one grid barrier
//   4. every CTA, redundantly: the N costs (Eq. 4-5) from the splits' sums, pbest (strict <,
//      NaN = +inf), gbest (lowest index on ties), trace, stop rule, its particle's mutation
//      mark (AMB-17) — identical inputs, identical bits in every CTA, so no second barrier.
// The arithmetic is the fused k_eval path's (same update order, same FK, same per-pixel
// formulas, integer sums), so the trajectory is bit for bit the multi-kernel fit's; what
// goes away is the per-generation launch, the grid drain, the ray-table restaging and the
// single-CTA bookkeeping tail.  Near-plane poses: NEARCODE = false (speculative, like the
// fused generation kernels); the host repeats the fit on the exact path if one appeared.
// ---------------------------------------------------------------------------------------
constexpr int kFitWarps = 32;
constexpr int kFitMaxN = 160;  // particles (<= one CTA per SM; B200 has 148 SMs)

// One grid-wide barrier: every CTA arrives once per generation on a monotone counter.
__device__ __forceinline__ void fit_grid_sync(unsigned int* count, unsigned int target) {
  // the CTA's writes happen before thread 0's release (bar.sync, then a cumulative
  // release at gpu scope); its acquire happens before every thread's later reads
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// The random numbers the update of generation k consumes (they depend only on the seed,
// the particle, the dimension and k): rd[d] = (r1, r2, mutation draw), computed by a warp
// outside the FK team one generation ahead, off the critical path.  Same draws as
// pso_update_warp: r1 / r2 of (i, 0 or d, k, tag 1), the re-draw of (i, d, k, tag 2) after
// the update, or of (i, d, k - 1, tag 2) before it in SPEC's order.
__device__ __forceinline__ void pso_draws_own(const PsoDev& p, const PsoDyn& dyn, int i, int k,
                                              const double* lo_s, const double* hi_s,
                                              double (*rd)[3]) {
  const int d = threadIdx.x & 31;
  if (d >= p.D) return;
  const uint4 r = draw(dyn.seed, (uint32_t)i, p.per_dim_r ? (uint32_t)d : 0u, (uint32_t)k, 1u);
  rd[d][0] = u01(r.x, r.y);
  rd[d][1] = u01(r.z, r.w);
  const uint4 m = draw(dyn.seed, (uint32_t)i, (uint32_t)d, (uint32_t)(p.mut_after ? k - 1 : k), 2u);
  rd[d][2] = lerp_rn(lo_s[d], hi_s[d], u01(m.x, m.y));
}

// Eq. (6)-(7) + clamp + mutation of the CTA's own particle i at generation k >= 1, from the
// shared-memory state: x, v (updated in place), pb = its pbest position, g = gbest, rd = the
// generation's draws.  The same operations in the same order as pso_update_warp (pso.cuh).
// One warp.
__device__ __forceinline__ void pso_update_own(const PsoDev& p, const PsoDyn& dyn, double* x_s,
                                               double* v_s, const double* pb_s,
                                               const double* g_s, const double* lo_s,
                                               const double* hi_s, const double (*rd)[3],
                                               bool marked) {
  const int d = threadIdx.x & 31;
  if (d >= p.D) return;
  const double r1 = rd[d][0], r2 = rd[d][1];
  double x0 = x_s[d], v0 = v_s[d];
  const double pb = pb_s[d], gb = g_s[d];
  const bool mdim = marked && d >= p.mut_lo && d < p.mut_hi;
  if (p.mut_after && mdim) {  // SPEC's order: re-drawn after generation k - 1
    x0 = rd[d][2];
    v0 = 0.0;
  }
  const double t1 = __dmul_rn(__dmul_rn(dyn.c1, r1), __dsub_rn(pb, x0));
  const double t2 = __dadd_rn(v0, t1);
  const double t3 = __dmul_rn(__dmul_rn(dyn.c2, r2), __dsub_rn(gb, x0));
  double v = __dmul_rn(dyn.w, __dadd_rn(t2, t3));
  double x = __dadd_rn(x0, v);
  if (x < lo_s[d]) {  // AMB-16
    x = lo_s[d];
    v = 0.0;
  } else if (x > hi_s[d]) {
    x = hi_s[d];
    v = 0.0;
  }
  if (!p.mut_after && mdim) {  // P:L152 (AMB-17: after the update)
    x = rd[d][2];
    v = 0.0;
  }
  x_s[d] = x;
  v_s[d] = v;
}

#if HP_GEN_PROF
// per-generation phase stamps: globaltimer min / max over CTAs (g_genprof), and clock64 of
// CTA 0 and of the last CTA (g_fitclk) for a per-CTA timeline
__device__ long long g_fitclk[64][2][8];
extern "C" int hp_debug_fit_clk(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_fitclk, sizeof(g_fitclk));
}
// stamps staged in shared memory (a global store per stamp would add a constant-bank load
// of the symbol's address, which misses: the loop's code evicts it), copied out at the end
__shared__ long long s_fitclk[64][8];
#define FITPROF_CLK(k, i) \
  if (threadIdx.x == 0 && (k) < 64) s_fitclk[(k)][i] = clock64();
#define FITPROF_MIN(k, i) FITPROF_CLK(k, i)
#define FITPROF_MAX(k, i) FITPROF_CLK(k, i)
#else
#define FITPROF_CLK(k, i)
#define FITPROF_MIN(k, i)
#define FITPROF_MAX(k, i)
#endif

#ifndef HP_FIT_DRAW_WARP
#define HP_FIT_DRAW_WARP kEvalFkTeam  // the warp drawing generation k + 1's numbers
#endif
template <bool NEARCODE>
__global__ void __launch_bounds__(kFitWarps * 32, 1)
    k_fit(const __grid_constant__ EvalArgs a, const __grid_constant__ CUtensorMap tmap) {
  __shared__ FkScratch s_fk;
  __shared__ __align__(16) FkOut s_out;
  __shared__ __align__(16) FkExact s_xr;
  __shared__ __align__(128) uint32_t s_obs[kFitWarps][kTileW * kTileH];
  __shared__ __align__(8) uint64_t s_bar[kFitWarps];
  __shared__ unsigned long long s_red[kFitWarps][4];
  __shared__ int s_next;
  // swarm state: this CTA's particle (x = the position generation k evaluates), gbest,
  // every particle's pbest cost and improvement flag, the bounds
  __shared__ double s_pose[32], s_v[32], s_pb[32], s_g[32];
  __shared__ double s_lo[32], s_hi[32];
  __shared__ double s_rd[2][32][3];  // the draws of generations k (parity) and k + 1
  __shared__ double s_pc[kFitMaxN];
  __shared__ int s_imp[kFitMaxN];
  __shared__ double s_bv[kFitWarps];
  __shared__ int s_bi[kFitWarps];
  __shared__ int s_g_idx, s_final, s_mark;
  // the hand model and the PSO parameters in shared memory: read every generation, and
  // kernel-parameter (constant-bank) reads that miss the constant cache after the tile loop
  // cost a round trip each on the generation's critical path
  __shared__ DimsD s_dims;
  __shared__ PsoDev s_ps;
  __shared__ PsoDyn s_dyn;
  __shared__ CamParams s_cam;  // FK's camera and kc rest term (no constant-bank reads per
  __shared__ double s_kcrest;  // generation: the parameter lines leave the constant cache)
  extern __shared__ float s_ray[];  // the ray table, then every particle's evaluated position

  const PsoDev& ps = s_ps;
  const int N = a.pso.N, D = a.pso.D, K = a.pso.K;
  const int G = gridDim.x, S = a.S;
  const int p = blockIdx.x % N, sidx = blockIdx.x / N;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const float* s_dx = s_ray;
  const float* s_dy = s_ray + ray_dx_len(a.cam.W);
  double(*s_xall)[kNdof] =
      reinterpret_cast<double(*)[kNdof]>(s_ray + ray_floats(a.cam.W, a.cam.H));
  const PsoDyn& dyn = s_dyn;

  // ---- prologue: ray table, mbarriers, bounds, generation-0 position of particle p ----
  {
    const int n4 = ray_floats(a.cam.W, a.cam.H) / 4;
    for (int i = tid; i < n4; i += kFitWarps * 32)
      reinterpret_cast<float4*>(s_ray)[i] = __ldg(reinterpret_cast<const float4*>(a.ray) + i);
  }
  for (int i = tid; i < (int)(sizeof(DimsD) / sizeof(double)); i += kFitWarps * 32)
    reinterpret_cast<double*>(&s_dims)[i] = reinterpret_cast<const double*>(&a.dims)[i];
  if (tid == 0) {
    s_ps = a.pso;
    s_dyn = *a.pso.dyn;
    s_cam = a.cam;
    s_kcrest = a.cost.kc_rest;
  }
  __syncthreads();
  const DimsD& dims = s_dims;
  if (tid == 0) {
    for (int w = 0; w < kFitWarps; w++) mbar_init(&s_bar[w], 1);
    fence_mbar_init();
    prefetch_tmap(&tmap);
    s_mark = 0;
  }
  if (tid < D) {
    s_lo[tid] = ps.lo[tid];
    s_hi[tid] = ps.hi[tid];
    // P:L146 random positions in the init box (k_pso_init's draw), v = 0
    const uint4 r = draw(dyn.seed, (uint32_t)p, (uint32_t)tid, 0u, 0u);
    s_pose[tid] = lerp_rn(ps.ilo[tid], ps.ihi[tid], u01(r.x, r.y));
    s_v[tid] = 0.0;
  }
  __syncthreads();

  uint32_t phase = 0;
  const uint32_t obs_s = smem_u32(s_obs[warp]), bar_s = smem_u32(&s_bar[warp]);
  int k = 0;
  for (;; k++) {
    FITPROF_MIN(k, 0)
    // ---- 1. update (k >= 1) and FK of particle p ----
    if (warp < kEvalFkTeam) {
      if (k >= 1 && warp == 0)
        pso_update_own(ps, dyn, s_pose, s_v, s_pb, s_g, s_lo, s_hi, s_rd[k & 1], s_mark != 0);
      __syncwarp();
      FITPROF_CLK(k, 5)
      // EXACT records only for the exact (near-plane) instantiation
      fk_team<double, kEvalFkTeam>(s_pose, dims, s_cam, s_kcrest, s_fk, s_out,
                                   NEARCODE ? &s_xr : nullptr);
    } else if (warp == HP_FIT_DRAW_WARP) {  // next generation's draws, while the team runs FK
      if (lane == 0) s_next = 0;
      if (k + 1 < K) pso_draws_own(ps, dyn, p, k + 1, s_lo, s_hi, s_rd[(k + 1) & 1]);
    }
    __syncthreads();
    FITPROF_MAX(k, 1)
    // ---- 2. this split's tiles ----
    TileSums acc;
    {
      const TileGrid g(s_out.ubox);
      const int nmine = g.ntiles > sidx ? (g.ntiles - sidx + S - 1) / S : 0;
      const TileRun r = run_tiles<kModeCost, NEARCODE>(a, &tmap, s_out, &s_xr, sidx, S, nmine,
                                                       &s_next, obs_s, bar_s, phase, s_dx,
                                                       s_dy, 0);
      acc = r.acc;
      phase = r.phase;
    }
    FITPROF_MAX(k, 2)
    // ---- 3. publish the CTA's sums (+ position and kc); grid barrier ----
    unpack_counts(acc);
    warp_reduce(acc);
    if (lane == 0) {
      s_red[warp][0] = acc.rm;
      s_red[warp][1] = acc.and_;
      s_red[warp][2] = acc.num;
      s_red[warp][3] = acc.both;
    }
    __syncthreads();
    const int buf = k & 1;
    if (tid < 4) {  // the rounding-free integer sums of the CTA's warps
      unsigned long long v = 0;
      for (int w = 0; w < kFitWarps; w++) v += s_red[w][tid];
      __stcg(a.fit_part + ((size_t)buf * G + blockIdx.x) * 4 + tid, v);
    }
    if (sidx == 0 && tid < 32) {
      double* xp = a.fit_xpub + ((size_t)buf * N + p) * 32;
      if (lane < D) xp[lane] = s_pose[lane];
      if (lane == 31) xp[31] = s_out.kc;
    }
    fit_grid_sync(a.fit_bar, (unsigned)(k + 1) * (unsigned)G);
    FITPROF_MAX(k, 3)
    // ---- 4. bookkeeping, redundantly in every CTA ----
    // the particle threads (warps 0 .. nwp - 1) load the sums and compute the costs; the
    // other warps copy every particle's evaluated position (for the gbest) meanwhile
    const int nwp = (N + 31) >> 5;
    double bv = INFINITY;
    int bi = 0x7fffffff;
    if (warp >= nwp) {
      for (int idx = tid - 32 * nwp; idx < N * D; idx += (kFitWarps - nwp) * 32) {
        const int i = idx / D, d = idx - i * D;
        s_xall[i][d] = __ldcg(a.fit_xpub + ((size_t)buf * N + i) * 32 + d);
      }
    } else if (tid < N) {
      const int i = tid;
      unsigned long long v0 = 0, v1 = 0, v2 = 0, v3 = 0;
      for (int s = 0; s < S; s++) {
        const ulonglong2* q = reinterpret_cast<const ulonglong2*>(
            a.fit_part + ((size_t)buf * G + (size_t)s * N + i) * 4);
        const ulonglong2 u0 = __ldcg(q), u1 = __ldcg(q + 1);
        v0 += u0.x;
        v1 += u0.y;
        v2 += u1.x;
        v3 += u1.y;
      }
      const unsigned long long v[4] = {v0, v1, v2, v3};
      const double kc = __ldcg(a.fit_xpub + ((size_t)buf * N + i) * 32 + 31);
      double e = finalize_cost(a, i, v, kc);  // Eq. (4)-(5); the fit's EvalArgs store nothing
      if (isnan(e)) e = INFINITY;
      const double pc_old = s_pc[i];
      const bool imp = k == 0 || e < pc_old;
      const double pc = imp ? e : pc_old;
      s_pc[i] = pc;
      s_imp[i] = imp;
      bv = pc;
      bi = i;
    }
    FITPROF_CLK(k, 6)
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov < bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      s_bv[warp] = bv;
      s_bi[warp] = bi;
    }
    __syncthreads();
    if (warp == 0) {
      // argmin over the warps that hold particles (lowest index on ties)
      const int nwp = (N + 31) >> 5;
      double v = lane < nwp ? s_bv[lane] : INFINITY;
      int g = lane < nwp ? s_bi[lane] : 0x7fffffff;
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, off);
        const int oi = __shfl_xor_sync(0xffffffffu, g, off);
        if (ov < v || (ov == v && oi < g)) {
          v = ov;
          g = oi;
        }
      }
      if (g >= N) g = 0;  // all +inf: lowest index
      // the mutation mark of particle p for generation k + 1 (AMB-17: the worst
      // floor(N frac) by pbest cost, ties: the higher index is worse)
      int m = 0;
      if (mutation_marks_due(ps, k)) {
        const double ci = s_pc[p];
        int rank = 0;
        for (int j = lane; j < N; j += 32) {
          const double cj = s_pc[j];
          rank += (cj < ci) || (cj == ci && j < p);
        }
        m = __reduce_add_sync(0xffffffffu, rank) >= N - ps.nmut;
      }
      if (lane == 0) {
        s_g_idx = g;
        const double gc = s_pc[g];
        const bool stopped = dyn.stop > -INFINITY && gc < dyn.stop;  // P:L148 stop rule
        s_final = stopped || k + 1 >= K;
        if (blockIdx.x == 0) {
          ps.trace[k] = gc;
          *ps.gens_run = k + 1;
          if (stopped) *ps.done = 1;
        }
        s_mark = m;
      }
    }
    FITPROF_CLK(k, 7)
    __syncthreads();
    // pbest position of p and gbest: the evaluated positions of the improved particles (a
    // gbest that changed improved in this generation, so its pbest is its position)
    const int g = s_g_idx;
    if (tid < D) {
      if (s_imp[p]) s_pb[tid] = s_pose[tid];
      if (s_imp[g]) s_g[tid] = s_xall[g][tid];
    }
    __syncthreads();
    FITPROF_MAX(k, 4)
    if (s_final) break;
  }
#if HP_GEN_PROF
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
    for (int q = 0; q < 64 * 8; q++)
      g_fitclk[q / 8][blockIdx.x == 0 ? 0 : 1][q % 8] = s_fitclk[q / 8][q % 8];
#endif
  // ---- the final state for the host (hp_pso_state): split 0 of every particle, gbest ----
  if (sidx == 0 && tid < D) {
    const size_t id = (size_t)p * D + tid;
    ps.X[id] = s_pose[tid];
    ps.V[id] = s_v[tid];
    ps.P[id] = s_pb[tid];
  }
  if (sidx == 0 && tid == 0) ps.Pc[p] = s_pc[p];
  if (blockIdx.x == 0) {
    if (tid < D) ps.G[tid] = s_g[tid];
    if (tid == 0) *ps.Gc = s_pc[s_g_idx];
  }
}

}  // namespace hp
