// eval.cuh — k_eval: one CTA per (pose, split) — small swarms, the depth hooks and the fused PSO generation (rows A2-A8)
// Part of the single translation unit kernels.cu (included after the observation kernels;
// shares its macros and helpers).
#pragma once

namespace hp {

// ---------------------------------------------------------------------------------------
// k_eval: one CTA per (particle, split).  Warp 0 runs FK into shared memory while the other
// warps stage the ray table; then all warps take tiles dynamically.  Used for small swarms
// (S > 1 splits per particle keep every SM busy) and for the depth-image hooks.
// ---------------------------------------------------------------------------------------
#ifndef HP_EVAL_FK_TEAM
#define HP_EVAL_FK_TEAM 5  // k_eval's / k_fit's FK team: warps 0..4 (fk_team<5>)
#endif
constexpr int kEvalFkTeam = HP_EVAL_FK_TEAM;
template <int NW, typename PoseT, int MODE, bool NEARCODE = true>
__global__ void __launch_bounds__(NW * 32, HP_MINB_WARPS_EVAL / NW)
    k_eval(const __grid_constant__ EvalArgs a, const __grid_constant__ CUtensorMap tmap) {
  __shared__ FkScratch s_fk;
  __shared__ __align__(16) FkOut s_out;
  __shared__ __align__(16) FkExact s_x;  // exact records: the near-plane tile loop's
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
      fk_team<double, kEvalFkTeam>(s_pose, a.dims, a.cam, a.cost.kc_rest, s_fk, s_out, &s_x);
    } else {
      const PoseT* pose = static_cast<const PoseT*>(a.poses) + (size_t)p * kNdof;
      fk_team<PoseT, kEvalFkTeam>(pose, a.dims, a.cam, a.cost.kc_rest, s_fk, s_out, &s_x);
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
  TileSums acc = run_tiles<MODE, NEARCODE>(a, &tmap, s_out, &s_x, sidx, a.S, nmine,
                                           &s_next, smem_u32(s_obs[warp]),
                                           smem_u32(&s_bar[warp]), 0u, s_dx, s_dy,
                                           frame_of(a, p) * a.cam.H)
                     .acc;

  GENPROF_MAX(2)
  if (MODE != kModeCost) return;
  // ---- reduction: warp shuffles, one atomic per sum per CTA ----
  unpack_counts(acc);
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


}  // namespace hp
