// pso.cuh — PSO device functions shared by the standalone PSO kernels (pso.cu) and the
// fused evaluation kernel (kernels.cu): Philox4x32-10, the Eq. (6)-(7) update of one
// particle by one warp, and the per-generation bookkeeping by one block
// (rows A7-A8).
//
// All swarm state is fp64 in device memory.  The update is evaluated in exactly the order
// v = w * ((v + (c1 r1)(P - x)) + (c2 r2)(G - x)), x = x + v with round-to-nearest
// intrinsics (no FMA contraction), so the trajectory is reproducible bit for bit
// (DESIGN §4).  Random numbers: Philox4x32-10 keyed by the seed, counter
// (particle, dim, generation, tag).
#pragma once
#include <math.h>

#include "common.cuh"

namespace hp {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    if (r > 0) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

// 53-bit uniform in [0, 1): every step is exact, so the value is unique.
__device__ __forceinline__ double u01(uint32_t w0, uint32_t w1) {
  return ((double)(w0 >> 5) * 67108864.0 + (double)(w1 >> 6)) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ uint4 draw(uint64_t seed, uint32_t i, uint32_t d, uint32_t k,
                                      uint32_t tag) {
  return philox4x32_10(make_uint4(i, d, k, tag),
                       make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}

// lo + u (hi - lo), rounded after each operation
__device__ __forceinline__ double lerp_rn(double lo, double hi, double u) {
  return __dadd_rn(lo, __dmul_rn(u, __dsub_rn(hi, lo)));
}

// One warp: Eq. (6)-(7) + clamp + mutation for particle i at generation k >= 1.  Reads
// x, v from Xin/Vin; if `write` stores them to Xout/Vout (may alias Xin/Vin when no other
// thread reads the old values); if pose != nullptr lane d also leaves x_d there.
// deferred (the fused generation kernel): the previous bookkeeping left P and G stale and
// recorded pimp[i] (particle i improved: its pbest is its evaluated position Xin[i]) and
// gsel = (g, pimp[g]); the update reads the values they stand for, and the writer CTA
// materialises P[i].  Same bits as the eager form.
__device__ __forceinline__ void pso_update_warp(const PsoDev& p, int i, int k, const double* Xin,
                                                const double* Vin, double* Xout, double* Vout,
                                                bool write, double* pose,
                                                bool deferred = false) {
  const int lane = threadIdx.x & 31;
  const PsoDyn dyn = *p.dyn;
  const bool imp_i = deferred && p.pimp[i] != 0;
  const int gi = deferred ? p.gsel[0] : 0;
  const bool g_from_x = deferred && p.gsel[1] != 0;
  double r1 = 0.0, r2 = 0.0;
  if (!p.per_dim_r) {
    const uint4 r = draw(dyn.seed, (uint32_t)i, 0u, (uint32_t)k, 1u);
    r1 = u01(r.x, r.y);
    r2 = u01(r.z, r.w);
  }
  const bool marked = p.mark[i] != 0;
  for (int d = lane; d < p.D; d += 32) {
    if (p.per_dim_r) {
      const uint4 r = draw(dyn.seed, (uint32_t)i, (uint32_t)d, (uint32_t)k, 1u);
      r1 = u01(r.x, r.y);
      r2 = u01(r.z, r.w);
    }
    const long long id = (long long)i * p.D + d;
    double x0 = Xin[id];  // the position generation k - 1 evaluated
    double pb, gb;
    if (deferred) {
      pb = imp_i ? x0 : p.P[id];
      if (imp_i && write) p.P[id] = x0;
      const long long gid = (long long)gi * p.D + d;  // P[g] is not written when g_from_x
      gb = g_from_x ? Xin[gid] : p.P[gid];
    } else {
      pb = p.P[id];
      gb = p.G[d];
    }
    double v0 = Vin[id];
    const bool mdim = marked && d >= p.mut_lo && d < p.mut_hi;
    if (p.mut_after && mdim) {
      // SPEC's order: the particle was re-drawn after generation k - 1's
      // bookkeeping (counter generation k - 1), so this update moves the re-drawn position
      const uint4 r = draw(dyn.seed, (uint32_t)i, (uint32_t)d, (uint32_t)(k - 1), 2u);
      x0 = lerp_rn(p.lo[d], p.hi[d], u01(r.x, r.y));
      v0 = 0.0;
    }
    // Eq. (6): v = w (v + c1 r1 (P - x) + c2 r2 (G - x));  Eq. (7): x = x + v
    const double t1 = __dmul_rn(__dmul_rn(dyn.c1, r1), __dsub_rn(pb, x0));
    const double t2 = __dadd_rn(v0, t1);
    const double t3 = __dmul_rn(__dmul_rn(dyn.c2, r2), __dsub_rn(gb, x0));
    double v = __dmul_rn(dyn.w, __dadd_rn(t2, t3));
    double x = __dadd_rn(x0, v);
    if (x < p.lo[d]) {  // AMB-16: clamp, zero that velocity component
      x = p.lo[d];
      v = 0.0;
    } else if (x > p.hi[d]) {
      x = p.hi[d];
      v = 0.0;
    }
    if (!p.mut_after && mdim) {  // P:L152 mutation (AMB-17: after the update)
      const uint4 r = draw(dyn.seed, (uint32_t)i, (uint32_t)d, (uint32_t)k, 2u);
      x = lerp_rn(p.lo[d], p.hi[d], u01(r.x, r.y));
      v = 0.0;
    }
    if (write) {
      Xout[id] = x;
      Vout[id] = v;
    }
    if (pose) pose[d] = x;
  }
}

// Are mutation marks for generation k + 1's update drawn at the end of generation k?
// Order 0 (AMB-17): generation k + 1 is a mutation generation (k + 1 = period, 2 period, ...).
// Order 1: generation k >= 1 is one, and the update of k + 1 moves the re-drawn
// particles.  Never after the last generation (nothing would see them).
__device__ __forceinline__ bool mutation_marks_due(const PsoDev& p, int k) {
  const int kn = k + 1;
  if (!(p.period > 0 && kn < p.K && p.nmut > 0)) return false;
  return p.mut_after ? (k >= 1 && k % p.period == 0) : (kn % p.period == 0);
}

// One block (any size, multiple of 32): bookkeeping after generation k's evaluation of the
// positions X — pbest (strict <), gbest (lowest index on ties, NaN = +inf), trace, stop
// rule, and the mutation marks for generation k + 1 (worst floor(N frac) by Pcost, ties:
// higher index worse).  Ends with __syncthreads.
constexpr int kPsoMaxFlags = 1024;  // particles whose pbest flags fit the shared bitmask
// e: this generation's costs (global p.E, or a shared-memory copy); spc: optional
// shared-memory scratch [N] for the personal-best costs (the global p.Pc is kept in step).
__device__ __forceinline__ void pso_book_block(const PsoDev& p, int k, const double* X,
                                               const double* e_in = nullptr,
                                               double* spc = nullptr,
                                               bool spc_loaded = false) {
  __shared__ double s_v[32];
  __shared__ int s_i[32];
  __shared__ int s_g;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nw = nt >> 5;
  const double* E = e_in ? e_in : p.E;
  double* PC = spc ? spc : p.Pc;
  const double stop = p.dyn->stop;  // loaded early: off the tail's critical path
  if (spc && !spc_loaded) {
    for (int i = tid; i < p.N; i += nt) spc[i] = p.Pc[i];
    __syncthreads();
  }
  // pbest: the improvement flags first (one thread per particle), then every (particle,
  // dim) copy in parallel so the global loads overlap instead of queueing per particle
  __shared__ unsigned s_imp[(kPsoMaxFlags + 31) / 32];
  const bool flags_in_smem = p.N <= kPsoMaxFlags;
  for (int i = tid; i < p.N; i += nt) {
    double e = E[i];
    if (isnan(e)) e = INFINITY;
    const bool imp = k == 0 || e < PC[i];
    if (imp) {
      PC[i] = e;
      if (spc) p.Pc[i] = e;
    }
    if (flags_in_smem) {
      if (imp) atomicOr(&s_imp[i >> 5], 1u << (i & 31));
      else atomicAnd(&s_imp[i >> 5], ~(1u << (i & 31)));
    } else if (imp) {
      for (int d = 0; d < p.D; d++) p.P[(long long)i * p.D + d] = X[(long long)i * p.D + d];
    }
  }
  __syncthreads();
  if (flags_in_smem) {
    const int nd = p.N * p.D;  // <= 1024 x 64
    for (int idx = tid; idx < nd; idx += nt) {
      const int i = idx / p.D;
      if ((s_imp[i >> 5] >> (i & 31)) & 1u) p.P[idx] = X[idx];
    }
  }
  __syncthreads();
  double bv = INFINITY;
  int bi = 0x7fffffff;
  for (int i = tid; i < p.N; i += nt) {
    const double v = PC[i];
    if (v < bv || (v == bv && i < bi)) {
      bv = v;
      bi = i;
    }
  }
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
    s_v[warp] = bv;
    s_i[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    double v = INFINITY;
    int g = 0x7fffffff;
    for (int w = 0; w < nw; w++)
      if (s_v[w] < v || (s_v[w] == v && s_i[w] < g)) {
        v = s_v[w];
        g = s_i[w];
      }
    if (g >= p.N) g = 0;  // all +inf (or NaN): lowest index
    s_g = g;
    *p.Gc = PC[g];
    p.trace[k] = PC[g];
    *p.gens_run = k + 1;
    if (stop > -INFINITY && PC[g] < stop) *p.done = 1;  // P:L148 stop rule
  }
  __syncthreads();
  const int g = s_g;
  for (int d = tid; d < p.D; d += nt) p.G[d] = p.P[(long long)g * p.D + d];
  const bool mut = mutation_marks_due(p, k);
  for (int i = tid; i < p.N; i += nt) {
    int m = 0;
    if (mut) {
      const double ci = PC[i];
      int rank = 0;
      for (int j = 0; j < p.N; j++) {
        const double cj = PC[j];
        rank += (cj < ci) || (cj == ci && j < i);
      }
      m = rank >= p.N - p.nmut;
    }
    p.mark[i] = m;
  }
  __syncthreads();
}

// The fused generation kernel's bookkeeping tail (deferred form, see pso_update_warp): the
// caller has finalised E, updated Pc / pimp and left each thread's (best pcost, index) in
// (bv, bi); pcs = the pbest costs (shared memory, or the global Pc).  Reduces the argmin,
// writes Gc / trace / stop, the deferred gbest (or, after the last generation or the stop,
// materialises P and G for the host), then the mutation marks.  Ends with __syncthreads.
__device__ __forceinline__ void pso_book_tail(const PsoDev& p, int k, const double* X,
                                              const double* pcs, double bv, int bi,
                                              double stop) {
  __shared__ double s_v[32];
  __shared__ int s_i[32];
  __shared__ int s_g, s_final;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nw = nt >> 5;
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
    s_v[warp] = bv;
    s_i[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    double v = INFINITY;
    int g = 0x7fffffff;
    for (int w = 0; w < nw; w++)
      if (s_v[w] < v || (s_v[w] == v && s_i[w] < g)) {
        v = s_v[w];
        g = s_i[w];
      }
    if (g >= p.N) g = 0;  // all +inf (or NaN): lowest index
    s_g = g;
    const double gc = pcs[g];
    *p.Gc = gc;
    p.trace[k] = gc;
    *p.gens_run = k + 1;
    const bool stopped = stop > -INFINITY && gc < stop;  // P:L148 stop rule
    if (stopped) *p.done = 1;
    s_final = stopped || k + 1 >= p.K;
  }
  __syncthreads();
  const int g = s_g;
  if (s_final) {  // materialise P and G for the host
    const int nd = p.N * p.D;
    for (int idx = tid; idx < nd; idx += nt)
      if (p.pimp[idx / p.D]) p.P[idx] = X[idx];
    for (int d = tid; d < p.D; d += nt)
      p.G[d] = p.pimp[g] ? X[(long long)g * p.D + d] : p.P[(long long)g * p.D + d];
  } else if (tid == 0) {
    p.gsel[0] = g;
    p.gsel[1] = p.pimp[g];
  }
  const bool mut = mutation_marks_due(p, k);
  for (int i = tid; i < p.N; i += nt) {
    int m = 0;
    if (mut) {
      const double ci = pcs[i];
      int rank = 0;
      for (int j = 0; j < p.N; j++) {
        const double cj = pcs[j];
        rank += (cj < ci) || (cj == ci && j < i);
      }
      m = rank >= p.N - p.nmut;
    }
    p.mark[i] = m;
  }
  __syncthreads();
}

}  // namespace hp
