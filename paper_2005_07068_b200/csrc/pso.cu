// pso.cu — PSO init / update / bookkeeping kernels (rows A7-A8; Eq. (6)-(7)).
//
// All swarm state is fp64 in device memory.  The update is evaluated in exactly the order
// v = w * ((v + (c1 r1)(P - x)) + (c2 r2)(G - x)), x = x + v with round-to-nearest
// intrinsics (no FMA contraction), so the trajectory is reproducible bit for bit
// (DESIGN §4).  Random numbers: Philox4x32-10 keyed by the seed, counter
// (particle, dim, generation, tag).
#include <math.h>

#include "pso.cuh"

namespace hp {

__global__ void k_pso_init(const PsoDev p) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx == 0) {
    *p.done = 0;
    *p.gens_run = 0;
  }
  if (idx < p.N) p.mark[idx] = 0;
  if (idx >= (long long)p.N * p.D) return;
  const int i = (int)(idx / p.D), d = (int)(idx % p.D);
  const uint4 r = draw(p.dyn->seed, (uint32_t)i, (uint32_t)d, 0u, 0u);
  p.X[idx] = lerp_rn(p.ilo[d], p.ihi[d], u01(r.x, r.y));  // P:L146 random positions
  p.V[idx] = 0.0;                                          // "initial velocity is 0"
}

// One warp per particle (standalone update; the hand fit fuses it into k_eval).
__global__ void k_pso_update(const PsoDev p, int k) {
  if (*p.done) return;
  pso_update_warp(p, blockIdx.x, k, p.X, p.V, p.X, p.V, true, nullptr);
}

constexpr int kBookThreads = 1024;
__global__ void __launch_bounds__(kBookThreads) k_pso_book(const PsoDev p, int k) {
  if (k > 0 && *p.done) return;
  pso_book_block(p, k, p.X);
}

// f(x) = sum_d (x_d - c_d)^2, left to right (hp_debug_pso_sphere).
__global__ void k_sphere_eval(const PsoDev p, const double* centre) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.N || *p.done) return;
  double acc = 0.0;
  for (int d = 0; d < p.D; d++) {
    const double t = __dsub_rn(p.X[(long long)i * p.D + d], centre[d]);
    acc = __dadd_rn(acc, __dmul_rn(t, t));
  }
  p.E[i] = acc;
}

cudaError_t launch_pso_init(const PsoDev& p, cudaStream_t st) {
  const long long n = (long long)p.N * p.D;
  const long long tot = n > p.N ? n : p.N;
  k_pso_init<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_pso_update(const PsoDev& p, int k, cudaStream_t st) {
  k_pso_update<<<p.N, 32, 0, st>>>(p, k);
  return cudaGetLastError();
}
cudaError_t launch_pso_book(const PsoDev& p, int k, cudaStream_t st) {
  k_pso_book<<<1, kBookThreads, 0, st>>>(p, k);
  return cudaGetLastError();
}
cudaError_t launch_sphere_eval(const PsoDev& p, const double* centre, cudaStream_t st) {
  k_sphere_eval<<<(p.N + 127) / 128, 128, 0, st>>>(p, centre);
  return cudaGetLastError();
}

}  // namespace hp
