// batch.cuh — the batch path: k_fk_batch (FK + tile lists) and the persistent renderer k_render_persist (rows A2-A5)
// Part of the single translation unit kernels.cu (included after the observation kernels;
// shares its macros and helpers).
#pragma once

namespace hp {

// ---------------------------------------------------------------------------------------
// Two-kernel batch path for large swarms.
//   k_fk_batch      : four particles per CTA — FK (fp64) and each particle's list of
//                     non-empty 16 x 16 blocks with the cull masks of their two 16 x 8
//                     halves, written to global memory (L2-resident), then a per-particle
//                     ready flag (the launch epoch, st.release).
//   k_render_persist: persistent CTAs, ALL warps render.  Per particle one thread pulls the
//                     FK record and tile list into shared memory with 1-D TMA bulk copies
//                     (three slots: particle i + 3 is fetched as soon as particle i is
//                     finished, while i + 1 and i + 2 render), so no warp waits on FK
//                     latency; launched under k_fk_batch (PDL), its first particles wait
//                     for their own flags, not for the whole FK grid.
// ---------------------------------------------------------------------------------------
// A tile (qx, qy) overlaps primitive j iff column qx's x-range and row qy's y-range both
// overlap box j — the same four compares as cull_tile — so the tile masks are the AND of
// per-column and per-row 38-bit masks (tx + ty sets of 38 tests instead of tx * ty).
constexpr int kMaxBand = 64;  // columns / rows of the per-warp band masks

// Tighter per-tile shapes than the boxes for the cones (the spheres' discs would remove only
// a fifth as much work: scripts/cull_stats.py).  A point p with |p - c| <= r projects within
// R = f r |c| / (c_z (c_z - r)) px of the projection P(c) (f = max(f_x, f_y); the image-plane
// offset is M (p - c) / (c_z (c_z + (p - c)_z)) with M = [[c_z, 0, -c_x], [0, c_z, -c_y]],
// whose largest singular value is |c|).  A cone — the convex hull of its two end discs —
// therefore lies in the 2-D capsule of radius max(R_0, R_1) around the segment
// P(J_0) P(J_1), and a tile whose rectangle projects on the segment's normal farther than R
// from it (separating axis) is skipped.  Stored per cone: (n_x, n_y, n . P(J_0), R); R = inf
// (no refinement) within 1 mm of the camera plane.  Margins: 1e-4 relative + 0.02 px for
// the fp32 / approximate-MUFU rounding of the record and of P (~1e-6 relative).
// A 16 x 8 tile's 38-bit cull mask: its column band's and row band's masks ANDed, then each
// cone's bit cleared if its projected capsule misses the tile (separating axis).
__device__ __forceinline__ uint2 tile_mask(uint2 c, uint2 r, int X0, int Y0, const float4* shp) {
  unsigned int lo = c.x & r.x, hi = c.y & r.y;
  // pixel x's centre is x + 1/2 in the projected coordinates f u + c
  const float tcx = (float)X0 + 0.5f * kTileW, tcy = (float)Y0 + 0.5f * kTileH;
  constexpr float hx = 0.5f * (kTileW - 1), hy = 0.5f * (kTileH - 1);
  unsigned int cm = ((lo >> kCone0) | (hi << (32 - kCone0))) & ((1u << kNcone) - 1u);
  for (unsigned int q = cm; q; q &= q - 1) {
    const int j = __ffs(q) - 1;
    const float4 sh = shp[j];
    if (fabsf(fmaf(sh.x, tcx, fmaf(sh.y, tcy, -sh.z))) >
        fmaf(hx, fabsf(sh.x), fmaf(hy, fabsf(sh.y), sh.w)))
      cm &= ~(1u << j);
  }
  // cones are bits 20..31 of lo and 0..1 of hi
  lo = (lo & ((1u << kCone0) - 1u)) | (cm << kCone0);
  hi = (hi & ~((1u << (kNcone - (32 - kCone0))) - 1u)) | (cm >> (32 - kCone0));
  return make_uint2(lo, hi);
}

// The particle's non-empty 16 x 16 blocks of its union grid (16 x 8 tiles, rows paired),
// each with its two halves' masks split per kind (BlockEnt, tile.cuh).  Returns the count,
// or -1 (too large: the renderer culls per tile).
__device__ __forceinline__ int build_block_list(const FkOut& fo, BlockEnt* out, uint2* s_cm,
                                                uint2* s_rm, const float4* shp) {
  const int lane = threadIdx.x & 31;
  const TileGrid g(fo.ubox);
  if (g.tx > kMaxBand) return -1;
  const int ty = g.tx > 0 ? g.ntiles / g.tx : 0;
  const int by = (ty + 1) >> 1;  // block rows
  if (ty > kMaxBand || g.tx * by > kMaxTiles) return -1;
  // band masks by ballot: lane j holds primitive j's (and j + 32's) band ranges; one pair
  // of ballots per column / row band
  int c0[2], c1[2], r0[2], r1[2];
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int j = lane + 32 * h;
    c0[h] = r0[h] = 1;
    c1[h] = r1[h] = 0;  // empty
    if (j < kNprim) {
      const int4 b = fo.box[j];
      if (b.x <= b.z) {  // band k covers [g.x0 + 16 k, g.x0 + 16 k + 15] (rows: 8)
        c0[h] = (b.x - g.x0) >> 4;
        c1[h] = (b.z - g.x0) >> 4;
        r0[h] = (b.y - g.y0) >> 3;
        r1[h] = (b.w - g.y0) >> 3;
      }
    }
  }
  static_assert(kTileW == 16 && kTileH == 8, "band shifts assume 16x8 tiles");
  for (int q = 0; q < g.tx; q++) {
    const unsigned int m0 = __ballot_sync(0xffffffffu, c0[0] <= q && q <= c1[0]);
    const unsigned int m1 = __ballot_sync(0xffffffffu, c0[1] <= q && q <= c1[1]);
    if (lane == 0) s_cm[q] = make_uint2(m0, m1);
  }
  for (int q = 0; q < 2 * by; q++) {  // an odd last row of tiles pairs with an empty band
    const unsigned int m0 = __ballot_sync(0xffffffffu, r0[0] <= q && q <= r1[0]);
    const unsigned int m1 = __ballot_sync(0xffffffffu, r0[1] <= q && q <= r1[1]);
    if (lane == 0) s_rm[q] = make_uint2(m0, m1);
  }
  __syncwarp();
  const int nb = g.tx * by;
  int cnt = 0;
  for (int base = 0; base < nb; base += 32) {  // one block per lane
    const int t = base + lane;
    uint2 top = make_uint2(0u, 0u), bot = make_uint2(0u, 0u);
    int X0 = 0, Y0 = 0;
    if (t < nb) {
      const int qy = t / g.tx, qx = t - qy * g.tx;
      X0 = g.x0 + qx * kTileW;
      Y0 = g.y0 + qy * kBlockH;
      HP_CHECK(qx < kMaxBand && 2 * qy + 1 < kMaxBand);
      const uint2 c = s_cm[qx];
      top = tile_mask(c, s_rm[2 * qy], X0, Y0, shp);
      bot = tile_mask(c, s_rm[2 * qy + 1], X0, Y0 + kTileH, shp);
    }
    const bool ne = (top.x | top.y | bot.x | bot.y) != 0;
    const unsigned int bal = __ballot_sync(0xffffffffu, ne);
    if (ne) {
      HP_CHECK(cnt + __popc(bal & ((1u << lane) - 1u)) < kMaxTiles);
      const BlockEnt e = make_block_ent(X0, Y0, split_kinds(top), split_kinds(bot));
      BlockEnt* dst = out + cnt + __popc(bal & ((1u << lane) - 1u));
      dst->a = e.a;
      dst->b = e.b;
    }
    cnt += __popc(bal);
  }
  return cnt;
}

#ifndef HP_PIN
#define HP_PIN(x) pin_u32(x)
#endif
#ifndef HP_FETCH
#define HP_FETCH 2  // renderer blocks a warp takes per shared-counter atomic
#endif
#ifndef HP_FK_PDL
#define HP_FK_PDL 1  // programmatic dependent launch of k_render_persist after k_fk_batch
#endif
#ifndef HP_FK_WARPS
#define HP_FK_WARPS 4  // particles (warps) per k_fk_batch CTA
#endif
constexpr int kFkWarps = HP_FK_WARPS;
static_assert(kFkWarps == 4, "k_fk_batch's work lists assume 4 poses per CTA");
// One CTA of 4 warps scores FK for 4 poses cooperatively, with every phase laid out over
// the CTA's 128 threads so that a warp runs one kind of work (no serialised branches of
// different primitive kinds in a warp, few idle lanes):
//   A  the 4 x 26 pose values and the 4 x 23 sincos (fp64), one per thread
//   B  the 4 x 5 finger chains (fp64), one per thread
//   C  the 4 x 38 boxes and FAST records, sorted by kind: 80 spheres (box + record), 72
//      quadric boxes, 72 quadric records, in passes of 128 threads
//   C' (a pose that may cross z_near: its EXACT records to global memory, warp per pose)
//   C" the 72 quadric records converted to the FAST layout (fp64), one pass
//   D  per warp (= pose): union box, near-plane flag, kc; the record leaves by one bulk
//      copy while the warp builds the pose's block list
#if HP_FKB_PROF
// clock64 stamps of k_fk_batch's phases (CTA 300, thread 0), staged in shared memory
__device__ long long g_fkbprof[16];
__device__ unsigned long long g_fkbcta[1024][2];  // per CTA: globaltimer at start / end
__device__ __forceinline__ unsigned long long fkb_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define FKBPROF(i) \
  if (blockIdx.x == 300 && threadIdx.x == 0) s_fkbp[i] = clock64();
#else
#define FKBPROF(i)
#endif
template <typename PoseT>
__global__ void __launch_bounds__(kFkWarps * 32, 32 / kFkWarps)
    k_fk_batch(const EvalArgs a) {
#if HP_FKB_PROF
  __shared__ long long s_fkbp[16];
#endif
  __shared__ __align__(16) FkScratch s_fk[kFkWarps];
  __shared__ __align__(16) FkOut s_out[kFkWarps];
  __shared__ __align__(16) float4 s_shp[kFkWarps][kNcone];  // cone capsules
  static_assert(sizeof(FkScratch) >= 2 * kMaxBand * sizeof(uint2), "band masks alias s_fk");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#if HP_FK_PDL
  // the renderer (launched with programmatic stream serialisation) may start its prologue
  // on SMs this grid frees; it waits for this grid's completion before reading its output
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  const int p0 = blockIdx.x * kFkWarps;
  const int np = min(kFkWarps, a.n - p0);  // poses of this CTA (the last CTA may be short)
  FKBPROF(0)
#if HP_FKB_PROF
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_fkbcta[blockIdx.x][0] = fkb_gtime();
#endif
  // ---- A: pose values and sincos ----
  if (tid < np * kNdof) {
    const int q = tid / kNdof, d = tid - q * kNdof;
    const double v = (double)static_cast<const PoseT*>(a.poses)[(size_t)(p0 + q) * kNdof + d];
    s_fk[q].h[d] = v;
    if (d >= 3) sincos(v, &s_fk[q].sn[d], &s_fk[q].cs[d]);
  }
  __syncthreads();
  FKBPROF(1)
  // ---- B: finger chains ----
  if (tid < np * 5) {
    const int q = tid / 5, f = tid - q * 5;
    int bad = 0;
    for (int d = 0; d < kNdof; d++) bad |= !isfinite(s_fk[q].h[d]);
    fk_finger_chain(s_fk[q], a.dims, f, bad);
  }
  __syncthreads();
  FKBPROF(2)
  // ---- C: records + boxes, kind-sorted items: the sphere records (EXACT = FAST) and boxes,
  // the quadrics' boxes, then their FAST records straight from the frames (build_fast) ----
  constexpr int kNs = kFkWarps * kCone0, kNq = kFkWarps * (kNprim - kCone0);
  constexpr int kItems = kNs + 2 * kNq;
#pragma unroll 1
  for (int i = tid; i < kItems; i += kFkWarps * 32) {
    if (i < kNs + kNq) {
      int q, j;
      if (i < kNs) {
        q = i / kCone0;
        j = i - q * kCone0;
      } else {
        const int k = i - kNs;
        q = k / (kNprim - kCone0);
        j = kCone0 + k - q * (kNprim - kCone0);
      }
      if (q < np) {
        float zmin;
        if (j < kCone0) {  // a sphere: box (the EXACT record is discarded), then FAST record
          build_prim(j, s_fk[q], a.dims, a.cam, s_out[q].rec[j], s_out[q].box[j], zmin);
          build_fast_sphere(j, s_fk[q], a.dims, s_out[q].rec[j]);
        } else {  // a quadric's EXACT record is not kept here (see C')
          float xr[kRec];
          build_prim(j, s_fk[q], a.dims, a.cam, xr, s_out[q].box[j], zmin,
                     j < kCyl ? &s_shp[q][j - kCone0] : nullptr);
        }
        s_fk[q].nearf[j] = zmin > a.cam.znear * 1.001f;
      }
    } else {
      const int k = i - kNs - kNq;
      const int q = k / (kNprim - kCone0), j = kCone0 + k - q * (kNprim - kCone0);
      if (q < np) build_fast(j, s_fk[q], a.dims, s_out[q].rec[j]);
    }
  }
  // the records were written by every thread of the CTA: each orders its writes before the
  // async proxy (the bulk copy in D) before the barrier
  fence_proxy_async();
  __syncthreads();
  FKBPROF(3)
  // ---- C': a pose that may cross z_near (rare) keeps its EXACT records (global memory) ----
  if (warp < np) {
    int nok = 1;
    for (int j = lane; j < kNprim; j += 32) nok &= s_fk[warp].nearf[j];
    if (!__all_sync(0xffffffffu, nok)) {
      FkExact* xg = static_cast<FkExact*>(a.fkx_g) + p0 + warp;
      for (int j = lane; j < kNprim; j += 32) {
        float zmin;
        int4 box;
        build_prim(j, s_fk[warp], a.dims, a.cam, xg->rec[j], box, zmin, nullptr);
      }
    }
  }
  if (warp >= np) return;  // warp-uniform; only warp-local synchronisation below
  // ---- D: per pose ----
  const int p = p0 + warp;
  FKBPROF(4)
  fk_finish_warp(s_fk[warp], s_out[warp], a.cost.kc_rest);
  FKBPROF(5)
  // the record leaves by one bulk copy while the warp builds the block list: every lane
  // orders its record writes before the async proxy, then lane 0 issues the copy
  fence_proxy_async();
  __syncwarp();
  if (lane == 0)
    bulk_s2g(static_cast<FkOut*>(a.fk_g) + p, &s_out[warp], (uint32_t)sizeof(FkOut));
  uint2* band = reinterpret_cast<uint2*>(&s_fk[warp]);  // FK scratch is dead by now
  const int cnt = build_block_list(s_out[warp],
                                   reinterpret_cast<BlockEnt*>(a.tiles_g) + (size_t)p * kMaxTiles, band,
                                   band + kMaxBand, s_shp[warp]);
  FKBPROF(6)
  __syncwarp();  // the warp's list (and C' record) stores precede lane 0's release
  if (lane == 0) {
    int ntl = cnt;
    if (!s_out[warp].near_ok) {  // some primitive may cross z_near: the exact pass renders it
      const unsigned slot_ = atomicAdd(a.near_count, 1u);
      HP_CHECK(slot_ < (unsigned)a.n);
      a.near_list[slot_] = p;
      ntl = -2;
    }
    a.ntl_g[p] = ntl;
    bulk_wait_all();  // the record's bulk write is complete (and the CTA's shared memory free)
    fence_proxy_async_global();
    // publish: the renderer (already running, PDL) may take pose p from here on
    st_release_u32(a.fk_ready + p, __ldcg(a.fk_epoch));
    FKBPROF(7)
#if HP_FKB_PROF
    if (blockIdx.x < 1024) atomicMax(&g_fkbcta[blockIdx.x][1], fkb_gtime());
    if (blockIdx.x == 300 && threadIdx.x == 0)
      for (int q = 0; q < 8; q++) g_fkbprof[q] = s_fkbp[q];
#endif
  }
}

// NEAR = false: the batch renderer, 16 x 16 warp blocks from k_fk_batch's block list (the
// tensor map's box is 16 x 16).  Particles whose FK found a primitive that may cross z_near
// were queued by k_fk_batch (ntl = -2) and are skipped here; NEAR = true renders exactly
// those (exact-solid path from their EXACT records; 16 x 8 tiles, box 16 x 8)
// in a second, normally empty launch, so the near-plane code never shares a register
// allocation with the hot loop.
#ifndef HP_STATIC_FIRST
#define HP_STATIC_FIRST 1  // CTA i's first poses are kSlots i + b (no atomic on the start path)
#endif
#ifndef HP_SLOTS
#define HP_SLOTS 3  // particle slots per renderer CTA (FK record + block list each)
#endif
constexpr int kSlots = HP_SLOTS;
#ifndef HP_RAY_GLOBAL
#define HP_RAY_GLOBAL 0  // 1: the block renderer reads the ray table through L1, not shared
#endif
// dynamic shared memory of k_render_persist: the ray table (the near pass, or HP_RAY_GLOBAL
// = 0), then the slots' block lists
__host__ __device__ constexpr size_t render_ray_bytes(int W, int H, bool near) {
  return near || !HP_RAY_GLOBAL ? (size_t)ray_floats(W, H) * sizeof(float) : 0;
}
__host__ __device__ constexpr size_t render_dyn_bytes(int W, int H, bool near = false) {
  return render_ray_bytes(W, H, near) + (size_t)kSlots * kMaxTiles * sizeof(BlockEnt);
}
#if HP_TAIL_PROF
// per CTA: globaltimer at entry, then per warp at loop exit (main pass only)
__device__ unsigned long long g_tailprof[1024][1 + 16];
__device__ __forceinline__ unsigned long long tail_time() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif
template <int NW, bool NEAR, bool SUMS>
__global__ void __launch_bounds__(NW * 32, HP_MINB_WARPS / NW)
    k_render_persist(const __grid_constant__ EvalArgs a,
                     const __grid_constant__ CUtensorMap tmap) {
  __shared__ __align__(16) FkOut s_out[kSlots];
  __shared__ __align__(16) FkExact s_x[NEAR ? kSlots : 1];
  __shared__ __align__(128) uint32_t s_obs[NW][kTileW * (NEAR ? kTileH : kBlockH)];
  __shared__ __align__(8) uint64_t s_bar[NW];
  __shared__ __align__(8) uint64_t s_full[kSlots];
  // per-warp partial sums of the particle in slot b: r_m, o_s AND r_m, numerator lo, hi
  __shared__ __align__(16) uint4 s_part[kSlots][NW];
  __shared__ unsigned int s_pboth[kSlots][NW];  // both-defined count (SUMS only)
  __shared__ int s_next[kSlots], s_done[kSlots], s_pid[kSlots], s_ntl[kSlots];
  __shared__ int s_fkdone;  // k_fk_batch's grid is known complete (griddepcontrol.wait ran)
  extern __shared__ float s_ray[];
  // the slots' block lists follow the ray table (16-byte aligned: ray_floats is a multiple
  // of 4)
  BlockEnt(*s_tiles)[kMaxTiles] = reinterpret_cast<BlockEnt(*)[kMaxTiles]>(
      reinterpret_cast<char*>(s_ray) + render_ray_bytes(a.cam.W, a.cam.H, NEAR));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if HP_TAIL_PROF
  if (!NEAR && threadIdx.x == 0 && blockIdx.x < 1024) {
    g_tailprof[blockIdx.x][0] = tail_time();
    for (int q = 9; q < 17; q++) g_tailprof[blockIdx.x][q] = 0;
  }
#endif
  const float* s_dx = s_ray;
  const float* s_dy = s_ray + ray_dx_len(a.cam.W);
  unsigned int* const counter = a.pcount + (NEAR ? 2 : 0);  // [taken, CTAs exited]
  // one thread: take the next particle (k: a counter value already taken, or -1) and pull
  // its FK record + tile list into slot b.  The record's copy starts before the list
  // length is known (expect_tx without arrival; the arrival follows with the list bytes)
  unsigned epoch = 0;  // thread 0: this launch's FK epoch (the first poses' flags)
  // ready: the pose's FK is known to be published (after griddepcontrol.wait); otherwise
  // (the first poses, taken while k_fk_batch may still run) wait for its flag first
  auto issue = [&](int b, int kt, bool ready) {
    int p = a.n;
    const unsigned k =
        kt >= 0 ? (unsigned)kt
                : atomicAdd(counter, 1u) +
                      (!NEAR && HP_STATIC_FIRST ? (unsigned)kSlots * gridDim.x : 0u);
    if (NEAR) {
      if (k < __ldcg(a.near_count)) p = __ldcg(a.near_list + k);
    } else {
      p = (int)k;
    }
    s_pid[b] = p;
    if (p < a.n) {
      if (NEAR) {
        mbar_expect_tx(&s_full[b], (uint32_t)(sizeof(FkOut) + sizeof(FkExact)));
        bulk_g2s(&s_out[b], static_cast<const FkOut*>(a.fk_g) + p, (uint32_t)sizeof(FkOut),
                 &s_full[b]);
        bulk_g2s(&s_x[NEAR ? b : 0], static_cast<const FkExact*>(a.fkx_g) + p,
                 (uint32_t)sizeof(FkExact), &s_full[b]);
        s_ntl[b] = -1;  // NEAR: cull every tile
        return;
      }
      if (!ready) {  // wait for this launch's epoch in the pose's flag
        while (ld_acquire_u32(a.fk_ready + p) != epoch) __nanosleep(256);
        fence_proxy_async_global();  // the record's bulk read below sees FK's bulk write
      }
      mbar_expect_tx_only(&s_full[b], (uint32_t)sizeof(FkOut));
      bulk_g2s(&s_out[b], static_cast<const FkOut*>(a.fk_g) + p, (uint32_t)sizeof(FkOut),
               &s_full[b]);
      const int ntl = __ldcg(a.ntl_g + p);
      s_ntl[b] = ntl;
      // ntl == -2: queued for the near-plane pass (the record is not used); -1: no list
      const uint32_t lb = ntl > 0 ? (uint32_t)ntl * (uint32_t)sizeof(BlockEnt) : 0u;
      mbar_expect_tx(&s_full[b], lb);
      if (lb)
        bulk_g2s(s_tiles[b], reinterpret_cast<const BlockEnt*>(a.tiles_g) + (size_t)p * kMaxTiles,
                 lb, &s_full[b]);
    } else {
#if HP_TAIL_PROF
      if (!NEAR && blockIdx.x < 1024 && g_tailprof[blockIdx.x][16] == 0)
        g_tailprof[blockIdx.x][16] = tail_time();  // the first terminator claim
#endif
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
    for (int b = 0; b < kSlots; b++) {
      mbar_init(&s_full[b], 1);
      s_next[b] = 0;
      s_done[b] = 0;
    }
    fence_mbar_init();
    prefetch_tmap(&tmap);
    s_fkdone = 0;
    // the first poses, one atomic; with PDL this grid starts on SMs k_fk_batch frees, so
    // each first pose waits for its own FK flag instead of the whole FK grid (NEAR: the
    // previous grid is complete first)
#if HP_FK_PDL
    if (NEAR) asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    // this launch's FK epoch (advanced only by the previous launch's end); needed only when
    // the first poses wait for their flags
    epoch = NEAR || !a.fk_wait ? 0u : __ldcg(a.fk_epoch);
    const unsigned k0 = NEAR || !HP_STATIC_FIRST ? atomicAdd(counter, (unsigned)kSlots)
                                                 : (unsigned)kSlots * blockIdx.x;
    for (int b = 0; b < kSlots; b++) issue(b, (int)(k0 + b), NEAR || !HP_FK_PDL || !a.fk_wait);
  }
  if (NEAR || !HP_RAY_GLOBAL) {
    const int n4 = ray_floats(a.cam.W, a.cam.H) / 4;
    for (int i = threadIdx.x; i < n4; i += NW * 32)
      reinterpret_cast<float4*>(s_ray)[i] = __ldg(reinterpret_cast<const float4*>(a.ray) + i);
  }
  __syncthreads();

  uint32_t phase = 0;
  const uint32_t obs_s = HP_PIN(smem_u32(s_obs[warp])), bar_s = HP_PIN(smem_u32(&s_bar[warp]));
  const uint32_t dx_s = HP_PIN(smem_u32(s_dx + (lane & 15)));
  const uint32_t dy_s = HP_PIN(smem_u32(s_dy + 4 * (lane >> 4)));
#if HP_RAY_GLOBAL
  // the lane's column / first row in the global ray table (L1-resident)
  const float* ray_x = a.ray + (lane & 15);
  const float4* ray_y = reinterpret_cast<const float4*>(a.ray + ray_dx_len(a.cam.W)) + (lane >> 4);
#endif
  // the lane's first observation pixel (column lane & 15, row lane >> 4) and the slots'
  // shared bases, computed once (the compiler otherwise re-derives them per block)
  const uint32_t obs_ls = HP_PIN(obs_s + 4u * ((lane >> 4) * kTileW + (lane & 15)));
  const uint32_t tiles_s0 = smem_u32(s_tiles[0]), rec_s0 = smem_u32(s_out[0].rec);
  const uint32_t next_s0 = smem_u32(&s_next[0]);
  for (int i = 0;; i++) {
    const int b = kSlots == 2 ? (i & 1) : i % kSlots;
    const uint32_t par = (kSlots == 2 ? (i >> 1) : i / kSlots) & 1;
#if HP_SLOT_SLEEP
    mbar_wait_sleep(&s_full[b], par);  // suspended, not spinning on issue slots
#else
    mbar_wait(&s_full[b], par);
#endif
    const int p = s_pid[b];
    if (p >= a.n) break;
    const FkOut& fo = s_out[b];
    const int nlist = s_ntl[b];
    const int yoff = frame_of(a, p) * a.cam.H;
    TileSums acc;
    if (nlist != -2) {
      // NEAR: every 16 x 8 tile of the union grid, culled here; otherwise the block list,
      // or (a close-up pose with more blocks than the list holds) every 16 x 16 block of
      // the union grid, both halves culled here.  The union grid (and its division) only
      // where it is used.
      TileGrid g;
      int nt = nlist;
      if (NEAR || nlist < 0) {
        g = TileGrid(fo.ubox);
        nt = NEAR ? g.ntiles : g.tx * ((g.ntiles / (g.tx > 0 ? g.tx : 1) + 1) >> 1);
      }
      // the slot's shared addresses pinned in registers: the primitive loops address
      // records as [rec_s + index * record size] instead of re-deriving the slot base
      const uint32_t next_s = HP_PIN(next_s0 + 4u * b);
      const uint32_t tiles_s = HP_PIN(tiles_s0 + (uint32_t)sizeof(s_tiles[0]) * b);
      const uint32_t rec_s = HP_PIN(rec_s0 + (uint32_t)sizeof(FkOut) * b);
      // blocks are taken HP_FETCH at a time (one shared atomic per HP_FETCH blocks)
      constexpr int kF = NEAR ? 1 : HP_FETCH;
      int t = warp_fetch_add<kF>(next_s), tend = t + kF;  // this warp's blocks [t, tend)
      while (t < nt) {
        int tn = t + 1;
        if (tn >= tend) {  // the next range, fetched early
          tn = warp_fetch_add<kF>(next_s);
          tend = tn + kF;
        }
        if (NEAR) {
          int X0, Y0;
          g.origin(t, X0, Y0);
          const uint3 km = cull_tile(fo, X0, Y0);
          if (km.x | km.y | km.z)
            do_tile<kModeCost, true, SUMS, 1>(a, &tmap, fo, &s_x[NEAR ? b : 0], X0, Y0, km,
                                              obs_s, bar_s, phase, dx_s, dy_s, acc, yoff);
        } else {
          BlockEnt ent;
          bool any = true;  // listed blocks are non-empty
          if (nlist >= 0) {
            HP_CHECK(t >= 0 && t < kMaxTiles);
            ent.a = lds_u4_nv(tiles_s + (uint32_t)sizeof(BlockEnt) * t);
            ent.b = lds_u4_nv(tiles_s + (uint32_t)sizeof(BlockEnt) * t + 16u);
          } else {
            const int qy = t / g.tx, qx = t - qy * g.tx;
            const int X0 = g.x0 + qx * kTileW, Y0 = g.y0 + qy * kBlockH;
            const uint3 kt = cull_tile(fo, X0, Y0), kb = cull_tile(fo, X0, Y0 + kTileH);
            ent = make_block_ent(X0, Y0, kt, kb);
            any = (kt.x | kt.y | kt.z | kb.x | kb.y | kb.z) != 0;
          }
          if (any)
#if HP_RAY_GLOBAL
            do_block<SUMS, true>(a, &tmap, rec_s, ent, obs_s, obs_ls, bar_s, phase, dx_s, dy_s,
                                 acc, yoff, ray_x, ray_y);
#else
            do_block<SUMS>(a, &tmap, rec_s, ent, obs_s, obs_ls, bar_s, phase, dx_s, dy_s, acc,
                           yoff);
#endif
        }
        t = tn;
      }
    }
    unpack_counts(acc);
    warp_reduce<SUMS>(acc);
    // publish this warp's partial sums; the last warp to arrive (acq_rel counter: its
    // acquire sees every other warp's partials) reduces them and refills the slot
    int last = 0;
    if (lane == 0) {
      s_part[b][warp] = make_uint4(acc.rm, acc.and_, (unsigned int)acc.num,
                                   (unsigned int)(acc.num >> 32));
      if (SUMS) s_pboth[b][warp] = acc.both;
      last = atom_add_acq_rel_cta(&s_done[b], 1) == NW - 1;
    }
    if (__shfl_sync(0xffffffffu, last, 0)) {
      __syncwarp();  // lane 0's acquire orders the other lanes' reads below
      TileSums t;
      if (lane < NW) {
        const uint4 v = s_part[b][lane];
        t.rm = v.x;
        t.and_ = v.y;
        t.num = ((unsigned long long)v.w << 32) | v.z;
        if (SUMS) t.both = s_pboth[b][lane];
      }
      warp_reduce<SUMS>(t);
      if (lane == 0) {
        const unsigned long long v[4] = {t.rm, t.and_, t.num, t.both};
        const double kc = fo.kc;  // read before the refill overwrites the slot
        s_next[b] = 0;
        s_done[b] = 0;
        fence_proxy_async();  // every warp's generic reads of slot b precede the refill
#if HP_FK_PDL
        // k_fk_batch complete before this refill reads its outputs: the first refilling
        // thread of the CTA waits for the grid (griddepcontrol.wait) and says so through
        // shared memory (release / acquire at CTA scope), later ones only read that
        if (!NEAR && ld_acquire_cta_s32(&s_fkdone) == 0) {
          asm volatile("griddepcontrol.wait;" ::: "memory");
          st_release_cta_s32(&s_fkdone, 1);
        }
#endif
        issue(b, -1, true);   // particle i + kSlots into the freed slot (before the cost:
                              // the refill's latency is the warps' critical path)
        if (nlist != -2) finalize_cost(a, p, v, kc);  // queued ones: the near pass
#if HP_TAIL_PROF
        if (!NEAR && blockIdx.x < 1024) {  // smid, particles, blocks, last two finish times
          unsigned long long* r = g_tailprof[blockIdx.x];
          unsigned smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          r[9] = smid;
          r[10] += 1;
          r[11] += nlist >= 0 ? nlist : 1000;
          r[12] = r[13];
          r[13] = tail_time();
          r[14] = p;
          r[15] = (unsigned)nlist;
        }
#endif
      }
    }
    __syncwarp();
  }
#if HP_TAIL_PROF
  if (!NEAR && lane == 0 && blockIdx.x < 1024) g_tailprof[blockIdx.x][1 + warp] = tail_time();
#endif
  // the last CTA to leave resets the counters for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(counter + 1, 1u) == gridDim.x - 1) {
      counter[0] = 0;
      counter[1] = 0;
      if (NEAR) *a.near_count = 0;
      else *a.fk_epoch += 1u;  // the next batch launch's flags
      __threadfence();
    }
  }
}


}  // namespace hp
