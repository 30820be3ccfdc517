// Fused sm_100a executor for the 3D heat chain (BASELINE.json configs[1];
// specs/heat3d.lf): fluxx, fluxy, fluxz -> divupd, fp64, periodic.
//
// HFAV contracts fx to a scalar carry, fy to 2 rows and fz to 2 planes
// (SURVEY.md App. A).  On B200 the same elision is done as 2.5-D streaming:
// one CTA owns a 64 x 16 (i, j) column of the grid and marches along k.
//   * a producer warp streams u planes (tile + 1-cell halo, 66 x 18 doubles)
//     into an S-stage shared-memory ring with TMA (cp.async.bulk.tensor.3d),
//     completion signalled on mbarriers; consumers free slots on a second
//     mbarrier set, so loads run S-2 planes ahead of the math;
//   * 8 consumer warps compute two rows x two cells each; fx/fy live only in
//     registers (recomputed per cell from the staged plane), fz(k-1) is the
//     register carry of the previous plane -- no intermediate touches HBM;
//   * the output is written once, and the periodic ghost layer of the goal
//     buffer is refilled by the CTAs that own the wrapped cells, so the next
//     step can stream the buffer straight back in (iterate: pairs).
// Compulsory traffic: 8 B read + 8 B written per cell-update.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "../../userkernels/stencil_kernels.h"
#include "common.cuh"
#include "exec.hpp"

namespace lfx {
namespace {

constexpr int TX = 64;                 // cells along i per CTA (32 lanes x 2)
constexpr int CWARPS = 8;              // consumer warps
constexpr int THREADS = (CWARPS + 1) * 32;
constexpr int LD = TX + 2;             // staged row length (halo 1 each side)

// Tunable shape: RPW rows per consumer warp (tile height TY = 8*RPW), S ring
// slots, KCH planes per work unit.
template <int RPW_, int S_, int KCH_>
struct Cfg {
  static constexpr int RPW = RPW_, S = S_, KCH = KCH_;
  static constexpr int TY = CWARPS * RPW;
  static constexpr int ROWS = TY + 2;
  static constexpr int STAGE_TX = LD * ROWS * 8;                    // bytes TMA delivers
  static constexpr int STAGE_BYTES = (STAGE_TX + 127) / 128 * 128;  // 128-B aligned slots
  static constexpr int SMEM = S * STAGE_BYTES + 2 * S * 8 + 128;
};

struct Params {
  int ni, nj, nk;       // interior sizes of this launch's domain (slab planes for multi-GPU)
  int k_lo, k_hi;       // planes this launch computes
  long long pj, pk;     // element strides of the (nk+2, nj+2, ni+2) layout
  int tiles_x, tiles;   // column tiles
  int kchunks;          // work units along k per column
  int units;            // tiles * kchunks
  int wrap_i, wrap_j, wrap_k;  // refill periodic ghosts along this dim
  int patch;                   // two-step pass: patch periodic images on face tiles
  int store_policy;            // L2 policy of the output stores (l2_store_policy)
};

// A row's two output columns (gi0, gi0 + 32 of cell row (k, j)) and their
// periodic images in the ghost layer: every combination of the own and the
// wrapped index along k, j and i -- the face images, and the edge and corner
// images as compositions of the face maps (the ghost fill of the oracle,
// oracle/stencils.c) -- so every cell of the goal buffer is written.  A single
// interior row / plane is the image of both ghost faces.
__device__ __noinline__ void store_ghost_images(double* out, long long pk, long long pj, int ni, int nk_, int nj_,
                                                bool wrap_k, bool wrap_j, int k, int j, int gi0, double v0, double v1,
                                                bool wrap_lo_i, bool wrap_hi_i, uint64_t pol) {
  int ks[3], js[3], nk = 0, nj = 0;
  ks[nk++] = k + 1;
  if (wrap_k && k == 0) ks[nk++] = nk_ + 1;
  if (wrap_k && k == nk_ - 1) ks[nk++] = 0;
  js[nj++] = j + 1;
  if (wrap_j && j == 0) js[nj++] = nj_ + 1;
  if (wrap_j && j == nj_ - 1) js[nj++] = 0;
  for (int a = 0; a < nk; ++a)
    for (int b = 0; b < nj; ++b) {
      if (a == 0 && b == 0) continue;  // the cell's own row: stored by the caller
      double* rowp = out + (long long)ks[a] * pk + (long long)js[b] * pj + 1;  // logical i = 0
      st_hint(rowp + gi0, v0, pol);
      st_hint(rowp + gi0 + 32, v1, pol);
      if (wrap_lo_i) st_hint(rowp + ni, v0, pol);
      if (wrap_hi_i) st_hint(rowp - 1, v1, pol);
    }
}
__device__ __forceinline__ void store_images(double* out, const Params& p, int k, int j, int gi0, double v0,
                                             double v1, bool wrap_lo_i, bool wrap_hi_i, uint64_t pol) {
  double* rowp = out + (long long)(k + 1) * p.pk + (long long)(j + 1) * p.pj + 1;  // logical i = 0
  st_hint(rowp + gi0, v0, pol);
  st_hint(rowp + gi0 + 32, v1, pol);
  if (wrap_lo_i) st_hint(rowp + p.ni, v0, pol);
  if (wrap_hi_i) st_hint(rowp - 1, v1, pol);
  // rows on a wrapped k or j face also have images in the ghost planes / rows
  // (out of line: only the boundary rows take it)
  if ((p.wrap_k && (k == 0 || k == p.nk - 1)) || (p.wrap_j && (j == 0 || j == p.nj - 1)))
    store_ghost_images(out, p.pk, p.pj, p.ni, p.nk, p.nj, p.wrap_k, p.wrap_j, k, j, gi0, v0, v1, wrap_lo_i, wrap_hi_i,
                       pol);
}

// Work unit u = (k chunk, column tile), k-chunk major: at any moment all
// persistent CTAs are inside the same one or two k chunks, so the halo rows a
// CTA stages were staged moments earlier by its neighbours and hit in L2.
struct Unit {
  int i0, j0, k0, kc;
};
template <int TY>
__device__ __forceinline__ Unit unit_of(const Params& p, int u) {
  const int kb = u / p.tiles, t = u - kb * p.tiles;
  Unit r;
  r.i0 = (t % p.tiles_x) * TX;
  r.j0 = (t / p.tiles_x) * TY;
  const int nk = p.k_hi - p.k_lo;
  r.k0 = p.k_lo + static_cast<int>((long long)kb * nk / p.kchunks);
  r.kc = p.k_lo + static_cast<int>((long long)(kb + 1) * nk / p.kchunks) - r.k0;
  return r;
}

template <class K>
__global__ void __launch_bounds__(THREADS, 2)
    heat3d_fused(const __grid_constant__ CUtensorMap tin, double* __restrict__ out, const Params p) {
  constexpr int RPW = K::RPW, S = K::S, TY = K::TY, STAGE_BYTES = K::STAGE_BYTES, STAGE_TX = K::STAGE_TX;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE_BYTES);
  uint64_t* empty = full + S;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CWARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == CWARPS) {
    // ---------------- producer: one elected lane streams planes ----------------
    if (lane == 0) {
      tma_prefetch_desc(&tin);
      int g = 0;  // running plane counter across this CTA's units
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const Unit w = unit_of<TY>(p, u);
        for (int q = 0; q < w.kc + 2; ++q, ++g) {
          const int slot = g % S;
          if (g >= S) mbar_wait(&empty[slot], ((g / S) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[slot], STAGE_TX);
          // storage coordinates = logical + 1 (terminal base is -1 in every dim):
          // box origin at logical (i0-1, j0-1, k0-1+q)
          tma_load_3d(ring + slot * STAGE_BYTES, &tin, &full[slot], w.i0, w.j0, w.k0 + q);
        }
      }
    }
    return;
  }

  // ---------------- consumers: warp w owns rows RPW*w .. RPW*w+RPW-1; lane owns cells lane, lane+32
  const uint64_t pol = l2_store_policy(p.store_policy);
  const int r0 = RPW * warp;
  auto stage = [&](int g) { return reinterpret_cast<const double*>(ring + (g % S) * STAGE_BYTES); };
  auto at = [&](const double* sp, int row, int col) { return sp[row * LD + col]; };
  int g = 0;
  for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
    const Unit w = unit_of<TY>(p, u);
    double uprev[RPW][2], ucur[RPW][2], unext[RPW][2];
    mbar_wait(&full[g % S], (g / S) & 1);
    {
      const double* sp = stage(g);
#pragma unroll
      for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) uprev[r][c] = at(sp, r0 + r + 1, lane + 32 * c + 1);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[g % S]);
    ++g;
    mbar_wait(&full[g % S], (g / S) & 1);
    {
      const double* sp = stage(g);
#pragma unroll
      for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) ucur[r][c] = at(sp, r0 + r + 1, lane + 32 * c + 1);
    }
    const int gi0 = w.i0 + lane;  // logical i of cell c=0 (c=1 is gi0+32)
    const bool wrap_lo_i = p.wrap_i && gi0 == 0;               // owns cell 0
    const bool wrap_hi_i = p.wrap_i && gi0 + 32 == p.ni - 1;   // owns cell ni-1
    for (int kk = 0; kk < w.kc; ++kk, ++g) {
      const int gn = g + 1;
      mbar_wait(&full[gn % S], (gn / S) & 1);
      const double* sn = stage(gn);
#pragma unroll
      for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) unext[r][c] = at(sn, r0 + r + 1, lane + 32 * c + 1);
      const double* sp = stage(g);
      const int k = w.k0 + kk;
      double o[RPW][2];
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const int row = r0 + r + 1;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int col = lane + 32 * c + 1;
          const double uc = ucur[r][c];
          const double uw = at(sp, row, col - 1);
          const double ue = at(sp, row, col + 1);
          const double un = r + 1 < RPW ? ucur[r + 1 < RPW ? r + 1 : r][c] : at(sp, row + 1, col);
          const double us = r > 0 ? ucur[r > 0 ? r - 1 : r][c] : at(sp, row - 1, col);
          double fxp, fxm, fyp, fym, fzp, fzm;
          face_flux(ue, uc, &fxp);
          face_flux(uc, uw, &fxm);
          face_flux(un, uc, &fyp);
          face_flux(uc, us, &fym);
          face_flux(unext[r][c], uc, &fzp);
          face_flux(uc, uprev[r][c], &fzm);
          heat_divupd(uc, fxp, fxm, fyp, fym, fzp, fzm, &o[r][c]);
        }
      }
      // plane k fully consumed: hand the slot back to the producer before the stores
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[g % S]);
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const int j = w.j0 + r0 + r;
        store_images(out, p, k, j, gi0, o[r][0], o[r][1], wrap_lo_i, wrap_hi_i, pol);
      }
#pragma unroll
      for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uprev[r][c] = ucur[r][c];
          ucur[r][c] = unext[r][c];
        }
    }
    // the unit's last staged plane (k0+kc) was only read for centres
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[g % S]);
    ++g;
  }
}

// ---------------------------------------------------------------------------
// Temporal blocking: two time steps per pass over the grid (the iterate pair
// of the chain fused in time, as HFAV fuses the chain's kernels in space).
// A CTA owns a 64 x 16 column tile and marches k; per plane it computes the
// first step (A) on the tile plus a one-cell ring (66 x 18) from the staged
// input (tile plus a two-cell ring, 70 x 20 from an aligned origin), keeps
// three A planes in shared memory, and computes the second step (B) on the
// tile from them.  Periodicity: k planes are loaded wrapped; on the tiles
// that touch an i/j face every staged cell outside the domain is replaced by
// its periodic image from the interior, so the pass never reads the input's
// ghost layer.  HBM: 8 B read + 8 B written per two cell-updates.
// ---------------------------------------------------------------------------
namespace tb {
constexpr int TY = 16;                  // B tile rows (8 consumer warps x 2)
constexpr int AX = TX + 2, AY = TY + 2;   // A ring tile: logical i0-1.., j0-1..
constexpr int LDI = TX + 6, RI = TY + 4;  // staged input: logical i0-3.., j0-2..
constexpr int STAGE_TX = LDI * RI * 8;
constexpr int STAGE_BYTES = (STAGE_TX + 127) / 128 * 128;
constexpr int APLANE = AX * AY;
template <int S_, int KCH_>
struct Cfg {
  static constexpr int S = S_, KCH = KCH_;
  static constexpr int SMEM = S * STAGE_BYTES + 4 * APLANE * 8 + (3 * S + 8) * 8 + 128;
};
__device__ __forceinline__ int wrapn(int x, int n) { return x < 0 ? x + n : (x >= n ? x - n : x); }
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"r"(CWARPS * 32) : "memory"); }

// Warp-specialised pipeline (no CTA-wide barrier): warp 8 streams input
// planes by TMA; warps 0-3 compute first-step planes A into a 4-slot ring;
// warps 4-7 compute the second step B from three A planes and store.
// Barriers: full/empty (input ring, producer <-> A warps), afull/aempty
// (A ring, A warps <-> B warps); A warps also patch the periodic images on
// face tiles (named barrier among the four of them).
constexpr int AW = 4, BW = 4;  // A and B warps
constexpr int THREADS2 = (AW + BW + 2) * 32;  // + TMA producer warp + patch warp
constexpr int ASLOTS = 4;
template <class K>
__global__ void __launch_bounds__(THREADS2, 2)
    heat3d_fused2(const __grid_constant__ CUtensorMap tin, const double* __restrict__ in, double* __restrict__ out,
                  const Params p) {
  constexpr int S = K::S;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;
  double* aring = reinterpret_cast<double*>(smem + S * STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE_BYTES + ASLOTS * APLANE * 8);
  uint64_t* empty = full + S;
  uint64_t* afull = empty + S;
  uint64_t* aempty = afull + ASLOTS;
  uint64_t* pfull = aempty + ASLOTS;  // stage landed and (face tiles) patched
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], AW);
    }
    for (int s = 0; s < ASLOTS; ++s) {
      mbar_init(&afull[s], AW);
      mbar_init(&aempty[s], BW);
    }
    for (int s = 0; s < S; ++s) mbar_init(&pfull[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto stage = [&](int g) { return reinterpret_cast<double*>(ring + (g % S) * STAGE_BYTES); };
  if (warp == AW + BW) {
    // ---------------- producer warp: streams input planes k0-2 .. k0+kc+1
    // (wrapped along k) by TMA, as far ahead as the ring allows
    if (lane == 0) {
      tma_prefetch_desc(&tin);
      int g = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const Unit w = unit_of<TY>(p, u);
        for (int q = 0; q < w.kc + 4; ++q, ++g) {
          const int slot = g % S;
          if (g >= S) mbar_wait(&empty[slot], ((g / S) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[slot], STAGE_TX);
          // storage = logical + 1: origin logical (i0-3, j0-2, k) -> storage (i0-2, j0-1, k+1)
          tma_load_3d(ring + slot * STAGE_BYTES, &tin, &full[slot], w.i0 - 2, w.j0 - 1,
                      wrapn(w.k0 - 2 + q, p.nk) + 1);
        }
      }
    }
    return;
  }
  if (warp == AW + BW + 1) {
    // ---------------- patch warp: publishes each landed plane on pfull, after
    // replacing (on face tiles) the staged cells outside the domain by their
    // periodic images -- so the patch's global loads stay off the A warps
    int g = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const Unit w = unit_of<TY>(p, u);
      const bool lo_i = w.i0 == 0, hi_i = w.i0 + TX == p.ni, lo_j = w.j0 == 0, hi_j = w.j0 + TY == p.nj;
      const bool face = p.patch && (lo_i || hi_i || lo_j || hi_j);
      for (int q = 0; q < w.kc + 4; ++q, ++g) {
        const int slot = g % S;
        mbar_wait(&full[slot], (g / S) & 1);
        if (face) {
          double* st = stage(g);
          const long long kp = (long long)(wrapn(w.k0 - 2 + q, p.nk) + 1) * p.pk;
          auto src = [&](int r, int c) {
            const int i = w.i0 - 3 + c, j = w.j0 - 2 + r;
            return __ldg(in + kp + (long long)(wrapn(j, p.nj) + 1) * p.pj + wrapn(i, p.ni) + 1);
          };
          // rows outside in j (two per face), columns outside in i (three per
          // face): every load issued before any store, one latency per plane
          constexpr int MR = (2 * LDI + 31) / 32, MC = (3 * RI + 31) / 32;
          double vr[2][MR], vc[2][MC];
#pragma unroll
          for (int m = 0; m < MR; ++m) {
            const int e = lane + 32 * m;
            if (e < 2 * LDI) {
              if (lo_j) vr[0][m] = src(e / LDI, e % LDI);
              if (hi_j) vr[1][m] = src(RI - 2 + e / LDI, e % LDI);
            }
          }
#pragma unroll
          for (int m = 0; m < MC; ++m) {
            const int e = lane + 32 * m;
            if (e < 3 * RI) {
              if (lo_i) vc[0][m] = src(e % RI, e / RI);
              if (hi_i) vc[1][m] = src(e % RI, LDI - 3 + e / RI);
            }
          }
#pragma unroll
          for (int m = 0; m < MR; ++m) {
            const int e = lane + 32 * m;
            if (e < 2 * LDI) {
              if (lo_j) st[(e / LDI) * LDI + e % LDI] = vr[0][m];
              if (hi_j) st[(RI - 2 + e / LDI) * LDI + e % LDI] = vr[1][m];
            }
          }
#pragma unroll
          for (int m = 0; m < MC; ++m) {
            const int e = lane + 32 * m;
            if (e < 3 * RI) {
              if (lo_i) st[(e % RI) * LDI + e / RI] = vc[0][m];
              if (hi_i) st[(e % RI) * LDI + LDI - 3 + e / RI] = vc[1][m];
            }
          }
          fence_proxy_async();  // generic writes before the slot's next TMA refill
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[slot]);
      }
    }
    return;
  }
  int gi = 0, ga = 0;  // running input-plane and A-plane counters
  if (warp < AW) {
    // ---------------- A warps: first step on the 66 x 18 ring tile.  Thread
    // t owns cells t + 128 m for the whole unit: the k-1 and k centres stay in
    // registers, so a plane costs one centre + four in-plane loads per cell.
    constexpr int MA = (APLANE + AW * 32 - 1) / (AW * 32);
    const int tid = threadIdx.x;  // 0..127
    auto off = [&](int m) {
      const int e = min(tid + AW * 32 * m, APLANE - 1);
      const int bb = e / AX, aa = e - bb * AX;
      return (bb + 1) * LDI + aa + 2;
    };
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const Unit w = unit_of<TY>(p, u);
      double pv[MA], cv[MA];  // centres of input planes q-2, q-1
      for (int q = 0; q < w.kc + 4; ++q) {
        const int g = gi + q;
        mbar_wait(&pfull[g % S], (g / S) & 1);
        const double* sq = stage(g);
        if (q < 2) {
#pragma unroll
          for (int m = 0; m < MA; ++m) (q == 0 ? pv : cv)[m] = sq[off(m)];
          if (q == 0) {  // plane 0 lives on in registers only
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[g % S]);
          }
          continue;
        }
        // A(q-1) from planes q-2 (registers), q-1 (centres + in-plane), q (centres)
        const int ai = ga + q - 2;
        if (ai >= ASLOTS) mbar_wait(&aempty[ai % ASLOTS], ((ai / ASLOTS) & 1) ^ 1);
        const double* sc = stage(g - 1);
        double* ao = aring + (ai % ASLOTS) * APLANE;
#pragma unroll
        for (int m = 0; m < MA; ++m) {
          const int e = tid + AW * 32 * m;
          const int o = off(m);
          const double uc = cv[m], up = sq[o];
          double fxp, fxm, fyp, fym, fzp, fzm, r;
          face_flux(sc[o + 1], uc, &fxp);
          face_flux(uc, sc[o - 1], &fxm);
          face_flux(sc[o + LDI], uc, &fyp);
          face_flux(uc, sc[o - LDI], &fym);
          face_flux(up, uc, &fzp);
          face_flux(uc, pv[m], &fzm);
          heat_divupd(uc, fxp, fxm, fyp, fym, fzp, fzm, &r);
          if (e < APLANE) ao[e] = r;
          pv[m] = uc;
          cv[m] = up;
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&afull[ai % ASLOTS]);
          mbar_arrive(&empty[(g - 1) % S]);  // plane q-1's in-plane reads are done
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[(gi + w.kc + 3) % S]);
      gi += w.kc + 4;
      ga += w.kc + 2;
    }
    return;
  }
  // ---------------- B warps: second step on the 64 x 16 tile, 4 rows x 2
  // cells per lane; the A(q-1) and A(q) centres of the lane's cells stay in
  // registers
  const int wb = warp - AW;
  const uint64_t pol = l2_evict_first_policy();
  for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
    const Unit w = unit_of<TY>(p, u);
    const int gi0 = w.i0 + lane;
    const bool wrap_lo_i = p.wrap_i && gi0 == 0;
    const bool wrap_hi_i = p.wrap_i && gi0 + 32 == p.ni - 1;
    double am[4][2], ac[4][2];
    for (int q = 2; q <= w.kc + 1; ++q) {
      // B(q) from A(q-1), A(q), A(q+1) = A-ring indices ga+q-2, ga+q-1, ga+q
      const int a0 = ga + q - 2;
      if (q == 2) {
        for (int d = 0; d < 2; ++d) mbar_wait(&afull[(a0 + d) % ASLOTS], ((a0 + d) / ASLOTS) & 1);
        const double* s0 = aring + (a0 % ASLOTS) * APLANE;
        const double* s1 = aring + ((a0 + 1) % ASLOTS) * APLANE;
#pragma unroll
        for (int rr = 0; rr < 4; ++rr)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int o = (4 * wb + rr + 1) * AX + lane + 32 * c + 1;
            am[rr][c] = s0[o];
            ac[rr][c] = s1[o];
          }
      }
      mbar_wait(&afull[(a0 + 2) % ASLOTS], ((a0 + 2) / ASLOTS) & 1);
      const double* sc = aring + ((a0 + 1) % ASLOTS) * APLANE;
      const double* sp = aring + ((a0 + 2) % ASLOTS) * APLANE;
      const int k = w.k0 - 2 + q;
      double o2[4][2];
#pragma unroll
      for (int rr = 0; rr < 4; ++rr)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int o = (4 * wb + rr + 1) * AX + lane + 32 * c + 1;
          const double uc = ac[rr][c], up = sp[o];
          double fxp, fxm, fyp, fym, fzp, fzm;
          face_flux(sc[o + 1], uc, &fxp);
          face_flux(uc, sc[o - 1], &fxm);
          face_flux(sc[o + AX], uc, &fyp);
          face_flux(uc, sc[o - AX], &fym);
          face_flux(up, uc, &fzp);
          face_flux(uc, am[rr][c], &fzm);
          heat_divupd(uc, fxp, fxm, fyp, fym, fzp, fzm, &o2[rr][c]);
          am[rr][c] = uc;
          ac[rr][c] = up;
        }
      // A(q-1) lives on in registers only
      __syncwarp();
      if (lane == 0) mbar_arrive(&aempty[a0 % ASLOTS]);
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const int j = w.j0 + 4 * wb + rr;
        store_images(out, p, k, j, gi0, o2[rr][0], o2[rr][1], wrap_lo_i, wrap_hi_i, pol);
      }
    }
    // the unit's last two A planes were only read by its last B planes
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&aempty[(ga + w.kc) % ASLOTS]);
      mbar_arrive(&aempty[(ga + w.kc + 1) % ASLOTS]);
    }
    ga += w.kc + 2;
  }
}
}  // namespace tb

struct Variant {
  const char* name;
  int ty, kch, smem;
  void (*kernel)(CUtensorMap, double*, Params);
};
template <class K>
Variant make_variant(const char* n) {
  return {n, K::TY, K::KCH, K::SMEM, heat3d_fused<K>};
}
// LF_HEAT3D_VARIANT=<index> overrides the default for tuning runs
const Variant& variant() {
  static const Variant table[] = {
      make_variant<Cfg<2, 6, 32>>("rpw2_s6_k32"), make_variant<Cfg<2, 8, 32>>("rpw2_s8_k32"),
      make_variant<Cfg<2, 6, 64>>("rpw2_s6_k64"), make_variant<Cfg<2, 6, 16>>("rpw2_s6_k16"),
      make_variant<Cfg<4, 5, 32>>("rpw4_s5_k32"), make_variant<Cfg<4, 6, 64>>("rpw4_s6_k64"),
      make_variant<Cfg<4, 4, 32>>("rpw4_s4_k32"), make_variant<Cfg<2, 6, 8>>("rpw2_s6_k8"),
      make_variant<Cfg<2, 5, 16>>("rpw2_s5_k16"), make_variant<Cfg<2, 7, 16>>("rpw2_s7_k16"),
      make_variant<Cfg<2, 4, 16>>("rpw2_s4_k16"), make_variant<Cfg<2, 6, 12>>("rpw2_s6_k12"),
  };
  static int idx = [] {
    const char* e = lfx::option("LF_HEAT3D_VARIANT");
    // default rpw2_s6_k16: best of the measured sweep (profiles/r01_heat3d_variants.txt)
    int i = e ? std::atoi(e) : 3;
    return (i >= 0 && i < (int)(sizeof table / sizeof table[0])) ? i : 3;
  }();
  return table[idx];
}

bool supports(const lf::Plan& plan, std::string& why) {
  const auto& r = plan.rs.ranges;
  long nk = r[0].trips(), nj = r[1].trips(), ni = r[2].trips();
  for (const auto& rg : r)
    if (rg.stride != 1 || rg.lo != 0) {
      why = "heat3d executor needs unit strides and ranges starting at 0";
      return false;
    }
  const int TY = variant().ty;
  if (ni % TX || nj % TY || nk < 1) {
    why = "heat3d executor needs N_i % 64 == 0 and N_j % " + std::to_string(TY) + " == 0 (got " +
          std::to_string(ni) + "x" + std::to_string(nj) + ")";
    return false;
  }
  if ((ni + 2) * 8 % 16) {
    why = "row pitch must be a multiple of 16 bytes";
    return false;
  }
  return true;
}

int launch_step(const double* in, double* out, int ni, int nj, int nk, int k_lo, int k_hi, bool wrap_k,
                cudaStream_t st, std::string& err) {
  const Variant& v = variant();
  static LaunchCache cache;  // the variant is fixed per process (LF_HEAT3D_VARIANT)
  int slots = 0;
  if (int s = resident_slots(cache, reinterpret_cast<const void*>(v.kernel), THREADS, v.smem, 0,
                             "cudaFuncSetAttribute(heat3d)", &slots, err))
    return s;
  CUtensorMap map;
  uint64_t dims[3] = {(uint64_t)ni + 2, (uint64_t)nj + 2, (uint64_t)nk + 2};
  uint32_t box[3] = {LD, (uint32_t)(v.ty + 2), 1};
  if (!make_tensor_map(&map, in, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 3, dims, box, err)) return LF_ERR_CUDA;
  Params p;
  p.ni = ni;
  p.nj = nj;
  p.nk = nk;
  p.pj = ni + 2;
  p.pk = (long long)(ni + 2) * (nj + 2);
  p.tiles_x = ni / TX;
  p.tiles = (ni / TX) * (nj / v.ty);
  p.k_lo = k_lo;
  p.k_hi = k_hi;
  p.kchunks = std::max(1, (k_hi - k_lo + v.kch - 1) / v.kch);
  p.units = p.tiles * p.kchunks;
  // evict_normal: same-box A/B 348.5 -> 351.2 G against evict_first; evict_last
  // (the 1 GB output cannot stay in L2) 343 G (LF_HEAT3D_STORE_POLICY)
  const int store_policy = [] {
    const char* e = lfx::option("LF_HEAT3D_STORE_POLICY");
    return e ? std::atoi(e) : 1;
  }();
  p.store_policy = store_policy;
  p.wrap_i = 1;
  p.wrap_j = 1;
  p.wrap_k = wrap_k ? 1 : 0;
  // persistent grid: every resident CTA slot on the chip, never more than units
  const int ctas = std::min(p.units, slots);
  // plain stream-ordered launch: measured A/B, programmatic dependent launch
  // costs heat3d ~8% (its one-wave 380-us kernels have no launch gap to hide)
  v.kernel<<<ctas, THREADS, v.smem, st>>>(map, out, p);
  return cuda_status(cudaGetLastError(), "heat3d_fused launch", err);
}

// two steps per pass (whole periodic domain only: a slab's k ghosts come from
// the caller's one-plane halo exchange)

// opt-in (LF_HEAT3D_TB=1): 382 vs 367 G cell-updates/s for the single-step
// kernel at 512^3 -- within a few percent, because the pass is bound by
// shared-memory traffic and latency rather than by the HBM bytes it saves
//
bool tb_enabled(int ni, int nj, int nk) {
  const char* e = lfx::option("LF_HEAT3D_TB");
  const bool on = e && std::atoi(e) != 0;
  return on && ni % TX == 0 && nj % tb::TY == 0 && nk >= 2 && ni >= TX && nj >= tb::TY;
}

template <class K>
int launch_pair_k(const double* in, double* out, int ni, int nj, int nk, cudaStream_t st, std::string& err) {
  static LaunchCache cache;
  int slots = 0;
  if (int s = resident_slots(cache, reinterpret_cast<const void*>(tb::heat3d_fused2<K>), tb::THREADS2, K::SMEM, 0,
                             "cudaFuncSetAttribute(heat3d pair)", &slots, err))
    return s;
  CUtensorMap map;
  uint64_t dims[3] = {(uint64_t)ni + 2, (uint64_t)nj + 2, (uint64_t)nk + 2};
  uint32_t box[3] = {tb::LDI, tb::RI, 1};
  if (!make_tensor_map(&map, in, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 3, dims, box, err)) return LF_ERR_CUDA;
  Params p;
  p.ni = ni;
  p.nj = nj;
  p.nk = nk;
  p.pj = ni + 2;
  p.pk = (long long)(ni + 2) * (nj + 2);
  p.tiles_x = ni / TX;
  p.tiles = (ni / TX) * (nj / tb::TY);
  p.k_lo = 0;
  p.k_hi = nk;
  p.kchunks = std::max(1, (nk + K::KCH - 1) / K::KCH);
  p.units = p.tiles * p.kchunks;
  p.store_policy = 0;
  p.wrap_i = p.wrap_j = p.wrap_k = 1;
  p.patch = lfx::option("LF_HEAT3D_NOPATCH") ? 0 : 1;  // timing experiments only (wrong at the faces)
  const int ctas = std::min(p.units, slots);
  tb::heat3d_fused2<K><<<ctas, tb::THREADS2, K::SMEM, st>>>(map, in, out, p);
  return cuda_status(cudaGetLastError(), "heat3d_fused2 launch", err);
}

// LF_HEAT3D_TBK: planes per work unit of the two-step pass (32 / 64 / 128; 64 measured best)
int launch_pair(const double* in, double* out, int ni, int nj, int nk, cudaStream_t st, std::string& err) {
  const int kch = [] {
    const char* e = lfx::option("LF_HEAT3D_TBK");
    return e ? std::atoi(e) : 64;
  }();
  if (kch >= 128) return launch_pair_k<tb::Cfg<6, 128>>(in, out, ni, nj, nk, st, err);
  if (kch >= 64) return launch_pair_k<tb::Cfg<6, 64>>(in, out, ni, nj, nk, st, err);
  return launch_pair_k<tb::Cfg<6, 32>>(in, out, ni, nj, nk, st, err);
}

int run(const ExecArgs& a, std::string& err) {
  const auto& r = a.plan->rs.ranges;
  const int nj = (int)r[1].trips(), ni = (int)r[2].trips();
  const RowPart rp = row_part(a, (int)r[0].trips());
  const int nk = rp.rows;
  // k ghosts of a slab come from the caller's halo exchange; the row parts of
  // a pipelined host run cover the whole domain and wrap themselves
  const bool wrap_k = a.slab == nullptr || a.whole_domain_parts;
  const double* src = static_cast<const double*>(a.terms[0]);
  double* goal = static_cast<double*>(a.terms[1]);
  double* scratch = a.steps > 1 ? static_cast<double*>(a.scratch[0]) : nullptr;
  // passes of one or two steps; they alternate goal/scratch so that the last
  // one lands in the goal and the axiom buffer is never written
  const bool pairs = a.slab == nullptr && a.steps >= 2 && tb_enabled(ni, nj, nk);
  const int passes = pairs ? (a.steps + 1) / 2 : a.steps;
  for (int s = 0; s < passes; ++s) {
    const bool to_goal = ((passes - 1 - s) % 2) == 0;
    double* dst = to_goal ? goal : scratch;
    // an odd step count runs its first step alone
    const bool two = pairs && !(s == 0 && a.steps % 2 == 1);
    int st = two ? launch_pair(src, dst, ni, nj, nk, a.stream, err)
                 : launch_step(src, dst, ni, nj, nk, rp.lo, rp.hi, wrap_k, a.stream, err);
    if (st != LF_OK) return st;
    src = dst;
  }
  return LF_OK;
}

}  // namespace

int heat3d_passes(const lf::Plan& plan, int steps, bool slab);
int heat3d_passes(const lf::Plan& plan, int steps, bool slab) {
  const auto& r = plan.rs.ranges;
  const bool pairs = !slab && steps >= 2 && tb_enabled((int)r[2].trips(), (int)r[1].trips(), (int)r[0].trips());
  return pairs ? (steps + 1) / 2 : steps;
}

namespace {

}  // namespace

extern const Executor heat3d_executor = {"heat3d_fused_tma", "heat3d.lf", 1, 16.0, supports, run, heat3d_passes};

}  // namespace lfx
