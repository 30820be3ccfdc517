// Row streaming for 2D chains marched along their outer loop dimension j
// (loop order (j, i)).  One warp per CTA owns a strip of columns and walks a
// contiguous run of rows, so every intermediate lives in per-lane register
// windows along j (HFAV's outer_rotate rows, storage.cpp:369-378) and moves
// between lanes with warp shuffles along i -- only terminals touch HBM.
//
// Work split: the strip-major linear row index L = strip * NJ + j is cut into
// one contiguous range per CTA (persistent grid, one resident wave), giving
// each CTA one or two segments (strip, [jb, je)).  Neighbouring strips are
// walked by CTAs that start at the same row at the same time, so the halo
// columns a CTA stages were staged moments earlier by its neighbour and hit
// in L2.
//
// Staging: lane 0 of the warp is also the TMA producer.  Rows [jb-H, je+H)
// of a segment are cut into stages of R rows, streamed by 2D TMA boxes into
// an S-slot shared-memory ring; a slot is refilled as soon as the marcher has
// consumed (and used) the last row of its stage.
#pragma once

#include <algorithm>

#include "common.cuh"

namespace lfx {

struct RowSeg {
  int strip, jb, je;  // output rows [jb, je) of column strip `strip`
};

// Segments of CTA `cta` of `ctas` over `strips` strips of rows [r0, r1).
__device__ __forceinline__ int cta_segments(int cta, int ctas, int strips, int r0, int r1, RowSeg* seg) {
  const int nj = r1 - r0;
  const long long total = (long long)strips * nj;
  long long a = total * cta / ctas, b = total * (cta + 1) / ctas;
  int n = 0;
  while (a < b && n < 3) {
    const int s = static_cast<int>(a / nj);
    const long long end = std::min<long long>(b, (long long)(s + 1) * nj);
    seg[n].strip = s;
    seg[n].jb = r0 + static_cast<int>(a - (long long)s * nj);
    seg[n].je = r0 + static_cast<int>(end - (long long)s * nj);
    ++n;
    a = end;
  }
  return n;
}

// Persistent grid for `strips` strips of `rows` rows on `slots` resident CTAs.
// A whole multiple of `strips` CTAs makes CTA c + ctas/strips start strip s+1
// at exactly the row where CTA c starts strip s, so the halo columns two
// neighbours share are fetched within moments of each other (one DRAM read,
// one L2 hit).  At least ceil(strips/2) CTAs: a CTA takes at most 3 segments.
inline int rowstream_ctas(long long slots, int strips, long long rows) {
  const long long work = (long long)strips * rows;
  long long ctas = std::max<long long>(1, std::min<long long>(slots, std::max<long long>(work / 16, (strips + 1) / 2)));
  if (ctas >= strips) ctas = ctas / strips * strips;
  return static_cast<int>(ctas);
}

// One-warp TMA row ring.  Stage g covers rows [jb-H + gg*R, +R) of its
// segment (gg = stage index within the segment).
template <int R, int S>
struct RowRing {
  const RowSeg* seg;
  int nseg, H, total;
  int nst[3];
  unsigned char* ring;
  uint64_t* full;
  int stage_bytes;
  uint32_t tx_bytes;
  int col0;       // storage column of strip 0's first staged column
  int row0;       // storage row of logical row 0 (= -terminal base along j)
  int strip_w;    // columns per strip

  __device__ void init(const RowSeg* s, int n, int halo, unsigned char* r, uint64_t* f, int sb, uint32_t tx,
                       int c0, int r0, int sw) {
    seg = s;
    nseg = n;
    H = halo;
    ring = r;
    full = f;
    stage_bytes = sb;
    tx_bytes = tx;
    col0 = c0;
    row0 = r0;
    strip_w = sw;
    total = 0;
    for (int k = 0; k < n; ++k) {
      nst[k] = (s[k].je - s[k].jb + 2 * H + R - 1) / R;
      total += nst[k];
    }
  }
  // lane 0 only: TMA for global stage g into slot g % S
  bool load_hint = false;  // fetch with an L2 cache policy (load_pol)
  uint64_t load_pol = 0;
  __device__ void issue(int g, const CUtensorMap* map) const {
    if (g >= total) return;
    int k = 0, gg = g;
    while (gg >= nst[k]) gg -= nst[k++];
    const int slot = g % S;
    fence_proxy_async();
    mbar_arrive_expect_tx(&full[slot], tx_bytes);
    if (load_hint)
      tma_load_2d_hint(ring + slot * stage_bytes, map, &full[slot], col0 + seg[k].strip * strip_w,
                       row0 + seg[k].jb - H + gg * R, load_pol);
    else
      tma_load_2d(ring + slot * stage_bytes, map, &full[slot], col0 + seg[k].strip * strip_w,
                  row0 + seg[k].jb - H + gg * R);
  }
  __device__ void wait(int g) const { mbar_wait(&full[g % S], (g / S) & 1); }
  __device__ const unsigned char* stage(int g) const { return ring + (g % S) * stage_bytes; }
};

}  // namespace lfx
