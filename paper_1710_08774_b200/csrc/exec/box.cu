// Fused sm_100a executor for the separable 3x3 box filter applied twice
// (BASELINE.json configs[3]; specs/box2x.lf): row1 -> col1 -> row2 -> col2,
// fp32, clamp-to-edge expressed as the caller's replicate padding of g_img.
//
// The three intermediates never leave the SM: one warp marches a 128-column
// strip down the image (rowstream.cuh), lane l owning columns 4l..4l+3.
// row passes read their i +- 1 neighbours from the adjacent lanes by shuffle
// (lanes 0/31 also carry the strip's halo column), column passes use 3-row
// register windows that rotate by renaming (rows unrolled by 3).  Image rows
// arrive by TMA into an 8-slot ring; each output row leaves as one 16-B store
// per lane.  Compulsory traffic: 4 B read + 4 B written per cell.
#include <algorithm>

#include "../../userkernels/stencil_kernels.h"
#include "common.cuh"
#include "exec.hpp"
#include "rowstream.cuh"

namespace lfx {
namespace {

constexpr int CPL = 4;                 // columns per lane
constexpr int SW = 32 * CPL;           // strip width: 128 columns
constexpr int H = 2;                   // chain radius
constexpr int LPAD = H;                // staged left pad (the box starts at the terminal's first column)
constexpr int BOXW = SW + 2 * LPAD;    // staged row: 132 floats = 528 B
constexpr int R = 3;                   // rows per stage (= register-window period)
constexpr int S = 8;                   // ring slots
constexpr int STAGE_TX = BOXW * R * 4;
constexpr int STAGE_BYTES = (STAGE_TX + 127) / 128 * 128;
constexpr int SMEM = S * STAGE_BYTES + S * 8 + 64;
constexpr int OCC = 16;

struct Params {
  int ni, nj;
  int row_lo, row_hi;   // rows this launch computes
  long long out_pitch;  // ni
  int strips;
};

struct Win {
  float r1[3][CPL];  // row pass 1, rows by index % 3
  float r1h[3];      // ... at the strip's halo column
  float r2[3][CPL];  // row pass 2
};

template <int P>
__device__ __forceinline__ void box_row(Win& w, const float* row, int t, int lane, int ex_col, float* orow,
                                        uint64_t pol) {
  constexpr int C = P, M1 = (P + 2) % 3, M2 = (P + 1) % 3;  // rows r, r-1, r-2
  // 8-B aligned halves: the staged row starts at logical i0-2
  const float2 v01 = *reinterpret_cast<const float2*>(row + LPAD + CPL * lane);
  const float2 v23 = *reinterpret_cast<const float2*>(row + LPAD + CPL * lane + 2);
  const float4 v = make_float4(v01.x, v01.y, v23.x, v23.y);
  const float2 ex = *reinterpret_cast<const float2*>(row + ex_col);
  // ---- row1 at row r
  {
    const float left = __shfl_up_sync(0xffffffffu, v.w, 1);
    const float right = __shfl_down_sync(0xffffffffu, v.x, 1);
    const float a = lane == 0 ? ex.y : left;       // logical -1 for lane 0
    const float b = lane == 31 ? ex.x : right;     // logical SW for lane 31
    box3(a, v.x, v.y, &w.r1[C][0]);
    box3(v.x, v.y, v.z, &w.r1[C][1]);
    box3(v.y, v.z, v.w, &w.r1[C][2]);
    box3(v.z, v.w, b, &w.r1[C][3]);
    // halo column: lane 0 -> logical -1 = box3(img[-2], img[-1], img[0]);
    //              lane 31 -> logical SW = box3(img[SW-1], img[SW], img[SW+1])
    const bool lo = lane == 0;
    box3(lo ? ex.x : v.w, lo ? ex.y : ex.x, lo ? v.x : ex.y, &w.r1h[C]);
  }
  if (t < 2) return;
  // ---- col1 at row r-1 (own columns and the halo column), then row2 at row r-1
  float c1[CPL], c1h;
#pragma unroll
  for (int c = 0; c < CPL; ++c) box3(w.r1[M2][c], w.r1[M1][c], w.r1[C][c], &c1[c]);
  box3(w.r1h[M2], w.r1h[M1], w.r1h[C], &c1h);
  {
    const float left = __shfl_up_sync(0xffffffffu, c1[CPL - 1], 1);
    const float right = __shfl_down_sync(0xffffffffu, c1[0], 1);
    const float a = lane == 0 ? c1h : left;
    const float b = lane == 31 ? c1h : right;
    box3(a, c1[0], c1[1], &w.r2[M1][0]);
    box3(c1[0], c1[1], c1[2], &w.r2[M1][1]);
    box3(c1[1], c1[2], c1[3], &w.r2[M1][2]);
    box3(c1[2], c1[3], b, &w.r2[M1][3]);
  }
  if (t < 4) return;
  // ---- col2 at row r-2: r2 rows r-3 (slot C), r-2 (M2), r-1 (M1)
  float o[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) box3(w.r2[C][c], w.r2[M2][c], w.r2[M1][c], &o[c]);
  st_hint4(orow + CPL * lane, o[0], o[1], o[2], o[3], pol);
}

__global__ void __launch_bounds__(32, OCC)
    box_fused(const __grid_constant__ CUtensorMap tin, float* __restrict__ out, const Params p) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE_BYTES);
  const int lane = threadIdx.x;

  RowSeg seg[3];
  const int nseg = cta_segments(blockIdx.x, gridDim.x, p.strips, p.row_lo, p.row_hi, seg);
  RowRing<R, S> rr;
  // staged column 0 = logical i0 - 2 = storage i0; storage row = logical + 2
  rr.init(seg, nseg, H, smem, full, STAGE_BYTES, STAGE_TX, 0, H, SW);
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    tma_prefetch_desc(&tin);
    for (int g = 0; g < S; ++g) rr.issue(g, &tin);
  }
  __syncwarp();

  const uint64_t pol = l2_evict_first_policy();
  // extra columns: lane 0 -> logical -2,-1 (staged 0,1); lane 31 -> SW, SW+1 (staged SW+2, SW+3)
  const int ex_col = lane == 0 ? LPAD - 2 : (lane == 31 ? LPAD + SW : LPAD + CPL * lane);
  int g = 0;
  Win w;
  for (int k = 0; k < nseg; ++k) {
    const RowSeg sg = seg[k];
    const int T = sg.je - sg.jb + 2 * H;
    float* orow = out + (long long)(sg.jb - 4) * p.out_pitch + sg.strip * SW;  // output row of t = 0
    for (int t0 = 0; t0 < T; t0 += R, ++g) {
      rr.wait(g);
      const float* st = reinterpret_cast<const float*>(rr.stage(g));
      box_row<0>(w, st, t0, lane, ex_col, orow, pol);
      orow += p.out_pitch;
      if (t0 + 1 < T) box_row<1>(w, st + BOXW, t0 + 1, lane, ex_col, orow, pol);
      orow += p.out_pitch;
      if (t0 + 2 < T) box_row<2>(w, st + 2 * BOXW, t0 + 2, lane, ex_col, orow, pol);
      orow += p.out_pitch;
      __syncwarp();
      if (lane == 0) rr.issue(g + S, &tin);
    }
  }
}

bool supports(const lf::Plan& plan, std::string& why) {
  const auto& r = plan.rs.ranges;
  for (const auto& rg : r)
    if (rg.stride != 1) {
      why = "box executor needs unit strides";
      return false;
    }
  long ni = r[1].trips();
  if (ni % SW) {
    why = "box executor needs N_i % 128 == 0 (got " + std::to_string(ni) + ")";
    return false;
  }
  return true;
}

int run(const ExecArgs& a, std::string& err) {
  static int slots = 0;
  if (!slots) {
    cudaError_t e = cudaFuncSetAttribute(box_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(box)", err);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, box_fused, 32, SMEM);
    slots = sms * std::max(1, std::min(per_sm, OCC));
  }
  const auto& r = a.plan->rs.ranges;
  const int ni = (int)r[1].trips();
  const RowPart rp = row_part(a, (int)r[0].trips());  // slab rows: halo rows supplied by the caller
  const int nj = rp.rows;
  CUtensorMap map;
  uint64_t dims[2] = {(uint64_t)ni + 4, (uint64_t)nj + 4};
  uint32_t box[2] = {BOXW, R};
  if (!make_tensor_map(&map, a.terms[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 2, dims, box, err))
    return LF_ERR_CUDA;
  Params p;
  p.ni = ni;
  p.nj = nj;
  p.row_lo = rp.lo;
  p.row_hi = rp.hi;
  p.out_pitch = ni;
  p.strips = ni / SW;
  const long long work = (long long)p.strips * (rp.hi - rp.lo);
  // each CTA must get at most 3 row segments (rowstream.cuh): at least
  // ceil(strips/2) CTAs when the row range is short
  const long long want = std::max<long long>(work / 16, (p.strips + 1) / 2);
  const int ctas = static_cast<int>(std::max<long long>(1, std::min<long long>(slots, want)));
  if ((long long)ctas * 2 < p.strips) {
    err = "row range too short for the resident grid";
    return LF_ERR_UNSUPPORTED;
  }
  // a single pass; `steps` re-applies the same pass (no iterate pairs)
  for (int s = 0; s < a.steps; ++s) {
    box_fused<<<ctas, 32, SMEM, a.stream>>>(map, static_cast<float*>(a.terms[1]), p);
    int st = cuda_status(cudaGetLastError(), "box_fused launch", err);
    if (st != LF_OK) return st;
  }
  return LF_OK;
}

}  // namespace

extern const Executor box_executor = {"box2x_fused_tma", "box2x.lf", 1, 8.0, supports, run};

}  // namespace lfx
