// Diffusion sub-step, activation detector, probe recording and layout
// kernels. Compiled with --fmad=false: every product and sum rounds exactly
// like the reference's x86-64 build, so diffusion is bit-identical to
// diffusion_substep (fem.cpp:194-207) and the detector to
// ActivationDetector::observe (postprocess.cpp:18-66).
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "launch.h"

namespace cwg {

static inline int blocks_for(long long n, int t, int cap);

// ---------------------------------------------------------------------------
// Stencil-2D: a regular sheet's 9-point rows with per-node coefficients taken
// verbatim from the CSR (absent boundary entries stored as 0 and skipped
// without reading V, so 0*Inf never appears). Row sums run in ascending
// column order starting from 0.0 like fem.cpp:202-205.
//   coef[c*cpitch + i], c = 0..8 for offsets {-w-1,-w,-w+1,-1,0,1,w-1,w,w+1}
//   cm[i] = dt_sub / m_i (the reference's own division)
// Local layout per rank: one halo row (w nodes) below and above the owned
// rows; the owned row r (0-based) starts at (r+1)*w.
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(256) diffuse_stencil2d(DiffArgs a, Stencil2D s) {
  const long long nown = s.rows * s.w;
  const long long seq = cur_seq(a.clock, a.step_off, a.evs, a.ev);
  // an earlier event failed: leave V where it stopped (host: restore_failed_state); a peer-linked rank still
  // takes part in the launch pacing so its neighbours do not wait for it
  const bool skip = earlier_failure(a.err, seq);
  peer_wait(a.pl);
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < nown && !skip;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = o + s.hrows_v * s.w;  // local V index
    const long long oc = o + s.hrows_c * s.w;  // local coefficient index
    const double vi = a.vin[i];
    const long long r = o / s.w, x = o - r * s.w;
    const long long gy = s.row_begin + r;
    const bool has_s = gy > 0, has_n = gy + 1 < s.ny1, has_w = x > 0, has_e = x + 1 < s.w;
    const double* c = s.coef + oc;
    const long long P = s.cpitch;
    double acc = 0.0;
    if (has_s) {
      if (has_w) acc += c[0 * P] * a.vin[i - s.w - 1];
      acc += c[1 * P] * a.vin[i - s.w];
      if (has_e) acc += c[2 * P] * a.vin[i - s.w + 1];
    }
    if (has_w) acc += c[3 * P] * a.vin[i - 1];
    acc += c[4 * P] * vi;
    if (has_e) acc += c[5 * P] * a.vin[i + 1];
    if (has_n) {
      if (has_w) acc += c[6 * P] * a.vin[i + s.w - 1];
      acc += c[7 * P] * a.vin[i + s.w];
      if (has_e) acc += c[8 * P] * a.vin[i + s.w + 1];
    }
    const double out = vi - s.cm[oc] * acc;
    a.vout[i] = out;
    peer_store(a, r, x, out);
    if (!isfinite(out))
      record_failure(a.err, static_cast<unsigned long long>(o + s.row_begin * s.w) << 22, seq, 2, 1, a.vin, a.vout);
  }
  peer_post(a.pl);
}

// ---------------------------------------------------------------------------
// Temporal blocking: T consecutive sub-steps in one kernel. A block owns a
// TBX x TBY output tile. Sub-step q (0-based) is computed on the tile plus a
// (T-1-q)-node halo, so the block needs V on the tile + T halo (shared memory,
// double-buffered) and the 9+1 coefficients of the tile + (T-1) halo: each
// thread owns up to R of those points for all T sub-steps and keeps their
// coefficients in registers (loaded once, all loads independent). Every
// node's arithmetic is exactly that of diffuse_stencil2d, so the result is
// bit-identical to T separate sub-steps. A non-finite value in sub-step q of
// the tile is keyed (q << 58) | (node << 22): atomicMin yields the earliest
// sub-step, then the lowest node (the order of separate launches).
// ---------------------------------------------------------------------------
// EDGE = false: the block's computed region plus one node lies inside the
// sheet and the rank's rows, so every point has all 8 neighbours (the CSR row
// is the full 9-point stencil) and no presence flags or selects are needed.
template <int T, int TBX, int TBY, int NT, bool EDGE>
__device__ __forceinline__ void tb_body(const DiffArgs& a, const Stencil2D& s, double (*Vs)[(TBY + 2 * T) * (TBX + 2 * T)],
                                        long long gx0, long long ly0, long long seq) {
  constexpr int VX = TBX + 2 * T;
  constexpr int CX = TBX + 2 * (T - 1), CY = TBY + 2 * (T - 1);  // computed region (sub-step 0)
  constexpr int R = (CX * CY + NT - 1) / NT;                     // points per thread
  const long long rows = s.rows, w = s.w;
  // Slots in ring order: the TBX x TBY tile first, then halo ring 1, 2, ...
  // so that the points active in sub-step q are a prefix of the slots and
  // whole warps skip the rest (warp-uniform branch). Per slot: coefficients,
  // V index, flags (bit0 own, 1 s, 2 n, 3 w, 4 e).
  double cf[R][10];
  int vi[R];
  unsigned fl[R];
  int px[R], py[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int p = threadIdx.x + r * NT;
    int rx = 0, ry = 0;
    const bool valid = p < CX * CY;
    if (p < TBX * TBY) {
      rx = p % TBX;
      ry = p / TBX;
    } else if (valid) {
      int e = p - TBX * TBY, k = 1;
      while (e >= 2 * (TBX + 2 * k) + 2 * (TBY + 2 * k - 2)) {
        e -= 2 * (TBX + 2 * k) + 2 * (TBY + 2 * k - 2);
        ++k;
      }
      const int wr = TBX + 2 * k, hr = TBY + 2 * k - 2;  // ring row length, column length (corners excluded)
      if (e < wr) {
        rx = e - k, ry = -k;
      } else if (e < 2 * wr) {
        rx = e - wr - k, ry = TBY - 1 + k;
      } else if (e < 2 * wr + hr) {
        rx = -k, ry = e - 2 * wr - k + 1;
      } else {
        rx = TBX - 1 + k, ry = e - 2 * wr - hr - k + 1;
      }
    }
    px[r] = rx;
    py[r] = ry;
    const long long x = gx0 + rx, yl = ly0 + ry, gy = s.row_begin + yl;
    // computed: inside the sheet and within the local coefficient rows (with
    // hrows_c > 0, halo points of a neighbouring rank are advanced too);
    // owned: written back and failure-checked
    const bool own = valid && (!EDGE || (x >= 0 && x < w && gy >= 0 && gy < s.ny1 && yl >= -s.hrows_c &&
                                         yl < rows + s.hrows_c));
    const bool mine = yl >= 0 && yl < rows;
    fl[r] = own ? (1u | (gy > 0 ? 2u : 0u) | (gy + 1 < s.ny1 ? 4u : 0u) | (x > 0 ? 8u : 0u) | (x + 1 < w ? 16u : 0u) |
                   (mine ? 32u : 0u))
                : 0u;
    vi[r] = own ? (ry + T) * VX + (rx + T) : VX + 1;  // inactive slots read a safe in-range cell
    const long long o = own ? (yl + s.hrows_c) * w + x : 0;
    const double* cp = s.coef + o;
#pragma unroll
    for (int c = 0; c < 9; ++c) cf[r][c] = own ? __ldg(cp + c * s.cpitch) : 0.0;
    cf[r][9] = own ? __ldg(s.cm + o) : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < T; ++q) {
    const double* src = Vs[q & 1];
    double* dst = Vs[(q + 1) & 1];
    const int hx = T - 1 - q;
    const int n_act = (TBX + 2 * hx) * (TBY + 2 * hx);  // active slots: a prefix
    double out[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      out[r] = 0.0;
      if (r * NT + (threadIdx.x & ~31) >= n_act) continue;  // warp-uniform
      const unsigned f = fl[r];
      const bool act = (f & 1u) && threadIdx.x + r * NT < n_act;
      const double* sp = src + vi[r];
      const double v0 = sp[0];
      double o;
      if (!EDGE) {
        // interior: the full 9-point row, same additions in the same order
        double acc = 0.0 + cf[r][0] * sp[-VX - 1];
        acc += cf[r][1] * sp[-VX];
        acc += cf[r][2] * sp[-VX + 1];
        acc += cf[r][3] * sp[-1];
        acc += cf[r][4] * v0;
        acc += cf[r][5] * sp[1];
        acc += cf[r][6] * sp[VX - 1];
        acc += cf[r][7] * sp[VX];
        acc += cf[r][8] * sp[VX + 1];
        o = v0 - cf[r][9] * acc;
      } else {
        const double vsw = sp[-VX - 1], vs = sp[-VX], vse = sp[-VX + 1], vw = sp[-1], ve = sp[1];
        const double vnw = sp[VX - 1], vn = sp[VX], vne = sp[VX + 1];
        const bool hs = f & 2u, hn = f & 4u, hw = f & 8u, he = f & 16u;
        // same additions, same order as diffuse_stencil2d; absent terms leave acc untouched
        double acc = 0.0, tmp;
        tmp = acc + cf[r][0] * vsw; acc = (hs && hw) ? tmp : acc;
        tmp = acc + cf[r][1] * vs;  acc = hs ? tmp : acc;
        tmp = acc + cf[r][2] * vse; acc = (hs && he) ? tmp : acc;
        tmp = acc + cf[r][3] * vw;  acc = hw ? tmp : acc;
        acc = acc + cf[r][4] * v0;
        tmp = acc + cf[r][5] * ve;  acc = he ? tmp : acc;
        tmp = acc + cf[r][6] * vnw; acc = (hn && hw) ? tmp : acc;
        tmp = acc + cf[r][7] * vn;  acc = hn ? tmp : acc;
        tmp = acc + cf[r][8] * vne; acc = (hn && he) ? tmp : acc;
        o = v0 - cf[r][9] * acc;
      }
      out[r] = o;
      if (q + 1 < T && act) dst[vi[r]] = o;
      if (act && (f & 32u) && threadIdx.x + r * NT < TBX * TBY && !isfinite(o)) {
        const long long x = gx0 + px[r], yl = ly0 + py[r];
        record_failure(a.err, (static_cast<unsigned long long>(q) << 58) |
                                  (static_cast<unsigned long long>(yl * w + x + s.row_begin * w) << 22), seq, 2, T,
                       a.vin, a.vout);
      }
    }
    if (q + 1 < T) {
      __syncthreads();
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r * NT >= TBX * TBY) break;
        if (fl[r] & 32u) {
          a.vout[(ly0 + py[r] + s.hrows_v) * w + gx0 + px[r]] = out[r];
          peer_store(a, ly0 + py[r], gx0 + px[r], out[r]);
        }
      }
    }
  }
}

template <int T, int TBX, int TBY, int NT>
__global__ void __launch_bounds__(NT) diffuse_stencil2d_tb(DiffArgs a, Stencil2D s) {
  constexpr int VX = TBX + 2 * T, VY = TBY + 2 * T;  // V region
  __shared__ double Vs[2][VY * VX];
  const long long seq = cur_seq(a.clock, a.step_off, a.evs, a.ev);
  const bool skip = earlier_failure(a.err, seq);
  peer_wait(a.pl);
  if (skip) {  // block-uniform: an earlier event failed, V stays where it stopped
    peer_post(a.pl);
    return;
  }
  const long long gx0 = static_cast<long long>(blockIdx.x) * TBX, ly0 = static_cast<long long>(blockIdx.y) * TBY;
  const long long rows = s.rows, w = s.w;
  {
    // V on the tile + T halo; rows outside the sheet are never read (presence flags)
    const double* vsrc = a.vin + (ly0 - T + s.hrows_v) * w + gx0 - T;
    for (int t = threadIdx.x; t < VX * VY; t += NT) {
      const int cx = t % VX, cy = t / VX;
      const long long x = gx0 - T + cx, gy = s.row_begin + ly0 - T + cy, yl = ly0 - T + cy;
      const bool in = x >= 0 && x < w && gy >= 0 && gy < s.ny1 && yl >= -s.hrows_v && yl < rows + s.hrows_v;
      Vs[0][t] = in ? vsrc[static_cast<long long>(cy) * w + cx] : 0.0;
    }
  }
  const bool interior = gx0 >= T && gx0 + TBX + T <= w && ly0 >= T && ly0 + TBY + T <= rows;
  if (interior)
    tb_body<T, TBX, TBY, NT, false>(a, s, Vs, gx0, ly0, seq);
  else
    tb_body<T, TBX, TBY, NT, true>(a, s, Vs, gx0, ly0, seq);
  peer_post(a.pl);
}

// ---------------------------------------------------------------------------
// Persistent temporal blocking with TMA: one CTA per SM walks the tiles. The
// coefficients live in a padded copy [10][rows][w_pad] (planes 0..8 = the 9
// stencil coefficients, 9 = dt/m; even row pitch so every global stride is a
// multiple of 16 bytes) described by a 3D tensor map; one thread issues ONE
// cp.async.bulk.tensor per tile for the whole (CX x CY x 10) box -- TMA
// zero-fills outside the sheet -- completing on an mbarrier while the CTA
// computes the previous tile. V regions (odd row pitch) come in by per-thread
// cp.async into a third buffer. Arithmetic, slot order and failure keys are
// those of diffuse_stencil2d_tb.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}

// TMA geometry. The padded tensor stores node (x, y) at column x + kTmaMargin
// (a zeroed left margin), and a box must start at a 16-byte aligned,
// non-negative inner coordinate: boxes start SX = 2*ceil((T-1)/2) columns
// left of the tile (even), BXW columns wide (even, covers the CX needed).
constexpr int kTmaMargin = 6;  // >= SX for T <= 6
template <int T, int TBX, int TBY, int NT>
struct TbmGeom {
  static constexpr int VX = TBX + 2 * T, VY = TBY + 2 * T, VXY = VX * VY;
  static constexpr int CX = TBX + 2 * (T - 1), CY = TBY + 2 * (T - 1);
  static constexpr int SX = 2 * ((T - 1 + 1) / 2);
  static constexpr int BXW = ((SX + TBX + (T - 1)) + 1) / 2 * 2;
  static constexpr int R = (CX * CY + NT - 1) / NT;
  static constexpr int BOX = 10 * BXW * CY;  // doubles per TMA box
  static_assert(SX <= kTmaMargin && (BXW * 8) % 16 == 0, "TMA box alignment");
  static constexpr size_t smem = (static_cast<size_t>(BOX) + 3ull * VXY) * sizeof(double) + 16;
};

template <int T, int TBX, int TBY, int NT>
__global__ void __launch_bounds__(NT, 1)
    diffuse_stencil2d_tbm(DiffArgs a, Stencil2D s, const __grid_constant__ CUtensorMap tmap, int tiles_x, int n_tiles) {
  using G = TbmGeom<T, TBX, TBY, NT>;
  constexpr int VX = G::VX, VXY = G::VXY, CX = G::CX, CY = G::CY, R = G::R, BOX = G::BOX, BXW = G::BXW, SX = G::SX;
  extern __shared__ __align__(128) double tbm_smem[];
  double* cfs = tbm_smem;  // [10][CY][BXW]: the TMA box
  double* vb0 = cfs + BOX;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(vb0 + 3 * VXY);
  const unsigned bar_a = smem_u32(bar);
  const long long seq = cur_seq(a.clock, a.step_off, a.evs, a.ev);
  const bool skip = earlier_failure(a.err, seq);
  if (skip) return;  // block-uniform: an earlier event failed, V stays where it stopped
  const long long rows = s.rows, w = s.w;
  int px[R], py[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int p = threadIdx.x + r * NT;
    int rx = 0, ry = 0;
    if (p < TBX * TBY) {
      rx = p % TBX;
      ry = p / TBX;
    } else if (p < CX * CY) {
      int e = p - TBX * TBY, k = 1;
      while (e >= 2 * (TBX + 2 * k) + 2 * (TBY + 2 * k - 2)) {
        e -= 2 * (TBX + 2 * k) + 2 * (TBY + 2 * k - 2);
        ++k;
      }
      const int wr = TBX + 2 * k, hr = TBY + 2 * k - 2;
      if (e < wr) {
        rx = e - k, ry = -k;
      } else if (e < 2 * wr) {
        rx = e - wr - k, ry = TBY - 1 + k;
      } else if (e < 2 * wr + hr) {
        rx = -k, ry = e - 2 * wr - k + 1;
      } else {
        rx = TBX - 1 + k, ry = e - 2 * wr - hr - k + 1;
      }
    }
    px[r] = rx;
    py[r] = ry;
  }
  auto issue_box = [&](int tile) {  // thread 0 only
    const int gx0 = (tile % tiles_x) * TBX, ly0 = (tile / tiles_x) * TBY;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of cfs before the async write
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a), "r"(BOX * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_u32(cfs)),
        "l"(&tmap), "r"(gx0 - SX + kTmaMargin), "r"(static_cast<int>(ly0 + s.hrows_c) - (T - 1)), "r"(0), "r"(bar_a)
        : "memory");
  };
  auto fetch_v = [&](int tile, double* vdst) {
    const long long gx0 = static_cast<long long>(tile % tiles_x) * TBX, ly0 = static_cast<long long>(tile / tiles_x) * TBY;
    const double* vsrc = a.vin + (ly0 - T + s.hrows_v) * w + gx0 - T;
    for (int t = threadIdx.x; t < VXY; t += NT) {
      const int cx = t % VX, cy = t / VX;
      const long long x = gx0 - T + cx, gy = s.row_begin + ly0 - T + cy, yl = ly0 - T + cy;
      if (x >= 0 && x < w && gy >= 0 && gy < s.ny1 && yl >= -s.hrows_v && yl < rows + s.hrows_v)
        cp_async8(vdst + t, vsrc + static_cast<long long>(cy) * w + cx);
      else
        vdst[t] = 0.0;  // outside the sheet: never read (presence flags)
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int tile = blockIdx.x;
  if (tile < n_tiles) {
    if (threadIdx.x == 0) issue_box(tile);
    fetch_v(tile, vb0);
  }
  int cur = 0;
  unsigned parity = 0;
  for (; tile < n_tiles; tile += gridDim.x) {
    const long long gx0 = static_cast<long long>(tile % tiles_x) * TBX, ly0 = static_cast<long long>(tile / tiles_x) * TBY;
    mbar_wait(bar_a, parity);
    parity ^= 1u;
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const bool interior = gx0 >= T && gx0 + TBX + T <= w && ly0 >= T && ly0 + TBY + T <= rows;
    double cf[R][10];
    int vi[R];
    unsigned fl[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long long x = gx0 + px[r], yl = ly0 + py[r], gy = s.row_begin + yl;
      const bool own = threadIdx.x + r * NT < CX * CY && x >= 0 && x < w && yl >= 0 && yl < rows;
      fl[r] = own ? (1u | (gy > 0 ? 2u : 0u) | (gy + 1 < s.ny1 ? 4u : 0u) | (x > 0 ? 8u : 0u) | (x + 1 < w ? 16u : 0u))
                  : 0u;
      vi[r] = own ? (py[r] + T) * VX + (px[r] + T) : VX + 1;
      const int bi = (py[r] + T - 1) * BXW + (px[r] + SX);
#pragma unroll
      for (int c = 0; c < 10; ++c) cf[r][c] = own ? cfs[c * BXW * CY + bi] : 0.0;
    }
    __syncthreads();  // cfs and the spare V buffer are free: start the next tile's copies
    const int nxt = tile + static_cast<int>(gridDim.x);
    double* vnext = vb0 + ((cur + 2) % 3) * VXY;
    if (nxt < n_tiles) {
      if (threadIdx.x == 0) issue_box(nxt);
      fetch_v(nxt, vnext);
    }
    double* va = vb0 + cur * VXY;
    double* vs = vb0 + ((cur + 1) % 3) * VXY;
#pragma unroll
    for (int q = 0; q < T; ++q) {
      const double* src = (q & 1) ? vs : va;
      double* dst = (q & 1) ? va : vs;
      const int hx = T - 1 - q;
      const int n_act = (TBX + 2 * hx) * (TBY + 2 * hx);
      double out[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        out[r] = 0.0;
        if (r * NT + (threadIdx.x & ~31) >= n_act) continue;  // warp-uniform
        const unsigned f = fl[r];
        const bool act = (f & 1u) && threadIdx.x + r * NT < n_act;
        const double* sp = src + vi[r];
        const double v0 = sp[0];
        double o;
        if (interior) {
          double acc = 0.0 + cf[r][0] * sp[-VX - 1];
          acc += cf[r][1] * sp[-VX];
          acc += cf[r][2] * sp[-VX + 1];
          acc += cf[r][3] * sp[-1];
          acc += cf[r][4] * v0;
          acc += cf[r][5] * sp[1];
          acc += cf[r][6] * sp[VX - 1];
          acc += cf[r][7] * sp[VX];
          acc += cf[r][8] * sp[VX + 1];
          o = v0 - cf[r][9] * acc;
        } else {
          const double vsw = sp[-VX - 1], vss = sp[-VX], vse = sp[-VX + 1], vw = sp[-1], ve = sp[1];
          const double vnw = sp[VX - 1], vn = sp[VX], vne = sp[VX + 1];
          const bool hs = f & 2u, hn = f & 4u, hw = f & 8u, he = f & 16u;
          double acc = 0.0, tmp;
          tmp = acc + cf[r][0] * vsw; acc = (hs && hw) ? tmp : acc;
          tmp = acc + cf[r][1] * vss; acc = hs ? tmp : acc;
          tmp = acc + cf[r][2] * vse; acc = (hs && he) ? tmp : acc;
          tmp = acc + cf[r][3] * vw;  acc = hw ? tmp : acc;
          acc = acc + cf[r][4] * v0;
          tmp = acc + cf[r][5] * ve;  acc = he ? tmp : acc;
          tmp = acc + cf[r][6] * vnw; acc = (hn && hw) ? tmp : acc;
          tmp = acc + cf[r][7] * vn;  acc = hn ? tmp : acc;
          tmp = acc + cf[r][8] * vne; acc = (hn && he) ? tmp : acc;
          o = v0 - cf[r][9] * acc;
        }
        out[r] = o;
        if (q + 1 < T && act) dst[vi[r]] = o;
        if (act && threadIdx.x + r * NT < TBX * TBY && !isfinite(o)) {
          const long long x = gx0 + px[r], yl = ly0 + py[r];
          record_failure(a.err, (static_cast<unsigned long long>(q) << 58) |
                                    (static_cast<unsigned long long>(yl * w + x + s.row_begin * w) << 22), seq, 2,
                         T, a.vin, a.vout);
        }
      }
      if (q + 1 < T) {
        __syncthreads();
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (r * NT >= TBX * TBY) break;
          if (fl[r] & 1u) a.vout[(ly0 + py[r] + s.hrows_v) * w + gx0 + px[r]] = out[r];
        }
      }
    }
    cur = (cur + 2) % 3;
  }
}

// ---------------------------------------------------------------------------
// TMA-fed fused diffusion, register quads (default for large one-GPU sheets).
// Same tiles, coefficient boxes (the tbm tensor maps), V prefetch and fused
// depth as diffuse_stencil2d_tbm, but each thread owns a 2 x 2 quad of points
// for all T sub-steps: its 40 coefficients live in registers (20 16-byte
// shared loads per tile: quads start at even x, so a quad row's two points
// are one aligned pair in every coefficient plane) and each sub-step streams
// the quad's 4 x 4 V neighbourhood row by row with two 16-byte shared loads
// per row -- 2 loads per point-sub-step instead of 9, and four independent
// accumulation chains per thread. Each point's 9 terms are added in ascending
// column order (row by row), exactly as diffuse_stencil2d. Absent neighbours
// meet a zero coefficient (stored 0, or TMA's zero fill) and a zero or finite
// V: 0 * v adds a signed zero, which never changes the sum (it starts at +0
// and so is never -0) -- the bits of skipping the term, with no presence
// tests. A quad computes while it touches the shrinking region; its points
// beyond the region hold finite values no counting point reads. Non-finite
// results of owned points set bits of a per-thread mask, resolved once per
// tile into the same failure keys the per-sub-step check would record (the
// minimum key is each point's first failing sub-step).
// ---------------------------------------------------------------------------
template <int T, int TBX, int TBY, int NT>
struct TbqGeom {
  using B = TbmGeom<T, TBX, TBY, NT>;                  // the coefficient box of the tbm tensor maps
  static constexpr int PX0 = -(T - 1) - ((T - 1) & 1);  // first quad column: even, <= -(T-1)
  static constexpr int QX = (TBX + T - PX0) / 2;        // quad columns covering PX0 .. TBX+T-2 (rounded up)
  static constexpr int QY = (TBY + 2 * (T - 1)) / 2;    // quad rows covering -(T-1) .. TBY+T-2
  static constexpr int VOFF = 1 - PX0;                  // V smem column of x: x + VOFF (x - 1 lands on an even column)
  static constexpr int VX = (PX0 + 2 * QX + VOFF + 2) / 2 * 2;  // even pitch: 16-byte aligned rows
  static constexpr int VY = TBY + 2 * T + 2;            // V smem row of y: y + T + 1
  static constexpr int VXY = VX * VY;
  static_assert(QX * QY <= NT && (TBY % 2) == 0 && VOFF % 2 == 1 && PX0 + 2 * QX - 1 >= TBX + T - 2, "quad geometry");
  static_assert(PX0 >= -B::SX && PX0 + 2 * QX <= B::BXW - B::SX, "quads inside the coefficient box");
  static constexpr size_t smem = (static_cast<size_t>(B::BOX) + 3ull * VXY) * sizeof(double) + 16;
};

template <int T, int TBX, int TBY, int NT>
__global__ void __launch_bounds__(NT, 1)
    diffuse_stencil2d_tbq(DiffArgs a, Stencil2D s, const __grid_constant__ CUtensorMap tmap, int tiles_x, int n_tiles) {
  using G = TbqGeom<T, TBX, TBY, NT>;
  using B = typename G::B;
  constexpr int VX = G::VX, VY = G::VY, VXY = G::VXY, QX = G::QX, QY = G::QY, VOFF = G::VOFF;
  constexpr int BOX = B::BOX, BXW = B::BXW, SX = B::SX, CY = B::CY;
  extern __shared__ __align__(128) double tbq_smem[];
  double* cfs = tbq_smem;  // [10][CY][BXW]: the TMA box
  double* vb0 = cfs + BOX;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(vb0 + 3 * VXY);
  const unsigned bar_a = smem_u32(bar);
  const long long seq = cur_seq(a.clock, a.step_off, a.evs, a.ev);
  if (earlier_failure(a.err, seq)) return;  // block-uniform: an earlier event failed, V stays where it stopped
  const long long rows = s.rows, w = s.w;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool has_quad = t < QX * QY;
  const int qx = G::PX0 + 2 * (t % QX), qy = 2 * (t / QX) - (T - 1);  // quad origin relative to the tile
  // the quad takes part in sub-steps q <= qlast: it touches region(q) = the tile grown by T-1-q
  const int dx = qx + 1 < 0 ? -(qx + 1) : (qx >= TBX ? qx - TBX + 1 : 0);
  const int dy = qy + 1 < 0 ? -(qy + 1) : (qy >= TBY ? qy - TBY + 1 : 0);
  const int qlast = has_quad ? T - 1 - (dx > dy ? dx : dy) : -1;
  const int cfo = (qy + T - 1) * BXW + qx + SX;     // box offset of the quad's (x, y) point: even
  const int wo = (qy - 1 + T + 1) * VX + qx - 1 + VOFF;  // V offset of the window's (x-1, y-1): even
  auto issue_box = [&](int tile) {  // thread 0 only
    const int gx0 = (tile % tiles_x) * TBX, ly0 = (tile / tiles_x) * TBY;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a), "r"(BOX * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_u32(cfs)),
        "l"(&tmap), "r"(gx0 - SX + kTmaMargin), "r"(static_cast<int>(ly0 + s.hrows_c) - (T - 1)), "r"(0), "r"(bar_a)
        : "memory");
  };
  // V rows ly0-T-1 .. ly0+TBY+T, columns gx0-VOFF .. gx0-VOFF+VX-1 (zero outside the sheet / local rows);
  // one warp per row, lanes along it
  auto fetch_v = [&](int tile, double* vdst) {
    const long long gx0 = static_cast<long long>(tile % tiles_x) * TBX, ly0 = static_cast<long long>(tile / tiles_x) * TBY;
    for (int cy = warp; cy < VY; cy += NT / 32) {
      const long long yl = ly0 - T - 1 + cy, gy = s.row_begin + yl;
      const bool row_in = gy >= 0 && gy < s.ny1 && yl >= -s.hrows_v && yl < rows + s.hrows_v;
      const double* vrow = a.vin + (yl + s.hrows_v) * w + gx0 - VOFF;
      double* drow = vdst + cy * VX;
      for (int cx = lane; cx < VX; cx += 32) {
        const long long x = gx0 - VOFF + cx;
        if (row_in && x >= 0 && x < w)
          cp_async8(drow + cx, vrow + cx);
        else
          drow[cx] = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // the second and third V frames start finite (quads read one point beyond the region they computed)
  for (int e = t; e < 2 * VXY; e += NT) vb0[VXY + e] = 0.0;
  __syncthreads();
  int tile = blockIdx.x;
  if (tile < n_tiles) {
    if (t == 0) issue_box(tile);
    fetch_v(tile, vb0);
  }
  int cur = 0;
  unsigned parity = 0;
  for (; tile < n_tiles; tile += gridDim.x) {
    const long long gx0 = static_cast<long long>(tile % tiles_x) * TBX, ly0 = static_cast<long long>(tile / tiles_x) * TBY;
    mbar_wait(bar_a, parity);
    parity ^= 1u;
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    // the quad's 4 x 10 coefficients (zero outside the local rows: those points never count)
    double cf[4][10];
    unsigned own = 0;  // bit k: point k lies in this tile and the sheet
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const long long yl = ly0 + qy + j;
      const bool in = has_quad && yl >= -s.hrows_c && yl < rows + s.hrows_c;
#pragma unroll
      for (int c = 0; c < 10; ++c) {
        double2 p = make_double2(0.0, 0.0);
        if (in) p = *reinterpret_cast<const double2*>(cfs + c * BXW * CY + cfo + j * BXW);
        cf[2 * j][c] = p.x;
        cf[2 * j + 1][c] = p.y;
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int px = qx + i, py = qy + j;
        if (has_quad && px >= 0 && px < TBX && py >= 0 && py < TBY && gx0 + px < w && yl < rows) own |= 1u << (2 * j + i);
      }
    }
    __syncthreads();  // cfs and the spare V frame are free: start the next tile's copies
    const int nxt = tile + static_cast<int>(gridDim.x);
    double* vnext = vb0 + ((cur + 2) % 3) * VXY;
    if (nxt < n_tiles) {
      if (t == 0) issue_box(nxt);
      fetch_v(nxt, vnext);
    }
    double* va = vb0 + cur * VXY;
    double* vs = vb0 + ((cur + 1) % 3) * VXY;
    double out[4] = {0.0, 0.0, 0.0, 0.0};
    unsigned bad = 0;  // bit 4q + k: point k non-finite after sub-step q
#pragma unroll
    for (int q = 0; q < T; ++q) {
      const double* src = (q & 1) ? vs : va;
      double* dst = (q & 1) ? va : vs;
      if (q <= qlast) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        double v0[4];
        // window rows y-1 .. y+2; quad row j (points k = 2j, 2j+1) takes rows y+j-1 .. y+j+1 in order
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const double* rp = src + wo + r * VX;
          const double2 p0 = *reinterpret_cast<const double2*>(rp);
          const double2 p1 = *reinterpret_cast<const double2*>(rp + 2);
          const double wv[4] = {p0.x, p0.y, p1.x, p1.y};  // x-1, x, x+1, x+2
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int ry = r - j;  // this window row is quad row j's row ry-1 (ry = 0, 1, 2)
            if (ry < 0 || ry > 2) continue;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int k = 2 * j + i;
              acc[k] += cf[k][ry * 3 + 0] * wv[i];
              acc[k] += cf[k][ry * 3 + 1] * wv[i + 1];
              acc[k] += cf[k][ry * 3 + 2] * wv[i + 2];
              if (ry == 1) v0[k] = wv[i + 1];
            }
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          out[k] = v0[k] - cf[k][9] * acc[k];
          bad |= (isfinite(out[k]) ? 0u : 1u) << (4 * q + k);
        }
        if (q + 1 < T) {
          double* dp = dst + wo + VX + 1;  // (x, y)
          dp[0] = out[0];
          dp[1] = out[1];
          dp[VX] = out[2];
          dp[VX + 1] = out[3];
        }
      }
      if (q + 1 < T) __syncthreads();
    }
    bad &= own * 0x11111111u;  // owned points only (own <= 0xF: the nibble replicated per sub-step)
    if (bad) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const unsigned m = (bad >> k) & 0x11111111u;
        if (!m) continue;
        const unsigned q = static_cast<unsigned>(__ffs(static_cast<int>(m)) - 1) / 4;
        const long long x = gx0 + qx + (k & 1), yl = ly0 + qy + (k >> 1);
        record_failure(a.err, (static_cast<unsigned long long>(q) << 58) |
                                  (static_cast<unsigned long long>(yl * w + x + s.row_begin * w) << 22), seq, 2, T,
                       a.vin, a.vout);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (own >> k & 1u) a.vout[(ly0 + qy + (k >> 1) + s.hrows_v) * w + gx0 + qx + (k & 1)] = out[k];
    cur = (cur + 2) % 3;
  }
}

template <int T>
static cudaError_t launch_tbq_t(const DiffArgs& a, const Stencil2D& s, const CUtensorMap& tm, int num_sms,
                                cudaStream_t st) {
  using G = TbqGeom<T, 64, 16, 512>;
  static std::atomic<uint64_t> attr_done{0};
  const cudaError_t e = ensure_dyn_smem(diffuse_stencil2d_tbq<T, 64, 16, 512>, static_cast<int>(G::smem), attr_done);
  if (e != cudaSuccess) return e;
  const int tiles_x = static_cast<int>((s.w + 63) / 64);
  const int n_tiles = tiles_x * static_cast<int>((s.rows + 15) / 16);
  diffuse_stencil2d_tbq<T, 64, 16, 512><<<std::min(num_sms, n_tiles), 512, G::smem, st>>>(a, s, tm, tiles_x, n_tiles);
  return cudaGetLastError();
}

template <int T>
static cudaError_t launch_tbm_t(const DiffArgs& a, const Stencil2D& s, const CUtensorMap& tm, int num_sms,
                                cudaStream_t st) {
  using G = TbmGeom<T, 64, 16, 512>;
  static std::atomic<uint64_t> attr_done{0};
  const cudaError_t e = ensure_dyn_smem(diffuse_stencil2d_tbm<T, 64, 16, 512>, static_cast<int>(G::smem), attr_done);
  if (e != cudaSuccess) return e;
  const int tiles_x = static_cast<int>((s.w + 63) / 64);
  const int n_tiles = tiles_x * static_cast<int>((s.rows + 15) / 16);
  diffuse_stencil2d_tbm<T, 64, 16, 512><<<std::min(num_sms, n_tiles), 512, G::smem, st>>>(a, s, tm, tiles_x, n_tiles);
  return cudaGetLastError();
}

// TMA box of the padded coefficient tensor for T fused sub-steps (64 x 16 tiles)
void tbm_box(int T, unsigned* cx, unsigned* cy, int* margin) {
  *margin = kTmaMargin;
  switch (T) {
    case 2: *cx = TbmGeom<2, 64, 16, 512>::BXW, *cy = TbmGeom<2, 64, 16, 512>::CY; break;
    case 3: *cx = TbmGeom<3, 64, 16, 512>::BXW, *cy = TbmGeom<3, 64, 16, 512>::CY; break;
    case 4: *cx = TbmGeom<4, 64, 16, 512>::BXW, *cy = TbmGeom<4, 64, 16, 512>::CY; break;
    case 5: *cx = TbmGeom<5, 64, 16, 512>::BXW, *cy = TbmGeom<5, 64, 16, 512>::CY; break;
    default: *cx = TbmGeom<6, 64, 16, 512>::BXW, *cy = TbmGeom<6, 64, 16, 512>::CY; break;
  }
}

cudaError_t launch_diffuse_stencil2d_tbm(int T, const DiffArgs& a, const Stencil2D& s, const CUtensorMap& tm,
                                         int num_sms, cudaStream_t st) {
  // register-quad kernel by default; CWG_TBQ=0: the slot kernel (A/B, one GPU only: it does not advance
  // a slab's halo rows)
  const char* e = getenv("CWG_TBQ");
  if (!(e && e[0] == '0') || s.hrows_c > 0) {
    switch (T) {
      case 2: return launch_tbq_t<2>(a, s, tm, num_sms, st);
      case 3: return launch_tbq_t<3>(a, s, tm, num_sms, st);
      case 4: return launch_tbq_t<4>(a, s, tm, num_sms, st);
      case 5: return launch_tbq_t<5>(a, s, tm, num_sms, st);
      case 6: return launch_tbq_t<6>(a, s, tm, num_sms, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (T) {
    case 2: return launch_tbm_t<2>(a, s, tm, num_sms, st);
    case 3: return launch_tbm_t<3>(a, s, tm, num_sms, st);
    case 4: return launch_tbm_t<4>(a, s, tm, num_sms, st);
    case 5: return launch_tbm_t<5>(a, s, tm, num_sms, st);
    case 6: return launch_tbm_t<6>(a, s, tm, num_sms, st);
    default: return cudaErrorInvalidValue;
  }
}

// dst[(c*rows + y)*w_pad + margin + x] = src[c*src_pitch + y*w + x] (padded coefficient planes)
__global__ void pad_planes(const double* src, long long src_pitch, int n_planes, long long w, long long rows,
                           double* dst, long long w_pad, int dst_plane0) {
  const long long n = w * rows;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < n * n_planes;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long c = o / n, r = o - c * n, y = r / w, x = r - y * w;
    dst[((c + dst_plane0) * rows + y) * w_pad + kTmaMargin + x] = src[c * src_pitch + r];
  }
}

cudaError_t launch_pad_planes(const double* src, long long src_pitch, int n_planes, long long w, long long rows,
                              double* dst, long long w_pad, int dst_plane0, cudaStream_t st) {
  pad_planes<<<blocks_for(w * rows * n_planes, 256, 148 * 32), 256, 0, st>>>(src, src_pitch, n_planes, w, rows, dst,
                                                                            w_pad, dst_plane0);
  return cudaGetLastError();
}

template <int T, int TBX, int TBY, int NT>
static cudaError_t launch_tb(const DiffArgs& a, const Stencil2D& s, cudaStream_t st) {
  const dim3 grid(static_cast<unsigned>((s.w + TBX - 1) / TBX), static_cast<unsigned>((s.rows + TBY - 1) / TBY));
  diffuse_stencil2d_tb<T, TBX, TBY, NT><<<grid, NT, 0, st>>>(a, s);
  return cudaGetLastError();
}

// T fused sub-steps (2..4): 64x16 tiles unless that leaves fewer than 2 blocks per SM
cudaError_t launch_diffuse_stencil2d_tb(int T, const DiffArgs& a, const Stencil2D& s, int num_sms, cudaStream_t st) {
  const long long big = ((s.w + 63) / 64) * ((s.rows + 15) / 16);
  const bool large = big >= 2ll * num_sms;
  switch (T) {
    case 2: return large ? launch_tb<2, 64, 16, 512>(a, s, st) : launch_tb<2, 32, 8, 256>(a, s, st);
    case 3: return large ? launch_tb<3, 64, 16, 512>(a, s, st) : launch_tb<3, 32, 8, 256>(a, s, st);
    case 4: return large ? launch_tb<4, 64, 16, 512>(a, s, st) : launch_tb<4, 32, 8, 256>(a, s, st);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------------------
// Structured 3D slab (EXTENSION): 27-point rows whose coefficients depend only
// on the node class (x face, y face, z layer); ascending-column order is
// (dy, dz, dx) lexicographic for the y-outer numbering. 16 B of node traffic
// per sub-step (V in/out) plus cached neighbour reads; bit-identical to the
// oracle's CSR assembly of the same operator.
// ---------------------------------------------------------------------------
// 2.5D blocking: a block owns a TX x TZ tile of the (x, z) plane and marches
// over a chunk of y-planes, keeping planes y-1, y, y+1 (tile + 1-node halo) in
// a shared-memory ring, so each V value is fetched from global memory ~1.3x
// per sub-step instead of up to 27x. No 64-bit division: (x, z, y) come from
// the launch geometry.
constexpr int S3_TX = 32, S3_TZ = 8;

__global__ void __launch_bounds__(S3_TX * S3_TZ, 6) diffuse_struct3d(DiffArgs a, Struct3D s) {
  constexpr int NT = S3_TX * S3_TZ;
  constexpr int PX = S3_TX + 2, PZ = S3_TZ + 2, PL = PX * PZ;
  constexpr int PR = (PL + NT - 1) / NT;  // plane values per thread
  __shared__ double ring[4][PL];
  const long long seq = cur_seq(a.clock, a.step_off, a.evs, a.ev);
  const bool skip = earlier_failure(a.err, seq);
  peer_wait(a.pl);
  if (skip) {  // block-uniform: an earlier event failed, V stays where it stopped
    peer_post(a.pl);
    return;
  }
  const int tx = threadIdx.x % S3_TX, tz = threadIdx.x / S3_TX;
  const int x0 = blockIdx.x * S3_TX, z0 = blockIdx.y * S3_TZ;
  const int ix = x0 + tx, iz = z0 + tz;
  const int nx1 = static_cast<int>(s.nx1), nz1 = static_cast<int>(s.nz1);
  const int nx = nx1 - 1, nz = nz1 - 1;
  const long long yb = static_cast<long long>(blockIdx.z) * s.ychunk;
  const long long ye = yb + s.ychunk < s.planes ? yb + s.ychunk : s.planes;
  const bool inside = ix < nx1 && iz < nz1;
  // this thread's share of a (tile + halo) plane: offsets within the plane, or -1
  int off[PR];
#pragma unroll
  for (int r = 0; r < PR; ++r) {
    const int t = threadIdx.x + r * NT;
    const int lx = x0 - 1 + t % PX, lz = z0 - 1 + t / PX;
    off[r] = (t < PL && lx >= 0 && lx < nx1 && lz >= 0 && lz < nz1) ? lz * nx1 + lx : -1;
  }
  // planes yl = -1 .. planes are valid memory (halo planes); beyond: zeros
  auto fetch = [&](long long yl, double (&reg)[PR]) {
    const double* src = a.vin + (yl + 1) * s.plane;
#pragma unroll
    for (int r = 0; r < PR; ++r) reg[r] = (off[r] >= 0 && yl <= s.planes) ? src[off[r]] : 0.0;
  };
  auto put = [&](const double (&reg)[PR], double* dst) {
#pragma unroll
    for (int r = 0; r < PR; ++r)
      if (threadIdx.x + r * NT < PL) dst[threadIdx.x + r * NT] = reg[r];
  };
  const int bx = ix == 0 ? 0 : (ix == nx ? 2 : 1);
  // Interior in x and z: all 27 neighbours exist on every y-interior plane;
  // the row's class (by = 1, bx, iz) is fixed for the whole march. Its
  // coefficients are read through the read-only cache: a warp spans one z
  // layer, so every load is a warp-uniform broadcast (registers would cut the
  // occupancy this latency-bound loop needs).
  const bool xz_interior = inside && bx == 1 && iz > 0 && iz < nz;
  const double* cfi = s.coef + ((3 + bx) * static_cast<long long>(nz1) + iz) * 27;
  const double* cmp = s.cm + (3 + bx) * static_cast<long long>(nz1) + iz;
  // 4-slot ring: planes y-1, y, y+1 are read while y+2 (prefetched into
  // registers one trip earlier) is written -- one barrier per plane, and the
  // global loads of a plane overlap the previous plane's arithmetic.
  double* pm = ring[0];  // y - 1
  double* p0 = ring[1];  // y
  double* pp = ring[2];  // y + 1
  double* pw = ring[3];  // y + 2 (being written)
  double reg[PR];
  fetch(yb - 1, reg);
  put(reg, pm);
  fetch(yb, reg);
  put(reg, p0);
  fetch(yb + 1, reg);
  put(reg, pp);
  fetch(yb + 2, reg);
  __syncthreads();
  const int c0 = (tz + 1) * PX + (tx + 1);
  for (long long yl = yb; yl < ye; ++yl) {
    if (inside) {
      const long long i = (yl + 1) * s.plane + static_cast<long long>(iz) * nx1 + ix;
      const double vi = p0[c0];
      const long long gy = s.row_begin + yl;
      const int by = gy == 0 ? 0 : (gy == s.ny1 - 1 ? 2 : 1);
      {
        double out;
        const double* pl[3] = {pm, p0, pp};
        if (xz_interior && by == 1) {
          // the full 27-point row in ascending column order (dy, dz, dx)
          double acc = 0.0;
#pragma unroll
          for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
              for (int dx = -1; dx <= 1; ++dx)
                acc += __ldg(cfi + dy * 9 + (dz + 1) * 3 + (dx + 1)) * pl[dy][c0 + dz * PX + dx];
          out = vi - __ldg(cmp) * acc;
        } else {
          const long long cls = (by * 3 + bx) * static_cast<long long>(nz1) + iz;
          const double* cf = s.coef + cls * 27;
          double acc = 0.0;
#pragma unroll
          for (int dy = -1; dy <= 1; ++dy) {
            if ((dy < 0 && by == 0) || (dy > 0 && by == 2)) continue;
#pragma unroll
            for (int dz = -1; dz <= 1; ++dz) {
              if ((dz < 0 && iz == 0) || (dz > 0 && iz == nz)) continue;
#pragma unroll
              for (int dx = -1; dx <= 1; ++dx) {
                if ((dx < 0 && bx == 0) || (dx > 0 && bx == 2)) continue;
                const int q = (dy + 1) * 9 + (dz + 1) * 3 + (dx + 1);
                acc += __ldg(cf + q) * pl[dy + 1][c0 + dz * PX + dx];
              }
            }
          }
          out = vi - __ldg(s.cm + cls) * acc;
        }
        a.vout[i] = out;
        peer_store(a, yl, static_cast<long long>(iz) * nx1 + ix, out);
        if (!isfinite(out))
          record_failure(a.err, static_cast<unsigned long long>(i - s.plane + s.row_begin * s.plane) << 22, seq, 2, 1,
                         a.vin, a.vout);
      }
    }
    if (yl + 1 < ye) {
      put(reg, pw);        // plane yl + 2
      fetch(yl + 3, reg);  // in flight during the next trip
    }
    __syncthreads();
    double* t = pm;
    pm = p0;
    p0 = pp;
    pp = pw;
    pw = t;
  }
  peer_post(a.pl);
}

// ---------------------------------------------------------------------------
// Structured 3D slab, register-blocked (default). The row sum is 27 DMUL +
// 27 DADD in a fixed order (bit-exactness: no FMA, no reassociation), so at
// 16 B of V traffic per node-substep the kernel is FP64-pipe bound unless the
// V values it multiplies are already in registers and the instructions that
// are not FP64 are few per node:
//   * a thread owns four x-adjacent nodes (x .. x+3) of one z row and marches
//     over y. All four have the same node class (x-interior, by, iz): the
//     warp-uniform 27 coefficients + dt/m of its row are read from shared
//     memory as broadcasts, each feeding four DMULs, and the four
//     accumulation chains (8-cycle DADD latency, measured) interleave;
//   * the 3 x 3 x 6 window of V (planes y-1, y, y+1; rows z-1..z+1; columns
//     x-1..x+4) lives in registers; a plane step brings in the 18 values of
//     plane y+1 with 3-4 shared-memory loads per row (~2.5 per node);
//   * plane rows arrive in shared memory by 1D bulk copies (cp.async.bulk,
//     the TMA engine: one instruction per 130-node row), NS - 2 planes ahead
//     of use, through a full/empty mbarrier ring -- no block-wide barrier: a
//     warp waits only for the rows it reads and the slot it refills. V rows
//     are not 16-byte aligned (odd nx+1), so each copy starts at the aligned
//     node at or below x0 - 1 and moves 132 nodes; the row's shift (0/1) is
//     the parity of its first index, and the window read picks its pattern;
//   * absent neighbours (z faces, y faces) meet a zero coefficient and a
//     zero V (rows outside the slab in z are zeroed once; the halo planes
//     beyond the global y faces are zero-initialised memory nothing writes):
//     0 * 0 adds +0, which leaves the sum (never -0: it starts at +0)
//     unchanged -- the same bits as skipping the term like fem.cpp;
//   * the two x faces (x = 0, x = nx; other classes) are rows of their own:
//     extra blocks of the same grid compute them one thread per node with
//     the generic class lookup.
// Warp w of a block owns row z0 + w; lane l owns x = xb + 4l .. xb + 4l + 3.
// ---------------------------------------------------------------------------
constexpr int S3R_NS = 6;      // plane stages in the ring (lead NS - 2 planes)
constexpr int S3R_TX = 128;    // nodes per tile row (32 lanes x 4)
constexpr int S3R_COPY = 132;  // nodes per row copy (1056 B, a multiple of 16): x0 - 1 - sh .. x0 + 130 - sh
constexpr int S3R_RS = 136;    // doubles per staged row

template <int W>
struct S3R {
  static constexpr int NT = 32 * W;
  static constexpr int ROWS = W + 2;
  static constexpr int STAGE = ROWS * S3R_RS;  // doubles per plane stage
  static constexpr int CF = 3 * W * 28;        // coefficient tables: [by][w][27 + dt/m]
  static constexpr size_t smem = (static_cast<size_t>(S3R_NS) * STAGE + CF) * sizeof(double) + 2 * S3R_NS * 8;
};

// Generic row (any class, presence tests): the x-face nodes and tiny slabs.
__device__ __forceinline__ void s3_generic_node(const DiffArgs& a, const Struct3D& s, int ix, int iz, long long yl,
                                                long long seq) {
  const int nx1 = static_cast<int>(s.nx1), nz1 = static_cast<int>(s.nz1);
  const int nx = nx1 - 1, nz = nz1 - 1;
  const long long gy = s.row_begin + yl;
  const int bx = ix == 0 ? 0 : (ix == nx ? 2 : 1);
  const int by = gy == 0 ? 0 : (gy == s.ny1 - 1 ? 2 : 1);
  const long long cls = (by * 3 + bx) * static_cast<long long>(nz1) + iz;
  const double* cf = s.coef + cls * 27;
  const long long i = (yl + 1) * s.plane + static_cast<long long>(iz) * nx1 + ix;
  double acc = 0.0;
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy) {
    if ((dy < 0 && by == 0) || (dy > 0 && by == 2)) continue;
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz) {
      if ((dz < 0 && iz == 0) || (dz > 0 && iz == nz)) continue;
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        if ((dx < 0 && bx == 0) || (dx > 0 && bx == 2)) continue;
        acc += __ldg(cf + (dy + 1) * 9 + (dz + 1) * 3 + (dx + 1)) * a.vin[i + dy * s.plane + dz * nx1 + dx];
      }
    }
  }
  const double out = a.vin[i] - __ldg(s.cm + cls) * acc;
  a.vout[i] = out;
  peer_store(a, yl, static_cast<long long>(iz) * nx1 + ix, out);
  if (!isfinite(out))
    record_failure(a.err, static_cast<unsigned long long>(i - s.plane + s.row_begin * s.plane) << 22, seq, 2, 1,
                   a.vin, a.vout);
}

// One plane step of a thread's four nodes: window planes (m, o, p) = (y-1, y,
// y+1), each [3 rows z-1..z+1][6 cols x-1..x+4]; cf = the row's 27
// coefficients and dt/m in shared memory (warp-uniform broadcasts).
__device__ __forceinline__ void s3r_quad(const double (&m)[18], const double (&o)[18], const double (&p)[18],
                                         const double* cf, double (&out)[4]) {
  const double* pl[3] = {m, o, p};
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int dy = 0; dy < 3; ++dy)
#pragma unroll
    for (int dz = 0; dz < 3; ++dz)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const double c = cf[dy * 9 + dz * 3 + dx];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] += c * pl[dy][dz * 6 + dx + j];
      }
  const double cm = cf[27];
#pragma unroll
  for (int j = 0; j < 4; ++j) out[j] = o[6 + 1 + j] - cm * acc[j];
}

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

template <int W>
__device__ __forceinline__ void struct3d_rb_body(const DiffArgs& a, const Struct3D& s, int tiles_x, int tiles_z,
                                                 int n_items, int ychunk, long long n_edge, long long seq);

template <int W>
__global__ void __launch_bounds__(32 * W, 2)
    diffuse_struct3d_rb(DiffArgs a, Struct3D s, int tiles_x, int tiles_z, int n_items, int ychunk,
                        long long n_edge) {
  const long long seq = cur_seq(a.clock, a.step_off, a.evs, a.ev);
  peer_wait(a.pl);
  // block-uniform: after an earlier failed event V stays where it stopped
  if (!earlier_failure(a.err, seq)) struct3d_rb_body<W>(a, s, tiles_x, tiles_z, n_items, ychunk, n_edge, seq);
  peer_post(a.pl);
}

template <int W>
__device__ __forceinline__ void struct3d_rb_body(const DiffArgs& a, const Struct3D& s, int tiles_x, int tiles_z,
                                                 int n_items, int ychunk, long long n_edge, long long seq) {
  using G = S3R<W>;
  extern __shared__ __align__(128) double s3r_smem[];
  const int nx1 = static_cast<int>(s.nx1), nz1 = static_cast<int>(s.nz1);
  const int nx = nx1 - 1;
  if (static_cast<int>(blockIdx.x) >= n_items) {
    // x-face rows (x = 0 and x = nx), one thread per node
    const long long per = static_cast<long long>(nz1) * s.planes;
    for (long long e = (blockIdx.x - n_items) * static_cast<long long>(G::NT) + threadIdx.x; e < n_edge;
         e += static_cast<long long>(gridDim.x - n_items) * G::NT) {
      const int side = static_cast<int>(e / per);
      const long long r = e - side * per;
      const long long yl = r / nz1;
      const int iz = static_cast<int>(r - yl * nz1);
      s3_generic_node(a, s, side == 0 ? 0 : nx, iz, yl, seq);
    }
    return;
  }
  const int item = blockIdx.x;
  const int tile = item % (tiles_x * tiles_z), ych = item / (tiles_x * tiles_z);
  const int xb = 1 + (tile % tiles_x) * S3R_TX;  // first node of the tile (x-interior rows start at x = 1)
  const int z0 = (tile / tiles_x) * W;
  const int planes = static_cast<int>(s.planes);
  const int yb = ych * ychunk;
  const int ye = yb + ychunk < planes ? yb + ychunk : planes;
  if (ye <= yb) return;  // an empty trailing chunk (block-uniform)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int x0 = xb + 4 * lane, z = z0 + w;
  const int zc = z < nz1 ? z : nz1 - 1;  // clamped row for the coefficient reads of idle threads
  const int nvalid = z < nz1 ? max(0, min(4, nx - x0)) : 0;  // nodes x0 .. x0+3 that are x-interior (<= nx - 1)
  const long long plane = s.plane;
  const int gy0 = static_cast<int>(s.row_begin), gny = static_cast<int>(s.ny1);
  double* cft = s3r_smem + S3R_NS * G::STAGE;  // [by][w][28]
  const unsigned long long* bars = reinterpret_cast<const unsigned long long*>(cft + G::CF);
  const unsigned full0 = static_cast<unsigned>(__cvta_generic_to_shared(bars));
  const unsigned empty0 = full0 + 8 * S3R_NS;
  const unsigned smem0 = static_cast<unsigned>(__cvta_generic_to_shared(s3r_smem));

  // rows of the stage this warp copies: its own row (stage row w + 1) and, for
  // the first / last warp, the halo row below / above the tile; rows outside
  // the slab in z are never copied (zeroed once below)
  const int rA = w + 1, rB = w == 0 ? 0 : (w == W - 1 ? W + 1 : -1);
  const bool vA = z0 - 1 + rA < nz1;  // z0 - 1 + rA = z >= 0 always
  const bool vB = rB >= 0 && z0 - 1 + rB >= 0 && z0 - 1 + rB < nz1;
  const unsigned bytes_w = (vA ? S3R_COPY * 8u : 0u) + (vB ? S3R_COPY * 8u : 0u);
  if (threadIdx.x == 0) {
    for (int k = 0; k < S3R_NS; ++k) {
      mbar_init(full0 + 8 * k, W);   // one arrival (with its bytes) per warp
      mbar_init(empty0 + 8 * k, W);  // one arrival per warp once it has read the slot
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int t = threadIdx.x; t < S3R_NS * G::ROWS * S3R_RS; t += G::NT) {
    const int r = (t / S3R_RS) % G::ROWS, zz = z0 - 1 + r;
    if (zz < 0 || zz >= nz1) s3r_smem[t] = 0.0;
  }
  for (int t = threadIdx.x; t < G::CF; t += G::NT) {  // the block's coefficient rows for by = 0, 1, 2
    const int by = t / (W * 28), ww = (t / 28) % W, q = t % 28;
    const int zz = min(z0 + ww, nz1 - 1);
    const long long cls = (by * 3 + 1) * static_cast<long long>(nz1) + zz;
    cft[t] = q < 27 ? __ldg(s.coef + cls * 27 + q) : __ldg(s.cm + cls);
  }
  __syncthreads();

  // plane P_k = yb - 1 + k -> slot k % NS; lane 0 of every warp arms the full
  // barrier with its bytes and copies its rows (after the slot's previous
  // plane was read by every warp)
  auto issue = [&](int k, int slot, unsigned empty_par, bool wait_empty) {
    if (lane != 0) return;
    if (wait_empty) mbar_wait(empty0 + 8 * slot, empty_par);
    mbar_arrive_tx(full0 + 8 * slot, bytes_w);
    const long long pbase = static_cast<long long>(yb + k) * plane + xb - 1;  // (yl + 1) * plane, yl = yb - 1 + k
    auto copy_row = [&](int r) {
      const long long idx = pbase + static_cast<long long>(z0 - 1 + r) * nx1;
      const unsigned dst = smem0 + static_cast<unsigned>((slot * G::STAGE + r * S3R_RS) * 8);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
          "l"(a.vin + (idx & ~1ll)), "r"(S3R_COPY * 8), "r"(full0 + 8 * slot)
          : "memory");
    };
    if (vA) copy_row(rA);
    if (vB) copy_row(rB);
  };
  // parity of row w + dz's first node index in plane P_0; P_k flips it when k * plane is odd
  int sh0 = 0;
#pragma unroll
  for (int dz = 0; dz < 3; ++dz)
    sh0 |= static_cast<int>((static_cast<long long>(yb) * plane + xb - 1 + static_cast<long long>(z0 - 1 + w + dz) * nx1) &
                            1) << dz;
  const int pflip = (plane & 1) ? 7 : 0;
  // this warp's 18 window values of plane P_k (in `slot`); row r's first
  // copied node is x0 - 1 - sh with sh the parity of the row start's index
  auto window = [&](int k, int slot, unsigned full_par, double (&wv)[18]) {
    mbar_wait(full0 + 8 * slot, full_par);
    const int shk = sh0 ^ ((k & 1) ? pflip : 0);
#pragma unroll
    for (int dz = 0; dz < 3; ++dz) {
      const double* rp = s3r_smem + slot * G::STAGE + (w + dz) * S3R_RS + 4 * lane;  // col c <-> x0 - 1 - sh + c
      if ((shk >> dz) & 1) {  // x-1 at col 4l + 1
        const double2 q0 = *reinterpret_cast<const double2*>(rp + 2);
        const double2 q1 = *reinterpret_cast<const double2*>(rp + 4);
        wv[dz * 6 + 0] = rp[1];
        wv[dz * 6 + 1] = q0.x;
        wv[dz * 6 + 2] = q0.y;
        wv[dz * 6 + 3] = q1.x;
        wv[dz * 6 + 4] = q1.y;
        wv[dz * 6 + 5] = rp[6];
      } else {  // x-1 at col 4l
        const double2 q0 = *reinterpret_cast<const double2*>(rp);
        const double2 q1 = *reinterpret_cast<const double2*>(rp + 2);
        const double2 q2 = *reinterpret_cast<const double2*>(rp + 4);
        wv[dz * 6 + 0] = q0.x;
        wv[dz * 6 + 1] = q0.y;
        wv[dz * 6 + 2] = q1.x;
        wv[dz * 6 + 3] = q1.y;
        wv[dz * 6 + 4] = q2.x;
        wv[dz * 6 + 5] = q2.y;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * slot);
  };

  const int n = ye - yb;
  const int last_k = ye - (yb - 1);  // planes P_0 .. P_{n+1} are needed (P_{n+1} = plane ye <= planes)
  // ring bookkeeping by counters (no divisions): slot and phase of the next plane to read / to issue
  int rd_slot = 0, wr_slot = 0;
  unsigned rd_par = 0, wr_par = 0;
  for (int k = 0; k < S3R_NS && k <= last_k; ++k) {
    issue(k, wr_slot, 0, false);
    if (++wr_slot == S3R_NS) {
      wr_slot = 0;
      wr_par ^= 1;
    }
  }
  double P0[18], P1[18], P2[18];
  auto read_next = [&](int k, double (&wv)[18]) {
    window(k, rd_slot, rd_par, wv);
    if (++rd_slot == S3R_NS) {
      rd_slot = 0;
      rd_par ^= 1;
    }
  };
  read_next(0, P0);
  read_next(1, P1);
  double* outp = a.vout + static_cast<long long>(yb + 1) * plane + static_cast<long long>(zc) * nx1 + x0;
  const unsigned long long key0 =
      static_cast<unsigned long long>(static_cast<long long>(yb) * plane + static_cast<long long>(zc) * nx1 + x0 +
                                      s.row_begin * plane);
  const double* cfw = cft + w * 28;
  // plane step i: output plane y = yb + i from (m, o, p); p <- P_{i+2}
  auto step = [&](int i, double (&m)[18], double (&o)[18], double (&p)[18]) {
    read_next(i + 2, p);
    if (i + S3R_NS <= last_k) {  // into the slot of P_i (read by every warp at step i-2)
      issue(i + S3R_NS, wr_slot, wr_par ^ 1u, true);
      if (++wr_slot == S3R_NS) {
        wr_slot = 0;
        wr_par ^= 1;
      }
    }
    const int gy = gy0 + yb + i;
    const int by = gy == 0 ? 0 : (gy == gny - 1 ? 2 : 1);
    double out[4];
    s3r_quad(m, o, p, cfw + by * (W * 28), out);
    if (nvalid == 4) {
      outp[0] = out[0];
      outp[1] = out[1];
      outp[2] = out[2];
      outp[3] = out[3];
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < nvalid) outp[j] = out[j];
    }
    if (a.pl.on && (yb + i == 0 || yb + i == planes - 1)) {  // the slab's edge planes: also the neighbours' halos
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < nvalid) peer_store(a, yb + i, static_cast<long long>(zc) * nx1 + x0 + j, out[j]);
    }
    // one check for the four (a non-finite output makes the sum non-finite; a finite overflow of the sum
    // only sends the thread to the exact per-node test)
    if (!isfinite((out[0] + out[1]) + (out[2] + out[3]))) {
      const unsigned long long k = key0 + static_cast<unsigned long long>(i) * plane;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < nvalid && !isfinite(out[j])) record_failure(a.err, (k + j) << 22, seq, 2, 1, a.vin, a.vout);
    }
    outp += plane;
  };
  int i = 0;
  for (; i + 3 <= n; i += 3) {
    step(i, P0, P1, P2);
    step(i + 1, P1, P2, P0);
    step(i + 2, P2, P0, P1);
  }
  if (i < n) step(i, P0, P1, P2);
  if (i + 1 < n) step(i + 1, P1, P2, P0);
  // every copy this block issued has been waited for (P_{n+1}, the last issued plane, was read at step n-1)
}

template <int W>
static cudaError_t launch_s3r(const DiffArgs& a, const Struct3D& s, int num_sms, cudaStream_t st) {
  using G = S3R<W>;
  static std::atomic<uint64_t> attr_done{0};
  cudaError_t e = ensure_dyn_smem(diffuse_struct3d_rb<W>, static_cast<int>(G::smem), attr_done);
  if (e != cudaSuccess) return e;
  const long long nxi = s.nx1 - 2;  // x-interior nodes 1 .. nx-1
  const int tiles_x = nxi > 0 ? static_cast<int>((nxi + S3R_TX - 1) / S3R_TX) : 0;
  const int tiles_z = static_cast<int>((s.nz1 + W - 1) / W);
  const long long tiles = static_cast<long long>(tiles_x) * tiles_z;
  // y chunks: whole waves of 2 blocks per SM, chunks of >= 8 planes
  const long long slots = 2ll * num_sms;
  int nch = 1;
  double best = 1e30;
  for (int c = 1; c <= 64; ++c) {
    if (c > 1 && (s.planes + c - 1) / c < 8) break;
    const long long items = tiles * c;
    const double waves = static_cast<double>((items + slots - 1) / slots);
    const double cost = waves * static_cast<double>((s.planes + c - 1) / c) + 3.0 * waves;  // + pipeline fill
    if (cost < best - 1e-9) {
      best = cost;
      nch = c;
    }
  }
  const int ychunk = static_cast<int>((s.planes + nch - 1) / nch);
  const int n_items = static_cast<int>(tiles * nch);
  const long long n_edge = 2ll * s.nz1 * s.planes;
  const int edge_blocks = static_cast<int>(std::min<long long>((n_edge + G::NT - 1) / G::NT, 2ll * num_sms));
  if (n_items + edge_blocks == 0) return cudaSuccess;
  diffuse_struct3d_rb<W><<<n_items + edge_blocks, G::NT, G::smem, st>>>(a, s, tiles_x, tiles_z, n_items, ychunk,
                                                                         n_edge);
  return cudaGetLastError();
}

// Peer-memory halo push (multi-GPU P2P transport): after the reaction changed
// V in place, this rank's edge rows/planes of V buffer `par` go into the
// neighbours' halo rows (paced like a diffusion launch; no compute).
__global__ void __launch_bounds__(256) push_halo(DiffArgs a) {
  peer_wait(a.pl);
  const PeerLink& pl = a.pl;
  const long long per = pl.lim * pl.w;  // nodes per side
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < 2 * per;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const bool up = e >= per;
    const long long k = up ? e - per : e;
    const long long r = up ? pl.rows - pl.lim + k / pl.w : k / pl.w, xo = k % pl.w;
    const double val = a.vin[a.halo + r * pl.w + xo];
    if (!up && pl.lo_dst[a.out_par]) pl.lo_dst[a.out_par][r * pl.w + xo] = val;
    if (up && pl.hi_dst[a.out_par]) pl.hi_dst[a.out_par][(r - pl.rows) * pl.w + xo] = val;
  }
  peer_post(a.pl);
}

cudaError_t launch_push_halo(const DiffArgs& a, cudaStream_t st) {
  const long long per = a.pl.lim * a.pl.w;
  push_halo<<<blocks_for(2 * per, 256, 1024), 256, 0, st>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Generic CSR (fem.cpp:201-206), one thread per row, ascending columns.
// cols are local indices into vin; row i (owned) lives at vin[halo + i].
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(256) diffuse_csr(DiffArgs a, CsrDev m) {
  const long long seq = cur_seq(a.clock, a.step_off, a.evs, a.ev);
  const bool skip = earlier_failure(a.err, seq);
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < a.n;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (skip) return;  // an earlier event failed: V stays where it stopped
    const long long i = o + a.halo;
    double acc = 0.0;
    const long long p1 = m.row_ptr[o + 1];
    for (long long p = m.row_ptr[o]; p < p1; ++p) acc += m.val[p] * a.vin[m.col[p]];
    const double out = a.vin[i] - m.cm[o] * acc;
    a.vout[i] = out;
    if (!isfinite(out))
      record_failure(a.err, static_cast<unsigned long long>(o + a.node_offset) << 22, seq, 2, 1, a.vin, a.vout);
  }
}

// ---------------------------------------------------------------------------
// ActivationDetector::observe (postprocess.cpp:18-66), SoA node state.
// t = S*dt, previous sample time = (S - every)*dt, both computed exactly as
// the reference computed the times it stored (splitting.cpp:272).
// ---------------------------------------------------------------------------

__global__ void detector_init(const double* v, long long n, long long halo, DetDev d) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double x = v[i + halo];
  d.prev_v[i] = x;
  d.v_rest[i] = x;
  d.max_slope[i] = -INFINITY;
  d.t_max_slope[i] = 0.0;
  d.v_peak[i] = 0.0;
  d.lat[i] = 0.0;
  d.apd[i] = 0.0;
  d.phase[i] = 0;
  d.has_lat[i] = 0;
  d.has_apd[i] = 0;
}

__global__ void detector_observe(const double* v, long long n, long long halo, DetDev d, const long long* clock,
                                 long long s_off, long long every, double dt) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const long long S = *clock + s_off;
  const double t = static_cast<double>(S) * dt;
  const double pt = static_cast<double>(S - every) * dt;
  const double h = t - pt;
  if (d.phase[i] == 2) return;
  const double x = v[i + halo], px = d.prev_v[i];
  const double slope = (x - px) / h;
  if (slope > d.max_slope[i]) {
    d.max_slope[i] = slope;
    d.t_max_slope[i] = pt + 0.5 * h;
  }
  const double thr = d.threshold;
  if (d.phase[i] == 0) {
    if (px < thr && x >= thr) {
      d.lat[i] = pt + (thr - px) / (x - px) * h;
      d.has_lat[i] = 1;
      d.phase[i] = 1;
      d.v_peak[i] = x;
    } else {
      const double r = d.v_rest[i];
      d.v_rest[i] = x < r ? x : r;  // std::min(r, x)
    }
  } else {
    double pk = d.v_peak[i];
    pk = pk < x ? x : pk;  // std::max(pk, x)
    d.v_peak[i] = pk;
    const double rest = d.v_rest[i];
    const double v90 = pk - 0.9 * (pk - rest);
    if (px >= v90 && x < v90 && pk - rest >= 20.0) {
      const double tc = pt + (px - v90) / (px - x) * h;
      d.apd[i] = tc - d.t_max_slope[i];
      d.has_apd[i] = 1;
      d.phase[i] = 2;
    }
  }
  d.prev_v[i] = x;
}

// probe samples: out[sample * np + p] = v[loc[p]] for owned probes (loc >= 0)
__global__ void record_probes(const double* v, const long long* loc, int np, double* out, const long long* clock,
                              long long s_off, long long every) {
  const int p = threadIdx.x + blockIdx.x * blockDim.x;
  if (p >= np) return;
  const long long S = *clock + s_off;
  const long long sample = S / every;
  const long long l = loc[p];
  out[sample * np + p] = l >= 0 ? v[l] : 0.0;
}

__global__ void set_clock(long long* clock, long long value) { *clock = value; }

// diastolic_threshold probe (stimulus.cpp:107): first step whose V[probe] > 0
__global__ void probe_cross(const double* v, long long probe, long long* cross, const long long* clock, long long off) {
  if (v[probe] > 0.0) atomicMin(reinterpret_cast<unsigned long long*>(cross), static_cast<unsigned long long>(*clock + off));
}
__global__ void tick_clock(long long* clock, long long by) { *clock += by; }

// AoS (NodeStateArray::s, ionic.hpp:44) <-> SoA chunk transposes
__global__ void aos_to_soa(const double* aos, int stride, int ns, long long count, double* soa, long long pitch,
                           long long dst0) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= count) return;
  for (int q = 0; q < ns; ++q) soa[sidx(q, dst0 + i, pitch)] = aos[i * stride + q];
}

__global__ void soa_to_aos(const double* soa, long long pitch, long long src0, int ns, long long count, double* aos,
                           int stride) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= count) return;
  for (int q = 0; q < ns; ++q) aos[i * stride + q] = soa[sidx(q, src0 + i, pitch)];
  for (int q = ns; q < stride; ++q) aos[i * stride + q] = 0.0;
}

// make_initial_state on the device (splitting.cpp:183-217 with rest states):
// V, all stride state slots (0 beyond the model's count) and last_dvdt = 0.
__global__ void init_rest(double* v, double* S, long long pitch, double* last, const int32_t* list, long long first,
                          long long count, const double* rest, int ns, int stride) {
  const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (p >= count) return;
  const long long i = list ? static_cast<long long>(list[p]) : first + p;
  v[i] = rest[0];
  last[i] = 0.0;
  for (int q = 0; q < stride; ++q) S[sidx(q, i, pitch)] = q < ns ? rest[q + 1] : 0.0;
}

// standalone diffusion_substep for cwg_diffusion_substep (no halo, no error record)
__global__ void diffuse_csr_plain(long long n, const long long* rp, const long long* col, const double* val,
                                  const double* mass, const double* v, double dt_sub, double* out) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (long long p = rp[i]; p < rp[i + 1]; ++p) acc += val[p] * v[col[p]];
  out[i] = v[i] - dt_sub / mass[i] * acc;
}

// cm[i] = dt_sub / m_i
__global__ void mass_factor(const double* mass, long long n, double dt_sub, double* cm) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i < n) cm[i] = dt_sub / mass[i];
}

// FP64 peak probe: 8 independent DFMA chains per thread (explicit fma(), so
// --fmad=false does not matter), iterated; one result store keeps it alive.
__global__ void __launch_bounds__(256) fp64_peak(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) x[q] = threadIdx.x * 1e-3 + q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = fma(x[q], a, b);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += x[q];
  if (s == 1.2345) out[0] = s;
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
static inline int blocks_for(long long n, int t, int cap) {
  long long b = (n + t - 1) / t;
  if (b > cap) b = cap;
  return static_cast<int>(b < 1 ? 1 : b);
}

cudaError_t launch_diffuse_stencil2d(const DiffArgs& a, const Stencil2D& s, int max_blocks, cudaStream_t st) {
  diffuse_stencil2d<<<blocks_for(s.rows * s.w, 256, max_blocks), 256, 0, st>>>(a, s);
  return cudaGetLastError();
}

// The y-chunk trades halo-plane reloads (a block loads chunk + 3 planes)
// against parallelism for this latency-bound loop: the largest chunk in
// [4, 16] that still gives >= 4 waves of resident blocks (C4: 4, C5: 16;
// measured C4 0.140 / 0.153 / 0.163 ms per step at 4 / 8 / 16, C5 flat).
// CWG_S3_YCHUNK overrides for experiments.
static cudaError_t launch_diffuse_struct3d_ring(const DiffArgs& a, const Struct3D& s_in, int num_sms, cudaStream_t st);

// Default: the register-blocked kernel; CWG_S3_KERNEL=0 selects the shared-memory ring kernel (A/B runs).
cudaError_t launch_diffuse_struct3d(const DiffArgs& a, const Struct3D& s, int num_sms, cudaStream_t st) {
  const char* e = getenv("CWG_S3_KERNEL");  // read per launch (graphs capture it once)
  if ((e && atoi(e) == 0) || s.nx1 < 2 || s.nz1 < 2) return launch_diffuse_struct3d_ring(a, s, num_sms, st);
  return launch_s3r<6>(a, s, num_sms, st);
}

static cudaError_t launch_diffuse_struct3d_ring(const DiffArgs& a, const Struct3D& s_in, int num_sms, cudaStream_t st) {
  static int capacity = 0;
  if (capacity == 0) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, diffuse_struct3d, S3_TX * S3_TZ, 0);
    capacity = std::max(1, per_sm) * num_sms;
  }
  static const int forced = [] {
    const char* e = getenv("CWG_S3_YCHUNK");
    return e ? atoi(e) : 0;
  }();
  Struct3D s = s_in;
  const long long xz = ((s.nx1 + S3_TX - 1) / S3_TX) * ((s.nz1 + S3_TZ - 1) / S3_TZ);
  s.ychunk = 4;
  for (int ch = 16; ch >= 4; --ch)
    if (xz * ((s.planes + ch - 1) / ch) >= 4ll * capacity) {
      s.ychunk = ch;
      break;
    }
  if (forced > 0) s.ychunk = forced;
  const dim3 grid(static_cast<unsigned>((s.nx1 + S3_TX - 1) / S3_TX), static_cast<unsigned>((s.nz1 + S3_TZ - 1) / S3_TZ),
                  static_cast<unsigned>((s.planes + s.ychunk - 1) / s.ychunk));
  diffuse_struct3d<<<grid, S3_TX * S3_TZ, 0, st>>>(a, s);
  return cudaGetLastError();
}

cudaError_t launch_diffuse_csr(const DiffArgs& a, const CsrDev& m, int max_blocks, cudaStream_t st) {
  diffuse_csr<<<blocks_for(a.n, 256, max_blocks), 256, 0, st>>>(a, m);
  return cudaGetLastError();
}

cudaError_t launch_detector_init(const double* v, long long n, long long halo, const DetDev& d, cudaStream_t st) {
  detector_init<<<blocks_for(n, 256, 1 << 30), 256, 0, st>>>(v, n, halo, d);
  return cudaGetLastError();
}

cudaError_t launch_detector_observe(const double* v, long long n, long long halo, const DetDev& d,
                                    const long long* clock, long long s_off, long long every, double dt,
                                    cudaStream_t st) {
  detector_observe<<<blocks_for(n, 256, 1 << 30), 256, 0, st>>>(v, n, halo, d, clock, s_off, every, dt);
  return cudaGetLastError();
}

cudaError_t launch_record_probes(const double* v, const long long* loc, int np, double* out, const long long* clock,
                                 long long s_off, long long every, cudaStream_t st) {
  if (np == 0) return cudaSuccess;
  record_probes<<<(np + 127) / 128, 128, 0, st>>>(v, loc, np, out, clock, s_off, every);
  return cudaGetLastError();
}

cudaError_t launch_probe_cross(const double* v, long long probe, long long* cross, const long long* clock,
                               long long off, cudaStream_t st) {
  probe_cross<<<1, 1, 0, st>>>(v, probe, cross, clock, off);
  return cudaGetLastError();
}

cudaError_t launch_set_clock(long long* clock, long long value, cudaStream_t st) {
  set_clock<<<1, 1, 0, st>>>(clock, value);
  return cudaGetLastError();
}

cudaError_t launch_tick_clock(long long* clock, long long by, cudaStream_t st) {
  tick_clock<<<1, 1, 0, st>>>(clock, by);
  return cudaGetLastError();
}

cudaError_t launch_aos_to_soa(const double* aos, int stride, int ns, long long count, double* soa, long long pitch,
                              long long dst0, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  aos_to_soa<<<blocks_for(count, 256, 1 << 30), 256, 0, st>>>(aos, stride, ns, count, soa, pitch, dst0);
  return cudaGetLastError();
}

cudaError_t launch_soa_to_aos(const double* soa, long long pitch, long long src0, int ns, long long count,
                              double* aos, int stride, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  soa_to_aos<<<blocks_for(count, 256, 1 << 30), 256, 0, st>>>(soa, pitch, src0, ns, count, aos, stride);
  return cudaGetLastError();
}

cudaError_t launch_diffuse_csr_plain(long long n, const long long* rp, const long long* col, const double* val,
                                     const double* mass, const double* v, double dt_sub, double* out,
                                     cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  diffuse_csr_plain<<<blocks_for(n, 256, 1 << 30), 256, 0, st>>>(n, rp, col, val, mass, v, dt_sub, out);
  return cudaGetLastError();
}

cudaError_t launch_fp64_peak(double* out, int blocks, int iters, cudaStream_t st) {
  fp64_peak<<<blocks, 256, 0, st>>>(out, iters, 0.999999, 1e-7);
  return cudaGetLastError();
}

cudaError_t launch_init_rest(double* v, double* S, long long pitch, double* last, const int32_t* list,
                              long long first, long long count, const double* rest, int ns, int stride,
                              cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  init_rest<<<blocks_for(count, 256, 1 << 30), 256, 0, st>>>(v, S, pitch, last, list, first, count, rest, ns, stride);
  return cudaGetLastError();
}

namespace {
__global__ void map_values(const double* val, const unsigned char* has, long long n, double* out) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = has[i] ? val[i] : __longlong_as_double(0x7ff8000000000000ll);
}

// ProtocolIndex pointer array of a slab context from the caller's global one
// (gptr = its owned slice, n_own + 1 entries): 0 over the lower halo, rebased
// over the owned nodes, the total over the upper halo.
__global__ void stim_local_ptr(const int32_t* gptr, long long n_own, long long halo, long long n_alloc,
                               int32_t* ptr) {
  const long long li = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (li > n_alloc) return;
  const int32_t base = gptr[0];
  int32_t v;
  if (li <= halo) v = 0;
  else if (li <= halo + n_own) v = gptr[li - halo] - base;
  else v = gptr[n_own] - base;
  ptr[li] = v;  // ptr[li] = entries of local nodes < li
}
}  // namespace

cudaError_t launch_map_values(const double* val, const unsigned char* has, long long n, double* out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  map_values<<<blocks_for(n, 256, 1 << 30), 256, 0, st>>>(val, has, n, out);
  return cudaGetLastError();
}

cudaError_t launch_stim_local_ptr(const int32_t* gptr, long long n_own, long long halo, long long n_alloc,
                                  int32_t* ptr, cudaStream_t st) {
  stim_local_ptr<<<blocks_for(n_alloc + 1, 256, 1 << 30), 256, 0, st>>>(gptr, n_own, halo, n_alloc, ptr);
  return cudaGetLastError();
}

cudaError_t launch_mass_factor(const double* mass, long long n, double dt_sub, double* cm, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  mass_factor<<<blocks_for(n, 256, 1 << 30), 256, 0, st>>>(mass, n, dt_sub, cm);
  return cudaGetLastError();
}

}  // namespace cwg
