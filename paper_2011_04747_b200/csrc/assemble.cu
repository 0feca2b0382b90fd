// Regular-sheet operator assembly ON THE DEVICE:
// build_diffusion_field (fem.cpp:21-51), the bilinear element integrals with
// row-sum lumping (fem.cpp:63-108), CSR accumulation (fem.cpp:112-152), the
// structural checks (fem.cpp:154-172) and gershgorin_step (fem.cpp:178-192),
// with no host triplet sort. One thread per node gathers the row of its
// (up to) four elements instead of scattering element matrices, and writes
// the stencil layout the diffusion kernels read (coef[slot][n], slot =
// (dy+1)*3 + (dx+1) = ascending column order).
//
// Bits (compiled with --fmad=false, the reference's evaluation order):
//  * lumped mass: sum over the node's elements in ascending element index
//    from 0.0 -- exactly mass[ia] += m[a] of the reference's element loop;
//  * off-diagonal entries: one or two element contributions, and a + b is
//    commutative -- identical to the reference whatever its sort order;
//  * diagonal: four contributions, summed here in ascending element index;
//    the reference sums them in the order std::sort leaves equal (i, i)
//    triplets (unstable, fem.cpp:135-137), so a diagonal can differ from the
//    reference's by 1-2 ulp (measured: tests/test_gpu_assembly.py).
// The host assembly (setup.cpp) stays the bit-identical path; this one is
// the scaling path (no O(nnz log nnz) host sort, no CSR upload).
#include "launch.h"

namespace cwg {

namespace {

constexpr double kGauss = 0.57735026918962576;  // 1/sqrt(3), fem.cpp:56

// Element e's diffusion tensor (fem.cpp:36-47, + the per-element scale extension)
__device__ __forceinline__ void element_tensor(const Sheet2DDev& g, long long ex, long long ey, double& dxx,
                                               double& dxy, double& dyy) {
  const long long w = g.nx + 1;
  const long long n0 = ey * w + ex;
  bool fib = false;
  if (g.tags) fib = g.tags[n0] == 1 || g.tags[n0 + 1] == 1 || g.tags[n0 + 1 + w] == 1 || g.tags[n0 + w] == 1;
  double dl = fib ? g.d0f : g.d0m;
  if (g.escale) dl = dl * g.escale[ey * g.nx + ex];
  const double dt = g.rho * dl;
  dxx = dl * g.fx * g.fx + dt * (1.0 - g.fx * g.fx);
  dxy = (dl - dt) * g.fx * g.fy;
  dyy = dl * g.fy * g.fy + dt * (1.0 - g.fy * g.fy);
}

// Row a of the element stiffness and m[a] (fem.cpp:63-108), element corners
// (x0, y0) + {(0,0), (h,0), (h,h), (0,h)}: the same operations in the same
// order as the reference's full 4x4 loop, only for the one row this node needs.
__device__ __forceinline__ bool element_row(double x0, double y0, double x1, double y1, double dxx, double dxy,
                                            double dyy, int a, double k[4], double& m) {
  const double xs[4] = {x0, x1, x1, x0}, ys[4] = {y0, y0, y1, y1};
  const double gp[2] = {-kGauss, kGauss};
  for (int b = 0; b < 4; ++b) k[b] = 0.0;
  m = 0.0;
  bool ok = true;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const double xi = gp[q], eta = gp[r];
      const double shp[4] = {0.25 * (1 - xi) * (1 - eta), 0.25 * (1 + xi) * (1 - eta), 0.25 * (1 + xi) * (1 + eta),
                             0.25 * (1 - xi) * (1 + eta)};
      const double dxi[4] = {-0.25 * (1 - eta), 0.25 * (1 - eta), 0.25 * (1 + eta), -0.25 * (1 + eta)};
      const double deta[4] = {-0.25 * (1 - xi), -0.25 * (1 + xi), 0.25 * (1 + xi), 0.25 * (1 - xi)};
      double j00 = 0, j01 = 0, j10 = 0, j11 = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        j00 += dxi[c] * xs[c];
        j01 += dxi[c] * ys[c];
        j10 += deta[c] * xs[c];
        j11 += deta[c] * ys[c];
      }
      const double det = j00 * j11 - j01 * j10;
      if (!(det > 0.0)) ok = false;
      const double i00 = j11 / det, i01 = -j01 / det;
      const double i10 = -j10 / det, i11 = j00 / det;
      double gx[4], gy[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        gx[c] = i00 * dxi[c] + i01 * deta[c];
        gy[c] = i10 * dxi[c] + i11 * deta[c];
      }
      const double fxa = dxx * gx[a] + dxy * gy[a];
      const double fya = dxy * gx[a] + dyy * gy[a];
#pragma unroll
      for (int b = 0; b < 4; ++b) k[b] += det * (fxa * gx[b] + fya * gy[b]);
      m += det * shp[a];
    }
  }
  return ok;
}

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* p, double x) {
  if (x == x) atomicMax(p, static_cast<unsigned long long>(__double_as_longlong(x)));  // NaN: std::max ignores it
}

// Pass 1: rows, masses, max |k_ij|, the first degenerate element.
__global__ void __launch_bounds__(256) sheet2d_rows_kernel(Sheet2DDev g, AsmOut o) {
  const long long w = g.nx + 1, n = w * (g.ny + 1);
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  double vmax = 0.0;
  if (i < n) {
    const long long iy = i / w, ix = i - iy * w;
    double acc[9];
    bool have[9];
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      acc[s] = 0.0;
      have[s] = false;
    }
    double mass = 0.0;
    // the node's elements in ascending element index, with its local vertex there
    const int dys[4] = {-1, -1, 0, 0}, dxs[4] = {-1, 0, -1, 0}, loc[4] = {2, 3, 1, 0};
    // local vertex b of an element -> (dx, dy) of that vertex from the element's corner n0
    const int vbx[4] = {0, 1, 1, 0}, vby[4] = {0, 0, 1, 1};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long ey = iy + dys[q], ex = ix + dxs[q];
      if (ey < 0 || ey >= g.ny || ex < 0 || ex >= g.nx) continue;
      double dxx, dxy, dyy;
      element_tensor(g, ex, ey, dxx, dxy, dyy);
      const double x0 = static_cast<double>(ex) * g.h, y0 = static_cast<double>(ey) * g.h;
      const double x1 = static_cast<double>(ex + 1) * g.h, y1 = static_cast<double>(ey + 1) * g.h;
      double k[4], m;
      const int a = loc[q];
      if (!element_row(x0, y0, x1, y1, dxx, dxy, dyy, a, k, m))
        atomicMin(o.keys + 0, static_cast<unsigned long long>(ey * g.nx + ex));
      mass += m;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        // neighbour = element corner + vertex b; offset from node i = (corner - i) + vertex b
        const int dx = static_cast<int>(ex - ix) + vbx[b], dy = static_cast<int>(ey - iy) + vby[b];
        const int s = (dy + 1) * 3 + (dx + 1);
        acc[s] = have[s] ? acc[s] + k[b] : k[b];  // "sum = first; sum += next" (fem.cpp:142-145)
        have[s] = true;
      }
    }
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      o.coef[s * n + i] = acc[s];  // absent neighbours: 0, never read
      if (have[s]) vmax = fmax(vmax, fabs(acc[s]));
    }
    o.mass[i] = mass;
    int cnt = 0;
#pragma unroll
    for (int s = 0; s < 9; ++s) cnt += have[s] ? 1 : 0;
    o.nnz_row[i] = static_cast<unsigned char>(cnt);
  }
  // block max of |k_ij|, one atomic per block
  __shared__ double red[8];
  for (int off = 16; off > 0; off >>= 1) vmax = fmax(vmax, __shfl_down_sync(0xffffffffu, vmax, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = vmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (blockDim.x + 31) / 32; ++q) vmax = fmax(vmax, red[q]);
    atomic_max_nonneg(o.keys + 3, vmax);
  }
}

// Pass 2 (needs the global max |k_ij|): structural checks (fem.cpp:154-172)
// and the Gershgorin ratio (fem.cpp:178-192) of every row.
//   keys[1] = min over failing nodes of node*16 + what (0 mass, 1+p symmetry at
//             the row's p-th entry, 15 row sum): the reference's first throw
//   keys[2] = first row with k_ii + sum|k_ij| <= 0;  keys[4] = min m_i / den_i
__global__ void __launch_bounds__(256) sheet2d_check_kernel(Sheet2DDev g, AsmOut o) {
  const long long w = g.nx + 1, n = w * (g.ny + 1);
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const long long iy = i / w, ix = i - iy * w;
  const double max_abs = __longlong_as_double(static_cast<long long>(o.keys[3]));
  const double tol_sym = 1e-12 * fmax(1.0, max_abs), tol_sum = 1e-10 * fmax(1e-300, max_abs);
  const double m = o.mass[i];
  unsigned long long fail = ~0ull;
  if (!(m > 0.0)) fail = static_cast<unsigned long long>(i) * 16;
  double row_sum = 0.0, den = 0.0;
  bool zero_row = true;
  int p = 0;
  for (int s = 0; s < 9; ++s) {
    const long long jy = iy + s / 3 - 1, jx = ix + s % 3 - 1;
    if (jy < 0 || jy > g.ny || jx < 0 || jx > g.nx) continue;
    const long long j = jy * w + jx;
    const double v = o.coef[s * n + i];
    row_sum += v;
    const double vt = o.coef[(8 - s) * n + j];  // entry (j, i): the opposite slot of row j
    if (fail == ~0ull && fabs(v - vt) > tol_sym) fail = static_cast<unsigned long long>(i) * 16 + 1 + p;
    den += s == 4 ? v : fabs(v);
    if (v != 0.0) zero_row = false;
    ++p;
  }
  if (fail == ~0ull && fabs(row_sum) > tol_sum) fail = static_cast<unsigned long long>(i) * 16 + 15;
  if (fail != ~0ull) atomicMin(o.keys + 1, fail);
  if (g.escale && zero_row) return;  // scar rows do not diffuse (extension, as setup.cpp)
  if (!(den > 0.0)) {
    atomicMin(o.keys + 2, static_cast<unsigned long long>(i));
    return;
  }
  const double ratio = m / den;
  if (ratio == ratio) atomicMin(o.keys + 4, static_cast<unsigned long long>(__double_as_longlong(ratio)));
}

// Copy rows [g0, g0 + rows) of the full [9][n] table into a [9][rows*w]
// slab table (rows outside the sheet: coefficients 0, mass 1 -- never read).
__global__ void sheet2d_slice_kernel(const double* coef, const double* mass, long long n, long long w, long long g0,
                                     long long cnt, double* coef_out, double* mass_out) {
  const long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (o >= cnt) return;
  const long long i = g0 + o;
  const bool in = i >= 0 && i < n;
  for (int s = 0; s < 9; ++s) coef_out[s * cnt + o] = in ? coef[s * n + i] : 0.0;
  mass_out[o] = in ? mass[i] : 1.0;
}

}  // namespace

cudaError_t launch_sheet2d_assemble(const Sheet2DDev& g, const AsmOut& o, cudaStream_t st) {
  const long long n = (g.nx + 1) * (g.ny + 1);
  const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
  const unsigned long long init[5] = {~0ull, ~0ull, ~0ull, 0ull, 0x7ff0000000000000ull};
  cudaError_t e = cudaMemcpyAsync(o.keys, init, sizeof(init), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  sheet2d_rows_kernel<<<blocks, 256, 0, st>>>(g, o);
  sheet2d_check_kernel<<<blocks, 256, 0, st>>>(g, o);
  return cudaGetLastError();
}

cudaError_t launch_sheet2d_slice(const double* coef, const double* mass, long long n, long long w, long long g0,
                                 long long cnt, double* coef_out, double* mass_out, cudaStream_t st) {
  if (cnt <= 0) return cudaSuccess;
  sheet2d_slice_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, st>>>(coef, mass, n, w, g0, cnt, coef_out,
                                                                                  mass_out);
  return cudaGetLastError();
}

}  // namespace cwg
