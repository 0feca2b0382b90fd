// Host-side problem setup (include/cwgpu_setup.h): the regular-sheet mesh,
// fibrosis tags, element diffusion tensors, bilinear-quad assembly with
// row-sum lumping and the Gershgorin step, restated from the reference setup
// path (mesh.cpp:72-180, fem.cpp:21-192) so that the GPU box can build
// BASELINE's operators without the reference tree. Compiled with g++ and
// -ffp-contract=off; the element integrals keep the reference's evaluation
// order and the triplets go through the same std::sort, so the CSR is
// bit-identical to cardwave::assemble (tests/test_setup_parity.py).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "../../include/cwgpu_setup.h"

struct cwg_sheet {
  int64_t nx = 0, ny = 0;  // element counts
  double h = 0.0;
  std::vector<double> xy;     // [n][2]
  std::vector<int32_t> tags;  // 0 myocyte-epi, 1 fibroblast
  std::vector<int64_t> row_ptr, col;
  std::vector<double> val, mass;
  double dt_s = 0.0;
  int64_t n() const { return (nx + 1) * (ny + 1); }
};

namespace {

struct SetupError {
  std::string msg;
};

void fail(cwg_error* e, const std::string& m) {
  if (!e) return;
  e->code = CWG_EVALIDATION;
  e->node = -1;
  e->t_ms = 0.0;
  e->phase = 0;
  std::snprintf(e->msg, sizeof(e->msg), "%s", m.c_str());
}

int64_t cells_along(double length, double h, const char* axis) {  // mesh.cpp:17-27
  const double q = length / h;
  const double r = std::round(q);
  if (r < 1.0 || std::abs(q - r) > 1e-9 * std::max(1.0, q))
    throw SetupError{std::string("mesh: ") + axis + " extent " + std::to_string(length) +
                     " cm is not a positive multiple of h = " + std::to_string(h) + " cm"};
  return static_cast<int64_t>(r);
}

struct Tensor2 {
  double xx, xy, yy;
};

// Element stiffness and lumped mass (fem.cpp:63-108): 2x2 Gauss on [-1,1]^2.
void element_integrals(const double xs[4], const double ys[4], const Tensor2& D, int64_t e, double k[4][4],
                       double m[4]) {
  constexpr double g = 0.57735026918962576;
  const double gp[2] = {-g, g};
  for (int a = 0; a < 4; ++a) {
    m[a] = 0.0;
    for (int b = 0; b < 4; ++b) k[a][b] = 0.0;
  }
  for (double xi : gp) {
    for (double eta : gp) {
      const double shp[4] = {0.25 * (1 - xi) * (1 - eta), 0.25 * (1 + xi) * (1 - eta), 0.25 * (1 + xi) * (1 + eta),
                             0.25 * (1 - xi) * (1 + eta)};
      const double dxi[4] = {-0.25 * (1 - eta), 0.25 * (1 - eta), 0.25 * (1 + eta), -0.25 * (1 + eta)};
      const double deta[4] = {-0.25 * (1 - xi), -0.25 * (1 + xi), 0.25 * (1 + xi), 0.25 * (1 - xi)};
      double j00 = 0, j01 = 0, j10 = 0, j11 = 0;
      for (int a = 0; a < 4; ++a) {
        j00 += dxi[a] * xs[a];
        j01 += dxi[a] * ys[a];
        j10 += deta[a] * xs[a];
        j11 += deta[a] * ys[a];
      }
      const double det = j00 * j11 - j01 * j10;
      if (!(det > 0.0))
        throw SetupError{"assemble: element " + std::to_string(e) +
                         " has non-positive Jacobian (degenerate or clockwise)"};
      const double i00 = j11 / det, i01 = -j01 / det;
      const double i10 = -j10 / det, i11 = j00 / det;
      double gx[4], gy[4];
      for (int a = 0; a < 4; ++a) {
        gx[a] = i00 * dxi[a] + i01 * deta[a];
        gy[a] = i10 * dxi[a] + i11 * deta[a];
      }
      for (int a = 0; a < 4; ++a) {
        const double fx = D.xx * gx[a] + D.xy * gy[a];
        const double fy = D.xy * gx[a] + D.yy * gy[a];
        for (int b = 0; b < 4; ++b) k[a][b] += det * (fx * gx[b] + fy * gy[b]);
        m[a] += det * shp[a];
      }
    }
  }
}

double entry(const cwg_sheet& s, int64_t i, int64_t j) {
  for (int64_t p = s.row_ptr[i]; p < s.row_ptr[i + 1]; ++p)
    if (s.col[p] == j) return s.val[p];
  return 0.0;
}

void build(cwg_sheet& s, double lx, double ly, double h, double angle, double d0m, double d0f, double rho,
           double frac, uint64_t seed, const double* elem_scale, bool assemble = true) {
  if (!(h > 0.0) || !std::isfinite(h)) throw SetupError{"mesh: spacing h must be positive and finite"};
  s.nx = cells_along(lx, h, "x");
  s.ny = cells_along(ly, h, "y");
  s.h = h;
  const int64_t w = s.nx + 1, n = s.n(), ne = s.nx * s.ny;
  s.xy.resize(static_cast<size_t>(2 * n));
  for (int64_t iy = 0; iy <= s.ny; ++iy)
    for (int64_t ix = 0; ix <= s.nx; ++ix) {
      s.xy[2 * (iy * w + ix)] = static_cast<double>(ix) * h;
      s.xy[2 * (iy * w + ix) + 1] = static_cast<double>(iy) * h;
    }
  s.tags.assign(static_cast<size_t>(n), 0);

  // assign_fibrosis (mesh.cpp:100-122): hand-rolled Fisher-Yates over mt19937_64
  if (frac < 0.0 || frac > 1.0) throw SetupError{"fibrosis: fraction must lie in [0, 1]"};
  const int64_t n_sel = static_cast<int64_t>(std::llround(frac * static_cast<double>(n)));
  bool any_fib = false;
  if (frac > 0.0 && n_sel > 0) {
    std::vector<int64_t> idx(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) idx[static_cast<size_t>(i)] = i;
    std::mt19937_64 gen(seed);
    for (int64_t i = n - 1; i > 0; --i) {
      const uint64_t j = gen() % static_cast<uint64_t>(i + 1);
      std::swap(idx[static_cast<size_t>(i)], idx[j]);
    }
    for (int64_t q = 0; q < n_sel; ++q) s.tags[static_cast<size_t>(idx[static_cast<size_t>(q)])] = 1;
    any_fib = true;
  }

  if (!assemble) return;  // mesh only: the operator is assembled on the device (assemble.cu)

  // build_diffusion_field (fem.cpp:21-51), D = dl f f^T + dt (I - f f^T)
  if (!(d0m > 0.0) || !(d0f > 0.0)) throw SetupError{"diffusion: coefficients must be positive"};
  if (!(rho > 0.0 && rho <= 1.0)) throw SetupError{"diffusion: rho must lie in (0, 1]"};
  const double fx = std::cos(angle), fy = std::sin(angle);

  // triplet assembly (fem.cpp:112-152)
  struct Triplet {
    int64_t i, j;
    double v;
  };
  std::vector<Triplet> trip;
  trip.reserve(static_cast<size_t>(ne) * 16);
  s.mass.assign(static_cast<size_t>(n), 0.0);
  for (int64_t ey = 0; ey < s.ny; ++ey)
    for (int64_t ex = 0; ex < s.nx; ++ex) {
      const int64_t e = ey * s.nx + ex;
      const int64_t n0 = ey * w + ex;
      const int64_t nodes[4] = {n0, n0 + 1, n0 + 1 + w, n0 + w};
      bool fib = false;
      if (any_fib)
        for (int a = 0; a < 4; ++a)
          if (s.tags[static_cast<size_t>(nodes[a])] == 1) fib = true;
      double dl = fib ? d0f : d0m;
      if (elem_scale) dl = dl * elem_scale[e];  // extension (x * 1.0 == x)
      const double dt = rho * dl;
      const Tensor2 D{dl * fx * fx + dt * (1.0 - fx * fx), (dl - dt) * fx * fy, dl * fy * fy + dt * (1.0 - fy * fy)};
      double xs[4], ys[4];
      for (int a = 0; a < 4; ++a) {
        xs[a] = s.xy[static_cast<size_t>(2 * nodes[a])];
        ys[a] = s.xy[static_cast<size_t>(2 * nodes[a] + 1)];
      }
      double k[4][4], m[4];
      element_integrals(xs, ys, D, e, k, m);
      for (int a = 0; a < 4; ++a) {
        s.mass[static_cast<size_t>(nodes[a])] += m[a];
        for (int b = 0; b < 4; ++b) trip.push_back({nodes[a], nodes[b], k[a][b]});
      }
    }
  std::sort(trip.begin(), trip.end(),
            [](const Triplet& a, const Triplet& b) { return a.i != b.i ? a.i < b.i : a.j < b.j; });
  s.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
  s.col.clear();
  s.val.clear();
  for (size_t t = 0; t < trip.size();) {
    size_t u = t + 1;
    double sum = trip[t].v;
    while (u < trip.size() && trip[u].i == trip[t].i && trip[u].j == trip[t].j) sum += trip[u++].v;
    s.col.push_back(trip[t].j);
    s.val.push_back(sum);
    ++s.row_ptr[static_cast<size_t>(trip[t].i + 1)];
    t = u;
  }
  for (int64_t i = 0; i < n; ++i) s.row_ptr[static_cast<size_t>(i + 1)] += s.row_ptr[static_cast<size_t>(i)];

  // structural checks (fem.cpp:154-172)
  double max_abs = 0.0;
  for (double v : s.val) max_abs = std::max(max_abs, std::abs(v));
  for (int64_t i = 0; i < n; ++i) {
    if (!(s.mass[static_cast<size_t>(i)] > 0.0))
      throw SetupError{"assemble: non-positive lumped mass at node " + std::to_string(i)};
    double row_sum = 0.0;
    for (int64_t p = s.row_ptr[i]; p < s.row_ptr[i + 1]; ++p) {
      row_sum += s.val[p];
      if (std::abs(s.val[p] - entry(s, s.col[p], i)) > 1e-12 * std::max(1.0, max_abs))
        throw SetupError{"assemble: stiffness not symmetric at (" + std::to_string(i) + ", " +
                         std::to_string(s.col[p]) + ")"};
    }
    if (std::abs(row_sum) > 1e-10 * std::max(1e-300, max_abs))
      throw SetupError{"assemble: row " + std::to_string(i) + " sum " + std::to_string(row_sum) + " not zero"};
  }

  // gershgorin_step (fem.cpp:178-192); with elem_scale, all-zero rows (scar
  // interior, extension) do not diffuse and are skipped.
  double min_ratio = std::numeric_limits<double>::infinity();
  for (int64_t i = 0; i < n; ++i) {
    double den = 0.0;
    bool zero_row = true;
    for (int64_t p = s.row_ptr[i]; p < s.row_ptr[i + 1]; ++p) {
      den += s.col[p] == i ? s.val[p] : std::abs(s.val[p]);
      if (s.val[p] != 0.0) zero_row = false;
    }
    if (elem_scale && zero_row) continue;
    if (!(den > 0.0))
      throw SetupError{"gershgorin: row " + std::to_string(i) +
                       " has non-positive k_ii + sum|k_ij|; operator is not diffusive"};
    min_ratio = std::min(min_ratio, s.mass[static_cast<size_t>(i)] / den);
  }
  if (!std::isfinite(min_ratio)) throw SetupError{"gershgorin: no diffusive row"};
  s.dt_s = 0.9 * min_ratio;
}

}  // namespace

extern "C" {

int cwg_sheet_build(double lx, double ly, double h, double angle, double d0m, double d0f, double rho, double frac,
                    uint64_t seed, const double* elem_scale, cwg_sheet** out, cwg_error* err) {
  auto* s = new cwg_sheet();
  try {
    build(*s, lx, ly, h, angle, d0m, d0f, rho, frac, seed, elem_scale);
  } catch (const SetupError& e) {
    delete s;
    *out = nullptr;
    fail(err, e.msg);
    return CWG_EVALIDATION;
  } catch (const std::bad_alloc&) {
    delete s;
    *out = nullptr;
    fail(err, "setup: out of host memory");
    return CWG_EVALIDATION;
  }
  *out = s;
  if (err) err->code = CWG_OK;
  return CWG_OK;
}

int cwg_sheet_mesh(double lx, double ly, double h, double frac, uint64_t seed, cwg_sheet** out, cwg_error* err) {
  auto* s = new cwg_sheet();
  try {
    build(*s, lx, ly, h, 0.0, 1.0, 1.0, 1.0, frac, seed, nullptr, false);
  } catch (const SetupError& e) {
    delete s;
    *out = nullptr;
    fail(err, e.msg);
    return CWG_EVALIDATION;
  } catch (const std::bad_alloc&) {
    delete s;
    *out = nullptr;
    fail(err, "setup: out of host memory");
    return CWG_EVALIDATION;
  }
  *out = s;
  if (err) err->code = CWG_OK;
  return CWG_OK;
}

void cwg_sheet_free(cwg_sheet* s) { delete s; }
int64_t cwg_sheet_nodes(const cwg_sheet* s) { return s->n(); }
int64_t cwg_sheet_elements(const cwg_sheet* s) { return s->nx * s->ny; }
int64_t cwg_sheet_nnz(const cwg_sheet* s) { return static_cast<int64_t>(s->val.size()); }
int64_t cwg_sheet_nx1(const cwg_sheet* s) { return s->nx + 1; }
int64_t cwg_sheet_ny1(const cwg_sheet* s) { return s->ny + 1; }
double cwg_sheet_dt_s(const cwg_sheet* s) { return s->dt_s; }
const int64_t* cwg_sheet_row_ptr(const cwg_sheet* s) { return s->row_ptr.data(); }
const int64_t* cwg_sheet_col(const cwg_sheet* s) { return s->col.data(); }
const double* cwg_sheet_val(const cwg_sheet* s) { return s->val.data(); }
const double* cwg_sheet_mass(const cwg_sheet* s) { return s->mass.data(); }
const double* cwg_sheet_coords(const cwg_sheet* s) { return s->xy.data(); }
const int32_t* cwg_sheet_tags(const cwg_sheet* s) { return s->tags.data(); }

// select_nodes (mesh.cpp:124-180)
int64_t cwg_sheet_select(const cwg_sheet* s, int kind, const double* prm, const int64_t* set_nodes, int64_t n_set,
                         int64_t* out, int64_t cap) {
  constexpr double tol = 1e-9;
  std::vector<int64_t> res;
  if (kind == CWG_SEL_NODE_SET) {
    res.assign(set_nodes, set_nodes + n_set);
    for (int64_t i : res)
      if (i < 0 || i >= s->n()) return -1;
    std::sort(res.begin(), res.end());
    res.erase(std::unique(res.begin(), res.end()), res.end());
  } else {
    const double value = prm[0], x0 = prm[1], x1 = prm[2], y0 = prm[3], y1 = prm[4], cx = prm[5], cy = prm[6],
                 rad = prm[7];
    for (int64_t i = 0; i < s->n(); ++i) {
      const double x = s->xy[static_cast<size_t>(2 * i)], y = s->xy[static_cast<size_t>(2 * i + 1)];
      bool in = false;
      switch (kind) {
        case CWG_SEL_X_LE: in = x <= value + tol; break;
        case CWG_SEL_X_GE: in = x >= value - tol; break;
        case CWG_SEL_Y_LE: in = y <= value + tol; break;
        case CWG_SEL_Y_GE: in = y >= value - tol; break;
        case CWG_SEL_RECT: in = x >= x0 - tol && x <= x1 + tol && y >= y0 - tol && y <= y1 + tol; break;
        case CWG_SEL_DISC: {
          const double dx = x - cx, dy = y - cy;
          in = std::sqrt(dx * dx + dy * dy) <= rad + tol;
          break;
        }
        default: return -1;
      }
      if (in) res.push_back(i);
    }
  }
  const int64_t m = static_cast<int64_t>(res.size());
  for (int64_t q = 0; q < m && q < cap; ++q) out[q] = res[static_cast<size_t>(q)];
  return m;
}

// nearest_node (mesh.cpp:43-57)
int64_t cwg_sheet_nearest(const cwg_sheet* s, double x, double y) {
  int64_t best = -1;
  double best_d2 = std::numeric_limits<double>::infinity();
  for (int64_t i = 0; i < s->n(); ++i) {
    const double dx = s->xy[static_cast<size_t>(2 * i)] - x;
    const double dy = s->xy[static_cast<size_t>(2 * i + 1)] - y;
    const double d2 = dx * dx + dy * dy;
    if (d2 < best_d2) {
      best_d2 = d2;
      best = i;
    }
  }
  return best;
}

}  // extern "C"

// ===================================================================== 3D slab
namespace {

// Trilinear hexahedron on the cube [0,h]^3 with a constant 3x3 tensor D:
// 2x2x2 Gauss, local node a = dx + 2*dy + 4*dz (dx, dy, dz in {0, 1}).
// Same evaluation order as oracle/cw_oracle.c:hex_integrals (bit-identical).
void hex_integrals(double h, const double D[3][3], double k[8][8], double m[8]) {
  constexpr double g = 0.57735026918962576;
  const double gp[2] = {-g, g};
  for (int a = 0; a < 8; ++a) {
    m[a] = 0.0;
    for (int b = 0; b < 8; ++b) k[a][b] = 0.0;
  }
  const double det = h * h * h / 8.0;
  const double sc = 2.0 / h;
  for (int q = 0; q < 8; ++q) {
    const double xi = gp[q & 1], eta = gp[(q >> 1) & 1], zeta = gp[q >> 2];
    double n[8], gx[8], gy[8], gz[8];
    for (int a = 0; a < 8; ++a) {
      const double sx = (a & 1) ? 1.0 : -1.0, sy = (a & 2) ? 1.0 : -1.0, sz = (a & 4) ? 1.0 : -1.0;
      const double fx = 1.0 + sx * xi, fy = 1.0 + sy * eta, fz = 1.0 + sz * zeta;
      n[a] = 0.125 * fx * fy * fz;
      gx[a] = sc * (0.125 * sx * fy * fz);
      gy[a] = sc * (0.125 * fx * sy * fz);
      gz[a] = sc * (0.125 * fx * fy * sz);
    }
    for (int a = 0; a < 8; ++a) {
      const double dgx = D[0][0] * gx[a] + D[0][1] * gy[a] + D[0][2] * gz[a];
      const double dgy = D[1][0] * gx[a] + D[1][1] * gy[a] + D[1][2] * gz[a];
      const double dgz = D[2][0] * gx[a] + D[2][1] * gy[a] + D[2][2] * gz[a];
      for (int b = 0; b < 8; ++b) k[a][b] += det * (dgx * gx[b] + dgy * gy[b] + dgz * gz[b]);
      m[a] += det * n[a];
    }
  }
}

// D = d_l f f^T + d_t (I - f f^T), f = (cos th, sin th, 0)
void layer_tensor(double dl, double rho, double th, double D[3][3]) {
  const double f[3] = {std::cos(th), std::sin(th), 0.0};
  const double dt = rho * dl;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const double ff = f[i] * f[j];
      D[i][j] = dl * ff + dt * ((i == j ? 1.0 : 0.0) - ff);
    }
}

}  // namespace

extern "C" double cwg_struct3d_tables(const cwg_struct3d* s, double* coef, double* mass) {
  if (!s || s->nx < 1 || s->ny < 1 || s->nz < 1 || !(s->h > 0.0) || !(s->d_long > 0.0) || !(s->rho > 0.0) ||
      !s->fiber_angle_of_layer)
    return -1.0;
  const int64_t nz = s->nz, nz1 = nz + 1;
  std::vector<std::array<std::array<double, 8>, 8>> K(static_cast<size_t>(nz));
  std::vector<std::array<double, 8>> M(static_cast<size_t>(nz));
  for (int64_t ez = 0; ez < nz; ++ez) {
    double D[3][3], k[8][8], m[8];
    layer_tensor(s->d_long, s->rho, s->fiber_angle_of_layer[ez], D);
    hex_integrals(s->h, D, k, m);
    for (int a = 0; a < 8; ++a) {
      M[ez][a] = m[a];
      for (int b = 0; b < 8; ++b) K[ez][a][b] = k[a][b];
    }
  }
  double min_ratio = std::numeric_limits<double>::infinity();
  for (int by = 0; by < 3; ++by)
    for (int bx = 0; bx < 3; ++bx)
      for (int64_t iz = 0; iz < nz1; ++iz) {
        const int64_t c = (by * 3 + bx) * nz1 + iz;
        double* cf = coef + c * 27;
        for (int q = 0; q < 27; ++q) cf[q] = 0.0;
        double ms = 0.0;
        // representative node of the class: ix/iy = 0 (low), 1 (interior), n (high)
        const int64_t ix = bx == 0 ? 0 : (bx == 1 ? 1 : s->nx), iy = by == 0 ? 0 : (by == 1 ? 1 : s->ny);
        if ((bx == 1 && s->nx < 2) || (by == 1 && s->ny < 2)) continue;  // class does not occur
        // adjacent elements in ascending element index (ey, ez, ex)
        for (int64_t ey = iy - 1; ey <= iy; ++ey) {
          if (ey < 0 || ey >= s->ny) continue;
          for (int64_t ez = iz - 1; ez <= iz; ++ez) {
            if (ez < 0 || ez >= nz) continue;
            for (int64_t ex = ix - 1; ex <= ix; ++ex) {
              if (ex < 0 || ex >= s->nx) continue;
              const int a = static_cast<int>((ix - ex) + 2 * (iy - ey) + 4 * (iz - ez));
              ms += M[ez][a];
              for (int b = 0; b < 8; ++b) {
                const int64_t dx = ex + (b & 1) - ix, dy = ey + ((b >> 1) & 1) - iy, dz = ez + ((b >> 2) & 1) - iz;
                cf[(dy + 1) * 9 + (dz + 1) * 3 + (dx + 1)] += K[ez][a][b];
              }
            }
          }
        }
        mass[c] = ms;
        double den = 0.0;
        for (int q = 0; q < 27; ++q) den += q == 13 ? cf[q] : std::abs(cf[q]);
        if (den > 0.0) min_ratio = std::min(min_ratio, ms / den);
      }
  return std::isfinite(min_ratio) ? 0.9 * min_ratio : -1.0;
}

extern "C" void cwg_uniform_mt64(uint64_t seed, int64_t n, double lo, double hi, double* out) {
  std::mt19937_64 gen(seed);
  const double w = hi - lo;
  for (int64_t i = 0; i < n; ++i) out[i] = lo + w * (static_cast<double>(gen() >> 11) * 0x1.0p-53);
}
