/*
 * cwgpu_setup.h -- host-side problem setup for benches and tests (C ABI).
 *
 * Restates the reference's setup path so that the GPU box can build the
 * operators of BASELINE.json's configurations without the reference tree:
 *   build_regular_sheet   mesh.cpp:72-98   (node numbering y-outer, x-inner)
 *   assign_fibrosis       mesh.cpp:100-122 (Fisher-Yates over mt19937_64)
 *   select_nodes          mesh.cpp:124-180 (1e-9 cm inclusive tolerance)
 *   nearest_node          mesh.cpp:43-57
 *   build_diffusion_field fem.cpp:21-51
 *   assemble              fem.cpp:63-176   (bilinear quad, 2x2 Gauss, row-sum lumping,
 *                                           triplet std::sort, CSR with ascending columns)
 *   gershgorin_step       fem.cpp:178-192
 * The 2D CSR is bit-identical to the reference's (tests/test_setup_parity.py).
 * Extension (config 3, parity unpinned by the reference): an optional
 * per-element conductivity scale (0 allowed: scar) with zero rows skipped by
 * Gershgorin.
 */
#ifndef CWGPU_SETUP_H
#define CWGPU_SETUP_H

#include <stdint.h>

#include "cwgpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cwg_sheet cwg_sheet;

/* RegionSelector kinds in reference declaration order (mesh.hpp:50-58) */
enum {
  CWG_SEL_X_LE = 0, CWG_SEL_X_GE = 1, CWG_SEL_Y_LE = 2, CWG_SEL_Y_GE = 3,
  CWG_SEL_RECT = 4, CWG_SEL_NODE_SET = 5, CWG_SEL_DISC = 6
};

/* build_regular_sheet (mesh.cpp:72-98) + assign_fibrosis (mesh.cpp:100-122,
 * fib_fraction > 0) + build_diffusion_field (fem.cpp:21-51) + assemble
 * (fem.cpp:63-176). elem_scale: optional [n_elements] multiplier of D
 * (extension). cwg_sheet_free releases it. */
int cwg_sheet_build(double lx_cm, double ly_cm, double h_cm, double fiber_angle_rad,
                    double d0_myocyte, double d0_fibrotic, double rho, double fib_fraction,
                    uint64_t seed, const double* elem_scale, cwg_sheet** out, cwg_error* err);
void cwg_sheet_free(cwg_sheet* s);
/* build_regular_sheet + assign_fibrosis only (mesh.cpp:72-122): coordinates
 * and tags for select / nearest, no host assembly -- the operator is then
 * assembled on the device (cwg_sheet2d, CWG_OP_SHEET2D in cwgpu.h). The
 * operator views below are empty (nnz 0, dt_s 0) for such a sheet. */
int cwg_sheet_mesh(double lx_cm, double ly_cm, double h_cm, double fib_fraction, uint64_t seed, cwg_sheet** out,
                   cwg_error* err);

/* Mesh::node_count / element_count (mesh.hpp), AssembledOperator nnz /
 * rows / dt_s (fem.hpp:23-32), grid node counts of build_regular_sheet */
int64_t cwg_sheet_nodes(const cwg_sheet* s);
int64_t cwg_sheet_elements(const cwg_sheet* s);
int64_t cwg_sheet_nnz(const cwg_sheet* s);
int64_t cwg_sheet_nx1(const cwg_sheet* s);
int64_t cwg_sheet_ny1(const cwg_sheet* s);
double cwg_sheet_dt_s(const cwg_sheet* s);
/* zero-copy views valid for the sheet's lifetime: AssembledOperator row_ptr /
 * col / val / lumped_mass (fem.hpp:23-32), Mesh::node_coords and node tags
 * (mesh.hpp) */
const int64_t* cwg_sheet_row_ptr(const cwg_sheet* s);
const int64_t* cwg_sheet_col(const cwg_sheet* s);
const double* cwg_sheet_val(const cwg_sheet* s);
const double* cwg_sheet_mass(const cwg_sheet* s);
const double* cwg_sheet_coords(const cwg_sheet* s); /* [n][2] */
const int32_t* cwg_sheet_tags(const cwg_sheet* s);  /* per node; 0 myocyte-epi, 1 fibroblast */

/* select_nodes (mesh.cpp:124-180); prm = {value, x0, x1, y0, y1, cx, cy,
 * radius}; returns count (writes <= cap) */
int64_t cwg_sheet_select(const cwg_sheet* s, int kind, const double* prm, const int64_t* set_nodes,
                         int64_t n_set, int64_t* out, int64_t cap);
int64_t cwg_sheet_nearest(const cwg_sheet* s, double x, double y); /* Mesh::nearest_node (mesh.cpp:43-57) */

/* ---- 3D slab (EXTENSION for BASELINE configs 4-5; parity pinned to the C
 * oracle's independent CSR assembly, oracle/cw_oracle.c cwo_assemble_slab3d).
 * Structured operator of cwg_struct3d (cwgpu.h): node (ix, iy, iz) has index
 * (iy*(nz+1) + iz)*(nx+1) + ix; hex element (ex, ey, ez) has index
 * (ey*nz + ez)*nx + ex and layer ez's fibre angle. Element integrals on the
 * cube [0,h]^3: trilinear shape functions, 2x2x2 Gauss, row-sum lumped mass
 * (the 3D analogue of fem.cpp:63-108). A row's coefficients depend only on the
 * node class c = (by*3 + bx)*(nz+1) + iz with bx/by = 0 (low face), 1
 * (interior), 2 (high face); each coefficient sums its element contributions
 * in ascending element index, exactly as a CSR assembly would.
 *   coef[c*27 + (dy+1)*9 + (dz+1)*3 + (dx+1)]  (0 where the neighbour is absent)
 *   mass[c]
 * n_classes = 9*(nz+1). Returns dt_s (Gershgorin, fem.cpp:178-192) or < 0. */
double cwg_struct3d_tables(const cwg_struct3d* s, double* coef, double* mass);

/* Seeded uniform draws for the synthetic configurations (EXTENSION; the
 * reference's RNG, std::mt19937_64 as in assign_fibrosis mesh.cpp:112):
 * out[i] = lo + (hi - lo) * ((x_i >> 11) * 2^-53) with x_i the i-th output
 * of std::mt19937_64(seed). Used for C3's per-node GKr jitter and C5's
 * stimulus sites; restated in the oracle (cwo_uniform_mt64). */
void cwg_uniform_mt64(uint64_t seed, int64_t n, double lo, double hi, double* out);

#ifdef __cplusplus
}
#endif
#endif
