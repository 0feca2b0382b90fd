/* TEST INFRASTRUCTURE ONLY -- the CPU restatement oracle.
 *
 * Plain C11 restatement of the reference's hot-path algorithm (cardwave,
 * /root/reference/proj/core). Used by tests/ (and __graft_entry__.smoke) as
 * the CHECKER for the CUDA path; never linked into or called by the product.
 * Pinned against the reference itself (oracle/_ref/libcwref.so) by
 * tests/test_oracle_pins.py, which requires bit-identical results for every
 * function below on the reference's own configurations.
 *
 * Extensions beyond the reference (3D sheets, zero-conductivity scar, GKr
 * jitter, the passive model) follow the reference conventions and are marked
 * "parity unpinned" where they are used.
 */
#ifndef CW_ORACLE_H
#define CW_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* model kinds (same ids as include/cwgpu.h) */
enum { CWO_AP = 0, CWO_ORD_ENDO = 1, CWO_ORD_EPI = 2, CWO_ORD_MID = 3, CWO_MAC = 4, CWO_PASSIVE = 5 };
enum { CWO_OST = 0, CWO_OSTAR = 1, CWO_DAETI = 2 };

int cwo_state_count(int kind);
double cwo_stable_step(int kind);
/* [V, s...] */
void cwo_rest_state(int kind, double* out);

/* One rates() evaluation (ionic.hpp:33). gkr_scale multiplies ORd GKr (1.0 = reference). */
void cwo_rates(int kind, double v, const double* s, double i_stim, double gkr_scale, double* dv,
               double* ds);
void cwo_rates_batch(int kind, int64_t n, const double* v, const double* s, const double* i_stim,
                     double* dv, double* ds);

int cwo_pace(int kind, double cycle_ms, int n_beats, double amp, double dur, double* state_out,
             double* apd_out, double* max_rel, int* fail_beat, double* fail_t);
int cwo_reaction_substeps(double dvdt_prev, int scheme, int k0_up, int k0_down, int k_max);
int cwo_diffusion_substeps(double dt, double dt_s, int strict, int scheme, int* l, double* dt_ad);
int cwo_k_max_for(double dt, double stable_step);

/* stimulus: flattened per-node entry lists */
typedef struct {
  const int32_t* node_ptr; /* n+1 */
  const int32_t* ids;      /* entry ids */
  const double* t_start;
  const double* duration;
  const double* amplitude;
  const double* period; /* NaN: single shot */
} cwo_protocol;

double cwo_stim_current(const cwo_protocol* p, int64_t node, double t);

void cwo_diffusion_substep_csr(int64_t n, const int64_t* row_ptr, const int64_t* col,
                               const double* val, const double* mass, const double* v,
                               double dt_sub, double* out);

/* One reaction pass (splitting.cpp:95-155). AoS states s[i*stride+q].
 * model_kind[m] for model id m, k_max[m]; gkr_scale may be NULL.
 * khist (len kmax_global+1) accumulated. Returns -1 or the lowest bad node;
 * *bad_t receives its sub-step time. */
int64_t cwo_reaction_step(int64_t n, int stride, double* v, double* s, double* last_dvdt,
                          const uint8_t* model_of_node, const int* model_kind, const int* k_max,
                          const double* gkr_scale, const cwo_protocol* prot, int scheme, int k0_up,
                          int k0_down, double dt, double t, int64_t* khist, double* bad_t);

/* Activation detector (postprocess.cpp:18-66), SoA node state. */
typedef struct {
  int64_t n;
  double threshold;
  double prev_t;
  int first;
  double *prev_v, *v_rest, *max_slope, *t_max_slope, *v_peak, *lat, *apd;
  uint8_t *phase, *has_lat, *has_apd;
} cwo_detector;

void cwo_detector_init(cwo_detector* d, int64_t n, double threshold);
void cwo_detector_free(cwo_detector* d);
void cwo_detector_observe(cwo_detector* d, double t, const double* v);

/* 3D slab operator (EXTENSION, BASELINE configs 4-5): CSR assembly of the
 * trilinear-hex / 2x2x2-Gauss / row-sum-lumped operator on an (nx, ny, nz)
 * element grid of spacing h, node index (iy*(nz+1)+iz)*(nx+1)+ix, element
 * index (ey*nz+ez)*nx+ex, fibre angle per element layer. Contributions are
 * accumulated per (row, column) in ascending element index; columns ascend.
 * Caller frees the arrays with free(). Returns dt_s (Gershgorin) or < 0. */
double cwo_assemble_slab3d(int64_t nx, int64_t ny, int64_t nz, double h, double d_long, double rho,
                           const double* angle_of_layer, int64_t** row_ptr, int64_t** col, double** val,
                           double** mass);
void cwo_free(void* p);

/* OpenMP variant of cwo_reaction_step (same results for any thread count). */
int64_t cwo_reaction_step_omp(int64_t n, int stride, double* v, double* s, double* last_dvdt,
                              const uint8_t* model_of_node, const int* model_kind, const int* k_max,
                              const double* gkr_scale, const cwo_protocol* prot, int scheme, int k0_up,
                              int k0_down, double dt, double t, int64_t* khist, int khist_len, double* bad_t);

/* Slab node-class tables (coef[9*(nz+1)][27], mass[9*(nz+1)]) from a small CSR assembly; returns dt_s. */
double cwo_slab3d_classes(int64_t nz, double h, double d_long, double rho, const double* angle_of_layer,
                          double* coef, double* mass);
/* Structured slab diffusion sub-step over those tables (OpenMP). */
void cwo_diffusion_substep_slab3d(int64_t nx1, int64_t ny1, int64_t nz1, const double* coef, const double* mass,
                                  const double* v, double dt_sub, double* out);

/* MT19937-64 (std::mt19937_64): raw outputs and uniform draws lo + (hi-lo)*((x >> 11) * 2^-53). */
void cwo_mt64_raw(uint64_t seed, int64_t n, uint64_t* out);
void cwo_uniform_mt64(uint64_t seed, int64_t n, double lo, double hi, double* out);

#ifdef __cplusplus
}
#endif
#endif
