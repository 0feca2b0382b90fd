// Host-side declarations of the kernel launchers (defined in the .cu files).
#pragma once

#include <cuda.h>

#include <atomic>
#include <cstdint>

#include "common.cuh"

namespace cwg {

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device property of a
// kernel: set it once per (kernel, device) -- `done` is the kernel's device
// bitmask -- and report the CUDA status instead of dropping it.
template <class K>
inline cudaError_t ensure_dyn_smem(K* kernel, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

cudaError_t launch_react_exact(int kind, const ReactArgs& a, int grid, cudaStream_t st);
int react_exact_threads(int kind);
cudaError_t launch_pace_exact(int kind, const PaceArgs& a, cudaStream_t st);
cudaError_t launch_pace_ord(int kind, const PaceArgs& a, cudaStream_t st);
int react_exact_occupancy(int kind);
cudaError_t launch_rates_exact(int kind, long long n, const double* v, const double* s, const double* ist,
                               double* dv, double* ds, cudaStream_t st);

cudaError_t launch_react_ord(int kind, int variant, const ReactArgs& a, int grid, cudaStream_t st);
int react_ord_threads(int variant);
bool react_ord_variant_valid(int variant);
int react_ord_occupancy(int kind, int variant);
cudaError_t launch_rates_ord(int kind, long long n, const double* v, const double* s, const double* ist, double* dv,
                             double* ds, cudaStream_t st);

cudaError_t launch_diffuse_stencil2d(const DiffArgs& a, const Stencil2D& s, int max_blocks, cudaStream_t st);
cudaError_t launch_diffuse_struct3d(const DiffArgs& a, const Struct3D& s, int max_blocks, cudaStream_t st);
cudaError_t launch_diffuse_stencil2d_tb(int T, const DiffArgs& a, const Stencil2D& s, int num_sms, cudaStream_t st);
void tbm_box(int T, unsigned* cx, unsigned* cy, int* margin);
cudaError_t launch_diffuse_stencil2d_tbm(int T, const DiffArgs& a, const Stencil2D& s, const CUtensorMap& tm,
                                         int num_sms, cudaStream_t st);
cudaError_t launch_pad_planes(const double* src, long long src_pitch, int n_planes, long long w, long long rows,
                              double* dst, long long w_pad, int dst_plane0, cudaStream_t st);
cudaError_t launch_diffuse_csr(const DiffArgs& a, const CsrDev& m, int max_blocks, cudaStream_t st);
cudaError_t launch_push_halo(const DiffArgs& a, cudaStream_t st);
cudaError_t launch_detector_init(const double* v, long long n, long long halo, const DetDev& d, cudaStream_t st);
cudaError_t launch_detector_observe(const double* v, long long n, long long halo, const DetDev& d,
                                    const long long* clock, long long s_off, long long every, double dt,
                                    cudaStream_t st);
cudaError_t launch_record_probes(const double* v, const long long* loc, int np, double* out, const long long* clock,
                                 long long s_off, long long every, cudaStream_t st);
cudaError_t launch_probe_cross(const double* v, long long probe, long long* cross, const long long* clock,
                               long long off, cudaStream_t st);
cudaError_t launch_set_clock(long long* clock, long long value, cudaStream_t st);
cudaError_t launch_tick_clock(long long* clock, long long by, cudaStream_t st);
cudaError_t launch_aos_to_soa(const double* aos, int stride, int ns, long long count, double* soa, long long pitch,
                              long long dst0, cudaStream_t st);
cudaError_t launch_soa_to_aos(const double* soa, long long pitch, long long src0, int ns, long long count,
                              double* aos, int stride, cudaStream_t st);
cudaError_t launch_diffuse_csr_plain(long long n, const long long* rp, const long long* col, const double* val,
                                     const double* mass, const double* v, double dt_sub, double* out,
                                     cudaStream_t st);
cudaError_t launch_fp64_peak(double* out, int blocks, int iters, cudaStream_t st);
cudaError_t launch_init_rest(double* v, double* S, long long pitch, double* last, const int32_t* list,
                              long long first, long long count, const double* rest, int ns, int stride,
                              cudaStream_t st);
// device assembly of a regular sheet (assemble.cu)
struct Sheet2DDev {
  long long nx, ny;                 // element counts
  double h, fx, fy;                 // spacing, fibre direction (cos, sin: computed by the host's libm)
  double d0m, d0f, rho;
  const int32_t* tags;              // [n] device, 1 = fibroblast; null = none
  const double* escale;             // [nx*ny] device; null = 1
};
struct AsmOut {
  double* coef;                     // [9][n] stencil coefficients (slot order = ascending column)
  double* mass;                     // [n] lumped mass
  unsigned char* nnz_row;           // [n] entries per row
  unsigned long long* keys;         // [5] element / structural / Gershgorin failure, max|k| bits, min m/den bits
};
cudaError_t launch_sheet2d_assemble(const Sheet2DDev& g, const AsmOut& o, cudaStream_t st);
cudaError_t launch_sheet2d_slice(const double* coef, const double* mass, long long n, long long w, long long g0,
                                 long long cnt, double* coef_out, double* mass_out, cudaStream_t st);
cudaError_t launch_mass_factor(const double* mass, long long n, double dt_sub, double* cm, cudaStream_t st);
cudaError_t launch_map_values(const double* val, const unsigned char* has, long long n, double* out, cudaStream_t st);
cudaError_t launch_stim_local_ptr(const int32_t* gptr, long long n_own, long long halo, long long n_alloc,
                                  int32_t* ptr, cudaStream_t st);

}  // namespace cwg
