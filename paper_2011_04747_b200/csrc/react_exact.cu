// Reaction kernels for the cheap cell models, compiled with --fmad=false so
// every +,-,*,/ rounds exactly like the reference's x86-64 build (no FMA):
// Aliev-Panfilov is bit-identical to the reference (no transcendentals);
// MacCannell differs only through libdevice exp/log vs glibc (tolerance).
#include "react.cuh"

namespace cwg {

// Aliev-Panfilov (aliev_panfilov.cpp:28-38)
struct ModelAP {
  static constexpr int NS = 1;
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 4;
  static constexpr bool kUsesGkr = false;
  static constexpr bool kBlockSync = false;
  __device__ __forceinline__ static void rates(double v, const double* s, double ist, double& dv, double* ds) {
    const double u = (v - (-80.0)) / 100.0;
    const double w = s[0];
    const double du = -8.0 * u * (u - 0.15) * (u - 1.0) - u * w;
    const double eps = 0.002 + 0.2 * w / (u + 0.3);
    const double dw = eps * (-w - 8.0 * u * (u - 0.15 - 1.0));
    dv = (100.0 / 12.9) * du + ist;
    ds[0] = dw / 12.9;
  }
  __device__ __forceinline__ static void advance(double& v, double* s, double ist, double, double h, double& dv) {
    double ds[1];
    rates(v, s, ist, dv, ds);
    v = fe(v, h, dv);
    s[0] = fe(s[0], h, ds[0]);
  }
};

// MacCannell 2007 fibroblast (maccannell_2007.cpp:31-70)
struct ModelMac {
  static constexpr int NS = 2;
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 4;
  static constexpr bool kUsesGkr = false;
  static constexpr bool kBlockSync = false;
  __device__ __forceinline__ static void rates(double v, const double* s, double ist, double& dv, double* ds) {
    const double rtf = 8314.0 * 306.15 / 96485.0;
    const double e_k = rtf * log(5.4 / 129.4349);
    const double e_na = rtf * log(130.0110 / 8.5547);
    const double r_inf = 1.0 / (1.0 + exp(-(v + 20.0) / 11.0));
    const double xr = (v + 20.0) / 25.9;
    const double tau_r = 20.3 + 138.0 * exp(-xr * xr);
    const double s_inf = 1.0 / (1.0 + exp((v + 23.0) / 7.0));
    const double xs = (v + 23.0) / 22.7;
    const double tau_s = 1574.0 + 5268.0 * exp(-xs * xs);
    const double i_kv = 0.25 * s[0] * s[1] * (v - e_k);
    const double vk = v - e_k;
    const double ak1 = 0.1 / (1.0 + exp(0.06 * (vk - 200.0)));
    const double bk1 = (3.0 * exp(0.0002 * (vk + 100.0)) + exp(0.1 * (vk - 10.0))) / (1.0 + exp(-0.5 * vk));
    const double i_k1 = 0.4822 * ak1 / (ak1 + bk1) * vk;
    const double na15 = pow(8.5547, 1.5);
    const double i_nak =
        2.002 * 5.4 / (5.4 + 1.0) * na15 / (na15 + pow(11.0, 1.5)) * (v - (-150.0)) / (v - (-200.0));
    const double i_bna = 0.0095 * (v - e_na);
    dv = -(i_kv + i_k1 + i_nak + i_bna) + ist;
    ds[0] = (r_inf - s[0]) / tau_r;
    ds[1] = (s_inf - s[1]) / tau_s;
  }
  __device__ __forceinline__ static void advance(double& v, double* s, double ist, double, double h, double& dv) {
    double ds[2];
    rates(v, s, ist, dv, ds);
    v = fe(v, h, dv);
    s[0] = fe(s[0], h, ds[0]);
    s[1] = fe(s[1], h, ds[1]);
  }
};

// Passive non-excitable membrane (EXTENSION for BASELINE config 3's scar):
// dV/dt = -g (V - E) + i_stim, g = 0.01 /ms, E = -85 mV, no states.
struct ModelPassive {
  static constexpr int NS = 0;
  static constexpr int kThreads = 256;
  static constexpr int kMinBlocks = 4;
  static constexpr bool kUsesGkr = false;
  static constexpr bool kBlockSync = false;
  __device__ __forceinline__ static void rates(double v, const double*, double ist, double& dv, double*) {
    dv = -0.01 * (v - (-85.0)) + ist;
  }
  __device__ __forceinline__ static void advance(double& v, double* s, double ist, double, double h, double& dv) {
    rates(v, s, ist, dv, nullptr);
    v = fe(v, h, dv);
  }
};

template <class M>
__global__ void rates_batch_kernel(long long n, const double* v, const double* s, const double* ist, double* dv,
                                   double* ds) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  double sl[M::NS > 0 ? M::NS : 1], dl[M::NS > 0 ? M::NS : 1];
  for (int q = 0; q < M::NS; ++q) sl[q] = s[i * M::NS + q];
  double d;
  M::rates(v[i], sl, ist[i], d, dl);
  dv[i] = d;
  for (int q = 0; q < M::NS; ++q) ds[i * M::NS + q] = dl[q];
}

}  // namespace cwg

// ---- host-visible launch helpers
namespace cwg {

template <class M>
static cudaError_t launch_react_t(const ReactArgs& a, int grid, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(a.khist_len) * sizeof(unsigned);
  react_kernel<M><<<grid, M::kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <class M>
static int occupancy_t() {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, react_kernel<M>, M::kThreads, 2048 * sizeof(unsigned));
  return b;
}

cudaError_t launch_react_exact(int kind, const ReactArgs& a, int grid, cudaStream_t st) {
  switch (kind) {
    case 0: return launch_react_t<ModelAP>(a, grid, st);
    case 4: return launch_react_t<ModelMac>(a, grid, st);
    case 5: return launch_react_t<ModelPassive>(a, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_pace_exact(int kind, const PaceArgs& a, cudaStream_t st) {
  switch (kind) {
    case 0: return launch_pace_t<ModelAP>(a, st);
    case 4: return launch_pace_t<ModelMac>(a, st);
    case 5: return launch_pace_t<ModelPassive>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

int react_exact_threads(int) { return 256; }

int react_exact_occupancy(int kind) {
  switch (kind) {
    case 0: return occupancy_t<ModelAP>();
    case 4: return occupancy_t<ModelMac>();
    case 5: return occupancy_t<ModelPassive>();
    default: return 0;
  }
}

cudaError_t launch_rates_exact(int kind, long long n, const double* v, const double* s, const double* ist,
                               double* dv, double* ds, cudaStream_t st) {
  const int grid = static_cast<int>((n + 255) / 256);
  if (n == 0) return cudaSuccess;
  switch (kind) {
    case 0: rates_batch_kernel<ModelAP><<<grid, 256, 0, st>>>(n, v, s, ist, dv, ds); break;
    case 4: rates_batch_kernel<ModelMac><<<grid, 256, 0, st>>>(n, v, s, ist, dv, ds); break;
    case 5: rates_batch_kernel<ModelPassive><<<grid, 256, 0, st>>>(n, v, s, ist, dv, ds); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace cwg
