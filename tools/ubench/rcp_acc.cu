// Accuracy of the short reciprocal (MUFU.RCP64H seed + one cubic Newton step,
// 3 DFMA) against the correctly rounded 1/x, over log-uniform x in
// [2^-40, 2^40] of both signs, plus the seed's own relative error.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rcp_acc rcp_acc.cu && ./rcp_acc
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcp3(double x, double* seed_err) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  *seed_err = fabs(e);
  e = fma(e, e, e);
  return fma(y, e, y);
}

__global__ void k(long long n, unsigned long long seed, unsigned long long* ulp_hist, double* max_seed) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  const double u = (z >> 11) * (1.0 / 9007199254740992.0);
  double x = exp2(-40.0 + 80.0 * u);
  if (z & 1) x = -x;
  double se;
  const double a = rcp3(x, &se);
  const double r = __drcp_rn(x);
  const long long d = llabs(__double_as_longlong(a) - __double_as_longlong(r));
  atomicAdd(ulp_hist + (d > 7 ? 7 : d), 1ull);
  // max of a non-negative double via its bit pattern
  atomicMax(reinterpret_cast<unsigned long long*>(max_seed), (unsigned long long)__double_as_longlong(se));
}

int main() {
  unsigned long long* h;
  double* m;
  cudaMalloc(&h, 8 * 8);
  cudaMalloc(&m, 8);
  cudaMemset(h, 0, 64);
  cudaMemset(m, 0, 8);
  const long long n = 1ll << 28;
  k<<<(unsigned)((n + 255) / 256), 256>>>(n, 12345, h, m);
  unsigned long long hh[8];
  double mm;
  cudaMemcpy(hh, h, 64, cudaMemcpyDeviceToHost);
  cudaMemcpy(&mm, m, 8, cudaMemcpyDeviceToHost);
  printf("rcp3 vs correctly rounded 1/x over %lld samples (|x| in [2^-40, 2^40]):\n", n);
  for (int i = 0; i < 8; ++i) printf("  %s%d ulp: %llu\n", i == 7 ? ">=" : "", i, hh[i]);
  printf("  max |1 - x*seed| = %.3e (2^%.1f)\n", mm, std::log2(mm));
  return cudaGetLastError() != cudaSuccess;
}
