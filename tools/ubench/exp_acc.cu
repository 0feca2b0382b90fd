// Accuracy of fastmath.cuh's table exp (fexp_nc: 2048-entry table, degree-3 polynomial, one reduction
// word) against libdevice's exp, in ulps of the libdevice result (itself within 1 ulp of the exact value).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I../../paper_2011_04747_b200/csrc \
//        -o exp_acc exp_acc.cu && ./exp_acc
#include <cstdio>
#include "fastmath.cuh"

__global__ void k(long long n, double lo, double hi, unsigned long long* h_exp) {
  cwg::exp_table_init();
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double x = lo + (hi - lo) * (static_cast<double>(i) / static_cast<double>(n - 1));
    const double c = cwg::fexp_nc(x), e = exp(x);
    const long long d2 = llabs(__double_as_longlong(c) - __double_as_longlong(e));
    atomicAdd(h_exp + (d2 > 7 ? 7 : d2), 1ull);
  }
}

int main() {
  unsigned long long *h;
  cudaMalloc(&h, 16 * 8);
  const double ranges[4][2] = {{-5.0, 5.0}, {-50.0, 50.0}, {-1e-3, 1e-3}, {-700.0, 700.0}};
  for (auto& r : ranges) {
    cudaMemset(h, 0, 128);
    const long long n = 1ll << 26;
    k<<<1184, 256>>>(n, r[0], r[1], h + 8);
    unsigned long long hh[16];
    cudaMemcpy(hh, h, 128, cudaMemcpyDeviceToHost);
    printf("x in [%g, %g], %lld points: ulps vs libdevice exp:", r[0], r[1], n);
    for (int i = 0; i < 8; ++i) printf(" %s%d:%llu", i == 7 ? ">=" : "", i, hh[8 + i]);
    printf("\n");
  }
  return cudaGetLastError() != cudaSuccess;
}
