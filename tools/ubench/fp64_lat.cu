// FP64 latency / throughput microbenchmark on sm_100a (clock64 around dependent chains).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_lat fp64_lat.cu && ./fp64_lat
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, long long* cyc, double a, double b, int iters) {
  double x = threadIdx.x * 1e-3 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (OP == 0) x = __dadd_rn(x, a);
      if (OP == 1) x = __dmul_rn(x, a);
      if (OP == 2) x = fma(x, a, b);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (x == 1.2345) out[0] = x;
}

// throughput: NC independent chains per thread, W warps per SM (one block per SM)
template <int NC>
__global__ void tput(double* out, long long* cyc, double a, int iters) {
  double x[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) x[c] = threadIdx.x * 1e-3 + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int c = 0; c < NC; ++c) x[c] = __dadd_rn(x[c], a);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) s += x[c];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8 * 1024);
  long long h[1024];
  const int iters = 1000;
  const char* names[3] = {"DADD", "DMUL", "DFMA"};
  for (int op = 0; op < 3; ++op) {
    if (op == 0) chain<0><<<1, 32>>>(out, cyc, 1e-9, 1e-9, iters);
    if (op == 1) chain<1><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, iters);
    if (op == 2) chain<2><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, iters);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%s dependent latency: %.2f cycles\n", names[op], double(h[0]) / (iters * 16.0));
  }
  for (int warps = 1; warps <= 16; warps *= 2) {
    for (int nc = 1; nc <= 8; nc *= 2) {
      const int T = 32 * warps;
      if (nc == 1) tput<1><<<1, T>>>(out, cyc, 1e-9, iters);
      if (nc == 2) tput<2><<<1, T>>>(out, cyc, 1e-9, iters);
      if (nc == 4) tput<4><<<1, T>>>(out, cyc, 1e-9, iters);
      if (nc == 8) tput<8><<<1, T>>>(out, cyc, 1e-9, iters);
      cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
      const double ops = double(iters) * 8 * nc * warps;  // warp-instructions per SM
      printf("warps/SM %2d chains/thread %d: %.3f DADD warp-instr per cycle per SM (%.1f%% of 2/cycle)\n", warps, nc,
             ops / h[0], 100.0 * ops / h[0] / 2.0);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
