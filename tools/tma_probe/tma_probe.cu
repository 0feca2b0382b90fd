// Standalone check of the TMA sequence used by diffuse_stencil2d_tbm:
// mbarrier init / expect_tx / cp.async.bulk.tensor.3d (zero-filled OOB) / try_wait.parity.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tma_probe tma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int BX = 70, BY = 22, BZ = 10;
__constant__ int cbox[3];

__global__ void probe(const __grid_constant__ CUtensorMap tmap, double* out, int x0, int y0, int mode, int nbox) {
  extern __shared__ __align__(128) double sm[];
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + nbox);
  const unsigned bar_a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a) : "memory");
    if (mode & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (mode & 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (mode & 8) {  // mbarrier only: plain arrive, no copy
      unsigned long long st;
      asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(bar_a) : "memory");
    } else {
    if (mode & 16) {
      unsigned long long st;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;" : "=l"(st) : "r"(bar_a), "r"(nbox * 8) : "memory");
    } else {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a), "r"(nbox * 8) : "memory");
    }
    if (mode & 4)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
          "l"(&tmap), "r"(x0), "r"(y0), "r"(0), "r"(bar_a)
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
          "l"(&tmap), "r"(x0), "r"(y0), "r"(0), "r"(bar_a)
          : "memory");
    }
  }
  unsigned done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(bar_a), "r"(0u)
                 : "memory");
  } while (!done);
  if (!(mode & 8))
    for (int i = threadIdx.x; i < nbox; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 3;
  if (argc > 6) { BX = atoi(argv[4]); BY = atoi(argv[5]); BZ = atoi(argv[6]); }
  const long long w = 1001, rows = 1001, wp = 1002;
  std::vector<double> h(10 * rows * wp);
  for (long long c = 0; c < 10; ++c)
    for (long long y = 0; y < rows; ++y)
      for (long long x = 0; x < wp; ++x) h[(c * rows + y) * wp + x] = c * 1e6 + y * 1e3 + x;
  double *d = nullptr, *out = nullptr;
  cudaMalloc(&d, h.size() * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&out, BX * BY * BZ * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)rows, 10};
  const cuuint64_t strides[2] = {(cuuint64_t)wp * 8, (cuuint64_t)(rows * wp) * 8};
  const cuuint32_t box[3] = {BX, BY, BZ}, es[3] = {1, 1, 1};
  CUresult r = reinterpret_cast<EncodeTiledFn>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es,
                                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode=%d entry=%d\n", (int)r, (int)q);
  const size_t smem = BX * BY * BZ * 8 + 16;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int x0 = argc > 2 ? atoi(argv[2]) : -3, y0 = argc > 3 ? atoi(argv[3]) : -3;
  probe<<<1, 256, smem>>>(tm, out, x0, y0, mode, BX * BY * BZ);
  cudaError_t e = cudaDeviceSynchronize();
  printf("mode %d kernel: %s\n", mode, cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  if (mode & 8) return 0;
  std::vector<double> o(BX * BY * BZ);
  cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int c = 0; c < BZ; ++c)
    for (int y = 0; y < BY; ++y)
      for (int x = 0; x < BX; ++x) {
        const long long gx = x0 + x, gy = y0 + y;
        const double want = (gx >= 0 && gx < w && gy >= 0 && gy < rows) ? c * 1e6 + gy * 1e3 + gx : 0.0;
        if (o[(c * BY + y) * BX + x] != want) ++bad;
      }
  printf("mismatches: %ld\n", bad);
  return bad ? 2 : 0;
}
