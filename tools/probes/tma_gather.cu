// Checks the two gather boxes of the lean panel: a G x 1 box (column part) and a 2 x G box
// (row part) of a column-major fp64 matrix, loaded with cp.async.bulk.tensor.2d into shared
// memory (cluster launch of CS CTAs like the panel), at arbitrary start coordinates.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_gather tma_gather.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap tmc, const __grid_constant__ CUtensorMap tmr, int G, int rbase0,
                  int pb, double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  double* gcol = (double*)smem;
  double* grow = (double*)(smem + ((8 * G + 127) & ~127));
  uint64_t* bar = (uint64_t*)(smem + ((8 * G + 127) & ~127) + ((16 * G + 127) & ~127));
  const int rbase = rbase0 + blockIdx.x * G;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 64) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(24u * G) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                     "r"(su32(gcol)), "l"((uint64_t)&tmc), "r"(rbase), "r"(pb), "r"(su32(bar)) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                     "r"(su32(grow)), "l"((uint64_t)&tmr), "r"(pb), "r"(rbase), "r"(su32(bar)) : "memory");
  }
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(su32(bar)) : "memory");
  for (int i = threadIdx.x; i < G; i += blockDim.x) {
    out[(size_t)blockIdx.x * 2 * G + i] = gcol[i];
    out[(size_t)blockIdx.x * 2 * G + G + i] = grow[2 * i];
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 4096, G = argc > 2 ? atoi(argv[2]) : 256, CS = argc > 3 ? atoi(argv[3]) : 16;
  const int pb = argc > 4 ? atoi(argv[4]) : 1001, rbase0 = argc > 5 ? atoi(argv[5]) : 3;
  const long long ld = n;
  std::vector<double> h((size_t)n * ld);
  for (long long j = 0; j < n; ++j)
    for (long long i = 0; i < n; ++i) h[j * ld + i] = 10000.0 * i + j;
  double *d, *out;
  cudaMalloc(&d, h.size() * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&out, (size_t)CS * 2 * G * 8);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap tmc, tmr;
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t es[2] = {1, 1};
  cuuint32_t bc[2] = {(cuuint32_t)G, 1}, br[2] = {2, (cuuint32_t)G};
  int r1 = enc(&tmc, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, bc, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int r2 = enc(&tmr, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, br, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: col %d row %d\n", r1, r2);
  const size_t smem = ((8 * G + 127) & ~127) + ((16 * G + 127) & ~127) + 64;
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = CS; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
  cfg.attrs = &attr; cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, tmc, tmr, G, rbase0, pb, out);
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("launch %s sync %s\n", cudaGetErrorString(e), cudaGetErrorString(e2));
  std::vector<double> o((size_t)CS * 2 * G);
  cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
  long long bad = 0;
  for (int c = 0; c < CS; ++c)
    for (int i = 0; i < G; ++i) {
      const long long row = rbase0 + (long long)c * G + i;
      const double ec = row < n ? 10000.0 * row + pb : 0.0;       // W(row, pb)
      const double er = row < n ? 10000.0 * pb + row : 0.0;       // W(pb, row)
      bad += o[(size_t)c * 2 * G + i] != ec;
      bad += o[(size_t)c * 2 * G + G + i] != er;
    }
  printf("n=%d G=%d CS=%d pb=%d rbase0=%d: mismatches %lld\n", n, G, CS, pb, rbase0, bad);
  return 0;
}
