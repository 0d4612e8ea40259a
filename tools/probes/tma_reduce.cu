// Checks cp.reduce.async.bulk.tensor .add on an FP64 tensor map with 128-byte
// swizzle (box 16 rows x 32 cols of a column-major matrix), and the fragment ->
// swizzled-smem mapping the trailing DGEMM epilogue uses.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_reduce tma_reduce.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <cstdint>

__global__ void k(const __grid_constant__ CUtensorMap tmap, int row0, int col0) {
  __shared__ __align__(1024) double buf[4][32 * 16];  // 4 boxes of 16 rows x 32 cols
  const int lane = threadIdx.x;
  // the warp's 64x32 "accumulator": value = 1000*row + col (local coords)
  for (int mi = 0; mi < 8; ++mi)
    for (int ni = 0; ni < 4; ++ni)
      for (int e = 0; e < 2; ++e) {
        const int row = mi * 8 + (lane >> 2), col = ni * 8 + 2 * (lane & 3) + e;
        const int box = mi >> 1, rin = row & 15;
        const int chunk = (rin >> 1) ^ (col & 7);
        double* p = &buf[box][0] + col * 16 + chunk * 2 + (rin & 1);
        *p = 1000.0 * row + col;
      }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    for (int b = 0; b < 4; ++b) {
      asm volatile(
          "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tmap),
          "r"(row0 + 16 * b), "r"(col0), "r"((unsigned)__cvta_generic_to_shared(&buf[b][0]))
          : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const int n = 200, ld = 202;
  std::vector<double> h((size_t)ld * n, 1.0);
  double* d;
  cudaMalloc(&d, h.size() * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no entry point\n"); return 1; }
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {16, 32}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  const int row0 = 160, col0 = 100;  // rows 160..223 clip at 200
  k<<<1, 32>>>(tm, row0, col0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
  int bad = 0, changed = 0;
  for (int c = 0; c < n; ++c)
    for (int rr = 0; rr < ld; ++rr) {
      double want = 1.0;
      if (rr < n && rr >= row0 && rr < row0 + 64 && c >= col0 && c < col0 + 32) want += 1000.0 * (rr - row0) + (c - col0);
      double got = h[(size_t)c * ld + rr];
      if (got != 1.0) ++changed;
      if (got != want) { if (bad++ < 5) printf("mismatch r=%d c=%d got %g want %g\n", rr, c, got, want); }
    }
  printf("bad=%d changed=%d (expect %d)\n", bad, changed, 40 * 32);
  return 0;
}
