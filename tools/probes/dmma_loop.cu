// Core-loop probe for the trailing DGEMM: 256 threads, 8 warps in 2x4, each a
// 64x32 warp tile = 8x4 DMMA.8x8x4 accumulators.  Variants isolate the loss of
// the real kernel's inner loop:
//   0: fragments from registers (pure issue rate)
//   1: fragments re-loaded from shared memory every k4 block (the real loop)
//   2: as 1, fully unrolled 4-block chunks
//   3: as 1, m16n8k16-style grouping (fragments of 2 k4 blocks loaded together)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_loop dmma_loop.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int V>
__global__ void __launch_bounds__(256, 1) loop(double* out, int iters) {
  __shared__ double sP[4 * 512], sQ[4 * 512];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, wm = warp >> 2, wn = warp & 3;
  for (int i = tid; i < 4 * 512; i += 256) { sP[i] = 1e-3 * i; sQ[i] = 1.0 + 1e-4 * i; }
  __syncthreads();
  double acc[8][4][2];
#pragma unroll
  for (int mi = 0; mi < 8; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  const double* ps = sP + wm * 8 * 32 + lane;
  const double* qs = sQ + wn * 4 * 32 + lane;
  if (V == 0) {
    double a[8], b[4];
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) a[mi] = ps[mi * 32];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = qs[ni * 32];
    for (int it = 0; it < iters * 4; ++it) {
#pragma unroll
      for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
  } else if (V == 1) {
    for (int it = 0; it < iters; ++it) {
      int nb = 4 - (it & 0);  // runtime-bounded like the kernel
      for (int kb = 0; kb < nb; ++kb) {
        double a[8], b[4];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) a[mi] = ps[kb * 512 + mi * 32];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) b[ni] = qs[kb * 512 + ni * 32];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
      }
    }
  } else if (V == 2) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kb = 0; kb < 4; ++kb) {
        double a[8], b[4];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) a[mi] = ps[kb * 512 + mi * 32];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) b[ni] = qs[kb * 512 + ni * 32];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
      }
    }
  } else {
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
      for (int kb = 0; kb < 4; kb += 2) {
        double a[2][8], b[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int mi = 0; mi < 8; ++mi) a[h][mi] = ps[(kb + h) * 512 + mi * 32];
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) b[h][ni] = qs[(kb + h) * 512 + ni * 32];
        }
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) dmma(acc[mi][ni][0], acc[mi][ni][1], a[h][mi], b[h][ni]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int mi = 0; mi < 8; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) s += acc[mi][ni][0] + acc[mi][ni][1];
  if (s == 1234.5) out[0] = s;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  void (*fns[4])(double*, int) = {loop<0>, loop<1>, loop<2>, loop<3>};
  for (int v = 0; v < 4; ++v) {
    fns[v]<<<nsm, 256>>>(out, 10);
    cudaEventRecord(e0);
    fns[v]<<<nsm, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 32 * 4 * (double)iters * 8 * nsm;
    printf("variant %d: %.2f TFLOP/s (%s)\n", v, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
