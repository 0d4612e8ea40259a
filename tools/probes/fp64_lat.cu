// FP64 latency / throughput probe (B200): dependent DFMA chain, independent
// DFMA throughput per SM, the IEEE fp64 division subroutine, redux.sync.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_chain(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int CH>
__global__ void dfma_tput(double* out, long long* cyc, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void ddiv_chain(double* out, long long* cyc, int iters, double d) {
  double x = 1.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x / d + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lds_chain(double* out, long long* cyc, int iters) {
  __shared__ int nxt[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) nxt[i] = (i + 33) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = nxt[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void redux_chain(double* out, long long* cyc, int iters) {
  unsigned v = threadIdx.x * 2654435761u;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __reduce_max_sync(0xffffffffu, v ^ (unsigned)i) + threadIdx.x;
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void sync_chain(double* out, long long* cyc, int iters) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 4096 * sizeof(long long));
  long long h[1024];
  const int it = 1000;
  dfma_chain<<<1, 32>>>(out, cyc, it, 1.0000001, 1e-9);
  dfma_chain<<<1, 32>>>(out, cyc, it, 1.0000001, 1e-9);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cyc\n", h[0] / (16.0 * it));
  for (int warps : {1, 2, 4, 8, 16, 32}) {
    dfma_tput<8><<<1, 32 * warps>>>(out, cyc, it, 1.0000001, 1e-9);
    dfma_tput<8><<<1, 32 * warps>>>(out, cyc, it, 1.0000001, 1e-9);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA throughput, %2d warps x 8 chains: %.2f DFMA/clk/SM\n", warps, 32.0 * warps * 8 * it / h[0]);
  }
  ddiv_chain<<<1, 32>>>(out, cyc, it, 1.37);
  ddiv_chain<<<1, 32>>>(out, cyc, it, 1.37);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DDIV+DADD dependent: %.1f cyc\n", h[0] / (double)it);
  lds_chain<<<1, 32>>>(out, cyc, it);
  lds_chain<<<1, 32>>>(out, cyc, it);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("LDS dependent latency: %.1f cyc\n", h[0] / (double)it);
  redux_chain<<<1, 32>>>(out, cyc, it);
  redux_chain<<<1, 32>>>(out, cyc, it);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("redux.sync dependent: %.1f cyc\n", h[0] / (double)it);
  for (int th : {256, 512, 1024}) {
    sync_chain<<<1, th>>>(out, cyc, it);
    sync_chain<<<1, th>>>(out, cyc, it);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads %4d thr: %.1f cyc\n", th, h[0] / (double)it);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
