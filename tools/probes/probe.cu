// Hardware probes for the FP64 pipe and grid-wide exchange latency on B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[2 * i]), "+d"(acc[2 * i + 1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma16_loop(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[4 * i]), "+d"(acc[4 * i + 1]), "+d"(acc[4 * i + 2]), "+d"(acc[4 * i + 3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double acc[16];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

// LL-style exchange: every CTA publishes (flag|payload) 8-byte words, then one warp polls all slots.
__global__ void exchange_loop(unsigned long long* slots, int nslots_pad, int rounds, long long* cyc) {
  int P = gridDim.x;
  long long t0 = clock64();
  __shared__ int done;
  for (int r = 1; r <= rounds; ++r) {
    int par = r & 1;
    if (threadIdx.x == 0) {
      unsigned long long w = ((unsigned long long)r << 32) | (unsigned)blockIdx.x;
      asm volatile("st.volatile.global.u64 [%0], %1;" :: "l"(slots + par * nslots_pad + blockIdx.x), "l"(w) : "memory");
    }
    if (threadIdx.x < 32) {
      for (int s = threadIdx.x; s < P; s += 32) {
        unsigned long long w;
        do {
          asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(w) : "l"(slots + par * nslots_pad + s) : "memory");
        } while ((unsigned)(w >> 32) != (unsigned)r);
      }
      __syncwarp();
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// Same but with a second dependent round trip (read a "winner row" of 130 doubles published by CTA r%P).
__global__ void exchange2_loop(unsigned long long* slots, int nslots_pad, unsigned long long* rows, int rounds) {
  int P = gridDim.x;
  for (int r = 1; r <= rounds; ++r) {
    int par = r & 1;
    int owner = r % P;
    if (blockIdx.x == owner && threadIdx.x < 130) {
      unsigned long long w = ((unsigned long long)r << 32) | (unsigned)threadIdx.x;
      asm volatile("st.volatile.global.u64 [%0], %1;" :: "l"(rows + par * 256 + threadIdx.x), "l"(w) : "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long w = ((unsigned long long)r << 32) | (unsigned)blockIdx.x;
      asm volatile("st.volatile.global.u64 [%0], %1;" :: "l"(slots + par * nslots_pad + blockIdx.x), "l"(w) : "memory");
    }
    if (threadIdx.x < 32) {
      for (int s = threadIdx.x; s < P; s += 32) {
        unsigned long long w;
        do {
          asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(w) : "l"(slots + par * nslots_pad + s) : "memory");
        } while ((unsigned)(w >> 32) != (unsigned)r);
      }
    }
    __syncthreads();
    if (threadIdx.x < 130) {
      unsigned long long w;
      do {
        asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(w) : "l"(rows + par * 256 + threadIdx.x) : "memory");
      } while ((unsigned)(w >> 32) != (unsigned)r);
    }
    __syncthreads();
  }
}

// dependent global load latency (pointer chase in HBM-sized buffer)
__global__ void chase(const unsigned long long* buf, int steps, unsigned long long* out, long long* cyc) {
  unsigned long long p = 0;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = buf[p];
  long long t1 = clock64();
  out[0] = p;
  cyc[0] = t1 - t0;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int nsm = prop.multiProcessorCount;
  printf("device %s sms=%d clock(kHz)=%d\n", prop.name, nsm, prop.clockRate);
  double* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  int iters = 20000;
  for (int bpsm = 1; bpsm <= 4; bpsm *= 2) {
    for (int threads = 128; threads <= 512; threads *= 2) {
      dim3 g(nsm * bpsm);
      dmma_loop<<<g, threads>>>(out, 100);
      cudaEventRecord(e0);
      dmma_loop<<<g, threads>>>(out, iters);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * (double)iters * (threads / 32) * g.x;
      printf("DMMA m8n8k4  blocks/sm=%d threads=%d : %.2f TFLOP/s\n", bpsm, threads, flops / ms / 1e9);
      dmma16_loop<<<g, threads>>>(out, 100);
      cudaEventRecord(e0);
      dmma16_loop<<<g, threads>>>(out, iters / 4);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 16 * 8 * 16 * 4 * (double)(iters / 4) * (threads / 32) * g.x;
      printf("DMMA m16n8k16 blocks/sm=%d threads=%d : %.2f TFLOP/s\n", bpsm, threads, flops / ms / 1e9);
      dfma_loop<<<g, threads>>>(out, 100);
      cudaEventRecord(e0);
      dfma_loop<<<g, threads>>>(out, iters);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 16 * (double)iters * threads * g.x;
      printf("DFMA         blocks/sm=%d threads=%d : %.2f TFLOP/s\n", bpsm, threads, flops / ms / 1e9);
    }
  }
  // exchange latency
  unsigned long long* slots;
  unsigned long long* rows;
  long long* cyc;
  CK(cudaMalloc(&slots, 2 * 256 * 8));
  CK(cudaMalloc(&rows, 2 * 256 * 8));
  CK(cudaMalloc(&cyc, 1024 * 8));
  for (int P : {8, 16, 32, 64, 128, nsm}) {
    CK(cudaMemset(slots, 0, 2 * 256 * 8));
    int rounds = 2000;
    void* args[] = {&slots, (void*)new int(256), &rounds, &cyc};
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)exchange_loop, P, 256, args, 0, 0));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("LL exchange P=%d : %.3f us/round\n", P, ms * 1e3 / rounds);
    CK(cudaMemset(slots, 0, 2 * 256 * 8));
    CK(cudaMemset(rows, 0, 2 * 256 * 8));
    void* args2[] = {&slots, (void*)new int(256), &rows, &rounds};
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)exchange2_loop, P, 256, args2, 0, 0));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("LL exchange+row P=%d : %.3f us/round\n", P, ms * 1e3 / rounds);
  }
  // pointer chase latency: L2-resident (4MB) and HBM (1GB)
  for (size_t bytes : {(size_t)4 << 20, (size_t)1 << 30}) {
    size_t n = bytes / 8;
    unsigned long long* h = (unsigned long long*)malloc(bytes);
    size_t stride = 4097 * 16 + 3;  // large odd stride in elements
    for (size_t i = 0; i < n; ++i) h[i] = (i + stride) % n;
    unsigned long long* d;
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
    unsigned long long* o;
    CK(cudaMalloc(&o, 8));
    chase<<<1, 1>>>(d, 1000, o, cyc);
    chase<<<1, 1>>>(d, 10000, o, cyc);
    long long c;
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf("chase %zu MB: %.1f cycles/load\n", bytes >> 20, c / 10000.0);
    cudaFree(d);
    free(h);
  }
  return 0;
}
