// Microbenchmark of candidate-exchange patterns for the pivoted panel step.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exchange exchange.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("CUDA %s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));      \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

template <bool kSys>
__device__ __forceinline__ void st2(uint64_t* p, uint64_t a, uint64_t b) {
  if (kSys)
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
  else
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
template <bool kSys>
__device__ __forceinline__ void ld2(const uint64_t* p, uint64_t& a, uint64_t& b) {
  if (kSys)
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  else
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// mode bits: 1 = publish+fetch a 130-double row; 2 = warp-0 polls all (else one thread per slot)
template <bool kSys>
__global__ void xchg(uint64_t* recs, uint64_t* rows, int rounds, int mode) {
  const int P = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  __shared__ int s_owner;
  __shared__ double s_row[160];
  for (int r = 1; r <= rounds; ++r) {
    const uint64_t tag = uint64_t(r) << 32;
    const int par = r & 1;
    if (mode & 1) {
      uint64_t* row = rows + ((size_t)cta * 2 + par) * 320;
      if (tid < 130) st2<kSys>(row + 2 * tid, tag | tid, tag | cta);
    }
    if (tid == 0) st2<kSys>(recs + ((size_t)par * P + cta) * 2, tag | cta, tag | ((cta * 7 + r) % 1000));
    if (mode & 2) {
      if (tid < 32) {
        int best = -1, bestv = -1;
        bool got[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) got[q] = tid + 32 * q >= P;
        bool all = false;
        while (!all) {
          all = true;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (!got[q]) {
              uint64_t a, b;
              ld2<kSys>(recs + ((size_t)par * P + tid + 32 * q) * 2, a, b);
              if ((a >> 32) == uint64_t(r) && (b >> 32) == uint64_t(r)) {
                got[q] = true;
                int v = int(uint32_t(b));
                if (v > bestv) bestv = v, best = tid + 32 * q;
              } else {
                all = false;
              }
            }
          }
        }
        for (int o = 16; o; o >>= 1) {
          int ov = __shfl_xor_sync(~0u, bestv, o), ob = __shfl_xor_sync(~0u, best, o);
          if (ov > bestv || (ov == bestv && ob < best)) bestv = ov, best = ob;
        }
        if (tid == 0) s_owner = best;
      }
    } else {
      __shared__ int s_v[256];
      if (tid < P) {
        uint64_t a, b;
        do {
          ld2<kSys>(recs + ((size_t)par * P + tid) * 2, a, b);
        } while ((a >> 32) != uint64_t(r) || (b >> 32) != uint64_t(r));
        s_v[tid] = int(uint32_t(b));
      }
      __syncthreads();
      if (tid == 0) {
        int best = 0;
        for (int t = 1; t < P; ++t)
          if (s_v[t] > s_v[best]) best = t;
        s_owner = best;
      }
    }
    __syncthreads();
    if (mode & 1) {
      const int owner = s_owner;
      const uint64_t* row = rows + ((size_t)owner * 2 + par) * 320;
      if (tid < 130) {
        uint64_t a, b;
        do {
          ld2<kSys>(row + 2 * tid, a, b);
        } while ((a >> 32) != uint64_t(r) || (b >> 32) != uint64_t(r));
        s_row[tid] = double(uint32_t(a));
      }
    }
    __syncthreads();
  }
}

int main() {
  uint64_t *recs, *rows;
  CK(cudaMalloc(&recs, 2 * 256 * 16));
  CK(cudaMalloc(&rows, 2 * 256 * 320 * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int rounds = 3000;
  for (int sys = 0; sys < 2; ++sys)
    for (int mode = 0; mode < 4; ++mode)
      for (int P : {16, 64, 148}) {
        CK(cudaMemset(recs, 0, 2 * 256 * 16));
        CK(cudaMemset(rows, 0, 2 * 256 * 320 * 8));
        void* args[] = {&recs, &rows, &rounds, &mode};
        void* fn = sys ? (void*)xchg<true> : (void*)xchg<false>;
        cudaEventRecord(e0);
        CK(cudaLaunchCooperativeKernel(fn, P, 256, args, 0, 0));
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%s mode=%d (row=%d warp0poll=%d) P=%3d : %.3f us/round\n", sys ? "volatile" : "relaxed ", mode,
               mode & 1, (mode >> 1) & 1, P, ms * 1e3 / rounds);
      }
  return 0;
}
