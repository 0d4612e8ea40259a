// Ring-buffer probe for the trailing DGEMM main loop (no epilogue): 148 CTAs x
// 256 threads, 64x32 warp tiles, k-chunks of K4 blocks (4 KiB per operand per
// block) streamed by cp.async.bulk through an S-stage ring.
//   mode 0: producer = tid 0, refills the stage of chunk q-1 after its empty barrier
//   mode 1: the last warp to release a stage refills it (shared counter, no waiting)
//   mode 2: as 0 but consumers never wait on `full` (race; pure-overhead bound)
//   mode 3: no bulk copies at all, consumers just run on stale smem (upper bound)
// operands come from a `span`-byte window of a large buffer (L2-resident or not).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gemm_ring gemm_ring.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int S = 3, K4 = 4, BLK = 512;
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su(b)), "r"(ph) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) ring(const double* __restrict__ P, const double* __restrict__ Q, long long span_blocks,
                                               int nchunks, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* sP = (double*)sm;
  double* sQ = sP + S * K4 * BLK;
  uint64_t* full = (uint64_t*)(sQ + S * K4 * BLK);
  uint64_t* empty = full + S;
  int* cnt = (int*)(empty + S);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, wm = warp >> 2, wn = warp & 3;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(su(&empty[s])));
      cnt[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int q) {
    const int s = q % S;
    long long blk, blkq;
    if (MODE == 5 || MODE == 6) {
      const int i = q / 35, c = q - i * 35;
      const int ti = MODE == 5 ? i + 130 : blockIdx.x, tj = MODE == 5 ? blockIdx.x % 130 : i;  // 5: shared P, 6: shared Q
      blk = ((long long)ti * 140 + c * K4) % (span_blocks - K4);
      blkq = ((long long)tj * 140 + c * K4) % (span_blocks - K4);
    } else if (MODE == 4) {
      // real trailing-update addressing: tile t = bid + i*grid, row-major lower
      // order, k4cap = 140 blocks per 128-row tile, 35 chunks per tile
      const int i = q / 35, c = q - i * 35;
      const int t = blockIdx.x + i * gridDim.x;
      int ti = int((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
      while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
      while (ti * (ti + 1) / 2 > t) --ti;
      const int tj = t - ti * (ti + 1) / 2;
      blk = ((long long)ti * 140 + c * K4) % (span_blocks - K4);
      blkq = ((long long)tj * 140 + c * K4) % (span_blocks - K4);
    } else {
      blk = ((long long)blockIdx.x * 977 + (long long)q * K4 * 13) % (span_blocks - K4);
      blkq = blk;
    }
    const uint32_t bytes = K4 * BLK * 8;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(2 * bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sP + s * K4 * BLK)),
                 "l"(P + blk * BLK), "r"(bytes), "r"(su(&full[s])) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sQ + s * K4 * BLK)),
                 "l"(Q + blkq * BLK), "r"(bytes), "r"(su(&full[s])) : "memory");
  };
  if (MODE != 3 && tid == 0)
    for (int q = 0; q < S && q < nchunks; ++q) issue(q);
  double acc[8][4][2];
#pragma unroll
  for (int mi = 0; mi < 8; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  for (int q = 0; q < nchunks; ++q) {
    const int s = q % S;
    if (MODE == 0 || MODE == 1 || MODE >= 4) mwait(&full[s], (q / S) & 1);
    const double* ps = sP + s * K4 * BLK + wm * 8 * 32 + lane;
    const double* qs = sQ + s * K4 * BLK + wn * 4 * 32 + lane;
    for (int kb = 0; kb < K4; ++kb) {
      double a[8], b[4];
#pragma unroll
      for (int mi = 0; mi < 8; ++mi) a[mi] = ps[kb * BLK + mi * 32];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = qs[kb * BLK + ni * 32];
#pragma unroll
      for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
    __syncwarp();
    if (MODE == 0 || MODE == 2 || MODE >= 4) {
      if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
      if (tid == 0 && q >= 1 && q - 1 + S < nchunks) {
        const int qp = q - 1;
        mwait(&empty[qp % S], (qp / S) & 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(qp + S);
      }
    } else if (MODE == 1) {
      if (lane == 0) {
        int old = atomicAdd(&cnt[s], 1);
        if (old == 7) {
          cnt[s] = 0;
          __threadfence_block();
          if (q + S < nchunks) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(q + S);
          }
        }
      }
    }
  }
  double sum = 0;
#pragma unroll
  for (int mi = 0; mi < 8; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) sum += acc[mi][ni][0] + acc[mi][ni][1];
  if (sum == 1234.5) out[0] = sum;
  // drain outstanding copies of mode 2 before exit
  if (MODE == 2 && tid == 0)
    for (int q = (nchunks > S ? nchunks - S : 0); q < nchunks; ++q) mwait(&full[q % S], (q / S) & 1);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = size_t(64) << 20;  // 64 MiB per operand
  double *P, *Q, *out;
  cudaMalloc(&P, big);
  cudaMalloc(&Q, big);
  cudaMalloc(&out, 64);
  cudaMemset(P, 0, big);
  cudaMemset(Q, 0, big);
  size_t smem = size_t(S) * 2 * K4 * BLK * 8 + 2 * S * 8 + 64;
  void (*fns[7])(const double*, const double*, long long, int, double*) = {ring<0>, ring<1>, ring<2>, ring<3>, ring<4>, ring<5>, ring<6>};
  for (int m = 0; m < 7; ++m) cudaFuncSetAttribute(fns[m], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int nchunks = 2000;
  for (long long span_mb : {36LL, 64LL}) {
    long long span_blocks = span_mb * (1 << 20) / (BLK * 8);
    for (int m = 0; m < 7; ++m) {
      if (m == 2 || m == 1 || m == 3) continue;
      fns[m]<<<nsm, 256, smem>>>(P, Q, span_blocks, 20, out);
      cudaEventRecord(e0);
      fns[m]<<<nsm, 256, smem>>>(P, Q, span_blocks, nchunks, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 128 * 128 * 4.0 * K4 * nchunks * nsm;
      printf("span %3lld MB mode %d: %.2f TFLOP/s  (%s)\n", span_mb, m, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
      fflush(stdout);
    }
  }
  return 0;
}
