// DSMEM broadcast probe: 16-CTA cluster, every CTA reads a K-double row that
// lives in one CTA's shared memory (the pivot-row broadcast of the panel step).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem dsmem.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void cbar() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int MODE>
__global__ void probe(int K, int rounds, long long* out) {
  __shared__ __align__(16) double row[1024];
  __shared__ __align__(16) double dst[1024];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank(), tid = threadIdx.x;
  for (int j = tid; j < K; j += blockDim.x) { row[j] = rank * 1000 + j; dst[j] = 0; }
  cbar();
  long long t_bar = 0, t_read = 0;
  for (int r = 0; r < rounds; ++r) {
    const int owner = r % 16;
    long long t0 = clock64();
    cbar();
    long long t1 = clock64();
    const double* src = cl.map_shared_rank(row, owner);
    if (MODE == 0) {  // 8-byte loads
      for (int j = tid; j < K; j += blockDim.x) dst[j] += src[j];
    } else if (MODE == 1) {  // 16-byte loads
      const double2* s2 = reinterpret_cast<const double2*>(src);
      double2* d2 = reinterpret_cast<double2*>(dst);
      for (int j = tid; j < K / 2; j += blockDim.x) { double2 v = s2[j]; double2 w = d2[j]; w.x += v.x; w.y += v.y; d2[j] = w; }
    } else if (MODE == 2) {  // local only (baseline)
      for (int j = tid; j < K; j += blockDim.x) dst[j] += row[j];
    } else {  // only CTA 0 reads (no contention)
      if (rank == 0)
        for (int j = tid; j < K; j += blockDim.x) dst[j] += src[j];
    }
    __syncthreads();
    long long t2 = clock64();
    t_bar += t1 - t0;
    t_read += t2 - t1;
  }
  __syncthreads();
  double chk = 0;
  for (int j = 0; j < K; ++j) chk += dst[j];
  if (tid == 0) {
    out[40 + rank] = (long long)chk;
    out[rank * 2] = t_bar / rounds;
    out[rank * 2 + 1] = t_read / rounds;
  }
}

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// every CTA pushes a K-double payload to all 16 CTAs (bulk DSMEM copy with
// complete_tx on the destination's mbarrier), then waits for 16 payloads.
__global__ void push_probe(int K, int rounds, long long* out) {
  __shared__ __align__(128) double sendbuf[2][160];
  __shared__ __align__(128) double recv[2][16][160];
  __shared__ __align__(8) unsigned long long mbar[2];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank(), tid = threadIdx.x;
  const unsigned bytes = (unsigned)(((K * 8) + 15) & ~15);
  if (tid == 0) {
    for (int p = 0; p < 2; ++p) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar[p])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cbar();
  long long t_tot = 0;
  double chk = 0;
  for (int r = 0; r < rounds; ++r) {
    const int par = r & 1;
    long long t0 = clock64();
    for (int j = tid; j < K; j += blockDim.x) sendbuf[par][j] = rank + j + r;
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mbar[par])), "r"(16 * bytes) : "memory");
    __syncthreads();
    if (tid < 16) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      unsigned dst = su32(&recv[par][rank][0]);
      unsigned bar = su32(&mbar[par]);
      unsigned rdst, rbar;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(dst), "r"(tid));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(bar), "r"(tid));
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rdst),
                   "r"(su32(&sendbuf[par][0])), "r"(bytes), "r"(rbar) : "memory");
    }
    // wait for all 16 payloads of this round
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su32(&mbar[par])),
                 "r"((unsigned)((r >> 1) & 1)) : "memory");
    if (tid == 0) chk += recv[par][(r * 7) % 16][K - 1];
    long long t1 = clock64();
    t_tot += t1 - t0;
  }
  cbar();
  if (tid == 0) {
    out[rank * 2] = 0;
    out[rank * 2 + 1] = t_tot / rounds;
    out[40 + rank] = (long long)chk;
  }
}

int main() {
  long long* out;
  cudaMalloc(&out, 64 * 8);
  long long h[64];
  for (int K : {64, 130, 260}) {
    for (int mode = 0; mode < 4; ++mode) {
      void (*fn)(int, int, long long*) =
          mode == 0 ? probe<0> : mode == 1 ? probe<1> : mode == 2 ? probe<2> : probe<3>;
      cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(16);
      cfg.blockDim = dim3(512);
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = 16;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      int rounds = 2000;
      cudaError_t e = cudaLaunchKernelEx(&cfg, fn, K, rounds, out);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("err %s\n", cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(h, out, 32 * 8, cudaMemcpyDeviceToHost);
      long long bmax = 0, rmax = 0, rsum = 0;
      for (int i = 0; i < 16; ++i) {
        bmax = h[2 * i] > bmax ? h[2 * i] : bmax;
        rmax = h[2 * i + 1] > rmax ? h[2 * i + 1] : rmax;
        rsum += h[2 * i + 1];
      }
      printf("K=%3d mode=%d (%s): barrier %lld cyc, read+sync max %lld avg %lld cyc\n", K, mode,
             mode == 0 ? "8B dsmem" : mode == 1 ? "16B dsmem" : mode == 2 ? "local" : "single reader", bmax, rmax,
             rsum / 16);
    }
  }
  for (int K : {64, 130}) {
    cudaFuncSetAttribute(push_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(512);
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 16;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int rounds = 2000;
    cudaError_t e = cudaLaunchKernelEx(&cfg, push_probe, K, rounds, out);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("push err %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, out, 32 * 8, cudaMemcpyDeviceToHost);
    long long rmax = 0;
    for (int i = 0; i < 16; ++i) rmax = h[2 * i + 1] > rmax ? h[2 * i + 1] : rmax;
    printf("K=%3d push-all bulk DSMEM round: %lld cyc\n", K, rmax);
  }
  return 0;
}
