// Row-broadcast alternatives after the 16-way candidate exchange (panel_push_kernel step):
//  mode 0: candidates only (baseline)
//  mode 1: push-all  -- every CTA st.async's its K-double row to all 16 (current kernel)
//  mode 3: pull      -- after the winner is known every CTA ld.shared::cluster.v2's the winner's row
//  mode 4: bulk      -- the winner CTA issues 16 cp.async.bulk shared::cta -> shared::cluster copies
//  mode 5: multicast -- every CTA writes its row to global before the exchange; the winner issues one
//                       cp.async.bulk global -> shared::cluster .multicast::cluster (ctaMask 0xffff)
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su(b)), "r"(ph) : "memory"); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(bytes) : "memory"); }

template <int MODE>
__global__ void __launch_bounds__(256, 1) xk(int K, int rounds, long long* out, double* gbuf) {
  __shared__ __align__(128) double rows[2][16][104];
  __shared__ __align__(128) double myrow[2][104];
  __shared__ __align__(16) double cand[2][16][2];
  __shared__ __align__(16) double slab[104 * 17];
  __shared__ __align__(8) uint64_t bar[4];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t rank = cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 104 * 17; i += 256) slab[i] = i * 1e-3 + rank;
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  const uint32_t dst = tid & 15;
  const uint32_t rrows = mapa(su(&rows[0][0][0]), dst), rb0 = mapa(su(&bar[2]), dst), rb1 = mapa(su(&bar[3]), dst);
  const uint32_t rc = mapa(su(&cand[0][0][0]), lane & 15), rc0 = mapa(su(&bar[0]), lane & 15), rc1 = mapa(su(&bar[1]), lane & 15);
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  const int np = (K + 1) / 2;
  const uint32_t rowbytes = uint32_t(np) * 16u;
  double acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    const int par = r & 1;
    const uint32_t ph = (r >> 1) & 1;
    if (tid == 0) {
      expect(&bar[par], 16 * 16);
      if (MODE == 1) expect(&bar[2 + par], 16u * rowbytes);
      if (MODE == 4 || MODE == 5) expect(&bar[2 + par], rowbytes);
    }
    const int lc = (r * 7 + rank) & 15;
    if (MODE == 4 || MODE == 3) {  // contiguous copy of this CTA's candidate row
      if (tid < K) myrow[par][tid] = slab[tid * 17 + lc];
      if (MODE == 4) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (MODE == 5) {
      if (tid < K) gbuf[(rank * 2 + par) * 104 + tid] = slab[tid * 17 + lc];
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    if (MODE >= 3) __syncthreads();
    if (tid < 16) {
      double v = 1.0 + ((r * 13 + rank * 5) & 15);
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                       rc + (par * 16 + rank) * 16), "d"(v), "d"((double)rank), "r"(par ? rc1 : rc0) : "memory");
    }
    if (MODE == 1)
      for (int p = tid >> 4; p < np; p += 16) {
        const double x0 = slab[(2 * p) * 17 + lc], x1 = slab[(2 * p + 1) * 17 + lc];
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                         rrows + ((par * 16 + rank) * 104 + 2 * p) * 8), "d"(x0), "d"(x1), "r"(par ? rb1 : rb0) : "memory");
      }
    mwait(&bar[par], ph);
    const double cv = lane < 16 ? cand[par][lane][0] : 0.0;
    const unsigned long long bits = __double_as_longlong(cv);
    unsigned hi = lane < 16 ? unsigned(bits >> 32) + 1 : 0;
    unsigned m1 = __reduce_max_sync(~0u, hi);
    unsigned m2 = __reduce_max_sync(~0u, hi == m1 ? unsigned(bits) : 0u);
    unsigned id = __reduce_min_sync(~0u, (hi == m1 && unsigned(bits) == m2) ? lane : 99u);
    const int owner = int(id) & 15;
    if (MODE == 3) {
      if (tid < np) {
        const uint32_t src = mapa(su(&myrow[par][2 * tid]), owner);
        double x0, x1;
        asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(x0), "=d"(x1) : "r"(src) : "memory");
        acc += x0 + x1;
      }
    }
    if (MODE == 4 && owner == int(rank) && tid < 16) {
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       rrows + (par * 16 * 104) * 8), "r"(su(&myrow[par][0])), "r"(rowbytes), "r"(par ? rb1 : rb0) : "memory");
    }
    if (MODE == 5 && owner == int(rank) && tid == 0) {
      const uint32_t dsm = su(&rows[par][0][0]);
      const double* src = gbuf + (rank * 2 + par) * 104;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
                       dsm), "l"(src), "r"(rowbytes), "r"(su(&bar[2 + par])), "h"((unsigned short)0xffff) : "memory");
    }
    if (MODE == 1 || MODE == 4 || MODE == 5) {
      mwait(&bar[2 + par], ph);
      if (tid < K) acc += rows[par][MODE == 1 ? owner : 0][tid];
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0 && rank == 0) out[0] = (t1 - t0) / rounds;
  if (acc == 12345.6) out[1] = 1;
}

template <int M>
void run(int K, long long* d, double* g) {
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(16); cfg.blockDim = dim3(256);
  cudaLaunchAttribute at; at.id = cudaLaunchAttributeClusterDimension; at.val.clusterDim.x = 16; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
  cfg.attrs = &at; cfg.numAttrs = 1;
  cudaFuncSetAttribute(xk<M>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int it = 0; it < 2; ++it) cudaLaunchKernelEx(&cfg, xk<M>, K, 2000, d, g);
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("mode %d K=%3d: %lld cycles/round (%s)\n", M, K, h, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  double* g; cudaMalloc(&g, 16 * 2 * 104 * 8);
  run<0>(0, d, g);
  for (int K : {16, 48, 96}) { run<1>(K, d, g); run<3>(K, d, g); run<4>(K, d, g); run<5>(K, d, g); }
  return 0;
}
