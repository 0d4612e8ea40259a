// Cluster exchange probe for the panel step: 16 CTAs each publish a candidate
// (16-byte header + K-double row); every CTA must end up with the winner's row.
//   A: pull   -- row to own smem, header to all via st.shared::cluster,
//               barrier.cluster, then ld.shared::cluster of the winner's row
//   B: push   -- header+row to all 16 via cp.async.bulk (DSMEM), mbarrier wait
//   C: push   -- header+row to all 16 via st.async.v2.f64 (32 lanes), mbarrier wait
//   D: as B, plus one CTA (the "row a" owner) pushes a second row to all
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xchg xchg.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;
constexpr int KMAX = 130, MSG = 2 + KMAX + 2;  // doubles per message slot (header + row, padded)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cbar() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mwait_cl(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su(b)), "r"(ph) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) xk(int K, int rounds, long long* out) {
  __shared__ __align__(128) double slab[2 * 256];
  __shared__ __align__(128) double pub[2][MSG];
  __shared__ __align__(128) double send[2][2][MSG];
  __shared__ __align__(128) double recv[2][17][MSG];
  __shared__ __align__(16) double cand[2][16][2];
  __shared__ __align__(16) double wrow[MSG];
  __shared__ __align__(8) uint64_t mbar[2];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank(), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 2 * 256; i += 256) slab[i] = rank + 1e-3 * i;
  const int bytes = ((2 + K) * 8 + 15) & ~15;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cbar();
  double chk = 0;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    const int par = r & 1;
    const int cand_row = (rank * 37 + r) & 255;
    const int winner = (r * 7) & 15;
    const int owner_a = (r >> 4) & 15;
    if (MODE == 0) {
      if (warp == 0) {
        for (int j = lane; j < K; j += 32) pub[par][j] = slab[(j & 1) * 256 + cand_row];
        __syncwarp();
        if (lane < 16) {
          double* dst = cl.map_shared_rank(&cand[par][rank][0], lane);
          dst[0] = 1.0 + rank;
          dst[1] = (double)cand_row;
        }
      }
      cbar();
      const double* wr = cl.map_shared_rank(&pub[par][0], winner);
      for (int j = tid; j < K; j += 256) wrow[j] = wr[j];
      __syncthreads();
      chk += wrow[K - 1] + cand[par][winner][0];
    } else if (MODE == 4 || MODE == 5) {
      // local publish: header + row into pub-like slot send[par][0]
      if (warp == 0) {
        for (int j = lane; j < K; j += 32) send[par][0][2 + j] = slab[(j & 1) * 256 + cand_row];
        if (lane == 0) { send[par][0][0] = 1.0 + rank; send[par][0][1] = cand_row; }
      } else if (MODE == 5 && warp == 1 && rank == owner_a) {
        for (int j = lane; j < K + 1; j += 32) send[par][1][j] = slab[(j & 1) * 256 + (cand_row ^ 1)];
      }
      cbar();
      const int L = K + 2;
      const int tot = 16 * L + (MODE == 5 ? K + 1 : 0);
#pragma unroll 4
      for (int e = tid; e < tot; e += 256) {
        double v;
        if (e < 16 * L) {
          const int m = e / L, j = e - m * L;
          v = *cl.map_shared_rank(&send[par][0][j], m);
          recv[par][m][j] = v;
        } else {
          v = *cl.map_shared_rank(&send[par][1][e - 16 * L], owner_a);
          recv[par][16][e - 16 * L] = v;
        }
      }
      __syncthreads();
      chk += recv[par][winner][2 + K - 1] + recv[par][winner][0];
    } else if (MODE == 1 || MODE == 3) {
      const bool extra = MODE == 3 && rank == owner_a;
      if (tid == 0) {
        const uint32_t tot = 16u * bytes + (MODE == 3 ? uint32_t(bytes) * 16u / 16u : 0u);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&mbar[par])), "r"(MODE == 3 ? 17u * bytes : tot) : "memory");
      }
      if (warp == 0) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        for (int j = lane; j < K; j += 32) send[par][0][2 + j] = slab[(j & 1) * 256 + cand_row];
        if (lane == 0) { send[par][0][0] = 1.0 + rank; send[par][0][1] = cand_row; }
        if (extra)
          for (int j = lane; j < K; j += 32) send[par][1][2 + j] = slab[(j & 1) * 256 + (cand_row ^ 1)];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane < 16) {
          uint32_t dst = su(&recv[par][rank][0]), bar = su(&mbar[par]), rdst, rbar;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(dst), "r"(lane));
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(bar), "r"(lane));
          asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rdst),
                       "r"(su(&send[par][0][0])), "r"(bytes), "r"(rbar) : "memory");
          if (extra) {
            uint32_t dst2 = su(&recv[par][16][0]), rdst2;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst2) : "r"(dst2), "r"(lane));
            asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rdst2),
                         "r"(su(&send[par][1][0])), "r"(bytes), "r"(rbar) : "memory");
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      mwait_cl(&mbar[par], (r >> 1) & 1);
      chk += recv[par][winner][2 + K - 1] + recv[par][winner][0];
      __syncthreads();
    } else {
      if (tid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&mbar[par])), "r"(16u * bytes) : "memory");
      if (warp == 0) {
        for (int j = lane; j < K; j += 32) send[par][0][2 + j] = slab[(j & 1) * 256 + cand_row];
        if (lane == 0) { send[par][0][0] = 1.0 + rank; send[par][0][1] = cand_row; }
        __syncwarp();
        const int n2 = bytes / 16;
        for (int e = lane; e < 16 * n2; e += 32) {
          const int d = e / n2, c = e - d * n2;
          uint32_t dst = su(&recv[par][rank][2 * c]), bar = su(&mbar[par]), rdst, rbar;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(dst), "r"(d));
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(bar), "r"(d));
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(rdst),
                       "d"(send[par][0][2 * c]), "d"(send[par][0][2 * c + 1]), "r"(rbar) : "memory");
        }
      }
      mwait_cl(&mbar[par], (r >> 1) & 1);
      chk += recv[par][winner][2 + K - 1] + recv[par][winner][0];
      __syncthreads();
    }
  }
  long long t1 = clock64();
  cbar();
  if (tid == 0) {
    out[rank] = (t1 - t0) / rounds;
    out[32 + rank] = (long long)chk;
  }
}

int main() {
  long long* out;
  cudaMalloc(&out, 64 * 8);
  long long h[64];
  void (*fns[6])(int, int, long long*) = {xk<0>, xk<1>, xk<2>, xk<3>, xk<4>, xk<5>};
  const char* names[6] = {"pull+cbar", "bulk push", "st.async push", "bulk push+rowA", "cbar+pull-all", "cbar+pull-all+rowA"};
  for (int K : {33, 65, 97, 129}) {
    for (int m = 0; m < 6; ++m) {
      if (m == 2) continue;
      cudaFuncSetAttribute(fns[m], cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(16);
      cfg.blockDim = dim3(256);
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = 16;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, fns[m], K, 4000, out);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("K=%d mode %d err %s\n", K, m, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, out, 64 * 8, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < 16; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("K=%3d %-16s %5lld cyc/round\n", K, names[m], mx);
      fflush(stdout);
    }
  }
  return 0;
}
