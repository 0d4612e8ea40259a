// Skeleton of one panel_push_kernel step (no gemv, no row delivery, no gathers) in a
// 16-CTA cluster of 256 threads, one row per thread: measure cycles per step while
// adding the pieces one by one (PIECES bitmask):
//   1 warp argmax + STS + __syncthreads      2 CTA argmax (every warp)
//   4 candidate st.async + mbarrier wait      8 winner argmax + lab swap
//  16 division v / vb                        32 z loop (threads j <= k) + taus + __syncthreads
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
__device__ __forceinline__ int lane_argmax(double v, int pos, bool valid) {
  const unsigned long long bits = valid ? (unsigned long long)__double_as_longlong(fabs(v)) : 0ull;
  const unsigned hi = valid ? unsigned(bits >> 32) + 1u : 0u;
  const unsigned m1 = __reduce_max_sync(0xffffffffu, hi);
  if (m1 == 0u) return -1;
  const bool c1 = hi == m1;
  const unsigned b1 = __ballot_sync(0xffffffffu, c1);
  if ((b1 & (b1 - 1u)) == 0u) return __ffs(b1) - 1;
  const unsigned lo = unsigned(bits);
  const unsigned m2 = __reduce_max_sync(0xffffffffu, c1 ? lo : 0u);
  const bool c2 = c1 && lo == m2;
  const unsigned id = __reduce_min_sync(0xffffffffu, c2 ? unsigned(pos) : 0xffffffffu);
  return __ffs(__ballot_sync(0xffffffffu, c2 && unsigned(pos) == id)) - 1;
}
struct __align__(16) C16 { double v; int pos; int ph; };
struct __align__(16) W32 { double v; int pos; int ph; int li; int pad[3]; };

template <int PIECES, int CL>
__global__ void __launch_bounds__(256, 1) sk(int steps, long long* out, double* sink) {
  __shared__ __align__(16) C16 cand[2][16];
  __shared__ __align__(16) W32 wc[8];
  __shared__ __align__(16) double zbuf[130], taus[130], col[256];
  __shared__ __align__(8) uint64_t bar[2];
  const uint32_t rank = cg::this_cluster().block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) { for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int j = tid; j < 130; j += 256) { zbuf[j] = 0; taus[j] = 1.0 + j; }
  const uint32_t rc = mapa(su(&cand[0][0]), lane & (CL - 1)), rc0 = mapa(su(&bar[0]), lane & (CL - 1)), rc1 = mapa(su(&bar[1]), lane & (CL - 1));
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  int lab = rank * 256 + tid + 1, ph = lab;
  double az = 0.001 * tid, cn = 1.0 + ((tid * 37 + rank * 11) & 255) * 0.01, vv = 0;
  long long t0 = clock64();
  for (int g = 0; g < steps; ++g) {
    const int par = g & 1, k = g % 96;
    const uint32_t phs = (g >> 1) & 1;
    if ((PIECES & 4) && tid == 0) expect(&bar[par], CL * 16);
    const double v = cn - az;
    vv = v;
    col[tid] = v;
    int wl = -1;
    if (PIECES & 1) {
      wl = lane_argmax(v, lab, lab > g);
      if (lane == (wl < 0 ? 0 : wl)) wc[warp] = W32{v, wl < 0 ? -1 : lab, ph, tid, {0, 0, 0}};
      __syncthreads();
    }
    W32 c{0.0, -1, 0, 0, {0, 0, 0}};
    if (PIECES & 2) {
      const W32 mine = lane < 8 ? wc[lane] : W32{0.0, -1, 0, 0, {0, 0, 0}};
      const int w2 = lane_argmax(mine.v, mine.pos, lane < 8 && mine.pos >= 0);
      c = wc[w2 < 0 ? 0 : w2];
    }
    int b = g + 2, pb = b;
    double vb = 1.5;
    if (PIECES & 4) {
      if (warp == 0 && lane < CL) {
        const unsigned long long v64 = __double_as_longlong(c.v + rank);
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                         rc + (par * 16 + rank) * 16), "r"(uint32_t(v64)), "r"(uint32_t(v64 >> 32)), "r"(uint32_t(c.pos)), "r"(uint32_t(c.ph)), "r"(par ? rc1 : rc0) : "memory");
      }
      mwait(&bar[par], phs);
      if (PIECES & 8) {
        const C16 mine = lane < CL ? cand[par][lane] : C16{0.0, -1, 0};
        int owner = lane_argmax(mine.v, mine.pos, lane < CL && mine.pos >= 0);
        if (owner < 0) owner = 0;
        const C16 w = cand[par][owner];
        b = w.pos; pb = w.ph; vb = w.v + 1.0;
        const int a_pos = g + 1;
        if (b != a_pos) lab = lab == b ? a_pos : (lab == a_pos ? b : lab);
      }
    }
    if (PIECES & 16) { vv = vv / vb; col[tid] = vv; }
    if (PIECES & 32) {
      for (int j = tid; j <= k; j += 256) {
        const double xm = j >= 1 ? col[j - 1] : 0.0, xp = j + 1 < k ? col[j + 1] : 1.0;
        zbuf[j] = (j >= 1 ? taus[j] * xm : 0.0) - taus[j + 1] * xp;
      }
      if (tid == 0) taus[k] = vb;
      __syncthreads();
      az += zbuf[k] * 1e-9;
    }
    cn += 1e-7 * (pb & 7);
  }
  long long t1 = clock64();
  if (tid == 0 && rank == 0) out[0] = (t1 - t0) / steps;
  sink[rank * 256 + tid] = vv + az;
}
template <int P, int CL> void run(long long* d, double* s) {
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(CL); cfg.blockDim = dim3(256);
  cudaLaunchAttribute at; at.id = cudaLaunchAttributeClusterDimension; at.val.clusterDim.x = CL; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
  cfg.attrs = &at; cfg.numAttrs = 1;
  cudaFuncSetAttribute(sk<P, CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int i = 0; i < 2; ++i) cudaLaunchKernelEx(&cfg, sk<P, CL>, 4000, d, s);
  long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("cluster %2d pieces %2d: %lld cycles/step (%s)\n", CL, P, h, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  long long* d; cudaMalloc(&d, 64); double* s; cudaMalloc(&s, 16 * 256 * 8);
  run<7, 16>(d, s); run<63, 16>(d, s);
  run<7, 8>(d, s); run<63, 8>(d, s);
  run<7, 4>(d, s); run<63, 4>(d, s);
  run<7, 2>(d, s); run<63, 2>(d, s);
  run<3, 1>(d, s); run<59, 1>(d, s);
  return 0;
}
