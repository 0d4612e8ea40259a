// Unblocked Wimmer two-step LTL^T with optional partial pivoting, fused into
// one single-cluster kernel.
//
// Reference semantics (restated): _panel_twostep unblocked.py:136-171,
// ltlt_unb_twostep unblocked.py:229-240, _eliminate unblocked.py:63-91,
// _sym_swap_lower core.py:294-324, trapezoid_rank2 / skew_rank2
// kernels2.py:93-131,296-312.  Per pair (g, g+1):
//   eliminate(g), eliminate(g+1)         iamax (ties -> lowest), symmetric swap, tau, scale
//   fold:  X[s:, g+2] -= tau[g+1] (X[g+2, g] l2 - l1)      (s = g+3)
//   wv  =  X[s:, g+2] - tau[g+1] l1
//   X[s:, s:] -= wv l2^T - l2 wv^T      (one skew rank-2 for both couplings)
//
// B200 mapping: the matrix lives in the shared memory of a 16-CTA cluster,
// column j owned by CTA j % C (whole columns, so the rank-2 and the column
// scans are local and coalesced); symmetric interchanges and the fold touch
// remote columns through DSMEM; the argmax of a column is a warp-shuffle /
// redux reduction inside its owner CTA; phases are separated by the
// hardware cluster barrier.  The rank-2 vectors (wv, l2) are broadcast
// through L2 (one writer, 16 readers) because a DSMEM fan-out from one SM is
// port-bandwidth bound.  For n too large for the cluster's shared memory
// the same kernel runs with the columns in global memory (the L buffer).
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace skl {
namespace {

constexpr int kTThreads = 512;
constexpr int kTWarps = kTThreads / 32;

__device__ __forceinline__ void tbarrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ int twarp_argmax(double v, int idx, bool valid) {
  const unsigned long long bits = valid ? (unsigned long long)__double_as_longlong(fabs(v)) : 0ull;
  const unsigned hi = valid ? unsigned(bits >> 32) + 1u : 0u;
  const unsigned lo = unsigned(bits);
  const unsigned m1 = __reduce_max_sync(0xffffffffu, hi);
  const bool c1 = valid && hi == m1;
  const unsigned m2 = __reduce_max_sync(0xffffffffu, c1 ? lo : 0u);
  const bool c2 = c1 && lo == m2;
  const unsigned id = __reduce_min_sync(0xffffffffu, c2 ? unsigned(idx) : 0xffffffffu);
  return id == 0xffffffffu ? -1 : int(id);
}

struct TArgs {
  const double* X;
  long long ldx;
  double* L;
  long long ldl;
  int n;
  int pivot;
  int smem_mode;  // 1: columns in cluster smem; 0: columns in L (global)
  double* tau;
  long long* piv;
  int* info;
  double* vec;    // global broadcast buffer [2][n]: wv, l2
};

struct TCtx {
  cg::cluster_group cl;
  double* local;  // smem column store (smem mode)
  int C, cta, n;
  int smem_mode;
  double* L;
  long long ldl;
  int lgC;        // C is a power of two (8 or 16)
  __device__ __forceinline__ double* col(int j) const {
    if (!smem_mode) return L + (long long)j * ldl;
    double* p = local + (size_t)(j >> lgC) * n;
    const int owner = j & (C - 1);
    return owner == cta ? p : cl.map_shared_rank(p, owner);
  }
};

// mailbox (per CTA smem): [0] pivot row b, [1] status flag, [2..3] tau bits
__device__ __forceinline__ void post_pivot(const TCtx& c, int* mbox, int b, int status) {
  const int lane = threadIdx.x & 31;
  if (lane < c.C) {
    int* dst = c.cl.map_shared_rank(mbox, lane);
    dst[0] = b;
    dst[1] = status;
  }
}

// Owner of column g: argmax |X[g+1:, g]| (ties -> lowest), or the unpivoted
// zero test.  Result posted to every CTA's mailbox (caller then barriers).
__device__ void choose_pivot(const TCtx& c, int g, int pivot, double* red_v, int* red_i, int* mbox) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, n = c.n;
  const double* x = c.col(g);
  if (pivot) {
    double bv = 0.0;
    int bi = -1;
    for (int i = g + 1 + tid; i < n; i += kTThreads) {
      double v = x[i];
      if (bi < 0 || fabs(v) > fabs(bv)) {
        bv = v;
        bi = i;
      }
    }
    const int id = twarp_argmax(bv, bi, bi >= 0);
    if (bi >= 0 && bi == id) {
      red_v[warp] = bv;
      red_i[warp] = bi;
    }
    if (lane == 0 && id < 0) red_i[warp] = -1;
    __syncthreads();
    if (warp == 0) {
      const bool ok = lane < kTWarps && red_i[lane] >= 0;
      const int id2 = twarp_argmax(ok ? red_v[lane] : 0.0, ok ? red_i[lane] : 0, ok);
      post_pivot(c, mbox, id2 < 0 ? g + 1 : id2, 0);
    }
  } else {
    // unpivoted: ZeroPivot(g) if X[g+1,g] == 0 with a nonzero below (unblocked.py:83-85)
    int nz = 0;
    const bool zero = x[g + 1] == 0.0;
    if (zero)
      for (int i = g + 2 + tid; i < n; i += kTThreads) nz |= x[i] != 0.0;
    nz = __syncthreads_or(nz);
    if (warp == 0) post_pivot(c, mbox, g + 1, zero && nz ? 1 : 0);
  }
}

// symmetric interchange of positions a < b over the whole matrix; every CTA
// handles the elements of the columns it owns (disjoint writes).
__device__ void sym_swap(const TCtx& c, int a, int b) {
  const int tid = threadIdx.x, n = c.n, C = c.C, cta = c.cta;
  // rows a and b of the columns j < a owned here
  for (int j = cta + C * (tid / 32); j < a; j += C * kTWarps) {
    if ((tid & 31) == 0) {
      double* p = c.col(j);
      double t = p[a];
      p[a] = p[b];
      p[b] = t;
    }
  }
  // columns a and b below row b: done by the owner of column a
  if (a % C == cta) {
    double* pa = c.col(a);
    double* pb = c.col(b);
    for (int i = b + 1 + tid; i < n; i += kTThreads) {
      double t = pa[i];
      pa[i] = pb[i];
      pb[i] = t;
    }
    if (tid == 0) pa[b] = -pa[b];
  }
  // crossing segment: (i, a) <-> -(b, i) for a < i < b, by the owner of column i
  {
    double* pa = c.col(a);
    for (int i = a + 1 + ((cta - (a + 1)) % C + C) % C + C * tid; i < b; i += C * kTThreads) {
      double* pi = c.col(i);
      double t = pi[b];
      double u = pa[i];
      pa[i] = -t;
      pi[b] = -u;
    }
  }
}

__global__ void __launch_bounds__(kTThreads, 1) twostep_kernel(TArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TCtx c{cg::this_cluster(), nullptr, (int)gridDim.x, (int)blockIdx.x, a.n, a.smem_mode, a.L, a.ldl,
         gridDim.x == 16 ? 4 : (gridDim.x == 8 ? 3 : (gridDim.x == 4 ? 2 : (gridDim.x == 2 ? 1 : 0)))};
  const int n = a.n, C = c.C, cta = c.cta, tid = threadIdx.x;
  const int ncl = (n + C - 1) / C;
  double* vbuf = reinterpret_cast<double*>(smem_raw);  // [2][n] staged wv, l2
  double* red_v = vbuf + 2 * n;
  int* red_i = reinterpret_cast<int*>(red_v + kTWarps);
  int* mbox = red_i + kTWarps;  // [4]
  c.local = reinterpret_cast<double*>(smem_raw + (((size_t)(2 * n + kTWarps) * 8 + kTWarps * 4 + 16 + 127) & ~size_t(127)));

  // load the owned columns (strictly-lower part)
  if (a.smem_mode) {
    for (int s = 0; s < ncl; ++s) {
      const int j = cta + s * C;
      if (j >= n) break;
      double* p = c.local + (size_t)s * n;
      for (int i = j + 1 + tid; i < n; i += kTThreads) p[i] = a.X[(long long)j * a.ldx + i];
    }
  }
  if (cta == 0 && tid == 0) {
    a.info[0] = 0;
    if (a.pivot) a.piv[0] = 0;
  }
  tbarrier();

  const int end = n - 1;
  int g = 0;
  int failed = 0;
  while (g < end && !failed) {
    const bool single = g + 1 >= end;
    // ---- eliminate(g) -------------------------------------------------------
    if (g % C == cta) choose_pivot(c, g, a.pivot, red_v, red_i, mbox);
    tbarrier();
    int b = mbox[0];
    if (mbox[1]) {
      if (cta == 0 && tid == 0) a.info[0] = g + 1;
      failed = 1;
      break;
    }
    if (a.pivot) {
      if (cta == 0 && tid == 0) a.piv[g + 1] = b - (g + 1);
      if (b != g + 1) sym_swap(c, g + 1, b);
    }
    tbarrier();
    // tau[g], scale column g (owner of g); eliminate(g+1) pivot choice (owner of g+1)
    if (g % C == cta) {
      double* x = c.col(g);
      const double t = x[g + 1];
      if (tid == 0) a.tau[g] = t;
      if (t != 0.0)
        for (int i = g + 2 + tid; i < n; i += kTThreads) x[i] = x[i] / t;
      __syncthreads();
      if (tid == 0) x[g + 1] = 1.0;
    }
    if (single) {
      // odd leftover: right-looking rank-2 on [g+2:, g+2:] (unblocked.py:151-156)
      tbarrier();
      if (g + 2 < n) {
        // wv = X[g+2:, g] (L col), l2 = X[g+2:, g+1]: X += wv l2^T - l2 wv^T
        const double* l1 = c.col(g);
        const double* l2 = c.col(g + 1);
        for (int i = g + 2 + tid; i < n; i += kTThreads) {
          vbuf[i] = l1[i];
          vbuf[n + i] = l2[i];
        }
        __syncthreads();
        for (int s = 0; s < ncl; ++s) {
          const int j = cta + s * C;
          if (j >= n) break;
          if (j < g + 2) continue;
          double* p = c.col(j);
          const double xj = vbuf[j], yj = vbuf[n + j];
          for (int i = j + 1 + tid; i < n; i += kTThreads) p[i] += vbuf[i] * yj - vbuf[n + i] * xj;
        }
      }
      g += 1;
      break;
    }
    if ((g + 1) % C == cta) choose_pivot(c, g + 1, a.pivot, red_v, red_i, mbox);
    tbarrier();
    b = mbox[0];
    if (mbox[1]) {
      if (cta == 0 && tid == 0) a.info[0] = g + 2;
      failed = 1;
      break;
    }
    if (a.pivot) {
      if (cta == 0 && tid == 0) a.piv[g + 2] = b - (g + 2);
      if (b != g + 2) sym_swap(c, g + 2, b);
    }
    tbarrier();
    // ---- tau[g+1], scale column g+1, fold into column g+2, rank-2 vectors ---
    const int s0 = g + 3;
    if ((g + 2) % C == cta || (g + 2 >= n && (g + 1) % C == cta)) {
      double* x1 = c.col(g + 1);
      const double t1 = x1[g + 2];
      if (tid == 0) a.tau[g + 1] = t1;
      if (g + 2 < n) {
        const double* l1 = c.col(g);
        double* x2 = c.col(g + 2);
        const double x20 = l1[g + 2];  // work[g+2, g]
        for (int i = s0 + tid; i < n; i += kTThreads) {
          const double l2 = t1 != 0.0 ? x1[i] / t1 : x1[i];
          x1[i] = l2;
          const double l1i = l1[i];
          const double f = x2[i] - t1 * (x20 * l2 - l1i);
          x2[i] = f;
          a.vec[i] = f - t1 * l1i;  // wv
          a.vec[n + i] = l2;
        }
      }
      __syncthreads();
      if (tid == 0) x1[g + 2] = 1.0;
    }
    __threadfence();
    tbarrier();
    // ---- X[s:, s:] -= wv l2^T - l2 wv^T on the owned columns ----------------
    if (s0 < n) {
      for (int i = s0 + tid; i < n; i += kTThreads) {
        vbuf[i] = __ldcg(a.vec + i);
        vbuf[n + i] = __ldcg(a.vec + n + i);
      }
      __syncthreads();
      for (int s = 0; s < ncl; ++s) {
        const int j = cta + s * C;
        if (j >= n) break;
        if (j < s0) continue;
        double* p = c.col(j);
        const double wj = vbuf[j], lj = vbuf[n + j];
        for (int i = j + 1 + tid; i < n; i += kTThreads) p[i] -= vbuf[i] * lj - vbuf[n + i] * wj;
      }
    }
    g += 2;
    // the next eliminate() barrier orders this rank-2 before the next interchange
  }
  tbarrier();
  // write back the strictly-lower part (smem mode); upper/diag from X if L != X
  if (a.smem_mode) {
    for (int s = 0; s < ncl; ++s) {
      const int j = cta + s * C;
      if (j >= n) break;
      const double* p = c.local + (size_t)s * n;
      for (int i = j + 1 + tid; i < n; i += kTThreads) a.L[(long long)j * a.ldl + i] = p[i];
    }
  }
}

__global__ void copy_matrix_kernel(const double* __restrict__ X, long long ldx, double* __restrict__ L,
                                   long long ldl, int n) {
  for (int j = blockIdx.y; j < n; j += gridDim.y)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
      L[(long long)j * ldl + i] = X[(long long)j * ldx + i];
}

size_t twostep_smem(int n, int C) {
  size_t head = (((size_t)(2 * n + kTWarps) * 8 + kTWarps * 4 + 16 + 127) & ~size_t(127));
  return head + (size_t)((n + C - 1) / C) * n * sizeof(double);
}

int twostep_cluster() {
  static int cs = -1;
  if (cs < 0) {
    cs = 0;
    for (int c : {16, 8}) {
      cudaFuncSetAttribute(twostep_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(twostep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c);
      cfg.blockDim = dim3(kTThreads);
      cfg.dynamicSmemBytes = 200 * 1024;
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = c;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, twostep_kernel, &cfg) == cudaSuccess && ncl >= 1) {
        cs = c;
        break;
      }
      cudaGetLastError();
    }
  }
  return cs;
}

}  // namespace

size_t twostep_workspace_bytes(int n) { return (size_t)2 * (n > 0 ? n : 1) * sizeof(double) + 256; }

cudaError_t launch_twostep(const double* X, long long ldx, double* L, long long ldl, int n, int pivot, double* tau,
                           long long* piv, int* info, void* workspace, cudaStream_t stream) {
  int C = twostep_cluster();
  if (C == 0) return cudaErrorNotSupported;
  int lim = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&lim, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const bool smem_mode = twostep_smem(n, C) <= (size_t)lim;
  size_t smem = smem_mode ? twostep_smem(n, C) : twostep_smem(n, C) - (size_t)((n + C - 1) / C) * n * sizeof(double);
  if (smem > (size_t)lim) return cudaErrorInvalidValue;  // n too large even for the staged vectors
  cudaError_t e;
  if (L != X || !smem_mode) {
    // the reference returns the work buffer: upper triangle / diagonal are the input's
    if (L != X) {
      dim3 grid((n + 255) / 256 < 8 ? (n + 255) / 256 : 8, n < 4096 ? n : 4096);
      copy_matrix_kernel<<<grid, 256, 0, stream>>>(X, ldx, L, ldl, n);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
  }
  if (n == 1) {
    if (pivot) return cudaMemsetAsync(piv, 0, sizeof(long long), stream);
    return cudaMemsetAsync(info, 0, sizeof(int), stream);
  }
  e = cudaFuncSetAttribute(twostep_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(twostep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  TArgs args{X, ldx, L, ldl, n, pivot, smem_mode ? 1 : 0, tau, piv, info, static_cast<double*>(workspace)};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kTThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = C;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, twostep_kernel, args);
}

}  // namespace skl
