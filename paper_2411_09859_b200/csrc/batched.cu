// Batched pivoted LTL^T + Pfaffian of many independent skew matrices
// (config 4: 8192 x n=256, fp32 and fp64).
//
// Reference path per matrix: pfaffian -> ltlt_blk_piv(x, b=min(256, m))
// (apps.py:12-30, blocked.py:303-363), i.e. one left-looking pivoted panel.
// The B200 kernel factors each matrix with the right-looking Wimmer two-step
// recurrence (unblocked.py:136-171) -- the same pivots and factors in exact
// arithmetic -- inside ONE CTA: the trailing matrix lives in shared memory
// (packed lower columns), the argmax is a warp redux over the column, the
// symmetric interchange and the rank-2 update are CTA-parallel with only
// __syncthreads between phases.  The rank-2 updates are blocked: kKB pairs stay
// pending (their w, l vectors in shared memory, interchanged with the matrix)
// and reach the trailing matrix as one rank-2kKB pass, while the columns
// eliminated in between get them applied on the fly (blocked.py:268-290's
// W = A S + skew rank-2k, per CTA).  The older L columns take their row
// interchanges once, at write-back (apply_row_pivots deferred and composed).
// Columns that do not fit the shared-memory budget (the first columns) live
// in the output L buffer.
// A persistent grid walks the batch; outputs: L ("ones" layout), tau,
// relative pivots, and sign / log|Pf| (overflow-free apps.py:26-30).
#include <cmath>

#include "common.cuh"
#include "internal.h"

namespace skl {
namespace {

#ifndef SKL_BATCHED_THREADS
#define SKL_BATCHED_THREADS 256
#endif
// matrices (CTAs) per SM: measured 8192 x n=256 with 8 pending pairs -- fp64
// 28.9 / 24.9 / 26.8 ms and fp32 21.8 / 18.6 / 16.9 ms for 2 / 3 / 4 per SM
#ifndef SKL_BATCHED_PER_SM
#define SKL_BATCHED_PER_SM_F64 3
#define SKL_BATCHED_PER_SM_F32 4
#else
#define SKL_BATCHED_PER_SM_F64 SKL_BATCHED_PER_SM
#define SKL_BATCHED_PER_SM_F32 SKL_BATCHED_PER_SM
#endif
template <typename T>
constexpr int per_sm() {
  return sizeof(T) == 8 ? SKL_BATCHED_PER_SM_F64 : SKL_BATCHED_PER_SM_F32;
}
#ifndef SKL_BATCHED_KB
#define SKL_BATCHED_KB 8  // fp64 31.5 / 26.4 / 24.9 / 35.5 ms (spills) for 2 / 4 / 8 / 16
#endif
constexpr int kBThreads = SKL_BATCHED_THREADS;
// pending two-step pairs: the trailing matrix receives one rank-2*kKB update
// every kKB pairs; the columns eliminated meanwhile get the pending pairs applied
// on the fly (the blocked two-step of blocked.py:268-290 inside one CTA)
constexpr int kKB = SKL_BATCHED_KB;
constexpr int kBWarps = kBThreads / 32;
constexpr size_t kRedBytes = 2 * kBWarps * (sizeof(double) + sizeof(int));

template <typename T>
struct BCtx {
  T* smem;           // packed columns j >= J0 (rows j+1..n-1)
  T* gl;             // L buffer of this matrix (columns j < J0 live here)
  const int* cofs;   // smem table: offset of column j in packed storage, minus (j+1)
  long long ldl;
  int n, J0;
  __device__ __forceinline__ T* col(int j) const {
    // pointer such that col(j)[i] is element (i, j), valid for i > j
    return j < J0 ? gl + (long long)j * ldl : smem + cofs[j];
  }
};

__device__ __forceinline__ int bwarp_argmax(double av, int idx, bool valid) {
  const unsigned long long bits = valid ? (unsigned long long)__double_as_longlong(av) : 0ull;
  const unsigned hi = valid ? unsigned(bits >> 32) + 1u : 0u;
  const unsigned lo = unsigned(bits);
  const unsigned m1 = __reduce_max_sync(0xffffffffu, hi);
  const bool c1 = valid && hi == m1;
  const unsigned m2 = __reduce_max_sync(0xffffffffu, c1 ? lo : 0u);
  const bool c2 = c1 && lo == m2;
  const unsigned id = __reduce_min_sync(0xffffffffu, c2 ? unsigned(idx) : 0xffffffffu);
  return id == 0xffffffffu ? -1 : int(id);
}

// iamax over X[g+1:, g] (ties -> lowest index).  One barrier: per-warp
// partials in smem, then every warp reduces the partials redundantly.
// `red` holds [2][kBWarps] (double-buffered by column parity).
// pending pairs p < np: column j of the trailing matrix still lacks
// sum_p (pw_p[i] pl_p[j] - pl_p[i] pw_p[j]) (pw/pl hold [kKB][n])
template <typename T>
__device__ __forceinline__ T pending_at(const T* pw, const T* pl, int n, int np, int i, int j) {
  T acc = T(0);
  for (int p = 0; p < np; ++p) acc += pw[p * n + i] * pl[p * n + j] - pl[p * n + i] * pw[p * n + j];
  return acc;
}

template <typename T>
__device__ int col_argmax(const BCtx<T>& c, int g, double* redv, int* redi, const T* pw = nullptr,
                          const T* pl = nullptr, int np = 0) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  T* x = c.col(g);
  double bv = -1.0;
  int bi = -1;
  for (int i = g + 1 + tid; i < c.n; i += kBThreads) {
    if (np > 0) x[i] -= pending_at(pw, pl, c.n, np, i, g);  // column g becomes current
    double v = fabs((double)x[i]);
    if (v > bv) {
      bv = v;
      bi = i;
    }
  }
  const int id = bwarp_argmax(bv, bi, bi >= 0);
  const int slot = (g & 1) * kBWarps;
  if (bi >= 0 && bi == id) {
    redv[slot + warp] = bv;
    redi[slot + warp] = bi;
  }
  if (lane == 0 && id < 0) redi[slot + warp] = -1;
  __syncthreads();
  const int cand = lane < kBWarps ? redi[slot + lane] : -1;
  const double v = cand >= 0 ? redv[slot + lane] : 0.0;
  const int id2 = bwarp_argmax(v, cand, cand >= 0);
  return id2 < 0 ? g + 1 : id2;
}

// Interchange (a = g+1, b) over the whole matrix fused with the elimination
// of column g: L[:, g] = X[:, g] / tau below the unit (tau = X[b, g] before the
// interchange), explicit 1 at [a, g].  Element sets are disjoint, so one pass.
template <typename T>
__device__ void swap_and_eliminate(const BCtx<T>& c, int g, int b, T tau, T* pw, T* pl, int np) {
  const int tid = threadIdx.x, n = c.n;
  const int a = g + 1;
  const bool sw = b != a;
  // P (X - sum w l^T - l w^T) P^T: the pending vectors take the interchange too
  if (sw && tid >= 32 && tid < 32 + 2 * np) {
    T* v = (tid - 32 < np ? pw : pl) + ((tid - 32) % np) * n;
    const T t = v[a];
    v[a] = v[b];
    v[b] = t;
  }
  // column g: finalize
  T* xg = c.col(g);
  {
    const T vb_old_a = xg[a];  // value that moves to row b
    for (int i = a + 1 + tid; i < n; i += kBThreads) {
      T v = (sw && i == b) ? vb_old_a : xg[i];
      xg[i] = tau != T(0) ? v / tau : v;
    }
  }
  if (!sw) return;
  // rows a, b of the older columns: only column g-1 now (the pair's fold reads
  // it); columns j < g-1 get this interchange at write-back (deferred, composed)
  if (tid == 0 && g >= 1) {
    T* p = c.col(g - 1);
    T t = p[a];
    p[a] = p[b];
    p[b] = t;
  }
  T* pa = c.col(a);
  T* pb = c.col(b);
  for (int i = b + 1 + tid; i < n; i += kBThreads) {
    T t = pa[i];
    pa[i] = pb[i];
    pb[i] = t;
  }
  for (int i = a + 1 + tid; i < b; i += kBThreads) {
    T* pi = c.col(i);
    T t = pi[b];
    T u = pa[i];
    pa[i] = -t;
    pi[b] = -u;
  }
  if (tid == 0) pa[b] = -pa[b];
}

#ifdef SKL_BATCHED_PROF
__device__ unsigned long long g_bprof[8];
}  // namespace
}  // namespace skl
extern "C" int skl_debug_read_bprof(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, skl::g_bprof, sizeof(unsigned long long) * 8);
}
namespace skl {
namespace {
#define BMARK(i)                                                         \
  do {                                                                   \
    long long _t = clock64();                                            \
    if (threadIdx.x == 0 && blockIdx.x == 0) bpt[i] += _t - bprev;       \
    bprev = _t;                                                          \
  } while (0)
#else
#define BMARK(i) \
  do {           \
  } while (0)
#endif

template <typename T>
__global__ void __launch_bounds__(kBThreads, per_sm<T>())
batched_kernel(int batch, int n, int J0, const T* __restrict__ X, long long ldx, long long strideX, T* __restrict__ L,
               long long ldl, long long strideL, T* __restrict__ tau, long long strideTau, long long* __restrict__ piv,
               long long stridePiv, double* __restrict__ pf_sign, double* __restrict__ pf_logabs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* redv = reinterpret_cast<double*>(smem_raw);  // [2][kBWarps] argmax partials
  int* redi = reinterpret_cast<int*>(redv + 2 * kBWarps);
  T* vec = reinterpret_cast<T*>(smem_raw + kRedBytes);  // [n] write-back staging
  T* pw = vec + n;                                       // [kKB][n] pending w vectors
  T* pl = pw + kKB * n;                                  // [kKB][n] pending l vectors
  int* cofs = reinterpret_cast<int*>(pl + kKB * n);      // [n] column offsets
  int* qmap = cofs + n;                                  // [n] write-back position map
  int* pvs = qmap + n;                                   // [n] relative pivots of this matrix
  T* store = reinterpret_cast<T*>(smem_raw + ((kRedBytes + (1 + 2 * kKB) * n * sizeof(T) + 3 * n * sizeof(int) + 15) &
                                               ~size_t(15)));
  const int tid = threadIdx.x;
  for (int j = tid; j < n; j += kBThreads) {
    // offset of column j >= J0: sum_{c=J0}^{j-1} (n-1-c), minus (j+1) so col(j)[i] indexes row i
    const long long off = (long long)(j - J0) * (n - 1) - ((long long)j * (j - 1) - (long long)J0 * (J0 - 1)) / 2;
    cofs[j] = j >= J0 ? int(off - (j + 1)) : 0;
  }
  __syncthreads();

  for (int m = blockIdx.x; m < batch; m += gridDim.x) {
    const T* x = X + (long long)m * strideX;
    T* l = L + (long long)m * strideL;
    T* tm = tau + (long long)m * strideTau;
    long long* pm = piv + (long long)m * stridePiv;
    BCtx<T> c{store, l, cofs, ldl, n, J0};
    // load (one flattened, coalesced pass): strictly-lower columns j >= J0 go
    // to shared memory, everything else (upper/diag, columns j < J0) to L
    {
      const int nn = n * n;
#pragma unroll 4
      for (int e = tid; e < nn; e += kBThreads) {
        const int j = e / n, i = e - j * n;
        const T v = x[(long long)j * ldx + i];
        if (i > j && j >= J0)
          c.col(j)[i] = v;
        else
          l[(long long)j * ldl + i] = v;
      }
    }
    if (tid == 0) {
      pm[0] = 0;
      pvs[0] = 0;
    }
    __syncthreads();

    int nswaps = 0;
    double logabs = 0.0, sgn = 1.0;
    const int end = n - 1;
    int g = 0;
#ifdef SKL_BATCHED_PROF
    long long bpt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long bprev = clock64();
#endif
    int np = 0;  // pending two-step pairs (rows/cols >= their s0 = g_p + 3)
    while (g < end) {
      // ---- eliminate(g): argmax, interchange + scale in one pass -------------
      // (column g is current: it was the previous pair's fold column)
      BMARK(7);
      int b = col_argmax(c, g, redv, redi);
      const T t0 = c.col(g)[b];  // becomes X[g+1, g] after the interchange
      __syncthreads();            // every warp has read the partials and tau
      BMARK(0);
      swap_and_eliminate(c, g, b, t0, pw, pl, np);
      if (tid == 0) {
        pm[g + 1] = b - (g + 1);
        pvs[g + 1] = b - (g + 1);
        nswaps += b != g + 1;
        tm[g] = t0;
        if ((g & 1) == 0) {  // Pf = sign(P) prod_{i even} (-tau_i)
          logabs += log(fabs((double)t0));
          sgn *= (t0 > T(0)) ? -1.0 : (t0 < T(0) ? 1.0 : 0.0);
        }
      }
      __syncthreads();
      BMARK(1);
      if (tid == 0) c.col(g)[g + 1] = T(1);
      if (g + 1 >= end) {
        __syncthreads();
        g += 1;
        break;
      }
      // ---- eliminate(g+1): the pending pairs are applied to column g+1 first --
      b = col_argmax(c, g + 1, redv, redi, pw, pl, np);
      const T t1 = c.col(g + 1)[b];
      __syncthreads();
      BMARK(2);
      swap_and_eliminate(c, g + 1, b, t1, pw, pl, np);
      if (tid == 0) {
        pm[g + 2] = b - (g + 2);
        pvs[g + 2] = b - (g + 2);
        nswaps += b != g + 2;
        tm[g + 1] = t1;
      }
      __syncthreads();
      BMARK(3);
      // ---- column g+2: pending pairs, then fold the first coupling; this pair's
      // rank-2 vectors become pending entry np -----------------------------------
      const int s0 = g + 3;
      T* xg = c.col(g);
      T* x1 = c.col(g + 1);
      T* x2 = c.col(g + 2);
      const T x20 = xg[g + 2];
      for (int i = s0 + tid; i < n; i += kBThreads) {
        const T l2 = x1[i];
        const T l1i = xg[i];
        const T x2i = np > 0 ? x2[i] - pending_at(pw, pl, n, np, i, g + 2) : x2[i];
        const T f = x2i - t1 * (x20 * l2 - l1i);
        x2[i] = f;
        pw[np * n + i] = f - t1 * l1i;  // wv
        pl[np * n + i] = l2;
      }
      ++np;
      __syncthreads();
      BMARK(4);
      if (tid == 0) x1[g + 2] = T(1);
      // ---- every kKB pairs: X[s:, s:] -= sum_p (w_p l_p^T - l_p w_p^T) ---------
      if (np == kKB) {
        // thread <-> row i (coalesced in every column; the pending row values in
        // registers), columns j in [s0, i) walked in lockstep (broadcast reads of
        // w_p[j], l_p[j]); loads of consecutive columns are independent
        for (int i = s0 + 1 + tid; i < n; i += kBThreads) {  // empty once s0 >= n - 1
          T wi[kKB], li[kKB];
#pragma unroll
          for (int p = 0; p < kKB; ++p) {
            wi[p] = pw[p * n + i];
            li[p] = pl[p * n + i];
          }
          int j = s0;
          for (; j + 1 < i; j += 2) {
            T* c0 = c.col(j);
            T* c1 = c.col(j + 1);
            T v0 = c0[i], v1 = c1[i];
#pragma unroll
            for (int p = 0; p < kKB; ++p) {
              v0 -= wi[p] * pl[p * n + j] - li[p] * pw[p * n + j];
              v1 -= wi[p] * pl[p * n + j + 1] - li[p] * pw[p * n + j + 1];
            }
            c0[i] = v0;
            c1[i] = v1;
          }
          if (j < i) {
            T* c0 = c.col(j);
            T v0 = c0[i];
#pragma unroll
            for (int p = 0; p < kKB; ++p) v0 -= wi[p] * pl[p * n + j] - li[p] * pw[p * n + j];
            c0[i] = v0;
          }
        }
        np = 0;
      }
      __syncthreads();
      BMARK(5);
      g += 2;
    }
#ifdef SKL_BATCHED_PROF
    if (tid == 0 && blockIdx.x == 0)
      for (int i = 0; i < 8; ++i) atomicAdd(&g_bprof[i], (unsigned long long)bpt[i]);
#endif
    if (tid == 0) {
      if (n % 2 == 1) {
        if (pf_sign) pf_sign[m] = 0.0;
        if (pf_logabs) pf_logabs[m] = -INFINITY;
      } else {
        if (nswaps & 1) sgn = -sgn;
        if (pf_sign) pf_sign[m] = sgn;
        if (pf_logabs) pf_logabs[m] = sgn == 0.0 ? -INFINITY : logabs;
      }
    }
    // write-back.  Column j still lacks the row interchanges of steps >= j+2
    // (swap_and_eliminate applies only step j+1's to it); walking j downwards,
    // qmap = s_{n-2} o ... o s_{j+2} maps a stored position to its final row
    // (the deferred row gather of apply_row_pivots, kernels2.py:232-271).
    // Row j+1 (the explicit 1) and rows <= j are fixed by every later swap.
    for (int i = tid; i < n; i += kBThreads) qmap[i] = i;
    __syncthreads();
    for (int j = n - 2; j >= 0; --j) {
      if (tid == 0 && j + 2 <= n - 2) {
        const int a = j + 3, bb = j + 3 + pvs[j + 3];  // s_{j+2} swaps positions j+3 and its pivot row
        const int t = qmap[a];
        qmap[a] = qmap[bb];
        qmap[bb] = t;
      }
      const T* cj = c.col(j);
      // read the whole column, then scatter (columns j < J0 live in l itself)
      for (int i = j + 1 + tid; i < n; i += kBThreads) vec[i] = cj[i];
      __syncthreads();
      for (int i = j + 1 + tid; i < n; i += kBThreads) l[(long long)j * ldl + qmap[i]] = vec[i];
      __syncthreads();
    }
  }
}

template <typename T>
size_t batched_smem(int n, int J0) {
  size_t head = (kRedBytes + (1 + 2 * kKB) * n * sizeof(T) + 3 * n * sizeof(int) + 15) & ~size_t(15);
  long long cols = 0;
  for (int j = J0; j < n - 1; ++j) cols += n - 1 - j;
  return head + (size_t)cols * sizeof(T);
}

}  // namespace

template <typename T>
cudaError_t launch_batched(int batch, int n, const T* X, long long ldx, long long strideX, T* L, long long ldl,
                           long long strideL, T* tau, long long strideTau, long long* piv, long long stridePiv,
                           double* pf_sign, double* pf_logabs, cudaStream_t stream) {
  int dev = 0, lim = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&lim, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // per_sm<T>() matrices share an SM (each CTA gets 1/k of the shared memory)
  constexpr int kPerSm = per_sm<T>();
  const size_t budget = kPerSm == 1 ? (size_t)lim : (size_t)(228 * 1024) / kPerSm - 1024;
  int J0 = 0;
  while (J0 < n - 1 && batched_smem<T>(n, J0) > budget) ++J0;
  size_t smem = batched_smem<T>(n, J0);
  cudaError_t e = cudaFuncSetAttribute(batched_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  long long g = (long long)nsm * kPerSm;
  int grid = batch < g ? batch : (int)g;
  batched_kernel<T><<<grid, kBThreads, smem, stream>>>(batch, n, J0, X, ldx, strideX, L, ldl, strideL, tau, strideTau,
                                                       piv, stridePiv, pf_sign, pf_logabs);
  return cudaGetLastError();
}

template cudaError_t launch_batched<double>(int, int, const double*, long long, long long, double*, long long,
                                            long long, double*, long long, long long*, long long, double*, double*,
                                            cudaStream_t);
template cudaError_t launch_batched<float>(int, int, const float*, long long, long long, float*, long long, long long,
                                           float*, long long, long long*, long long, double*, double*, cudaStream_t);

}  // namespace skl
