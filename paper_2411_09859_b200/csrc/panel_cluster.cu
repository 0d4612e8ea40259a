// Pivoted left-looking panel on ONE thread-block cluster (16 CTAs).
//
// Same reference semantics as panel.cu (_panel_ll unblocked.py:94-119,
// _eliminate unblocked.py:63-91, _sym_swap_lower core.py:294-324), but the
// per-step argmax exchange runs through distributed shared memory and the
// hardware cluster barrier instead of global-memory flags: a grid-wide
// exchange over 148 SMs measured ~2 us per round on B200, a cluster barrier
// is a few hundred cycles.  Each elimination step is
//   v = c - A z (A z precomputed while the column gather was in flight)
//   -> CTA argmax -> candidate pushed into every CTA's smem (st.shared::cluster)
//   -> barrier.cluster (release/acquire) -> every warp reduces 16 candidates
//   -> winner row read from its owner's smem (ld.shared::cluster), next
//      column gathered from the pre-panel matrix (lazy symmetric swaps)
//   -> local row interchange + scale -> A z for the next column.
// The panel block lives in shared memory across the 16 CTAs; the driver
// narrows the panel when it would not fit (the factorization is invariant to
// the GPU block width; pivots stay those of the reference).
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace skl {
namespace {

constexpr int kCThreads = 256;
constexpr int kBank = 32;  // register-cached slab columns per bank (2 banks, rows li = tid only)
constexpr int kCWarps = kCThreads / 32;
constexpr int kClusterMax = 16;

struct __align__(16) CCand {
  double v;
  int idx;
  int perm;
};

__device__ __forceinline__ bool cbetter(double av, int ai, double bv, int bi) {
  if (ai < 0) return false;
  if (bi < 0) return true;
  double aa = fabs(av), bb = fabs(bv);
  return aa > bb || (aa == bb && ai < bi);
}

__device__ __forceinline__ void cwarp_argmax(CCand& c, int& owner) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, c.v, o);
    int oi = __shfl_xor_sync(0xffffffffu, c.idx, o);
    int op = __shfl_xor_sync(0xffffffffu, c.perm, o);
    int ow = __shfl_xor_sync(0xffffffffu, owner, o);
    if (cbetter(ov, oi, c.v, c.idx)) {
      c.v = ov;
      c.idx = oi;
      c.perm = op;
      owner = ow;
    }
  }
}

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Exact warp argmax of |v| with ties to the lowest index, using three
// redux.sync reductions on the bit pattern of |v| (monotone for v >= 0)
// instead of a 5-round shuffle tree.  Returns the winning index or -1.
__device__ __forceinline__ int warp_argmax_redux(double v, int idx, bool valid) {
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

struct CSmem {
  double* slab;    // [kmax][Rs]
  double* wrow;    // winner row (pivot row of the next step)   [kmax+2]
  double* arow;    // displaced row a                           [kmax+2]
  double* taus;    // taus[j] = tau[lo+j]                       [kmax+2]
  double* zbuf;    // z = T x                                    [kmax+2]
  double* pubrow;  // [2][kmax+2] own candidate row, read remotely
  double* pubA;    // [2][kmax+2] row a (if owned), read remotely
  double* part;    // gemv partials [kCThreads]
  double* az;      // A z for the next column [Rs]
  double* ycol;    // [Rs]
  int* perm;       // [Rs]
  CCand* cand;     // [2][kClusterMax] written by every CTA of the cluster
  CCand* wcand;    // [kCWarps]
  int* misc;       // [0..1] pubA perm per parity, [2] local cand idx
  int* pivbuf;     // [nelim] pivot offsets of this panel (flushed at the end)
};

__host__ __device__ inline int cslab_stride(int rows_per) { return rows_per | 1; }

__host__ __device__ inline size_t csmem_layout(int R, int kmax, CSmem* s, unsigned char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 15) & ~size_t(15);
    return base ? base + o : nullptr;
  };
  const int Rs = cslab_stride(R);
  const size_t kv = sizeof(double) * (kmax + 2);
  unsigned char* p;
  p = take(sizeof(double) * (size_t)kmax * Rs);
  if (s) s->slab = (double*)p;
  p = take(kv);
  if (s) s->wrow = (double*)p;
  p = take(kv);
  if (s) s->arow = (double*)p;
  p = take(kv);
  if (s) s->taus = (double*)p;
  p = take(kv);
  if (s) s->zbuf = (double*)p;
  p = take(2 * kv);
  if (s) s->pubrow = (double*)p;
  p = take(2 * kv);
  if (s) s->pubA = (double*)p;
  p = take(sizeof(double) * kCThreads);
  if (s) s->part = (double*)p;
  p = take(sizeof(double) * Rs);
  if (s) s->az = (double*)p;
  p = take(sizeof(double) * Rs);
  if (s) s->ycol = (double*)p;
  p = take(sizeof(int) * Rs);
  if (s) s->perm = (int*)p;
  p = take(sizeof(CCand) * 2 * kClusterMax);
  if (s) s->cand = (CCand*)p;
  p = take(sizeof(CCand) * kCWarps);
  if (s) s->wcand = (CCand*)p;
  p = take(sizeof(int) * 8);
  if (s) s->misc = (int*)p;
  p = take(sizeof(int) * (kmax + 2));
  if (s) s->pivbuf = (int*)p;
  return off;
}

// az[li] = sum_{j<k} slab[j][li] z_j for local rows li >= l0 (G groups split k)
__device__ __forceinline__ void compute_az(const CSmem& s, int Rs, int R, int rcount, int G, int k, int l0,
                                           int tid) {
  if (k < 2) {
    for (int li = tid; li < rcount; li += kCThreads) s.az[li] = 0.0;
    return;
  }
  if (G > 1) {
    if (tid < G * R) {
      const int gi = tid / R, li = tid - gi * R;
      if (li >= l0 && li < rcount) {
        const int kc = (k + G - 1) / G;
        const int j0 = gi * kc, j1 = min(k, j0 + kc);
        double a0 = 0.0, a1 = 0.0;
        int j = j0;
        for (; j + 1 < j1; j += 2) {
          a0 = fma(s.slab[(size_t)j * Rs + li], s.zbuf[j], a0);
          a1 = fma(s.slab[(size_t)(j + 1) * Rs + li], s.zbuf[j + 1], a1);
        }
        if (j < j1) a0 = fma(s.slab[(size_t)j * Rs + li], s.zbuf[j], a0);
        s.part[gi * R + li] = a0 + a1;
      }
    }
    __syncthreads();
    for (int li = l0 + tid; li < rcount; li += kCThreads) {
      double acc = 0.0;
      for (int gi = 0; gi < G; ++gi) acc += s.part[gi * R + li];
      s.az[li] = acc;
    }
  } else {
    for (int li = l0 + tid; li < rcount; li += kCThreads) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int j = 0;
      for (; j + 3 < k; j += 4) {
        a0 = fma(s.slab[(size_t)j * Rs + li], s.zbuf[j], a0);
        a1 = fma(s.slab[(size_t)(j + 1) * Rs + li], s.zbuf[j + 1], a1);
        a2 = fma(s.slab[(size_t)(j + 2) * Rs + li], s.zbuf[j + 2], a2);
        a3 = fma(s.slab[(size_t)(j + 3) * Rs + li], s.zbuf[j + 3], a3);
      }
      for (; j < k; ++j) a0 = fma(s.slab[(size_t)j * Rs + li], s.zbuf[j], a0);
      s.az[li] = (a0 + a1) + (a2 + a3);
    }
  }
}

__global__ void __launch_bounds__(kCThreads, 1) panel_cluster_kernel(PanelArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const int C = gridDim.x, cta = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n, lo = a.lo, r = a.r, nelim = a.nelim, kmax = a.kmax;
  const int R = a.rows_per, Rs = cslab_stride(R);
  const int G = R <= kCThreads ? max(1, min(kCThreads / max(R, 1), 16)) : 1;
  const long long ld = a.ld;
  double* __restrict__ W = a.W;
  const int row0 = lo + 1;
  const int rbase = row0 + cta * R;
  const int rcount = max(0, min(R, n - rbase));
  const int rt = r + nelim;

  CSmem s;
  csmem_layout(R, kmax, &s, smem_raw);

  for (int li = tid; li < rcount; li += kCThreads) {
    s.perm[li] = rbase + li;
    s.az[li] = 0.0;
  }
  if (lo < r) {
    for (int li = tid; li < rcount; li += kCThreads) s.slab[li] = W[(long long)lo * ld + rbase + li];
  }
  for (int j = tid; j < kmax + 2; j += kCThreads) {
    s.taus[j] = (j == 0 && lo >= 0 && lo < n - 1) ? a.tau[lo] : 0.0;
    s.wrow[j] = 0.0;
    s.zbuf[j] = 0.0;
  }
  {
    double* col = s.slab + (size_t)(r - lo) * Rs;
    for (int li = tid; li < rcount; li += kCThreads) {
      int pos = rbase + li;
      col[li] = pos > r ? W[(long long)r * ld + pos] : 0.0;
    }
  }
  cluster_barrier();
  long long pt[6] = {0, 0, 0, 0, 0, 0};
  long long t_prev = clock64();
#define CMARK(i)                    \
  do {                              \
    long long _t = clock64();       \
    pt[i] += _t - t_prev;           \
    t_prev = _t;                    \
  } while (0)

  // register cache of slab columns [0, kBank*nbank) for row li = tid (the gemv re-reads
  // the slab every step; shared-memory bandwidth is its bound otherwise)
  double rb[2][kBank];
  int nbank = 0;
  // per-thread rows: li = tid + u * kCThreads (R <= 2 * kCThreads)
  double cnext[2] = {0.0, 0.0};
  bool cneg[2] = {false, false};  // gathered from the row part: negate at use (keeps the load in flight)
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int li = tid + u * kCThreads;
    if (li < rcount) cnext[u] = s.slab[(size_t)(r - lo) * Rs + li];
  }
  __syncthreads();

  for (int g = r; g < rt; ++g) {
    const int k = g - lo;
    const int par = g & 1;
    double* col = s.slab + (size_t)k * Rs;
    const int a_pos = g + 1;
    const int owner_a = (a_pos - row0) / R;
    const bool own_a = owner_a == cta;

    // ---- (1) v = c - A z; per-warp argmax -----------------------------------
    double vbest = 0.0;
    int ibest = -1;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int li = tid + u * kCThreads;
      const int pos = rbase + li;
      if (li < rcount && pos > g) {
        const double v = (cneg[u] ? -cnext[u] : cnext[u]) - s.az[li];
        col[li] = v;
        if (ibest < 0 || fabs(v) > fabs(vbest)) {
          vbest = v;
          ibest = pos;
        }
      }
    }
    {
      const int id = warp_argmax_redux(vbest, ibest, ibest >= 0);
      if (ibest >= 0 && ibest == id) s.wcand[warp] = CCand{vbest, ibest, 0};
      if (lane == 0 && id < 0) s.wcand[warp] = CCand{0.0, -1, 0};
    }
    CMARK(0);
    __syncthreads();

    // ---- (2) CTA candidate -> every CTA of the cluster; publish rows ------------
    if (warp == 0) {
      const bool ok = lane < kCWarps && s.wcand[lane].idx >= 0;
      const CCand mine = lane < kCWarps ? s.wcand[lane] : CCand{0.0, -1, 0};
      const int id = warp_argmax_redux(mine.v, mine.idx, ok);
      const unsigned bal = __ballot_sync(0xffffffffu, ok && mine.idx == id);
      CCand c = CCand{0.0, -1, -1};
      if (id >= 0) {
        c = s.wcand[__ffs(bal) - 1];
        c.perm = s.perm[c.idx - rbase];
        const int lc = c.idx - rbase;
        double* pr = s.pubrow + par * (kmax + 2);
        for (int j = lane; j <= k; j += 32) pr[j] = s.slab[(size_t)j * Rs + lc];
      }
      __syncwarp();
      if (lane < C) *cluster.map_shared_rank(s.cand + par * kClusterMax + cta, lane) = c;
    } else if (warp == 1 && own_a) {
      const int la = a_pos - rbase;
      double* pa = s.pubA + par * (kmax + 2);
      for (int j = lane; j <= k; j += 32) pa[j] = s.slab[(size_t)j * Rs + la];
      if (lane == 0) s.misc[par] = s.perm[la];
    }
    CMARK(1);
    cluster_barrier();
    CMARK(2);

    // ---- (3) winner, next-column gather, winner row / row a via DSMEM ---------
    int owner;
    CCand w;
    {
      const bool ok = lane < C && s.cand[par * kClusterMax + lane].idx >= 0;
      const CCand mine = lane < C ? s.cand[par * kClusterMax + lane] : CCand{0.0, -1, -1};
      const int id = warp_argmax_redux(mine.v, mine.idx, ok);
      owner = __ffs(__ballot_sync(0xffffffffu, ok && mine.idx == id)) - 1;
      w = s.cand[par * kClusterMax + owner];
    }
    const int b = w.idx, pb = w.perm;
    const double vb = w.v;
    const bool own_b = b >= rbase && b < rbase + rcount;
    const bool swapped = b != a_pos;
    const bool more = (g + 1 < rt) || a.want_y;
    int perm_a = 0;
    if (own_b && swapped) perm_a = *cluster.map_shared_rank(s.misc + par, owner_a);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int li = tid + u * kCThreads;
      const int pos = rbase + li;
      cnext[u] = 0.0;
      cneg[u] = false;
      if (more && li < rcount && pos > a_pos) {
        const int ph = (swapped && pos == b) ? perm_a : s.perm[li];
        // X(ph, pb) in skew-lower storage; the sign is applied when consumed
        cneg[u] = ph < pb;
        cnext[u] = cneg[u] ? W[(long long)ph * ld + pb] : W[(long long)pb * ld + ph];
      }
    }
    {
      const double* wr = cluster.map_shared_rank(s.pubrow + par * (kmax + 2), owner);
      for (int j = tid; j <= k; j += kCThreads) s.wrow[j] = wr[j];
      if (own_b && swapped) {
        const double* ar = cluster.map_shared_rank(s.pubA + par * (kmax + 2), owner_a);
        for (int j = tid; j <= k; j += kCThreads) s.arow[j] = ar[j];
      }
    }
    __syncthreads();
    CMARK(3);

    // ---- (4) interchange rows a/b, scale column k, z for the next step -------
    if (swapped) {
      if (own_a) {
        const int la = a_pos - rbase;
        for (int j = tid; j < k; j += kCThreads) s.slab[(size_t)j * Rs + la] = s.wrow[j];
        if (tid == la && nbank > 0) {
#pragma unroll
          for (int q = 0; q < kBank; ++q) rb[0][q] = s.wrow[q];
          if (nbank > 1) {
#pragma unroll
            for (int q = 0; q < kBank; ++q) rb[1][q] = s.wrow[kBank + q];
          }
        }
      }
      if (own_b) {
        const int lb = b - rbase;
        for (int j = tid; j < k; j += kCThreads) s.slab[(size_t)j * Rs + lb] = s.arow[j];
        if (tid == lb && nbank > 0) {
#pragma unroll
          for (int q = 0; q < kBank; ++q) rb[0][q] = s.arow[q];
          if (nbank > 1) {
#pragma unroll
            for (int q = 0; q < kBank; ++q) rb[1][q] = s.arow[kBank + q];
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int li = tid + u * kCThreads;
      if (li < rcount) {
        const int pos = rbase + li;
        if (pos == a_pos) {
          col[li] = 1.0;
          if (swapped) s.perm[li] = pb;
        } else if (pos > a_pos) {
          const bool isb = swapped && pos == b;
          const double v = isb ? s.arow[k] : col[li];
          col[li] = vb != 0.0 ? v / vb : v;
          if (isb) s.perm[li] = perm_a;
        }
      }
    }
    for (int j = tid; j <= k; j += kCThreads) {
      const double xm = j >= 1 ? s.wrow[j - 1] : 0.0;
      const double xp = (j + 1 < k) ? s.wrow[j + 1] : (j + 1 == k ? 1.0 : 0.0);
      const double tj = j == k ? vb : s.taus[j];
      const double tj1 = (j + 1 == k) ? vb : s.taus[j + 1];
      s.zbuf[j] = (j >= 1 ? tj * xm : 0.0) - (j + 1 <= k ? tj1 * xp : 0.0);
    }
    if (tid == 0) s.pivbuf[g - r] = b - a_pos;  // tau is kept in s.taus
    __syncthreads();
    if (tid == 0) {
      s.taus[k] = vb;
      s.wrow[k] = 1.0;
    }
    CMARK(5);

    // ---- (5) A z for the next column, one thread per row (overlaps the gather) --
    if (more) {
      const int kk = k + 1;
      // columns [kBank*m, kBank*(m+1)) are final once the next column is kk >= kBank*(m+1)
      if (nbank < 2 && kk >= kBank * (nbank + 1) && tid < rcount) {
        if (nbank == 0) {
#pragma unroll
          for (int q = 0; q < kBank; ++q) rb[0][q] = s.slab[(size_t)q * Rs + tid];
        } else {
#pragma unroll
          for (int q = 0; q < kBank; ++q) rb[1][q] = s.slab[(size_t)(kBank + q) * Rs + tid];
        }
      }
      if (nbank < 2 && kk >= kBank * (nbank + 1)) ++nbank;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int li = tid + u * kCThreads;
        if (li < rcount && rbase + li > a_pos) {
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          int j = 0;
          if (u == 0 && nbank > 0) {
            const double2* z2 = reinterpret_cast<const double2*>(s.zbuf);
#pragma unroll
            for (int q = 0; q < kBank; q += 4) {
              const double2 za = z2[q >> 1], zb = z2[(q >> 1) + 1];
              a0 = fma(rb[0][q], za.x, a0);
              a1 = fma(rb[0][q + 1], za.y, a1);
              a2 = fma(rb[0][q + 2], zb.x, a2);
              a3 = fma(rb[0][q + 3], zb.y, a3);
            }
            if (nbank > 1) {
#pragma unroll
              for (int q = 0; q < kBank; q += 4) {
                const double2 za = z2[(kBank + q) >> 1], zb = z2[((kBank + q) >> 1) + 1];
                a0 = fma(rb[1][q], za.x, a0);
                a1 = fma(rb[1][q + 1], za.y, a1);
                a2 = fma(rb[1][q + 2], zb.x, a2);
                a3 = fma(rb[1][q + 3], zb.y, a3);
              }
            }
            j = kBank * nbank;
          }
          for (; j + 3 < kk; j += 4) {
            a0 = fma(s.slab[(size_t)j * Rs + li], s.zbuf[j], a0);
            a1 = fma(s.slab[(size_t)(j + 1) * Rs + li], s.zbuf[j + 1], a1);
            a2 = fma(s.slab[(size_t)(j + 2) * Rs + li], s.zbuf[j + 2], a2);
            a3 = fma(s.slab[(size_t)(j + 3) * Rs + li], s.zbuf[j + 3], a3);
          }
          for (; j < kk; ++j) a0 = fma(s.slab[(size_t)j * Rs + li], s.zbuf[j], a0);
          s.az[li] = kk >= 2 ? (a0 + a1) + (a2 + a3) : 0.0;
        }
      }
    }
    CMARK(4);
  }
  __syncthreads();
  if (cta == 0) {
    for (int g = r + tid; g < rt; g += kCThreads) {
      a.tau[g] = s.taus[g - lo];
      a.piv[g + 1] = (long long)s.pivbuf[g - r];
    }
  }
  if (a.prof && tid == 0) {
    for (int i = 0; i < 6; ++i) a.prof[cta * 8 + i] += (unsigned long long)pt[i];
    a.prof[cta * 8 + 6] += (unsigned long long)(rt - r);
  }
  if (a.want_y) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int li = tid + u * kCThreads;
      if (li < rcount) s.ycol[li] = cneg[u] ? -cnext[u] : cnext[u];
    }
  }
  __syncthreads();

  // ---- var1: y = column rt after the couplings (straggler operand) --------
  if (a.want_y && rt < n) {
    const int l0 = max(0, rt + 1 - rbase);
    for (int li = l0 + tid; li < rcount; li += kCThreads) a.y[rbase + li] = s.ycol[li] - s.az[li];
  }

  // ---- materialise displaced trailing lines, write back ------------------
  for (int li = tid; li < rcount; li += kCThreads) {
    int pos = rbase + li, ph = s.perm[li];
    a.gperm[pos] = ph;
    if (pos >= rt && ph != pos) {
      int q = atomicAdd(a.disp_count, 1);
      a.disp_list[q] = pos;
    }
  }
  if (cta == 0) {
    for (int i = tid; i < row0; i += kCThreads) a.gperm[i] = i;
  }
  __threadfence();
  cluster_barrier();
  const int nd = *((volatile int*)a.disp_count);
  const int ntr = n - rt;
  for (int q = cta; q < nd; q += C) {
    const int p = a.disp_list[q];
    const int pp = a.gperm[p];
    double* line = a.side + (size_t)q * ntr;
    for (int i = rt + tid; i < n; i += kCThreads) line[i - rt] = (i == p) ? 0.0 : skew_at(W, ld, a.gperm[i], pp);
  }
  __threadfence();
  cluster_barrier();
  for (int j = 0; j < kmax; ++j) {
    const int c = lo + j;
    const double* sc = s.slab + (size_t)j * Rs;
    for (int li = tid; li < rcount; li += kCThreads) {
      int pos = rbase + li;
      if (pos > c) W[(long long)c * ld + pos] = sc[li];
    }
  }
  for (int q = cta; q < nd; q += C) {
    const int p = a.disp_list[q];
    const double* line = a.side + (size_t)q * ntr;
    for (int i = rt + tid; i < n; i += kCThreads) {
      double v = line[i - rt];
      if (i > p)
        W[(long long)p * ld + i] = v;
      else if (i < p)
        W[(long long)i * ld + p] = -v;
    }
  }
}

}  // namespace

size_t panel_cluster_smem_bytes(int rows_per, int kmax) { return csmem_layout(rows_per, kmax, nullptr, nullptr); }

int panel_cluster_size() {
  static int cs = -1;
  if (cs < 0) {
    cs = 0;
    for (int c : {16, 8}) {
      cudaFuncSetAttribute(panel_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c);
      cfg.blockDim = dim3(kCThreads);
      cfg.dynamicSmemBytes = 200 * 1024;
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = c;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, panel_cluster_kernel, &cfg) == cudaSuccess && ncl >= 1) {
        cs = c;
        break;
      }
      cudaGetLastError();
    }
  }
  return cs;
}

cudaError_t launch_panel_cluster(const PanelArgs& a, cudaStream_t stream) {
  const int C = a.nblocks;
  size_t smem = csmem_layout(a.rows_per, a.kmax, nullptr, nullptr);
  cudaError_t e = cudaFuncSetAttribute(panel_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(a.disp_count, 0, sizeof(int), stream);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kCThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = C;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, panel_cluster_kernel, a);
}

}  // namespace skl
