// Pivoted left-looking panel of the blocked LTL^T factorization.
//
// Reference semantics (restated, not ported):
//   _panel_ll        unblocked.py:94-119   column g += -A (T x), x = row g of A
//   skew_tridiag_gemv kernels2.py:178-229  (T x formed in O(k), then a gemv)
//   _eliminate        unblocked.py:63-91   iamax (ties -> lowest index), record
//                                          offset, symmetric swap, tau, scale,
//                                          explicit unit at [g+1, g]
//   _sym_swap_lower   core.py:294-324
//   _block_pivots     blocked.py:293-300   (deferred here, see finalize_l)
//
// B200 design.  One cooperative launch per panel, one CTA per SM.  The rows
// [lo+1, n) of the panel block ("slab": columns lo..r+nelim-1) are split into
// contiguous chunks, one per CTA, and live in shared memory for the whole
// panel, so the per-step left-looking gemv never touches HBM.  The trailing
// matrix is NOT swapped eagerly: a position->physical map `perm` is kept and
// the next column is gathered straight from the pre-panel matrix
// (X_cur[i, g] = X0[perm[i], perm[g]], read through the skew-lower rule).
// Each elimination step is one all-to-all exchange of per-CTA argmax
// candidates in LL (flag-in-word) format plus a read of the winning row, so
// a step costs ~2 L2 round trips instead of a grid barrier + reductions.
// At panel end the displaced trailing lines are materialised (gather into a
// side buffer, grid sync, scatter), which equals applying all the panel's
// symmetric swaps to the trailing matrix; older L columns get their row
// pivots once, at the very end (finalize_l), which equals the reference's
// per-panel apply_row_pivots (kernels2.py:232-271) composed.
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace skl {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxZ = 16;  // z register slots per lane -> kmax <= 512

#ifdef SKL_PANEL_PROFILE
__device__ unsigned long long g_panel_prof[2][16];
__device__ unsigned long long g_panel_ts[8][160][4];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TS_MARK(slot)                                                               \
  do {                                                                              \
    if (tid == 0 && r == 0 && g >= 100 && g < 108 && cta < 160) g_panel_ts[g - 100][cta][slot] = gtime(); \
  } while (0)
#define PROF_MARK(ph)                                                        \
  do {                                                                       \
    if (tid == 0 && (cta == 0 || cta == P - 1)) {                            \
      long long _t = clock64();                                              \
      atomicAdd(&g_panel_prof[cta == 0 ? 0 : 1][ph], (unsigned long long)(_t - _pt)); \
      _pt = _t;                                                              \
    }                                                                        \
  } while (0)
#else
#define TS_MARK(slot) \
  do {                \
  } while (0)
#define PROF_MARK(ph) \
  do {                \
  } while (0)
#endif

struct __align__(16) Cand {
  double v;
  int idx;
  int perm;
};

__device__ __forceinline__ bool better(double av, int ai, double bv, int bi) {
  // larger |v| wins; ties -> lower position; idx < 0 means "no candidate"
  if (ai < 0) return false;
  if (bi < 0) return true;
  double aa = fabs(av), bb = fabs(bv);
  return aa > bb || (aa == bb && ai < bi);
}

__device__ __forceinline__ void warp_argmax(double& v, int& idx, int& perm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    int op = __shfl_xor_sync(0xffffffffu, perm, o);
    if (better(ov, oi, v, idx)) {
      v = ov;
      idx = oi;
      perm = op;
    }
  }
}

struct Smem {
  double* slab;   // [kmax][Rs]
  double* wrow;   // winner row / pivot row x   [kmax + 2]
  double* arow;   // row a (displaced row)      [kmax + 2]
  double* taus;   // taus[j] = tau[lo + j]      [kmax + 2]
  double* zbuf;   // z = T x for the next gemv  [kmax + 2]
  double* part;   // gemv partial sums          [kThreads]
  double* ycol;   // scratch column             [Rs]
  int* perm;      // position -> physical       [Rs]
  Cand* wcand;    // per-warp candidates        [kWarps]
  int* misc;      // [0]=winner cta, [1]=winner idx, [2]=winner perm, [3]=perm_a, [4..7] cta cand
};

__host__ __device__ inline int slab_stride(int rows_per) { return rows_per | 1; }

__host__ __device__ inline size_t smem_layout(int rows_per, int kmax, int P, Smem* s, unsigned char* base) {
  (void)P;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 15) & ~size_t(15);
    return base ? base + o : nullptr;
  };
  int Rs = slab_stride(rows_per);
  unsigned char* p;
  p = take(sizeof(double) * (size_t)kmax * Rs);
  if (s) s->slab = (double*)p;
  p = take(sizeof(double) * (kmax + 2));
  if (s) s->wrow = (double*)p;
  p = take(sizeof(double) * (kmax + 2));
  if (s) s->arow = (double*)p;
  p = take(sizeof(double) * (kmax + 2));
  if (s) s->taus = (double*)p;
  p = take(sizeof(double) * (kmax + 2));
  if (s) s->zbuf = (double*)p;
  p = take(sizeof(double) * kThreads);
  if (s) s->part = (double*)p;
  p = take(sizeof(double) * Rs);
  if (s) s->ycol = (double*)p;
  p = take(sizeof(int) * Rs);
  if (s) s->perm = (int*)p;
  p = take(sizeof(Cand) * kWarps);
  if (s) s->wcand = (Cand*)p;
  p = take(sizeof(int) * 8);
  if (s) s->misc = (int*)p;
  return off;
}

// Partial left-looking products: part[gi*R + li] = sum_{j in group gi} slab[j][li] z_j.
// G groups of R threads split the k columns (short FMA chains, 2 accumulators).
__device__ __forceinline__ void gemv_partials(const Smem& s, int Rs, int R, int G, int k, int l0, int tid) {
  if (G > 1) {
    if (tid < G * R) {
      const int gi = tid / R, li = tid - gi * R;
      if (li >= l0) {
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
  }
}

// v = c - sum of partials (or the full dot product when G == 1), for local row li
__device__ __forceinline__ double gemv_finish(const Smem& s, int Rs, int R, int G, int k, int li, double c) {
  if (k < 2) return c;
  if (G > 1) {
    double acc = 0.0;
    for (int gi = 0; gi < G; ++gi) acc += s.part[gi * R + li];
    return c - acc;
  }
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int j = 0;
  for (; j + 3 < k; j += 4) {
    a0 = fma(s.slab[(size_t)j * Rs + li], s.zbuf[j], a0);
    a1 = fma(s.slab[(size_t)(j + 1) * Rs + li], s.zbuf[j + 1], a1);
    a2 = fma(s.slab[(size_t)(j + 2) * Rs + li], s.zbuf[j + 2], a2);
    a3 = fma(s.slab[(size_t)(j + 3) * Rs + li], s.zbuf[j + 3], a3);
  }
  for (; j < k; ++j) a0 = fma(s.slab[(size_t)j * Rs + li], s.zbuf[j], a0);
  return c - ((a0 + a1) + (a2 + a3));
}

__global__ void __launch_bounds__(kThreads, 1) panel_kernel(PanelArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::grid_group grid = cg::this_grid();
  const int P = gridDim.x, cta = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n, lo = a.lo, r = a.r, nelim = a.nelim, kmax = a.kmax;
  const int R = a.rows_per, Rs = slab_stride(R);
  const int G = R <= kThreads ? max(1, min(kThreads / max(R, 1), 16)) : 1;
  const long long ld = a.ld;
  double* __restrict__ W = a.W;
  const int row0 = lo + 1;
  const int rbase = row0 + cta * R;
  const int rcount = max(0, min(R, n - rbase));  // rows owned by this CTA
  const int rt = r + nelim;

  Smem s;
  smem_layout(R, kmax, P, &s, smem_raw);

  // ---- panel start: identity perm, carry column, first column ------------
  for (int li = tid; li < rcount; li += kThreads) s.perm[li] = rbase + li;
  if (lo < r) {
    for (int li = tid; li < rcount; li += kThreads) s.slab[li] = W[(long long)lo * ld + rbase + li];
  }
  for (int j = tid; j < kmax + 2; j += kThreads) {
    s.taus[j] = (j == 0 && lo >= 0 && lo < n - 1) ? a.tau[lo] : 0.0;
    s.wrow[j] = 0.0;
    s.zbuf[j] = 0.0;
  }
  {
    double* col = s.slab + (size_t)(r - lo) * Rs;
    for (int li = tid; li < rcount; li += kThreads) {
      int pos = rbase + li;
      col[li] = pos > r ? W[(long long)r * ld + pos] : 0.0;
    }
  }
  __syncthreads();

  const int slot_words = a.slot_words;
  long long _pt = clock64();
  (void)_pt;
  for (int g = r; g < rt; ++g) {
    const int k = g - lo;  // slab column of the current column
    const uint32_t tag = a.tag0 + uint32_t(g - r);
    const int par = tag & 1;
    double* col = s.slab + (size_t)k * Rs;
    const int l_first = max(0, g + 1 - rbase);  // first local row with position >= g+1
    const int a_pos = g + 1;
    const bool own_a = a_pos >= rbase && a_pos < rbase + rcount;
    TS_MARK(0);

    // ---- A/B: left-looking update v = c - A z, local argmax -----------------
    const int kk = (a.dbg & 1) ? 0 : k;
    if (kk >= 2 && G > 1) {
      gemv_partials(s, Rs, R, G, kk, l_first, tid);
      __syncthreads();
    }
    Cand best;
    best.v = 0.0;
    best.idx = -1;
    best.perm = -1;
    for (int li = l_first + tid; li < rcount; li += kThreads) {
      double v = gemv_finish(s, Rs, R, G, kk, li, col[li]);
      col[li] = v;
      if (better(v, rbase + li, best.v, best.idx)) {
        best.v = v;
        best.idx = rbase + li;
        best.perm = s.perm[li];
      }
    }
    PROF_MARK(0);
    warp_argmax(best.v, best.idx, best.perm);
    if (lane == 0) s.wcand[warp] = best;
    __syncthreads();
    PROF_MARK(1);

    // ---- C: publish (warp 0: candidate + row; warp 1: row a), poll, reduce ----
    if (warp == 0) {
      Cand c = lane < kWarps ? s.wcand[lane] : Cand{0.0, -1, -1};
      warp_argmax(c.v, c.idx, c.perm);
      uint64_t* slot = a.slots + ((size_t)cta * 2 + par) * slot_words;
      uint64_t* rec = a.recs + ((size_t)par * P + cta) * 4;
      if (c.idx >= 0 && !(a.dbg & 8)) {
        const int lc = c.idx - rbase;
        for (int j = lane; j <= k; j += 32) ll_put_double(slot + 4 + 2 * j, s.slab[(size_t)j * Rs + lc], tag);
      }
      if (lane == 0) {
        uint64_t bits = __double_as_longlong(c.v);
        ll_put2(rec + 2, uint32_t(c.idx), uint32_t(c.perm), tag);
        ll_put2(rec, uint32_t(bits), uint32_t(bits >> 32), tag);
      }
      PROF_MARK(2);
      TS_MARK(1);
      // poll all P records: lane handles slots lane, lane+32, ...
      Cand w{0.0, -1, -1};
      int owner = -1;
      constexpr int kMaxPoll = 8;  // P <= 256
      bool got[kMaxPoll];
#pragma unroll
      for (int q = 0; q < kMaxPoll; ++q) got[q] = (lane + 32 * q) >= P;
      bool all = (a.dbg & 16) != 0;
      if (all) { w = c; owner = cta; }
      int spins = 0;
      while (!all) {
        (void)spins;
        all = true;
#pragma unroll
        for (int q = 0; q < kMaxPoll; ++q) {
          if (!got[q]) {
            const int t = lane + 32 * q;
            const uint64_t* sl = a.recs + ((size_t)par * P + t) * 4;
            uint64_t w0, w1, w2, w3;
            asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(sl) : "memory");
            asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w2), "=l"(w3) : "l"(sl + 2) : "memory");
            if (uint32_t(w0 >> 32) == tag && uint32_t(w1 >> 32) == tag && uint32_t(w2 >> 32) == tag &&
                uint32_t(w3 >> 32) == tag) {
              got[q] = true;
              Cand o;
              o.v = __longlong_as_double((long long)((w1 << 32) | (w0 & 0xffffffffull)));
              o.idx = int(uint32_t(w2));
              o.perm = int(uint32_t(w3));
              if (better(o.v, o.idx, w.v, w.idx)) {
                w = o;
                owner = t;
              }
            } else {
              all = false;
            }
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, w.v, o);
        int oi = __shfl_xor_sync(0xffffffffu, w.idx, o);
        int op = __shfl_xor_sync(0xffffffffu, w.perm, o);
        int ow = __shfl_xor_sync(0xffffffffu, owner, o);
        if (better(ov, oi, w.v, w.idx)) {
          w.v = ov;
          w.idx = oi;
          w.perm = op;
          owner = ow;
        }
      }
      if (lane == 0) {
        s.misc[0] = owner;
        s.misc[1] = w.idx;
        s.misc[2] = w.perm;
        reinterpret_cast<double*>(s.misc + 6)[0] = w.v;
      }
    } else if (warp == 1 && own_a) {
      uint64_t* ra = a.rowa + (size_t)par * slot_words;
      const int la = a_pos - rbase;
      for (int j = lane; j <= k; j += 32) ll_put_double(ra + 4 + 2 * j, s.slab[(size_t)j * Rs + la], tag);
      if (lane == 0) ll_put2(ra, uint32_t(s.perm[la]), 0u, tag);
    }
    __syncthreads();
    TS_MARK(2);
    PROF_MARK(3);

    // ---- D: gather next column (overlapped with the winner-row fetch) --------
    const int owner = s.misc[0], b = s.misc[1], pb = s.misc[2];
    const double vb = reinterpret_cast<double*>(s.misc + 6)[0];
    const bool own_b = b >= rbase && b < rbase + rcount;
    const bool swapped = b != a_pos;
    const bool more = (g + 1 < rt) || a.want_y;
    double cnext[2] = {0.0, 0.0};
    const uint64_t* ra = a.rowa + (size_t)par * slot_words;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int li = tid + u * kThreads;
      const int pos = rbase + li;
      if (more && li < rcount && pos > a_pos) {
        int ph;
        if (swapped && pos == b) {
          uint32_t pa = 0, dummy;
          if (!(a.dbg & 4)) ll_get2(ra, tag, pa, dummy);
          ph = int(pa);
        } else {
          ph = s.perm[li];
        }
        cnext[u] = (a.dbg & 2) ? 0.0 : skew_at(W, ld, ph, pb);
      }
    }
    {
      const uint64_t* wslot = a.slots + ((size_t)owner * 2 + par) * slot_words;
      if (!(a.dbg & 4)) for (int j = tid; j <= k; j += kThreads) s.wrow[j] = ll_get_double(wslot + 4 + 2 * j, tag);
      if (own_b && swapped && !(a.dbg & 4)) {
        for (int j = tid; j <= k; j += kThreads) s.arow[j] = ll_get_double(ra + 4 + 2 * j, tag);
        if (tid == 0) {
          uint32_t pa, dummy;
          ll_get2(ra, tag, pa, dummy);
          s.misc[3] = int(pa);
        }
      }
    }
    PROF_MARK(4);
    __syncthreads();
    PROF_MARK(5);

    // ---- E: interchange, scale, next column, z for the next step -------------
    if (swapped) {
      if (own_a) {
        const int la = a_pos - rbase;
        for (int j = tid; j < k; j += kThreads) s.slab[(size_t)j * Rs + la] = s.wrow[j];
      }
      if (own_b) {
        const int lb = b - rbase;
        for (int j = tid; j < k; j += kThreads) s.slab[(size_t)j * Rs + lb] = s.arow[j];
      }
    }
    double* ncol = (g + 1 < rt) ? s.slab + (size_t)(k + 1) * Rs : s.ycol;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int li = tid + u * kThreads;
      if (li < rcount) {
        const int pos = rbase + li;
        if (pos == a_pos) {
          col[li] = 1.0;
          if (swapped) s.perm[li] = pb;
        } else if (pos > a_pos) {
          double v = (swapped && pos == b) ? s.arow[k] : col[li];
          col[li] = vb != 0.0 ? v / vb : v;
          if (swapped && pos == b) s.perm[li] = s.misc[3];
        }
        if (more) ncol[li] = cnext[u];
      }
    }
    // z for the next step: x = [wrow[0..k-1], 1], taus[k] = vb
    for (int j = tid; j <= k; j += kThreads) {
      double xm = j >= 1 ? s.wrow[j - 1] : 0.0;
      double xp = (j + 1 < k) ? s.wrow[j + 1] : (j + 1 == k ? 1.0 : 0.0);
      double tj = j == k ? vb : s.taus[j];
      double tj1 = (j + 1 == k) ? vb : s.taus[j + 1];
      s.zbuf[j] = (j >= 1 ? tj * xm : 0.0) - (j + 1 <= k ? tj1 * xp : 0.0);
    }
    __syncthreads();
    if (tid == 0) {
      s.taus[k] = vb;
      s.wrow[k] = 1.0;
      if (cta == 0) {
        a.tau[g] = vb;
        a.piv[g + 1] = (long long)(b - a_pos);
      }
    }
    PROF_MARK(6);
    PROF_MARK(7);
  }

  // ---- var1: y = column rt after the panel's couplings (for the straggler) --
  __syncthreads();
  if (a.want_y && rt < n) {
    const int k = rt - lo;
    const int l_first = max(0, rt + 1 - rbase);
    if (G > 1) {
      gemv_partials(s, Rs, R, G, k, l_first, tid);
      __syncthreads();
    }
    for (int li = l_first + tid; li < rcount; li += kThreads)
      a.y[rbase + li] = gemv_finish(s, Rs, R, G, k, li, s.ycol[li]);
  }

  // ---- materialise the displaced trailing lines -------------------------
  for (int li = tid; li < rcount; li += kThreads) {
    int pos = rbase + li, ph = s.perm[li];
    a.gperm[pos] = ph;
    if (pos >= rt && ph != pos) {
      int q = atomicAdd(a.disp_count, 1);
      a.disp_list[q] = pos;
    }
  }
  if (cta == 0) {
    for (int i = tid; i < row0; i += kThreads) a.gperm[i] = i;
  }
  grid.sync();
  const int nd = *a.disp_count;
  const int ntr = n - rt;
  for (int q = cta; q < nd; q += P) {
    const int p = a.disp_list[q];
    const int pp = a.gperm[p];
    double* line = a.side + (size_t)q * ntr;
    for (int i = rt + tid; i < n; i += kThreads) line[i - rt] = (i == p) ? 0.0 : skew_at(W, ld, a.gperm[i], pp);
  }
  grid.sync();

  // ---- write back: slab -> L columns [lo, rt); side -> trailing lines ------
  for (int j = 0; j < kmax; ++j) {
    const int c = lo + j;
    const double* sc = s.slab + (size_t)j * Rs;
    for (int li = tid; li < rcount; li += kThreads) {
      int pos = rbase + li;
      if (pos > c) W[(long long)c * ld + pos] = sc[li];
    }
  }
  for (int q = cta; q < nd; q += P) {
    const int p = a.disp_list[q];
    const double* line = a.side + (size_t)q * ntr;
    for (int i = rt + tid; i < n; i += kThreads) {
      double v = line[i - rt];
      if (i > p)
        W[(long long)p * ld + i] = v;
      else if (i < p)
        W[(long long)i * ld + p] = -v;
    }
  }
}

// sigma_all[k][i] = (pi_{k+1} o ... o pi_{np-1})(i): the row gather still
// owed by L columns whose last panel was k (composition of the reference's
// per-panel apply_row_pivots, kernels2.py:232-271 / blocked.py:293-300).
__global__ void compose_suffix_kernel(const int* __restrict__ gperm_all, int np, int n, int* __restrict__ sigma_all) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int sidx = i;
    for (int k = np - 1; k >= 0; --k) {
      sigma_all[(size_t)k * n + i] = sidx;
      sidx = gperm_all[(size_t)k * n + sidx];
    }
  }
}

// L[i, c] = W[sigma_{grp(c)}[i], c] for i > c; upper/diag copied from X.
__global__ void finalize_l_kernel(const double* __restrict__ W, long long ldw, const double* __restrict__ X,
                                  long long ldx, double* __restrict__ L, long long ldl, int n,
                                  const int* __restrict__ col_group, const int* __restrict__ sigma_all,
                                  int copy_upper, int own_nbd, int own_g, int own_rank) {
  for (int c = blockIdx.y; c < n; c += gridDim.y) {
    if (own_g > 1 && (c / own_nbd) % own_g != own_rank) continue;  // another rank's column
    const int grp = col_group[c];
    const int* sg = sigma_all + (size_t)grp * n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      if (i > c) {
        L[(long long)c * ldl + i] = W[(long long)c * ldw + sg[i]];
      } else if (copy_upper) {
        L[(long long)c * ldl + i] = X[(long long)c * ldx + i];
      }
    }
  }
}

}  // namespace

int panel_threads() { return kThreads; }

size_t panel_smem_bytes(int rows_per, int kmax) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return smem_layout(rows_per, kmax, nsm, nullptr, nullptr);
}

int panel_max_ctas() {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return nsm;
}

cudaError_t launch_panel(const PanelArgs& a, cudaStream_t stream) {
  size_t smem = smem_layout(a.rows_per, a.kmax, a.nblocks, nullptr, nullptr);
  cudaError_t e = cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(a.disp_count, 0, sizeof(int), stream);
  if (e != cudaSuccess) return e;
  PanelArgs copy = a;
  void* args[] = {&copy};
  return cudaLaunchCooperativeKernel((void*)panel_kernel, dim3(a.nblocks), dim3(kThreads), args, smem, stream);
}

cudaError_t launch_compose_suffix(const int* gperm_all, int npanels, const int* row0s, int n, int* sigma_all,
                                  cudaStream_t stream) {
  (void)row0s;
  int grid = (n + 255) / 256;
  compose_suffix_kernel<<<grid, 256, 0, stream>>>(gperm_all, npanels, n, sigma_all);
  return cudaGetLastError();
}

cudaError_t launch_finalize_l(const double* W, long long ldw, const double* X, long long ldx, double* L,
                              long long ldl, int n, const int* col_group, const int* sigma_all, int copy_upper,
                              cudaStream_t stream, int own_nbd, int own_g, int own_rank) {
  dim3 grid((n + 255) / 256 < 8 ? (n + 255) / 256 : 8, n < 4096 ? n : 4096);
  finalize_l_kernel<<<grid, 256, 0, stream>>>(W, ldw, X, ldx, L, ldl, n, col_group, sigma_all, copy_upper, own_nbd,
                                              own_g, own_rank);
  return cudaGetLastError();
}

}  // namespace skl

#ifdef SKL_PANEL_PROFILE
extern "C" int skl_debug_panel_ts(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, skl::g_panel_ts, sizeof(unsigned long long) * 8 * 160 * 4);
}
extern "C" int skl_debug_panel_profile(unsigned long long* out32) {
  return (int)cudaMemcpyFromSymbol(out32, skl::g_panel_prof, sizeof(unsigned long long) * 32);
}
#endif
