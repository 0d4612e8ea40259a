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
  double* ycol;   // scratch column             [Rs]
  int* perm;      // position -> physical       [Rs]
  Cand* wcand;    // per-warp candidates        [kWarps]
  Cand* ccand;    // per-CTA candidates         [P]
  int* misc;      // [0]=winner cta, [1]=winner idx, [2]=winner perm, [3]=perm_a
};

__host__ __device__ inline int slab_stride(int rows_per) { return rows_per | 1; }

__host__ __device__ inline size_t smem_layout(int rows_per, int kmax, int P, Smem* s, unsigned char* base) {
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
  p = take(sizeof(double) * Rs);
  if (s) s->ycol = (double*)p;
  p = take(sizeof(int) * Rs);
  if (s) s->perm = (int*)p;
  p = take(sizeof(Cand) * kWarps);
  if (s) s->wcand = (Cand*)p;
  p = take(sizeof(Cand) * P);
  if (s) s->ccand = (Cand*)p;
  p = take(sizeof(int) * 8);
  if (s) s->misc = (int*)p;
  return off;
}

// v[li] = c[li] - sum_j slab[j][li] z_j  for local rows li in [l0, R), written
// in place into slab column k (which holds c on entry).  z = T x with
// T = tridiag(taus[1..k-1]), x = wrow[0..k-1].  Returns per-lane best
// candidate over processed rows (lane 0 only meaningful after warp reduce).
__device__ __forceinline__ void gemv_rows(const Smem& s, int Rs, int k, int l0, int R, int rbase, int warp,
                                          int lane, double* outcol, Cand& best) {
  double z[kMaxZ];
#pragma unroll
  for (int m = 0; m < kMaxZ; ++m) {
    int j = lane + 32 * m;
    double zz = 0.0;
    if (j < k) {
      if (j >= 1) zz = s.taus[j] * s.wrow[j - 1];
      if (j + 1 < k) zz -= s.taus[j + 1] * s.wrow[j + 1];
    }
    z[m] = zz;
  }
  const int nm = (k + 31) >> 5;
  for (int li = l0 + warp; li < R; li += kWarps) {
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < kMaxZ; ++m) {
      if (m < nm) {
        int j = lane + 32 * m;
        if (j < k) acc = fma(s.slab[(size_t)j * Rs + li], z[m], acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      double v = outcol[li] - acc;
      outcol[li] = v;
      if (better(v, rbase + li, best.v, best.idx)) {
        best.v = v;
        best.idx = rbase + li;
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) panel_kernel(PanelArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::grid_group grid = cg::this_grid();
  const int P = gridDim.x, cta = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n, lo = a.lo, r = a.r, nelim = a.nelim, kmax = a.kmax;
  const int R = a.rows_per, Rs = slab_stride(R);
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
  }
  // first column g = r: X_cur[i, r] = X0[i, r] for i > r
  {
    double* col = s.slab + (size_t)(r - lo) * Rs;
    for (int li = tid; li < rcount; li += kThreads) {
      int pos = rbase + li;
      col[li] = pos > r ? W[(long long)r * ld + pos] : 0.0;
    }
  }
  int pg = r;  // physical index of the current column's position
  __syncthreads();

  const int slot_words = a.slot_words;
  for (int g = r; g < rt; ++g) {
    const int k = g - lo;  // slab column of the current column
    const uint32_t tag = a.tag0 + uint32_t(g - r);
    const int par = tag & 1;
    double* col = s.slab + (size_t)k * Rs;
    const int l_first = max(0, g + 1 - rbase);  // first local row with position >= g+1

    // ---- left-looking update + local argmax ------------------------------
    Cand best;
    best.v = 0.0;
    best.idx = -1;
    best.perm = -1;
    if (k >= 2) {
      gemv_rows(s, Rs, k, l_first, rcount, rbase, warp, lane, col, best);
    } else {
      for (int li = l_first + tid; li < rcount; li += kThreads) {
        double v = col[li];
        if (better(v, rbase + li, best.v, best.idx)) {
          best.v = v;
          best.idx = rbase + li;
        }
      }
    }
    warp_argmax(best.v, best.idx, best.perm);
    if (lane == 0) s.wcand[warp] = best;
    __syncthreads();
    if (warp == 0) {
      Cand c = lane < kWarps ? s.wcand[lane] : Cand{0.0, -1, -1};
      warp_argmax(c.v, c.idx, c.perm);
      if (lane == 0) {
        if (c.idx >= 0) c.perm = s.perm[c.idx - rbase];
        s.misc[4] = c.idx;
        s.misc[5] = c.perm;
        reinterpret_cast<double*>(s.misc + 6)[0] = c.v;  // misc[6..7]
      }
    }
    __syncthreads();

    // ---- publish candidate (+ its row) and, if owned, row a ---------------
    const int a_pos = g + 1;
    const bool own_a = a_pos >= rbase && a_pos < rbase + rcount;
    {
      uint64_t* slot = a.slots + ((size_t)cta * 2 + par) * slot_words;
      const int cidx = s.misc[4];
      if (cidx >= 0) {
        const int lc = cidx - rbase;
        for (int j = tid; j <= k; j += kThreads) ll_put_double(slot + 4 + 2 * j, s.slab[(size_t)j * Rs + lc], tag);
      }
      if (own_a) {
        uint64_t* ra = a.rowa + (size_t)par * slot_words;
        const int la = a_pos - rbase;
        for (int j = tid; j <= k; j += kThreads) ll_put_double(ra + 4 + 2 * j, s.slab[(size_t)j * Rs + la], tag);
        if (tid == 0) ll_put2(ra, uint32_t(s.perm[la]), 0u, tag);
      }
      if (tid == 0) {
        double cv = reinterpret_cast<double*>(s.misc + 6)[0];
        uint64_t bits = __double_as_longlong(cv);
        ll_put2(slot, uint32_t(bits), uint32_t(bits >> 32), tag);
        ll_put2(slot + 2, uint32_t(cidx), uint32_t(s.misc[5]), tag);
      }
    }

    // ---- poll every CTA's candidate ---------------------------------------
    for (int t = tid; t < P; t += kThreads) {
      const uint64_t* slot = a.slots + ((size_t)t * 2 + par) * slot_words;
      uint32_t lo32, hi32, ci, cp;
      ll_get2(slot, tag, lo32, hi32);
      ll_get2(slot + 2, tag, ci, cp);
      Cand c;
      c.v = __longlong_as_double((long long)((uint64_t(hi32) << 32) | lo32));
      c.idx = int(ci);
      c.perm = int(cp);
      s.ccand[t] = c;
    }
    __syncthreads();
    if (warp == 0) {
      Cand c{0.0, -1, -1};
      int owner = -1;
      for (int t = lane; t < P; t += 32) {
        Cand o = s.ccand[t];
        if (better(o.v, o.idx, c.v, c.idx)) {
          c = o;
          owner = t;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, c.v, o);
        int oi = __shfl_xor_sync(0xffffffffu, c.idx, o);
        int op = __shfl_xor_sync(0xffffffffu, c.perm, o);
        int ow = __shfl_xor_sync(0xffffffffu, owner, o);
        if (better(ov, oi, c.v, c.idx)) {
          c.v = ov;
          c.idx = oi;
          c.perm = op;
          owner = ow;
        }
      }
      if (lane == 0) {
        s.misc[0] = owner;
        s.misc[1] = c.idx;
        s.misc[2] = c.perm;
        reinterpret_cast<double*>(s.misc + 6)[0] = c.v;
      }
    }
    __syncthreads();
    const int owner = s.misc[0], b = s.misc[1], pb = s.misc[2];
    const double vb = reinterpret_cast<double*>(s.misc + 6)[0];
    const bool own_b = b >= rbase && b < rbase + rcount;

    // ---- fetch the winning row (and row a if we own b) -------------------
    {
      const uint64_t* wslot = a.slots + ((size_t)owner * 2 + par) * slot_words;
      for (int j = tid; j <= k; j += kThreads) s.wrow[j] = ll_get_double(wslot + 4 + 2 * j, tag);
      if (own_b && b != a_pos) {
        const uint64_t* ra = a.rowa + (size_t)par * slot_words;
        for (int j = tid; j <= k; j += kThreads) s.arow[j] = ll_get_double(ra + 4 + 2 * j, tag);
        if (tid == 0) {
          uint32_t pa, dummy;
          ll_get2(ra, tag, pa, dummy);
          s.misc[3] = int(pa);
        }
      }
    }
    __syncthreads();

    // ---- symmetric interchange restricted to the slab rows + perm ----------
    if (b != a_pos) {
      if (own_a) {
        const int la = a_pos - rbase;
        for (int j = tid; j <= k; j += kThreads) s.slab[(size_t)j * Rs + la] = s.wrow[j];
      }
      if (own_b) {
        const int lb = b - rbase;
        for (int j = tid; j <= k; j += kThreads) s.slab[(size_t)j * Rs + lb] = s.arow[j];
      }
    }
    __syncthreads();
    if (tid == 0) {
      if (b != a_pos) {
        if (own_a) s.perm[a_pos - rbase] = pb;
        if (own_b) s.perm[b - rbase] = s.misc[3];
      }
      s.taus[k] = vb;
      s.wrow[k] = 1.0;  // pivot row of the next step: [A[b, 0..k-1], 1]
      if (cta == 0) {
        a.tau[g] = vb;
        a.piv[g + 1] = (long long)(b - a_pos);
      }
    }
    __syncthreads();

    // ---- scale: L column g+1 = v / tau below the unit --------------------
    const double inv = vb != 0.0 ? 1.0 / vb : 0.0;
    (void)inv;
    for (int li = tid; li < rcount; li += kThreads) {
      int pos = rbase + li;
      if (pos == a_pos) {
        col[li] = 1.0;
      } else if (pos > a_pos && vb != 0.0) {
        col[li] = col[li] / vb;
      }
    }
    // ---- next column: gather X_cur[i, a] = X0[perm[i], perm[a]] ---------
    pg = pb;
    if (g + 1 < rt || a.want_y) {
      double* ncol = (g + 1 < rt) ? s.slab + (size_t)(k + 1) * Rs : s.ycol;
      for (int li = tid; li < rcount; li += kThreads) {
        int pos = rbase + li;
        double c = 0.0;
        if (pos > a_pos) c = skew_at(W, ld, s.perm[li], pg);
        ncol[li] = c;
      }
    }
    __syncthreads();
  }

  // ---- var1: y = column rt after the panel's couplings (for the straggler) --
  if (a.want_y && rt < n) {
    const int k = rt - lo;
    const int l_first = max(0, rt + 1 - rbase);
    Cand dummy;
    dummy.v = 0.0;
    dummy.idx = -1;
    gemv_rows(s, Rs, k, l_first, rcount, rbase, warp, lane, s.ycol, dummy);
    __syncthreads();
    for (int li = l_first + tid; li < rcount; li += kThreads) a.y[rbase + li] = s.ycol[li];
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
                                  int copy_upper) {
  for (int c = blockIdx.y; c < n; c += gridDim.y) {
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
                              cudaStream_t stream) {
  dim3 grid((n + 255) / 256 < 8 ? (n + 255) / 256 : 8, n < 4096 ? n : 4096);
  finalize_l_kernel<<<grid, 256, 0, stream>>>(W, ldw, X, ldx, L, ldl, n, col_group, sigma_all, copy_upper);
  return cudaGetLastError();
}

}  // namespace skl
