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
#include <algorithm>
#include <cassert>

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
// 16-byte candidate -> the same smem slot in CTA `rank`, completing 16 bytes of
// transaction on that CTA's mbarrier (same offset as `bar`)
__device__ __forceinline__ void st_async_cand(CCand* slot_local, uint64_t* bar_local, uint32_t rank, const CCand& c) {
  uint32_t rdst, rbar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(smem_u32(slot_local)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(bar_local)), "r"(rank));
  const unsigned long long vb = (unsigned long long)__double_as_longlong(c.v);
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(rdst),
               "r"(uint32_t(vb)), "r"(uint32_t(vb >> 32)), "r"(uint32_t(c.idx)), "r"(uint32_t(c.perm)), "r"(rbar)
               : "memory");
}

// two doubles -> the same smem offset in CTA `rank`, completing 16 bytes on its mbarrier
__device__ __forceinline__ void st_async_f64x2(double* dst_local, uint64_t* bar_local, uint32_t rank, double x,
                                               double y) {
  uint32_t rdst, rbar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(smem_u32(dst_local)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(bar_local)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(rdst),
               "d"(x), "d"(y), "r"(rbar)
               : "memory");
}

__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
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
  int* misc;       // [0..1] pubA perm per parity, [4..5] global winner owner (MULTI)
  int* pivbuf;     // [nelim] pivot offsets of this panel (flushed at the end)
  CCand* gwin;     // [2] global winner (MULTI)
  uint64_t* xbar;  // MULTI: [0..1] candidate all-to-all, [2..3] global-winner delivery (st.async)
  int* lab;        // [Rs] final position of each slab row (written after the step loop)
  double* crows;   // push mode: [2][C][crow_stride(kmax)] candidate rows pushed by every CTA
};

__host__ __device__ inline int crow_stride(int kmax) { return (kmax + 3) & ~1; }  // even: 16-byte rows

__host__ __device__ inline int cslab_stride(int rows_per) { return rows_per | 1; }

__host__ __device__ inline size_t csmem_layout(int R, int kmax, CSmem* s, unsigned char* base, int npush = 0) {
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
  p = take(sizeof(CCand) * 2);
  if (s) s->gwin = (CCand*)p;
  p = take(sizeof(uint64_t) * 4);
  if (s) s->xbar = (uint64_t*)p;
  p = take(sizeof(int) * Rs);
  if (s) s->lab = (int*)p;
  p = take(sizeof(double) * 2 * (size_t)npush * crow_stride(kmax));
  if (s) s->crows = (double*)p;
  return off;
}

// MULTI = several co-resident clusters (cooperative launch): candidates are
// reduced inside each cluster through DSMEM, then the cluster leaders exchange
// their cluster's best through global LL records; pivot rows travel through L2.
template <bool MULTI>
__global__ void __launch_bounds__(kCThreads, 1) panel_cluster_kernel(PanelArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const long long t_kernel0 = clock64();
  cg::cluster_group cluster = cg::this_cluster();
  const int C = MULTI ? int(cluster.num_blocks()) : int(gridDim.x);
  const int crank = MULTI ? int(cluster.block_rank()) : int(blockIdx.x);  // rank inside the cluster
  const int gcta = blockIdx.x;                                             // global CTA id (row owner)
  const int Q = MULTI ? int(gridDim.x) / C : 1;                            // clusters
  const int qid = gcta / C;
  const int cta = gcta;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n, lo = a.lo, r = a.r, nelim = a.nelim, kmax = a.kmax;
  const int R = a.rows_per, Rs = cslab_stride(R);
  const long long ld = a.ld;
  double* __restrict__ W = a.W;
  const int row0 = lo + 1;
  const int rbase = row0 + cta * R;
  const int rcount = max(0, min(R, n - rbase));
  const int rt = r + nelim;

  CSmem s;
  // push mode (one cluster, pivoted): every CTA pushes its candidate's row to every CTA
  // with st.async next to the candidate, and symmetric interchanges are LAZY -- a slab row
  // keeps its data and carries its position as a label (lab[]), so no row ever moves
  // between CTAs and no pivot row is fetched through L2
  const bool push = MULTI && Q == 1 && a.pivot && a.push;
  csmem_layout(R, kmax, &s, smem_raw, push ? C : 0);
  const int CRS = crow_stride(kmax);
  const bool spread_pub = a.dbg & 64 ? false : true;  // dbg bit 6: the warp-0 publication (A/B)
  if (MULTI && tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&s.xbar[i], 1);  // one local arrival (expect_tx) per phase
    fence_mbar_init();  // made visible to the cluster by the cluster barrier below
  }

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
  long long sub[3] = {0, 0, 0};  // phase-3 split (profiling only): winner | gathers issued | row poll done
  long long t_prev = clock64();
  const long long t_loop0 = t_prev;
#ifdef SKL_PANEL_PROFILE
#define SUBMARK(i)                  \
  do {                              \
    sub[i] += clock64() - t_prev;   \
  } while (0)
#define CMARK(i)                    \
  do {                              \
    long long _t = clock64();       \
    pt[i] += _t - t_prev;           \
    t_prev = _t;                    \
  } while (0)
#else  // phase clocks only in the profiling build (make prof)
#define SUBMARK(i) \
  do {             \
  } while (0)
#define CMARK(i) \
  do {           \
  } while (0)
#endif

  // register cache of slab columns [0, kBank*nbank) for row li = tid (the gemv re-reads
  // the slab every step; shared-memory bandwidth is its bound otherwise)
  double rb[2][kBank];
  int nbank = 0;
  // per-thread rows: li = tid + u * kCThreads (R <= 2 * kCThreads)
  double cnext[2] = {0.0, 0.0};
  bool cneg[2] = {false, false};  // gathered from the row part: negate at use (keeps the load in flight)
  int lab[2] = {rbase + tid, rbase + tid + kCThreads};  // position of row li = tid + u * kCThreads
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
    const int owner_a = (a_pos - row0) / R;  // global CTA id owning position a
    const bool own_a = owner_a == cta;
    const uint32_t tag = a.tag0 + uint32_t(g - r);

    if (MULTI && tid == 0) {
      // this step's deliveries: C candidates (16 B each) and the global winner (16 B)
      // push mode: the candidate rows complete on their own barrier (xbar[2 + par], unused
      // with one cluster), so the winner is found while the rows are still in flight
      mbar_arrive_expect_tx(&s.xbar[par], uint32_t(C) * uint32_t(sizeof(CCand)));
      if (push) mbar_arrive_expect_tx(&s.xbar[2 + par], uint32_t(C) * 16u * uint32_t((k + 2) >> 1));
      if (Q > 1) mbar_arrive_expect_tx(&s.xbar[2 + par], sizeof(CCand));
    }

    // ---- (1) v = c - A z; per-warp argmax -----------------------------------
    double vbest = 0.0;
    int ibest = -1, lbest = 0;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int li = tid + u * kCThreads;
      const int pos = lab[u];
      if (li < rcount && pos > g) {
        const double v = (cneg[u] ? -cnext[u] : cnext[u]) - s.az[li];
        col[li] = v;
        if (ibest < 0 || fabs(v) > fabs(vbest)) {
          vbest = v;
          ibest = pos;
          lbest = li;
        }
      }
    }
    {
      // the perm field carries the local slab row until the CTA candidate is formed
      const int id = warp_argmax_redux(vbest, ibest, ibest >= 0);
      if (ibest >= 0 && ibest == id) s.wcand[warp] = CCand{vbest, ibest, lbest};
      if (lane == 0 && id < 0) s.wcand[warp] = CCand{0.0, -1, 0};
    }
    CMARK(0);
    __syncthreads();

    // ---- (2) CTA candidate -> every CTA of the cluster; publish rows ------------
    int lc_pub = -1;  // local row of this CTA's candidate
    if (MULTI && spread_pub) {
      // every warp derives the CTA candidate from the 8 warp candidates (one redux), so
      // warp 0 sends it while warps 2-5 publish its row and warps 1/6/7 row a, in parallel:
      // the rows reach L2 before the receivers poll them (one round trip in phase 3)
      const bool ok = lane < kCWarps && s.wcand[lane].idx >= 0;
      const CCand mine = lane < kCWarps ? s.wcand[lane] : CCand{0.0, -1, 0};
      const int id = warp_argmax_redux(mine.v, mine.idx, ok);
      const unsigned bal = __ballot_sync(0xffffffffu, ok && mine.idx == id);
      CCand c = CCand{0.0, -1, -1};
      if (id >= 0) {
        c = s.wcand[__ffs(bal) - 1];
        lc_pub = c.perm;
        c.perm = s.perm[lc_pub];
      }
      if (warp == 0) {
        if (lane < C) st_async_cand(s.cand + par * kClusterMax + crank, &s.xbar[par], lane, c);
      } else if (push) {
        // candidate row [0, k] (pairs of doubles) -> crows[par][crank] of every CTA
        const int np = (k + 2) >> 1;
        const int lc = lc_pub >= 0 ? lc_pub : 0;
        double* dst = s.crows + ((size_t)par * C + crank) * CRS;
        const float inv_np = 1.0f / float(np);  // f < 16 * 66: the float quotient is exact after rz
        for (int f = tid - 32; f < C * np; f += kCThreads - 32) {
          const int d = __float2int_rz((float(f) + 0.5f) * inv_np), pp = f - d * np;
          const int j0 = 2 * pp;
          const double x0 = s.slab[(size_t)j0 * Rs + lc];
          const double x1 = j0 + 1 <= k ? s.slab[(size_t)(j0 + 1) * Rs + lc] : 0.0;
          st_async_f64x2(dst + j0, &s.xbar[2 + par], uint32_t(d), x0, x1);
        }
      } else if (warp >= 2 && warp <= 5) {
        if (lc_pub >= 0) {
          uint64_t* gr = a.slots + ((size_t)gcta * 2 + par) * a.slot_words + 4;
          for (int j = (warp - 2) * 32 + lane; j <= k; j += 128)
            ll_put_double(gr + 2 * j, s.slab[(size_t)j * Rs + lc_pub], tag);
        }
      } else if (own_a) {
        const int la = a_pos - rbase;
        uint64_t* ra = a.rowa + (size_t)par * a.slot_words;
        const int w3 = warp == 1 ? 0 : warp - 5;
        for (int j = w3 * 32 + lane; j <= k; j += 96) ll_put_double(ra + 4 + 2 * j, s.slab[(size_t)j * Rs + la], tag);
        if (warp == 1 && lane == 0) ll_put2(ra, uint32_t(s.perm[la]), 0u, tag);
      }
      CMARK(1);
      mbar_wait_delivered(&s.xbar[par], (uint32_t(g - r) >> 1) & 1u);
    } else {
      if (warp == 0) {
        const bool ok = lane < kCWarps && s.wcand[lane].idx >= 0;
        const CCand mine = lane < kCWarps ? s.wcand[lane] : CCand{0.0, -1, 0};
        const int id = warp_argmax_redux(mine.v, mine.idx, ok);
        const unsigned bal = __ballot_sync(0xffffffffu, ok && mine.idx == id);
        CCand c = CCand{0.0, -1, -1};
        if (id >= 0) {
          c = s.wcand[__ffs(bal) - 1];
          lc_pub = c.perm;
          c.perm = s.perm[lc_pub];
          if (!MULTI) {
            double* pr = s.pubrow + par * (kmax + 2);
            for (int j = lane; j <= k; j += 32) pr[j] = s.slab[(size_t)j * Rs + lc_pub];
          }
        }
        __syncwarp();
        if (MULTI) {
          // candidate -> slot crank of every cluster CTA, delivered with its mbarrier
          if (lane < C) st_async_cand(s.cand + par * kClusterMax + crank, &s.xbar[par], lane, c);
        } else if (lane < C) {
          *cluster.map_shared_rank(s.cand + par * kClusterMax + crank, lane) = c;
        }
      } else if (!MULTI && warp == 1 && own_a) {
        const int la = a_pos - rbase;
        double* pa = s.pubA + par * (kmax + 2);
        for (int j = lane; j <= k; j += 32) pa[j] = s.slab[(size_t)j * Rs + la];
        if (lane == 0) s.misc[par] = s.perm[la];
      }
      CMARK(1);
      if (MULTI) {
        // the global LL publications (candidate row, row a) carry their own flags and
        // need no ordering; the candidates arrive by st.async on xbar[par] (no
        // cluster barrier: nothing else is read across CTAs in this mode)
        if (warp == 0 && lc_pub >= 0) {
          uint64_t* gr = a.slots + ((size_t)gcta * 2 + par) * a.slot_words + 4;
          for (int j = lane; j <= k; j += 32) ll_put_double(gr + 2 * j, s.slab[(size_t)j * Rs + lc_pub], tag);
        } else if (warp == 1 && own_a) {
          const int la = a_pos - rbase;
          uint64_t* ra = a.rowa + (size_t)par * a.slot_words;
          for (int j = lane; j <= k; j += 32) ll_put_double(ra + 4 + 2 * j, s.slab[(size_t)j * Rs + la], tag);
          if (lane == 0) ll_put2(ra, uint32_t(s.perm[la]), 0u, tag);
        }
        mbar_wait_delivered(&s.xbar[par], (uint32_t(g - r) >> 1) & 1u);
      } else {
        cluster_barrier();
      }
    }
    CMARK(2);

    // ---- (3) winner, next-column gather, winner row / row a via DSMEM ---------
    int owner;
    CCand w;
    const double* xrow = s.wrow;  // pivot row of this step (push: in place in crows)
    {
      const bool ok = lane < C && s.cand[par * kClusterMax + lane].idx >= 0;
      const CCand mine = lane < C ? s.cand[par * kClusterMax + lane] : CCand{0.0, -1, -1};
      const int id = warp_argmax_redux(mine.v, mine.idx, ok);
      owner = __ffs(__ballot_sync(0xffffffffu, ok && mine.idx == id)) - 1;
      if (owner < 0) {  // no row of this cluster is below g (small multi-cluster panels)
        w = CCand{0.0, -1, -1};
        owner = 0;
      } else {
        w = s.cand[par * kClusterMax + owner];
      }
      owner += qid * C;  // global CTA id of the cluster's best
    }
    if (MULTI && Q > 1) {
      if (crank == 0 && warp == 0) {
        // leader: publish the cluster's best, gather every cluster's best (one lane each)
        uint64_t* rec = a.recs + ((size_t)par * Q + qid) * 6;
        if (lane == 0) {
          const uint64_t bits = __double_as_longlong(w.v);
          ll_put2(rec, uint32_t(bits), uint32_t(bits >> 32), tag);
          ll_put2(rec + 2, uint32_t(w.idx), uint32_t(w.perm), tag);
          ll_put2(rec + 4, uint32_t(owner), 0u, tag);
        }
        CCand o{0.0, -1, -1};
        int oo = -1;
        if (lane < Q) {
          const uint64_t* rq = a.recs + ((size_t)par * Q + lane) * 6;
          uint32_t lo32, hi32, ci, cp, ow, dummy;
          ll_get6(rq, tag, lo32, hi32, ci, cp, ow, dummy);
          o.v = __longlong_as_double((long long)((uint64_t(hi32) << 32) | lo32));
          o.idx = int(ci);
          o.perm = int(cp);
          oo = int(ow);
        }
        const bool ok = lane < Q && o.idx >= 0;
        const int id = warp_argmax_redux(o.v, o.idx, ok);
        const int wl = __ffs(__ballot_sync(0xffffffffu, ok && o.idx == id)) - 1;
        CCand gw;
        gw.v = __shfl_sync(0xffffffffu, o.v, wl);
        gw.idx = __shfl_sync(0xffffffffu, o.idx, wl);
        gw.perm = __shfl_sync(0xffffffffu, o.perm, wl);
        (void)oo;
        if (lane < C) st_async_cand(s.gwin + par, &s.xbar[2 + par], lane, gw);
      }
      mbar_wait_delivered(&s.xbar[2 + par], (uint32_t(g - r) >> 1) & 1u);
      w = s.gwin[par];
      owner = w.idx >= 0 ? (w.idx - row0) / R : 0;  // rows are dealt out contiguously
    }
    if (!a.pivot) {
      // unpivoted drivers (blocked.py:162-290, unblocked.py:192-226): the pivot row is
      // row a itself; the argmax above only says whether the column below g is all
      // zero, for the exact-zero breakdown test (ZeroPivot, unblocked.py:83-85)
      const bool colnz = w.idx >= 0 && w.v != 0.0;
      double va;
      int pa_perm;
      if (MULTI) {
        const uint64_t* ra = a.rowa + (size_t)par * a.slot_words;
        uint32_t p32, dummy;
        ll_get2(ra, tag, p32, dummy);
        pa_perm = int(p32);
        va = ll_get_double(ra + 4 + 2 * k, tag);
      } else {
        va = *cluster.map_shared_rank(s.pubA + par * (kmax + 2) + k, owner_a);
        pa_perm = *cluster.map_shared_rank(s.misc + par, owner_a);
      }
      if (colnz && va == 0.0 && gcta == 0 && tid == 0 && a.info != nullptr && *a.info == 0) *a.info = g + 1;
      w = CCand{va, a_pos, pa_perm};
      owner = owner_a;
    }
    const int b = w.idx, pb = w.perm;
    const double vb = w.v;
    const bool own_b = b >= rbase && b < rbase + rcount;
    const bool swapped = b != a_pos;
    const bool more = (g + 1 < rt) || a.want_y;
    int perm_a = 0;
    const bool need_a = !push && own_b && swapped;  // row b's owner receives row a
    const int lb_thread = (b - rbase) & (kCThreads - 1);
    SUBMARK(0);
    // gathers of the next column for every row but b (row b's physical index
    // perm_a arrives with row a; its gather is issued once that is known)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int li = tid + u * kCThreads;
      int pos = lab[u];  // == rbase + li unless push (then: the label after this step's swap)
      if (push && swapped) pos = pos == b ? a_pos : (pos == a_pos ? b : pos);
      cnext[u] = 0.0;
      cneg[u] = false;
      if (more && li < rcount && pos > a_pos && !(need_a && pos == b)) {
        const int ph = s.perm[li];
        // X(ph, pb) in skew-lower storage; the sign is applied when consumed
        cneg[u] = ph < pb;
        cnext[u] = cneg[u] ? W[(long long)ph * ld + pb] : W[(long long)pb * ld + ph];
      }
    }
    SUBMARK(1);
    if (push) {
      // the winner's row (pushed with its candidate) is read in place by phase 4
      mbar_wait_delivered(&s.xbar[2 + par], (uint32_t(g - r) >> 1) & 1u);
      xrow = s.crows + ((size_t)par * C + owner) * CRS;
    } else if (MULTI) {
      const uint64_t* gr = a.pivot ? a.slots + ((size_t)owner * 2 + par) * a.slot_words + 4
                                   : a.rowa + (size_t)par * a.slot_words + 4;
      const uint64_t* ra = a.rowa + (size_t)par * a.slot_words;
      if (need_a) {
        // pivot row, row a and row a's header polled together (one round trip)
        for (int j = tid; j <= k; j += kCThreads) ll_get_double2(gr + 2 * j, ra + 4 + 2 * j, tag, s.wrow[j], s.arow[j]);
        if (tid == lb_thread) {
          uint32_t pa32, dummy;
          ll_get2(ra, tag, pa32, dummy);
          perm_a = int(pa32);
        }
      } else {
        for (int j = tid; j <= k; j += kCThreads) s.wrow[j] = ll_get_double(gr + 2 * j, tag);
      }
    } else {
      const double* wr = a.pivot ? cluster.map_shared_rank(s.pubrow + par * (kmax + 2), owner)
                                 : cluster.map_shared_rank(s.pubA + par * (kmax + 2), owner_a);
      if (need_a) {
        const double* ar = cluster.map_shared_rank(s.pubA + par * (kmax + 2), owner_a);
        if (tid == lb_thread) perm_a = *cluster.map_shared_rank(s.misc + par, owner_a);
        for (int j = tid; j <= k; j += kCThreads) {
          const double wv = wr[j], av = ar[j];
          s.wrow[j] = wv;
          s.arow[j] = av;
        }
      } else {
        for (int j = tid; j <= k; j += kCThreads) s.wrow[j] = wr[j];
      }
    }
    SUBMARK(2);
    if (need_a && tid == lb_thread) {
      const int u = (b - rbase) >> 8;  // kCThreads == 256
#pragma unroll
      for (int uu = 0; uu < 2; ++uu)
        if (uu == u && more) {
          cneg[uu] = perm_a < pb;
          cnext[uu] = cneg[uu] ? W[(long long)perm_a * ld + pb] : W[(long long)pb * ld + perm_a];
        }
    }
    if (!push) __syncthreads();  // push: nothing phase 4 reads was written by another thread here
    CMARK(3);

    // ---- (4) interchange rows a/b, scale column k, z for the next step -------
    if (swapped && !push) {
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
      if (li < rcount && push) {
        // lazy interchange: labels a <-> b swap, the rows' data stay
        int pos = lab[u];
        if (swapped) {
          pos = pos == b ? a_pos : (pos == a_pos ? b : pos);
          lab[u] = pos;
        }
        if (pos == a_pos) {
          col[li] = 1.0;
        } else if (pos > a_pos) {
          const double v = col[li];
          col[li] = vb != 0.0 ? v / vb : v;
        }
      } else if (li < rcount) {
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
      const double xm = j >= 1 ? xrow[j - 1] : 0.0;
      const double xp = (j + 1 < k) ? xrow[j + 1] : (j + 1 == k ? 1.0 : 0.0);
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
        if (li < rcount && lab[u] > a_pos) {
          // eight independent FMA chains (the phase is bound by the chain latency)
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0, a5 = 0.0, a6 = 0.0, a7 = 0.0;
          int j = 0;
          if (u == 0 && nbank > 0) {
            const double2* z2 = reinterpret_cast<const double2*>(s.zbuf);
#pragma unroll
            for (int q = 0; q < kBank; q += 8) {
              const double2 za = z2[q >> 1], zb = z2[(q >> 1) + 1], zc = z2[(q >> 1) + 2], zd = z2[(q >> 1) + 3];
              a0 = fma(rb[0][q], za.x, a0);
              a1 = fma(rb[0][q + 1], za.y, a1);
              a2 = fma(rb[0][q + 2], zb.x, a2);
              a3 = fma(rb[0][q + 3], zb.y, a3);
              a4 = fma(rb[0][q + 4], zc.x, a4);
              a5 = fma(rb[0][q + 5], zc.y, a5);
              a6 = fma(rb[0][q + 6], zd.x, a6);
              a7 = fma(rb[0][q + 7], zd.y, a7);
            }
            if (nbank > 1) {
#pragma unroll
              for (int q = 0; q < kBank; q += 8) {
                const int h = (kBank + q) >> 1;
                const double2 za = z2[h], zb = z2[h + 1], zc = z2[h + 2], zd = z2[h + 3];
                a0 = fma(rb[1][q], za.x, a0);
                a1 = fma(rb[1][q + 1], za.y, a1);
                a2 = fma(rb[1][q + 2], zb.x, a2);
                a3 = fma(rb[1][q + 3], zb.y, a3);
                a4 = fma(rb[1][q + 4], zc.x, a4);
                a5 = fma(rb[1][q + 5], zc.y, a5);
                a6 = fma(rb[1][q + 6], zd.x, a6);
                a7 = fma(rb[1][q + 7], zd.y, a7);
              }
            }
            j = kBank * nbank;
          }
          for (; j + 7 < kk; j += 8) {
            a0 = fma(s.slab[(size_t)j * Rs + li], s.zbuf[j], a0);
            a1 = fma(s.slab[(size_t)(j + 1) * Rs + li], s.zbuf[j + 1], a1);
            a2 = fma(s.slab[(size_t)(j + 2) * Rs + li], s.zbuf[j + 2], a2);
            a3 = fma(s.slab[(size_t)(j + 3) * Rs + li], s.zbuf[j + 3], a3);
            a4 = fma(s.slab[(size_t)(j + 4) * Rs + li], s.zbuf[j + 4], a4);
            a5 = fma(s.slab[(size_t)(j + 5) * Rs + li], s.zbuf[j + 5], a5);
            a6 = fma(s.slab[(size_t)(j + 6) * Rs + li], s.zbuf[j + 6], a6);
            a7 = fma(s.slab[(size_t)(j + 7) * Rs + li], s.zbuf[j + 7], a7);
          }
          if (j + 3 < kk) {
            a0 = fma(s.slab[(size_t)j * Rs + li], s.zbuf[j], a0);
            a1 = fma(s.slab[(size_t)(j + 1) * Rs + li], s.zbuf[j + 1], a1);
            a2 = fma(s.slab[(size_t)(j + 2) * Rs + li], s.zbuf[j + 2], a2);
            a3 = fma(s.slab[(size_t)(j + 3) * Rs + li], s.zbuf[j + 3], a3);
            j += 4;
          }
          if (j + 1 < kk) {
            a4 = fma(s.slab[(size_t)j * Rs + li], s.zbuf[j], a4);
            a5 = fma(s.slab[(size_t)(j + 1) * Rs + li], s.zbuf[j + 1], a5);
            j += 2;
          }
          if (j < kk) a6 = fma(s.slab[(size_t)j * Rs + li], s.zbuf[j], a6);
          s.az[li] = kk >= 2 ? ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7)) : 0.0;
        }
      }
    }
    CMARK(4);
  }
  __syncthreads();
  if (cta == 0) {
    for (int g = r + tid; g < rt; g += kCThreads) {
      a.tau[g] = s.taus[g - lo];
      if (a.piv != nullptr) a.piv[g + 1] = (long long)s.pivbuf[g - r];
    }
  }
  if (a.prof && tid == 0) {
    for (int i = 0; i < 6; ++i) a.prof[cta * 16 + i] += (unsigned long long)pt[i];
    for (int i = 0; i < 3; ++i) a.prof[cta * 16 + 12 + i] += (unsigned long long)sub[i];
    a.prof[cta * 16 + 6] += (unsigned long long)(rt - r);
    a.prof[cta * 16 + 8] += (unsigned long long)(t_loop0 - t_kernel0);
    a.prof[cta * 16 + 9] += (unsigned long long)(clock64() - t_prev);
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int li = tid + u * kCThreads;
    if (li < rcount) {
      s.lab[li] = lab[u];
      if (a.want_y) s.ycol[li] = cneg[u] ? -cnext[u] : cnext[u];
    }
  }
  __syncthreads();

  // ---- var1: y = column rt after the couplings (straggler operand) --------
  if (a.want_y && rt < n) {
    for (int li = tid; li < rcount; li += kCThreads)
      if (s.lab[li] >= rt + 1) a.y[s.lab[li]] = s.ycol[li] - s.az[li];
  }

  // ---- materialise displaced trailing lines, write back ------------------
  for (int li = tid; li < rcount; li += kCThreads) {
    int pos = s.lab[li], ph = s.perm[li];
    a.gperm[pos] = ph;
    if (pos >= rt && ph != pos) {
      int q = atomicAdd(a.disp_count, 1);
      a.disp_list[q] = pos;
    }
  }
  if (cta == 0) {
    for (int i = tid; i < row0; i += kCThreads) a.gperm[i] = i;
  }
  const long long t_tail1 = clock64();
  {
    // the slab goes to the panel buffer; panel_finish_* (separate grid-wide launches,
    // also the ordering point) materialise the displaced lines and write the L
    // columns with every SM instead of this kernel's 16: the displaced lines are
    // row accesses of column-major storage (one sector per element)
    for (int li = tid; li < rcount; li += kCThreads) {
      double* dst = a.pbuf + s.lab[li];
      int j = 0;
      for (; j + 8 <= kmax; j += 8) {  // 8 loads in flight, then 8 streaming stores
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = s.slab[(size_t)(j + u) * Rs + li];
#pragma unroll
        for (int u = 0; u < 8; ++u) __stcs(dst + (size_t)(j + u) * n, v[u]);
      }
      for (; j < kmax; ++j) __stcs(dst + (size_t)j * n, s.slab[(size_t)j * Rs + li]);
    }
    if (a.prof && tid == 0) {
      const long long t_end = clock64();
      a.prof[cta * 16 + 7] += (unsigned long long)(t_end - t_kernel0);
      a.prof[cta * 16 + 10] += (unsigned long long)(t_tail1 - t_kernel0);
      a.prof[cta * 16 + 11] += (unsigned long long)(t_end - t_tail1);
    }
    return;
  }
}

// MULTI panel epilogue, launch 1: displaced trailing lines -> side buffer (reads W only)
__global__ void panel_finish_gather(PanelArgs a) {
  const int n = a.n, rt = a.r + a.nelim, ntr = n - rt;
  const int nd = *a.disp_count;
  for (int q = blockIdx.y; q < nd; q += gridDim.y) {
    const int p = a.disp_list[q];
    const int pp = a.gperm[p];
    double* line = a.side + (size_t)q * ntr;
    for (int i = rt + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
      line[i - rt] = (i == p) ? 0.0 : skew_at(a.W, a.ld, a.gperm[i], pp);
  }
}

// MULTI panel epilogue, launch 2: panel buffer -> L columns [lo, rt); side -> trailing lines
__global__ void panel_finish_write(PanelArgs a) {
  const int n = a.n, lo = a.lo, rt = a.r + a.nelim, ntr = n - rt, row0 = lo + 1;
  const long long ld = a.ld;
  for (int j = blockIdx.y; j < a.kmax; j += gridDim.y) {
    const int c = lo + j;
    for (int pos = max(row0, c + 1) + blockIdx.x * blockDim.x + threadIdx.x; pos < n; pos += gridDim.x * blockDim.x)
      a.W[(long long)c * ld + pos] = a.pbuf[(size_t)j * n + pos];
  }
  const int nd = *a.disp_count;
  for (int q = blockIdx.y; q < nd; q += gridDim.y) {
    const int p = a.disp_list[q];
    const double* line = a.side + (size_t)q * ntr;
    for (int i = rt + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      const double v = line[i - rt];
      if (i > p)
        a.W[(long long)p * ld + i] = v;
      else if (i < p)
        a.W[(long long)i * ld + p] = -v;
    }
  }
}


// displaced trailing lines -> side buffer, then panel buffer -> L columns and
// side -> trailing lines (two launches: the gather must see the pre-panel W)
cudaError_t launch_panel_finish(const PanelArgs& a, cudaStream_t stream) {
  const int ntr = a.n - (a.r + a.nelim);
  dim3 grid(ntr > 0 ? (ntr + 255) / 256 : 1, 2 * (a.nelim + 1));
  if (grid.x > 16) grid.x = 16;
  panel_finish_gather<<<grid, 256, 0, stream>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 grid2(grid.x, a.kmax > 2 * (a.nelim + 1) ? a.kmax : 2 * (a.nelim + 1));
  panel_finish_write<<<grid2, 256, 0, stream>>>(a);
  return cudaGetLastError();
}


// The panel epilogue and the packing of the trailing update's operands as one cooperative
// kernel.  Phase A reads only: the displaced trailing lines go to the side buffer (they must
// see the pre-panel W), and P = -A, Q = A T^T (+ the var1 straggler pair) are packed
// straight from the panel buffer (by position, rows >= rt) -- the same values finish_write
// is about to copy into W's columns [lo, rt).  Grid barrier.  Phase B writes W: panel
// buffer -> L columns, side buffer -> trailing lines.  Three dependent ~6 us launches per
// panel become one.
__device__ __forceinline__ size_t fp_packed_elems(int rows, int k4cap) {
  return (size_t)tiles_for(rows) * kTile * 4 * k4cap;
}
__global__ void __launch_bounds__(256) panel_finish_pack_kernel(PanelArgs a, FinishPack f) {
  const int n = a.n, lo = a.lo, rt = a.r + a.nelim, ntr = n - rt, row0 = lo + 1;
  const long long ld = a.ld;
  const int nd = *a.disp_count;
  const int GX = min(16, max(1, (ntr + 255) / 256));  // row chunks of a line, as in the two-launch epilogue
  const int nb = int(gridDim.x);
  // ---- A1: displaced trailing lines -> side buffer
  for (int w = blockIdx.x; w < nd * GX; w += nb) {
    const int q = w / GX, bx = w - q * GX;
    const int p = a.disp_list[q];
    const int pp = a.gperm[p];
    double* line = a.side + (size_t)q * ntr;
    for (int i = rt + bx * 256 + threadIdx.x; i < n; i += GX * 256)
      line[i - rt] = (i == p) ? 0.0 : skew_at(a.W, a.ld, a.gperm[i], pp);
  }
  // ---- A2: packed operands from the panel buffer (pack_rankk_kernel, trailing.cu)
  if (f.rows > 0) {
    const double* A = a.pbuf + rt;  // A[row, col] = pbuf[col * n + rt + row]
    const size_t total = fp_packed_elems(f.rows + f.shift, f.k4cap);
    for (size_t off = blockIdx.x * (size_t)256 + threadIdx.x; off < total; off += (size_t)nb * 256) {
      const int lane = int(off & 31), mb = int((off >> 5) & 15);
      const size_t rest = off >> 9;
      const int qk = int(rest % (size_t)f.k4cap), tl = int(rest / (size_t)f.k4cap);
      const int row = tl * kTile + mb * 8 + (lane >> 2) - f.shift;
      const int col = qk * 4 + (lane & 3);
      double pv = 0.0, qv = 0.0;
      if (row >= 0 && row < f.rows) {
        if (col < f.ka) {
          const double* ar = A + row;
          pv = -1.0 * ar[(size_t)col * n];
          double acc = 0.0;
          if (col >= 1) acc = f.t[col - 1] * ar[(size_t)(col - 1) * n];
          if (col + 1 < f.ka) acc -= f.t[col] * ar[(size_t)(col + 1) * n];
          qv = acc;
        } else if (f.y != nullptr && row >= 1 && col < f.ka + 2) {
          const double lv = A[(size_t)(f.ka - 1) * n + row];
          const double yv = f.y[row];
          if (col == f.ka) {
            pv = lv;
            qv = yv;
          } else {
            pv = -yv;
            qv = lv;
          }
        }
      }
      f.P[off] = pv;
      f.Q[off] = qv;
    }
  }
  __threadfence();
  cg::this_grid().sync();
  // ---- B1: panel buffer -> L columns [lo, rt)
  const int GY = a.kmax;
  for (int w = blockIdx.x; w < GY * GX; w += nb) {
    const int j = w / GX, bx = w - j * GX;
    const int c = lo + j;
    for (int pos = max(row0, c + 1) + bx * 256 + threadIdx.x; pos < n; pos += GX * 256)
      a.W[(long long)c * ld + pos] = a.pbuf[(size_t)j * n + pos];
  }
  // ---- B2: side buffer -> trailing lines
  for (int w = blockIdx.x; w < nd * GX; w += nb) {
    const int q = w / GX, bx = w - q * GX;
    const int p = a.disp_list[q];
    const double* line = a.side + (size_t)q * ntr;
    for (int i = rt + bx * 256 + threadIdx.x; i < n; i += GX * 256) {
      const double v = line[i - rt];
      if (i > p)
        a.W[(long long)p * ld + i] = v;
      else if (i < p)
        a.W[(long long)i * ld + p] = -v;
    }
  }
  // every thread read the count at kernel entry: reset it for the next panel (its launcher
  // then skips the memset)
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.disp_count = 0;
}

// ===========================================================================
// panel_push_kernel: the single-cluster pivoted panel, rebuilt for the shortest
// per-elimination dependency chain (configs 1 and 2, and the tail panels of
// configs 3 and 5).  Same reference semantics and outputs as the push mode of
// panel_cluster_kernel<true> (lazy interchanges: slab rows never move, a row
// carries its position as a label), but:
//  * every per-row quantity lives in registers of the owning thread (label,
//    physical row, the next column's value, A z, this step's v), so the step
//    touches shared memory only for the slab columns, the candidates and z;
//  * the CTA candidate and the winner are found by every warp redundantly
//    (one exact 3-redux argmax each), so a step has exactly two CTA barriers;
//  * remote addresses (candidate slots, row slots, mbarriers of every peer)
//    are computed once (mapa) before the step loop;
//  * the candidate row push is laid out as (destination = tid % 16, pair =
//    tid / 16), so no integer division sits on the step;
//  * the column scaling v / vb runs on the value still in a register, in the
//    shadow of the pushed-row wait and the z barrier, and the gemv reads the
//    freshly scaled column k from that register;
//  * slab columns [0, 32 * NBANK) of a thread's row are register-cached.
// ===========================================================================
constexpr int kPThreads = 256;
constexpr int kPWarps = kPThreads / 32;
constexpr int kPC = 16;  // cluster size of the push panel

struct __align__(16) PCand {  // pushed to every CTA of the cluster
  double v;
  int pos;
  int ph;
};
struct __align__(16) PWCand {  // CTA-local warp candidate
  double v;
  int pos;
  int ph;
  int li;
  int pad[3];
};

__host__ __device__ inline int push_crs(int kmax) { return (kmax + 2) & ~1; }  // even -> 16-byte rows

struct PSmem {
  double* slab;   // [kmax][Rs]
  double* crows;  // [2][16][CRS]
  double* zbuf;   // [kmax + 2]
  double* taus;   // [kmax + 2]
  PCand* cand;    // [2][16]
  PWCand* wcand;  // [8]
  int* pivbuf;    // [kmax]
  uint64_t* xbar; // [4]: candidates (par), rows (2 + par)
};

// nslots: pivot-row slots per parity (1 with the multicast delivery, 16 with the DSMEM push)
__host__ __device__ inline size_t psmem_layout(int R, int kmax, PSmem* s, unsigned char* base, int nslots = 1) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 15) & ~size_t(15);
    return base ? base + o : nullptr;
  };
  const int Rs = cslab_stride(R);
  unsigned char* p;
  p = take(sizeof(double) * (size_t)kmax * Rs);
  if (s) s->slab = (double*)p;
  p = take(sizeof(double) * 2 * nslots * (size_t)push_crs(kmax));
  if (s) s->crows = (double*)p;
  p = take(sizeof(double) * (kmax + 10));  // + 8 zeroed spares: gemv_slab_cols reads z in groups of eight
  if (s) s->zbuf = (double*)p;
  p = take(sizeof(double) * (kmax + 2));
  if (s) s->taus = (double*)p;
  p = take(sizeof(PCand) * (2 * kPC + 4));  // + [2][2]: the global winner's record (multi-cluster panel)
  if (s) s->cand = (PCand*)p;
  p = take(sizeof(PWCand) * kPWarps);
  if (s) s->wcand = (PWCand*)p;
  p = take(sizeof(int) * (kmax + 2));
  if (s) s->pivbuf = (int*)p;
  p = take(sizeof(uint64_t) * 6);  // [4 + par]: winner record (multi-cluster panel)
  if (s) s->xbar = (uint64_t*)p;
  return off;
}

__device__ __forceinline__ uint32_t mapa_u32(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_v4(uint32_t rdst, uint32_t rbar, uint32_t a, uint32_t b, uint32_t c,
                                            uint32_t d) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   rdst),
               "r"(a), "r"(b), "r"(c), "r"(d), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_v2f64(uint32_t rdst, uint32_t rbar, double x, double y) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(rdst),
               "d"(x), "d"(y), "r"(rbar)
               : "memory");
}

// exact argmax of |v| over the lanes (ties -> lowest pos); returns the winning lane or -1.
// Fast path: one redux on the top 32 bits of |v| (+1, so a valid 0.0 beats an empty
// lane); when exactly one lane holds that top word it is the maximum.  Otherwise the
// low words and then the positions decide among the tied lanes (two more reduxes).
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

// A z over the shared-memory slab columns [j0, k) of one row (j0 even): eight column loads
// issued before the FMAs of a trip, columns >= k predicated off (z beyond k is zero or
// finite: zbuf carries eight spare zeroed entries), no remainder loop.  Chains by column % 4.
__device__ __forceinline__ void gemv_slab_cols(const double* __restrict__ sl, int Rs, const double2* __restrict__ z2,
                                               int j0, int k, double& c0, double& c1, double& c2, double& c3) {
  for (int j = j0; j < k; j += 8) {
    double x[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) x[e] = j + e < k ? sl[(size_t)(j + e) * Rs] : 0.0;
    const double2 za = z2[j >> 1], zb = z2[(j >> 1) + 1], zc = z2[(j >> 1) + 2], zd = z2[(j >> 1) + 3];
    c0 = fma(x[0], za.x, c0);
    c1 = fma(x[1], za.y, c1);
    c2 = fma(x[2], zb.x, c2);
    c3 = fma(x[3], zb.y, c3);
    c0 = fma(x[4], zc.x, c0);
    c1 = fma(x[5], zc.y, c1);
    c2 = fma(x[6], zd.x, c2);
    c3 = fma(x[7], zd.y, c3);
  }
}

// RPT rows per thread (TPR == 1), or TPR threads per row (RPT == 1): the TPR threads of a
// row are consecutive lanes; they hold the row's state redundantly and split the gemv's
// columns (j % TPR == part), combining the partial sums with xor-shuffles.  NBANK banks
// of 32 slab columns are register-cached (each of the TPR threads caches its 32/TPR).
// MCAST: pivot-row delivery.  0 = every CTA pushes its candidate row to every CTA by
// st.async; 1 = the winning CTA multicasts its row (written to a global slot during the
// exchange) once the winner is known; 2 = every CTA multicasts its candidate row straight
// from the row-major global mirror of the slab (a.rowmir, kept current by the owning
// threads) at the same time as it sends its candidate, so the rows travel during the
// candidate exchange and no delivery follows the winner.
template <int RPT, int NBANK, int TPR, int MCAST>
__global__ void __launch_bounds__(kPThreads, 1) panel_push_kernel(PanelArgs a) {
  static_assert(RPT == 1 || TPR == 1, "either rows per thread or threads per row");
  constexpr int RPB = kPThreads / TPR;   // rows per row-block of the CTA's threads
  constexpr int CPB = 32 / TPR;          // cached columns per bank and thread
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int crank = int(cg::this_cluster().block_rank());
  const int C = int(cg::this_cluster().num_blocks());  // <= 16
  constexpr int NSLOT = MCAST == 1 ? 1 : kPC;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int part = TPR > 1 ? (tid & (TPR - 1)) : 0;
  const int rowt = TPR > 1 ? tid / TPR : tid;  // this thread's (first) local row
  const int n = a.n, lo = a.lo, r = a.r, nelim = a.nelim, kmax = a.kmax;
  const int R = a.rows_per, Rs = cslab_stride(R);
  const long long ld = a.ld;
  const double* __restrict__ W = a.W;
  const int row0 = lo + 1;
  const int rbase = row0 + crank * R;
  const int rcount = max(0, min(R, n - rbase));
  const int rt = r + nelim;
  const int CRS = push_crs(kmax);
#ifdef SKL_PANEL_DBG_BUILD
  const int dbg = a.dbg;  // timing experiments only (make variant VFLAGS=-DSKL_PANEL_DBG_BUILD)
#else
  constexpr int dbg = 0;
#endif
  PSmem s;
  psmem_layout(R, kmax, &s, smem_raw, NSLOT);

  // the deliveries of step g complete on xbar[g & 1] (candidates) and xbar[2 + (g & 1)]
  // (pivot row); the last thread arms each barrier for step g + 2 as soon as step g's
  // wait returns, so no arming sits on warp 0's path to the candidate send
  constexpr int kArm = kPThreads - 1;
  auto row_bytes = [&](int gg) { return (MCAST == 1 ? 1u : uint32_t(C)) * 16u * uint32_t((gg - lo + 2) >> 1); };
  if (tid == kArm) {
    for (int i = 0; i < 4; ++i) mbar_init(&s.xbar[i], 1);
    fence_mbar_init();
    for (int gg = r; gg < rt && gg < r + 2; ++gg) {
      mbar_arrive_expect_tx(&s.xbar[gg & 1], uint32_t(C * sizeof(PCand)));
      mbar_arrive_expect_tx(&s.xbar[2 + (gg & 1)], row_bytes(gg));
    }
  }
  for (int j = tid; j < kmax + 10; j += kPThreads) {
    if (j < kmax + 2) s.taus[j] = (j == 0 && lo >= 0 && lo < n - 1) ? a.tau[lo] : 0.0;
    s.zbuf[j] = 0.0;
  }
#ifdef SKL_CHECKED
  assert(C >= 1 && C <= kPC && R <= RPT * RPB && kmax <= n && lo >= -1 && r >= lo && rt <= n - 1 + 1);
  assert(psmem_layout(R, kmax, nullptr, nullptr, MCAST == 1 ? 1 : kPC) <= 232448);
#endif
  // per-row state in registers: row li = rowt + u * RPB
  int lab[RPT], ph[RPT];
  double cn[RPT], az[RPT], vv[RPT];
  bool cneg[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int li = rowt + u * RPB;
    const int pos = rbase + li;
    lab[u] = li < rcount ? pos : -1;  // -1: no row (never a candidate, never written)
    ph[u] = pos;
    az[u] = 0.0;
    vv[u] = 0.0;
    cneg[u] = false;
    cn[u] = (li < rcount && pos > r) ? W[(long long)r * ld + pos] : 0.0;
    if (part == 0 && li < rcount && lo < r) {  // var2a carry column
      const double c0 = W[(long long)lo * ld + pos];
      s.slab[li] = c0;
      if (MCAST == 2) a.rowmir[(size_t)(crank * R + li) * CRS] = c0;
    }
  }
  double rb[RPT][CPB * NBANK];
  int nbank = 0;
  // remote addresses, fixed for the whole panel
  const uint32_t dst = uint32_t(tid & (kPC - 1));  // DSMEM push: this thread's destination CTA (if < C)
  const uint32_t dstc = dst < uint32_t(C) ? dst : 0u;
  const uint32_t r_crows = mapa_u32(smem_u32(s.crows), dstc);
  const uint32_t r_rbar0 = mapa_u32(smem_u32(&s.xbar[2]), dstc);
  const uint32_t r_rbar1 = mapa_u32(smem_u32(&s.xbar[3]), dstc);
  const uint32_t lanec = uint32_t(lane < C ? lane : 0);
  const uint32_t r_cand = mapa_u32(smem_u32(s.cand), lanec);
  const uint32_t r_cbar0 = mapa_u32(smem_u32(&s.xbar[0]), lanec);
  const uint32_t r_cbar1 = mapa_u32(smem_u32(&s.xbar[1]), lanec);
  cluster_barrier();  // barriers initialised and visible cluster-wide; smem initialised
#ifdef SKL_PANEL_PROFILE
  long long pp[13] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long wp[4] = {0, 0, 0, 0};
  long long tp = clock64();
#define PMARK(i)                \
  do {                          \
    long long _t = clock64();   \
    pp[i] += _t - tp;           \
    tp = _t;                    \
  } while (0)
#define PSUB(i)                 \
  do {                          \
    pp[i] += clock64() - tp;    \
  } while (0)
#else
#define PMARK(i) \
  do {           \
  } while (0)
#define PSUB(i) \
  do {          \
  } while (0)
#endif

  for (int g = r; g < rt; ++g) {
    const int k = g - lo;
    const int par = g & 1;
    const int np = (k + 2) >> 1;  // pairs of the pushed candidate row (values 0..k)
    const uint32_t phase = (uint32_t(g - r) >> 1) & 1u;
    double* col = s.slab + (size_t)k * Rs;
    PSUB(11);
    // ---- (1) v = c - A z; exact warp argmax --------------------------------
    double bv = 0.0;
    int bpos = -1, bph = 0, bli = 0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      if (lab[u] > g) {
        const double v = (cneg[u] ? -cn[u] : cn[u]) - az[u];
        vv[u] = v;
        if (part == 0) {
          col[rowt + u * RPB] = v;
          if (bpos < 0 || fabs(v) > fabs(bv)) {
            bv = v;
            bpos = lab[u];
            bph = ph[u];
            bli = rowt + u * RPB;
          }
        }
      }
    }
    PSUB(12);  // v computed (gathered value consumed)
    {
      const int wl = lane_argmax(bv, bpos, bpos >= 0);
      if (lane == (wl < 0 ? 0 : wl)) s.wcand[warp] = PWCand{bv, wl < 0 ? -1 : bpos, bph, bli, {0, 0, 0}};
    }
    PMARK(0);
    // mode 2: this thread's mirror stores of the previous step (long landed) become visible
    // to the bulk-copy engine before any thread of the CTA can issue this step's multicast
    if (MCAST == 2) asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    PMARK(1);
    // ---- (2) CTA candidate -> every CTA; its row -> every CTA ---------------
    {
      const PWCand mine = lane < kPWarps ? s.wcand[lane] : PWCand{0.0, -1, 0, 0, {0, 0, 0}};
      const int wl = lane_argmax(mine.v, mine.pos, lane < kPWarps && mine.pos >= 0);
      const int src = wl < 0 ? 0 : wl;
      const PWCand c = s.wcand[src];  // smem broadcast
      const int lc = wl < 0 ? 0 : c.li;
      if (warp == 0) {
        if (lane < C) {
          const unsigned long long vb64 = (unsigned long long)__double_as_longlong(wl < 0 ? 0.0 : c.v);
          st_async_v4(r_cand + uint32_t((par * kPC + crank) * sizeof(PCand)), par ? r_cbar1 : r_cbar0,
                      uint32_t(vb64), uint32_t(vb64 >> 32), uint32_t(wl < 0 ? -1 : c.pos), uint32_t(c.ph));
        }
      }
      // candidate row values [0, k] as pairs (DSMEM push; an LL-flagged L2 row slot polled by
      // every CTA was measured slower: ~1000 cycles per poll round on B200)
      // this thread -> CTA dst, pairs tid/16 + 16 i
      if (dbg & 8) {
      } else if (MCAST == 2) {
        // the candidate row, contiguous in the global mirror, to slot [par][crank] of every CTA
        if (tid == 32) {
          const double* src = a.rowmir + (size_t)(crank * R + lc) * CRS;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, "
              "[%3], %4;" ::"r"(smem_u32(s.crows + ((size_t)par * kPC + crank) * CRS)),
              "l"(src), "r"(16u * uint32_t(np)), "r"(smem_u32(&s.xbar[2 + par])),
              "h"((unsigned short)((1u << C) - 1u))
              : "memory");
        }
      } else if (MCAST == 1) {
        // the candidate row -> this CTA's global slot (warp 0, after the candidate send); if it
        // wins, ONE multicast bulk copy delivers it to all 16 CTAs (one L2 read, no DSMEM port
        // traffic: the speculative st.async push of 16 rows to 16 CTAs costs ~18 cycles per
        // row double on B200, the multicast is flat in the row length -- tools/probes/xchg3.cu)
        // (the proxy fence that orders these generic stores before the bulk copy's read is
        // issued only by the winning CTA's warp 0, right before the copy: the stores have
        // long landed by then, and the 15 other CTAs never wait on it)
        if (warp == 0) {
          double* gs = a.crow + ((size_t)par * kPC + crank) * CRS;  // global slots: [2][16][CRS]
          for (int j = lane; j <= k; j += 32) gs[j] = s.slab[(size_t)j * Rs + lc];
        }
      } else {
        const uint32_t rbar = par ? r_rbar1 : r_rbar0;
        const uint32_t rrow = r_crows + uint32_t(((par * kPC + crank) * CRS) * sizeof(double));
        for (int p = tid >> 4; dst < uint32_t(C) && p < np; p += kPThreads / kPC) {
          const int j0 = 2 * p;
          const double x0 = s.slab[(size_t)j0 * Rs + lc];
          const double x1 = j0 + 1 <= k ? s.slab[(size_t)(j0 + 1) * Rs + lc] : 0.0;
          st_async_v2f64(rrow + uint32_t(j0 * sizeof(double)), rbar, x0, x1);
        }
      }
    }
    PMARK(2);
    // ---- (3) winner ---------------------------------------------------------
    mbar_wait_delivered(&s.xbar[par], phase);
    if (tid == kArm && g + 2 < rt) mbar_arrive_expect_tx(&s.xbar[par], uint32_t(C * sizeof(PCand)));
    PMARK(3);
#ifdef SKL_PANEL_PROFILE
    const long long wt0 = clock64();
#endif
    const PCand* cs = s.cand + par * kPC;
    int owner;
    {
      const PCand mine = lane < C ? cs[lane] : PCand{0.0, -1, 0};
      owner = lane_argmax(mine.v, mine.pos, lane < C && mine.pos >= 0);
      if (owner < 0) owner = 0;
    }
    if (MCAST == 1 && owner == crank && warp == 0 && !(dbg & 8)) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncwarp();
    }
    if (MCAST == 1 && owner == crank && tid == 0 && !(dbg & 8)) {
      const double* src = a.crow + ((size_t)par * kPC + crank) * CRS;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
          "%4;" ::"r"(smem_u32(s.crows + (size_t)par * CRS)),
          "l"(src), "r"(16u * uint32_t(np)), "r"(smem_u32(&s.xbar[2 + par])), "h"((unsigned short)((1u << C) - 1u))
          : "memory");
    }
    const PCand w = cs[owner];
    const int a_pos = g + 1, b = w.pos, pb = w.ph;
    const double vb = w.v;
#ifdef SKL_CHECKED
    // checked build (make variant V=checked VFLAGS=-DSKL_CHECKED): the invariants the
    // exchange relies on -- a real winner below g, inside the panel's rows, identical
    // in every CTA (each CTA re-derives it from the same delivered candidates)
    assert(owner >= 0 && owner < C);
    assert(b >= a_pos && b < n && pb >= row0 && pb < n);
    assert(w.pos == cs[owner].pos);
#endif
    const bool swapped = b != a_pos;
    const bool more = (g + 1 < rt) || a.want_y;
    // lazy interchange a_pos <-> b, then the next column's gathers (X(ph, pb), skew-lower)
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      if (swapped) lab[u] = lab[u] == b ? a_pos : (lab[u] == a_pos ? b : lab[u]);
      cneg[u] = ph[u] < pb;
      if (more && lab[u] > a_pos && !(dbg & 16)) {
        if (dbg & 1)  // timing experiment only: a contiguous, cache-hot gather (wrong values)
          cn[u] = W[(long long)r * ld + rbase + rowt + u * RPB];
        else if (dbg & 64)  // timing experiment only: every gather from column pb (mirrored-storage proxy)
          cn[u] = W[(long long)pb * ld + ph[u]];
        else
          cn[u] = cneg[u] ? W[(long long)ph[u] * ld + pb] : W[(long long)pb * ld + ph[u]];
        if (dbg & 32) {
          // remote-gather proxy: the gathered value additionally waits on a chain of
          // (dbg >> 8) dependent L2 loads (peer-memory latency stand-in, timing only)
          long long idx = (long long)pb * ld + ph[u];
          double acc = 0.0;
          for (int h = 0; h < (dbg >> 8); ++h) {
            const double t = __ldcg(W + (idx & ((1ll << 20) - 1)));  // within the first 8 MB of W
            acc += t * 0.0;
            idx += 1 + (long long)(t != t);
          }
          cn[u] += acc;
        }
      }
    }
    // column k: explicit 1 at a_pos, v / vb below (the value is still in a register)
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      if (lab[u] == a_pos) {
        vv[u] = 1.0;
        if (part == 0) col[rowt + u * RPB] = 1.0;
      } else if (lab[u] > a_pos) {
        const double sv = (dbg & 4) ? vv[u] : (vb != 0.0 ? vv[u] / vb : vv[u]);
        vv[u] = sv;
        if (part == 0) {
          col[rowt + u * RPB] = sv;
          // dbg 128 (timing only): no mirror store.  (Issuing this store behind the z barrier
          // instead measured +0.09 ms on config 2.)
          if (MCAST == 2 && !(dbg & 128)) a.rowmir[(size_t)(crank * R + rowt + u * RPB) * CRS + k] = sv;
        }
      }
    }
    PMARK(4);
#ifdef SKL_PANEL_PROFILE
    const long long wt1 = clock64();
#endif
    // ---- (4) z = T x for the next column (x = pivot row, pushed) -----------
    if (!(dbg & 8)) mbar_wait_delivered(&s.xbar[2 + par], phase);
#ifdef SKL_PANEL_PROFILE
    const long long wt2 = clock64();
#endif
    if (tid == kArm && g + 2 < rt && !(dbg & 8)) mbar_arrive_expect_tx(&s.xbar[2 + par], row_bytes(g + 2));
    PMARK(5);
    if (more) {
      const double* xrow = s.crows + ((size_t)par * NSLOT + (MCAST == 1 ? 0 : owner)) * CRS;
      for (int j = tid; j <= k; j += kPThreads) {
        const double xm = j >= 1 ? xrow[j - 1] : 0.0;
        const double xp = (j + 1 < k) ? xrow[j + 1] : (j + 1 == k ? 1.0 : 0.0);
        const double tj = j == k ? vb : s.taus[j];
        const double tj1 = (j + 1 == k) ? vb : s.taus[j + 1];
        s.zbuf[j] = (j >= 1 ? tj * xm : 0.0) - (j + 1 <= k ? tj1 * xp : 0.0);
      }
    }
    if (tid == 0) {
      s.pivbuf[g - r] = b - a_pos;
      s.taus[k] = vb;
    }
#ifdef SKL_PANEL_PROFILE
    const long long wt3 = clock64();
#endif
    __syncthreads();
#ifdef SKL_PANEL_PROFILE
    if (lane == 0) {  // per warp: winner..scale, pivot-row wait, z, wait at the second barrier
      const long long wt4 = clock64();
      wp[0] += wt1 - wt0;
      wp[1] += wt2 - wt1;
      wp[2] += wt3 - wt2;
      wp[3] += wt4 - wt3;
    }
#endif
    PMARK(6);
    if (!more) break;
    // ---- (5) A z for the next column: kk = k + 1 columns ---------------------
    const int kk = k + 1;
    if (nbank < NBANK && k >= 32 * (nbank + 1)) {
      // columns [32 nbank, 32 nbank + 32) are final: cache this thread's share of them
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int li = rowt + u * RPB;
#pragma unroll
        for (int b2 = 0; b2 < NBANK; ++b2)
          if (b2 == nbank) {
#pragma unroll
            for (int q = 0; q < CPB; ++q) rb[u][CPB * b2 + q] = s.slab[(size_t)(32 * b2 + part + TPR * q) * Rs + li];
          }
      }
      ++nbank;
    }
    if (dbg & 2) continue;  // timing experiment only: no gemv
    const double zk = s.zbuf[k];
    PSUB(8);
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int li = rowt + u * RPB;
      double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
      if (lab[u] > a_pos) {
#pragma unroll
        for (int b2 = 0; b2 < NBANK; ++b2) {
          if (b2 < nbank) {
            if constexpr (TPR == 1) {
              const double2* z2 = reinterpret_cast<const double2*>(s.zbuf);
#pragma unroll
              for (int q = 0; q < 32; q += 4) {
                const double2 za = z2[(32 * b2 + q) >> 1], zb = z2[((32 * b2 + q) >> 1) + 1];
                c0 = fma(rb[u][32 * b2 + q], za.x, c0);
                c1 = fma(rb[u][32 * b2 + q + 1], za.y, c1);
                c2 = fma(rb[u][32 * b2 + q + 2], zb.x, c2);
                c3 = fma(rb[u][32 * b2 + q + 3], zb.y, c3);
              }
            } else {
#pragma unroll
              for (int q = 0; q < CPB; q += 2) {
                c0 = fma(rb[u][CPB * b2 + q], s.zbuf[32 * b2 + part + TPR * q], c0);
                if (q + 1 < CPB) c1 = fma(rb[u][CPB * b2 + q + 1], s.zbuf[32 * b2 + part + TPR * (q + 1)], c1);
              }
            }
          }
        }
        PSUB(9);
        const double* sl = s.slab + li;
        if constexpr (TPR == 1) {
          gemv_slab_cols(sl, Rs, reinterpret_cast<const double2*>(s.zbuf), 32 * nbank, k, c0, c1, c2, c3);
          c1 = fma(vv[u], zk, c1);  // column k, freshly scaled, from the register
        } else {
          // four predicated column loads per trip, all issued before the FMAs (a short
          // dependent LDS -> FMA chain: with TPR threads per row a thread has few columns)
          for (int j = 32 * nbank + part; j < k; j += 4 * TPR) {
            double x[4], zz[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int jj = j + e * TPR;
              x[e] = jj < k ? sl[(size_t)jj * Rs] : 0.0;
              zz[e] = jj < k ? s.zbuf[jj] : 0.0;
            }
            c0 = fma(x[0], zz[0], c0);
            c1 = fma(x[1], zz[1], c1);
            c2 = fma(x[2], zz[2], c2);
            c3 = fma(x[3], zz[3], c3);
          }
          if (part == 0) c1 = fma(vv[u], zk, c1);
        }
      }
      PSUB(10);
      double t = (c0 + c1) + (c2 + c3);
      if constexpr (TPR > 1) {
#pragma unroll
        for (int o = 1; o < TPR; o <<= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      }
      if (lab[u] > a_pos) az[u] = kk >= 2 ? t : 0.0;
    }
    PMARK(7);
  }
#ifdef SKL_PANEL_PROFILE
  if (a.prof && tid == 0) {
    for (int i = 0; i < 8; ++i) a.prof[crank * 16 + i] += (unsigned long long)pp[i];
    a.prof[crank * 16 + 8] += (unsigned long long)(rt - r);
    for (int i = 8; i < 13; ++i) a.prof[crank * 16 + 1 + i] += (unsigned long long)pp[i];
  }
  if (a.prof && lane == 0 && crank < 16)  // rows 32..159: per (CTA, warp) sub-phase clocks
    for (int i = 0; i < 4; ++i) a.prof[(32 + crank * kPWarps + warp) * 16 + i] += (unsigned long long)wp[i];
#endif
#undef PMARK
#undef PSUB
  __syncthreads();
  // ---- outputs: tau / pivots, y (var1 straggler), position map, panel buffer ----
  if (crank == 0) {
    for (int g = r + tid; g < rt; g += kPThreads) {
      a.tau[g] = s.taus[g - lo];
      if (a.piv != nullptr) a.piv[g + 1] = (long long)s.pivbuf[g - r];
    }
    for (int i = tid; i < row0; i += kPThreads) a.gperm[i] = i;
  }
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int li = rowt + u * RPB;
    if (li < rcount && part == 0) {
      const int pos = lab[u];
#ifdef SKL_CHECKED
      assert(pos >= row0 && pos < n && ph[u] >= row0 && ph[u] < n);
#endif
      if (a.want_y && rt < n && pos >= rt + 1) a.y[pos] = (cneg[u] ? -cn[u] : cn[u]) - az[u];
      a.gperm[pos] = ph[u];
      if (pos >= rt && ph[u] != pos) {
        const int q = atomicAdd(a.disp_count, 1);
        a.disp_list[q] = pos;
      }
    }
  }
  // panel buffer (by position); the TPR threads of a row split its columns
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int li = rowt + u * RPB;
    if (li < rcount) {
      double* dstp = a.pbuf + lab[u];
      for (int j = part; j < kmax; j += TPR) __stcs(dstp + (size_t)j * n, s.slab[(size_t)j * Rs + li]);
    }
  }
  // no CTA may exit while a peer can still st.async into its shared memory: every
  // delivery of the last step has been waited on above, and nothing is sent after it
}


// ===========================================================================
// panel_multi2_kernel: the pivoted panel on Q co-resident clusters of C CTAs
// (tall panels of configs 3 and 5), on the lean structure of panel_push_kernel.
// Per step: the intra-cluster exchange is panel_push_kernel's (candidates by
// st.async, every CTA re-derives its cluster's winner); the CTA holding a
// cluster's winner publishes ONE record {v, position, physical row} and the
// winner's row [0, k] as LL-flagged words (value + step tag, no fence needed)
// into its cluster's L2 slot; warp 0 of every CTA polls the Q records (one lane
// each) and picks the global winner; every thread j <= k polls the two words of
// the winning row that z_j needs.  Two L2 round trips per step (record, row)
// instead of the leader relay + separate pivot-row and row-a exchanges of
// panel_cluster_kernel<MULTI>.
// ===========================================================================
template <int RPT, int NBANK>
__global__ void __launch_bounds__(kPThreads, 1) panel_multi2_kernel(PanelArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const int C = int(cluster.num_blocks());
  const int crank = int(cluster.block_rank());
  const int gcta = blockIdx.x;
  const int Q = int(gridDim.x) / C;
  const int qid = gcta / C;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n, lo = a.lo, r = a.r, nelim = a.nelim, kmax = a.kmax;
  const int R = a.rows_per, Rs = cslab_stride(R);
  const long long ld = a.ld;
  const double* __restrict__ W = a.W;
  const int row0 = lo + 1;
  const int rbase = row0 + gcta * R;
  const int rcount = max(0, min(R, n - rbase));
  const int rt = r + nelim;
  PSmem s;
  psmem_layout(R, kmax, &s, smem_raw, 3);
  // the winning cluster's L2 slot (record: 3 flagged pairs; row: k+1 flagged doubles)
  // lands here by one multicast bulk copy issued by the cluster leader, per parity
  const int SW = 6 + 2 * (kmax + 1);
  uint64_t* mslot = reinterpret_cast<uint64_t*>(s.crows);
  constexpr int kArm = kPThreads - 1;
  auto slot_bytes = [&](int gg) { return uint32_t(sizeof(uint64_t)) * uint32_t(6 + 2 * (gg - lo + 1)); };
  if (tid == kArm) {
    for (int i = 0; i < 6; ++i) mbar_init(&s.xbar[i], 1);
    fence_mbar_init();
    for (int gg = r; gg < rt && gg < r + 2; ++gg) {
      mbar_arrive_expect_tx(&s.xbar[gg & 1], uint32_t(C * sizeof(PCand)));
      mbar_arrive_expect_tx(&s.xbar[2 + (gg & 1)], slot_bytes(gg));
      mbar_arrive_expect_tx(&s.xbar[4 + (gg & 1)], uint32_t(2 * sizeof(PCand)));
    }
  }
  for (int j = tid; j < kmax + 10; j += kPThreads) {
    if (j < kmax + 2) s.taus[j] = (j == 0 && lo >= 0 && lo < n - 1) ? a.tau[lo] : 0.0;
    s.zbuf[j] = 0.0;
  }
  int lab[RPT], ph[RPT];
  double cn[RPT], az[RPT], vv[RPT];
  bool cneg[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int li = tid + u * kPThreads;
    const int pos = rbase + li;
    lab[u] = li < rcount ? pos : -1;
    ph[u] = pos;
    az[u] = 0.0;
    vv[u] = 0.0;
    cneg[u] = false;
    cn[u] = (li < rcount && pos > r) ? W[(long long)r * ld + pos] : 0.0;
    if (li < rcount && lo < r) s.slab[li] = W[(long long)lo * ld + pos];
  }
  double rb[RPT][32 * NBANK];
  int nbank = 0;
  const uint32_t lanec = uint32_t(lane < C ? lane : 0);
  const uint32_t r_cand = mapa_u32(smem_u32(s.cand), lanec);
  const uint32_t r_cbar0 = mapa_u32(smem_u32(&s.xbar[0]), lanec);
  const uint32_t r_cbar1 = mapa_u32(smem_u32(&s.xbar[1]), lanec);
  const uint32_t r_wbar0 = mapa_u32(smem_u32(&s.xbar[4]), lanec);
  const uint32_t r_wbar1 = mapa_u32(smem_u32(&s.xbar[5]), lanec);
  cluster_barrier();
#ifdef SKL_PANEL_PROFILE
  long long pp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tp = clock64();
#define QMARK(i)              \
  do {                        \
    long long _t = clock64(); \
    pp[i] += _t - tp;         \
    tp = _t;                  \
  } while (0)
#else
#define QMARK(i) \
  do {           \
  } while (0)
#endif

  for (int g = r; g < rt; ++g) {
    const int k = g - lo;
    const int par = g & 1;
    const uint32_t phase = (uint32_t(g - r) >> 1) & 1u;
    const uint32_t tag = a.tag0 + uint32_t(g - r);
    double* col = s.slab + (size_t)k * Rs;
    // ---- (1) v = c - A z; exact warp argmax --------------------------------
    double bv = 0.0;
    int bpos = -1, bph = 0, bli = 0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      if (lab[u] > g) {
        const double v = (cneg[u] ? -cn[u] : cn[u]) - az[u];
        vv[u] = v;
        col[tid + u * kPThreads] = v;
        if (bpos < 0 || fabs(v) > fabs(bv)) {
          bv = v;
          bpos = lab[u];
          bph = ph[u];
          bli = tid + u * kPThreads;
        }
      }
    }
    {
      const int wl = lane_argmax(bv, bpos, bpos >= 0);
      if (lane == (wl < 0 ? 0 : wl)) s.wcand[warp] = PWCand{bv, wl < 0 ? -1 : bpos, bph, bli, {0, 0, 0}};
    }
    __syncthreads();
    QMARK(0);
    // ---- (2) CTA candidate -> every CTA of the cluster ------------------------
    int lc;
    {
      const PWCand mine = lane < kPWarps ? s.wcand[lane] : PWCand{0.0, -1, 0, 0, {0, 0, 0}};
      const int wl = lane_argmax(mine.v, mine.pos, lane < kPWarps && mine.pos >= 0);
      const PWCand c = s.wcand[wl < 0 ? 0 : wl];
      lc = wl < 0 ? 0 : c.li;
      if (warp == 0 && lane < C) {
        const unsigned long long vb64 = (unsigned long long)__double_as_longlong(wl < 0 ? 0.0 : c.v);
        st_async_v4(r_cand + uint32_t((par * kPC + crank) * sizeof(PCand)), par ? r_cbar1 : r_cbar0,
                    uint32_t(vb64), uint32_t(vb64 >> 32), uint32_t(wl < 0 ? -1 : c.pos), uint32_t(c.ph));
      }
    }
    QMARK(1);
    // ---- (3) cluster winner; its CTA publishes record + row to the cluster's L2 slot
    mbar_wait_delivered(&s.xbar[par], phase);
    QMARK(2);
    if (tid == kArm && g + 2 < rt) mbar_arrive_expect_tx(&s.xbar[par], uint32_t(C * sizeof(PCand)));
    {
      const PCand* cs = s.cand + par * kPC;
      const PCand mine = lane < C ? cs[lane] : PCand{0.0, -1, 0};
      int cown = lane_argmax(mine.v, mine.pos, lane < C && mine.pos >= 0);
      if (cown < 0) cown = 0;
      if (cown == crank) {
        const PCand cw = cs[cown];
        uint64_t* slot = a.slots + ((size_t)qid * 2 + par) * a.slot_words;
        if (tid == 0) {
          const unsigned long long vb64 = (unsigned long long)__double_as_longlong(cw.v);
          ll_put2(slot, uint32_t(vb64), uint32_t(vb64 >> 32), tag);
          ll_put2(slot + 2, uint32_t(cw.pos), uint32_t(cw.ph), tag);
          ll_put2(slot + 4, uint32_t(qid), 0u, tag);
        }
        for (int j = tid; j <= k; j += kPThreads) ll_put_double(slot + 6 + 2 * j, s.slab[(size_t)j * Rs + lc], tag);
      }
    }
    QMARK(3);
    // ---- (4) global winner: the cluster leader's warp 0 polls the Q records (one lane
    // each) and multicasts the winning cluster's slot -- record and row -- into every
    // CTA of its cluster; the copy is checked against the step tag (L2 fallback) ------
    if (crank == 0 && warp == 0) {
      PCand rec{0.0, -1, 0};
      if (lane < Q) {
        const uint64_t* slot = a.slots + ((size_t)lane * 2 + par) * a.slot_words;
        uint32_t vlo, vhi, pp, pph;
        ll_get4(slot, tag, vlo, vhi, pp, pph);  // both flagged pairs in one poll round
        rec = PCand{__longlong_as_double((long long)((uint64_t(vhi) << 32) | vlo)), int(pp), int(pph)};
      }
      const int gl = lane_argmax(rec.v, rec.pos, lane < Q && rec.pos >= 0);
      // the winning record straight to the CTAs of this cluster by st.async (it is what the
      // interchange, the gathers and the scaling wait for); the row follows by the multicast
      // and is only needed for z
      {
        const int src = gl < 0 ? 0 : gl;
        const unsigned long long vw = (unsigned long long)__double_as_longlong(__shfl_sync(0xffffffffu, rec.v, src));
        const int posw = __shfl_sync(0xffffffffu, rec.pos, src);
        const int phw = __shfl_sync(0xffffffffu, rec.ph, src);
        if (lane < C) {
          const uint32_t rdst = r_cand + uint32_t((2 * kPC + 2 * par) * sizeof(PCand));
          const uint32_t rbar = par ? r_wbar1 : r_wbar0;
          st_async_v4(rdst, rbar, uint32_t(vw), uint32_t(vw >> 32), uint32_t(posw), uint32_t(phw));
          st_async_v4(rdst + uint32_t(sizeof(PCand)), rbar, uint32_t(src), 0u, 0u, 0u);
        }
      }
      if (lane == 0) {
        const uint64_t* src = a.slots + ((size_t)(gl < 0 ? 0 : gl) * 2 + par) * a.slot_words;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, "
            "[%3], %4;" ::"r"(smem_u32(mslot + (size_t)par * SW)),
            "l"(src), "r"(slot_bytes(g)), "r"(smem_u32(&s.xbar[2 + par])), "h"((unsigned short)((1u << C) - 1u))
            : "memory");
      }
    }
    QMARK(3);
    mbar_wait_delivered(&s.xbar[4 + par], phase);
    if (tid == kArm && g + 2 < rt) mbar_arrive_expect_tx(&s.xbar[4 + par], uint32_t(2 * sizeof(PCand)));
    const uint64_t* ms = mslot + (size_t)par * SW;
    PCand w;
    int wq;
    {
      const PCand* ws2 = s.cand + 2 * kPC + 2 * par;
      w = ws2[0];
      wq = *reinterpret_cast<const int*>(ws2 + 1);
    }
    QMARK(4);
    const int a_pos = g + 1, b = w.pos, pb = w.ph;
    const double vb = w.v;
    const bool swapped = b != a_pos;
    const bool more = (g + 1 < rt) || a.want_y;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      if (swapped) lab[u] = lab[u] == b ? a_pos : (lab[u] == a_pos ? b : lab[u]);
      cneg[u] = ph[u] < pb;
      if (more && lab[u] > a_pos) cn[u] = cneg[u] ? W[(long long)ph[u] * ld + pb] : W[(long long)pb * ld + ph[u]];
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      if (lab[u] == a_pos) {
        vv[u] = 1.0;
        col[tid + u * kPThreads] = 1.0;
      } else if (lab[u] > a_pos) {
        const double sv = vb != 0.0 ? vv[u] / vb : vv[u];
        vv[u] = sv;
        col[tid + u * kPThreads] = sv;
      }
    }
    QMARK(5);
    // ---- (5) z = T x (x = the winning row, from the multicast copy) ----------------
    mbar_wait_delivered(&s.xbar[2 + par], phase);
    if (tid == kArm && g + 2 < rt) mbar_arrive_expect_tx(&s.xbar[2 + par], slot_bytes(g + 2));
    if (more) {
      const uint64_t* xs = ms + 6;
      const uint64_t* xr = a.slots + ((size_t)wq * 2 + par) * a.slot_words + 6;
      auto xval = [&](int j) {
        const uint64_t lo = xs[2 * j], hi = xs[2 * j + 1];
        if (uint32_t(lo >> 32) == tag && uint32_t(hi >> 32) == tag)
          return __longlong_as_double((long long)((uint64_t(uint32_t(hi)) << 32) | uint32_t(lo)));
        return ll_get_double(xr + 2 * j, tag);  // fallback through L2 (never seen)
      };
      for (int j = tid; j <= k; j += kPThreads) {
        const double xm = j >= 1 ? xval(j - 1) : 0.0;
        const double xp = (j + 1 < k) ? xval(j + 1) : (j + 1 == k ? 1.0 : 0.0);
        const double tj = j == k ? vb : s.taus[j];
        const double tj1 = (j + 1 == k) ? vb : s.taus[j + 1];
        s.zbuf[j] = (j >= 1 ? tj * xm : 0.0) - (j + 1 <= k ? tj1 * xp : 0.0);
      }
    }
    if (tid == 0) {
      s.pivbuf[g - r] = b - a_pos;
      s.taus[k] = vb;
    }
    __syncthreads();
    QMARK(6);
    if (!more) break;
    // ---- (6) A z for the next column ---------------------------------------------
    const int kk = k + 1;
    if (nbank < NBANK && k >= 32 * (nbank + 1)) {
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int li = tid + u * kPThreads;
#pragma unroll
        for (int b2 = 0; b2 < NBANK; ++b2)
          if (b2 == nbank) {
#pragma unroll
            for (int q = 0; q < 32; ++q) rb[u][32 * b2 + q] = s.slab[(size_t)(32 * b2 + q) * Rs + li];
          }
      }
      ++nbank;
    }
    const double2* z2 = reinterpret_cast<const double2*>(s.zbuf);
    const double zk = s.zbuf[k];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int li = tid + u * kPThreads;
      if (lab[u] > a_pos) {
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
#pragma unroll
        for (int b2 = 0; b2 < NBANK; ++b2) {
          if (b2 < nbank) {
#pragma unroll
            for (int q = 0; q < 32; q += 4) {
              const double2 za = z2[(32 * b2 + q) >> 1], zb = z2[((32 * b2 + q) >> 1) + 1];
              c0 = fma(rb[u][32 * b2 + q], za.x, c0);
              c1 = fma(rb[u][32 * b2 + q + 1], za.y, c1);
              c2 = fma(rb[u][32 * b2 + q + 2], zb.x, c2);
              c3 = fma(rb[u][32 * b2 + q + 3], zb.y, c3);
            }
          }
        }
        const double* sl = s.slab + li;
        gemv_slab_cols(sl, Rs, z2, 32 * nbank, k, c0, c1, c2, c3);
        c1 = fma(vv[u], zk, c1);
        az[u] = kk >= 2 ? (c0 + c1) + (c2 + c3) : 0.0;
      }
    }
    QMARK(7);
  }
#ifdef SKL_PANEL_PROFILE
  if (a.prof && tid == 0 && gcta < 160) {
    for (int i = 0; i < 8; ++i) a.prof[gcta * 16 + i] += (unsigned long long)pp[i];
    a.prof[gcta * 16 + 8] += (unsigned long long)(rt - r);
  }
#endif
#undef QMARK
  __syncthreads();
  if (gcta == 0) {
    for (int g = r + tid; g < rt; g += kPThreads) {
      a.tau[g] = s.taus[g - lo];
      if (a.piv != nullptr) a.piv[g + 1] = (long long)s.pivbuf[g - r];
    }
    for (int i = tid; i < row0; i += kPThreads) a.gperm[i] = i;
  }
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int li = tid + u * kPThreads;
    if (li < rcount) {
      const int pos = lab[u];
      if (a.want_y && rt < n && pos >= rt + 1) a.y[pos] = (cneg[u] ? -cn[u] : cn[u]) - az[u];
      a.gperm[pos] = ph[u];
      if (pos >= rt && ph[u] != pos) {
        const int q = atomicAdd(a.disp_count, 1);
        a.disp_list[q] = pos;
      }
      double* dstp = a.pbuf + pos;
      for (int j = 0; j < kmax; ++j) __stcs(dstp + (size_t)j * n, s.slab[(size_t)j * Rs + li]);
    }
  }
}

}  // namespace

cudaError_t launch_panel_finish_pack(const PanelArgs& a, const FinishPack& f, cudaStream_t stream) {
  static int maxgrid = 0;
  if (!maxgrid) {
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, panel_finish_pack_kernel, 256, 0) != cudaSuccess || per < 1)
      per = 1;
    maxgrid = nsm * (per > 4 ? 4 : per);
  }
  // enough CTAs for the largest phase (256 elements each), at most the co-resident grid
  const int ntr = a.n - (a.r + a.nelim);
  const size_t pk = f.rows > 0 ? (size_t)tiles_for(f.rows + f.shift) * kTile * 4 * f.k4cap : 0;
  const size_t wr = (size_t)a.kmax * (size_t)(ntr > 0 ? ntr : 1);
  size_t want = (std::max(pk, wr) + 255) / 256;
  int grid = (int)std::min<size_t>(std::max<size_t>(want, 1), (size_t)maxgrid);
  PanelArgs ac = a;
  FinishPack fc = f;
  void* args[] = {&ac, &fc};
  return cudaLaunchCooperativeKernel((void*)panel_finish_pack_kernel, dim3(grid), dim3(256), args, 0, stream);
}

size_t panel_cluster_smem_bytes(int rows_per, int kmax, int npush) {
  return csmem_layout(rows_per, kmax, nullptr, nullptr, npush);
}

int panel_cluster_size() {
  static int cs = -1;
  if (cs < 0) {
    cs = 0;
    for (int c : {16, 8}) {
      cudaFuncSetAttribute(panel_cluster_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(panel_cluster_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
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
      if (cudaOccupancyMaxActiveClusters(&ncl, panel_cluster_kernel<false>, &cfg) == cudaSuccess && ncl >= 1) {
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
  cudaError_t e = cudaFuncSetAttribute(panel_cluster_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(panel_cluster_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = a.count_zeroed ? cudaSuccess : cudaMemsetAsync(a.disp_count, 0, sizeof(int), stream);
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
  e = cudaLaunchKernelEx(&cfg, panel_cluster_kernel<false>, a);
  if (e != cudaSuccess) return e;
  return a.defer_finish ? cudaSuccess : launch_panel_finish(a, stream);
}

// Largest number of co-resident clusters of size `csize` for a given smem size (0: none).
int panel_multi_clusters(int csize, size_t smem) {
  cudaFuncSetAttribute(panel_cluster_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (cudaFuncSetAttribute(panel_cluster_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize);
  cfg.blockDim = dim3(kCThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = csize;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, panel_cluster_kernel<true>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return ncl > 32 ? 32 : ncl;
}

int push_mcast();
size_t panel_push_smem_bytes(int rows_per, int kmax) {
  return psmem_layout(rows_per, kmax, nullptr, nullptr, push_mcast() == 1 ? 1 : kPC);
}

bool panel_push_v2();
bool panel_push_usable(bool push_pivot, int ctas, int csize, int rows_per, int kmax) {
  static int lim = 0;
  if (!lim) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&lim, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || lim <= 0)
      lim = 232448;
  }
  return push_pivot && ctas == csize && csize >= 1 && csize <= kPC && rows_per <= 2 * kPThreads && panel_push_v2() &&
         panel_push_smem_bytes(rows_per, kmax) <= (size_t)lim;
}

bool panel_push_v2() {
  static int on = [] {
    const char* v = getenv("SKL_PANEL_V2");
    return v && *v ? atoi(v) : 1;
  }();
  return on != 0;
}

// SKL_PUSH_MCAST: 0 = speculative DSMEM push of every candidate row, 1 = winner multicast,
// 2 = every candidate row multicast from the global row mirror during the exchange
int push_mcast() {
  static const int mcast = [] {
    const char* v = getenv("SKL_PUSH_MCAST");
    const int m = v && *v ? atoi(v) : 2;
    return m < 0 || m > 2 ? 2 : m;
  }();
  return mcast;
}

template <int RPT, int NB, int TPR>
cudaError_t launch_push_t(const PanelArgs& a, size_t smem, cudaStream_t stream) {
  const int mode = push_mcast();
  auto kern = mode == 2 ? panel_push_kernel<RPT, NB, TPR, 2>
                        : (mode == 1 ? panel_push_kernel<RPT, NB, TPR, 1> : panel_push_kernel<RPT, NB, TPR, 0>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.nblocks);
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = a.nblocks;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

// single 16-CTA cluster, pivoted: the lean push-mode panel (panel_push_kernel); the
// threads per row grow as the rows per CTA shrink (SKL_PUSH_TPR caps it, 1 = off)
cudaError_t launch_panel_push(const PanelArgs& a, cudaStream_t stream) {
  const size_t smem = panel_push_smem_bytes(a.rows_per, a.kmax);
  cudaError_t e = a.count_zeroed ? cudaSuccess : cudaMemsetAsync(a.disp_count, 0, sizeof(int), stream);
  if (e != cudaSuccess) return e;
  static const int tpr_cap = [] {
    const char* v = getenv("SKL_PUSH_TPR");
    return v && *v ? atoi(v) : 8;
  }();
  const int R = a.rows_per;
  if (R > kPThreads)
    e = launch_push_t<2, 1, 1>(a, smem, stream);
  else if (R > kPThreads / 2 || tpr_cap < 2)
    e = launch_push_t<1, 2, 1>(a, smem, stream);
  else if (R > kPThreads / 4 || tpr_cap < 4)
    e = launch_push_t<1, 2, 2>(a, smem, stream);
  else if (R > kPThreads / 8 || tpr_cap < 8)
    e = launch_push_t<1, 2, 4>(a, smem, stream);
  else
    e = launch_push_t<1, 2, 8>(a, smem, stream);
  if (e != cudaSuccess) return e;
  return a.defer_finish ? cudaSuccess : launch_panel_finish(a, stream);
}

size_t panel_multi2_smem_bytes(int rows_per, int kmax) { return psmem_layout(rows_per, kmax, nullptr, nullptr, 3); }

// several co-resident clusters, pivoted: panel_multi2_kernel (SKL_PANEL_MULTI2=0 keeps the
// round-1 panel_cluster_kernel<MULTI>)
bool panel_multi2_usable(const PanelArgs& a, int csize) {
  static const int on = [] {
    const char* v = getenv("SKL_PANEL_MULTI2");
    return v && *v ? atoi(v) : 1;
  }();
  if (!on || !a.pivot || csize < 1 || csize > kPC || a.nblocks % csize != 0 || a.nblocks / csize > 32 ||
      a.rows_per > 2 * kPThreads || a.slot_words < 6 + 2 * (a.kmax + 1) ||
      6 * push_crs(a.kmax) < 2 * (6 + 2 * (a.kmax + 1)))
    return false;
  return panel_multi2_smem_bytes(a.rows_per, a.kmax) <= 232448;
}

template <int RPT, int NB>
cudaError_t launch_multi2_t(const PanelArgs& a, int csize, size_t smem, cudaStream_t stream) {
  auto kern = panel_multi2_kernel<RPT, NB>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.nblocks);
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = csize;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeCooperative;
  attrs[1].val.cooperative = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

cudaError_t launch_panel_multi2(const PanelArgs& a, int csize, cudaStream_t stream) {
  const size_t smem = panel_multi2_smem_bytes(a.rows_per, a.kmax);
  cudaError_t e = a.count_zeroed ? cudaSuccess : cudaMemsetAsync(a.disp_count, 0, sizeof(int), stream);
  if (e != cudaSuccess) return e;
  e = a.rows_per > kPThreads ? launch_multi2_t<2, 1>(a, csize, smem, stream)
                             : launch_multi2_t<1, 2>(a, csize, smem, stream);
  if (e != cudaSuccess) return e;
  return a.defer_finish ? cudaSuccess : launch_panel_finish(a, stream);
}

// a.nblocks = total CTAs (Q clusters x a.csize); cooperative so all clusters are co-resident
cudaError_t launch_panel_multi(const PanelArgs& a, int csize, cudaStream_t stream) {
  if (panel_push_usable(a.push && a.pivot, a.nblocks, csize, a.rows_per, a.kmax)) return launch_panel_push(a, stream);
  if (a.nblocks > csize && panel_multi2_usable(a, csize)) return launch_panel_multi2(a, csize, stream);
  const bool push = a.push && a.pivot && a.nblocks == csize;
  size_t smem = csmem_layout(a.rows_per, a.kmax, nullptr, nullptr, push ? csize : 0);
  cudaError_t e = cudaFuncSetAttribute(panel_cluster_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(panel_cluster_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = a.count_zeroed ? cudaSuccess : cudaMemsetAsync(a.disp_count, 0, sizeof(int), stream);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.nblocks);
  cfg.blockDim = dim3(kCThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = csize;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeCooperative;
  attrs[1].val.cooperative = 1;
  cfg.attrs = attrs;
  // co-residency only matters across clusters; one cluster is co-resident by
  // construction (and a plain cluster launch stays replayable under ncu)
  cfg.numAttrs = a.nblocks > csize ? 2 : 1;
  e = cudaLaunchKernelEx(&cfg, panel_cluster_kernel<true>, a);
  if (e != cudaSuccess) return e;
  return a.defer_finish ? cudaSuccess : launch_panel_finish(a, stream);
}

}  // namespace skl
