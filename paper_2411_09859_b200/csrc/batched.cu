// Batched pivoted LTL^T + Pfaffian of many independent skew matrices
// (config 4: 8192 x n=256, fp32 and fp64).
//
// Reference path per matrix: pfaffian -> ltlt_blk_piv(x, b=min(256, m))
// (apps.py:12-30, blocked.py:303-363), i.e. one left-looking pivoted panel.
// The B200 kernel factors each matrix with the right-looking Wimmer two-step
// recurrence (unblocked.py:136-171) -- the same pivots and factors in exact
// arithmetic -- inside ONE CTA, with the symmetric interchanges made LAZY:
//
//  * The trailing matrix never moves.  It stays where it was loaded, in
//    "physical" coordinates (packed strictly-lower columns: the short last
//    columns in shared memory, the rest in a per-CTA global scratch that the
//    persistent CTA reuses for every matrix, so it stays L2-resident).  A
//    logical row/column i lives at physical index ph[i]; the interchange of
//    rows/columns a and b (_sym_swap_lower, core.py:294-324) only exchanges
//    two labels.  Element (i, j) is read with the skew rule
//    X(p, q) = p > q ? S[p][q] : -S[q][p].
//  * Thread t owns physical rows t (+256): it holds that row's current-column
//    value, its two L values of the running pair, and its logical label in
//    registers.  A column elimination (_eliminate, unblocked.py:63-91) is a
//    gather, an exact argmax (warp redux on the bit pattern of |v|, ties to
//    the lowest LOGICAL index) and ONE __syncthreads; the L column is written
//    out by physical row and every later row interchange of older L columns
//    (apply_row_pivots, kernels2.py:232-271) reduces to one final gather with
//    the final label map.
//  * The two-step rank-2 updates are blocked: kKB pairs stay pending (their
//    w, l vectors by physical row in shared memory); columns gathered meanwhile
//    get them applied on the fly, and every kKB pairs one skew rank-2kKB pass
//    (blocked.py:268-290's W = A S + skew rank-2k) updates the active part of
//    the trailing matrix, tiled 32 x 32 over the compacted active index list.
//
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
constexpr int kBT = SKL_BATCHED_THREADS;  // threads per CTA (thread t owns physical rows t, t + kBT, ...)
constexpr int kBW = kBT / 32;
#ifndef SKL_BATCHED_KB
#define SKL_BATCHED_KB 8
#endif
constexpr int kKB = SKL_BATCHED_KB;  // pending two-step pairs between trailing passes

// CTAs per SM (each gets 1/k of the shared memory for its cache of S columns)
// (8192 x n=256: fp64 19.1 / 20.9 ms and fp32 13.9 / 11.4 ms at 2 / 3 per SM; 128-thread
// CTAs at 3-6 per SM and 4 pending pairs were slower)
#ifndef SKL_BATCHED_CPS_F64
#define SKL_BATCHED_CPS_F64 2
#endif
#ifndef SKL_BATCHED_CPS_F32
#define SKL_BATCHED_CPS_F32 3
#endif
template <typename T>
constexpr int ctas_per_sm() {
  return sizeof(T) == 8 ? SKL_BATCHED_CPS_F64 : SKL_BATCHED_CPS_F32;
}

// pending vectors of physical index q: pend[q * PS + k] = w_k, pend[q * PS + kKB + k] = l_k.
// The 16-byte pad keeps 16-byte alignment and spreads consecutive rows over the banks.
template <typename T>
__host__ __device__ constexpr int pend_stride() {
  return 2 * kKB + int(16 / sizeof(T));
}

__host__ __device__ inline long long pk_off(int n, int q) {
  return (long long)q * (n - 1) - ((long long)q * (q - 1)) / 2;
}

struct BCand {
  double v;  // signed column value (tau if it wins)
  double x;  // carry: the candidate row's L value of the pair's first column
  int lg;    // logical index (argmax tie-break)
  int p;     // physical index
};

template <typename T>
struct PhysS {
  T* sm;  // packed columns [J0, n-1) in shared memory
  T* gs;  // packed columns [0, J0) in the CTA's global scratch
  const int* coff;  // [n] offset of column q's pointer inside its region (shared memory table:
                    // the 64-bit packed-offset arithmetic was 20 % of the kernel's stall samples)
  int J0;
  // pointer such that col(q)[p] = S[p][q] for p > q
  __device__ __forceinline__ T* col(int q) const { return (q >= J0 ? sm : gs) + coff[q]; }
  __device__ __forceinline__ T at(int p, int q) const {
    const int hi = max(p, q), lo = min(p, q);
    const T v = col(lo)[hi];
    return p > q ? v : -v;
  }
  // storage slot of the pair {p, q} (p != q), no sign
  __device__ __forceinline__ T* slot(int p, int q) const { return col(min(p, q)) + max(p, q); }
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

// sum_k (w_k[p] l_k[q] - l_k[p] w_k[q]) over the np pending pairs
template <typename T>
__device__ __forceinline__ T pending_dot(const T* pp, const T* pq, int np) {
  T acc = T(0), acc2 = T(0);
  for (int k = 0; k < np; ++k) {
    acc += pp[k] * pq[kKB + k];
    acc2 += pp[kKB + k] * pq[k];
  }
  return acc - acc2;
}

// the 2 kKB pending values of one physical index with 16-byte loads (rows are 16-byte aligned)
__device__ __forceinline__ void load_pend_row(double* q, const double* src) {
#pragma unroll
  for (int k = 0; k < 2 * kKB; k += 2) {
    const double2 t = *reinterpret_cast<const double2*>(src + k);
    q[k] = t.x;
    q[k + 1] = t.y;
  }
}
__device__ __forceinline__ void load_pend_row(float* q, const float* src) {
#pragma unroll
  for (int k = 0; k < 2 * kKB; k += 4) {
    const float4 t = *reinterpret_cast<const float4*>(src + k);
    q[k] = t.x;
    q[k + 1] = t.y;
    q[k + 2] = t.z;
    q[k + 3] = t.w;
  }
}

// sum_k (w_k q_l,k - l_k q_w,k) with four independent FMA chains (the pass is
// otherwise bound by the dependent-DFMA latency)
template <typename T>
__device__ __forceinline__ T pair_dot(const T* wp, const T* lp, const T* q) {
  T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
#pragma unroll
  for (int k = 0; k < kKB; k += 2) {
    a0 = fma(wp[k], q[kKB + k], a0);
    a1 = fma(lp[k], q[k], a1);
    a2 = fma(wp[k + 1], q[kKB + k + 1], a2);
    a3 = fma(lp[k + 1], q[k + 1], a3);
  }
  return (a0 + a2) - (a1 + a3);
}

template <typename T, int RPT>
struct RowState {
  T cur[RPT];  // current column value of this physical row
  T la[RPT];   // L value, first column of the running pair
  T lb[RPT];   // L value, second column
  int lg[RPT]; // logical label of this physical row
};

// One column elimination (_eliminate, unblocked.py:63-91) over the rows with
// logical label > g, values in st.cur; c = physical index of column g.
// Candidates carry the row's `la`.  Returns the winner and relabels; the L
// column goes to the storage slots {p, c} of S: physical row/column c is dead
// from now on (never read as part of the trailing matrix again), so its n - 1
// slots hold L(:, g) by physical row until the final write-back.
template <typename T, int RPT>
__device__ __forceinline__ BCand eliminate(RowState<T, RPT>& st, int g, int n, BCand* red, int* paslot,
                                           const PhysS<T>& S, int c) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int a = g + 1;
  const int par = g & 1;
  double bv = -1.0;
  BCand mine{0.0, 0.0, -1, -1};
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int p = tid + u * kBT;
    if (p < n && st.lg[u] > g) {
      const double av = fabs((double)st.cur[u]);
      if (av > bv || (av == bv && st.lg[u] < mine.lg)) {
        bv = av;
        mine = BCand{(double)st.cur[u], (double)st.la[u], st.lg[u], p};
      }
      if (st.lg[u] == a) paslot[par] = p;
    }
  }
  const int id = bwarp_argmax(bv, mine.lg, mine.lg >= 0);
  if (mine.lg >= 0 && mine.lg == id) red[par * kBW + warp] = mine;
  if (lane == 0 && id < 0) red[par * kBW + warp].lg = -1;
  __syncthreads();
  BCand w;
  {
    const BCand c = lane < kBW ? red[par * kBW + lane] : BCand{0.0, 0.0, -1, -1};
    const bool ok = lane < kBW && c.lg >= 0;
    const int id2 = bwarp_argmax(fabs(c.v), c.lg, ok);
    const int src = __ffs(__ballot_sync(0xffffffffu, ok && c.lg == id2)) - 1;
    w.v = __shfl_sync(0xffffffffu, c.v, src);
    w.x = __shfl_sync(0xffffffffu, c.x, src);
    w.lg = id2;
    w.p = __shfl_sync(0xffffffffu, c.p, src);
  }
  const int pa = paslot[par];
  const T t0 = (T)w.v;
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int p = tid + u * kBT;
    if (p < n && st.lg[u] > g) {
      if (p == w.p) {
        st.lg[u] = a;  // the pivot row takes position a (explicit 1 of L)
      } else {
        const T v = st.cur[u];
        const T l = t0 != T(0) ? v / t0 : v;
        st.lb[u] = l;
        *S.slot(p, c) = l;
        if (p == pa) st.lg[u] = w.lg;  // row a moves to position b
      }
    }
  }
  return w;
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
#define BMARK(i)                                  \
  do {                                            \
    long long _t = clock64();                     \
    bpt[i] += _t - bprev;                         \
    bprev = _t;                                   \
  } while (0)
#else
#define BMARK(i) \
  do {           \
  } while (0)
#endif

template <typename T, int RPT>
__global__ void __launch_bounds__(kBT, ctas_per_sm<T>())
batched_kernel(int batch, int n, int J0, const T* __restrict__ X, long long ldx, long long strideX, T* __restrict__ L,
               long long ldl, long long strideL, T* __restrict__ tau, long long strideTau, long long* __restrict__ piv,
               long long stridePiv, double* __restrict__ pf_sign, double* __restrict__ pf_logabs, T* __restrict__ scr,
               long long scr_stride) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int PS = pend_stride<T>();
  BCand* red = reinterpret_cast<BCand*>(smem_raw);         // [2][kBW]
  int* ibuf = reinterpret_cast<int*>(red + 2 * kBW);       // [0..1] pa slots, [2..2+kBW) warp counts
  int* actl = ibuf + 2 + 2 * kBW;                                   // [n] compact active list / final label map
  int* coff = actl + n;                                             // [n] column pointer offsets
  T** cptr = reinterpret_cast<T**>(smem_raw + ((sizeof(BCand) * 2 * kBW + sizeof(int) * (2 + 2 * kBW + 2 * n) + 15) & ~size_t(15)));
  double* taus = reinterpret_cast<double*>(cptr + n);      // [n] tau (Pfaffian factors)
  double* pfred = taus + n;                                // [kBW] log|Pf| partials
  T* pend = reinterpret_cast<T*>(pfred + kBW);             // [n][PS]
  T* smS = pend + (size_t)n * PS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    const int offJ0 = int(pk_off(n, J0));
    for (int q = tid; q < n; q += kBT) {
      const int o = int(pk_off(n, q)) - (q + 1);
      coff[q] = q >= J0 ? o - offJ0 : o;
    }
  }
  PhysS<T> S{smS, scr + (long long)blockIdx.x * scr_stride, coff, J0};
  __syncthreads();

#ifdef SKL_BATCHED_PROF
  long long bpt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long bprev = clock64();
#endif
  for (int m = blockIdx.x; m < batch; m += gridDim.x) {
    const T* x = X + (long long)m * strideX;
    T* l = L + (long long)m * strideL;
    T* tm = tau + (long long)m * strideTau;
    long long* pm = piv + (long long)m * stridePiv;
    // ---- load the strict lower triangle into S (warp per column, coalesced) ----
    for (int j = warp; j < n - 1; j += kBW) {
      T* cj = S.col(j);
      const T* xj = x + (long long)j * ldx;
      T v[RPT * kBT / 32];
#pragma unroll
      for (int s = 0; s < RPT * kBT / 32; ++s) {
        const int i = j + 1 + lane + 32 * s;
        if (i < n) v[s] = __ldcs(xj + i);  // streamed: keep L2 for the scratch
      }
#pragma unroll
      for (int s = 0; s < RPT * kBT / 32; ++s) {
        const int i = j + 1 + lane + 32 * s;
        if (i < n) cj[i] = v[s];
      }
    }
    RowState<T, RPT> st;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      st.lg[u] = tid + u * kBT;
      st.la[u] = T(0);
      st.lb[u] = T(0);
      st.cur[u] = T(0);
    }
    if (tid == 0) pm[0] = 0;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int p = tid + u * kBT;
      if (p >= 1 && p < n) st.cur[u] = S.col(0)[p];
    }

    BMARK(0);
    int nswaps = 0;
    const int end = n - 1;
    int g = 0;
    int np = 0;
    int cg = 0;  // physical index of column g
    while (g < end) {
      // ---- eliminate(g): column g is current (loaded, or the previous pair's fold) ----
      BCand w0 = eliminate<T, RPT>(st, g, n, red, ibuf, S, cg);
      if (tid == 0) {
        const int b = w0.lg;
        pm[g + 1] = b - (g + 1);
        nswaps += b != g + 1;
        tm[g] = (T)w0.v;
        taus[g] = w0.v;  // even g: Pfaffian factor, reduced after the loop
      }
#pragma unroll
      for (int u = 0; u < RPT; ++u) st.la[u] = st.lb[u];
      BMARK(1);
      if (g + 1 >= end) {
        g += 1;
        break;
      }
      // ---- eliminate(g+1): gather column g+1 (physical w0.p), pending pairs applied ----
      {
        const int c = w0.p;
        const T* pc = pend + (size_t)c * PS;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int p = tid + u * kBT;
          if (p < n && st.lg[u] > g + 1) {
            T v = S.at(p, c);
            if (np > 0) v -= pending_dot(pend + (size_t)p * PS, pc, np);
            st.cur[u] = v;
          }
        }
      }
      BMARK(2);
      BCand w1 = eliminate<T, RPT>(st, g + 1, n, red, ibuf, S, w0.p);
      if (tid == 0) {
        const int b = w1.lg;
        pm[g + 2] = b - (g + 2);
        nswaps += b != g + 2;
        tm[g + 1] = (T)w1.v;
      }
      BMARK(3);
      // ---- column g+2 (physical w1.p): pending pairs, then fold the first coupling;
      // this pair's rank-2 vectors become pending entry np -------------------------
      {
        const int c = w1.p;
        const T* pc = pend + (size_t)c * PS;
        const T t1 = (T)w1.v;
        const T x20 = (T)w1.x;  // L(g+2, g): the winner's first-column L value
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int p = tid + u * kBT;
          if (p < n && st.lg[u] > g + 2) {
            T* pp = pend + (size_t)p * PS;
            T x2 = S.at(p, c);
            if (np > 0) x2 -= pending_dot(pp, pc, np);
            const T l2 = st.lb[u], l1 = st.la[u];
            const T f = x2 - t1 * (x20 * l2 - l1);
            st.cur[u] = f;
            pp[np] = f - t1 * l1;
            pp[kKB + np] = l2;
          }
        }
      }
      ++np;
      g += 2;
      cg = w1.p;
      BMARK(4);
      // ---- every kKB pairs: S[act, act] -= sum_k (w_k l_k^T - l_k w_k^T) ---------
      if (np == kKB && g + 1 < end) {
        // compact the active physical indices (label >= g + 1), ascending
        int base = 0;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int p = tid + u * kBT;
          const bool act = p < n && st.lg[u] >= g + 1;
          const unsigned bal = __ballot_sync(0xffffffffu, act);
          if (lane == 0) ibuf[2 + warp] = __popc(bal);
          __syncthreads();  // also orders the fold's pend writes before the pass
          int off = base, tot = 0;
#pragma unroll
          for (int w = 0; w < kBW; ++w) {
            const int cnt = ibuf[2 + w];
            off += w < warp ? cnt : 0;
            tot += cnt;
          }
          if (act) {
            const int r = off + __popc(bal & ((1u << lane) - 1u));
            actl[r] = p;
            cptr[r] = S.col(p);
          }
          base += tot;
          __syncthreads();
        }
        const int mact = base;
        const int nbk = (mact + 31) >> 5;
        const int ntiles = nbk * (nbk + 1) / 2;
        for (int t = warp; t < ntiles; t += kBW) {
          int R = int((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
          while ((R + 1) * (R + 2) / 2 <= t) ++R;
          while (R * (R + 1) / 2 > t) --R;
          const int Cb = t - R * (R + 1) / 2;
          const int r = R * 32 + lane;
          if (r >= mact) continue;
          const int p = actl[r];
          T wp[kKB], lp[kKB];
          {
            T q[2 * kKB];
            load_pend_row(q, pend + (size_t)p * PS);
#pragma unroll
            for (int k = 0; k < kKB; ++k) {
              wp[k] = q[k];
              lp[k] = q[kKB + k];
            }
          }
          const int c0 = Cb * 32;
          const int c1 = min(c0 + 32, r);  // columns c < r (strict lower)
          int c = c0;
          constexpr int U = 4;  // S loads in flight per lane
          for (; c + U - 1 < c1; c += U) {
            T* e[U];
            T v[U];
#pragma unroll
            for (int t2 = 0; t2 < U; ++t2) {
              e[t2] = cptr[c + t2] + p;
              v[t2] = *e[t2];
            }
#pragma unroll
            for (int t2 = 0; t2 < U; ++t2) {
              T q[2 * kKB];
              load_pend_row(q, pend + (size_t)actl[c + t2] * PS);
              v[t2] -= pair_dot(wp, lp, q);
              *e[t2] = v[t2];
            }
          }
          for (; c < c1; ++c) {
            T* e0 = cptr[c] + p;
            T v0 = *e0;
            T q[2 * kKB];
            load_pend_row(q, pend + (size_t)actl[c] * PS);
            v0 -= pair_dot(wp, lp, q);
            *e0 = v0;
          }
        }
        np = 0;
        __syncthreads();
        BMARK(5);
      }
    }
    // Pf = sign(P) prod_{i even} (-tau_i) (apps.py:26-30) as (sign, log|Pf|):
    // per-thread partial sums over the even taus, warp + CTA reduction
    __syncthreads();
    {
      double lsum = 0.0;
      int npos = 0, nzero = 0;
      for (int i = 2 * tid; i < n - 1; i += 2 * kBT) {
        const double t = taus[i];
        lsum += log(fabs(t));
        npos += t > 0.0;
        nzero += t == 0.0;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
      npos = __reduce_add_sync(0xffffffffu, npos);
      nzero = __reduce_add_sync(0xffffffffu, nzero);
      if (lane == 0) {
        pfred[warp] = lsum;
        ibuf[2 + warp] = npos;
        ibuf[2 + kBW + warp] = nzero;
      }
    }
    // ---- write-back: final label map; L column j is read from the slots
    // {ph[i], ph[j]} in final row order (every deferred row interchange at
    // once), the upper triangle and diagonal are copied from X; one warp per
    // output column, coalesced ----------------------------------------------------
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int p = tid + u * kBT;
      if (p < n) actl[st.lg[u]] = p;  // actl = final ph: logical -> physical
    }
    __syncthreads();
    if (tid == 0) {
      double lsum = 0.0;
      int npos = 0, nzero = 0;
      for (int w = 0; w < kBW; ++w) {
        lsum += pfred[w];
        npos += ibuf[2 + w];
        nzero += ibuf[2 + kBW + w];
      }
      double sgn = nzero ? 0.0 : (((npos + nswaps) & 1) ? -1.0 : 1.0);
      if (n % 2 == 1) sgn = 0.0;
      if (pf_sign) pf_sign[m] = sgn;
      if (pf_logabs) pf_logabs[m] = sgn == 0.0 ? -INFINITY : lsum;
    }
    for (int j = warp; j < n; j += kBW) {
      T* lj = l + (long long)j * ldl;
      const T* xj = x + (long long)j * ldx;
      const int cj = actl[j];
      T v[RPT * kBT / 32];
#pragma unroll
      for (int s = 0; s < RPT * kBT / 32; ++s) {
        const int i = lane + 32 * s;
        if (i < n) v[s] = i <= j ? __ldcs(xj + i) : (i == j + 1 ? T(1) : *S.slot(actl[i], cj));
      }
#pragma unroll
      for (int s = 0; s < RPT * kBT / 32; ++s) {
        const int i = lane + 32 * s;
        if (i < n) __stcs(lj + i, v[s]);
      }
    }
    __syncthreads();
    BMARK(6);
  }
#ifdef SKL_BATCHED_PROF
  if (tid == 0 && blockIdx.x == 0)
    for (int i = 0; i < 8; ++i) atomicAdd(&g_bprof[i], (unsigned long long)bpt[i]);
#endif
}

template <typename T>
size_t batched_head(int n) {
  size_t h = (sizeof(BCand) * 2 * kBW + sizeof(int) * (2 + 2 * kBW + 2 * n) + 15) & ~size_t(15);
  return h + sizeof(T*) * (size_t)n + sizeof(double) * (size_t)(n + kBW) + sizeof(T) * (size_t)n * pend_stride<T>();
}

template <typename T>
size_t batched_smem(int n, int J0) {
  return batched_head<T>(n) + sizeof(T) * (size_t)(pk_off(n, n - 1) - pk_off(n, J0));
}

template <typename T, int RPT>
cudaError_t launch_rpt(int batch, int n, const T* X, long long ldx, long long strideX, T* L, long long ldl,
                       long long strideL, T* tau, long long strideTau, long long* piv, long long stridePiv,
                       double* pf_sign, double* pf_logabs, cudaStream_t stream) {
  int dev = 0, lim = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&lim, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  constexpr int kPerSm = ctas_per_sm<T>();
  const size_t budget = kPerSm == 1 ? (size_t)lim : (size_t)(228 * 1024) / kPerSm - 1024;
  if (batched_head<T>(n) > budget) return cudaErrorInvalidValue;
  int J0 = 0;
  while (J0 < n - 1 && batched_smem<T>(n, J0) > budget) ++J0;
  const size_t smem = batched_smem<T>(n, J0);
  cudaError_t e =
      cudaFuncSetAttribute(batched_kernel<T, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long gmax = (long long)nsm * kPerSm;
  const int grid = batch < gmax ? batch : (int)gmax;
  // per-CTA scratch for the packed columns that do not fit shared memory
  const long long scr_stride = (pk_off(n, J0) + 31) / 32 * 32;
  T* scr = nullptr;
  if (scr_stride > 0) {
    static bool pool_kept = false;
    if (!pool_kept) {
      // keep freed stream-ordered memory in the pool across calls (the default
      // threshold 0 returns it to the driver at every synchronisation)
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        unsigned long long keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      pool_kept = true;
    }
    e = cudaMallocAsync(reinterpret_cast<void**>(&scr), sizeof(T) * (size_t)scr_stride * grid, stream);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kBT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  e = cudaLaunchKernelEx(&cfg, batched_kernel<T, RPT>, batch, n, J0, X, ldx, strideX, L, ldl, strideL, tau, strideTau,
                         piv, stridePiv, pf_sign, pf_logabs, scr, scr_stride);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (scr) {
    cudaError_t e2 = cudaFreeAsync(scr, stream);
    if (e == cudaSuccess) e = e2;
  }
  return e;
}

}  // namespace

template <typename T>
cudaError_t launch_batched(int batch, int n, const T* X, long long ldx, long long strideX, T* L, long long ldl,
                           long long strideL, T* tau, long long strideTau, long long* piv, long long stridePiv,
                           double* pf_sign, double* pf_logabs, cudaStream_t stream) {
  // n <= 512: at most 512 / kBT physical rows per thread
  if (n <= kBT)
    return launch_rpt<T, 1>(batch, n, X, ldx, strideX, L, ldl, strideL, tau, strideTau, piv, stridePiv, pf_sign,
                            pf_logabs, stream);
  if (n <= 2 * kBT)
    return launch_rpt<T, 2>(batch, n, X, ldx, strideX, L, ldl, strideL, tau, strideTau, piv, stridePiv, pf_sign,
                            pf_logabs, stream);
  if constexpr (kBT < 256) {
    if (n <= 4 * kBT)
      return launch_rpt<T, 4>(batch, n, X, ldx, strideX, L, ldl, strideL, tau, strideTau, piv, stridePiv, pf_sign,
                              pf_logabs, stream);
  }
  return cudaErrorInvalidValue;
}

template cudaError_t launch_batched<double>(int, int, const double*, long long, long long, double*, long long,
                                            long long, double*, long long, long long*, long long, double*, double*,
                                            cudaStream_t);
template cudaError_t launch_batched<float>(int, int, const float*, long long, long long, float*, long long, long long,
                                           float*, long long, long long*, long long, double*, double*, cudaStream_t);

}  // namespace skl
