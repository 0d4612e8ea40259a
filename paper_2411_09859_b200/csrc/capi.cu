// extern "C" boundary and the host-side blocked driver.
//
// The driver is the B200 counterpart of ltlt_blk_piv (blocked.py:303-363):
// per panel it launches (1) the cooperative pivoted panel kernel, (2) the
// operand pack (B = A T^T on the fly, plus the var1 straggler pair), and
// (3) the lower-triangular DMMA GEMM on the trailing matrix; after the last
// panel, one gather applies the deferred row interchanges to the L columns.
// Everything is enqueued on the caller's stream with no host synchronisation.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "internal.h"
#include "skewltl_b200.h"

namespace {

thread_local std::string g_last_error;
unsigned long long* g_prof = nullptr;  // debug: panel phase profile (device)

// ---- optional per-kernel-class timing of the blocked driver (CUDA events on
// the launching stream; bench.py uses it for the roofline of the top kernel)
enum { KPANEL = 0, KPACK = 1, KGEMM = 2, KFINAL = 3, KNUM = 4 };
struct KTimer {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[KNUM];
  long long launches = 0;
} g_kt;

// NVTX ranges over the same scopes (SKL_NVTX=1): the host-side phase names of a timeline --
// the counterpart of the reference's scope("panel") / scope("update") tagging
// (instrument.py:74-94, blocked.py:92,331,347).  Header-only NVTX v3: no library to link.
const char* const kScopeName[] = {"skl.panel", "skl.pack", "skl.trailing_gemm", "skl.finalize"};
bool nvtx_on() {
  static const bool on = [] {
    const char* v = getenv("SKL_NVTX");
    return v && *v && *v != '0';
  }();
  return on;
}

struct KScope {
  int kind;
  cudaStream_t st;
  cudaEvent_t b = nullptr, e = nullptr;
  KScope(int k, cudaStream_t s) : kind(k), st(s) {
    g_kt.launches++;
    if (nvtx_on()) nvtxRangePushA(kScopeName[kind]);
    if (g_kt.on) {
      cudaEventCreate(&b);
      cudaEventCreate(&e);
      cudaEventRecord(b, st);
    }
  }
  ~KScope() {
    if (g_kt.on) {
      cudaEventRecord(e, st);
      g_kt.ev[kind].push_back({b, e});
    }
    if (nvtx_on()) nvtxRangePop();
  }
};

int fail_cuda(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return SKL_CUDA_ERROR;
}

#define SKL_TRY(expr)                                  \
  do {                                                 \
    cudaError_t _e = (expr);                           \
    if (_e != cudaSuccess) return fail_cuda(_e, #expr); \
  } while (0)

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// simple bump allocator over a caller-provided workspace (or a size query)
struct Bump {
  unsigned char* base;
  size_t off = 0;
  explicit Bump(void* b) : base(static_cast<unsigned char*>(b)) {}
  template <typename T>
  T* take(size_t count) {
    size_t o = align_up(off);
    off = o + count * sizeof(T);
    return base ? reinterpret_cast<T*>(base + o) : nullptr;
  }
};

bool overlaps(const void* a, size_t abytes, const void* b, size_t bbytes) {
  auto pa = reinterpret_cast<uintptr_t>(a), pb = reinterpret_cast<uintptr_t>(b);
  return pa < pb + bbytes && pb < pa + abytes;
}

size_t mat_bytes(int rows, int cols, long long ld) {
  if (rows <= 0 || cols <= 0) return 0;
  return ((size_t)(cols - 1) * ld + rows) * sizeof(double);
}

// ---------------------------------------------------------------------------
// panel schedule of the pivoted blocked driver (blocked.py:325-362), with the
// panel width shrunk when the panel block would not fit in shared memory
// ---------------------------------------------------------------------------
struct PanelPlan {
  int r, nelim, lo;
  int ctas, rows_per, kmax;
  int cluster;  // 2: multi-cluster kernel, 1: single-cluster DSMEM panel kernel, 0: grid-wide kernel
  int csize;    // cluster size (multi)
};

size_t smem_limit() {
  static int lim = 0;
  if (!lim) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&lim, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || lim <= 0)
      lim = 232448;
  }
  return (size_t)lim;
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// single-cluster pivoted panel: candidate rows pushed through DSMEM with lazy
// interchanges (panel_cluster.cu, push mode); SKL_PANEL_PUSH=0 keeps the L2 row exchange
bool panel_push() {
  static int on = env_int("SKL_PANEL_PUSH", 1);
  return on != 0;
}

bool plan_panel(int n, int r, int want, int lo, int nsm, PanelPlan& p) {
  int rows = n - (lo + 1);
  // GPU panel width cap for the cluster panel (per-step cost grows with the width while the
  // trailing DMMA GEMM is already efficient at K ~ 96); SKL_GPU_NB overrides.
  static int gpu_nb = env_int("SKL_GPU_NB", 94);  // K = 94 + 2 (straggler) = 96: whole 16-wide GEMM k-chunks
  static int no_cluster = env_int("SKL_NO_CLUSTER", 0);
  const int Cmax = no_cluster ? 0 : skl::panel_cluster_size();
  // SKL_FORCE_MULTI=1: skip the single-cluster plan (tests drive the multi-cluster
  // exchange at small n with it; SKL_MULTI_Q caps the cluster count)
  static int force_multi = env_int("SKL_FORCE_MULTI", 0);
  if (Cmax > 0 && !force_multi) {
    // smallest cluster that keeps <= rows_target rows per CTA: fewer CTAs means a
    // cheaper cluster barrier and less DSMEM fan-out of the pivot row per step
    static int rows_target = env_int("SKL_CLUSTER_ROWS", 16);
    int C = (rows + rows_target - 1) / rows_target;
    if (C < 2) C = 2;
    if (C > Cmax) C = Cmax;
    int Rc = (rows + C - 1) / C;
    // the cluster kernels hold at most two rows per thread (R <= 512); a larger R
    // (reachable with SKL_MIN_CLUSTER_W < 56) used to fault
    if (Rc <= 2 * skl::panel_threads()) {
      static int min_w = env_int("SKL_MIN_CLUSTER_W", 64);
      static int ll_single = env_int("SKL_LL_SINGLE", 1);
      const int npush = (ll_single && panel_push()) ? C : 0;  // room for the pushed candidate rows
      // (round 2 measured and dropped: 64-column tall panels and one full-width final panel,
      // DESIGN.md §4)
      // short trailing matrices take wider panels (fewer panel / GEMM launches; the per-step
      // gemv is cheap at few rows per CTA): SKL_GPU_NB_SHORT columns from SKL_SHORT_ROWS rows down
      static int short_rows = env_int("SKL_SHORT_ROWS", 600);
      static int gpu_nb_short = env_int("SKL_GPU_NB_SHORT", 142);  // K = 144: nine 16-wide k-chunks
      const int cap = (short_rows > 0 && rows <= short_rows && gpu_nb_short > gpu_nb) ? gpu_nb_short : gpu_nb;
      int w = (cap > 0 && want > cap) ? cap : want;
      auto fits = [&](int ww) {
        const int km = r + ww - lo;
        if (ll_single && skl::panel_push_usable(panel_push(), C, C, Rc, km)) return true;
        return skl::panel_cluster_smem_bytes(Rc, km, npush) <= smem_limit();
      };
      while (w >= 1 && !fits(w)) --w;
      if (w >= 1 && w >= std::min(want, min_w)) {
        // default (SKL_LL_SINGLE=1): the one cluster runs the multi-cluster kernel with
        // Q = 1 -- st.async candidate all-to-all + flagged pivot rows through L2, no
        // cluster barrier per step (2-3 % faster than the DSMEM-pull variant, which
        // SKL_LL_SINGLE=0 keeps)
        p = ll_single ? PanelPlan{r, w, lo, C, Rc, r + w - lo, 2, C} : PanelPlan{r, w, lo, C, Rc, r + w - lo, 1, C};
        return true;
      }
    }
  }
  static int multi = env_int("SKL_MULTI_CLUSTER", 1);
  static int multi_q = env_int("SKL_MULTI_Q", 0);    // cap on the co-resident clusters used
  // cap on the multi-cluster panel width: n=16384 sweep (tools/sweep_multi.sh) 117.8-118.6 ms at 128
  // vs 120.7 ms uncapped (256): the per-step gemv grows with the width faster than the GEMM gains
  static int multi_nb = env_int("SKL_MULTI_NB", 190);  // round 2 (lean multi-cluster panel): 128/158/190 -> 103.3/101.6/101.4 ms at config 3
  if (Cmax > 0 && multi) {
    for (int csize : {Cmax, 8}) {
      int Q = skl::panel_multi_clusters(csize, smem_limit());
      if (multi_q > 0 && Q > multi_q) {
        Q = std::max(multi_q, 2);
      }
      if (Q < 2) continue;
      const int P = Q * csize;
      const int Rm = (rows + P - 1) / P;
      if (Rm > 512) continue;
      int w = (multi_nb > 0 && want > multi_nb) ? multi_nb : want;
      while (w >= 1 && skl::panel_cluster_smem_bytes(Rm, r + w - lo) > smem_limit()) --w;
      if (w >= 1 && w >= std::min(want, 64)) {
        p = PanelPlan{r, w, lo, P, Rm, r + w - lo, 2, csize};
        return true;
      }
    }
  }
  static int min_rows = env_int("SKL_PANEL_MIN_ROWS", 8);
  int ctas = (rows + min_rows - 1) / min_rows;
  if (ctas > nsm) ctas = nsm;
  if (ctas < 1) ctas = 1;
  int R = (rows + ctas - 1) / ctas;
  if (R > 2 * skl::panel_threads()) return false;
  int nelim = want;
  while (nelim >= 1 && skl::panel_smem_bytes(R, r + nelim - lo) > smem_limit()) --nelim;
  if (nelim < 1) return false;
  p = PanelPlan{r, nelim, lo, ctas, R, r + nelim - lo, 0, 0};
  return true;
}

// panels eliminating columns [0, ncols) (ncols = n - 1: the whole factorization)
bool make_schedule(int n, int nb, int variant, std::vector<PanelPlan>& out, int ncols = -1) {
  out.clear();
  int nsm = skl::panel_max_ctas();
  PanelPlan p;
  const int end = ncols < 0 ? n - 1 : std::min(ncols, n - 1);
  if (variant == SKL_VAR2B) {
    int done = 0;
    bool first = true;
    while (done < end) {
      int want = std::min(nb + (first ? 1 : 0), end - done);
      int lo = first ? 0 : done - 1;
      if (!plan_panel(n, done, want, lo, nsm, p)) return false;
      out.push_back(p);
      done += p.nelim;
      first = false;
    }
  } else {
    int r = 0;
    bool pending = false;
    while (r < end) {
      int want = std::min(nb, end - r);
      int lo = (variant == SKL_VAR2A && pending) ? r - 1 : r;
      if (!plan_panel(n, r, want, lo, nsm, p)) return false;
      out.push_back(p);
      r += p.nelim;
      pending = true;
    }
  }
  return true;
}

struct BlkWorkspace {
  double* W;
  double* P;
  double* Q;
  double* side;
  double* y;
  int* gperm_all;
  int* sigma_all;
  int* col_group;
  int* disp_list;
  int* disp_count;
  uint64_t* slots;
  uint64_t* rowa;
  uint64_t* recs;
  double* crow;
  double* arowg;
  double* rowmir;
  double* pbuf;
  size_t ll_bytes;
  int k4cap, slot_words, np;
  double* PL;  // left-looking driver: packed A = W[r:, 0:r] and (T B)^T of the panel rows
  double* QL;
  int* ltab;   // [np][owner_table_ints(kmax)] tile tables of the panel blocks
  size_t ltab_stride;
};

size_t layout_blk(int n, int nb, const std::vector<PanelPlan>& plan, void* base, BlkWorkspace* ws,
                  bool left = false) {
  Bump b(base);
  int kmax = 1, nelim_max = 1, ctas = 1;
  for (auto& p : plan) {
    kmax = std::max(kmax, p.kmax);
    nelim_max = std::max(nelim_max, p.nelim);
    ctas = std::max(ctas, p.ctas);
  }
  (void)nb;
  int np = (int)plan.size();
  int k4cap = (kmax + 2 + 3) / 4;
  int slot_words = 4 + 2 * (kmax + 2);
  BlkWorkspace w{};
  w.W = b.take<double>((size_t)n * n);
  w.pbuf = b.take<double>((size_t)kmax * n);
  w.P = b.take<double>(skl::packed_elems(n, k4cap));
  w.Q = b.take<double>(skl::packed_elems(n, k4cap));
  w.side = b.take<double>((size_t)2 * (nelim_max + 1) * n);
  w.y = b.take<double>(n);
  w.gperm_all = b.take<int>((size_t)std::max(np, 1) * n);
  w.sigma_all = b.take<int>((size_t)std::max(np, 1) * n);
  w.col_group = b.take<int>(n);
  w.disp_list = b.take<int>(2 * (nelim_max + 1));
  w.disp_count = b.take<int>(1);
  w.rowmir = b.take<double>((size_t)n * (kmax + 4));
  size_t ll_start = align_up(b.off);
  w.slots = b.take<uint64_t>((size_t)ctas * 2 * slot_words);
  w.rowa = b.take<uint64_t>((size_t)2 * slot_words);
  w.recs = b.take<uint64_t>((size_t)2 * ctas * 4);
  w.crow = b.take<double>((size_t)2 * 16 * (kmax + 2));
  w.arowg = b.take<double>((size_t)2 * (kmax + 2));
  w.ll_bytes = b.off - ll_start;
  w.k4cap = k4cap;
  w.slot_words = slot_words;
  w.np = np;
  if (left) {
    size_t pl = 1, ql = 1;
    for (auto& p : plan) {
      const int k4 = (p.r + 3) / 4;
      if (p.r < 2) continue;
      pl = std::max(pl, skl::packed_elems(n - p.r, k4));
      ql = std::max(ql, skl::packed_elems(p.nelim, k4));
    }
    w.PL = b.take<double>(pl);
    w.QL = b.take<double>(ql);
    w.ltab_stride = skl::owner_table_ints(kmax);
    w.ltab = b.take<int>((size_t)std::max(np, 1) * w.ltab_stride);
  }
  if (ws) *ws = w;
  return b.off + 256;
}

}  // namespace

extern "C" {

const char* skl_version(void) { return "skewltl_b200 0.1.0 (sm_100a)"; }
const char* skl_last_error(void) { return g_last_error.c_str(); }

// per-kernel-class timing: enable/disable (clears), read after the stream has synced
int skl_timing_enable(int on) {
  for (auto& v : g_kt.ev)
    for (auto& p : v) {
      cudaEventDestroy(p.first);
      cudaEventDestroy(p.second);
    }
  for (auto& v : g_kt.ev) v.clear();
  g_kt.on = on != 0;
  g_kt.launches = 0;
  return SKL_OK;
}

// ms[k] = total milliseconds of kernel class k (panel, pack, gemm, finalize); cnt[k] = launches
int skl_timing_read(double* ms, int* cnt) {
  for (int k = 0; k < KNUM; ++k) {
    double tot = 0.0;
    for (auto& p : g_kt.ev[k]) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, p.first, p.second) != cudaSuccess) return fail_cuda(cudaGetLastError(), "timing");
      tot += t;
    }
    ms[k] = tot;
    cnt[k] = (int)g_kt.ev[k].size();
  }
  return SKL_OK;
}

// number of kernel launches issued by the library since the last skl_timing_enable()
long long skl_launch_count(void) { return g_kt.launches; }

// debug hook: route per-CTA panel phase cycle counters to a device buffer (NULL disables)
int skl_debug_set_panel_profile(unsigned long long* dev_buf) {
  g_prof = dev_buf;
  return SKL_OK;
}

// ---------------------------------------------------------------------------
size_t skl_skr2k_workspace_size(int n, int k) {
  Bump b(nullptr);
  int k4cap = (2 * std::max(k, 1) + 3) / 4;
  b.take<double>(skl::packed_elems(std::max(n, 1), k4cap));
  b.take<double>(skl::packed_elems(std::max(n, 1), k4cap));
  b.take<int>(std::max(k, 1));
  b.take<int>(4 + std::max(k, 1));
  b.take<unsigned>(skl::rank2k_prep_scratch_words(k));
  return b.off + 256;
}

int skl_skr2k_lower(int n, int k, double alpha, const double* A, long long lda, const double* B, long long ldb,
                    double beta, double* C, long long ldc, int skip_zero_cols, void* workspace,
                    size_t workspace_bytes, int* keff_dev, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n < 0 || k < 0 || (n > 0 && (lda < n || ldb < n || ldc < n))) return SKL_BAD_ARGUMENT;
  if (workspace_bytes < skl_skr2k_workspace_size(n, k)) return SKL_BAD_ARGUMENT;
  size_t cb = mat_bytes(n, n, ldc);
  if (overlaps(C, cb, A, mat_bytes(n, k, lda)) && k > 0) return SKL_ALIAS;
  if (overlaps(C, cb, B, mat_bytes(n, k, ldb)) && k > 0) return SKL_ALIAS;
  Bump b(workspace);
  int k4cap = (2 * std::max(k, 1) + 3) / 4;
  double* P = b.take<double>(skl::packed_elems(std::max(n, 1), k4cap));
  double* Q = b.take<double>(skl::packed_elems(std::max(n, 1), k4cap));
  int* keep = b.take<int>(std::max(k, 1));
  int* cnt = b.take<int>(4 + std::max(k, 1));  // [0] keff, [1] nk4, [2..] per-column flags
  if (n <= 1 || k == 0 || alpha == 0.0) {
    if (n <= 1) {
      if (keff_dev) {
        if (k == 0 || n <= 0) {
          SKL_TRY(cudaMemsetAsync(keff_dev, 0, sizeof(int), st));
        } else {
          SKL_TRY(skl::launch_rank2k_keep(A, lda, B, ldb, n, k, skip_zero_cols, keep, cnt, cnt + 1, st));
          SKL_TRY(cudaMemcpyAsync(keff_dev, cnt, sizeof(int), cudaMemcpyDeviceToDevice, st));
        }
      }
      return SKL_OK;
    }
    SKL_TRY(skl::launch_scale_lower<double>(C, ldc, n, beta, st));
    if (keff_dev) {
      if (k == 0) {
        SKL_TRY(cudaMemsetAsync(keff_dev, 0, sizeof(int), st));
      } else {
        SKL_TRY(skl::launch_rank2k_keep(A, lda, B, ldb, n, k, skip_zero_cols, keep, cnt, cnt + 1, st));
        SKL_TRY(cudaMemcpyAsync(keff_dev, cnt, sizeof(int), cudaMemcpyDeviceToDevice, st));
      }
    }
    return SKL_OK;
  }
  // keep list + packed operands in one cooperative launch (SKL_SKR2K_PREP=0: the
  // four-launch prologue, kept for A/B), then the lower-triangular DMMA GEMM
  static const bool fused_prep = [] {
    const char* v = getenv("SKL_SKR2K_PREP");
    return !(v && *v == '0');
  }();
  if (fused_prep) {
    unsigned* part = b.take<unsigned>(skl::rank2k_prep_scratch_words(k));
    g_kt.launches += 2;
    SKL_TRY(skl::launch_rank2k_prep(A, lda, B, ldb, n, k, skip_zero_cols, alpha, k4cap, part, keep, cnt, P, Q, st));
  } else {
    g_kt.launches += 4;
    SKL_TRY(skl::launch_rank2k_keep(A, lda, B, ldb, n, k, skip_zero_cols, keep, cnt, cnt + 1, st));
    SKL_TRY(skl::launch_pack_rank2k(A, lda, B, ldb, n, k, alpha, keep, cnt, k4cap, P, Q, st));
  }
  SKL_TRY(skl::launch_gemm_lower(P, Q, k4cap, k4cap, cnt + 1, C, ldc, n, beta, st));
  if (keff_dev) SKL_TRY(cudaMemcpyAsync(keff_dev, cnt, sizeof(int), cudaMemcpyDeviceToDevice, st));
  return SKL_OK;
}

// skew_tridiag_gemm (kernels3.py:239-302): C (p x q) := beta C + alpha A (T B);
// tril: only row > col of the view.  The same DMMA kernel in tile-table mode.
size_t skl_skew_tridiag_gemm_workspace_size(int p, int q, int k) {
  Bump b(nullptr);
  const int k4cap = (std::max(k, 1) + 3) / 4;
  b.take<double>(skl::packed_elems(std::max(p, 1), k4cap));
  b.take<double>(skl::packed_elems(std::max(q, 1), k4cap));
  b.take<int>(skl::owner_table_ints(std::max(q, 1)));
  return b.off + 256;
}

int skl_skew_tridiag_gemm(int p, int q, int k, double alpha, const double* A, long long lda, const double* tau,
                          const double* B, long long ldb, double beta, double* C, long long ldc, int tril,
                          void* workspace, size_t workspace_bytes, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p < 0 || q < 0 || k < 0 || (p > 0 && ldc < p) || (p > 0 && k > 0 && lda < p) || (q > 0 && k > 0 && ldb < k))
    return SKL_BAD_ARGUMENT;
  if (workspace_bytes < skl_skew_tridiag_gemm_workspace_size(p, q, k)) return SKL_BAD_ARGUMENT;
  if (k > 0 && overlaps(C, mat_bytes(p, q, ldc), A, mat_bytes(p, k, lda))) return SKL_ALIAS;
  if (k > 0 && overlaps(C, mat_bytes(p, q, ldc), B, mat_bytes(k, q, ldb))) return SKL_ALIAS;
  if (p == 0 || q == 0) return SKL_OK;
  if (alpha == 0.0 || k == 0) {
    g_kt.launches += beta != 1.0 ? 1 : 0;
    SKL_TRY(skl::launch_scale_block(C, ldc, p, q, beta, tril ? 1 : 0, st));
    return SKL_OK;
  }
  Bump b(workspace);
  const int k4cap = (k + 3) / 4;
  double* P = b.take<double>(skl::packed_elems(p, k4cap));
  double* Q = b.take<double>(skl::packed_elems(q, k4cap));
  int* tab_dev = b.take<int>(skl::owner_table_ints(q));
  std::vector<int> tab(skl::owner_table_ints(q), 0);
  const int ntiles = skl::build_rect_table(p, q, tril ? 1 : 0, tab.data());
  if (ntiles == 0) return SKL_OK;  // tril with q >= p... nothing strictly below the diagonal
  SKL_TRY(cudaMemcpyAsync(tab_dev, tab.data(), sizeof(int) * tab.size(), cudaMemcpyHostToDevice, st));
  g_kt.launches += 2;
  SKL_TRY(skl::launch_pack_gemm(A, lda, p, B, ldb, q, k, tau, alpha, k4cap, P, Q, st, 0));
  skl::ColOwner own{tab_dev, ntiles, 0, 1 << 30, 1, 0};
  SKL_TRY(skl::launch_gemm_lower(P, Q, k4cap, k4cap, nullptr, C, ldc, p, beta, st, &own, q, tril ? 1 : 0));
  return SKL_OK;
}

size_t skl_sktri_rankk_workspace_size(int n, int k) {
  Bump b(nullptr);
  int k4cap = (std::max(k, 1) + 3) / 4;
  b.take<double>(skl::packed_elems(std::max(n, 1), k4cap));
  b.take<double>(skl::packed_elems(std::max(n, 1), k4cap));
  return b.off + 256;
}

int skl_sktri_rankk_lower(int n, int k, double alpha, const double* A, long long lda, const double* tau,
                          double beta, double* C, long long ldc, void* workspace, size_t workspace_bytes,
                          void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n < 0 || k < 0 || (n > 0 && (lda < n || ldc < n))) return SKL_BAD_ARGUMENT;
  if (workspace_bytes < skl_sktri_rankk_workspace_size(n, k)) return SKL_BAD_ARGUMENT;
  if (k > 0 && overlaps(C, mat_bytes(n, n, ldc), A, mat_bytes(n, k, lda))) return SKL_ALIAS;
  if (n <= 1) return SKL_OK;
  if (alpha == 0.0 || k == 0) {
    SKL_TRY(skl::launch_scale_lower<double>(C, ldc, n, beta, st));
    return SKL_OK;
  }
  Bump b(workspace);
  int k4cap = (k + 3) / 4;
  double* P = b.take<double>(skl::packed_elems(n, k4cap));
  double* Q = b.take<double>(skl::packed_elems(n, k4cap));
  SKL_TRY(skl::launch_pack_rankk(A, lda, n, k, tau, alpha, nullptr, k4cap, P, Q, st));
  SKL_TRY(skl::launch_gemm_lower(P, Q, k4cap, k4cap, nullptr, C, ldc, n, beta, st));
  return SKL_OK;
}

int skl_form_w(int n, int k, const double* A, long long lda, const double* tau, double* W, long long ldw,
               void* stream) {
  if (n < 0 || k < 0 || (n > 0 && (lda < n || ldw < n))) return SKL_BAD_ARGUMENT;
  SKL_TRY(skl::launch_form_w(A, lda, n, k, tau, W, ldw, static_cast<cudaStream_t>(stream)));
  return SKL_OK;
}

int skl_skew_rank2_lower(int n, double alpha, const double* x, const double* y, double beta, double* A,
                         long long lda, void* stream) {
  if (n < 0 || (n > 0 && lda < n)) return SKL_BAD_ARGUMENT;
  if (alpha == 0.0 && beta == 1.0) return SKL_OK;
  SKL_TRY(skl::launch_skew_rank2(A, lda, n, alpha, x, y, beta, static_cast<cudaStream_t>(stream)));
  return SKL_OK;
}

int skl_gen_rank2(int p, int q, double alpha, const double* x, const double* u, const double* y, const double* v,
                  double beta, double* A, long long lda, void* stream) {
  if (p < 0 || q < 0 || (p > 0 && q > 0 && lda < p)) return SKL_BAD_ARGUMENT;
  if (p == 0 || q == 0 || (alpha == 0.0 && beta == 1.0)) return SKL_OK;
  SKL_TRY(skl::launch_gen_rank2(A, lda, p, q, alpha, x, u, y, v, beta, static_cast<cudaStream_t>(stream)));
  g_kt.launches++;
  return SKL_OK;
}

int skl_skew_tridiag_gemv(int p, int k, double alpha, const double* A, long long lda, const double* tau,
                          const double* x, double beta, double* y, int tail_from, void* stream) {
  if (p < 0 || k < 0 || tail_from < 0 || tail_from > p || (p > 0 && lda < p)) return SKL_BAD_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (alpha == 0.0) {
    if (beta != 1.0) SKL_TRY(skl::launch_skew_tridiag_gemv(y, 0.0, A, lda, p, 0, tau, x, beta, tail_from, st));
    return SKL_OK;
  }
  SKL_TRY(skl::launch_skew_tridiag_gemv(y, alpha, A, lda, p, k, tau, x, beta, tail_from, st));
  return SKL_OK;
}

size_t skl_apply_row_pivots_workspace_size(int q, int lo, int hi) {
  return (size_t)std::max(q, 1) * std::max(hi - lo, 1) * sizeof(double) + 256;
}

int skl_apply_row_pivots(int n, int q, double* block, long long ld, const long long* idx, int lo, int hi,
                         void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 0 || q < 0 || lo < 0 || hi > n || (q > 0 && ld < n)) return SKL_BAD_ARGUMENT;
  if (hi <= lo || q == 0) return SKL_OK;
  if (workspace_bytes < skl_apply_row_pivots_workspace_size(q, lo, hi)) return SKL_BAD_ARGUMENT;
  SKL_TRY(skl::launch_gather_rows(block, ld, q, lo, hi, idx, static_cast<double*>(workspace),
                                  static_cast<cudaStream_t>(stream)));
  return SKL_OK;
}

int skl_apply_symmetric_pivot(int n, double* X, long long ld, int k, long long pi, void* stream) {
  if (pi == 0) return SKL_OK;
  if (pi < 0 || k < 0 || k + pi >= n) return SKL_BAD_PIVOT;
  SKL_TRY(skl::launch_sym_swap(X, ld, n, k, (int)(k + pi), static_cast<cudaStream_t>(stream)));
  return SKL_OK;
}

int skl_pack_factor(int n, const double* L, long long ldl, const double* tau, double* X, long long ldx, void* stream) {
  if (n < 1 || ldl < n || ldx < n) return SKL_BAD_ARGUMENT;
  g_kt.launches += n > 1 ? 1 : 0;
  SKL_TRY(skl::launch_pack_factor(n, L, ldl, tau, X, ldx, static_cast<cudaStream_t>(stream)));
  return SKL_OK;
}

int skl_unpack_factor(int n, const double* X, long long ldx, double* L, long long ldl, double* tau, void* stream) {
  if (n < 1 || ldl < n || ldx < n) return SKL_BAD_ARGUMENT;
  if (L == X) return SKL_ALIAS;
  g_kt.launches += 1;
  SKL_TRY(skl::launch_unpack_factor(n, X, ldx, L, ldl, tau, static_cast<cudaStream_t>(stream)));
  return SKL_OK;
}

// ---------------------------------------------------------------------------
size_t skl_ltlt_blk_piv_workspace_size(int n, int nb, int variant) {
  if (n < 1 || nb < 1 || variant < SKL_VAR1 || variant > SKL_LEFT) return 0;
  const bool left = variant == SKL_LEFT;
  std::vector<PanelPlan> plan;
  if (!make_schedule(n, nb, left ? SKL_VAR2A : variant, plan)) return 0;
  return layout_blk(n, nb, plan, nullptr, nullptr, left);
}

int skl_ltlt_blk_piv_plan(int n, int nb, int variant, int* r, int* nelim, int* kind, int* ctas, int* csize,
                          int cap) {
  if (n < 1 || nb < 1 || variant < SKL_VAR1 || variant > SKL_VAR2B) return -1;
  std::vector<PanelPlan> plan;
  if (!make_schedule(n, nb, variant, plan)) return -1;
  for (int i = 0; i < (int)plan.size() && i < cap; ++i) {
    if (r) r[i] = plan[i].r;
    if (nelim) nelim[i] = plan[i].nelim;
    if (kind) kind[i] = plan[i].cluster;
    if (ctas) ctas[i] = plan[i].ctas;
    if (csize) csize[i] = plan[i].csize;
  }
  return (int)plan.size();
}

namespace {
// blocked driver behind skl_ltlt_blk_piv / skl_ltlt_blk / skl_ltlt_unb_panel:
// eliminates columns [0, ncols); pivot = 0 runs the unpivoted drivers (pivot row
// fixed, exact-zero breakdown reported in *info)
int blk_driver(int n, int nb, int variant, int pivot, int ncols, const double* X, long long ldx, double* L,
               long long ldl, double* tau, long long* piv, int* info, void* workspace, size_t workspace_bytes,
               void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (variant < SKL_VAR1 || variant > SKL_LEFT) return SKL_UNSUPPORTED;
  // blocked left-looking (blocked.py:236-265): every panel first pulls all prior
  // couplings into its own columns (skew_tridiag_gemm, tril) and the trailing
  // matrix is never updated; pivoting is impossible there (PivotUnsupported)
  const bool left = variant == SKL_LEFT;
  if (left && pivot) return SKL_UNSUPPORTED;
  if (left) variant = SKL_VAR2A;  // the carry-column panel schedule
  if (n < 1 || nb < 1 || ldx < n || ldl < n) return SKL_BAD_ARGUMENT;
  if ((pivot && piv == nullptr) || (!pivot && info == nullptr)) return SKL_BAD_ARGUMENT;
  std::vector<PanelPlan> plan;
  if (!make_schedule(n, nb, variant, plan, ncols)) {
    g_last_error = "panel block does not fit the shared-memory budget";
    return SKL_UNSUPPORTED;
  }
  if (!pivot)
    for (const PanelPlan& p : plan)
      if (p.cluster == 0) {
        g_last_error = "the unpivoted drivers need the cluster panel kernels";
        return SKL_UNSUPPORTED;
      }
  size_t need = layout_blk(n, nb, plan, nullptr, nullptr, left);
  if (workspace_bytes < need) return SKL_BAD_ARGUMENT;
  BlkWorkspace ws;
  layout_blk(n, nb, plan, workspace, &ws, left);
  const long long ld = n;
  std::vector<int> ltiles;
  if (left) {
    std::vector<int> tabs((size_t)std::max((int)plan.size(), 1) * ws.ltab_stride, 0);
    ltiles.assign(plan.size(), 0);
    for (int k = 0; k < (int)plan.size(); ++k)
      if (plan[k].r >= 2)
        ltiles[k] = skl::build_rect_table(n - plan[k].r, plan[k].nelim, 1, tabs.data() + (size_t)k * ws.ltab_stride);
    SKL_TRY(cudaMemcpyAsync(ws.ltab, tabs.data(), sizeof(int) * tabs.size(), cudaMemcpyHostToDevice, st));
  }

  if (piv != nullptr) SKL_TRY(cudaMemsetAsync(piv, 0, sizeof(long long) * n, st));
  if (info != nullptr) SKL_TRY(cudaMemsetAsync(info, 0, sizeof(int), st));
  if (n == 1) {
    if (L != X) SKL_TRY(cudaMemcpyAsync(L, X, sizeof(double), cudaMemcpyDeviceToDevice, st));
    return SKL_OK;
  }
  SKL_TRY(cudaMemcpy2DAsync(ws.W, ld * sizeof(double), X, ldx * sizeof(double), n * sizeof(double), n,
                            cudaMemcpyDeviceToDevice, st));
  SKL_TRY(cudaMemsetAsync(tau, 0, sizeof(double) * (n - 1), st));
  SKL_TRY(cudaMemsetAsync(ws.slots, 0, ws.ll_bytes, st));

  // column -> last panel containing it (for the deferred row gather)
  std::vector<int> group(n, 0);
  for (int k = 0; k < (int)plan.size(); ++k)
    for (int c = plan[k].lo; c < n; ++c) group[c] = k;
  SKL_TRY(cudaMemcpyAsync(ws.col_group, group.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));

  uint32_t tag = 1;
  bool count_zeroed = false;  // disp_count left at zero by the previous panel's fused epilogue
  for (int k = 0; k < (int)plan.size(); ++k) {
    const PanelPlan& p = plan[k];
    const int rt = p.r + p.nelim;
    const bool straggler = (variant == SKL_VAR1) && (n - rt >= 2);
    if (left && p.r >= 2 && ltiles[k] > 0) {
      // work[r:, r:r+be] -= work[r:, 0:r] T(tau[1:r]) work[r:r+be, 0:r]^T, row > col only
      const int rr = p.r, k4 = (rr + 3) / 4;
      {
        KScope ks(KPACK, st);
        SKL_TRY(skl::launch_pack_gemm(ws.W + rr, ld, n - rr, ws.W + rr, ld, p.nelim, rr, tau + 1, -1.0, k4, ws.PL,
                                      ws.QL, st, 1));
      }
      {
        KScope ks(KGEMM, st);
        skl::ColOwner own{ws.ltab + (size_t)k * ws.ltab_stride, ltiles[k], 0, 1 << 30, 1, 0};
        SKL_TRY(skl::launch_gemm_lower(ws.PL, ws.QL, k4, k4, nullptr, ws.W + (size_t)rr * ld + rr, ld, n - rr, 1.0,
                                       st, &own, p.nelim, 1));
      }
    }
    skl::PanelArgs a{};
    a.W = ws.W;
    a.ld = ld;
    a.n = n;
    a.r = p.r;
    a.nelim = p.nelim;
    a.lo = p.lo;
    a.want_y = straggler ? 1 : 0;
    a.tau = tau;
    a.piv = piv;
    a.y = ws.y;
    a.gperm = ws.gperm_all + (size_t)k * n;
    a.disp_list = ws.disp_list;
    a.disp_count = ws.disp_count;
    a.side = ws.side;
    a.slots = ws.slots;
    a.rowa = ws.rowa;
    a.recs = ws.recs;
    a.crow = ws.crow;
    a.rowmir = ws.rowmir;
    a.arowg = ws.arowg;
    a.pbuf = ws.pbuf;
    a.tag0 = tag;
    a.nblocks = p.ctas;
    a.rows_per = p.rows_per;
    a.kmax = p.kmax;
    a.slot_words = ws.slot_words;
    static int dbg = env_int("SKL_PANEL_DBG", 0);
    a.dbg = dbg;
    a.prof = g_prof;
    a.pivot = pivot;
    a.info = info;
    a.push = (p.cluster == 2 && p.ctas == p.csize && pivot && panel_push()) ? 1 : 0;
    const int ntr = n - rt;
    // cluster panels followed by a trailing update: epilogue + operand packing as ONE
    // cooperative launch (SKL_FUSED_FINISH=0: finish_gather, finish_write, pack_rankk)
    // (worth ~12 us per panel while the three kernels are launch-bound: config 1 0.868 -> 0.842 ms,
    // config 2 8.56 -> 8.50 ms; from ~8K trailing rows on the separate, wider grids win: config 3
    // 100.6 -> 101.2 ms with every panel fused, hence the row limit)
    static const int fused_rows = env_int("SKL_FUSED_FINISH", 8192);
    const bool fuse = ntr < fused_rows && p.cluster != 0 && ntr >= 2 && !left;
    a.defer_finish = fuse ? 1 : 0;
    a.count_zeroed = count_zeroed ? 1 : 0;
    count_zeroed = fuse;  // the fused epilogue leaves disp_count at zero
    {
      KScope ks(KPANEL, st);
      if (p.cluster == 2)
        SKL_TRY(skl::launch_panel_multi(a, p.csize, st));
      else if (p.cluster == 1)
        SKL_TRY(skl::launch_panel_cluster(a, st));
      else
        SKL_TRY(skl::launch_panel(a, st));
      if (p.cluster != 0 && !fuse) g_kt.launches += 2;  // + panel_finish_gather / panel_finish_write
    }
    tag += (uint32_t)p.nelim + 1;

    if (ntr >= 2 && !left) {
      const int ka = rt - p.lo;
      const int K = ka + (straggler ? 2 : 0);
      const int nk4 = (K + 3) / 4;
      const int sh0 = skl::align_shift(rt, ld), rt0 = rt - sh0;
      {
        KScope ks(KPACK, st);
        if (fuse) {
          skl::FinishPack f{ntr, ka, ws.k4cap, sh0, tau + p.lo + 1, straggler ? ws.y + rt : nullptr, ws.P, ws.Q};
          SKL_TRY(skl::launch_panel_finish_pack(a, f, st));
        } else {
          SKL_TRY(skl::launch_pack_rankk(ws.W + (size_t)p.lo * ld + rt, ld, ntr, ka, tau + p.lo + 1, -1.0,
                                         straggler ? ws.y + rt : nullptr, ws.k4cap, ws.P, ws.Q, st, sh0));
        }
      }
      {
        // the C region starts sh0 rows/columns early (zero operand rows there) so
        // every C tile begins on a 128-byte line
        KScope ks(KGEMM, st);
        SKL_TRY(skl::launch_gemm_lower(ws.P, ws.Q, ws.k4cap, nk4, nullptr, ws.W + (size_t)rt0 * ld + rt0, ld,
                                       ntr + sh0, 1.0, st));
      }
    }
  }
  {
    KScope ks(KFINAL, st);
    SKL_TRY(skl::launch_compose_suffix(ws.gperm_all, (int)plan.size(), nullptr, n, ws.sigma_all, st));
    g_kt.launches++;
    SKL_TRY(skl::launch_finalize_l(ws.W, ld, X, ldx, L, ldl, n, ws.col_group, ws.sigma_all, L != X ? 1 : 0, st));
  }
  return SKL_OK;
}
}  // namespace

// ---------------------------------------------------------------------------
// Block-cyclic multi-GPU driver (config 5).  The work matrix W is
// ONE virtual address range on every rank whose nbd-column blocks are backed by
// the HBM of rank (block % G) (CUDA VMM, mapped by the host layer), so the
// panel kernels address remote columns exactly like local ones over NVLink.
// Per panel: the owner of the panel's first column runs the pivoted panel and
// its finish kernels (pivot-column gathers and interchanges read/write peer
// memory); barrier; every rank packs the panel operands and runs the DMMA
// trailing GEMM on the columns it owns; barrier.  tau / piv / y / gperm live
// in a shared region (one rank's memory, mapped by all).
namespace {
struct DistShared {
  double* tau;
  long long* piv;
  double* y;
  int* gperm_all;
};
size_t layout_dist_shared(int n, int np, void* base, DistShared* out) {
  Bump b(base);
  DistShared d{};
  d.tau = b.take<double>(n);
  d.piv = b.take<long long>(n);
  d.y = b.take<double>(n);
  d.gperm_all = b.take<int>((size_t)std::max(np, 1) * n);
  if (out) *out = d;
  return b.off + 256;
}
struct DistWs {
  BlkWorkspace blk;  // W unused (the global matrix is the caller's)
  int* own_tab;      // [np][nr][owner_table_ints(n)]
  size_t tab_stride;
};
size_t layout_dist(int n, int nb, int nr, const std::vector<PanelPlan>& plan, void* base, DistWs* ws) {
  Bump b(base);
  int kmax = 1, nelim_max = 1, ctas = 1;
  for (auto& p : plan) {
    kmax = std::max(kmax, p.kmax);
    nelim_max = std::max(nelim_max, p.nelim);
    ctas = std::max(ctas, p.ctas);
  }
  (void)nb;
  const int np = (int)plan.size();
  BlkWorkspace w{};
  const int k4cap = (kmax + 2 + 3) / 4;
  const int slot_words = 4 + 2 * (kmax + 2);
  w.W = nullptr;
  w.pbuf = b.take<double>((size_t)kmax * n);
  w.P = b.take<double>(skl::packed_elems(n, k4cap));
  w.Q = b.take<double>(skl::packed_elems(n, k4cap));
  w.side = b.take<double>((size_t)2 * (nelim_max + 1) * n);
  w.sigma_all = b.take<int>((size_t)std::max(np, 1) * n);
  w.col_group = b.take<int>(n);
  w.disp_list = b.take<int>(2 * (nelim_max + 1));
  w.disp_count = b.take<int>(1);
  w.rowmir = b.take<double>((size_t)n * (kmax + 4));
  size_t ll_start = align_up(b.off);
  w.slots = b.take<uint64_t>((size_t)ctas * 2 * slot_words);
  w.rowa = b.take<uint64_t>((size_t)2 * slot_words);
  w.recs = b.take<uint64_t>((size_t)2 * ctas * 4);
  w.crow = b.take<double>((size_t)2 * 16 * (kmax + 2));
  w.arowg = b.take<double>((size_t)2 * (kmax + 2));
  w.ll_bytes = b.off - ll_start;
  w.k4cap = k4cap;
  w.slot_words = slot_words;
  w.np = np;
  DistWs d{};
  d.blk = w;
  d.tab_stride = skl::owner_table_ints(n);
  d.own_tab = b.take<int>((size_t)std::max(np, 1) * nr * d.tab_stride);
  if (ws) *ws = d;
  return b.off + 256;
}
}  // namespace

size_t skl_ltlt_dist_shared_size(int n, int nb, int variant) {
  if (n < 2 || nb < 1 || variant < SKL_VAR1 || variant > SKL_VAR2B) return 0;
  std::vector<PanelPlan> plan;
  if (!make_schedule(n, nb, variant, plan)) return 0;
  return layout_dist_shared(n, (int)plan.size(), nullptr, nullptr);
}

size_t skl_ltlt_dist_workspace_size(int n, int nb, int variant, int nranks_local) {
  if (n < 2 || nb < 1 || nranks_local < 1 || variant < SKL_VAR1 || variant > SKL_VAR2B) return 0;
  std::vector<PanelPlan> plan;
  if (!make_schedule(n, nb, variant, plan)) return 0;
  return layout_dist(n, nb, nranks_local, plan, nullptr, nullptr);
}

int skl_ltlt_dist_offsets(int n, int nb, int variant, size_t* off_tau, size_t* off_piv, size_t* off_gperm,
                          int* npanels) {
  std::vector<PanelPlan> plan;
  if (n < 2 || nb < 1 || variant < SKL_VAR1 || variant > SKL_VAR2B || !make_schedule(n, nb, variant, plan))
    return SKL_BAD_ARGUMENT;
  DistShared d;
  layout_dist_shared(n, (int)plan.size(), reinterpret_cast<void*>(uintptr_t(0x100000)), &d);
  const uintptr_t b0 = 0x100000;
  if (off_tau) *off_tau = reinterpret_cast<uintptr_t>(d.tau) - b0;
  if (off_piv) *off_piv = reinterpret_cast<uintptr_t>(d.piv) - b0;
  if (off_gperm) *off_gperm = reinterpret_cast<uintptr_t>(d.gperm_all) - b0;
  if (npanels) *npanels = (int)plan.size();
  return SKL_OK;
}

int skl_dist_owner_table(int n, long long cbase, int nbd, int nranks, int rank, int* tab, size_t tab_ints) {
  if (n < 1 || nbd < 1 || nranks < 1 || rank < 0 || rank >= nranks || !tab) return SKL_BAD_ARGUMENT;
  if (tab_ints < skl::owner_table_ints(n)) return SKL_BAD_ARGUMENT;
  return skl::build_owner_table(n, cbase, nbd, nranks, rank, tab) >= 0 ? SKL_OK : SKL_BAD_ARGUMENT;
}

int skl_ltlt_blk_piv_dist(int n, int nb, int variant, int nbd, int nranks, int rank_lo, int rank_hi, double* W,
                          long long ldw, double* L, long long ldl, void* shared, void* workspace,
                          size_t workspace_bytes, skl_barrier_fn barrier, void* barrier_ctx, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (variant < SKL_VAR1 || variant > SKL_VAR2B) return SKL_UNSUPPORTED;
  if (n < 2 || nb < 1 || nbd < 1 || nranks < 1 || rank_lo < 0 || rank_hi > nranks || rank_lo >= rank_hi ||
      ldw < n || ldl < n || !W || !L || !shared || !workspace)
    return SKL_BAD_ARGUMENT;
  const bool all_local = rank_lo == 0 && rank_hi == nranks;
  if (!all_local && !barrier) return SKL_BAD_ARGUMENT;
  const int nr = rank_hi - rank_lo;
  std::vector<PanelPlan> plan;
  if (!make_schedule(n, nb, variant, plan)) {
    g_last_error = "panel block does not fit the shared-memory budget";
    return SKL_UNSUPPORTED;
  }
  const int np = (int)plan.size();
  if (workspace_bytes < layout_dist(n, nb, nr, plan, nullptr, nullptr)) return SKL_BAD_ARGUMENT;
  DistWs dw;
  layout_dist(n, nb, nr, plan, workspace, &dw);
  BlkWorkspace& ws = dw.blk;
  DistShared sh;
  layout_dist_shared(n, np, shared, &sh);
  auto sync = [&]() -> int {
    if (all_local) return SKL_OK;
    const int rc = barrier(barrier_ctx, stream);
    if (rc != 0) {
      g_last_error = "distributed barrier failed";
      return SKL_CUDA_ERROR;
    }
    return SKL_OK;
  };

  // host tables: column -> last panel containing it; per (panel, rank) owned GEMM tiles
  std::vector<int> group(n, 0);
  for (int k = 0; k < np; ++k)
    for (int c = plan[k].lo; c < n; ++c) group[c] = k;
  std::vector<int> tabs((size_t)np * nr * dw.tab_stride, 0);
  std::vector<int> ntiles((size_t)np * nr, 0);
  for (int k = 0; k < np; ++k) {
    const int rt = plan[k].r + plan[k].nelim;
    if (n - rt < 2) continue;
    const int rt0 = rt - skl::align_shift(rt, ldw);  // the GEMM's (line-aligned) region origin
    for (int q = 0; q < nr; ++q)
      ntiles[(size_t)k * nr + q] = skl::build_owner_table(n - rt0, rt0, nbd, nranks, rank_lo + q,
                                                          tabs.data() + ((size_t)k * nr + q) * dw.tab_stride);
  }
  SKL_TRY(cudaMemcpyAsync(ws.col_group, group.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
  SKL_TRY(cudaMemcpyAsync(dw.own_tab, tabs.data(), sizeof(int) * tabs.size(), cudaMemcpyHostToDevice, st));
  SKL_TRY(cudaMemsetAsync(ws.slots, 0, ws.ll_bytes, st));
  if (rank_lo == 0) {
    SKL_TRY(cudaMemsetAsync(sh.tau, 0, sizeof(double) * (n - 1), st));
    SKL_TRY(cudaMemsetAsync(sh.piv, 0, sizeof(long long) * n, st));
  }
  // the host tables are pageable: the copies above complete before this returns
  int rc = sync();
  if (rc) return rc;

  uint32_t tag = 1;
  for (int k = 0; k < np; ++k) {
    const PanelPlan& p = plan[k];
    const int rt = p.r + p.nelim;
    const bool straggler = (variant == SKL_VAR1) && (n - rt >= 2);
    const int runner = (p.r / nbd) % nranks;
    if (runner >= rank_lo && runner < rank_hi) {
      skl::PanelArgs a{};
      a.W = W;
      a.ld = ldw;
      a.n = n;
      a.r = p.r;
      a.nelim = p.nelim;
      a.lo = p.lo;
      a.want_y = straggler ? 1 : 0;
      a.tau = sh.tau;
      a.piv = sh.piv;
      a.y = sh.y;
      a.gperm = sh.gperm_all + (size_t)k * n;
      a.disp_list = ws.disp_list;
      a.disp_count = ws.disp_count;
      a.side = ws.side;
      a.slots = ws.slots;
      a.rowa = ws.rowa;
      a.recs = ws.recs;
      a.crow = ws.crow;
      a.rowmir = ws.rowmir;
      a.arowg = ws.arowg;
      a.pbuf = ws.pbuf;
      a.tag0 = tag;
      a.nblocks = p.ctas;
      a.rows_per = p.rows_per;
      a.kmax = p.kmax;
      a.slot_words = ws.slot_words;
      a.prof = nullptr;
      a.pivot = 1;
      a.info = nullptr;
      // the same panel kernel as the single-device driver (bit-identical factorizations)
      a.push = (p.cluster == 2 && p.ctas == p.csize && panel_push()) ? 1 : 0;
      KScope ks(KPANEL, st);
      if (p.cluster == 2)
        SKL_TRY(skl::launch_panel_multi(a, p.csize, st));
      else if (p.cluster == 1)
        SKL_TRY(skl::launch_panel_cluster(a, st));
      else
        SKL_TRY(skl::launch_panel(a, st));
      if (p.cluster != 0) g_kt.launches += 2;
    }
    tag += (uint32_t)p.nelim + 1;  // every process advances the LL tag identically
    if ((rc = sync())) return rc;

    const int ntr = n - rt;
    if (ntr >= 2) {
      const int ka = rt - p.lo;
      const int K = ka + (straggler ? 2 : 0);
      const int nk4 = (K + 3) / 4;
      const int sh0 = skl::align_shift(rt, ldw), rt0 = rt - sh0;
      {
        KScope ks(KPACK, st);
        SKL_TRY(skl::launch_pack_rankk(W + (size_t)p.lo * ldw + rt, ldw, ntr, ka, sh.tau + p.lo + 1, -1.0,
                                       straggler ? sh.y + rt : nullptr, ws.k4cap, ws.P, ws.Q, st, sh0));
      }
      for (int q = 0; q < nr; ++q) {
        const int nt = ntiles[(size_t)k * nr + q];
        if (nt == 0) continue;
        skl::ColOwner own{dw.own_tab + ((size_t)k * nr + q) * dw.tab_stride, nt, (long long)rt0, nbd, nranks,
                          rank_lo + q};
        KScope ks(KGEMM, st);
        SKL_TRY(skl::launch_gemm_lower(ws.P, ws.Q, ws.k4cap, nk4, nullptr, W + (size_t)rt0 * ldw + rt0, ldw,
                                       ntr + sh0, 1.0, st, &own));
      }
      if ((rc = sync())) return rc;
    }
  }
  {
    KScope ks(KFINAL, st);
    SKL_TRY(skl::launch_compose_suffix(sh.gperm_all, np, nullptr, n, ws.sigma_all, st));
    for (int q = 0; q < nr; ++q) {
      g_kt.launches++;
      SKL_TRY(skl::launch_finalize_l(W, ldw, W, ldw, L, ldl, n, ws.col_group, ws.sigma_all, 0, st, nbd, nranks,
                                     rank_lo + q));
    }
  }
  return sync();
}

int skl_ltlt_blk_piv(int n, int nb, int variant, const double* X, long long ldx, double* L, long long ldl,
                     double* tau, long long* piv, void* workspace, size_t workspace_bytes, void* stream) {
  return blk_driver(n, nb, variant, 1, -1, X, ldx, L, ldl, tau, piv, nullptr, workspace, workspace_bytes, stream);
}

int skl_ltlt_blk(int n, int nb, int variant, int pivot, const double* X, long long ldx, double* L, long long ldl,
                 double* tau, long long* piv, int* info, void* workspace, size_t workspace_bytes, void* stream) {
  return blk_driver(n, nb, variant, pivot ? 1 : 0, -1, X, ldx, L, ldl, tau, pivot ? piv : nullptr, info, workspace,
                    workspace_bytes, stream);
}

size_t skl_ltlt_unb_panel_workspace_size(int n, int width) {
  if (n < 1 || width < 1) return 0;
  std::vector<PanelPlan> plan;
  if (!make_schedule(n, width, SKL_VAR2A, plan, width)) return 0;
  return layout_blk(n, width, plan, nullptr, nullptr);
}

int skl_ltlt_unb_panel(int n, int width, int pivot, const double* X, long long ldx, double* L, long long ldl,
                       double* tau, long long* piv, int* info, void* workspace, size_t workspace_bytes,
                       void* stream) {
  if (width < 1) return SKL_BAD_ARGUMENT;
  return blk_driver(n, width, SKL_VAR2A, pivot ? 1 : 0, width, X, ldx, L, ldl, tau, pivot ? piv : nullptr, info,
                    workspace, workspace_bytes, stream);
}

// ---------------------------------------------------------------------------
// host-buffer driver: [dXL (n*n) | tau (n) | piv (n) | blk workspace]
namespace {
constexpr int kHostBlock = 128;
size_t host_ws_head(int n) {
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  return al(sizeof(double) * (size_t)n * n) + al(sizeof(double) * n) + al(sizeof(long long) * n);
}
}  // namespace

size_t skl_ltlt_blk_piv_host_workspace_size(int n, int nb, int variant) {
  if (n < 1 || nb < 1) return 0;
  size_t blk = skl_ltlt_blk_piv_workspace_size(n, nb, variant);
  if (blk == 0 && n > 1) return 0;
  return host_ws_head(n) + blk;
}

int skl_ltlt_blk_piv_host(int n, int nb, int variant, const double* X_host, long long ldx, double* L_host,
                          long long ldl, double* tau_host, long long* piv_host, void* workspace,
                          size_t workspace_bytes, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (variant < SKL_VAR1 || variant > SKL_VAR2B) return SKL_UNSUPPORTED;
  if (n < 1 || nb < 1 || ldx < n || ldl < n || !X_host || !L_host || (n > 1 && !tau_host) || !piv_host)
    return SKL_BAD_ARGUMENT;
  const size_t need = skl_ltlt_blk_piv_host_workspace_size(n, nb, variant);
  if (need == 0) return SKL_UNSUPPORTED;
  if (workspace_bytes < need) return SKL_BAD_ARGUMENT;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  unsigned char* base = static_cast<unsigned char*>(workspace);
  double* dXL = reinterpret_cast<double*>(base);
  double* dtau = reinterpret_cast<double*>(base + al(sizeof(double) * (size_t)n * n));
  long long* dpiv = reinterpret_cast<long long*>(base + al(sizeof(double) * (size_t)n * n) + al(sizeof(double) * n));
  void* wsb = base + host_ws_head(n);
  const size_t wsb_bytes = workspace_bytes - host_ws_head(n);
  // lower trapezoid of X, one 2-D copy per 128-column block
  for (int j0 = 0; j0 < n; j0 += kHostBlock) {
    const int w = std::min(kHostBlock, n - j0);
    SKL_TRY(cudaMemcpy2DAsync(dXL + (size_t)j0 * n + j0, sizeof(double) * n, X_host + (size_t)j0 * ldx + j0,
                              sizeof(double) * ldx, sizeof(double) * (n - j0), w, cudaMemcpyHostToDevice, st));
  }
  // in place on the device (L == X): the diagonal blocks keep X's upper values
  int rc = skl_ltlt_blk_piv(n, nb, variant, dXL, n, dXL, n, dtau, dpiv, wsb, wsb_bytes, stream);
  if (rc != SKL_OK) return rc;
  for (int j0 = 0; j0 < n; j0 += kHostBlock) {
    const int w = std::min(kHostBlock, n - j0);
    SKL_TRY(cudaMemcpy2DAsync(L_host + (size_t)j0 * ldl + j0, sizeof(double) * ldl, dXL + (size_t)j0 * n + j0,
                              sizeof(double) * n, sizeof(double) * (n - j0), w, cudaMemcpyDeviceToHost, st));
  }
  if (n > 1) SKL_TRY(cudaMemcpyAsync(tau_host, dtau, sizeof(double) * (n - 1), cudaMemcpyDeviceToHost, st));
  SKL_TRY(cudaMemcpyAsync(piv_host, dpiv, sizeof(long long) * n, cudaMemcpyDeviceToHost, st));
  return SKL_OK;
}

// ---------------------------------------------------------------------------
size_t skl_ltlt_solve_workspace_size(int n, int nrhs) {
  if (n < 1 || nrhs < 1) return 0;
  return skl::solve_workspace_bytes(n, nrhs);
}

int skl_ltlt_solve(int n, int nrhs, const double* L, long long ldl, const double* tau, const long long* piv,
                   double* B, long long ldb, double tol_scale, int* info, void* workspace, size_t workspace_bytes,
                   void* stream) {
  if (n < 1 || nrhs < 1 || ldl < n || ldb < n || !L || !piv || !B || !info || (n > 1 && !tau))
    return SKL_BAD_ARGUMENT;
  if (workspace_bytes < skl::solve_workspace_bytes(n, nrhs)) return SKL_BAD_ARGUMENT;
  g_kt.launches += 6 + 4 * ((n + 63) / 64);
  SKL_TRY(skl::launch_solve(n, nrhs, L, ldl, tau, piv, B, ldb, tol_scale, info, workspace,
                            static_cast<cudaStream_t>(stream)));
  return SKL_OK;
}

// ---------------------------------------------------------------------------
// From n = 128 up the two-step factorization is computed faster by the blocked
// driver (left-looking cluster panel + DMMA trailing update): the same L, T and
// pivots in exact arithmetic, and the cluster two-step kernel pays five cluster
// barriers per column pair (n=512: 1.50 vs 2.54 ms; n=1024: 2.9 vs 13.2 ms).
namespace {
constexpr int kTwostepViaBlocked = 128;
size_t twostep_blocked_ws(int n) {
  std::vector<PanelPlan> plan;
  if (n < kTwostepViaBlocked || !make_schedule(n, n, SKL_VAR1, plan)) return 0;
  return layout_blk(n, n, plan, nullptr, nullptr);
}
}  // namespace

size_t skl_ltlt_unb_twostep_workspace_size(int n) {
  return std::max(skl::twostep_workspace_bytes(n), twostep_blocked_ws(n));
}

int skl_ltlt_unb_twostep(int n, int pivot, const double* X, long long ldx, double* L, long long ldl, double* tau,
                         long long* piv, int* info_dev, void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 1 || ldx < n || ldl < n) return SKL_BAD_ARGUMENT;
  static int via_blocked = env_int("SKL_TWOSTEP_VIA_BLOCKED", 1);
  const size_t blk_ws = via_blocked ? twostep_blocked_ws(n) : 0;
  if (blk_ws > 0 && workspace_bytes >= blk_ws && info_dev != nullptr)
    return blk_driver(n, n, SKL_VAR1, pivot ? 1 : 0, -1, X, ldx, L, ldl, tau, pivot ? piv : nullptr, info_dev,
                      workspace, workspace_bytes, stream);
  if (workspace_bytes < skl::twostep_workspace_bytes(n)) return SKL_BAD_ARGUMENT;
  g_kt.launches += (L != X) ? 2 : 1;
  SKL_TRY(skl::launch_twostep(X, ldx, L, ldl, n, pivot, tau, piv, info_dev, workspace,
                              static_cast<cudaStream_t>(stream)));
  return SKL_OK;
}

int skl_ltlt_batched_piv(int batch, int n, int dtype, const void* X, long long ldx, long long strideX, void* L,
                         long long ldl, long long strideL, void* tau, long long* piv, double* pf_sign,
                         double* pf_logabs, void* stream) {
  if (batch < 0 || n < 1 || ldx < n || ldl < n) return SKL_BAD_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (batch == 0) return SKL_OK;
  if (n > 512) {
    g_last_error = "batched factorization: n > 512 (one CTA per matrix, at most two rows per thread)";
    return SKL_UNSUPPORTED;
  }
  {
    // L is written while X is still read (the upper triangle is copied last)
    const size_t es = dtype == SKL_F32 ? sizeof(float) : sizeof(double);
    const size_t xb = es * (size_t)((long long)(batch - 1) * strideX + ldx * (n - 1) + n);
    const size_t lb = es * (size_t)((long long)(batch - 1) * strideL + ldl * (n - 1) + n);
    if (overlaps(X, xb, L, lb)) return SKL_ALIAS;
  }
  if (dtype == SKL_F64) {
    SKL_TRY(skl::launch_batched<double>(batch, n, static_cast<const double*>(X), ldx, strideX,
                                        static_cast<double*>(L), ldl, strideL, static_cast<double*>(tau), n - 1,
                                        piv, n, pf_sign, pf_logabs, st));
  } else if (dtype == SKL_F32) {
    SKL_TRY(skl::launch_batched<float>(batch, n, static_cast<const float*>(X), ldx, strideX, static_cast<float*>(L),
                                       ldl, strideL, static_cast<float*>(tau), n - 1, piv, n, pf_sign, pf_logabs,
                                       st));
  } else {
    return SKL_UNSUPPORTED;
  }
  return SKL_OK;
}

}  // extern "C"
