// Internal (non-exported) launchers shared between the translation units of
// libskewltl_b200.so.  Every launcher enqueues on `stream` and never syncs.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace skl {

// ---- packed operand layout for the lower-triangular DGEMM-NT --------------
// An operand X (rows x K) is stored as 128-row tiles; inside a tile, K is
// split into k4 blocks of 4 columns and rows into 16 blocks of 8; the 32
// doubles of an (8 x 4) block are in DMMA-fragment lane order
// (lane = 4*(row%8) + col%4).  One k4 block of one tile is 4 KiB contiguous.
constexpr int kTile = 128;
__host__ __device__ inline int tiles_for(int rows) { return (rows + kTile - 1) / kTile; }
__host__ __device__ inline size_t packed_elems(int rows, int k4cap) { return (size_t)tiles_for(rows) * kTile * 4 * k4cap; }

// Block-cyclic column ownership of a GEMM launch (multi-GPU driver): only C
// columns c (global index cbase + c) with (c / nbd) % G == rank are written;
// tab (device) is the owned-tile table build_owner_table() fills.
struct ColOwner {
  const int* tab;
  int ntiles;
  long long cbase;
  int nbd, G, rank;
};
// host: owned-tile table for the lower triangle of an n x n region whose column
// 0 is global column cbase; tab needs 2 + 3*tiles_for(n) ints; returns the tile count
int build_owner_table(int n, long long cbase, int nbd, int G, int rank, int* tab);
inline size_t owner_table_ints(int n) { return 2 + 4 * (size_t)tiles_for(n); }
// host: tile table of a general p x q block (tri = 0) or of its strictly-lower
// trapezoid (tri = 1) for launch_gemm_lower(..., own, q, tri); tab needs
// owner_table_ints(q) ints; returns the tile count
int build_rect_table(int p, int q, int tri, int* tab);

// C[i,j] (i>j, i,j < n) = beta*C[i,j] + sum_k P[i,k] Q[j,k]
// nk4_dev (optional) overrides nk4 with a device-resident count; own (optional)
// restricts the update to one rank's columns.
cudaError_t launch_gemm_lower(const double* P, const double* Q, int k4cap, int nk4, const int* nk4_dev,
                              double* C, long long ldc, int n, double beta, cudaStream_t stream,
                              const ColOwner* own = nullptr, int ncols = -1, int tri = 1);

// skew_tridiag_gemm operands: P = alpha*A (p x k), Q = (T B)^T (q x k) with
// B (k x q, column stride ldb) and T tridiag(t): Q[j,c] = t[c-1] B[c-1,j] - t[c] B[c+1,j]
// btrans = 1: B is passed as B^T (q x k column-major, stride ldb)
cudaError_t launch_pack_gemm(const double* A, long long lda, int p, const double* B, long long ldb, int q, int k,
                             const double* t, double alpha, int k4cap, double* P, double* Q, cudaStream_t stream,
                             int btrans = 0);
// C (p x q) *= beta on every entry (tri = 0) or on row > col only
cudaError_t launch_scale_block(double* C, long long ldc, int p, int q, double beta, int tri, cudaStream_t stream);

// P = alpha*A, Q = A T^T with T tridiag(t) (t = tau_base[0..ka-2]); optional
// var1 straggler columns (l = A[:, ka-1], y) zeroed on row 0.  shift > 0
// prepends that many zero rows (P, Q then hold rows + shift rows).
cudaError_t launch_pack_rankk(const double* A, long long lda, int rows, int ka, const double* tau_base,
                              double alpha, const double* y, int k4cap, double* P, double* Q,
                              cudaStream_t stream, int shift = 0);

// rows/columns of zero padding that put the trailing C region [rt:, rt:] of a
// column-major matrix with leading dimension ld on 128-byte lines (TMA boxes
// and L2 lines then never straddle); 0 when ld is not a multiple of 16
inline int align_shift(int rt, long long ld) { return (ld % 16 == 0) ? (rt & 15) : 0; }

// skr2k: keep[] (device) lists columns nonzero in both A and B; count at keff_dev.
cudaError_t launch_rank2k_keep(const double* A, long long lda, const double* B, long long ldb, int n, int k,
                               int skip_zero, int* keep, int* keff_dev, int* nk4_dev, cudaStream_t stream);
cudaError_t launch_pack_rank2k(const double* A, long long lda, const double* B, long long ldb, int n, int k,
                               double alpha, const int* keep, const int* keff_dev, int k4cap, double* P,
                               double* Q, cudaStream_t stream);

// the same prologue (keep list + packed operands) in one cooperative launch;
// part: rank2k_prep_scratch_words(k) words of scratch; cnt[0] = keff, cnt[1] = nk4
size_t rank2k_prep_scratch_words(int k);
cudaError_t launch_rank2k_prep(const double* A, long long lda, const double* B, long long ldb, int n, int k,
                               int skip_zero, double alpha, int k4cap, unsigned* part, int* keep, int* cnt, double* P,
                               double* Q, cudaStream_t stream);

cudaError_t launch_form_w(const double* A, long long lda, int n, int k, const double* tau, double* W,
                          long long ldw, cudaStream_t stream);

// ---- level-2 kernels ------------------------------------------------------
cudaError_t launch_skew_rank2(double* A, long long lda, int n, double alpha, const double* x, const double* y,
                              double beta, cudaStream_t stream);
cudaError_t launch_gen_rank2(double* A, long long lda, int p, int q, double alpha, const double* x,
                            const double* u, const double* y, const double* v, double beta, cudaStream_t stream);
cudaError_t launch_skew_tridiag_gemv(double* y, double alpha, const double* A, long long lda, int p, int k,
                                     const double* tau, const double* x, double beta, int tail_from,
                                     cudaStream_t stream);
cudaError_t launch_gather_rows(double* block, long long ld, int q, int lo, int hi, const long long* idx_dev,
                               double* tmp, cudaStream_t stream);
cudaError_t launch_sym_swap(double* X, long long ld, int n, int a, int b, cudaStream_t stream);
template <typename T>
cudaError_t launch_scale_lower(T* C, long long ldc, int n, T beta, cudaStream_t stream);

// ---- factorization pieces -------------------------------------------------
struct PanelArgs {
  double* W;             // n x n work buffer (lower storage, column-major)
  long long ld;
  int n;
  int r, nelim, lo;      // eliminate columns [r, r+nelim); leftmost participating column lo
  int want_y;            // var1: compute y = column rt after the trailing couplings
  double* tau;           // device tau (length n-1)
  long long* piv;        // device pivots (length n)
  double* y;             // device y vector (position indexed), var1 only
  int* gperm;            // out: position -> physical map of this panel (length n)
  int* disp_list;        // scratch: displaced trailing positions
  int* disp_count;       // scratch counter (zeroed by the kernel launcher)
  double* side;          // scratch: displaced trailing lines (2*nelim x n)
  uint64_t* slots;       // LL exchange area
  uint64_t* rowa;        // LL exchange area for the row being displaced
  uint64_t* recs;        // LL candidate records [2][P][4]
  double* crow;          // cluster panel: candidate rows [2][C][kmax+2]
  double* arowg;         // cluster panel: row a [2][kmax+2]
  double* rowmir;        // lean panel: row-major mirror of the slab [rows][push_crs(kmax)] (multicast source)
  double* pbuf;          // multi-cluster panel: slab output [kmax][n]
  uint32_t tag0;         // first LL tag of this panel
  int nblocks;           // CTAs (co-resident)
  int rows_per;          // rows per CTA
  int kmax;              // slab columns (= r + nelim - lo)
  int slot_words;
  int dbg;               // timing experiments only (bitmask of skipped phases)
  unsigned long long* prof;  // optional per-CTA phase cycle totals [C][16]
  int pivot;             // 0: unpivoted (pivot row = row g+1), exact-zero breakdown -> *info
  int* info;             // device: first breaking column + 1 (0 = none); may be null when pivot
  int push;              // single-cluster pivoted panel: candidate rows pushed by st.async, lazy interchanges
  int defer_finish;      // 1: the launcher leaves the finish kernels to launch_panel_finish_pack()
  int count_zeroed;      // 1: disp_count is already zero (the previous panel's fused epilogue reset it)
};
size_t panel_smem_bytes(int rows_per, int kmax);
int panel_max_ctas();
int panel_threads();
cudaError_t launch_panel(const PanelArgs& a, cudaStream_t stream);
// single-cluster variant (DSMEM exchange); cluster size 16 (or 8), 0 if unavailable
int panel_cluster_size();
size_t panel_cluster_smem_bytes(int rows_per, int kmax, int npush = 0);
// the lean single-cluster push panel (panel_push_kernel): shared memory, and whether a plan runs on it
size_t panel_push_smem_bytes(int rows_per, int kmax);
bool panel_push_usable(bool push_pivot, int ctas, int csize, int rows_per, int kmax);
cudaError_t launch_panel_cluster(const PanelArgs& a, cudaStream_t stream);
// multi-cluster variant (cooperative; intra-cluster DSMEM + inter-cluster LL exchange)
int panel_multi_clusters(int csize, size_t smem);
cudaError_t launch_panel_multi(const PanelArgs& a, int csize, cudaStream_t stream);
// Panel epilogue and operand packing in ONE cooperative launch (a.defer_finish = 1 panels):
// displaced trailing lines -> side buffer and P / Q packed straight from the panel buffer,
// grid barrier, panel buffer -> L columns and side -> trailing lines.  Same results as
// launch_panel_finish + launch_pack_rankk (three launches of ~6 us each per panel).
struct FinishPack {
  int rows, ka, k4cap, shift;  // trailing rows, panel columns, packed k4 capacity, alignment shift
  const double* t;             // tau of the panel columns (ka - 1 couplings)
  const double* y;             // var1 straggler vector (position indexed from rt) or null
  double* P;
  double* Q;
};
cudaError_t launch_panel_finish_pack(const PanelArgs& a, const FinishPack& f, cudaStream_t stream);

// packed factor layout (core.py:349-375)
cudaError_t launch_pack_factor(int n, const double* L, long long ldl, const double* tau, double* X, long long ldx,
                               cudaStream_t stream);
cudaError_t launch_unpack_factor(int n, const double* X, long long ldx, double* L, long long ldl, double* tau,
                                 cudaStream_t stream);

// linear solve on top of the factorization (solve.cu); B (n x nrhs) is overwritten
size_t solve_workspace_bytes(int n, int nrhs);
cudaError_t launch_solve(int n, int nrhs, const double* L, long long ldl, const double* tau, const long long* piv,
                         double* B, long long ldb, double tol_scale, int* info, void* ws, cudaStream_t stream);

cudaError_t launch_compose_suffix(const int* gperm_all, int npanels, const int* row0s, int n, int* sigma_all,
                                  cudaStream_t stream);
// own_g > 1: only the columns c with (c / own_nbd) % own_g == own_rank
cudaError_t launch_finalize_l(const double* W, long long ldw, const double* X, long long ldx, double* L,
                              long long ldl, int n, const int* col_group, const int* sigma_all, int copy_upper,
                              cudaStream_t stream, int own_nbd = 1, int own_g = 1, int own_rank = 0);

// ---- unblocked two-step (config 1) and batched (config 4) ------------------
cudaError_t launch_twostep(const double* X, long long ldx, double* L, long long ldl, int n, int pivot,
                           double* tau, long long* piv, int* info, void* workspace, cudaStream_t stream);
size_t twostep_workspace_bytes(int n);

template <typename T>
cudaError_t launch_batched(int batch, int n, const T* X, long long ldx, long long strideX, T* L, long long ldl,
                           long long strideL, T* tau, long long strideTau, long long* piv, long long stridePiv,
                           double* pf_sign, double* pf_logabs, cudaStream_t stream);

}  // namespace skl
