/*
 * skewltl_b200 — C ABI of the B200 (sm_100a) pivoted LTL^T hot path.
 *
 * Drop-in boundary for the reference `skewltl` package (arXiv 2411.09859
 * artefact).  The reference is pure Python (numpy/OpenBLAS); each entry point
 * below replaces the reference function named in its comment, with the same
 * argument meaning, in-place/ownership rules and error behaviour, expressed
 * as plain pointers and sizes.  The Python mirror package
 * `paper_2411_09859_b200` binds these with ctypes.
 *
 * Conventions
 *   - every matrix pointer is DEVICE memory, column-major, with explicit ld;
 *     skew matrices are stored as their strictly-lower triangle, entries on or
 *     above the diagonal are never read (and never written except where a
 *     function says it copies them);
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream); no
 *     function synchronises the stream;
 *   - device scalars/arrays documented as such are written asynchronously;
 *   - return value: skl_status; on SKL_CUDA_ERROR skl_last_error() describes it.
 */
#ifndef SKEWLTL_B200_H
#define SKEWLTL_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SKL_OK = 0,
  SKL_ZERO_PIVOT = 1,  /* unpivoted breakdown; column in *info (core.py:17-22 ZeroPivot) */
  SKL_BAD_ARGUMENT = 2, /* dimension / ld / block mismatch (ValueError) */
  SKL_ALIAS = 3,        /* output aliases an operand (kernels3.py:64-66) */
  SKL_CUDA_ERROR = 4,
  SKL_UNSUPPORTED = 5,  /* e.g. variant name (InvalidVariant, blocked.py:314-315) */
  SKL_BAD_PIVOT = 6     /* pivot index out of range (IndexError, core.py:306-307) */
} skl_status;

/* trailing-update scheme of the pivoted blocked driver (blocked.py:35) */
enum { SKL_VAR1 = 0, SKL_VAR2A = 1, SKL_VAR2B = 2, SKL_LEFT = 3 /* skl_ltlt_blk, unpivoted only */ };
enum { SKL_F64 = 0, SKL_F32 = 1 };

const char* skl_version(void);
const char* skl_last_error(void);

/* ---- level-3: trailing sandwiched updates --------------------------------
 * skew_rank2k (kernels3.py:305-351):
 *   C_lower := beta*C + alpha*(A B^T - B A^T); A, B are n x k; with
 *   skip_zero_cols, columns zero in A or in B are dropped (keff <= k).
 *   *keff_dev (device int, may be NULL) receives keff.                     */
size_t skl_skr2k_workspace_size(int n, int k);
int skl_skr2k_lower(int n, int k, double alpha, const double* A, long long lda, const double* B, long long ldb,
                    double beta, double* C, long long ldc, int skip_zero_cols, void* workspace,
                    size_t workspace_bytes, int* keff_dev, void* stream);

/* skew_tridiag_rankk (kernels3.py:151-209):
 *   C_lower := beta*C + alpha * A T A^T, T = tridiag(tau[0..k-2]) skew.     */
/* skew_tridiag_gemm (kernels3.py:239-302): C (p x q) := beta*C + alpha*A (T B)
 *   with A (p x k), B (k x q), T = tridiag(tau) skew (T[i+1,i] = tau_i,
 *   T[i,i+1] = -tau_i).  tril != 0 writes only the entries with row > col
 *   (the trapezoidal from-the-left update of ltlt_blk_left, blocked.py:236-265);
 *   otherwise every entry.  C must not alias A or B (SKL_ALIAS).            */
size_t skl_skew_tridiag_gemm_workspace_size(int p, int q, int k);
int skl_skew_tridiag_gemm(int p, int q, int k, double alpha, const double* A, long long lda, const double* tau,
                          const double* B, long long ldb, double beta, double* C, long long ldc, int tril,
                          void* workspace, size_t workspace_bytes, void* stream);

size_t skl_sktri_rankk_workspace_size(int n, int k);
int skl_sktri_rankk_lower(int n, int k, double alpha, const double* A, long long lda, const double* tau,
                          double beta, double* C, long long ldc, void* workspace, size_t workspace_bytes,
                          void* stream);

/* form_w + form_s_splitting (kernels3.py:354-364, core.py:153-169):
 *   W = A S with T = S - S^T, tau of length k-1; even columns of W are 0.   */
int skl_form_w(int n, int k, const double* A, long long lda, const double* tau, double* W, long long ldw,
               void* stream);

/* ---- level-2 --------------------------------------------------------------
 * skew_rank2 (kernels2.py:93-131): A_lower := beta*A + alpha*(x y^T - y x^T) */
int skl_skew_rank2_lower(int n, double alpha, const double* x, const double* y, double beta, double* A,
                         long long lda, void* stream);

/* gen_rank2 (kernels2.py:134-163): A := beta*A + alpha*(x u^T + y v^T) on a p x q
 * column-major rectangle (x, y length p; u, v length q) */
int skl_gen_rank2(int p, int q, double alpha, const double* x, const double* u, const double* y, const double* v,
                  double beta, double* A, long long lda, void* stream);

/* skew_tridiag_gemv (kernels2.py:178-229):
 *   y := beta*y + alpha*(A (T x))[tail_from:], A is p x k, T = tridiag(tau[0..k-2]) */
int skl_skew_tridiag_gemv(int p, int k, double alpha, const double* A, long long lda, const double* tau,
                          const double* x, double beta, double* y, int tail_from, void* stream);

/* apply_row_pivots (kernels2.py:232-271): rows [lo, hi) of the n x q block
 *   := rows idx[lo..hi) (idx: device int64 gather index of length n, composed
 *   on the host from the pivot vector exactly as the reference does).       */
size_t skl_apply_row_pivots_workspace_size(int q, int lo, int hi);
int skl_apply_row_pivots(int n, int q, double* block, long long ld, const long long* idx, int lo, int hi,
                         void* workspace, size_t workspace_bytes, void* stream);

/* apply_symmetric_pivot (core.py:327-333): X := P X P^T, P = (k, k+pi).     */
int skl_apply_symmetric_pivot(int n, double* X, long long ld, int k, long long pi, void* stream);

/* pack_in_place (core.py:349-362): X[j+1, j] = tau[j], X[j+2:, j] = L[j+2:, j]
 *   (the LAPACK-style packed factor; only the strictly-lower triangle of X is
 *   written).  unpack_in_place (core.py:365-375): the exact inverse into a
 *   fresh "ones" L buffer (every entry written) and tau (n-1); L must not
 *   alias X.                                                                  */
int skl_pack_factor(int n, const double* L, long long ldl, const double* tau, double* X, long long ldx, void* stream);
int skl_unpack_factor(int n, const double* X, long long ldx, double* L, long long ldl, double* tau, void* stream);

/* ---- factorization drivers -------------------------------------------------
 * ltlt_blk_piv (blocked.py:303-363): pivoted blocked right-looking LTL^T.
 *   X (n x n, lower read) is not modified.  L (n x n) receives the work
 *   buffer of the reference: L column j (j>=1) in column j-1 below the
 *   diagonal with an explicit 1 at [j, j-1] (UnitLowerFactor "ones",
 *   core.py:172-186); if L != X its upper triangle and diagonal are copied
 *   from X.  tau (n-1) and piv (n, int64 relative offsets, piv[0] = 0) are
 *   device outputs.  variant: SKL_VAR1 / SKL_VAR2A / SKL_VAR2B.             */
size_t skl_ltlt_blk_piv_workspace_size(int n, int nb, int variant);
/* GPU panel schedule of skl_ltlt_blk_piv (a query, no device work): the panel
 *   width on the GPU may be narrower than nb when the panel block would not fit
 *   on-chip (the factorization is invariant to it).  Writes up to cap entries
 *   r[i] (first column), nelim[i] (columns eliminated), kind[i] (2: cluster
 *   panel, ctas[i] CTAs in clusters of csize[i]; 0: grid-wide panel); returns
 *   the number of panels, or -1 when the configuration is unsupported.      */
int skl_ltlt_blk_piv_plan(int n, int nb, int variant, int* r, int* nelim, int* kind, int* ctas, int* csize,
                          int cap);
int skl_ltlt_blk_piv(int n, int nb, int variant, const double* X, long long ldx, double* L, long long ldl,
                     double* tau, long long* piv, void* workspace, size_t workspace_bytes, void* stream);

/* Pivoted or unpivoted blocked LTL^T (blocked.py:162-233 ltlt_blk_var1/2a/2b,
 *   blocked.py:303-363 ltlt_blk_piv).  pivot = 1: identical to skl_ltlt_blk_piv
 *   (piv required).  pivot = 0: the pivot row of every step is row g+1; an exact
 *   zero pivot with a nonzero column below it (unblocked.py:83-85) stores the
 *   first such column + 1 in the device int *info (0 = success) -- ZeroPivot
 *   on the host -- and the factors are then meaningless; piv is not written
 *   (may be null).  Same layout/workspace as skl_ltlt_blk_piv (its size query). */
int skl_ltlt_blk(int n, int nb, int variant, int pivot, const double* X, long long ldx, double* L, long long ldl,
                 double* tau, long long* piv, int* info, void* workspace, size_t workspace_bytes, void* stream);

/* ltlt_unb_panel (unblocked.py:243-275): eliminate only columns [0, width) of
 *   the whole matrix (left-looking, optional pivoting).  L receives the work
 *   buffer; only its columns [0, min(width, n-1)) are meaningful (the
 *   reference returns zeros elsewhere), tau[0:width), piv[0:width+1).         */
size_t skl_ltlt_unb_panel_workspace_size(int n, int width);
int skl_ltlt_unb_panel(int n, int width, int pivot, const double* X, long long ldx, double* L, long long ldl,
                       double* tau, long long* piv, int* info, void* workspace, size_t workspace_bytes,
                       void* stream);

/* solve (apps.py:76-100): X y = b from a pivoted factorization (L "ones"
 *   buffer, tau, piv as written by skl_ltlt_blk_piv).  B (n x nrhs, device,
 *   column-major) is overwritten by y.  A numerically singular T (a pivot at or
 *   below tol_scale * eps * max|tau|, apps.py:47-65; every odd n) stores the
 *   row + 1 in the device int *info (0 = success) -- SingularT on the host --
 *   and B is then meaningless.                                                */
size_t skl_ltlt_solve_workspace_size(int n, int nrhs);
int skl_ltlt_solve(int n, int nrhs, const double* L, long long ldl, const double* tau, const long long* piv,
                   double* B, long long ldb, double tol_scale, int* info, void* workspace, size_t workspace_bytes,
                   void* stream);

/* Same factorization from HOST buffers (the drop-in call with H2D/D2H inside;
 * X_host/L_host column-major, pinned for asynchronous copies).  Only the
 * lower part travels: column blocks [j0, j0+128) move rows [j0, n), i.e. the
 * strict lower triangle plus the 128x128 diagonal blocks.  L_host receives
 * the reference's work buffer on those blocks (the factor with its explicit
 * ones below the diagonal; X's values on/above the diagonal inside the
 * diagonal blocks); the rest of L_host's upper triangle is not written (it is
 * X's upper triangle in the reference's buffer: pass L_host == X_host, or a
 * copy of X, for a bit-identical buffer).  tau_host (n-1), piv_host (n).
 * workspace: device bytes from skl_ltlt_blk_piv_host_workspace_size.  The
 * call is stream-ordered: outputs are valid after the stream synchronizes. */
size_t skl_ltlt_blk_piv_host_workspace_size(int n, int nb, int variant);
int skl_ltlt_blk_piv_host(int n, int nb, int variant, const double* X_host, long long ldx, double* L_host,
                          long long ldl, double* tau_host, long long* piv_host, void* workspace,
                          size_t workspace_bytes, void* stream);

/* ltlt_unb_twostep (unblocked.py:229-240): Wimmer two-step, optional pivoting.
 *   Same output layout.  Unpivoted breakdown: *info_dev (device int) is set
 *   to the column + 1 (0 = success) — ZeroPivot(column) on the host.        */
size_t skl_ltlt_unb_twostep_workspace_size(int n);
int skl_ltlt_unb_twostep(int n, int pivot, const double* X, long long ldx, double* L, long long ldl, double* tau,
                         long long* piv, int* info_dev, void* workspace, size_t workspace_bytes, void* stream);

/* Batched pivoted factorization + Pfaffian (pfaffian, apps.py:12-30, applied
 * to `batch` independent matrices).  dtype SKL_F64 or SKL_F32 selects the
 * element type of X, L and tau.  Matrix b lives at X + b*strideX (elements).
 * pf_sign/pf_logabs (device doubles, may be NULL) receive sign(Pf) and
 * log|Pf| (overflow-free form of apps.py:26-30).                            */
int skl_ltlt_batched_piv(int batch, int n, int dtype, const void* X, long long ldx, long long strideX, void* L,
                         long long ldl, long long strideL, void* tau, long long* piv, double* pf_sign,
                         double* pf_logabs, void* stream);

/* ---- block-cyclic multi-GPU factorization (config 5) ----------
 * The reference has no distributed path; this is the GPU counterpart of
 * ltlt_blk_piv (blocked.py:303-363) over G ranks, one process per GPU.
 *
 * W (n x n, column stride ldw) is ONE virtual address range on every rank in
 *   which column block j = [j*nbd, (j+1)*nbd) is backed by the memory of rank
 *   j % G (skl_vmm_* below; the host layer maps it).  On entry every rank's
 *   blocks hold X's lower triangle; W is the work buffer (destroyed).
 * L (same block-cyclic mapping, stride ldl) receives, for the columns this
 *   process drives, the "ones" L buffer of skl_ltlt_blk_piv (strict lower part).
 * shared (skl_ltlt_dist_shared_size bytes, one range visible to all ranks):
 *   tau (n-1 doubles) at off_tau and piv (n int64) at off_piv
 *   (skl_ltlt_dist_offsets); the rest is panel state.
 * Ranks [rank_lo, rank_hi) are driven by this process: one rank per process on
 *   a multi-GPU node (barrier required: a stream-ordered cross-rank barrier,
 *   e.g. skl_nccl_barrier), or all G ranks in one process on one device (no
 *   barrier; the same kernels with every rank's column filter).
 * Per panel: the owner of the panel's first column runs the pivoted panel
 *   (pivot-column gathers and interchanges over peer memory), barrier, every
 *   rank packs the panel operands and updates the trailing columns it owns
 *   (column-filtered DMMA GEMM), barrier.                                     */
typedef int (*skl_barrier_fn)(void* ctx, void* stream);
size_t skl_ltlt_dist_shared_size(int n, int nb, int variant);
size_t skl_ltlt_dist_workspace_size(int n, int nb, int variant, int nranks_local);
int skl_ltlt_dist_offsets(int n, int nb, int variant, size_t* off_tau, size_t* off_piv, size_t* off_gperm,
                          int* npanels);
int skl_ltlt_blk_piv_dist(int n, int nb, int variant, int nbd, int nranks, int rank_lo, int rank_hi, double* W,
                          long long ldw, double* L, long long ldl, void* shared, void* workspace,
                          size_t workspace_bytes, skl_barrier_fn barrier, void* barrier_ctx, void* stream);
/* host only: owned-tile table of the column-filtered trailing GEMM (the lower
 *   triangle of an n x n region whose column 0 is global column cbase):
 *   tab = [m, total, (tile column, first tile, partial, first tile row) x m];
 *   tab_ints >= 2 + 4*ceil(n/128).                                                       */
int skl_dist_owner_table(int n, long long cbase, int nbd, int nranks, int rank, int* tab, size_t tab_ints);

/* CUDA VMM plumbing (driver API through cudaGetDriverEntryPoint): physical
 * allocations (exportable as POSIX fds for the peer processes), virtual ranges,
 * block mapping with read/write access for `device`.                        */
int skl_vmm_available(void);
int skl_vmm_last_result(void); /* CUresult of the last skl_vmm_* driver call */
int skl_vmm_granularity(int device, size_t* gran);
int skl_vmm_create(size_t bytes, int device, int exportable, unsigned long long* handle);
int skl_vmm_export_fd(unsigned long long handle, int* fd);
int skl_vmm_import_fd(int fd, unsigned long long* handle);
int skl_vmm_release(unsigned long long handle);
int skl_vmm_reserve(size_t bytes, size_t align, unsigned long long* va);
int skl_vmm_free_va(unsigned long long va, size_t bytes);
int skl_vmm_map(unsigned long long va, size_t bytes, unsigned long long handle, size_t offset, int device);
int skl_vmm_unmap(unsigned long long va, size_t bytes);

/* NCCL stream-ordered barrier (libnccl.so.2 via dlopen): a one-word
 * all-reduce on the caller's stream; skl_nccl_barrier matches skl_barrier_fn. */
int skl_nccl_available(void);
int skl_nccl_unique_id(unsigned char* out, size_t bytes);
int skl_nccl_barrier_create(int nranks, int rank, const unsigned char* id, void** ctx);
int skl_nccl_barrier(void* ctx, void* stream);
int skl_nccl_barrier_destroy(void* ctx);

/* ---- instrumentation (bench / profiling) ---------------------------------
 * skl_timing_enable(1) records CUDA events around every kernel the blocked
 * driver launches, by class (0 panel, 1 operand pack, 2 trailing GEMM,
 * 3 finalize); skl_timing_read() returns total ms and launch counts per class
 * after the caller synchronised the stream.  skl_launch_count() counts
 * library kernel launches since the last skl_timing_enable().               */
int skl_timing_enable(int on);
int skl_timing_read(double* ms4, int* count4);
long long skl_launch_count(void);
int skl_debug_set_panel_profile(unsigned long long* dev_buf);

#ifdef __cplusplus
}
#endif

#endif /* SKEWLTL_B200_H */
