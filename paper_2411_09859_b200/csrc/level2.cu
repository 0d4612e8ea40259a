// Level-2 kernels behind the reference's kernels2.py API.
//   skew_rank2         kernels2.py:93-131   A_lower := beta A + alpha (x y^T - y x^T)
//   gen_rank2          kernels2.py:134-163  A := beta A + alpha (x u^T + y v^T), p x q rectangle
//   skew_tridiag_gemv  kernels2.py:178-229  y := beta y + alpha (A (T x))[tail_from:]
//   apply_row_pivots   kernels2.py:232-271  rows [lo, hi) := rows idx[lo:hi] (one gather)
//   _sym_swap_lower    core.py:294-324      X := P X P^T for one transposition
// These are the stand-alone API kernels; inside the factorization the same
// operations are fused into the panel / trailing kernels.
#include "common.cuh"
#include "internal.h"

namespace skl {
namespace {

// one CTA per column block; threads stride rows (coalesced in column-major)
__global__ void skew_rank2_kernel(double* __restrict__ A, long long lda, int n, double alpha,
                                  const double* __restrict__ x, const double* __restrict__ y, double beta) {
  for (int j = blockIdx.y; j < n; j += gridDim.y) {
    const double xj = x[j], yj = y[j];
    for (int i = j + 1 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      double* p = A + (long long)j * lda + i;
      double upd = alpha * (x[i] * yj - y[i] * xj);
      *p = (beta == 1.0) ? *p + upd : beta * *p + upd;
    }
  }
}

// general rank-2 on a p x q column-major rectangle (HBM-bound: one read + one write per entry)
__global__ void gen_rank2_kernel(double* __restrict__ A, long long lda, int p, int q, double alpha,
                                 const double* __restrict__ x, const double* __restrict__ u,
                                 const double* __restrict__ y, const double* __restrict__ v, double beta) {
  for (int j = blockIdx.y; j < q; j += gridDim.y) {
    const double uj = alpha * u[j], vj = alpha * v[j];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p; i += gridDim.x * blockDim.x) {
      double* e = A + (long long)j * lda + i;
      const double upd = fma(x[i], uj, y[i] * vj);
      *e = (beta == 1.0) ? *e + upd : fma(beta, *e, upd);
    }
  }
}

// z = T x (O(k)), then y[r] = beta y[r] + alpha sum_j A[tail_from + r, j] z_j
__global__ void skew_tridiag_gemv_kernel(double* __restrict__ y, double alpha, const double* __restrict__ A,
                                         long long lda, int p, int k, const double* __restrict__ tau,
                                         const double* __restrict__ x, double beta, int tail_from) {
  extern __shared__ double z[];
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    double v = 0.0;
    if (j >= 1) v = tau[j - 1] * x[j - 1];
    if (j + 1 < k) v -= tau[j] * x[j + 1];
    z[j] = v;
  }
  __syncthreads();
  const int rows = p - tail_from;
  for (int rr = blockIdx.x * blockDim.x + threadIdx.x; rr < rows; rr += gridDim.x * blockDim.x) {
    const double* ar = A + tail_from + rr;
    double acc = 0.0;
    for (int j = 0; j < k; ++j) acc = fma(ar[(long long)j * lda], z[j], acc);
    y[rr] = (beta == 1.0) ? y[rr] + alpha * acc : beta * y[rr] + alpha * acc;
  }
}

// tmp[c][r] = block[idx[lo + r], c]; then block[lo + r, c] = tmp[c][r]
__global__ void gather_rows_a(const double* __restrict__ block, long long ld, int q, int lo, int hi,
                              const long long* __restrict__ idx, double* __restrict__ tmp) {
  const int h = hi - lo;
  for (int c = blockIdx.y; c < q; c += gridDim.y)
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < h; r += gridDim.x * blockDim.x)
      tmp[(size_t)c * h + r] = block[(long long)c * ld + idx[lo + r]];
}
__global__ void gather_rows_b(double* __restrict__ block, long long ld, int q, int lo, int hi,
                              const double* __restrict__ tmp) {
  const int h = hi - lo;
  for (int c = blockIdx.y; c < q; c += gridDim.y)
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < h; r += gridDim.x * blockDim.x)
      block[(long long)c * ld + lo + r] = tmp[(size_t)c * h + r];
}

// one symmetric interchange (a < b) of a lower-stored skew matrix
__global__ void sym_swap_kernel(double* __restrict__ X, long long ld, int n, int a, int b) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  // rows a and b left of column a
  for (int c = t; c < a; c += stride) {
    double u = X[(long long)c * ld + a], v = X[(long long)c * ld + b];
    X[(long long)c * ld + a] = v;
    X[(long long)c * ld + b] = u;
  }
  // columns a and b below row b
  for (int i = b + 1 + t; i < n; i += stride) {
    double u = X[(long long)a * ld + i], v = X[(long long)b * ld + i];
    X[(long long)a * ld + i] = v;
    X[(long long)b * ld + i] = u;
  }
  // crossing segment: (i, a) <-> -(b, i), a < i < b
  for (int i = a + 1 + t; i < b; i += stride) {
    double u = X[(long long)a * ld + i], v = X[(long long)i * ld + b];
    X[(long long)a * ld + i] = -v;
    X[(long long)i * ld + b] = -u;
  }
  if (t == 0) X[(long long)a * ld + b] = -X[(long long)a * ld + b];
}

template <typename T>
__global__ void scale_lower_kernel(T* __restrict__ C, long long ldc, int n, T beta) {
  for (int j = blockIdx.y; j < n; j += gridDim.y)
    for (int i = j + 1 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
      C[(long long)j * ldc + i] = beta == T(0) ? T(0) : beta * C[(long long)j * ldc + i];
}

inline dim3 col_grid(int rows, int cols) {
  int gx = (rows + 255) / 256;
  gx = gx < 1 ? 1 : (gx > 8 ? 8 : gx);
  int gy = cols < 1 ? 1 : (cols > 8192 ? 8192 : cols);
  return dim3(gx, gy);
}

// packed factor layout (core.py:349-362): X[j+1, j] = tau[j], X[j+2:, j] = L[j+2:, j]
__global__ void pack_factor_kernel(int n, const double* __restrict__ L, long long ldl, const double* __restrict__ tau,
                                   double* __restrict__ X, long long ldx) {
  const int j = blockIdx.y;
  for (int i = j + 1 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    X[(long long)j * ldx + i] = i == j + 1 ? tau[j] : L[(long long)j * ldl + i];
}

// exact inverse (core.py:365-375): tau[j] = X[j+1, j]; "ones" L buffer with zeros elsewhere
__global__ void unpack_factor_kernel(int n, const double* __restrict__ X, long long ldx, double* __restrict__ L,
                                     long long ldl, double* __restrict__ tau) {
  const int j = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double v = 0.0;
    if (j < n - 1) {
      if (i == j + 1) {
        v = 1.0;
        tau[j] = X[(long long)j * ldx + i];
      } else if (i > j + 1) {
        v = X[(long long)j * ldx + i];
      }
    }
    L[(long long)j * ldl + i] = v;
  }
}

}  // namespace

cudaError_t launch_pack_factor(int n, const double* L, long long ldl, const double* tau, double* X, long long ldx,
                               cudaStream_t stream) {
  if (n < 2) return cudaSuccess;
  pack_factor_kernel<<<dim3((n + 255) / 256, n - 1), 256, 0, stream>>>(n, L, ldl, tau, X, ldx);
  return cudaGetLastError();
}

cudaError_t launch_unpack_factor(int n, const double* X, long long ldx, double* L, long long ldl, double* tau,
                                 cudaStream_t stream) {
  unpack_factor_kernel<<<dim3((n + 255) / 256, n), 256, 0, stream>>>(n, X, ldx, L, ldl, tau);
  return cudaGetLastError();
}

cudaError_t launch_skew_rank2(double* A, long long lda, int n, double alpha, const double* x, const double* y,
                              double beta, cudaStream_t stream) {
  if (n <= 1) return cudaSuccess;
  skew_rank2_kernel<<<col_grid(n, n), 256, 0, stream>>>(A, lda, n, alpha, x, y, beta);
  return cudaGetLastError();
}

cudaError_t launch_gen_rank2(double* A, long long lda, int p, int q, double alpha, const double* x,
                            const double* u, const double* y, const double* v, double beta, cudaStream_t stream) {
  if (p <= 0 || q <= 0) return cudaSuccess;
  gen_rank2_kernel<<<col_grid(p, q), 256, 0, stream>>>(A, lda, p, q, alpha, x, u, y, v, beta);
  return cudaGetLastError();
}

cudaError_t launch_skew_tridiag_gemv(double* y, double alpha, const double* A, long long lda, int p, int k,
                                     const double* tau, const double* x, double beta, int tail_from,
                                     cudaStream_t stream) {
  int rows = p - tail_from;
  if (rows <= 0) return cudaSuccess;
  int grid = (rows + 255) / 256;
  if (grid > 1184) grid = 1184;
  const size_t zbytes = sizeof(double) * (k > 0 ? k : 1);  // z = T x staged in shared memory
  if (zbytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(skew_tridiag_gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)zbytes);
    if (e != cudaSuccess) return e;  // k beyond the shared-memory budget (~29K columns)
  }
  skew_tridiag_gemv_kernel<<<grid, 256, zbytes, stream>>>(y, alpha, A, lda, p, k, tau, x, beta, tail_from);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(double* block, long long ld, int q, int lo, int hi, const long long* idx_dev,
                               double* tmp, cudaStream_t stream) {
  if (hi <= lo || q <= 0) return cudaSuccess;
  gather_rows_a<<<col_grid(hi - lo, q), 256, 0, stream>>>(block, ld, q, lo, hi, idx_dev, tmp);
  gather_rows_b<<<col_grid(hi - lo, q), 256, 0, stream>>>(block, ld, q, lo, hi, tmp);
  return cudaGetLastError();
}

cudaError_t launch_sym_swap(double* X, long long ld, int n, int a, int b, cudaStream_t stream) {
  if (a == b) return cudaSuccess;
  if (a > b) {
    int t = a;
    a = b;
    b = t;
  }
  sym_swap_kernel<<<(n + 255) / 256, 256, 0, stream>>>(X, ld, n, a, b);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_scale_lower(T* C, long long ldc, int n, T beta, cudaStream_t stream) {
  if (n <= 1) return cudaSuccess;
  scale_lower_kernel<T><<<col_grid(n, n), 256, 0, stream>>>(C, ldc, n, beta);
  return cudaGetLastError();
}
template cudaError_t launch_scale_lower<double>(double*, long long, int, double, cudaStream_t);
template cudaError_t launch_scale_lower<float>(float*, long long, int, float, cudaStream_t);

}  // namespace skl
