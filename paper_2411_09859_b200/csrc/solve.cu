// Linear solve X y = b on top of the pivoted factorization (apps.py:76-100,
// SURVEY.md 8f rank 2): permute, unit-lower solve, pivoted skew-tridiagonal
// solve (apps.py:33-73), transposed unit-lower solve, permute back.
//
// L is read in the reference's "ones" work-buffer layout: L[i, j] =
// buf[i, j-1] for i > j >= 1, L[:, 0] = e_0 (core.py:172-220).  The
// triangular solves are blocked: a one-CTA-per-right-hand-side solve of the
// 64x64 diagonal block, then a grid-wide update of the remaining rows (one
// thread per row going down, one warp per row going up so that the column
// reads of L stay coalesced).  The tridiagonal elimination is factored once by
// a single thread in the reference's operation order (no FMA contraction),
// then applied to every right-hand side in parallel (back substitution by the
// reciprocal pivots).
#include <cooperative_groups.h>
#include <cfloat>
#include <map>
#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace skl {
namespace {

constexpr int kSolveBlk = 64;

__device__ __forceinline__ double l_at(const double* __restrict__ L, long long ld, int i, int j) {
  return j >= 1 ? L[(long long)(j - 1) * ld + i] : 0.0;  // i > j
}

// perm[i] with (P x)[i] = x[perm[i]] (core.py:274-285): the swap chain runs in
// shared memory (one thread; n ints of dynamic shared memory, or perm itself in
// global memory when n does not fit), the offsets are staged in chunks and the
// result is written out coalesced
constexpr int kPermChunk = 2048;
__global__ void compose_perm_kernel(int n, const long long* __restrict__ piv, int* __restrict__ perm, int in_smem) {
  extern __shared__ int sp_dyn[];
  __shared__ int soff[kPermChunk];
  int* sp = in_smem ? sp_dyn : perm;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sp[i] = i;
  __syncthreads();
  for (int k0 = 0; k0 < n; k0 += kPermChunk) {
    const int k1 = min(n, k0 + kPermChunk);
    for (int t = threadIdx.x; t < k1 - k0; t += blockDim.x) soff[t] = int(piv[k0 + t]);
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = k0; k < k1; ++k) {
        const int off = soff[k - k0];
        if (off) {
          const int j = k + off;
          const int t = sp[k];
          sp[k] = sp[j];
          sp[j] = t;
        }
      }
    }
    __syncthreads();
  }
  if (in_smem)
    for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = sp[i];
}

// dst = src[perm] (gather) or dst[perm] = src (scatter), column-major n x nrhs
__global__ void permute_rows_kernel(int n, int nrhs, const double* __restrict__ src, long long lds,
                                    double* __restrict__ dst, long long ldd, const int* __restrict__ perm,
                                    int scatter) {
  const long long total = (long long)n * nrhs;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int c = int(e / n), i = int(e - (long long)c * n);
    if (scatter)
      dst[(long long)c * ldd + perm[i]] = src[(long long)c * lds + i];
    else
      dst[(long long)c * ldd + i] = src[(long long)c * lds + perm[i]];
  }
}

// in-place solve of the diagonal block [j0, j1) for right-hand side blockIdx.x;
// the block of L is staged in shared memory first (one coalesced pass)
template <bool TRANS>
__global__ void trsm_diag_kernel(int n, const double* __restrict__ L, long long ld, double* __restrict__ Z,
                                 long long ldz, int j0, int j1) {
  __shared__ double lb[kSolveBlk][kSolveBlk + 1];  // lb[col][row] = L[j0+row, j0+col]
  __shared__ double zb[kSolveBlk];
  double* z = Z + (long long)blockIdx.x * ldz;
  const int w = j1 - j0;
  // column cc of the block (rows j0..j1) is L buffer column j0+cc-1; a warp per column
  for (int cc = threadIdx.x >> 5; cc < w; cc += blockDim.x >> 5) {
    const int lane = threadIdx.x & 31;
    const double* col = j0 + cc >= 1 ? L + (long long)(j0 + cc - 1) * ld + j0 : nullptr;
    const double v0 = (col && lane > cc && lane < w) ? col[lane] : 0.0;
    const double v1 = (col && lane + 32 > cc && lane + 32 < w) ? col[lane + 32] : 0.0;
    lb[cc][lane] = v0;
    if (lane + 32 < kSolveBlk) lb[cc][lane + 32] = v1;
  }
  for (int t = threadIdx.x; t < w; t += blockDim.x) zb[t] = z[j0 + t];
  __syncthreads();
  if (!TRANS) {
    for (int jj = 0; jj < w; ++jj) {
      const double y = zb[jj];
      for (int t = jj + 1 + threadIdx.x; t < w; t += blockDim.x) zb[t] -= lb[jj][t] * y;
      __syncthreads();
    }
  } else {
    for (int jj = w - 1; jj >= 0; --jj) {
      const double y = zb[jj];
      for (int t = threadIdx.x; t < jj; t += blockDim.x) zb[t] -= lb[t][jj] * y;
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < w; t += blockDim.x) z[j0 + t] = zb[t];
}

// rows below the block: z[i] -= sum_{j in [j0,j1)} L[i, j] z[j]   (thread per row,
// loads of the 64 L entries unrolled so they are in flight together)
__global__ void trsm_update_down_kernel(int n, int nrhs, const double* __restrict__ L, long long ld,
                                        double* __restrict__ Z, long long ldz, int j0, int j1) {
  __shared__ double zb[kSolveBlk];
  const int c = blockIdx.y;
  double* z = Z + (long long)c * ldz;
  const int w = j1 - j0;
  for (int t = threadIdx.x; t < w; t += blockDim.x) zb[t] = z[j0 + t];
  __syncthreads();
  for (int i = j1 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int t = 0;
    if (w == kSolveBlk) {
#pragma unroll 16
      for (; t < kSolveBlk; t += 4) {
        a0 = fma(l_at(L, ld, i, j0 + t), zb[t], a0);
        a1 = fma(l_at(L, ld, i, j0 + t + 1), zb[t + 1], a1);
        a2 = fma(l_at(L, ld, i, j0 + t + 2), zb[t + 2], a2);
        a3 = fma(l_at(L, ld, i, j0 + t + 3), zb[t + 3], a3);
      }
    }
    for (; t < w; ++t) a0 = fma(l_at(L, ld, i, j0 + t), zb[t], a0);
    z[i] -= (a0 + a1) + (a2 + a3);
  }
}

// rows above the block: z[i] -= sum_{m in [j0,j1)} L[m, i] z[m]   (warp per row)
__global__ void trsm_update_up_kernel(int n, int nrhs, const double* __restrict__ L, long long ld,
                                      double* __restrict__ Z, long long ldz, int j0, int j1) {
  __shared__ double zb[kSolveBlk];
  const int c = blockIdx.y;
  double* z = Z + (long long)c * ldz;
  const int w = j1 - j0;
  for (int t = threadIdx.x; t < w; t += blockDim.x) zb[t] = z[j0 + t];
  __syncthreads();
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < j0; i += gridDim.x * wpb) {
    double acc = 0.0;
    if (i >= 1) {
      const double* col = L + (long long)(i - 1) * ld + j0;
      const double v0 = lane < w ? col[lane] : 0.0;
      const double v1 = lane + 32 < w ? col[lane + 32] : 0.0;
      acc = fma(v0, lane < w ? zb[lane] : 0.0, v1 * (lane + 32 < w ? zb[lane + 32] : 0.0));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) z[i] -= acc;
  }
}

// One launch per 64-column block (instead of a diagonal launch + an update launch):
// every CTA stages and solves the diagonal block of its right-hand side itself (the
// same arithmetic as trsm_diag_kernel, so all CTAs hold the same solution), CTA 0
// writes the solved block to the OTHER buffer (zout: nobody in this launch reads it),
// and the CTA updates its share of the remaining rows of zin from shared memory (as
// trsm_update_*).  Forward: Z -> B (B is free scratch between the gather and the final
// scatter); backward: B -> Z.  Bit-identical to the two-launch scheme.
template <bool TRANS>
__global__ void __launch_bounds__(256) trsm_fused_kernel(int n, const double* __restrict__ L, long long ld,
                                                         double* __restrict__ zin_all, long long ldi,
                                                         double* __restrict__ zout_all, long long ldo, int j0,
                                                         int j1) {
  __shared__ double lb[kSolveBlk][kSolveBlk + 1];  // lb[col][row] = L[j0+row, j0+col]
  __shared__ double zb[kSolveBlk];
  const int c = blockIdx.y;
  double* zin = zin_all + (long long)c * ldi;
  double* zout = zout_all + (long long)c * ldo;
  const int w = j1 - j0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int cc = warp; cc < w; cc += nw) {
    const double* col = j0 + cc >= 1 ? L + (long long)(j0 + cc - 1) * ld + j0 : nullptr;
    const double v0 = (col && lane > cc && lane < w) ? col[lane] : 0.0;
    const double v1 = (col && lane + 32 > cc && lane + 32 < w) ? col[lane + 32] : 0.0;
    lb[cc][lane] = v0;
    lb[cc][lane + 32] = v1;
  }
  for (int t = threadIdx.x; t < w; t += blockDim.x) zb[t] = zin[j0 + t];
  __syncthreads();
  if (!TRANS) {
    for (int jj = 0; jj < w; ++jj) {
      const double y = zb[jj];
      for (int t = jj + 1 + threadIdx.x; t < w; t += blockDim.x) zb[t] -= lb[jj][t] * y;
      __syncthreads();
    }
  } else {
    for (int jj = w - 1; jj >= 0; --jj) {
      const double y = zb[jj];
      for (int t = threadIdx.x; t < jj; t += blockDim.x) zb[t] -= lb[t][jj] * y;
      __syncthreads();
    }
  }
  if (blockIdx.x == 0)
    for (int t = threadIdx.x; t < w; t += blockDim.x) zout[j0 + t] = zb[t];
  if (!TRANS) {
    // rows below the block, thread per row
    for (int i = j1 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int t = 0;
      if (w == kSolveBlk) {
#pragma unroll 16
        for (; t < kSolveBlk; t += 4) {
          a0 = fma(l_at(L, ld, i, j0 + t), zb[t], a0);
          a1 = fma(l_at(L, ld, i, j0 + t + 1), zb[t + 1], a1);
          a2 = fma(l_at(L, ld, i, j0 + t + 2), zb[t + 2], a2);
          a3 = fma(l_at(L, ld, i, j0 + t + 3), zb[t + 3], a3);
        }
      }
      for (; t < w; ++t) a0 = fma(l_at(L, ld, i, j0 + t), zb[t], a0);
      zin[i] -= (a0 + a1) + (a2 + a3);
    }
  } else {
    // rows above the block, warp per row
    for (int i = blockIdx.x * nw + warp; i < j0; i += gridDim.x * nw) {
      double acc = 0.0;
      if (i >= 1) {
        const double* col = L + (long long)(i - 1) * ld + j0;
        const double v0 = lane < w ? col[lane] : 0.0;
        const double v1 = lane + 32 < w ? col[lane + 32] : 0.0;
        acc = fma(v0, lane < w ? zb[lane] : 0.0, v1 * (lane + 32 < w ? zb[lane + 32] : 0.0));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) zin[i] -= acc;
    }
  }
}

// The whole triangular sweep of 1-2 right-hand sides as ONE cooperative kernel: the loop over
// the 64-column blocks of trsm_fused_kernel with a grid barrier between blocks instead of a
// launch per block (n = 4096: 64 + 64 launches of 12-18 us each).  Per block every CTA stages
// the diagonal block, warp 0 solves it with register shuffles (two entries per lane, the same
// operations in the same order as the barrier-per-step loop of trsm_fused_kernel), CTA 0
// writes the solved block to the other buffer and every CTA updates its share of the
// remaining rows of zin.  A block's solve reads rows the previous block's updates wrote,
// hence the barrier; the solved block itself is never read again.  Bit-identical results.
template <bool TRANS>
__global__ void __launch_bounds__(256) trsm_sweep_kernel(int n, const double* __restrict__ L, long long ld,
                                                         double* __restrict__ zin_all, long long ldi,
                                                         double* __restrict__ zout_all, long long ldo) {
  // lbuf[2][col][row] = L[j0+row, j0+col] of the current and the NEXT block (L is constant: the
  // next diagonal block is staged while this block's rows are updated, off the critical path)
  extern __shared__ __align__(16) unsigned char sweep_smem[];
  typedef double LB[kSolveBlk][kSolveBlk + 1];
  LB* lbuf = reinterpret_cast<LB*>(sweep_smem);
  double* zb = reinterpret_cast<double*>(lbuf + 2);
  static_assert(kSolveBlk == 64, "two entries per lane");
  const int c = blockIdx.y;
  double* zin = zin_all + (long long)c * ldi;
  double* zout = zout_all + (long long)c * ldo;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nblk = (n + kSolveBlk - 1) / kSolveBlk;
  // the strictly-lower part of diagonal block bi: 16 entries per thread, loaded in one go
  // (stage_load) and stored to shared memory later (stage_store), so the loads of the next
  // block fly while this block's rows are updated
  constexpr int kPerThread = kSolveBlk * kSolveBlk / 256;
  double sv[kPerThread];
  auto stage_load = [&](int bi) {
    const int j0 = bi * kSolveBlk, w = min(n, j0 + kSolveBlk) - j0;
#pragma unroll
    for (int e = 0; e < kPerThread; ++e) {
      const int idx = threadIdx.x + e * 256, cc = idx >> 6, rr = idx & 63;
      sv[e] = (cc < w && rr > cc && rr < w && j0 + cc >= 1) ? L[(long long)(j0 + cc - 1) * ld + j0 + rr] : 0.0;
    }
  };
  auto stage_store = [&](LB& lb) {
#pragma unroll
    for (int e = 0; e < kPerThread; ++e) {
      const int idx = threadIdx.x + e * 256;
      lb[idx >> 6][idx & 63] = sv[e];
    }
  };
  stage_load(TRANS ? nblk - 1 : 0);
  stage_store(lbuf[0]);
  for (int bi0 = 0; bi0 < nblk; ++bi0) {
    const int bi = TRANS ? nblk - 1 - bi0 : bi0;
    const int j0 = bi * kSolveBlk, j1 = min(n, j0 + kSolveBlk);
    const int w = j1 - j0;
    LB& lb = lbuf[bi0 & 1];
    for (int t = threadIdx.x; t < w; t += blockDim.x) zb[t] = __ldcg(zin + j0 + t);
    // the L entries of this CTA's first pass over the rows to update do not depend on the
    // block's solution: load them now, so their latency hides behind warp 0's serial solve
    double lv[16];
    const int q = threadIdx.x & 3;
    const int ipre = TRANS ? blockIdx.x * nw + warp : j1 + blockIdx.x * 64 + (threadIdx.x >> 2);
    if (!TRANS) {
      if (w == kSolveBlk && ipre < n) {
#pragma unroll
        for (int e = 0; e < 16; ++e) lv[e] = l_at(L, ld, ipre, j0 + q + 4 * e);
      }
    } else {
      lv[0] = lv[1] = 0.0;
      if (ipre >= 1 && ipre < j0) {
        const double* col = L + (long long)(ipre - 1) * ld + j0;
        lv[0] = lane < w ? col[lane] : 0.0;
        lv[1] = lane + 32 < w ? col[lane + 32] : 0.0;
      }
    }
    __syncthreads();
    if (warp == 0) {
      double z0 = lane < w ? zb[lane] : 0.0, z1 = lane + 32 < w ? zb[lane + 32] : 0.0;
      if (!TRANS) {
        for (int jj = 0; jj < w; ++jj) {
          const double y = jj < 32 ? __shfl_sync(0xffffffffu, z0, jj) : __shfl_sync(0xffffffffu, z1, jj - 32);
          if (lane > jj) z0 -= lb[jj][lane] * y;
          if (lane + 32 > jj && lane + 32 < w) z1 -= lb[jj][lane + 32] * y;
        }
      } else {
        for (int jj = w - 1; jj >= 0; --jj) {
          const double y = jj < 32 ? __shfl_sync(0xffffffffu, z0, jj) : __shfl_sync(0xffffffffu, z1, jj - 32);
          if (lane < jj) z0 -= lb[lane][jj] * y;
          if (lane + 32 < jj) z1 -= lb[lane + 32][jj] * y;
        }
      }
      if (lane < w) zb[lane] = z0;
      if (lane + 32 < w) zb[lane + 32] = z1;
    }
    __syncthreads();
    if (bi0 + 1 < nblk) stage_load(TRANS ? bi - 1 : bi + 1);
    if (blockIdx.x == 0)
      for (int t = threadIdx.x; t < w; t += blockDim.x) zout[j0 + t] = zb[t];
    if (!TRANS) {
      // rows below the block: four consecutive lanes per row, lane q takes the columns
      // t = q (mod 4) -- the four accumulation chains of the thread-per-row update, one per
      // lane, all 16 loads of a lane in flight at once -- combined as (a0 + a1) + (a2 + a3)
      for (int i0 = j1 + blockIdx.x * 64; i0 < n; i0 += gridDim.x * 64) {
        const int i = i0 + (threadIdx.x >> 2);
        double a = 0.0;
        if (i < n) {
          if (w == kSolveBlk) {
            if (i != ipre) {
#pragma unroll
              for (int e = 0; e < 16; ++e) lv[e] = l_at(L, ld, i, j0 + q + 4 * e);
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) a = fma(lv[e], zb[q + 4 * e], a);
          } else {
            // a partial last block keeps the thread-per-row order: chain 0 takes every column
            if (q == 0)
              for (int t = 0; t < w; ++t) a = fma(l_at(L, ld, i, j0 + t), zb[t], a);
          }
        }
        a += __shfl_xor_sync(0xffffffffu, a, 1);
        a += __shfl_xor_sync(0xffffffffu, a, 2);
        if (q == 0 && i < n) zin[i] = __ldcg(zin + i) - a;
      }
    } else {
      for (int i = blockIdx.x * nw + warp; i < j0; i += gridDim.x * nw) {
        double acc = 0.0;
        if (i >= 1) {
          double v0 = lv[0], v1 = lv[1];
          if (i != ipre) {
            const double* col = L + (long long)(i - 1) * ld + j0;
            v0 = lane < w ? col[lane] : 0.0;
            v1 = lane + 32 < w ? col[lane + 32] : 0.0;
          }
          acc = fma(v0, lane < w ? zb[lane] : 0.0, v1 * (lane + 32 < w ? zb[lane + 32] : 0.0));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) zin[i] = __ldcg(zin + i) - acc;
      }
    }
    if (bi0 + 1 < nblk) stage_store(lbuf[(bi0 + 1) & 1]);
    __threadfence();
    cooperative_groups::this_grid().sync();
  }
}

constexpr int kChunk = 512;  // steps staged in shared memory per round

// factor T (subdiagonal tau) by Gaussian elimination with partial pivoting, one
// superdiagonal of fill (apps.py:33-73).  The recurrence is sequential: thread
// 0 runs it in the reference's operation order with the two live rows in
// registers, while the block stages tau chunks into shared memory and streams
// the per-step outputs (d, e, f2, multiplier, swap flag) back out coalesced.
__global__ void tridiag_factor_kernel(int m, const double* __restrict__ tau, double tol_scale, double* d, double* e,
                                      double* f2, double* mult, int* swp, int* info) {
  __shared__ double st[kChunk + 1];
  __shared__ double so[4][kChunk];
  __shared__ int ss[kChunk];
  __shared__ double red[32];
  __shared__ int stop;
  const int tid = threadIdx.x;
  double big = 0.0;
  for (int k = tid; k < m - 1; k += blockDim.x) big = fmax(big, fabs(tau[k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) big = fmax(big, __shfl_xor_sync(0xffffffffu, big, o));
  if ((tid & 31) == 0) red[tid >> 5] = big;
  if (tid == 0) stop = 0;
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < int(blockDim.x >> 5); ++w) big = fmax(big, red[w]);
    red[0] = big;
  }
  __syncthreads();
  const double thresh = __dmul_rn(__dmul_rn(tol_scale, DBL_EPSILON), red[0]);
  double dk = 0.0, ek = m > 1 ? -tau[0] : 0.0;  // thread 0's live state
  for (int k0 = 0; k0 < m - 1; k0 += kChunk) {
    const int k1 = min(m - 1, k0 + kChunk);
    for (int t = tid; t <= k1 - k0; t += blockDim.x) st[t] = (k0 + t < m - 1) ? tau[k0 + t] : 0.0;
    __syncthreads();
    if (tid == 0) {
      for (int k = k0; k < k1; ++k) {
        double sub = st[k - k0];
        double dk1 = 0.0, ek1 = k + 1 < m - 1 ? -st[k + 1 - k0] : 0.0, f2k = 0.0;
        int sw = 0;
        if (fabs(sub) > fabs(dk)) {
          double t = dk;
          dk = sub;
          sub = t;
          t = ek;
          ek = dk1;
          dk1 = t;
          if (k + 2 < m) {
            t = f2k;
            f2k = ek1;
            ek1 = t;
          }
          sw = 1;
        }
        if (fabs(dk) <= thresh) {
          *info = k + 1;
          stop = 1;
          break;
        }
        const double mu = __dmul_rn(sub, __drcp_rn(dk));  // short dependent chain (tolerance-level vs /)
        dk1 = __dsub_rn(dk1, __dmul_rn(mu, ek));
        if (k + 2 < m) ek1 = __dsub_rn(ek1, __dmul_rn(mu, f2k));
        so[0][k - k0] = dk;
        so[1][k - k0] = ek;
        so[2][k - k0] = f2k;
        so[3][k - k0] = mu;
        ss[k - k0] = sw;
        dk = dk1;
        ek = ek1;
      }
    }
    __syncthreads();
    if (stop) return;
    for (int t = tid; t < k1 - k0; t += blockDim.x) {
      d[k0 + t] = so[0][t];
      e[k0 + t] = so[1][t];
      f2[k0 + t] = so[2][t];
      mult[k0 + t] = so[3][t];
      swp[k0 + t] = ss[t];
    }
    __syncthreads();
  }
  if (tid == 0) {
    d[m - 1] = dk;
    e[m - 1] = ek;
    f2[m - 1] = 0.0;
    if (fabs(dk) <= thresh) *info = m;
  }
}

// d[k] := 1 / d[k] for the back substitution (multiplications instead of one
// division per step on the right-hand sides' dependent chain)
__global__ void tridiag_recip_kernel(int m, double* d, const int* __restrict__ info) {
  if (*info != 0) return;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) d[k] = 1.0 / d[k];
}

// apply the factored T to right-hand side blockIdx.x: chunks of the column and
// of the factor are staged in shared memory, thread 0 runs the recurrences
__global__ void tridiag_apply_kernel(int m, int nrhs, const double* __restrict__ d, const double* __restrict__ e,
                                     const double* __restrict__ f2, const double* __restrict__ mult,
                                     const int* __restrict__ swp, const int* __restrict__ info,
                                     double* __restrict__ Z, long long ldz) {
  __shared__ double xs[kChunk + 2];
  __shared__ double a0[kChunk], a1[kChunk], a2[kChunk];
  __shared__ int sw[kChunk];
  if (*info != 0) return;
  const int tid = threadIdx.x;
  double* x = Z + (long long)blockIdx.x * ldz;
  // forward: x[k+1] -= mult[k] x[k] after the optional row swap (k, k+1)
  double xk = x[0];
  for (int k0 = 0; k0 < m - 1; k0 += kChunk) {
    const int k1 = min(m - 1, k0 + kChunk);
    for (int t = tid; t < k1 - k0; t += blockDim.x) {
      xs[t] = x[k0 + 1 + t];
      a0[t] = mult[k0 + t];
      sw[t] = swp[k0 + t];
    }
    __syncthreads();
    if (tid == 0) {
      for (int k = k0; k < k1; ++k) {
        double xk1 = xs[k - k0];
        if (sw[k - k0]) {
          const double t = xk;
          xk = xk1;
          xk1 = t;
        }
        xk1 = __dsub_rn(xk1, __dmul_rn(a0[k - k0], xk));
        xs[k - k0] = xk;  // final x[k] (slot of x[k+1] reused: x[k] goes out below)
        xk = xk1;
      }
    }
    __syncthreads();
    for (int t = tid; t < k1 - k0; t += blockDim.x) x[k0 + t] = xs[t];
    __syncthreads();
  }
  if (tid == 0) x[m - 1] = xk;
  __syncthreads();
  // back substitution with one extra superdiagonal (d holds 1/d)
  double xp1 = 0.0, xp2 = 0.0;  // x[k+1], x[k+2] (thread 0)
  for (int k1 = m; k1 > 0; k1 -= kChunk) {
    const int k0 = max(0, k1 - kChunk);
    for (int t = tid; t < k1 - k0; t += blockDim.x) {
      xs[t] = x[k0 + t];
      a0[t] = d[k0 + t];
      a1[t] = e[k0 + t];
      a2[t] = f2[k0 + t];
    }
    __syncthreads();
    if (tid == 0) {
      for (int k = k1 - 1; k >= k0; --k) {
        double v;
        if (k == m - 1)
          v = xs[k - k0] * a0[k - k0];
        else if (k == m - 2)
          v = __dsub_rn(xs[k - k0], __dmul_rn(a1[k - k0], xp1)) * a0[k - k0];
        else
          v = __dsub_rn(__dsub_rn(xs[k - k0], __dmul_rn(a1[k - k0], xp1)), __dmul_rn(a2[k - k0], xp2)) * a0[k - k0];
        xs[k - k0] = v;
        xp2 = xp1;
        xp1 = v;
      }
    }
    __syncthreads();
    for (int t = tid; t < k1 - k0; t += blockDim.x) x[k0 + t] = xs[t];
    __syncthreads();
  }
}

}  // namespace

size_t solve_workspace_bytes(int n, int nrhs) {
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  return al(sizeof(int) * n) + al(sizeof(double) * (size_t)n * nrhs) + 4 * al(sizeof(double) * n) +
         al(sizeof(int) * n);
}

namespace {
// per-device side stream for the overlapped tridiagonal factorization
cudaError_t side_stream_for(cudaStream_t stream, cudaStream_t* out) {
  static std::mutex mu;
  static std::map<int, cudaStream_t> sides;
  int dev = 0;
  cudaError_t err = cudaStreamGetDevice(stream, &dev);
  if (err != cudaSuccess) return err;
  std::lock_guard<std::mutex> lk(mu);
  auto it = sides.find(dev);
  if (it != sides.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  int cur = 0;
  if ((err = cudaGetDevice(&cur)) != cudaSuccess) return err;
  if (cur != dev && (err = cudaSetDevice(dev)) != cudaSuccess) return err;
  cudaStream_t s = nullptr;
  err = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (cur != dev) cudaSetDevice(cur);
  if (err != cudaSuccess) return err;
  sides[dev] = s;
  *out = s;
  return cudaSuccess;
}

// fork/join events owned by one call; destroyed when the call returns (CUDA
// releases them once the recorded work has completed)
struct EventPair {
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaError_t create() {
    cudaError_t e = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
    return e;
  }
  ~EventPair() {
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
  }
};

}  // namespace

cudaError_t launch_solve(int n, int nrhs, const double* L, long long ldl, const double* tau, const long long* piv,
                         double* B, long long ldb, double tol_scale, int* info, void* ws, cudaStream_t stream) {
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  unsigned char* p = static_cast<unsigned char*>(ws);
  int* perm = reinterpret_cast<int*>(p);
  p += al(sizeof(int) * n);
  double* Z = reinterpret_cast<double*>(p);
  p += al(sizeof(double) * (size_t)n * nrhs);
  double* d = reinterpret_cast<double*>(p);
  p += al(sizeof(double) * n);
  double* e = reinterpret_cast<double*>(p);
  p += al(sizeof(double) * n);
  double* f2 = reinterpret_cast<double*>(p);
  p += al(sizeof(double) * n);
  double* mult = reinterpret_cast<double*>(p);
  p += al(sizeof(double) * n);
  int* swp = reinterpret_cast<int*>(p);
  const long long ldz = n;
  cudaError_t err = cudaMemsetAsync(info, 0, sizeof(int), stream);
  if (err != cudaSuccess) return err;
  {
    // the swap chain in shared memory when n ints fit next to the static chunk buffer
    static int optin = 0;
    if (optin == 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || optin <= 0)
        optin = 48 * 1024;
      optin -= int(sizeof(int)) * kPermChunk + 1024;
    }
    const size_t pbytes = sizeof(int) * (size_t)n;
    const int in_smem = pbytes <= (size_t)optin ? 1 : 0;
    if (in_smem && pbytes > 48 * 1024) {
      err = cudaFuncSetAttribute(compose_perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pbytes);
      if (err != cudaSuccess) return err;
    }
    compose_perm_kernel<<<1, 256, in_smem ? pbytes : 0, stream>>>(n, piv, perm, in_smem);
  }
  const long long tot = (long long)n * nrhs;
  const int pg = int(std::min<long long>((tot + 255) / 256, 148 * 8));
  permute_rows_kernel<<<pg, 256, 0, stream>>>(n, nrhs, B, ldb, Z, ldz, perm, 0);
  // the tridiagonal factorization depends on tau only: it runs on a side stream,
  // overlapped with the permutation and the forward sweep (one thread's sequential
  // recurrence, ~0.6 ms at n = 4096, would otherwise sit on the critical path)
  // one side stream per device (the caller's stream's device, not the current one);
  // the fork/join events are per call, so concurrent calls never wait on each other's
  cudaStream_t side = nullptr;
  if ((err = side_stream_for(stream, &side)) != cudaSuccess) return err;
  EventPair evs;
  if ((err = evs.create()) != cudaSuccess) return err;
  cudaEvent_t ev_fork = evs.fork, ev_join = evs.join;
  if ((err = cudaEventRecord(ev_fork, stream)) != cudaSuccess) return err;  // info zeroed, inputs ready
  if ((err = cudaStreamWaitEvent(side, ev_fork, 0)) != cudaSuccess) return err;
  tridiag_factor_kernel<<<1, 256, 0, side>>>(n, tau, tol_scale, d, e, f2, mult, swp, info);
  tridiag_recip_kernel<<<(n + 255) / 256, 256, 0, side>>>(n, d, info);
  if ((err = cudaEventRecord(ev_join, side)) != cudaSuccess) return err;
  // fused launches for one or two right-hand sides (n=4096, 1 rhs: 2.52 -> 2.24 ms); with
  // many the redundant per-CTA diagonal solves and L reads lose (16 rhs: 3.0 -> 5.1 ms)
  static const bool fused_on = [] {
    const char* v = getenv("SKL_SOLVE_FUSED");
    return !(v && *v == '0');
  }();
  const bool fused = fused_on && nrhs <= 2;
  // 1-2 right-hand sides: each triangular sweep as one cooperative kernel (SKL_SOLVE_SWEEP=0: a
  // fused launch per 64-column block)
  static const bool sweep_on = [] {
    const char* v = getenv("SKL_SOLVE_SWEEP");
    return !(v && *v == '0');
  }();
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const bool sweep = fused && sweep_on;
  auto launch_sweep = [&](bool trans, double* zin, long long ldi, double* zout, long long ldo) {
    const int work = trans ? (n + 7) / 8 : (n + 63) / 64;  // warp per row / four lanes per row
    dim3 grid(std::max(1, std::min(work, 2 * nsm / nrhs)), nrhs);
    void* args[] = {&n, &L, &ldl, &zin, &ldi, &zout, &ldo};
    const size_t smem = sizeof(double) * (2 * kSolveBlk * (kSolveBlk + 1) + kSolveBlk);
    void* kern = trans ? (void*)trsm_sweep_kernel<true> : (void*)trsm_sweep_kernel<false>;
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e2 != cudaSuccess) return e2;
    return cudaLaunchCooperativeKernel(kern, grid, dim3(256), args, smem, stream);
  };
  if (sweep && (err = launch_sweep(false, Z, ldz, B, ldb)) != cudaSuccess) return err;
  // L z = P b (forward, blocks of 64 columns); fused: the solved z lands in B
  for (int j0 = 0; j0 < n && !sweep; j0 += kSolveBlk) {
    const int j1 = std::min(n, j0 + kSolveBlk);
    const int rows = n - j1;
    if (fused) {
      dim3 grid(std::max(1, std::min((rows + 255) / 256, 148 * 2)), nrhs);
      trsm_fused_kernel<false><<<grid, 256, 0, stream>>>(n, L, ldl, Z, ldz, B, ldb, j0, j1);
      continue;
    }
    trsm_diag_kernel<false><<<nrhs, 256, 0, stream>>>(n, L, ldl, Z, ldz, j0, j1);
    if (j1 < n) {
      dim3 grid(std::max(1, std::min((rows + 63) / 64, 148 * 8)), nrhs);
      trsm_update_down_kernel<<<grid, 64, 0, stream>>>(n, nrhs, L, ldl, Z, ldz, j0, j1);
    }
  }
  double* Zt = fused ? B : Z;  // the forward solution
  const long long ldt = fused ? ldb : ldz;
  if ((err = cudaStreamWaitEvent(stream, ev_join, 0)) != cudaSuccess) return err;
  tridiag_apply_kernel<<<nrhs, 128, 0, stream>>>(n, nrhs, d, e, f2, mult, swp, info, Zt, ldt);
  // L^T y = z (backward); fused: the solved y lands back in Z
  const int nblk = (n + kSolveBlk - 1) / kSolveBlk;
  if (sweep && (err = launch_sweep(true, B, ldb, Z, ldz)) != cudaSuccess) return err;
  for (int bi = nblk - 1; bi >= 0 && !sweep; --bi) {
    const int j0 = bi * kSolveBlk, j1 = std::min(n, j0 + kSolveBlk);
    if (fused) {
      dim3 grid(std::max(1, std::min((j0 + 7) / 8, 148 * 4)), nrhs);
      trsm_fused_kernel<true><<<grid, 256, 0, stream>>>(n, L, ldl, B, ldb, Z, ldz, j0, j1);
      continue;
    }
    trsm_diag_kernel<true><<<nrhs, 256, 0, stream>>>(n, L, ldl, Z, ldz, j0, j1);
    if (j0 > 0) {
      dim3 grid(std::max(1, std::min((j0 + 7) / 8, 148 * 4)), nrhs);
      trsm_update_up_kernel<<<grid, 256, 0, stream>>>(n, nrhs, L, ldl, Z, ldz, j0, j1);
    }
  }
  permute_rows_kernel<<<pg, 256, 0, stream>>>(n, nrhs, Z, ldz, B, ldb, perm, 1);
  return cudaGetLastError();
}

}  // namespace skl
