// Trailing "sandwiched" update on the FP64 tensor pipe.
//
// The reference realizes C := C - A T A^T (kernels3.py:151-209,
// skew_tridiag_rankk) and C := C + alpha (A B^T - B A^T) (kernels3.py:305-351,
// skew_rank2k) as Goto-blocked NumPy/OpenBLAS tiles with a masked merge on
// diagonal tiles.  Here both are ONE lower-triangular DGEMM-NT
//     C[i,j] = beta*C[i,j] + sum_k P[i,k] Q[j,k]      (i > j only)
// whose operands P, Q are packed by a small kernel that also forms the
// tridiagonal-multiplied operand (B = A T^T, or W = A S for skr2k) on the fly,
// the GPU analogue of the reference's "T rides along with packing"
// (_pack_bt_panel, kernels3.py:134-148).
//
// GEMM kernel: 128x128 C tile per CTA, 8 compute warps in a 2x4 grid of
// 64x32 warp tiles, DMMA.8x8x4 (mma.sync m8n8k4 f64).  Operand k-chunks are
// streamed by the bulk-copy engine (cp.async.bulk -> mbarrier complete_tx)
// through a 4-stage shared-memory ring; the packed layout puts every DMMA
// fragment in lane order so fragment loads are conflict-free 256-byte rows.
// Only lower tiles are launched (triangle-aware schedule); diagonal tiles
// mask i <= j at load and store, so the upper triangle is never read or
// written (test_core.py:39-58 NaN-poison invariant).
#include <algorithm>
#include <cstdlib>
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "internal.h"

namespace skl {

namespace {

#ifndef SKL_GEMM_STAGES
#define SKL_GEMM_STAGES 3
#define SKL_GEMM_K4_PER_STAGE 4
#endif
constexpr int kStages = SKL_GEMM_STAGES;
constexpr int kK4PerStage = SKL_GEMM_K4_PER_STAGE;  // 4*kK4PerStage k per stage
constexpr int kBlkDoubles = 16 * 32;              // one k4 block of a 128-row tile
constexpr int kStageDoubles = kK4PerStage * kBlkDoubles;
constexpr int kGemmThreads = 256;
constexpr int kGemmWarps = kGemmThreads / 32;
// C staging of the tensor-reduce epilogue: per warp, its 64x32 block as four
// 16-row x 32-col boxes (4 KiB each, 128-byte swizzled, 1 KiB aligned) that
// cp.reduce.async.bulk.tensor adds into C through a tensor map.
constexpr int kBoxRows = 16, kBoxCols = 32;
constexpr int kBoxDoubles = kBoxRows * kBoxCols;
constexpr size_t kRingBytes = size_t(kStages) * 2 * kStageDoubles * sizeof(double);
constexpr size_t kCbufBytes = size_t(kGemmWarps) * 4 * kBoxDoubles * sizeof(double);
constexpr size_t kGemmSmem = 1024 + kRingBytes + kCbufBytes + 2 * kStages * sizeof(uint64_t);
static_assert(kGemmSmem <= 232448, "GEMM shared memory exceeds the sm_100 opt-in limit");

__device__ __forceinline__ size_t packed_off(int row, int col, int k4cap) {
  int t = row >> 7, mb = (row >> 3) & 15, r8 = row & 7;
  int q = col >> 2, c4 = col & 3;
  return (((size_t)t * k4cap + q) * 16 + mb) * 32 + (r8 * 4 + c4);
}

// Tile raster: bands of kBand tile-rows; inside a band, columns ascend and rows
// ascend within a column.  The ~148 tiles in flight at once then span ~kBand P
// tiles and ~148/kBand Q tiles, so no packed operand tile is read by every SM
// at the same moment (a plain row-major walk has all SMs on one P tile, which
// hot-spots the L2 slices holding it).
#ifndef SKL_GEMM_BAND
#define SKL_GEMM_BAND 8
#endif
constexpr int kBand = SKL_GEMM_BAND;
__host__ __device__ __forceinline__ void lower_tile_swizzled(int t, int nt, int& ti, int& tj) {
  // full band b holds G^2 b + G(G+1)/2 tiles; cum(b) = G^2 b(b-1)/2 + b G(G+1)/2
  constexpr long long G = kBand;
  auto cum = [](long long b) { return G * G * b * (b - 1) / 2 + b * G * (G + 1) / 2; };
  const float a = 0.5f * G * G, bb = 0.5f * G * (G + 1) - 0.5f * G * G;
  long long b = (long long)((-bb + sqrtf(bb * bb + 4.f * a * (float)t)) / (2.f * a));
  if (b < 0) b = 0;
  while (b > 0 && cum(b) > t) --b;
  while (cum(b + 1) <= t) ++b;
  const int r0 = int(b * G);
  const int h = min(int(G), nt - r0);
  int u = int(t - cum(b));
  if (u < h * r0) {
    tj = u / h;
    ti = r0 + (u - tj * h);
    return;
  }
  u -= h * r0;
  int j = 0;
  while (u >= h - j) {
    u -= h - j;
    ++j;
  }
  tj = r0 + j;
  ti = tj + u;
}

// Tile-table mode (kOwned): tab = [m, total, (tcol, first, partial, row0) x m]
// lists tile columns; column entry c holds the tiles t with first[c] <= t <
// first[c+1], tile column tcol[c] and rows row0[c] + (t - first[c]).  Used by
//  * the block-cyclic multi-GPU driver: the lower tiles (row0 = tcol) of the
//    columns one rank owns; `partial` tiles straddle an owner boundary and take
//    the column-masked register epilogue;
//  * skew_tridiag_gemm: a general p x q block (row0 = 0, tri = 0) or its
//    strictly-lower trapezoid (row0 = tcol, tri = 1).
// The CTA's tiles t = blockIdx.x + i*gridDim.x ascend, so each walker (producer
// and consumers) keeps its own column cursor c and only moves it forward: no
// dependent binary-search loads on the producer's critical path.
__device__ __forceinline__ void owned_tile(const int* __restrict__ tab, int t, int& c, int& ti, int& tj, int& part) {
  const int m = tab[0];
  const int* e = tab + 2;
  while (c + 1 < m && __ldg(e + 4 * (c + 1) + 1) <= t) ++c;
  tj = __ldg(e + 4 * c);
  ti = __ldg(e + 4 * c + 3) + (t - __ldg(e + 4 * c + 1));
  part = __ldg(e + 4 * c + 2);
}

// Persistent lower-triangular DGEMM-NT: one CTA per SM walks the lower tiles
// (ti >= tj) round-robin; the bulk-copy ring runs ahead across tile
// boundaries so the next tile's operands stream in during the epilogue.  The
// C tile is prefetched into L2 when a tile starts and read-modified-written
// in the epilogue (accumulators start at zero).
template <bool kOwned>
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_lower_nt_kernel(const __grid_constant__ CUtensorMap cmap, const __grid_constant__ CUtensorMap pmap, int use_tmap,
                     const double* __restrict__ P,
                     const double* __restrict__ Q, int k4cap, int nk4_host,
                     const int* __restrict__ nk4_dev, double* __restrict__ C, long long ldc, int n, double beta,
                     const int* __restrict__ own_tab, long long own_cbase, int own_nbd, int own_g, int own_rank,
                     int ncols, int tri) {
  // n: C rows; ncols: C columns (== n and tri == 1 except for the tile-table
  // rectangular mode of skew_tridiag_gemm); tri: only row > col is written
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // 1 KiB-align the carve-up (the swizzled boxes need it)
  unsigned char* smem_al = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* sP = reinterpret_cast<double*>(smem_al);
  double* sQ = sP + kStages * kStageDoubles;
  double* cbuf = sQ + kStages * kStageDoubles;
  uint64_t* full = reinterpret_cast<uint64_t*>(cbuf + kGemmWarps * 4 * kBoxDoubles);
  uint64_t* empty = full + kStages;
  // off-diagonal tiles with beta == 1 finish through the bulk engine: accumulators
  // -> swizzled shared boxes -> cp.reduce.async.bulk.tensor .add into C (rows
  // past n clipped by the tensor map), overlapping C's read-modify-write with
  // the next tile's MMAs; diagonal tiles keep the masked register epilogue
  const bool bulk_ok = use_tmap && beta == 1.0;
  const int nt = tiles_for(n);
  const int ntiles = kOwned ? own_tab[1] : nt * (nt + 1) / 2;
  const int nk4 = nk4_dev ? *nk4_dev : nk4_host;
  const int nchunks = (nk4 + kK4PerStage - 1) / kK4PerStage;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int total_chunks = my_tiles * nchunks;
  if (my_tiles == 0 || nchunks == 0) {
    // nothing to multiply: still apply beta to the owned tiles (the column-owned
    // launches always carry K >= 1)
    for (int t = blockIdx.x; t < ntiles && nchunks == 0 && !kOwned; t += gridDim.x) {
      int ti = int((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
      while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
      while (ti * (ti + 1) / 2 > t) --ti;
      const int tj = t - ti * (ti + 1) / 2;
      for (int e = tid; e < kTile * kTile; e += kGemmThreads) {
        int row = ti * kTile + (e & (kTile - 1)), col = tj * kTile + (e >> 7);
        if (row < n && col < n && row > col) {
          double* p = C + (long long)col * ldc + row;
          *p = beta == 0.0 ? 0.0 : beta * *p;
        }
      }
    }
    return;
  }

  int part_dummy, cur_iss = 0, cur_mma = 0;
  auto tile_of = [&](int i, int& ti, int& tj) {
    if constexpr (kOwned) owned_tile(own_tab, blockIdx.x + i * gridDim.x, cur_iss, ti, tj, part_dummy);
    else lower_tile_swizzled(blockIdx.x + i * gridDim.x, nt, ti, tj);
  };
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kGemmWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // global chunk q -> (tile i = q / nchunks, chunk c = q % nchunks)
  // producer state (tid 0): chunks are issued strictly in order, so the tile
  // coordinates are recomputed only when the issue cursor enters a new tile --
  // the per-chunk cost stays a few integer ops on warp 0's critical path
  int iss_q = 0, iss_i = -1, iss_c = 0, iss_ti = 0, iss_tj = 0;
  auto issue = [&](int q) {
    (void)q;  // == iss_q
    if (iss_i < 0 || iss_c == nchunks) {
      ++iss_i;
      iss_c = 0;
      tile_of(iss_i, iss_ti, iss_tj);
    }
    const int s = iss_q % kStages;
    const int q0 = iss_c * kK4PerStage;
    const int nb = min(kK4PerStage, nk4 - q0);
    const uint32_t bytes = uint32_t(nb) * kBlkDoubles * sizeof(double);
    mbar_arrive_expect_tx(&full[s], 2 * bytes);
    bulk_g2s(sP + s * kStageDoubles, P + ((size_t)iss_ti * k4cap + q0) * kBlkDoubles, bytes, &full[s]);
    bulk_g2s(sQ + s * kStageDoubles, Q + ((size_t)iss_tj * k4cap + q0) * kBlkDoubles, bytes, &full[s]);
    ++iss_q;
    ++iss_c;
  };

  if (tid == 0) {
    for (int q = 0; q < min(kStages, total_chunks); ++q) issue(q);
  }

  int q = 0;
  for (int i = 0; i < my_tiles; ++i) {
    int ti, tj, part = 0;
    if constexpr (kOwned) owned_tile(own_tab, blockIdx.x + i * gridDim.x, cur_mma, ti, tj, part);
    else lower_tile_swizzled(blockIdx.x + i * gridDim.x, nt, ti, tj);
    // warm L2 with the NEXT tile's C block (read-modify-written in its
    // epilogue): one 128x128 tensor prefetch issued a whole tile ahead by a
    // thread that is not the operand producer
    if (tid == 32 && use_tmap) {
      if (i == 0) prefetch_l2_tensor_2d(&pmap, ti * kTile, tj * kTile);
      if (i + 1 < my_tiles) {
        int nti, ntj, npart;
        if constexpr (kOwned) {
          int cur_pf = cur_mma;
          owned_tile(own_tab, blockIdx.x + (i + 1) * gridDim.x, cur_pf, nti, ntj, npart);
        } else {
          lower_tile_swizzled(blockIdx.x + (i + 1) * gridDim.x, nt, nti, ntj);
        }
        prefetch_l2_tensor_2d(&pmap, nti * kTile, ntj * kTile);
      }
    } else if (!use_tmap && tid < kTile) {
      const int col = tj * kTile + tid;
      const int r0 = ti * kTile;
      if (col < ncols && r0 < n) {
        const int rows = min(kTile, n - r0);
        const double* src = C + (long long)col * ldc + r0;
        uintptr_t a0 = reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15);
        uintptr_t a1 = (reinterpret_cast<uintptr_t>(src + rows) + 15) & ~uintptr_t(15);
        prefetch_l2_bulk(reinterpret_cast<const void*>(a0), uint32_t(a1 - a0));
      }
    }
    double acc[8][4][2];
#pragma unroll
    for (int mi = 0; mi < 8; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

    for (int c = 0; c < nchunks; ++c, ++q) {
      const int s = q % kStages;
      mbar_wait(&full[s], (q / kStages) & 1);
      const int nb = min(kK4PerStage, nk4 - c * kK4PerStage);
      const double* ps = sP + s * kStageDoubles + (wm * 8) * 32 + lane;
      const double* qs = sQ + s * kStageDoubles + (wn * 4) * 32 + lane;
      for (int kb = 0; kb < nb; ++kb) {
        double a[8], b[4];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) a[mi] = ps[kb * kBlkDoubles + mi * 32];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) b[ni] = qs[kb * kBlkDoubles + ni * 32];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done reading stage s
      // refill the stage the PREVIOUS chunk used: the other warps are at most a
      // chunk behind warp 0, so the wait is short and stalls only warp 0
      if (tid == 0 && q >= 1 && q - 1 + kStages < total_chunks) {
        const int qp = q - 1;
        mbar_wait(&empty[qp % kStages], (qp / kStages) & 1);
        fence_proxy_async();
        issue(qp + kStages);
      }
    }

    if (bulk_ok && !part && (ti > tj || (kOwned && !tri))) {
      // warp-local: the warp's boxes are private, so no CTA barrier; lane 0
      // issued this warp's previous reduces and waits for them to drain
      bulk_wait_read0();
      __syncwarp();
      double* wbuf = cbuf + warp * 4 * kBoxDoubles;
#pragma unroll
      for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            // element (row, col) of the warp block -> box mi/2, 16-byte chunk
            // (row%16)/2 XOR col%8 of the box's 128-byte column (SWIZZLE_128B)
            const int r = (mi & 1) * 8 + (lane >> 2), col = ni * 8 + 2 * (lane & 3) + e;
            wbuf[(mi >> 1) * kBoxDoubles + col * kBoxRows + (((r >> 1) ^ (col & 7)) << 1) + (r & 1)] =
                acc[mi][ni][e];
          }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int b = 0; b < 4; ++b)
          tensor_reduce_add_2d(&cmap, ti * kTile + wm * 64 + b * kBoxRows, tj * kTile + wn * 32,
                               wbuf + b * kBoxDoubles);
        bulk_commit();
      }
      continue;
    }

    const int row_base = ti * kTile + wm * 64 + (lane >> 2);
    const int col_base = tj * kTile + wn * 32 + 2 * (lane & 3);
    // straddling tile of the column-owned launch: columns of other ranks stay untouched
    auto mine = [&](int col) {
      if constexpr (kOwned) return !part || int(((own_cbase + col) / own_nbd) % own_g) == own_rank;
      else return true;
    };
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // epilogue in two halves to bound register use
      double cin[4][4][2];
#pragma unroll
      for (int mm = 0; mm < 4; ++mm)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int row = row_base + (h * 4 + mm) * 8, col = col_base + ni * 8 + e;
            cin[mm][ni][e] =
                (beta != 0.0 && row < n && col < ncols && (row > col || !tri) && mine(col))
                    ? C[(long long)col * ldc + row]
                    : 0.0;
          }
#pragma unroll
      for (int mm = 0; mm < 4; ++mm)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int row = row_base + (h * 4 + mm) * 8, col = col_base + ni * 8 + e;
            if (row < n && col < ncols && (row > col || !tri) && mine(col))
              C[(long long)col * ldc + row] =
                  (beta == 1.0 ? cin[mm][ni][e] : beta * cin[mm][ni][e]) + acc[h * 4 + mm][ni][e];
          }
    }
  }
  bulk_wait0();
}

// Small trailing updates (few 128x128 tiles: the late panels of config 2, config 1):
// one CTA of 4 warps per 64x64 lower tile, several CTAs per SM.  A 64-row tile is
// one half (m8 blocks 0-7 or 8-15) of a packed 128-row tile, i.e. a contiguous 2 KiB
// piece of every 4 KiB k4 block, streamed by bulk copies through a 3-stage ring.
// Each C element accumulates the same DMMA k4 blocks in the same order as in
// gemm_lower_nt_kernel and is added to C once, so the result is bit-identical.
constexpr int kSmT = 64, kSmThreads = 128, kSmStages = 3, kSmK4 = 4;
constexpr int kSmHalf = 8 * 32;  // doubles of a half k4 block (8 m8 blocks)
constexpr size_t kSmSmem = size_t(kSmStages) * 2 * kSmK4 * kSmHalf * sizeof(double) + 2 * kSmStages * 8 + 128;

__global__ void __launch_bounds__(kSmThreads) gemm_lower_small_kernel(const double* __restrict__ P,
                                                                      const double* __restrict__ Q, int k4cap,
                                                                      int nk4_host, const int* __restrict__ nk4_dev,
                                                                      double* __restrict__ C, long long ldc, int n,
                                                                      double beta) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sP = reinterpret_cast<double*>(smem_raw);
  double* sQ = sP + kSmStages * kSmK4 * kSmHalf;
  uint64_t* full = reinterpret_cast<uint64_t*>(sQ + kSmStages * kSmK4 * kSmHalf);
  const int nk4 = nk4_dev ? *nk4_dev : nk4_host;
  const int t = blockIdx.x;
  int ti = int((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
  while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
  while (ti * (ti + 1) / 2 > t) --ti;
  const int tj = t - ti * (ti + 1) / 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 1, wn = warp & 1;
  const int nch = (nk4 + kSmK4 - 1) / kSmK4;
  if (tid == 0) {
    for (int s2 = 0; s2 < kSmStages; ++s2) mbar_init(&full[s2], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // half k4 block q of 64-tile x: packed 128-tile x/2, m8 blocks (x&1)*8 .. +7
  auto issue = [&](int c) {
    const int s2 = c % kSmStages;
    const int q0 = c * kSmK4, nb = min(kSmK4, nk4 - q0);
    mbar_arrive_expect_tx(&full[s2], uint32_t(2 * nb * kSmHalf * sizeof(double)));
    for (int q = 0; q < nb; ++q) {
      const double* ps = P + (((size_t)(ti >> 1) * k4cap + q0 + q) * 16 + (ti & 1) * 8) * 32;
      const double* qs = Q + (((size_t)(tj >> 1) * k4cap + q0 + q) * 16 + (tj & 1) * 8) * 32;
      bulk_g2s(sP + ((size_t)s2 * kSmK4 + q) * kSmHalf, ps, kSmHalf * sizeof(double), &full[s2]);
      bulk_g2s(sQ + ((size_t)s2 * kSmK4 + q) * kSmHalf, qs, kSmHalf * sizeof(double), &full[s2]);
    }
  };
  if (tid == 0)
    for (int c = 0; c < min(kSmStages, nch); ++c) issue(c);
  // this thread's C entries, loaded now so their latency hides behind the k loop
  const int row_base = ti * kSmT + wm * 32 + (lane >> 2);
  const int col_base = tj * kSmT + wn * 32 + 2 * (lane & 3);
  double cin[4][4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = row_base + mi * 8, col = col_base + ni * 8 + e;
        cin[mi][ni][e] = (beta != 0.0 && row < n && col < n && row > col) ? C[(long long)col * ldc + row] : 0.0;
      }
  double acc[4][4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  for (int c = 0; c < nch; ++c) {
    const int s2 = c % kSmStages;
    mbar_wait(&full[s2], (c / kSmStages) & 1);
    const int nb = min(kSmK4, nk4 - c * kSmK4);
    const double* ps = sP + (size_t)s2 * kSmK4 * kSmHalf + (wm * 4) * 32 + lane;
    const double* qs = sQ + (size_t)s2 * kSmK4 * kSmHalf + (wn * 4) * 32 + lane;
    for (int kb = 0; kb < nb; ++kb) {
      double a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = ps[kb * kSmHalf + mi * 32];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = qs[kb * kSmHalf + ni * 32];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
    __syncthreads();  // stage s2 consumed by every warp
    if (tid == 0 && c + kSmStages < nch) {
      fence_proxy_async();
      issue(c + kSmStages);
    }
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = row_base + mi * 8, col = col_base + ni * 8 + e;
        if (row < n && col < n && row > col)
          C[(long long)col * ldc + row] = (beta == 1.0 ? cin[mi][ni][e] : beta * cin[mi][ni][e]) + acc[mi][ni][e];
      }
}

__device__ __forceinline__ void packed_decode(size_t off, int k4cap, int& row, int& col) {
  int lane = int(off & 31);
  int mb = int((off >> 5) & 15);
  size_t rest = off >> 9;
  int q = int(rest % (size_t)k4cap);
  int t = int(rest / (size_t)k4cap);
  row = t * kTile + mb * 8 + (lane >> 2);
  col = q * 4 + (lane & 3);
}

// P = alpha*A, Q[:, j] = t[j-1] A[:, j-1] - t[j] A[:, j+1]   (Q = A T^T, T = tridiag(t))
// optional var1 straggler pair (rows >= 1 only; l = A[:, ka-1]):
//   P[:, ka] = l,  P[:, ka+1] = -y,  Q[:, ka] = y,  Q[:, ka+1] = l
// so that sum_k P Q^T = alpha A T A^T + l y^T - y l^T.
// shift > 0: packed rows [0, shift) are zero and packed row r holds A row
// r - shift (the driver aligns the C region to 128-byte lines that way)
__global__ void pack_rankk_kernel(const double* __restrict__ A, long long lda, int rows, int ka,
                                  const double* __restrict__ t, double alpha, const double* __restrict__ y,
                                  int k4cap, double* __restrict__ P, double* __restrict__ Q, int shift) {
  const size_t total = (size_t)tiles_for(rows + shift) * kTile * 4 * k4cap;
  for (size_t off = blockIdx.x * (size_t)blockDim.x + threadIdx.x; off < total;
       off += (size_t)gridDim.x * blockDim.x) {
    int row, col;
    packed_decode(off, k4cap, row, col);
    row -= shift;
    double p = 0.0, q = 0.0;
    if (row >= 0 && row < rows) {
      if (col < ka) {
        const double* ar = A + row;
        p = alpha * ar[(long long)col * lda];
        double acc = 0.0;
        if (col >= 1) acc = t[col - 1] * ar[(long long)(col - 1) * lda];
        if (col + 1 < ka) acc -= t[col] * ar[(long long)(col + 1) * lda];
        q = acc;
      } else if (y != nullptr && row >= 1 && col < ka + 2) {
        double lv = A[(long long)(ka - 1) * lda + row];
        double yv = y[row];
        if (col == ka) {
          p = lv;
          q = yv;
        } else {
          p = -yv;
          q = lv;
        }
      }
    }
    P[off] = p;
    Q[off] = q;
  }
}

// skew_tridiag_gemm (kernels3.py:239-302): P = alpha*A (p rows), Q = (T B)^T
// (q rows) with Q[j, c] = t[c-1] B[c-1, j] - t[c] B[c+1, j]
__global__ void pack_gemm_kernel(const double* __restrict__ A, long long lda, int p, const double* __restrict__ B,
                                 long long ldb, int q, int k, const double* __restrict__ t, double alpha, int k4cap,
                                 double* __restrict__ P, double* __restrict__ Q, int btrans) {
  // btrans: B is given as B^T (q x k, column stride ldb), i.e. B[c, j] = B_arg[j + c*ldb]
  const long long bs_row = btrans ? 1 : ldb, bs_col = btrans ? ldb : 1;
  const size_t totp = (size_t)tiles_for(p) * kTile * 4 * k4cap, totq = (size_t)tiles_for(q) * kTile * 4 * k4cap;
  const size_t total = totp > totq ? totp : totq;
  for (size_t off = blockIdx.x * (size_t)blockDim.x + threadIdx.x; off < total;
       off += (size_t)gridDim.x * blockDim.x) {
    int row, col;
    packed_decode(off, k4cap, row, col);
    if (off < totp) P[off] = (row < p && col < k) ? alpha * A[(long long)col * lda + row] : 0.0;
    if (off < totq) {
      double v = 0.0;
      if (row < q && col < k) {
        const double* bj = B + (long long)row * bs_row;
        if (col >= 1) v = t[col - 1] * bj[(long long)(col - 1) * bs_col];
        if (col + 1 < k) v -= t[col] * bj[(long long)(col + 1) * bs_col];
      }
      Q[off] = v;
    }
  }
}

__global__ void scale_block_kernel(double* __restrict__ C, long long ldc, int p, int q, double beta, int tri) {
  for (int j = blockIdx.y; j < q; j += gridDim.y)
    for (int i = (tri ? j + 1 : 0) + blockIdx.x * blockDim.x + threadIdx.x; i < p; i += gridDim.x * blockDim.x) {
      double* c = C + (long long)j * ldc + i;
      *c = beta == 0.0 ? 0.0 : beta * *c;
    }
}

// keep[j] = column j is nonzero in both A and B (kernels3.py:318-321);
// single CTA: flags, then an ordered compaction.
// grid (column groups, row chunks); flags[j] |= (chunk of A[:, j] nonzero) etc.
// flags[j] bit 0: A column nonzero, bit 1: B column nonzero (zeroed by the launcher)
__global__ void rank2k_flags_kernel(const double* __restrict__ A, long long lda, const double* __restrict__ B,
                                    long long ldb, int n, int k, int skip_zero, int* __restrict__ flags) {
  const int wpb = blockDim.x >> 5;
  const int rchunk = (n + gridDim.y - 1) / gridDim.y;
  const int r0 = blockIdx.y * rchunk, r1 = min(n, r0 + rchunk);
  for (int j = blockIdx.x * wpb + (threadIdx.x >> 5); j < k; j += gridDim.x * wpb) {
    int lane = threadIdx.x & 31;
    int nzA = 0, nzB = 0;
    if (skip_zero) {
      for (int i = r0 + lane; i < r1; i += 32) {
        nzA |= A[(long long)j * lda + i] != 0.0;
        nzB |= B[(long long)j * ldb + i] != 0.0;
      }
      nzA = __any_sync(0xffffffffu, nzA);
      nzB = __any_sync(0xffffffffu, nzB);
    } else {
      nzA = nzB = 1;
    }
    if (lane == 0 && (nzA || nzB)) atomicOr(flags + j, (nzA ? 1 : 0) | (nzB ? 2 : 0));
  }
}

__global__ void rank2k_compact_kernel(const int* __restrict__ flags, int k, int* __restrict__ keep,
                                      int* __restrict__ keff_dev, int* __restrict__ nk4_dev) {
  __shared__ int cnt[1024];
  const int per = (k + blockDim.x - 1) / blockDim.x;
  const int j0 = threadIdx.x * per, j1 = min(k, j0 + per);
  int c = 0;
  for (int j = j0; j < j1; ++j) c += flags[j] == 3;
  cnt[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      int v = cnt[t];
      cnt[t] = acc;
      acc += v;
    }
    *keff_dev = acc;
    *nk4_dev = (2 * acc + 3) / 4;
  }
  __syncthreads();
  int o = cnt[threadIdx.x];
  for (int j = j0; j < j1; ++j)
    if (flags[j] == 3) keep[o++] = j;
}

// P = alpha*[A_keep | B_keep], Q = [B_keep | -A_keep]  => sum P Q^T = alpha (A B^T - B A^T)
__global__ void pack_rank2k_kernel(const double* __restrict__ A, long long lda, const double* __restrict__ B,
                                   long long ldb, int n, double alpha, const int* __restrict__ keep,
                                   const int* __restrict__ keff_dev, int k4cap, double* __restrict__ P,
                                   double* __restrict__ Q) {
  const int keff = *keff_dev;
  const size_t total = (size_t)tiles_for(n) * kTile * 4 * k4cap;
  for (size_t off = blockIdx.x * (size_t)blockDim.x + threadIdx.x; off < total;
       off += (size_t)gridDim.x * blockDim.x) {
    int row, col;
    packed_decode(off, k4cap, row, col);
    double p = 0.0, q = 0.0;
    if (row < n && col < 2 * keff) {
      int j = keep[col < keff ? col : col - keff];
      double av = A[(long long)j * lda + row], bv = B[(long long)j * ldb + row];
      if (col < keff) {
        p = alpha * av;
        q = bv;
      } else {
        p = alpha * bv;
        q = -av;
      }
    }
    P[off] = p;
    Q[off] = q;
  }
}

// skr2k prologue in ONE cooperative launch (kernels3.py:318-321 + the packing):
//  phase 1  every CTA scans a block of rows of A and B and records, per column,
//           "this block holds a nonzero of A / of B" as two bits (plain stores to
//           its own words of `part`, so nothing needs zeroing);
//  grid barrier;
//  phase 2  every CTA ORs the per-block words, builds the ordered keep list in
//           shared memory (columns nonzero in both factors), CTA 0 publishes keep /
//           keff / nk4, and all CTAs pack P = alpha [A_keep | B_keep], Q = [B_keep | -A_keep].
// Replaces memset + flags + compact + pack (four dependent launches, ~30 us of the
// 120 us config-2b microbench) by one.
constexpr int kPrepThreads = 1024;
__global__ void __launch_bounds__(kPrepThreads, 1)
rank2k_prep_kernel(const double* __restrict__ A, long long lda, const double* __restrict__ B, long long ldb, int n,
                   int k, int skip_zero, double alpha, int k4cap, unsigned* __restrict__ part, int* __restrict__ keep,
                   int* __restrict__ cnt, double* __restrict__ P, double* __restrict__ Q) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int words = (k + 15) >> 4;  // two bits per column
  unsigned* bits = reinterpret_cast<unsigned*>(smem_raw);  // [words]
  int* skeep = reinterpret_cast<int*>(bits + words);       // [k]
  __shared__ int s_keff;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = kPrepThreads >> 5;
  for (int i = tid; i < words; i += kPrepThreads) bits[i] = 0u;
  __syncthreads();
  if (skip_zero) {
    // row blocks of a multiple of 32 rows, one per CTA
    int rc = (n + gridDim.x - 1) / gridDim.x;
    rc = (rc + 31) & ~31;
    const int r0 = blockIdx.x * rc, r1 = min(n, r0 + rc);
    if (r0 < r1) {
      // four columns per warp and trip: the eight loads of a row group are issued before
      // any of them is reduced (one column at a time waited out a DRAM latency per column)
      for (int j0 = warp; j0 < k; j0 += 4 * nw) {
        int nzA[4] = {0, 0, 0, 0}, nzB[4] = {0, 0, 0, 0};
        for (int i = r0 + lane; i < r1; i += 32) {
          double av[4], bv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int j = j0 + e * nw;
            av[e] = j < k ? A[(long long)j * lda + i] : 0.0;
            bv[e] = j < k ? B[(long long)j * ldb + i] : 0.0;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            nzA[e] |= av[e] != 0.0;
            nzB[e] |= bv[e] != 0.0;
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = j0 + e * nw;
          const int a1 = __any_sync(0xffffffffu, nzA[e]), b1 = __any_sync(0xffffffffu, nzB[e]);
          if (lane == 0 && j < k && (a1 || b1))
            atomicOr(&bits[j >> 4], unsigned((a1 ? 1 : 0) | (b1 ? 2 : 0)) << (2 * (j & 15)));
        }
      }
    }
    __syncthreads();
    for (int i = tid; i < words; i += kPrepThreads) part[(size_t)blockIdx.x * words + i] = bits[i];
    __threadfence();
    cooperative_groups::this_grid().sync();
    for (int i = tid; i < words; i += kPrepThreads) bits[i] = 0u;
    __syncthreads();
    const int tot = (int)gridDim.x * words;
    for (int i = tid; i < tot; i += kPrepThreads) {
      const unsigned v = __ldcg(part + i);
      if (v) atomicOr(&bits[i % words], v);
    }
    __syncthreads();
  }
  if (warp == 0) {
    int base = 0;
    for (int j0 = 0; j0 < k; j0 += 32) {
      const int j = j0 + lane;
      const bool on = j < k && (!skip_zero || ((bits[j >> 4] >> (2 * (j & 15))) & 3u) == 3u);
      const unsigned bal = __ballot_sync(0xffffffffu, on);
      if (on) skeep[base + __popc(bal & ((1u << lane) - 1u))] = j;
      base += __popc(bal);
    }
    if (lane == 0) s_keff = base;
  }
  __syncthreads();
  const int keff = s_keff;
  if (blockIdx.x == 0) {
    for (int i = tid; i < keff; i += kPrepThreads) keep[i] = skeep[i];
    if (tid == 0) {
      cnt[0] = keff;
      cnt[1] = (2 * keff + 3) / 4;
    }
  }
  const size_t total = (size_t)tiles_for(n) * kTile * 4 * k4cap;
  const size_t stride = (size_t)gridDim.x * kPrepThreads;
  for (size_t off0 = blockIdx.x * (size_t)kPrepThreads + tid; off0 < total; off0 += 4 * stride) {
    // four packed entries per trip, their loads issued together
    double av[4], bv[4];
    bool lowh[4], on[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const size_t off = off0 + e * stride;
      int row = 0, col = 0;
      if (off < total) packed_decode(off, k4cap, row, col);
      on[e] = off < total && row < n && col < 2 * keff;
      lowh[e] = col < keff;
      const int j = on[e] ? skeep[lowh[e] ? col : col - keff] : 0;
      av[e] = on[e] ? A[(long long)j * lda + row] : 0.0;
      bv[e] = on[e] ? B[(long long)j * ldb + row] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const size_t off = off0 + e * stride;
      if (off < total) {
        P[off] = on[e] ? (lowh[e] ? alpha * av[e] : alpha * bv[e]) : 0.0;
        Q[off] = on[e] ? (lowh[e] ? bv[e] : -av[e]) : 0.0;
      }
    }
  }
}

// W = A S with T = S - S^T (core.py:153-169, kernels3.py:354-364):
// even columns zero; odd j: W[:, j] = -tau[j-1] A[:, j-1] + tau[j] A[:, j+1] (second term if j+1 < k)
__global__ void form_w_kernel(const double* __restrict__ A, long long lda, int n, int k,
                              const double* __restrict__ tau, double* __restrict__ W, long long ldw) {
  const size_t total = (size_t)n * k;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    int j = int(e / n), i = int(e % n);
    double w = 0.0;
    if (j & 1) {
      // two roundings, in the reference's entry order (no FMA contraction): bit-identical W
      w = __dmul_rn(-tau[j - 1], A[(long long)(j - 1) * lda + i]);
      if (j + 1 < k) w = __dadd_rn(w, __dmul_rn(tau[j], A[(long long)(j + 1) * lda + i]));
    }
    W[(long long)j * ldw + i] = w;
  }
}

int grid_for(size_t total, int threads) {
  size_t g = (total + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  return int(g < 1 ? 1 : g);
}

}  // namespace

namespace {
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      enc = nullptr;
  }
  return enc;
}
}  // namespace

cudaError_t launch_gemm_lower(const double* P, const double* Q, int k4cap, int nk4, const int* nk4_dev,
                              double* C, long long ldc, int n, double beta, cudaStream_t stream,
                              const ColOwner* own, int ncols, int tri) {
  if (ncols < 0) ncols = n;
  if (n < 1 || (own == nullptr && n < 2)) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_lower_nt_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kGemmSmem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(gemm_lower_nt_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  // tensor map over C (rows x cols = n x n, column stride ldc) for the
  // bulk-reduce epilogue; needs a 16-byte aligned base and an even ldc
  CUtensorMap cmap, pmap;
  memset(&cmap, 0, sizeof(cmap));
  memset(&pmap, 0, sizeof(pmap));
  int use_tmap = 0;
  PFN_cuTensorMapEncodeTiled_v12000 enc = tmap_encoder();
  if (enc && beta == 1.0 && (ldc & 1) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0) {
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)ncols};
    cuuint64_t strides[1] = {(cuuint64_t)ldc * sizeof(double)};
    cuuint32_t box[2] = {(cuuint32_t)kBoxRows, (cuuint32_t)kBoxCols}, es[2] = {1, 1};
    use_tmap = enc(&cmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, C, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    // L2 prefetch map: one 128 x 128 box per C tile (no swizzle; prefetch only)
    cuuint32_t pbox[2] = {(cuuint32_t)kTile, (cuuint32_t)kTile};
    use_tmap = use_tmap &&
               enc(&pmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, C, dims, strides, pbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  int nt = tiles_for(n);
  int ntiles = own ? own->ntiles : nt * (nt + 1) / 2;
  if (ntiles == 0) return cudaSuccess;
  // few 128x128 tiles (under ~four waves): 64x64 tiles, one 4-warp CTA each (bit-identical)
  static const int small_max = [] {
    const char* v = getenv("SKL_GEMM_SMALL_TILES");
    return v && *v ? atoi(v) : 600;  // ~4 waves of 128x128 tiles (config 2: 1.40 -> 1.34 ms against 296)
  }();
  static bool sattr = false;
  if (!sattr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_lower_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmSmem);
    if (e != cudaSuccess) return e;
    sattr = true;
  }
  if (!own && tri && ncols == n && ntiles < small_max) {
    const int nt64 = (n + kSmT - 1) / kSmT;
    gemm_lower_small_kernel<<<nt64 * (nt64 + 1) / 2, kSmThreads, kSmSmem, stream>>>(P, Q, k4cap, nk4, nk4_dev, C,
                                                                                   ldc, n, beta);
    return cudaGetLastError();
  }
  // (a split of a partial last wave into 64x64 quarters measured no gain: DESIGN.md §4)
  int grid = ntiles < nsm ? ntiles : nsm;
  if (own)
    gemm_lower_nt_kernel<true><<<grid, kGemmThreads, kGemmSmem, stream>>>(
        cmap, pmap, use_tmap, P, Q, k4cap, nk4, nk4_dev, C, ldc, n, beta, own->tab, own->cbase, own->nbd, own->G,
        own->rank, ncols, tri);
  else
    gemm_lower_nt_kernel<false><<<grid, kGemmThreads, kGemmSmem, stream>>>(cmap, pmap, use_tmap, P, Q, k4cap, nk4,
                                                                           nk4_dev, C, ldc, n, beta, nullptr, 0, 1,
                                                                           1, 0, n, 1);
  return cudaGetLastError();
}

int build_owner_table(int n, long long cbase, int nbd, int G, int rank, int* tab) {
  const int nt = tiles_for(n);
  int m = 0, total = 0;
  for (int tj = 0; tj < nt; ++tj) {
    const long long c0 = cbase + (long long)tj * kTile, c1 = std::min(cbase + n, c0 + kTile);
    int owned = 0;
    for (long long c = c0; c < c1;) {  // walk the distribution blocks the tile column crosses
      const long long bend = std::min(c1, (c / nbd + 1) * nbd);
      if ((c / nbd) % G == rank) owned += int(bend - c);
      c = bend;
    }
    if (owned == 0) continue;
    int* e = tab + 2 + 4 * m;
    e[0] = tj;
    e[1] = total;
    e[2] = owned < int(c1 - c0) ? 1 : 0;
    e[3] = tj;
    total += nt - tj;
    ++m;
  }
  tab[0] = m;
  tab[1] = total;
  return total;
}

int build_rect_table(int p, int q, int tri, int* tab) {
  const int ntr = tiles_for(p), ntc = tiles_for(q);
  int m = 0, total = 0;
  for (int tj = 0; tj < ntc; ++tj) {
    const int row0 = tri ? tj : 0;
    if (row0 >= ntr) break;
    int* e = tab + 2 + 4 * m;
    e[0] = tj;
    e[1] = total;
    e[2] = 0;
    e[3] = row0;
    total += ntr - row0;
    ++m;
  }
  tab[0] = m;
  tab[1] = total;
  return total;
}

cudaError_t launch_pack_rankk(const double* A, long long lda, int rows, int ka, const double* tau_base,
                              double alpha, const double* y, int k4cap, double* P, double* Q,
                              cudaStream_t stream, int shift) {
  size_t total = packed_elems(rows + shift, k4cap);
  pack_rankk_kernel<<<grid_for(total, 256), 256, 0, stream>>>(A, lda, rows, ka, tau_base, alpha, y, k4cap, P, Q,
                                                              shift);
  return cudaGetLastError();
}

cudaError_t launch_pack_gemm(const double* A, long long lda, int p, const double* B, long long ldb, int q, int k,
                             const double* t, double alpha, int k4cap, double* P, double* Q, cudaStream_t stream,
                             int btrans) {
  const size_t total = std::max(packed_elems(p, k4cap), packed_elems(q, k4cap));
  pack_gemm_kernel<<<grid_for(total, 256), 256, 0, stream>>>(A, lda, p, B, ldb, q, k, t, alpha, k4cap, P, Q,
                                                             btrans);
  return cudaGetLastError();
}

cudaError_t launch_scale_block(double* C, long long ldc, int p, int q, double beta, int tri, cudaStream_t stream) {
  if (p <= 0 || q <= 0 || beta == 1.0) return cudaSuccess;
  dim3 grid((p + 255) / 256 < 8 ? (p + 255) / 256 : 8, q < 4096 ? q : 4096);
  scale_block_kernel<<<grid, 256, 0, stream>>>(C, ldc, p, q, beta, tri);
  return cudaGetLastError();
}

cudaError_t launch_rank2k_keep(const double* A, long long lda, const double* B, long long ldb, int n, int k,
                               int skip_zero, int* keep, int* keff_dev, int* nk4_dev, cudaStream_t stream) {
  // flags live in keep's tail half: keep has room for k entries, flags reuse nk4_dev+1.. is unsafe, so use
  // the upper part of the keep array when k is small enough; the launcher passes a scratch via keff_dev+2
  int* flags = keff_dev + 2;
  cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int) * (k > 0 ? k : 1), stream);
  if (e != cudaSuccess) return e;
  int bx = (k + 7) / 8;
  if (bx < 1) bx = 1;
  int by = (n + 255) / 256;
  if (by > 64) by = 64;
  if (by < 1) by = 1;
  rank2k_flags_kernel<<<dim3(bx, by), 256, 0, stream>>>(A, lda, B, ldb, n, k, skip_zero, flags);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  rank2k_compact_kernel<<<1, 1024, 0, stream>>>(flags, k, keep, keff_dev, nk4_dev);
  return cudaGetLastError();
}

cudaError_t launch_pack_rank2k(const double* A, long long lda, const double* B, long long ldb, int n, int k,
                               double alpha, const int* keep, const int* keff_dev, int k4cap, double* P,
                               double* Q, cudaStream_t stream) {
  (void)k;
  size_t total = packed_elems(n, k4cap);
  pack_rank2k_kernel<<<grid_for(total, 256), 256, 0, stream>>>(A, lda, B, ldb, n, alpha, keep, keff_dev, k4cap, P,
                                                               Q);
  return cudaGetLastError();
}

size_t rank2k_prep_scratch_words(int k) {
  // one (k + 15) / 16-word bit row per CTA of the cooperative grid (at most one CTA per SM; 256 bounds the SM count)
  return (size_t)256 * (size_t)((std::max(k, 1) + 15) / 16);
}

cudaError_t launch_rank2k_prep(const double* A, long long lda, const double* B, long long ldb, int n, int k,
                               int skip_zero, double alpha, int k4cap, unsigned* part, int* keep, int* cnt, double* P,
                               double* Q, cudaStream_t stream) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t smem = sizeof(unsigned) * (size_t)((k + 15) / 16) + sizeof(int) * (size_t)std::max(k, 1);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  if (smem > 40 * 1024) {
    cudaError_t e =
        cudaFuncSetAttribute(rank2k_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int grid = std::min(nsm, 256);
  void* args[] = {&A, &lda, &B, &ldb, &n, &k, &skip_zero, &alpha, &k4cap, &part, &keep, &cnt, &P, &Q};
  return cudaLaunchCooperativeKernel((void*)rank2k_prep_kernel, dim3(grid), dim3(kPrepThreads), args, smem, stream);
}

cudaError_t launch_form_w(const double* A, long long lda, int n, int k, const double* tau, double* W,
                          long long ldw, cudaStream_t stream) {
  size_t total = (size_t)n * k;
  if (total == 0) return cudaSuccess;
  form_w_kernel<<<grid_for(total, 256), 256, 0, stream>>>(A, lda, n, k, tau, W, ldw);
  return cudaGetLastError();
}

}  // namespace skl
