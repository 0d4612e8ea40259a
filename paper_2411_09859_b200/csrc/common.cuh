// Shared device helpers for the skewltl B200 kernels (sm_100a only).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef __CUDA_ARCH__
#define SKL_HOST_ONLY 1
#endif

namespace skl {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// LL ("low-latency") flagged words: every 8-byte word carries a 32-bit flag
// next to 32 bits of payload, so a reader can poll the data itself and needs
// no fence or separate flag (8-byte accesses are single-copy atomic).  A
// double travels as two flagged words written with one 16-byte store.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ll_put2(uint64_t* p, uint32_t d0, uint32_t d1, uint32_t flag) {
  uint64_t w0 = (uint64_t(flag) << 32) | d0;
  uint64_t w1 = (uint64_t(flag) << 32) | d1;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}

__device__ __forceinline__ void ll_put_double(uint64_t* p, double v, uint32_t flag) {
  uint64_t bits = __double_as_longlong(v);
  ll_put2(p, uint32_t(bits), uint32_t(bits >> 32), flag);
}

// spin until both words carry `flag`; returns the 2 payloads
__device__ __forceinline__ void ll_get2(const uint64_t* p, uint32_t flag, uint32_t& d0, uint32_t& d1) {
  uint64_t w0, w1;
  do {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
  } while (uint32_t(w0 >> 32) != flag || uint32_t(w1 >> 32) != flag);
  d0 = uint32_t(w0);
  d1 = uint32_t(w1);
}

// two flagged pairs (a 4-word record) polled together: one L2 round trip per attempt
__device__ __forceinline__ void ll_get4(const uint64_t* p, uint32_t flag, uint32_t& d0, uint32_t& d1, uint32_t& d2,
                                        uint32_t& d3) {
  uint64_t w0, w1, w2, w3;
  do {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w2), "=l"(w3) : "l"(p + 2) : "memory");
  } while (uint32_t(w0 >> 32) != flag || uint32_t(w1 >> 32) != flag || uint32_t(w2 >> 32) != flag ||
           uint32_t(w3 >> 32) != flag);
  d0 = uint32_t(w0);
  d1 = uint32_t(w1);
  d2 = uint32_t(w2);
  d3 = uint32_t(w3);
}

// three flagged pairs (a 6-word record) polled together: one L2 round trip per
// attempt instead of three dependent ones
__device__ __forceinline__ void ll_get6(const uint64_t* p, uint32_t flag, uint32_t& d0, uint32_t& d1, uint32_t& d2,
                                        uint32_t& d3, uint32_t& d4, uint32_t& d5) {
  uint64_t w0, w1, w2, w3, w4, w5;
  do {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w2), "=l"(w3) : "l"(p + 2) : "memory");
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w4), "=l"(w5) : "l"(p + 4) : "memory");
  } while (uint32_t(w0 >> 32) != flag || uint32_t(w1 >> 32) != flag || uint32_t(w2 >> 32) != flag ||
           uint32_t(w3 >> 32) != flag || uint32_t(w4 >> 32) != flag || uint32_t(w5 >> 32) != flag);
  d0 = uint32_t(w0);
  d1 = uint32_t(w1);
  d2 = uint32_t(w2);
  d3 = uint32_t(w3);
  d4 = uint32_t(w4);
  d5 = uint32_t(w5);
}

// two flagged doubles from independent places, polled together
__device__ __forceinline__ void ll_get_double2(const uint64_t* p, const uint64_t* q, uint32_t flag, double& x,
                                               double& y) {
  uint64_t w0, w1, w2, w3;
  do {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w2), "=l"(w3) : "l"(q) : "memory");
  } while (uint32_t(w0 >> 32) != flag || uint32_t(w1 >> 32) != flag || uint32_t(w2 >> 32) != flag ||
           uint32_t(w3 >> 32) != flag);
  x = __longlong_as_double((long long)((uint64_t(uint32_t(w1)) << 32) | uint32_t(w0)));
  y = __longlong_as_double((long long)((uint64_t(uint32_t(w3)) << 32) | uint32_t(w2)));
}

__device__ __forceinline__ double ll_get_double(const uint64_t* p, uint32_t flag) {
  uint32_t lo, hi;
  ll_get2(p, flag, lo, hi);
  return __longlong_as_double((long long)((uint64_t(hi) << 32) | lo));
}

// ---------------------------------------------------------------------------
// FP64 tensor pipe: DMMA.8x8x4.  Fragment layout (lane l):
//   A (8x4, row): a = A[l/4][l%4];  B (4x8, col): b = B[l%4][l/4]
//   C/D (8x8): d0 = D[l/4][2(l%4)], d1 = D[l/4][2(l%4)+1]
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// mbarrier + bulk async copy (TMA bulk engine, UBLKCP)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// wait for a phase with cluster-scope acquire (data delivered by remote CTAs)
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// wait for a phase whose payload was delivered into THIS CTA's shared memory by
// st.async / bulk copies completing on the barrier (complete_tx): the bytes are
// in local smem once the phase flips, so a CTA-scope acquire is enough (the
// cluster-scope form compiles to an extra CCTL.IVALL -- an L1 invalidate -- per
// wait).  SKL_XBAR_ACQ_CLUSTER=1 restores the cluster-scope wait (A/B builds).
__device__ __forceinline__ void mbar_wait_delivered(uint64_t* bar, uint32_t parity) {
#if defined(SKL_XBAR_ACQ_CLUSTER) && SKL_XBAR_ACQ_CLUSTER
  mbar_wait_acq_cluster(bar, parity);
#else
  mbar_wait(bar, parity);
#endif
}

// global -> shared bulk copy, completion signalled on `bar` (bytes multiple of 16)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// shared -> global tensor add-reduction of one box at (c0 = inner/row, c1 = col)
__device__ __forceinline__ void tensor_reduce_add_2d(const void* tmap, int c0, int c1, const void* src) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   tmap),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void prefetch_l2_tensor_2d(const void* tmap, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(tmap), "r"(c0), "r"(c1)
               : "memory");
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// ---------------------------------------------------------------------------
// skew-lower element access: X(p, q) of the full skew matrix whose strictly
// lower triangle is stored column-major in W (p != q).
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T skew_at(const T* __restrict__ W, long long ld, int p, int q) {
  return p > q ? W[(long long)q * ld + p] : -W[(long long)p * ld + q];
}

}  // namespace skl
