// Does the L2 round-trip latency of a flagged-word poll (ld.relaxed.gpu) depend on
// which die the polling SM sits on relative to the line's home?  One CTA per SM;
// thread 0 times dependent ld.relaxed.gpu loads to NCHUNK lines spread over a buffer
// (each line first touched so it is L2-resident), min of 8 per line.
// Output: smid, then NCHUNK latencies (cycles) per CTA.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

constexpr int NCHUNK = 512;
constexpr size_t STRIDE = 4096 + 128;  // bytes between probed lines (walks the slice hash)

__global__ void probe(const uint64_t* buf, unsigned* out) {
  if (threadIdx.x) return;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  out[blockIdx.x * (NCHUNK + 1)] = smid;
  uint64_t sink = 0;
  for (int c = 0; c < NCHUNK; ++c) {
    const uint64_t* p = buf + (size_t)c * STRIDE / 8;
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    sink += v;
    long long best = 1ll << 40;
    for (int r = 0; r < 8; ++r) {
      const uint64_t* q = p + (sink & 0);  // dependent address
      long long t0 = clock64();
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(q) : "memory");
      sink += v;
      long long t1 = clock64();
      if (sink == 12345) t1 += 1;  // keep the load ordered before t1
      if (t1 - t0 < best) best = t1 - t0;
    }
    out[blockIdx.x * (NCHUNK + 1) + 1 + c] = (unsigned)best;
  }
  if (sink == 0xdeadbeef) out[0] = 0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint64_t* buf;
  unsigned* out;
  cudaMalloc(&buf, NCHUNK * STRIDE + 4096);
  cudaMemset(buf, 0, NCHUNK * STRIDE + 4096);
  cudaMalloc(&out, sizeof(unsigned) * nsm * (NCHUNK + 1));
  probe<<<nsm, 32>>>(buf, out);
  cudaDeviceSynchronize();
  probe<<<nsm, 32>>>(buf, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<unsigned> h(nsm * (NCHUNK + 1));
  cudaMemcpy(h.data(), out, sizeof(unsigned) * h.size(), cudaMemcpyDeviceToHost);
  for (int b = 0; b < nsm; ++b) {
    printf("%u", h[b * (NCHUNK + 1)]);
    for (int c = 0; c < NCHUNK; ++c) printf(" %u", h[b * (NCHUNK + 1) + 1 + c]);
    printf("\n");
  }
  return 0;
}
