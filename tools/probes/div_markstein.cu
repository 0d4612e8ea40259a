// Is q = fma(fma(-q0, b, a), r, q0), q0 = a * r, r = __drcp_rn(b) bit-identical to a / b
// for |a| <= |b| (the panel's column scaling, |v| <= |pivot|)?  Counts mismatches over
// random and adversarial pairs.
#include <cstdio>
#include <cstdint>
#include <curand_kernel.h>

__global__ void check(unsigned long long seed, long long per, unsigned long long* bad, double* ex) {
  curandStatePhilox4_32_10_t st;
  curand_init(seed, blockIdx.x * blockDim.x + threadIdx.x, 0, &st);
  unsigned long long nb = 0;
  for (long long i = 0; i < per; ++i) {
    const uint4 u = curand4(&st);
    double b = __longlong_as_double(((long long)(u.x & 0x7fffffffu) << 32) | u.y);  // random bits
    double a = __longlong_as_double(((long long)(u.z & 0x7fffffffu) << 32) | u.w);
    if (!(isfinite(a) && isfinite(b)) || b == 0.0) continue;
    if (fabs(a) > fabs(b)) { double t = a; a = b; b = t; }
    if (u.x & 0x80000000u) a = -a;
    if (u.z & 0x80000000u) b = -b;
    if (fabs(b) < 1e-300 || fabs(b) > 1e300) continue;  // pivots far from over/underflow
    if (fabs(a) < 1e-290 && a != 0.0) continue;      // residual would underflow: exact division there
    const double q1 = a / b;
    const double r = __drcp_rn(b);
    const double q0 = a * r;
    const double q = fma(fma(-q0, b, a), r, q0);
    if (__double_as_longlong(q) != __double_as_longlong(q1)) {
      if (nb == 0) { ex[0] = a; ex[1] = b; }
      ++nb;
    }
  }
  atomicAdd(bad, nb);
}

int main() {
  unsigned long long* bad;
  double* ex;
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&ex, 16);
  *bad = 0;
  check<<<148 * 8, 256>>>(1234, 20000, bad, ex);
  cudaDeviceSynchronize();
  printf("pairs %lld mismatches %llu example a=%.17g b=%.17g\n", 148LL * 8 * 256 * 20000, *bad, ex[0], ex[1]);
  return 0;
}
