// Temporary placeholders (replaced by twostep.cu / batched.cu).
#include "internal.h"
namespace skl {
template <typename T>
cudaError_t launch_batched(int, int, const T*, long long, long long, T*, long long, long long, T*, long long,
                           long long*, long long, double*, double*, cudaStream_t) {
  return cudaErrorNotSupported;
}
template cudaError_t launch_batched<double>(int, int, const double*, long long, long long, double*, long long,
                                            long long, double*, long long, long long*, long long, double*, double*,
                                            cudaStream_t);
template cudaError_t launch_batched<float>(int, int, const float*, long long, long long, float*, long long, long long,
                                           float*, long long, long long*, long long, double*, double*, cudaStream_t);
}  // namespace skl
