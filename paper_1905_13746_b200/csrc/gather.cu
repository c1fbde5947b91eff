// GATHER: route + FeatureSet gather on the device.
//
// x_vocab [N, V] (full vocabulary, mnemonic-sorted columns) -> x_out [N, F]
// holding each row's routed model's features in FeatureSet order, zero
// padded: the predict input layout.  Restates the per-sample lookups of
// engine._classify_slice (pkg/src/groupnb/engine.py:198-202) and the
// `histogram.entries.get(op)` walk over `_packed` in classifier.log_posterior
// (pkg/src/groupnb/classifier.py:142-147) as one streaming pass.
#include <cstdint>

#include "gnb_internal.h"

namespace gnb {

__global__ void __launch_bounds__(256)
    gather_kernel(const int32_t* __restrict__ x, int64_t n_rows, int32_t V, int64_t ldx,
                  const int32_t* __restrict__ size, int32_t width, int32_t limit,
                  const int32_t* __restrict__ route, const int32_t* __restrict__ features,
                  const int32_t* __restrict__ n_features, int32_t F, int32_t* __restrict__ out,
                  int64_t ldo) {
  const int64_t total = n_rows * F;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / F;
    const int j = static_cast<int>(i - r * F);
    const int sz = __ldg(size + r);
    int v = 0;
    if (sz >= 0 && sz < limit) {
      const int s = __ldg(route + sz / width);
      if (j < __ldg(n_features + s)) {
        const int col = __ldg(features + static_cast<int64_t>(s) * F + j);
        if (col >= 0 && col < V) v = __ldg(x + r * ldx + col);
      }
    }
    out[r * ldo + j] = v;
  }
}

cudaError_t gather_launch(const int32_t* x, int64_t n_rows, int32_t V, int64_t ldx,
                          const int32_t* size, int32_t width, int32_t limit,
                          const int32_t* route, const int32_t* features,
                          const int32_t* n_features, int32_t F, int32_t* out, int64_t ldo,
                          cudaStream_t stream) {
  const int64_t total = n_rows * F;
  if (total == 0) return cudaSuccess;
  const int64_t b = (total + 255) / 256;
  gather_kernel<<<static_cast<int>(b < 148 * 32 ? b : 148 * 32), 256, 0, stream>>>(
      x, n_rows, V, ldx, size, width, limit, route, features, n_features, F, out, ldo);
  return cudaGetLastError();
}

}  // namespace gnb
