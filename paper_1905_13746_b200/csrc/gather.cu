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

// UNPACK-U4: one thread per 8 packed bytes (16 counts) -> one 16-B store.
// Byte j holds feature 2j (low nibble) and 2j+1 (high nibble).
__global__ void __launch_bounds__(256)
    unpack_u4_kernel(const uint2* __restrict__ in, int64_t words, uint4* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < words;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint2 w = __ldg(in + i);
    // spread the 8 nibbles of each 32-bit half into 8 bytes (low nibble first)
    auto spread = [](uint32_t v, uint32_t& lo, uint32_t& hi) {
      lo = __byte_perm(v & 0x0f0f0f0fu, (v >> 4) & 0x0f0f0f0fu, 0x5140);
      hi = __byte_perm(v & 0x0f0f0f0fu, (v >> 4) & 0x0f0f0f0fu, 0x7362);
    };
    uint4 o;
    spread(w.x, o.x, o.y);
    spread(w.y, o.z, o.w);
    out[i] = o;
  }
}

cudaError_t unpack_u4_launch(const uint8_t* packed, int64_t n_rows, int64_t packed_pitch,
                             uint8_t* out, cudaStream_t stream) {
  const int64_t words = n_rows * (packed_pitch / 8);
  if (words == 0) return cudaSuccess;
  const int64_t b = (words + 255) / 256;
  unpack_u4_kernel<<<static_cast<int>(b < 148 * 16 ? b : 148 * 16), 256, 0, stream>>>(
      reinterpret_cast<const uint2*>(packed), words, reinterpret_cast<uint4*>(out));
  return cudaGetLastError();
}

}  // namespace gnb
