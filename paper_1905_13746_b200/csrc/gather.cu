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

// One warp per row (grid-stride over rows): lane j writes output columns j,
// j+32, ... (coalesced stores); the reads are the row's routed feature
// columns, gathered from a row that is one contiguous V-element span (L1/L2
// sectors shared by the warp).  T: the caller's storage (int32 / uint16 /
// uint8) in and out -- narrow rows stay narrow for K-PRED.
template <typename T>
__global__ void __launch_bounds__(256)
    gather_kernel(const T* __restrict__ x, int64_t n_rows, int32_t V, int64_t ldx,
                  const int32_t* __restrict__ size, int32_t width, int32_t limit,
                  const int32_t* __restrict__ route, const int32_t* __restrict__ features,
                  const int32_t* __restrict__ n_features, int32_t F, T* __restrict__ out,
                  int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
       r < n_rows; r += warps) {
    const int sz = __ldg(size + r);
    const int s = (sz >= 0 && sz < limit) ? __ldg(route + sz / width) : -1;
    const int nf = s >= 0 ? __ldg(n_features + s) : 0;
    const T* row = x + r * ldx;
    const int32_t* fs = features + static_cast<int64_t>(s < 0 ? 0 : s) * F;
    for (int j = lane; j < F; j += 32) {
      T v = 0;
      if (j < nf) {
        const int col = __ldg(fs + j);
        if (col >= 0 && col < V) v = row[col];
      }
      out[r * ldo + j] = v;
    }
  }
}

template <typename T>
static cudaError_t gather_launch_t(const void* x, int64_t n_rows, int32_t V, int64_t ldx,
                                   const int32_t* size, int32_t width, int32_t limit,
                                   const int32_t* route, const int32_t* features,
                                   const int32_t* n_features, int32_t F, void* out, int64_t ldo,
                                   cudaStream_t stream) {
  const int64_t b = (n_rows + 7) / 8;  // 8 rows (warps) per block
  gather_kernel<T><<<static_cast<int>(b < 148 * 16 ? b : 148 * 16), 256, 0, stream>>>(
      static_cast<const T*>(x), n_rows, V, ldx, size, width, limit, route, features, n_features,
      F, static_cast<T*>(out), ldo);
  return cudaGetLastError();
}

cudaError_t gather_launch(const void* x, int x_type, int64_t n_rows, int32_t V, int64_t ldx,
                          const int32_t* size, int32_t width, int32_t limit,
                          const int32_t* route, const int32_t* features,
                          const int32_t* n_features, int32_t F, void* out, int64_t ldo,
                          cudaStream_t stream) {
  if (n_rows == 0 || F == 0) return cudaSuccess;
  switch (x_type) {
    case GNB_X_U8:
      return gather_launch_t<uint8_t>(x, n_rows, V, ldx, size, width, limit, route, features,
                                      n_features, F, out, ldo, stream);
    case GNB_X_U16:
      return gather_launch_t<uint16_t>(x, n_rows, V, ldx, size, width, limit, route, features,
                                       n_features, F, out, ldo, stream);
    default:
      return gather_launch_t<int32_t>(x, n_rows, V, ldx, size, width, limit, route, features,
                                      n_features, F, out, ldo, stream);
  }
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
