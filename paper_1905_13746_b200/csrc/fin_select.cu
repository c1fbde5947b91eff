// FIN-SELECT (device): feature scoring + top-k for every size group at once
// (SURVEY 8f rank 3), for vocabularies / group counts where the host FIN's
// O(G V log V) starts to matter.  One CTA per group:
//   class totals over the full vocabulary        features.py:51-53
//   candidates = opcodes with a nonzero count     features.py:71
//   score = |S_m/T_m - S_b/T_b| (IEEE, same ops)  features.py:72-74
//   order by (-score, column) = (-score, mnemonic) features.py:85
// via a shared-memory bitonic sort of (~bits(score), column) keys (scores are
// >= 0, so their IEEE bit patterns order like the values).  The CTA then
// gathers the selected columns' per-class sums; the host finishes the
// logarithms with libm (gnb_fin_tables), so bundles stay bit-identical.
#include <cstdint>

#include "gnb_internal.h"

namespace gnb {

constexpr int kSelectThreads = 1024;

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(~0u, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  return red[0];
}

// smem: keys[P] (u64) + cols[P] (i32), P = next pow2 >= V
__global__ void __launch_bounds__(kSelectThreads)
    fin_select_kernel(const double* __restrict__ sums, const double* __restrict__ counts, int V,
                      int P, int k, int min_per_class, int32_t* __restrict__ state,
                      int32_t* __restrict__ n_features, int32_t* __restrict__ features,
                      double* __restrict__ selected /* [G][2][k] */) {
  extern __shared__ unsigned long long keys[];
  int* cols = reinterpret_cast<int*>(keys + P);
  __shared__ double red[32];
  __shared__ int n_cand;
  const int g = blockIdx.x;
  const double* Sb = sums + static_cast<int64_t>(g) * 2 * V;  // class 0 benign
  const double* Sm = Sb + V;                                  // class 1 malware
  const double nb = counts[2 * g], nm = counts[2 * g + 1];
  if (nb < min_per_class || nm < min_per_class) {
    if (threadIdx.x == 0) {
      state[g] = 0;
      n_features[g] = 0;
    }
    return;
  }
  double tb = 0.0, tm = 0.0;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    tb += Sb[v];
    tm += Sm[v];
  }
  tb = block_sum(tb, red);  // integer-valued: exact in any order below 2^53
  tm = block_sum(tm, red);
  if (tm == 0.0 || tb == 0.0) {  // malware checked first (features.py:67-70)
    if (threadIdx.x == 0) {
      state[g] = tm == 0.0 ? -1 : -2;
      n_features[g] = 0;
    }
    return;
  }
  if (threadIdx.x == 0) n_cand = 0;
  __syncthreads();
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const double cb = Sb[v], cm = Sm[v];
    if (cb == 0.0 && cm == 0.0) continue;
    const double score = fabs(cm / tm - cb / tb);
    const int slot = atomicAdd(&n_cand, 1);
    keys[slot] = ~static_cast<unsigned long long>(__double_as_longlong(score));
    cols[slot] = v;
  }
  __syncthreads();
  const int m = n_cand;
  for (int i = m + threadIdx.x; i < P; i += blockDim.x) {
    keys[i] = ~0ull;
    cols[i] = INT32_MAX;
  }
  __syncthreads();
  // bitonic sort ascending by (key, col)
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const unsigned long long a = keys[lo], b = keys[hi];
        const int ca = cols[lo], cb = cols[hi];
        const bool gt = a > b || (a == b && ca > cb);
        if (gt == up) {
          keys[lo] = b;
          keys[hi] = a;
          cols[lo] = cb;
          cols[hi] = ca;
        }
      }
      __syncthreads();
    }
  }
  const int F = m < k ? m : k;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const int c = j < F ? cols[j] : 0;
    features[static_cast<int64_t>(g) * k + j] = c;
    selected[(static_cast<int64_t>(g) * 2 + 0) * k + j] = j < F ? Sb[c] : 0.0;
    selected[(static_cast<int64_t>(g) * 2 + 1) * k + j] = j < F ? Sm[c] : 0.0;
  }
  if (threadIdx.x == 0) {
    state[g] = 1;
    n_features[g] = F;
  }
}

int fin_select_max_vocab() { return 16384; }

cudaError_t fin_select_launch(const double* sums, const double* counts, int G, int V, int k,
                              int min_per_class, int32_t* state, int32_t* n_features,
                              int32_t* features, double* selected, cudaStream_t stream) {
  int P = 1;
  while (P < V) P <<= 1;
  const size_t smem = static_cast<size_t>(P) * (8 + 4);
  cudaError_t e = cudaFuncSetAttribute(fin_select_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  fin_select_kernel<<<G, kSelectThreads, smem, stream>>>(sums, counts, V, P, k, min_per_class,
                                                         state, n_features, features, selected);
  return cudaGetLastError();
}

}  // namespace gnb
