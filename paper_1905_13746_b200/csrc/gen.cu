// GEN: device-side synthetic corpus following the reference's generator law
// (pkg/src/groupnb/synth.py:64-116) at scales the Python generator cannot
// reach.  Rows are laid out group by group (as GroupedCorpus.all_samples()
// orders them, corpus.py:111-116); every value is a pure function of
// (seed, global row index, column), so sharding the index space over GPUs
// or chunks reproduces the same matrix.
//
// Per row:  class c = row % C (balanced, synth.py:447-451 draws per class),
//           size ~ U[g*w, (g+1)*w) (synth.py:452), T = 64 + size/64 draws
//           (synth.py:453), count_v ~ Poisson(T * p_c[v]) -- the per-cell
//           Poisson limit of rng.multinomial(T, p_c) (synth.py:454), with
//           p_c from class_distributions (synth.py:412-428): weight 1 on the
//           class's block of columns, 1 - divergence elsewhere.  For C = 2
//           malware (c=1) owns the first ceil(V/2) columns, benign the rest.
#include <cmath>
#include <cstdint>

#include "gnb_internal.h"

namespace gnb {

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double unit(unsigned long long h) {  // [0, 1)
  return static_cast<double>(h >> 11) * 0x1p-53;
}

// Block b of C blocks over V columns: [ceil(b V / C), ceil((b+1) V / C)).
__device__ __forceinline__ int block_lo(int b, int V, int C) {
  return static_cast<int>((static_cast<long long>(b) * V + C - 1) / C);
}

__global__ void generate_kernel(const GenParams p) {
  const int NC = p.n_cols, V = p.vocab_cols, C = p.n_classes;
  const int64_t total = p.n_rows * static_cast<int64_t>(NC);
  const double low = 1.0 - p.divergence;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / NC;
    const int j = static_cast<int>(i - r * NC);
    const int v = p.col_map ? __ldg(p.col_map + j) : j;  // vocabulary column
    const long long R = p.row_offset + r;
    int g = 0;
    while (g < p.n_groups - 1 && R >= p.group_end[g]) ++g;
    const int c = static_cast<int>(R % C);
    const unsigned long long hr = mix64(p.seed ^ mix64(static_cast<unsigned long long>(R)));
    const int size = g * p.width + static_cast<int>(unit(hr) * p.width);
    if (j == 0) {
      p.size[r] = size;
      p.labels[r] = c;
    }
    const double draws = 64.0 + static_cast<double>(size / 64);
    const int b = C - 1 - c;  // class c owns block C-1-c
    const int lo = block_lo(b, V, C), hi = block_lo(b + 1, V, C);
    const double wsum = (hi - lo) + (V - (hi - lo)) * low;
    const double w = (v >= lo && v < hi) ? 1.0 : low;
    const double lam = draws * w / wsum;
    const unsigned long long hc = mix64(hr ^ (0xd1b54a32d192ed03ull * (v + 1)));
    double u = unit(hc);
    int k = 0;
    if (lam <= 0.0) {
      k = 0;
    } else if (lam < 64.0) {
      double pk = exp(-lam), cdf = pk;
      while (u > cdf && k < 4096) {
        ++k;
        pk *= lam / k;
        cdf += pk;
      }
    } else {  // normal approximation for large means
      const double u2 = unit(mix64(hc));
      const double z = sqrt(-2.0 * log(u > 0.0 ? u : 0x1p-53)) * cospi(2.0 * u2);
      k = static_cast<int>(fmax(0.0, rint(lam + sqrt(lam) * z)));
    }
    p.x[r * p.ldx + j] = k;
  }
}

cudaError_t generate_launch(const GenParams& p, cudaStream_t stream) {
  const int64_t total = p.n_rows * static_cast<int64_t>(p.n_cols);
  if (total == 0) return cudaSuccess;
  const int64_t blocks64 = (total + 255) / 256;
  const int blocks = static_cast<int>(blocks64 < 148 * 64 ? blocks64 : 148 * 64);
  generate_kernel<<<blocks, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace gnb
