// SLOT SORT: rows grouped by routed model slot (SURVEY 8f rank 2,
// "device group-sort"), so a K-PRED tile of a shuffled ragged batch shares one
// model and reads its tables from shared memory.  Replaces nothing in the
// reference (which routes per sample, engine.py:198-202); it is the B200
// batching of the paper's "model of the group and its files in the same core"
// (PAPER.md:96).
//
// Counting sort in three launches over the 4-byte sizes only:
//   hist    per-block slot histograms (shared atomics), slot-major [S+1][B]
//   scan    one-block exclusive scan over the (S+1)*B counts
//   scatter per-block cursors start at the scanned offsets; perm[pos] = row
// Bucket S collects rows whose size is out of range.  Order inside one
// (block, slot) bucket is not defined; K-PRED writes by row id.
#include <cstdint>

#include "gnb_internal.h"

namespace gnb {

constexpr int kSortThreads = 512;
constexpr int kSortMaxBlocks = 1024;
constexpr int kSortMaxSlots = 4096;

__device__ __forceinline__ int slot_of(const int32_t* size, int64_t r, int width, int limit,
                                       const int32_t* route, int S) {
  const int sz = __ldg(size + r);
  return (sz >= 0 && sz < limit) ? __ldg(route + sz / width) : S;
}

__global__ void __launch_bounds__(kSortThreads)
    slot_hist_kernel(const int32_t* __restrict__ size, int64_t n, int width, int limit,
                     const int32_t* __restrict__ route, int S, int64_t chunk,
                     int* __restrict__ counts) {
  extern __shared__ int hist[];
  const int B = gridDim.x, b = blockIdx.x;
  for (int s = threadIdx.x; s <= S; s += blockDim.x) hist[s] = 0;
  __syncthreads();
  const int64_t lo = b * chunk, hi = lo + chunk < n ? lo + chunk : n;
  for (int64_t r = lo + threadIdx.x; r < hi; r += blockDim.x)
    atomicAdd(&hist[slot_of(size, r, width, limit, route, S)], 1);
  __syncthreads();
  for (int s = threadIdx.x; s <= S; s += blockDim.x) counts[static_cast<int64_t>(s) * B + b] = hist[s];
}

// exclusive scan of m ints in place, one block
__global__ void __launch_bounds__(1024) slot_scan_kernel(int* __restrict__ v, int m) {
  __shared__ int part[1024];
  const int t = threadIdx.x, T = blockDim.x;
  const int per = (m + T - 1) / T;
  const int lo = t * per, hi = lo + per < m ? lo + per : m;
  int sum = 0;
  for (int i = lo; i < hi; ++i) sum += v[i];
  part[t] = sum;
  __syncthreads();
  for (int o = 1; o < T; o <<= 1) {  // inclusive Hillis-Steele over the thread sums
    const int add = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += add;
    __syncthreads();
  }
  int run = part[t] - sum;
  for (int i = lo; i < hi; ++i) {
    const int c = v[i];
    v[i] = run;
    run += c;
  }
}

__global__ void __launch_bounds__(kSortThreads)
    slot_scatter_kernel(const int32_t* __restrict__ size, int64_t n, int width, int limit,
                        const int32_t* __restrict__ route, int S, int64_t chunk,
                        const int* __restrict__ offsets, int32_t* __restrict__ perm) {
  extern __shared__ int cursor[];
  const int B = gridDim.x, b = blockIdx.x;
  for (int s = threadIdx.x; s <= S; s += blockDim.x)
    cursor[s] = offsets[static_cast<int64_t>(s) * B + b];
  __syncthreads();
  const int64_t lo = b * chunk, hi = lo + chunk < n ? lo + chunk : n;
  for (int64_t r = lo + threadIdx.x; r < hi; r += blockDim.x) {
    const int pos = atomicAdd(&cursor[slot_of(size, r, width, limit, route, S)], 1);
    perm[pos] = static_cast<int32_t>(r);
  }
}

static int sort_blocks(int64_t n) {
  const int64_t b = (n + 4095) / 4096;
  return static_cast<int>(b < 1 ? 1 : b > kSortMaxBlocks ? kSortMaxBlocks : b);
}

size_t slot_sort_workspace(int64_t n, int S) {
  return static_cast<size_t>(S + 1) * sort_blocks(n) * sizeof(int);
}

cudaError_t slot_sort(const int32_t* size, int64_t n, int width, int limit, const int32_t* route,
                      int S, int32_t* perm, void* workspace, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  if (S + 1 > kSortMaxSlots) return cudaErrorInvalidValue;
  const int B = sort_blocks(n);
  const int64_t chunk = (n + B - 1) / B;
  int* counts = static_cast<int*>(workspace);
  const size_t sm = static_cast<size_t>(S + 1) * sizeof(int);
  slot_hist_kernel<<<B, kSortThreads, sm, stream>>>(size, n, width, limit, route, S, chunk,
                                                    counts);
  slot_scan_kernel<<<1, 1024, 0, stream>>>(counts, (S + 1) * B);
  slot_scatter_kernel<<<B, kSortThreads, sm, stream>>>(size, n, width, limit, route, S, chunk,
                                                       counts, perm);
  return cudaGetLastError();
}

}  // namespace gnb
