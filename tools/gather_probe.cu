// Probe: how fast can a CTA stream rows at ARBITRARY positions (the slot-sorted
// order of a shuffled ragged batch) from HBM into shared memory?
//   mode 0: contiguous tiles, one 1-D bulk copy per tile      (the sequential bound)
//   mode 1: one 1-D bulk copy per row, rows in `perm` order   (whole-row gather)
// Consumers touch every row (one LDS.128 per 16-B quad) so stages are really
// consumed before release.  Prints achieved GB/s of row bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1905_13746_b200/csrc \
//        tools/gather_probe.cu -o tools/gather_probe
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>

#include "gnb_device.cuh"

using namespace gnb;

struct Args {
  const uint8_t* x;
  const int* perm;
  int64_t n_rows;
  int row_bytes;   // multiple of 16
  int pitch;       // smem row pitch (bytes)
  int rows;        // rows per tile
  int stages;
  int mode;
  unsigned long long* sink;
};

__global__ void __launch_bounds__(160) probe(Args a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int NW = 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * a.rows * a.pitch);
  uint64_t* empty = full + a.stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t n_tiles = (a.n_rows + a.rows - 1) / a.rows;
  if (warp == NW) {
    int stage = 0;
    uint32_t phase = 0;
    const uint64_t pol = policy_evict_first();
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      mbar_wait(&empty[stage], phase ^ 1);
      const int64_t r0 = t * a.rows;
      const int nr = static_cast<int>(a.n_rows - r0 < a.rows ? a.n_rows - r0 : a.rows);
      uint8_t* dst = smem + stage * a.rows * a.pitch;
      if (a.mode == 0) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[stage], nr * a.row_bytes);
          bulk_load(dst, a.x + r0 * a.row_bytes, nr * a.row_bytes, &full[stage], pol);
        }
      } else {
        if (lane == 0) mbar_expect_tx(&full[stage], nr * a.row_bytes);
        __syncwarp();
        for (int i = lane; i < nr; i += 32) {
          const int64_t src = a.perm[r0 + i];
          bulk_load(dst + i * a.pitch, a.x + src * a.row_bytes, a.row_bytes, &full[stage], pol);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[stage]);
      }
      if (++stage == a.stages) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else {
    int stage = 0;
    uint32_t phase = 0;
    unsigned long long acc = 0;
    const int pitch = a.mode == 0 ? a.row_bytes : a.pitch;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      mbar_wait(&full[stage], phase);
      const uint8_t* src = smem + stage * a.rows * a.pitch;
      for (int r = threadIdx.x; r < a.rows; r += NW * 32) {
        const uint8_t* row = src + r * pitch;
        for (int q = 0; q < a.row_bytes / 16; ++q) {
          const uint4 v = *reinterpret_cast<const uint4*>(row + 16 * q);
          acc += v.x ^ v.w;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == a.stages) {
        stage = 0;
        phase ^= 1;
      }
    }
    if (acc == 0x123456789ull) *a.sink = acc;
  }
}

int main(int argc, char** argv) {
  const int64_t n = 4194304;
  const int row_bytes = argc > 1 ? atoi(argv[1]) : 800;
  const int groups = 32;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* x;
  int *perm_sorted, *perm_id;
  unsigned long long* sink;
  cudaMalloc(&x, n * row_bytes);
  cudaMemset(x, 1, n * row_bytes);
  cudaMalloc(&perm_sorted, n * 4);
  cudaMalloc(&perm_id, n * 4);
  cudaMalloc(&sink, 8);
  // shuffled ragged batch (group g has weight 0.9^g), then a stable counting
  // sort by group: the perm the slot sort produces
  std::mt19937_64 rng(1);
  std::vector<double> w(groups);
  for (int g = 0; g < groups; ++g) w[g] = std::pow(0.9, g);
  std::discrete_distribution<int> pick(w.begin(), w.end());
  std::vector<int> grp(n);
  for (auto& g : grp) g = pick(rng);
  std::vector<int> ps;
  ps.reserve(n);
  for (int g = 0; g < groups; ++g)
    for (int64_t i = 0; i < n; ++i)
      if (grp[i] == g) ps.push_back(static_cast<int>(i));
  std::vector<int> pid(n);
  for (int64_t i = 0; i < n; ++i) pid[i] = static_cast<int>(i);
  cudaMemcpy(perm_sorted, ps.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(perm_id, pid.data(), n * 4, cudaMemcpyHostToDevice);
  uint8_t* flush;
  cudaMalloc(&flush, 512 << 20);

  struct Cfg { int mode, rows, stages, ctas; const char* perm; };
  std::vector<Cfg> cfgs;
  for (int rows : {32, 64, 128})
    for (int stages : {2, 3, 4})
      for (int ctas : {1, 2, 3, 4, 6}) {
        cfgs.push_back({1, rows, stages, ctas, "sorted"});
      }
  cfgs.push_back({0, 128, 2, 6, "contig"});
  cfgs.push_back({0, 64, 3, 4, "contig"});
  cfgs.push_back({1, 64, 3, 3, "identity"});
  for (const Cfg& c : cfgs) {
    const int pitch = ((row_bytes / 16) | 1) * 16;
    const size_t smem = size_t(c.stages) * c.rows * pitch + 2 * c.stages * 8;
    if (smem * c.ctas > 227 * 1024) continue;
    if (cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024))
      return 1;
    Args a{x, strcmp(c.perm, "identity") == 0 ? perm_id : perm_sorted, n, row_bytes, pitch,
           c.rows, c.stages, c.mode, sink};
    const int grid = sms * c.ctas;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f, sum = 0;
    const int reps = 6;
    for (int it = 0; it < reps + 1; ++it) {
      cudaMemset(flush, it, 512 << 20);
      cudaEventRecord(e0);
      probe<<<grid, 160, smem>>>(a);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it) {
        best = std::min(best, ms);
        sum += ms;
      }
    }
    cudaError_t err = cudaGetLastError();
    printf("{\"mode\": \"%s\", \"row_bytes\": %d, \"rows\": %d, \"stages\": %d, \"ctas_per_sm\": %d, "
           "\"smem\": %zu, \"mean_ms\": %.4f, \"gbs\": %.1f, \"err\": \"%s\"}\n",
           c.mode == 0 ? "contig_tile" : c.perm, row_bytes, c.rows, c.stages, c.ctas, smem,
           sum / reps, double(n) * row_bytes / (sum / reps / 1e3) / 1e9, cudaGetErrorString(err));
  }
  return 0;
}
