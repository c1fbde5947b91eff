// K-FIT: per-(size group, class, column) sufficient statistics on sm_100a.
//
// Replaces the count loops of features.class_frequency
// (pkg/src/groupnb/features.py:48-53), classifier.train_group
// (pkg/src/groupnb/classifier.py:94-101) and the per-class sample counts of
// corpus.trainable_groups (pkg/src/groupnb/corpus.py:302-305).
//
// Segmented reduction keyed by key = group * C + label:
//   * X [N, V] is streamed once by TMA in boxes of 32 columns x 64 rows
//     (no swizzle: a warp reads one 128-B box row per step, conflict-free).  Column chunk c of every tile goes to consumer warp
//     c mod NW, so a warp always owns the same columns and its shared-memory
//     partials need no atomics.
//   * the producer warp routes the tile's rows (size -> group, label ->
//     class), drops out-of-range / unlabeled rows, and groups the rest by key
//     with warp ballots (a counting sort without a histogram).  It publishes
//     the permutation and the key runs with every stage.
//   * a consumer lane owns one column: for each key run it accumulates
//     sum x and sum x^2 in 64-bit integer registers (IMAD.WIDE, no FP64),
//     then adds the run into the CTA's shared partial [key][col].  Integer
//     arithmetic is exact and associative, so the result does not depend on
//     the tiling, the grid, or how rows are sharded across GPUs.
//   * at exit every CTA adds its partials into the fp64 outputs with
//     RED.ADD.F64 (exact: integer values < 2^53).
#include <cstdint>

#include "gnb_device.cuh"
#include "gnb_internal.h"

namespace gnb {

constexpr int kFitRows = 64;  // rows per tile (u8 permutation)
constexpr int kFitSPW = 3;    // ring stages per consumer warp

struct FitHdr {
  int n_runs;
  int pad[3];
  uint8_t perm[kFitRows];
  int2 runs[kFitRows];  // {key, start | len << 16}
};

template <int NW>
struct FitSmem {
  static constexpr int kBox = kFitRows * kChunkBytesPerRow;  // 8 KB
  static constexpr int kStages = NW * kFitSPW;
  static constexpr int kX = 0;
  static constexpr int kHdr = kX + kStages * kBox;
  static constexpr int kScratch = kHdr + kStages * static_cast<int>(sizeof(FitHdr));
  static constexpr int kBar = kScratch + static_cast<int>(sizeof(FitHdr));
  static constexpr int kPart = kBar + 2 * kStages * 8;  // 8-B aligned
  static constexpr int kFixed = kPart + 1024;           // + alignment slack
};

template <int NW>
__global__ void __launch_bounds__((NW + 1) * 32)
    fit_tma_kernel(const __grid_constant__ CUtensorMap xmap, const FitParams p) {
  using L = FitSmem<NW>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for SWIZZLE_128B, keeping the pointer in the shared window
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* empty = full + L::kStages;
  const int Fp = p.n_chunks * kChunkCols;
  const int KS = p.smem_keys;
  unsigned long long* part_s = reinterpret_cast<unsigned long long*>(smem + L::kPart);
  unsigned long long* part_q = part_s + static_cast<int64_t>(KS) * Fp;  // if sumsq
  unsigned long long* part_n = part_q + (p.sumsq ? static_cast<int64_t>(KS) * Fp : 0);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nthreads = blockDim.x;
  const int64_t part_words = static_cast<int64_t>(KS) * Fp * (p.sumsq ? 2 : 1) + KS;
  for (int64_t i = threadIdx.x; i < part_words; i += nthreads) part_s[i] = 0ull;
  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int NCH = p.n_chunks;
  if (warp == NW) {
    // ------------------------------------------------------------ producer
    const uint64_t pol_x = policy_evict_first();
    FitHdr* scratch = reinterpret_cast<FitHdr*>(smem + L::kScratch);
    int stage_of[NW];
    uint32_t phase_of[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      stage_of[w] = 0;
      phase_of[w] = 0;
    }
    unsigned long long bad_label = 0, out_of_range = 0;
    const uint32_t lt = (1u << lane) - 1u;
    for (int64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
      const int64_t r0 = tile * kFitRows;
      int key[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int64_t r = r0 + lane + 32 * i;
        key[i] = -1;
        if (r < p.n_rows) {
          const int sz = __ldg(p.size + r);
          if (sz >= 0 && sz < p.limit) {
            const int lab = __ldg(p.labels + r);
            if (lab >= 0 && lab < p.n_classes)
              key[i] = (sz / p.width) * p.n_classes + lab;
            else
              ++bad_label;
          } else {
            ++out_of_range;
          }
        }
      }
      // group rows by key: repeatedly take the first remaining row's key
      uint32_t rem0 = __ballot_sync(~0u, key[0] >= 0);
      uint32_t rem1 = __ballot_sync(~0u, key[1] >= 0);
      int pos = 0, n_runs = 0;
      while (rem0 | rem1) {
        const int src = rem0 ? __ffs(rem0) - 1 : __ffs(rem1) - 1;
        const int k = rem0 ? __shfl_sync(~0u, key[0], src) : __shfl_sync(~0u, key[1], src);
        const uint32_t m0 = __ballot_sync(~0u, key[0] == k) & rem0;
        const uint32_t m1 = __ballot_sync(~0u, key[1] == k) & rem1;
        const int c0 = __popc(m0), len = c0 + __popc(m1);
        if (m0 & (1u << lane)) scratch->perm[pos + __popc(m0 & lt)] = static_cast<uint8_t>(lane);
        if (m1 & (1u << lane))
          scratch->perm[pos + c0 + __popc(m1 & lt)] = static_cast<uint8_t>(lane + 32);
        if (lane == 0) {
          scratch->runs[n_runs] = make_int2(k, pos | (len << 16));
          if (k < KS) part_n[k] += static_cast<unsigned long long>(len);
          else atomicAdd(p.counts + k, static_cast<double>(len));
        }
        pos += len;
        ++n_runs;
        rem0 &= ~m0;
        rem1 &= ~m1;
      }
      __syncwarp();
      // copy perm + runs, then ship each column chunk to its owner warp
      const int hdr_words = (16 + kFitRows + n_runs * 8 + 15) / 16;  // 16-B units
      for (int ch = 0; ch < NCH; ++ch) {
        const int w = ch % NW;
        const int st = w * kFitSPW + stage_of[w];
        mbar_wait(&empty[st], phase_of[w] ^ 1);
        FitHdr* hdr = reinterpret_cast<FitHdr*>(smem + L::kHdr + st * sizeof(FitHdr));
        const int4* src4 = reinterpret_cast<const int4*>(scratch);
        int4* dst4 = reinterpret_cast<int4*>(hdr);
        for (int i = lane; i < hdr_words; i += 32) dst4[i] = src4[i];
        if (lane == 0) hdr->n_runs = n_runs;
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[st], L::kBox);
          tma_load_2d(smem + L::kX + st * L::kBox, &xmap, ch * kChunkCols,
                      static_cast<int32_t>(r0), &full[st], pol_x);
        } else {
          mbar_arrive(&full[st]);
        }
        if (++stage_of[w] == kFitSPW) {
          stage_of[w] = 0;
          phase_of[w] ^= 1;
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      bad_label += __shfl_xor_sync(~0u, bad_label, o);
      out_of_range += __shfl_xor_sync(~0u, out_of_range, o);
    }
    if (lane == 0 && p.status != nullptr) {
      if (bad_label) atomicAdd(p.status + 0, bad_label);
      if (out_of_range) atomicAdd(p.status + 1, out_of_range);
    }
  } else {
    // ------------------------------------------------------------ consumers
    const uint32_t lane4 = static_cast<uint32_t>(lane) * 4u;  // unswizzled box: row r at r*128
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
      for (int ch = warp; ch < NCH; ch += NW) {
        const int st = warp * kFitSPW + stage;
        mbar_wait(&full[st], phase);
        const FitHdr* hdr = reinterpret_cast<const FitHdr*>(smem + L::kHdr + st * sizeof(FitHdr));
        const uint8_t* box = smem + L::kX + st * L::kBox;
        const int col = ch * kChunkCols + lane;
        const int n_runs = hdr->n_runs;
        for (int ri = 0; ri < n_runs; ++ri) {
          const int2 run = hdr->runs[ri];
          const int start = run.y & 0xffff, len = run.y >> 16;
          unsigned long long s = 0, s2 = 0;
          int i = 0;
          for (; i + 4 <= len; i += 4) {
            uint32_t x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const uint32_t r = hdr->perm[start + i + u];
              x[u] = *reinterpret_cast<const uint32_t*>(box + (r << 7) + lane4);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              s += x[u];
              s2 += static_cast<unsigned long long>(x[u]) * x[u];
            }
          }
          for (; i < len; ++i) {
            const uint32_t r = hdr->perm[start + i];
            const uint32_t x = *reinterpret_cast<const uint32_t*>(box + (r << 7) + lane4);
            s += x;
            s2 += static_cast<unsigned long long>(x) * x;
          }
          const int k = run.x;
          if (k < KS) {
            part_s[static_cast<int64_t>(k) * Fp + col] += s;
            if (p.sumsq) part_q[static_cast<int64_t>(k) * Fp + col] += s2;
          } else if (col < p.n_cols) {
            if (s) atomicAdd(p.sums + static_cast<int64_t>(k) * p.n_cols + col, static_cast<double>(s));
            if (p.sumsq && s2)
              atomicAdd(p.sumsq + static_cast<int64_t>(k) * p.n_cols + col, static_cast<double>(s2));
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (++stage == kFitSPW) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  }
  __syncthreads();
  // ------------------------------------------------------------ flush partials
  for (int64_t i = threadIdx.x; i < static_cast<int64_t>(KS) * Fp; i += nthreads) {
    const int k = static_cast<int>(i / Fp), col = static_cast<int>(i % Fp);
    if (col >= p.n_cols) continue;
    const int64_t o = static_cast<int64_t>(k) * p.n_cols + col;
    if (part_s[i]) atomicAdd(p.sums + o, static_cast<double>(part_s[i]));
    if (p.sumsq && part_q[i]) atomicAdd(p.sumsq + o, static_cast<double>(part_q[i]));
  }
  for (int k = threadIdx.x; k < KS; k += nthreads)
    if (part_n[k]) atomicAdd(p.counts + k, static_cast<double>(part_n[k]));
}

template <int NW>
static cudaError_t launch_fit(const CUtensorMap& map, FitParams p, cudaStream_t stream) {
  using L = FitSmem<NW>;
  auto kern = fit_tma_kernel<NW>;
  int dev = 0, sms = 0, max_smem = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int Fp = p.n_chunks * kChunkCols;
  const int per_key = Fp * 8 * (p.sumsq ? 2 : 1) + 8;
  // keep partials modest so two CTAs fit per SM when keys are few
  const int budget = max_smem - L::kFixed;
  int ks = budget / per_key;
  if (ks > p.n_keys) ks = p.n_keys;
  if (ks < 0) ks = 0;
  p.smem_keys = ks;
  const int smem = L::kFixed + ks * per_key;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (NW + 1) * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t want = static_cast<int64_t>(sms) * per_sm;
  const int grid = static_cast<int>(p.n_tiles < want ? p.n_tiles : want);
  if (grid == 0) return cudaSuccess;
  kern<<<grid, (NW + 1) * 32, smem, stream>>>(map, p);
  return cudaGetLastError();
}

cudaError_t fit_launch(const CUtensorMap& map, FitParams p, cudaStream_t stream) {
  p.n_chunks = (p.n_cols + kChunkCols - 1) / kChunkCols;
  p.n_tiles = (p.n_rows + kFitRows - 1) / kFitRows;
  if (p.n_chunks >= 4) return launch_fit<4>(map, p, stream);
  if (p.n_chunks >= 2) return launch_fit<2>(map, p, stream);
  return launch_fit<1>(map, p, stream);
}

}  // namespace gnb
