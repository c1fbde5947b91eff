// K-FIT: per-(size group, class, column) sufficient statistics on sm_100a.
//
// Replaces the count loops of features.class_frequency
// (pkg/src/groupnb/features.py:48-53), classifier.train_group
// (pkg/src/groupnb/classifier.py:94-101) and the per-class sample counts of
// corpus.trainable_groups (pkg/src/groupnb/corpus.py:302-305).
//
// Segmented reduction keyed by key = group * C + label:
//   * X [N, V] is streamed once by TMA.  A stage is one tile of kFitRows rows
//     x one 64-column group (two 32-column boxes, unswizzled), so a warp reads
//     a whole 256-B row segment per step: lane l owns columns 2l, 2l+1 (one
//     LDS.64, conflict-free per half warp).
//   * the producer warp routes the tile's rows (size -> group, label ->
//     class), drops out-of-range / unlabeled rows, and counting-sorts the rest
//     by key through a shared histogram (match_any leaders reserve places for
//     their lanes).  The next tile's sizes/labels are prefetched while the
//     current one sorts.  It publishes the permutation and the key runs with
//     every stage.
//   * every consumer warp reads every stage but only accumulates the runs of
//     the keys it owns (key mod NW == warp), so its shared-memory partials
//     [key][column] are private to it: no atomics, no replicas.  Within a run
//     the sums of x and x^2 stay in 64-bit integer registers (IMAD.WIDE, no
//     FP64); the run is then added into the partial (one read-modify-write
//     per run, not per row).  Integer arithmetic is exact and associative, so
//     the result does not depend on tiling, grid, or GPU sharding.
//   * at exit every CTA adds its partials into the fp64 outputs with
//     RED.ADD.F64 (exact: integer values < 2^53).  Keys beyond the shared
//     memory capacity go straight to global RED per run.
#include <climits>
#include <cstdint>
#include <cstdlib>

#include "gnb_device.cuh"
#include "gnb_internal.h"

namespace gnb {

constexpr int kMaxHistKeys = 4096;   // keys sorted by the shared-memory histogram

// Stage geometry per X storage: a lane owns CPL consecutive columns.
//   int32 : 2 boxes x 32 columns = 64 columns, CPL 2 (LDS.64)
//   uint16: 1 box  x 64 columns  = 64 columns, CPL 2 (LDS.32)
//   uint8 : 1 box  x 128 columns = 128 columns, CPL 4 (LDS.32)
template <typename T, int BX = (sizeof(T) == 4 ? 2 : 1)>
struct FitGeom {
  // rows per tile (u8 permutation).  256-row tiles for narrow rows were
  // measured slower (fewer CTAs per SM), profiles/r01_tuning.md.
  static constexpr int kRows = 128;
  static constexpr int kBoxCols = kChunkBytesPerRow / static_cast<int>(sizeof(T));
  static constexpr int kBoxes = BX;
  static constexpr int kGroupCols = kBoxCols * kBoxes;
  static constexpr int kCPL = kGroupCols / 32;
  static constexpr int kLaneBytes = kCPL * static_cast<int>(sizeof(T));
};

template <int ROWS>
struct FitHdr {
  int n_runs;
  int pad[3];
  uint8_t perm[ROWS];
  int2 runs[ROWS];  // {key, start | len << 16}
};

template <typename T, int NW, int STAGES, int BX, int NP = 1>
struct FitSmem {
  using Geo = FitGeom<T, BX>;
  using Hdr = FitHdr<Geo::kRows>;
  static constexpr int kBox = Geo::kRows * kChunkBytesPerRow;  // 16 KB
  static constexpr int kStage = Geo::kBoxes * kBox;             // 16 / 32 KB
  static constexpr int kX = 0;
  static constexpr int kHdr = kX + STAGES * kStage;
  static constexpr int kScratch = kHdr + STAGES * static_cast<int>(sizeof(Hdr));
  static constexpr int kBar = kScratch + NP * static_cast<int>(sizeof(Hdr));
  static constexpr int kPart = (kBar + 2 * STAGES * 8 + 15) / 16 * 16;
  static constexpr int kFixed = kPart + 1024;  // + alignment slack
};

__device__ __forceinline__ void add_u64x2(unsigned long long* p, unsigned long long a,
                                          unsigned long long b) {
  ulonglong2 v = *reinterpret_cast<ulonglong2*>(p);
  v.x += a;
  v.y += b;
  *reinterpret_cast<ulonglong2*>(p) = v;
}

// the CPL columns of a lane's slice of one box row
template <typename T, int CPL>
__device__ __forceinline__ void load_lane(const uint8_t* at, uint32_t (&x)[CPL]) {
  constexpr int bytes = CPL * static_cast<int>(sizeof(T));
  uint32_t w[bytes / 4];
  if constexpr (bytes == 4) {
    w[0] = *reinterpret_cast<const uint32_t*>(at);
  } else if constexpr (bytes == 8) {
    const uint2 v = *reinterpret_cast<const uint2*>(at);
    w[0] = v.x;
    w[1] = v.y;
  } else {
    const uint4 v = *reinterpret_cast<const uint4*>(at);
    w[0] = v.x;
    w[1] = v.y;
    w[2] = v.z;
    w[3] = v.w;
  }
#pragma unroll
  for (int e = 0; e < CPL; ++e) {
    if constexpr (sizeof(T) == 4) {
      x[e] = w[e];
    } else {
      constexpr int per = 4 / static_cast<int>(sizeof(T));
      constexpr uint32_t mask = sizeof(T) == 2 ? 0xffffu : 0xffu;
      x[e] = (w[e / per] >> (8 * sizeof(T) * (e % per))) & mask;
    }
  }
}

// NP producer warps (1 or 2) sort alternate tiles; their latency-bound sorts
// overlap, and a pair of named barriers keeps the stage issue in tile order
// (mbarrier parity waits must never run two phases ahead).
__device__ __forceinline__ void named_sync(int id) {
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}
__device__ __forceinline__ void named_arrive(int id) {
  asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory");
}

template <typename T, int NW, int STAGES, int BX, int NP>
__global__ void __launch_bounds__((NW + NP) * 32, 2)
    fit_tma_kernel(const __grid_constant__ CUtensorMap xmap, const FitParams p) {
  using L = FitSmem<T, NW, STAGES, BX, NP>;
  using Geo = typename L::Geo;
  using FitHdrT = typename L::Hdr;
  constexpr int kGroupCols = Geo::kGroupCols;
  constexpr int CPL = Geo::kCPL;
  constexpr int kFitRows = Geo::kRows;
  constexpr int kKeysPerLane = kFitRows / 32;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* empty = full + STAGES;
  const int NG = p.n_chunks;         // column groups of kGroupCols
  const int Vp = NG * kGroupCols;
  const int KS = p.smem_keys;
  unsigned long long* part_s = reinterpret_cast<unsigned long long*>(smem + L::kPart);
  unsigned long long* part_q = part_s + static_cast<int64_t>(KS) * Vp;  // if sumsq
  unsigned long long* part_n = part_q + (p.sumsq ? static_cast<int64_t>(KS) * Vp : 0);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nthreads = blockDim.x;
  const int64_t part_words = static_cast<int64_t>(KS) * Vp * (p.sumsq ? 2 : 1) + KS;
  for (int64_t i = threadIdx.x; i < part_words; i += nthreads) part_s[i] = 0ull;
  // histogram sort scratch after the partials: per producer hist[HK], kstart[HK]
  const int HK = p.n_keys <= kMaxHistKeys ? p.n_keys : 0;
  const int pid = warp >= NW ? warp - NW : 0;
  int* hist = reinterpret_cast<int*>(part_n + KS) + pid * 2 * HK;
  int* kstart = hist + HK;
  for (int i = threadIdx.x; i < NP * 2 * HK; i += nthreads)
    reinterpret_cast<int*>(part_n + KS)[i] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], NW);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp >= NW) {
    // ------------------------------------------------------------ producer(s)
    const uint64_t pol_x = policy_evict_normal();
    FitHdrT* scratch = reinterpret_cast<FitHdrT*>(smem + L::kScratch + pid * sizeof(FitHdrT));
    const int64_t my_iters =
        blockIdx.x < p.n_tiles ? (p.n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    unsigned long long bad_label = 0, out_of_range = 0;
    const uint32_t lt = (1u << lane) - 1u;
    const bool hist_sort = HK > 0;
    // Sizes/labels of the NEXT tile are loaded while this tile sorts; they are
    // only turned into keys (and status counts) one iteration later, so the
    // global-load latency never stalls the producer.
    auto load_raw = [&](int64_t tile, int (&sz)[kKeysPerLane], int (&lab)[kKeysPerLane]) {
#pragma unroll
      for (int i = 0; i < kKeysPerLane; ++i) {
        const int64_t r = tile * kFitRows + lane + 32 * i;
        const bool in = tile < p.n_tiles && r < p.n_rows;
        sz[i] = in ? __ldg(p.size + r) : INT_MIN;  // INT_MIN: no row
        lab[i] = in ? __ldg(p.labels + r) : 0;
      }
    };
    int nsz[kKeysPerLane], nlab[kKeysPerLane];
    load_raw(blockIdx.x + int64_t(pid) * gridDim.x, nsz, nlab);
    for (int64_t it = pid; it < my_iters; it += NP) {
      const int64_t tile = blockIdx.x + it * gridDim.x;
      const int64_t r0 = tile * kFitRows;
      int key[kKeysPerLane];
#pragma unroll
      for (int i = 0; i < kKeysPerLane; ++i) {
        const int sz = nsz[i], lab = nlab[i];
        key[i] = -1;
        if (sz == INT_MIN) continue;
        if (sz >= 0 && sz < p.limit) {
          if (lab >= 0 && lab < p.n_classes)
            key[i] = (sz / p.width) * p.n_classes + lab;
          else
            ++bad_label;
        } else {
          ++out_of_range;
        }
      }
      load_raw(tile + int64_t(NP) * gridDim.x, nsz, nlab);  // prefetch
      int n_runs = 0;
      if (hist_sort) {
        // counting sort through a shared histogram: per key slot, lanes with
        // equal keys elect a leader that reserves popc(lanes) places at once
        int rank[kKeysPerLane];
        uint32_t mine = 0;  // bit i: this lane's slot-i key is new in the tile
#pragma unroll
        for (int i = 0; i < kKeysPerLane; ++i) {
          const uint32_t m = __match_any_sync(~0u, key[i]);
          const int leader = __ffs(m) - 1;
          int base = 0;
          if (key[i] >= 0 && lane == leader) base = atomicAdd(&hist[key[i]], __popc(m));
          base = __shfl_sync(~0u, base, leader);
          rank[i] = base + __popc(m & lt);
          if (key[i] >= 0 && lane == leader && base == 0) mine |= 1u << i;
        }
        __syncwarp();
        // list the tile's keys, exclusive-scan their counts into run starts
        int cnt[kKeysPerLane], kk[kKeysPerLane];
        int total = 0;
#pragma unroll
        for (int i = 0; i < kKeysPerLane; ++i) {
          const bool is_new = (mine >> i) & 1u;
          const uint32_t b = __ballot_sync(~0u, is_new);
          const int slot = n_runs + __popc(b & lt);
          kk[i] = is_new ? key[i] : -1;
          cnt[i] = is_new ? hist[key[i]] : 0;
          // inclusive warp scan of cnt[i] in run order (slot order)
          int v = cnt[i];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(~0u, v, o);
            if (lane >= o) v += t;
          }
          const int start = total + v - cnt[i];
          if (is_new) {
            kstart[key[i]] = start;
            scratch->runs[slot] = make_int2(key[i], start | (cnt[i] << 16));
          }
          total += __shfl_sync(~0u, v, 31);
          n_runs += __popc(b);
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < kKeysPerLane; ++i)
          if (key[i] >= 0)
            scratch->perm[kstart[key[i]] + rank[i]] = static_cast<uint8_t>(lane + 32 * i);
        // counts + reset the histogram entries this tile touched
#pragma unroll
        for (int i = 0; i < kKeysPerLane; ++i) {
          if (kk[i] >= 0) {
            if (kk[i] < KS) {
              if (NP == 1) part_n[kk[i]] += static_cast<unsigned long long>(cnt[i]);
              else atomicAdd(part_n + kk[i], static_cast<unsigned long long>(cnt[i]));
            } else {
              atomicAdd(p.counts + kk[i], static_cast<double>(cnt[i]));
            }
            hist[kk[i]] = 0;
          }
        }
      } else {
        // huge key spaces: take the first remaining row's key, ballot its rows
        uint32_t rem[kKeysPerLane];
#pragma unroll
        for (int i = 0; i < kKeysPerLane; ++i) rem[i] = __ballot_sync(~0u, key[i] >= 0);
        int pos = 0;
        while (true) {
          int src_i = -1;
#pragma unroll
          for (int i = kKeysPerLane - 1; i >= 0; --i)
            if (rem[i]) src_i = i;
          if (src_i < 0) break;
          int k = 0;
#pragma unroll
          for (int i = 0; i < kKeysPerLane; ++i)
            if (i == src_i) k = __shfl_sync(~0u, key[i], __ffs(rem[i]) - 1);
          int len = 0;
#pragma unroll
          for (int i = 0; i < kKeysPerLane; ++i) {
            const uint32_t m = __ballot_sync(~0u, key[i] == k) & rem[i];
            if (m & (1u << lane))
              scratch->perm[pos + len + __popc(m & lt)] = static_cast<uint8_t>(lane + 32 * i);
            len += __popc(m);
            rem[i] &= ~m;
          }
          if (lane == 0) {
            scratch->runs[n_runs] = make_int2(k, pos | (len << 16));
            if (k < KS) {
              if (NP == 1) part_n[k] += static_cast<unsigned long long>(len);
              else atomicAdd(part_n + k, static_cast<unsigned long long>(len));
            } else {
              atomicAdd(p.counts + k, static_cast<double>(len));
            }
          }
          pos += len;
          ++n_runs;
        }
      }
      __syncwarp();
      const int hdr_words = (16 + kFitRows + n_runs * 8 + 15) / 16;  // 16-B units
      if (NP > 1 && it > 0) named_sync(1 + ((it - 1) & 1));  // tile it-1 issued
      int64_t g = it * NG;  // global stage sequence number of this tile's first chunk
      for (int cg = 0; cg < NG; ++cg, ++g) {
        const int stage = static_cast<int>(g % STAGES);
        const uint32_t phase = static_cast<uint32_t>(g / STAGES) & 1u;
        mbar_wait(&empty[stage], phase ^ 1);
        FitHdrT* hdr = reinterpret_cast<FitHdrT*>(smem + L::kHdr + stage * sizeof(FitHdrT));
        const int4* src4 = reinterpret_cast<const int4*>(scratch);
        int4* dst4 = reinterpret_cast<int4*>(hdr);
        for (int i = lane; i < hdr_words; i += 32) dst4[i] = src4[i];
        if (lane == 0) hdr->n_runs = n_runs;
        __syncwarp();
        if (lane == 0) {
          const int boxes = min(Geo::kBoxes, (p.n_cols - cg * kGroupCols + Geo::kBoxCols - 1) /
                                                 Geo::kBoxCols);
          mbar_arrive_expect_tx(&full[stage], boxes * L::kBox);
          for (int b = 0; b < boxes; ++b)
            tma_load_2d(smem + L::kX + stage * L::kStage + b * L::kBox, &xmap,
                        cg * kGroupCols + b * Geo::kBoxCols, static_cast<int32_t>(r0),
                        &full[stage], pol_x);
        } else {
          mbar_arrive(&full[stage]);
        }
      }
      __syncwarp();
      if (NP > 1 && it + 1 < my_iters) named_arrive(1 + (it & 1));
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
    // lane owns columns CPL*lane .. CPL*lane+CPL-1 of the group
    const uint32_t lane_byte = static_cast<uint32_t>(lane) * Geo::kLaneBytes;
    const uint32_t lane_off = (lane_byte / kChunkBytesPerRow) * L::kBox + lane_byte % kChunkBytesPerRow;
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
      for (int cg = 0; cg < NG; ++cg) {
        mbar_wait(&full[stage], phase);
        const FitHdrT* hdr =
            reinterpret_cast<const FitHdrT*>(smem + L::kHdr + stage * sizeof(FitHdrT));
        const uint8_t* xs = smem + L::kX + stage * L::kStage + lane_off;
        const int col0 = cg * kGroupCols + CPL * lane;
        const int n_runs = hdr->n_runs;
        for (int rb = 0; rb < n_runs; rb += 32) {
          // lane j holds run rb+j; the warp walks only the runs of its keys
          int2 mine = make_int2(-1, 0);
          if (rb + lane < n_runs) mine = hdr->runs[rb + lane];
          uint32_t todo = __ballot_sync(~0u, mine.x >= 0 && mine.x % NW == warp);
          while (todo) {
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            const int k = __shfl_sync(~0u, mine.x, j);
            const int packed = __shfl_sync(~0u, mine.y, j);
            const int start = packed & 0xffff, len = packed >> 16;
            unsigned long long sa[CPL], qa[CPL];
#pragma unroll
            for (int e = 0; e < CPL; ++e) sa[e] = qa[e] = 0;
            int i = 0;
            for (; i + 4 <= len; i += 4) {
              uint32_t v[4][CPL];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const uint32_t r = hdr->perm[start + i + u];
                load_lane<T, CPL>(xs + (r << 7), v[u]);
              }
#pragma unroll
              for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int e = 0; e < CPL; ++e) {
                  sa[e] += v[u][e];
                  qa[e] += static_cast<unsigned long long>(v[u][e]) * v[u][e];
                }
            }
            for (; i < len; ++i) {
              uint32_t v[CPL];
              load_lane<T, CPL>(xs + (static_cast<uint32_t>(hdr->perm[start + i]) << 7), v);
#pragma unroll
              for (int e = 0; e < CPL; ++e) {
                sa[e] += v[e];
                qa[e] += static_cast<unsigned long long>(v[e]) * v[e];
              }
            }
            if (k < KS) {
              if constexpr (CPL == 1) {
                part_s[static_cast<int64_t>(k) * Vp + col0] += sa[0];
                if (p.sumsq) part_q[static_cast<int64_t>(k) * Vp + col0] += qa[0];
              } else {
#pragma unroll
                for (int e = 0; e < CPL; e += 2) {
                  add_u64x2(part_s + static_cast<int64_t>(k) * Vp + col0 + e, sa[e], sa[e + 1]);
                  if (p.sumsq)
                    add_u64x2(part_q + static_cast<int64_t>(k) * Vp + col0 + e, qa[e], qa[e + 1]);
                }
              }
            } else {
#pragma unroll
              for (int e = 0; e < CPL; ++e) {
                if (col0 + e >= p.n_cols) break;
                const int64_t o = static_cast<int64_t>(k) * p.n_cols + col0 + e;
                if (sa[e]) atomicAdd(p.sums + o, static_cast<double>(sa[e]));
                if (p.sumsq && qa[e]) atomicAdd(p.sumsq + o, static_cast<double>(qa[e]));
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  }
  __syncthreads();
  // ------------------------------------------------------------ flush partials
  for (int64_t i = threadIdx.x; i < static_cast<int64_t>(KS) * Vp; i += nthreads) {
    const int k = static_cast<int>(i / Vp), col = static_cast<int>(i % Vp);
    if (col >= p.n_cols) continue;
    const int64_t o = static_cast<int64_t>(k) * p.n_cols + col;
    if (part_s[i]) atomicAdd(p.sums + o, static_cast<double>(part_s[i]));
    if (p.sumsq && part_q[i]) atomicAdd(p.sumsq + o, static_cast<double>(part_q[i]));
  }
  for (int k = threadIdx.x; k < KS; k += nthreads)
    if (part_n[k]) atomicAdd(p.counts + k, static_cast<double>(part_n[k]));
}

template <typename T, int NW, int STAGES, int BX, int NP>
static cudaError_t launch_fit_np(const CUtensorMap& map, FitParams p, cudaStream_t stream,
                                 int ctas_per_sm) {
  using L = FitSmem<T, NW, STAGES, BX, NP>;
  auto kern = fit_tma_kernel<T, NW, STAGES, BX, NP>;
  constexpr int kGroupCols = L::Geo::kGroupCols;
  p.n_chunks = (p.n_cols + kGroupCols - 1) / kGroupCols;
  int dev = 0, sms = 0, max_smem = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int Vp = p.n_chunks * kGroupCols;
  const int per_key = Vp * 8 * (p.sumsq ? 2 : 1) + 8;
  const int hist_bytes = p.n_keys <= kMaxHistKeys ? 8 * NP * p.n_keys : 0;
  // Partials sized so `ctas_per_sm` CTAs share an SM; keys beyond the cap
  // (large group counts) accumulate per run in global memory.
  const int budget = (max_smem + 1024) / ctas_per_sm - 1024 - L::kFixed - hist_bytes;
  int ks = budget > 0 ? budget / per_key : 0;
  if (ks < 1) ks = (max_smem - L::kFixed - hist_bytes) / per_key;
  if (ks > p.n_keys) ks = p.n_keys;
  if (ks < 0) ks = 0;
  p.smem_keys = ks;
  const int smem = L::kFixed + ks * per_key + hist_bytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (NW + NP) * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t want = static_cast<int64_t>(sms) * per_sm;
  const int grid = static_cast<int>(p.n_tiles < want ? p.n_tiles : want);
  if (grid == 0) return cudaSuccess;
  kern<<<grid, (NW + NP) * 32, smem, stream>>>(map, p);
  return cudaGetLastError();
}

// Producer warps per CTA: 2 unless GNB_FIT_NP=1 (A/B).  One producer warp's
// sort is a latency-bound dependent chain (~7k cycles per 128-row tile under
// load) that capped K-FIT at ~85 % of HBM with int32 rows (profiles/).
static int fit_producers() {
  static const int v = [] {  // read once (thread-safe static init)
    int v = -1;
    const char* e = getenv("GNB_FIT_NP");
    v = e ? atoi(e) : 2;
    if (v != 1) v = 2;
    return v;
  }();
  return v;
}

template <typename T, int NW, int STAGES, int BX = (sizeof(T) == 4 ? 2 : 1)>
static cudaError_t launch_fit(const CUtensorMap& map, const FitParams& p, cudaStream_t stream,
                              int ctas_per_sm) {
  // large key spaces keep one producer (per-producer histograms double)
  if (fit_producers() == 2 && p.n_keys <= 1024)
    return launch_fit_np<T, NW, STAGES, BX, 2>(map, p, stream, ctas_per_sm);
  return launch_fit_np<T, NW, STAGES, BX, 1>(map, p, stream, ctas_per_sm);
}

int fit_box_rows(int x_type) {
  return x_type == GNB_X_I32 ? FitGeom<int32_t>::kRows : FitGeom<uint8_t>::kRows;
}

// GNB_FIT_VARIANT (profiling only): 0 = 2 stages x 2 CTAs/SM (default; measured
// best on B200, profiles/r01_tuning.md), 1 = 4 stages x 1 CTA/SM,
// 2 = one-box (16 KB) stages x 4 x 2 CTAs/SM, 3 = one-box stages x 3 x 2 CTAs/SM.
static int fit_variant() {
  static const int v = [] {  // read once (thread-safe static init)
    int v = -1;
    const char* e = getenv("GNB_FIT_VARIANT");
    v = e ? atoi(e) : 0;
    if (v < 0 || v > 3) v = 0;
    return v;
  }();
  return v;
}

// CTAs per SM the partial-sum budget is sized for, narrow rows (GNB_FIT_CTAS).
static int narrow_ctas() {
  static const int v = [] {  // read once (thread-safe static init)
    int v = -1;
    const char* e = getenv("GNB_FIT_CTAS");
    v = e ? atoi(e) : 2;
    if (v < 1 || v > 8) v = 2;
    return v;
  }();
  return v;
}

template <typename T, int NW>
static cudaError_t launch_fit_nw(const CUtensorMap& map, const FitParams& p, cudaStream_t stream) {
  switch (fit_variant()) {
    case 1: return launch_fit<T, NW, 4>(map, p, stream, 1);
    case 2: return launch_fit<T, NW, 4, 1>(map, p, stream, 2);  // 16-KB stages, 4 deep
    case 3: return launch_fit<T, NW, 3, 1>(map, p, stream, 2);
    default: return launch_fit<T, NW, 2>(map, p, stream, sizeof(T) == 4 ? 2 : narrow_ctas());
  }
}

template <typename T>
static cudaError_t launch_fit_typed(const CUtensorMap& map, const FitParams& p,
                                   cudaStream_t stream) {
  // keys are dealt to warps round-robin: no more warps than keys
  static const int nw8 = [] {  // read once (thread-safe static init)  // GNB_FIT_NW8=0 disables the 8-consumer-warp CTA (profiling)
    int nw8 = -1;
    const char* e = getenv("GNB_FIT_NW8");
    nw8 = e ? atoi(e) : 1;
    return nw8;
  }();
  // 8 consumer warps pay off for int32 rows (32-KB stages, consumer-bound); for
  // uint8/uint16 tiles the producer's sort is the limit (profiles/r01_tuning.md)
  if ((sizeof(T) == 4 || nw8 == 2) && p.n_keys >= 8 && nw8)  // 2: any storage (A/B)
    return launch_fit_nw<T, 8>(map, p, stream);
  if (p.n_keys >= 4) return launch_fit_nw<T, 4>(map, p, stream);
  if (p.n_keys >= 2) return launch_fit_nw<T, 2>(map, p, stream);
  return launch_fit_nw<T, 1>(map, p, stream);
}

cudaError_t fit_launch(const CUtensorMap& map, FitParams p, cudaStream_t stream) {
  p.n_tiles = (p.n_rows + fit_box_rows(p.x_type) - 1) / fit_box_rows(p.x_type);
  switch (p.x_type) {
    case GNB_X_U16: return launch_fit_typed<uint16_t>(map, p, stream);
    case GNB_X_U8: return launch_fit_typed<uint8_t>(map, p, stream);
    default: return launch_fit_typed<int32_t>(map, p, stream);
  }
}

}  // namespace gnb
