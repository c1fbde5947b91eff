// K-PRED: group-wise Naive Bayes scoring + fused argmax on sm_100a.
//
// Replaces the reference's per-sample loop (pkg/src/groupnb/engine.py:198-205)
// and its kernel classifier.log_posterior / predict
// (pkg/src/groupnb/classifier.py:132-158).
//
// Data path:
//   * X [N, F] counts (int32, or uint16 / uint8 when the counts fit -- the same
//     integers, fewer bytes) are streamed from HBM exactly once by TMA: 2-D
//     boxes of 128 B (32/64/128 features) x ROWS rows, SWIZZLE_128B, through a
//     STAGES-deep mbarrier ring filled by one producer warp.
//   * each consumer thread owns one row and walks its features in FeatureSet
//     order: acc_c = acc_c + x * ll_c as one DMUL (x converted exactly by
//     I2F.F64) and one DADD -- the same two roundings as the reference's
//     `score += n * ll`, so log-posteriors are bit-identical.
//   * the producer routes the tile's rows (size -> group -> slot, the whole
//     route table lookup of engine.py:202) and, when every valid row of the tile
//     shares a slot (G=1, or rows grouped by size group as the reference's
//     GroupedCorpus orders them), also bulk-copies that slot's table slice for
//     the chunk next to the X box, so table reads are smem broadcasts.  Mixed
//     tiles read per-row tables through L1 instead.  All groups: one launch.
//   * argmax (ties -> lowest class index = benign) and the out-of-range status
//     are fused into the epilogue; label (+ optional log-posteriors) written
//     once, coalesced.
//   * persistent CTAs claim tiles dynamically (first tile blockIdx.x, then the
//     next unclaimed index from a per-stream atomic counter; the tile index
//     travels in the stage header, an end-marker stage stops the consumers),
//     so SMs that get less DRAM bandwidth simply take fewer tiles.
//   * kernels: 128-B boxes (predict_tma_kernel, also gather mode for slot-
//     sorted batches), whole-row boxes for short rows (predict_rowbox_kernel),
//     every slot's table resident for batches in any row order
//     (predict_mixed_kernel), and an L1 kernel for any layout.
//
// This header holds the kernels and their launch templates; the translation
// units predict_<storage>_<mode>.cu instantiate launch_typed<T, FMA> (so the
// build compiles them in parallel) and predict.cu holds the dispatch.
#pragma once
#include <atomic>
#include <cfloat>
#include <climits>
#include <cstdint>
#include <cstdlib>

#include "gnb_device.cuh"
#include "gnb_internal.h"

namespace gnb {

// ------------------------------------------------------------------ tables
// packed = [prior: S][CP] | [tab: S][NB][32 features][CP] log-likelihoods.
// NB = ceil(F/32) rounded up to a multiple of 4, so a 128-feature chunk (uint8
// X) of any slot is one in-bounds contiguous block; padding entries are 0.
inline constexpr int kTabBlockFeatures = 32;
inline constexpr int kTabBlockAlign = 4;
int table_blocks(int F);
int class_pad(int C);

// ------------------------------------------------------------------ element types
template <typename T>
struct Elem {
  static constexpr int kPerQuad = 16 / static_cast<int>(sizeof(T));   // per 16-B chunk
  static constexpr int kPerRow = 128 / static_cast<int>(sizeof(T));   // per 128-B box row
  static constexpr bool kSigned = false;
};
template <>
struct Elem<int32_t> {
  static constexpr int kPerQuad = 4, kPerRow = 32;
  static constexpr bool kSigned = true;  // negative counts are flagged, not scored
};

// Element e (0 <= e < kPerQuad) of a 16-B chunk as a double.  The conversion
// is exact (counts < 2^32) and runs on the conversion unit (I2F.F64; for
// uint8/uint16 with a byte/half-word source select), so the product below is
// ONE DMUL rounding, exactly the reference's `n * ll` (a Python float multiply).
// FMA mode on uint8 rows (XU-bound): odd elements are converted on the FP64
// pipe instead, as (2^52 | x) - 2^52 (exact: one PRMT builds the low word, one
// DADD), so I2F and the DFMA chain share the load.
template <typename T, bool FMA = false>
__device__ __forceinline__ double converted(const uint4& v, int e) {
  constexpr int sz = static_cast<int>(sizeof(T));
  const uint32_t w = (e * sz) < 4 ? v.x : (e * sz) < 8 ? v.y : (e * sz) < 12 ? v.z : v.w;
  if constexpr (FMA && sz == 1) {
    if (e & 1)  // half: 3 of 4 measured slower (13.3 vs 13.7 G/s)
      return __dadd_rn(__hiloint2double(0x43300000, static_cast<int>(__byte_perm(w, 0, 0x4440 + (e & 3)))),
                       -4503599627370496.0);
  }
  if constexpr (sz == 4) {
    return __uint2double_rn(w);
  } else {
    // cvt from a .u8/.u16 source of the shifted word: ptxas folds the shift
    // into the I2F byte/half-word selector (I2F.F64.U8 Rx.B1..B3, .U16 Rx.H1),
    // where `(w >> s) & mask` cost a SHF + LOP3 per element before the I2F
    constexpr int bits = 8 * sz;
    const uint32_t s = w >> ((e * bits) & 31);
    double d;
    if constexpr (sz == 1) asm("cvt.rn.f64.u8 %0, %1;" : "=d"(d) : "r"(s));
    else asm("cvt.rn.f64.u16 %0, %1;" : "=d"(d) : "r"(s));
    return d;
  }
}

// ------------------------------------------------------------------ inner loops
// Negative-count flag (int32 rows only).  TMA tensor boxes zero-fill columns
// >= F, but the row-box kernel's 1-D bulk tile copy moves the HBM row pitch
// raw, and callers need not initialise pitch padding: when F is not a
// multiple of 4 the last quad of a row carries padding, and only its first
// (F - 4*(nq-1)) elements may count towards the flag (TAILMASK instances).
struct QuadMask {
  uint32_t y, z, w;
};
__device__ __forceinline__ QuadMask last_quad_mask(int nf) {
  const int rem = nf - ((nf - 1) >> 2) * 4;  // valid int32 elements of the last quad, 1..4
  return {rem > 1 ? ~0u : 0u, rem > 2 ? ~0u : 0u, rem > 3 ? ~0u : 0u};
}
__device__ __forceinline__ uint32_t quad_neg(const uint4& v, bool last, const QuadMask& m) {
  return last ? (v.x | (v.y & m.y) | (v.z & m.z) | (v.w & m.w)) : (v.x | v.y | v.z | v.w);
}

struct GlobalTab {
  const double* p;
  __device__ __forceinline__ double get(int idx) const { return __ldg(p + idx); }
};

// acc + x*t: exact mode = the reference's two roundings (DMUL then DADD);
// fma mode (GNB_MODE_FMA) = one rounding, within the north star's 1e-5.
template <bool FMA>
__device__ __forceinline__ double madd(double acc, double x, double t) {
  if constexpr (FMA) return __fma_rn(x, t, acc);
  else return __dadd_rn(acc, __dmul_rn(x, t));
}

// One 16-B chunk (kPerQuad consecutive features) of one row, all classes.
template <int CP, typename T, typename Tab, bool FMA>
__device__ __forceinline__ void score_quad(double (&acc)[CP], const uint4 v, const Tab& tab,
                                           int feat0) {
#pragma unroll
  for (int e = 0; e < Elem<T>::kPerQuad; ++e) {
    const double xd = converted<T, FMA>(v, e);
#pragma unroll
    for (int c = 0; c < CP; ++c)
      acc[c] = madd<FMA>(acc[c], xd, tab.get((feat0 + e) * CP + c));
  }
}

template <int CP, typename T, typename Tab, bool FMA>
__device__ __forceinline__ void score_chunk(double (&acc)[CP], const uint8_t* box, uint32_t row,
                                            const Tab& tab, int nq, uint32_t& neg) {
  constexpr int EQ = Elem<T>::kPerQuad;
  if (nq == 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 v = *reinterpret_cast<const uint4*>(box + swz128(row, q));
      if (Elem<T>::kSigned) neg |= v.x | v.y | v.z | v.w;
      score_quad<CP, T, Tab, FMA>(acc, v, tab, EQ * q);
    }
  } else {
#pragma unroll 1
    for (int q = 0; q < nq; ++q) {
      const uint4 v = *reinterpret_cast<const uint4*>(box + swz128(row, q));
      if (Elem<T>::kSigned) neg |= v.x | v.y | v.z | v.w;
      score_quad<CP, T, Tab, FMA>(acc, v, tab, EQ * q);
    }
  }
}

template <int CP>
__device__ __forceinline__ void write_row(const PredictParams& p, int64_t r, int slot,
                                          uint32_t neg, const double (&acc)[CP]) {
  int lab;
  if (slot < 0) {
    lab = GNB_ROW_OUT_OF_RANGE;
  } else if (neg & 0x80000000u) {
    lab = GNB_ROW_NEGATIVE_COUNT;
  } else {
    lab = 0;
    double best = acc[0];
#pragma unroll
    for (int c = 1; c < CP; ++c) {
      if (acc[c] > best) {  // strict: ties keep the lower index (benign)
        best = acc[c];
        lab = c;
      }
    }
  }
  p.label[r] = lab;
  if (p.logpost != nullptr) {
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    double* out = p.logpost + r * p.n_classes;
    if (p.n_classes == 2 && CP == 2) {
      const double2 v = slot < 0 ? make_double2(nan, nan) : make_double2(acc[0], acc[CP - 1]);
      *reinterpret_cast<double2*>(out) = v;
    } else {
#pragma unroll
      for (int c = 0; c < CP; ++c)
        if (c < p.n_classes) out[c] = slot < 0 ? nan : acc[c];
    }
  }
}

// Device-side kernel gate (GNB_ORDER_AUTO): both K-PRED kernels are launched
// and the one not chosen by the tile-mix count exits at once.
__device__ __forceinline__ bool gated_off(const PredictParams& p) {
  return p.gate != nullptr && __ldg(p.gate) != p.gate_want;
}

// ------------------------------------------------------------------ TMA kernel
// A consumer thread owns R rows of the tile (rows lane + 32*(w + NW*i)), so one
// broadcast table read feeds R*CP independent accumulator chains.
// A stage holds B consecutive 128-B column chunks of the tile (B boxes).
template <int CP, typename T, int R, int NW, int STAGES, bool GATHER = false, int B = 1>
struct PredictSmem {
  static constexpr int kRows = NW * 32 * R;                          // rows per tile (<= 256)
  static constexpr int kBox = kRows * kChunkBytesPerRow;               // one box
  static constexpr int kXBytes = B * kBox;                             // one stage
  static constexpr int kTabChunk = Elem<T>::kPerRow * CP * 8;          // one chunk's table
  static constexpr int kPrior = CP * 8;                                // the slot's prior
  static constexpr int kTabBytes = kPrior + B * kTabChunk;             // prior + tables
  // tile_slot + tile + row_slot[kRows] (+ row_id[kRows] in gather mode)
  static constexpr int kHdrBytes = ((8 + kRows * 4 * (GATHER ? 2 : 1)) + 15) / 16 * 16;
  static constexpr int kX = 0;
  static constexpr int kTab = kX + STAGES * kXBytes;
  static constexpr int kHdr = kTab + STAGES * kTabBytes;
  static constexpr int kBar = kHdr + STAGES * kHdrBytes;
  static constexpr int kTotal = kBar + 2 * STAGES * 8;
  static constexpr int kAlloc = kTotal + 1024;  // slack for 1024-B alignment
  static_assert(kRows <= 256, "TMA box rows <= 256");
};

struct StageHdr {
  int tile_slot;  // >= 0: every valid row uses this slot; table slice staged
  int tile;       // the tile this stage belongs to; -1 = no more tiles (end marker)
  int row_slot[1];  // [kRows]; in gather mode followed by row_id[kRows]
};

// Table of slot s, chunk ch (kPerRow features per chunk).
template <int CP, typename T>
__device__ __forceinline__ const double* chunk_table(const PredictParams& p, int s, int ch) {
  constexpr int blocks_per_chunk = Elem<T>::kPerRow / kTabBlockFeatures;
  return p.tab + (static_cast<int64_t>(s) * p.n_tab_blocks + ch * blocks_per_chunk) *
                     (kTabBlockFeatures * CP);
}

// Uniform tile: the chunk's table slice is in smem and shared by all R rows.
template <int CP, typename T, int R, bool FMA>
__device__ __forceinline__ void score_chunk_uniform(double (&acc)[R][CP], const uint8_t* box,
                                                    const uint32_t (&rows)[R], const double* tab,
                                                    int nq, uint32_t (&neg)[R]) {
  constexpr int EQ = Elem<T>::kPerQuad;
  auto quad = [&](int q) {
    uint4 v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      v[i] = *reinterpret_cast<const uint4*>(box + swz128(rows[i], q));
      if (Elem<T>::kSigned) neg[i] |= v[i].x | v[i].y | v[i].z | v[i].w;
    }
#pragma unroll
    for (int e = 0; e < EQ; ++e) {
      double t[CP];  // one broadcast LDS.128 per 2 classes
#pragma unroll
      for (int c = 0; c < CP; c += 2) {
        const double2 t2 = *reinterpret_cast<const double2*>(tab + (EQ * q + e) * CP + c);
        t[c] = t2.x;
        t[c + 1] = t2.y;
      }
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const double xd = converted<T, FMA>(v[i], e);
#pragma unroll
        for (int c = 0; c < CP; ++c) acc[i][c] = madd<FMA>(acc[i][c], xd, t[c]);
      }
    }
  };
  if (nq == 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) quad(q);
  } else {
#pragma unroll 1
    for (int q = 0; q < nq; ++q) quad(q);
  }
}

// Mixed tile: every row reads its own slot's table through L1.
template <int CP, typename T, int R, bool FMA>
__device__ __forceinline__ void score_chunk_mixed(const PredictParams& p, double (&acc)[R][CP],
                                                  const uint8_t* box, const uint32_t (&rows)[R],
                                                  const int (&slot)[R], int ch, int nq,
                                                  uint32_t (&neg)[R]) {
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const GlobalTab tab{chunk_table<CP, T>(p, max(slot[i], 0), ch)};
    double a[CP];
#pragma unroll
    for (int c = 0; c < CP; ++c) a[c] = acc[i][c];
    score_chunk<CP, T, GlobalTab, FMA>(a, box, rows[i], tab, nq, neg[i]);
#pragma unroll
    for (int c = 0; c < CP; ++c) acc[i][c] = a[c];
  }
}

// GATHER: tile rows are perm[tile*ROWS ...] (rows sorted by routed slot by
// slot_sort), loaded with TMA tile::gather4 (4 arbitrary rows per
// instruction, one instruction per producer lane) into the same swizzled box
// layout; outputs go back to the original row index.
template <int CP, typename T, int R, int NW, int STAGES, bool GATHER, int B, bool FMA>
__global__ void __launch_bounds__((NW + 1) * 32)
    predict_tma_kernel(const __grid_constant__ PredictMaps maps, const PredictParams p) {
  if (gated_off(p)) return;
  const CUtensorMap& xmap = maps.main;
  using L = PredictSmem<CP, T, R, NW, STAGES, GATHER, B>;
  constexpr int ROWS = L::kRows;
  constexpr int CF = Elem<T>::kPerRow;
  constexpr int EQ = Elem<T>::kPerQuad;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for SWIZZLE_128B, keeping the pointer in the shared window
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 32);   // all producer lanes arrive (lane 0 with tx)
      mbar_init(&empty[s], NW);  // one arrive per consumer warp
    }
    mbar_fence_init();
  }
  if (warp == NW && lane == 0) {
    prefetch_tensormap(&xmap);
    if (GATHER) prefetch_tensormap(&maps.tail);
  }
  __syncthreads();

  const int NCH = p.n_chunks;
  const int NSC = (NCH + B - 1) / B;  // stages per tile
  const int64_t n_tiles = p.n_tiles;

  if (warp == NW) {
    // ---------------------------------------------------------- producer
    const uint64_t pol_x = p.x_policy == 1 ? policy_evict_first() : policy_evict_normal();
    const uint64_t pol_t = policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    // Tiles: the CTA's first is blockIdx.x; after that, with p.tile_ctr, the
    // next unclaimed tile in index order (one atomic per tile) -- CTAs whose
    // SM gets less DRAM bandwidth take fewer tiles, so they all finish
    // together instead of spreading the launch's last ~20 us (a static
    // grid-stride split finished CTAs of equal tile count 113-134 us apart
    // at 1M x 200).  Tiles are still handed out in order (DRAM locality).
    for (int64_t tile = blockIdx.x; tile < n_tiles;) {
      const int64_t r0 = tile * ROWS;
      int slots[ROWS / 32], ids[ROWS / 32];
      int lo = INT_MAX, hi = INT_MIN;
#pragma unroll
      for (int i = 0; i < ROWS / 32; ++i) {
        int64_t r = r0 + lane + 32 * i;
        int s = -1;
        if (GATHER) r = r < p.n_rows ? __ldg(p.perm + r) : -1;
        ids[i] = static_cast<int>(GATHER ? r : 0);
        if (r >= 0 && r < p.n_rows) {
          const int sz = __ldg(p.size + r);
          if (sz >= 0 && sz < p.limit) {
            s = __ldg(p.route + sz / p.width);
            lo = min(lo, s);
            hi = max(hi, s);
          }
        }
        slots[i] = s;
      }
      lo = __reduce_min_sync(0xffffffffu, lo);
      hi = __reduce_max_sync(0xffffffffu, hi);
      const int tile_slot = (lo == INT_MAX) ? 0 : (lo == hi ? lo : -1);
      for (int sc = 0; sc < NSC; ++sc) {
        const int ch = sc * B;
        const int nb = min(B, NCH - ch);
        mbar_wait(&empty[stage], phase ^ 1);
        StageHdr* hdr = reinterpret_cast<StageHdr*>(smem + L::kHdr + stage * L::kHdrBytes);
        if (ch == 0) {
#pragma unroll
          for (int i = 0; i < ROWS / 32; ++i) {
            hdr->row_slot[lane + 32 * i] = slots[i];
            if (GATHER) hdr->row_slot[ROWS + lane + 32 * i] = ids[i];
          }
        }
        if (lane == 0) {
          hdr->tile_slot = tile_slot;
          hdr->tile = static_cast<int>(tile);
        }
        __syncwarp();
        uint8_t* box = smem + L::kX + stage * L::kXBytes;
        if (lane == 0) {
          const uint32_t bytes = nb * (L::kBox + (tile_slot >= 0 ? L::kTabChunk : 0)) +
                                 (tile_slot >= 0 && ch == 0 ? L::kPrior : 0);
          mbar_arrive_expect_tx(&full[stage], bytes);
          if (!GATHER)
            for (int b = 0; b < nb; ++b)
              tma_load_2d(box + b * L::kBox, &xmap, (ch + b) * CF, static_cast<int32_t>(r0),
                          &full[stage], pol_x);
          if (tile_slot >= 0) {
            uint8_t* dst = smem + L::kTab + stage * L::kTabBytes;
            if (ch == 0)  // first stage of the tile: the slot's prior too
              bulk_load(dst, p.prior + tile_slot * CP, L::kPrior, &full[stage], pol_t);
            bulk_load(dst + L::kPrior, chunk_table<CP, T>(p, tile_slot, ch), nb * L::kTabChunk,
                      &full[stage], pol_t);
          }
        }
        if (GATHER) {
          __syncwarp();  // expect_tx precedes every completion
#pragma unroll
          for (int g = lane; g < ROWS / 4; g += 32) {
            int rr[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int64_t pos = r0 + 4 * g + k;
              rr[k] = __ldg(p.perm + (pos < p.n_rows ? pos : p.n_rows - 1));
            }
            for (int b = 0; b < nb; ++b)
              tma_gather4(box + b * L::kBox + 4 * g * kChunkBytesPerRow,
                          ch + b == NCH - 1 ? &maps.tail : &xmap, (ch + b) * CF, rr,
                          &full[stage]);
          }
        }
        if (lane != 0) mbar_arrive(&full[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (p.tile_ctr != nullptr) {
        int next = 0;
        if (lane == 0) next = static_cast<int>(gridDim.x) + atomicAdd(p.tile_ctr, 1);
        tile = __shfl_sync(0xffffffffu, next, 0);
      } else {
        tile += gridDim.x;
      }
    }
    // end marker: one more stage whose header says "no more tiles"
    mbar_wait(&empty[stage], phase ^ 1);
    if (lane == 0) reinterpret_cast<StageHdr*>(smem + L::kHdr + stage * L::kHdrBytes)->tile = -1;
    __syncwarp();
    mbar_arrive(&full[stage]);
    if (p.tile_ctr != nullptr && lane == 0) {
      // the last producer to finish leaves the counters at 0 for the next launch
      __threadfence();
      if (atomicAdd(p.tile_ctr + 1, 1) == static_cast<int>(gridDim.x) - 1) {
        p.tile_ctr[0] = 0;
        p.tile_ctr[1] = 0;
        __threadfence();
      }
    }
  } else {
    // ---------------------------------------------------------- consumers
    uint32_t rows[R];
#pragma unroll
    for (int i = 0; i < R; ++i) rows[i] = lane + 32 * (warp + NW * i);
    int stage = 0;
    uint32_t phase = 0;
    for (;;) {
      double acc[R][CP];
      int slot[R], rid[R];
      uint32_t neg[R];
      int64_t tile = 0;
#pragma unroll
      for (int i = 0; i < R; ++i) neg[i] = 0;
      for (int sc = 0; sc < NSC; ++sc) {
        mbar_wait(&full[stage], phase);
        const StageHdr* hdr =
            reinterpret_cast<const StageHdr*>(smem + L::kHdr + stage * L::kHdrBytes);
        const int ts = hdr->tile_slot;
        if (sc == 0) {
          tile = hdr->tile;
          if (tile < 0) break;  // end marker (released below)
        }
        if (sc == 0) {
#pragma unroll
          for (int i = 0; i < R; ++i) {
            slot[i] = hdr->row_slot[rows[i]];
            rid[i] = GATHER ? hdr->row_slot[ROWS + rows[i]] : 0;
            const int s = ts >= 0 ? ts : max(slot[i], 0);
            const double* sp =
                reinterpret_cast<const double*>(smem + L::kTab + stage * L::kTabBytes);
#pragma unroll
            for (int c = 0; c < CP; ++c) acc[i][c] = ts >= 0 ? sp[c] : __ldg(p.prior + s * CP + c);
          }
        }
#pragma unroll
        for (int b = 0; b < B; ++b) {
          const int ch = sc * B + b;
          if (B > 1 && ch >= NCH) break;
          const int nf = min(CF, p.n_features - ch * CF);
          const int nq = (nf + EQ - 1) / EQ;
          const uint8_t* box = smem + L::kX + stage * L::kXBytes + b * L::kBox;
          if (ts >= 0) {
            score_chunk_uniform<CP, T, R, FMA>(
                acc, box, rows,
                reinterpret_cast<const double*>(smem + L::kTab + stage * L::kTabBytes +
                                                L::kPrior + b * L::kTabChunk),
                nq, neg);
          } else {
            score_chunk_mixed<CP, T, R, FMA>(p, acc, box, rows, slot, ch, nq, neg);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (tile < 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        break;
      }
#pragma unroll
      for (int i = 0; i < R; ++i) {
        if (GATHER) {
          if (tile * ROWS + rows[i] < p.n_rows) write_row<CP>(p, rid[i], slot[i], neg[i], acc[i]);
        } else {
          const int64_t r = tile * ROWS + rows[i];
          if (r < p.n_rows) write_row<CP>(p, r, slot[i], neg[i], acc[i]);
        }
      }
    }
  }
}

// ------------------------------------------------------------------ row-box kernel
// Short rows (F <= ~100 int32 features): one stage holds kRowBoxRows whole
// rows, WQ 16-B quads per smem row with WQ odd so the 8 lanes of an LDS.128
// phase (consecutive rows, stride WQ*16 B) hit 8 distinct bank groups.  When
// the HBM row pitch equals WQ*16 B the tile is one contiguous 1-D bulk copy;
// otherwise a 2-D tensor box (unswizzled).  One stage per tile, no partial
// 128-B chunks: the 128-B-box kernel above spends a whole 16-KB stage on e.g.
// the 18 trailing features of F=50, so short rows kept too few bytes in flight
// per SM.  Same arithmetic and order as every path.
//
// Resident tables (p.rowbox_resident): every slot's prior + table is copied
// into smem once per CTA, so a stage carries X only.  Rows of <= kRegQuads
// quads are then moved to registers and the stage is released BEFORE the
// DMUL/DADD chain runs: a stage is held for a few LDS instead of the whole
// scoring time, which is what bounds the bytes in flight per SM for short rows.
// Register budget: the default instance (__launch_bounds__(160, 4): <= 102
// per thread) holds 13 quads of X next to 2 accumulators (14 spill), 8 next to
// 4; wider class pads keep the stage.  Rows of 14-26 quads at C=2 (int32
// F <= 104: 2-3 CTAs/SM anyway, 30-55-KB tiles) take a second instance with
// __launch_bounds__(160, 2) and 26 quads of registers.
template <int CP>
inline constexpr int kRegQuads = CP <= 2 ? 13 : CP == 4 ? 8 : 0;
inline constexpr int kRegQuadsWide = 26;

struct RowBoxSmem {
  uint32_t x_bytes, tab_bytes, hdr_bytes, res_stride, x, res, tab, hdr, sizes, bar, total;
  // ahead: tiles whose row sizes are in flight ahead of routing;
  // resident_slots > 0: all slot tables resident (no per-stage tables)
  __host__ __device__ RowBoxSmem(int wq, int tab_feats, int cp, int stages, int ahead,
                                 int resident_slots) {
    x_bytes = static_cast<uint32_t>(kRowBoxRows) * wq * 16;
    // one slot = [prior: cp doubles][tab_feats x cp log-likelihoods]
    res_stride = static_cast<uint32_t>(1 + tab_feats) * cp;  // doubles
    tab_bytes = resident_slots > 0 ? 0u : res_stride * 8;
    hdr_bytes = (8 + kRowBoxRows * 4 + 15) / 16 * 16;  // tile_slot, tile, slot[rows]
    x = 0;
    res = x + stages * x_bytes;
    tab = res + static_cast<uint32_t>(resident_slots) * res_stride * 8;
    hdr = tab + stages * tab_bytes;
    sizes = hdr + stages * hdr_bytes;  // [ahead][kRowBoxRows] prefetched sizes
    bar = sizes + ahead * kRowBoxRows * 4;
    total = bar + 2 * stages * 8;
  }
};

__host__ __device__ inline int rowbox_tab_feats(int F, int EQ, int n_tab_blocks) {
  const int nq = (F + EQ - 1) / EQ;
  const int want = nq * EQ, have = n_tab_blocks * kTabBlockFeatures;
  return want < have ? want : have;
}

// the nq quads of one row against one slot's smem table (prior excluded)
template <int CP, typename T, bool FMA, bool TAILMASK>
__device__ __forceinline__ void rowbox_score_smem(double (&acc)[CP], const uint8_t* xrow,
                                                  const double* tab, int nq, uint32_t& neg,
                                                  const QuadMask& lm) {
  constexpr int EQ = Elem<T>::kPerQuad;
#pragma unroll 2
  for (int q = 0; q < nq; ++q) {
    const uint4 v = *reinterpret_cast<const uint4*>(xrow + 16 * q);
    if (Elem<T>::kSigned) neg |= TAILMASK ? quad_neg(v, q == nq - 1, lm) : (v.x | v.y | v.z | v.w);
#pragma unroll
    for (int e = 0; e < EQ; ++e) {
      const double xd = converted<T, FMA>(v, e);
#pragma unroll
      for (int c = 0; c < CP; c += 2) {  // broadcast LDS.128 per 2 classes
        const double2 t2 = *reinterpret_cast<const double2*>(tab + (EQ * q + e) * CP + c);
        acc[c] = madd<FMA>(acc[c], xd, t2.x);
        acc[c + 1] = madd<FMA>(acc[c + 1], xd, t2.y);
      }
    }
  }
}

template <int CP, typename T, int kRowBoxAhead, bool FMA, int RQ = kRegQuads<CP>, int MINB = 4,
          bool TAILMASK = false>
__global__ void __launch_bounds__(5 * 32, MINB)
    predict_rowbox_kernel(const __grid_constant__ PredictMaps maps, const PredictParams p) {
  const CUtensorMap& xmap = maps.main;
  constexpr int NW = 4, ROWS = kRowBoxRows, EQ = Elem<T>::kPerQuad;
  static_assert(ROWS == NW * 32, "one row per consumer thread");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  const int ST = p.rowbox_stages, WQ = p.rowbox_quads;
  const int tab_feats = rowbox_tab_feats(p.n_features, EQ, p.n_tab_blocks);
  const bool resident = p.rowbox_resident != 0;
  const RowBoxSmem L(WQ, tab_feats, CP, ST, kRowBoxAhead, resident ? p.n_slots : 0);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* empty = full + ST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t slot_tab = static_cast<int64_t>(p.n_tab_blocks) * kTabBlockFeatures * CP;
  // Prologue: the producer initialises the barriers and starts streaming at
  // once; the consumers copy the resident tables meanwhile and wait (named
  // barrier 1) for the producer's init and each other's copies -- the first X
  // copies do not queue behind the table loads.
  if (warp == NW) {
    if (lane == 0) {
      for (int s = 0; s < ST; ++s) {
        mbar_init(&full[s], 32);
        mbar_init(&empty[s], NW);
      }
      mbar_fence_init();
      prefetch_tensormap(&xmap);
    }
    __syncwarp();
    named_bar_arrive(1, (NW + 1) * 32);
  } else {
    if (resident) {  // all slots' [prior | table] once per CTA
      double* res = reinterpret_cast<double*>(smem + L.res);
      const int stride = static_cast<int>(L.res_stride);
      for (int i = threadIdx.x; i < p.n_slots * stride; i += NW * 32) {
        const int s = i / stride, k = i - s * stride;
        res[i] = k < CP ? __ldg(p.prior + s * CP + k) : __ldg(p.tab + s * slot_tab + (k - CP));
      }
    }
    named_bar_sync(1, (NW + 1) * 32);
  }
  const int64_t n_tiles = p.n_tiles;

  if (warp == NW) {
    // ---------------------------------------------------------- producer
    const uint64_t pol_x = p.x_policy == 1 ? policy_evict_first() : policy_evict_normal();
    const uint64_t pol_t = policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    // Row sizes travel kRowBoxAhead tiles ahead of routing (LDGSTS into a
    // smem ring, each lane reading back only its own entries): with one stage
    // per tile, a size load per tile on the critical path capped the rate at
    // one tile per loaded-HBM round trip.
    int* szr = reinterpret_cast<int*>(smem + L.sizes);
    auto fetch_sizes = [&](int64_t tile, int k) {
      if (tile < n_tiles) {
#pragma unroll
        for (int i = 0; i < ROWS / 32; ++i) {
          const int64_t r = tile * ROWS + lane + 32 * i;
          cp_async4(szr + k * ROWS + lane + 32 * i, p.size + (r < p.n_rows ? r : p.n_rows - 1));
        }
      }
      cp_async_commit();
    };
    // Tiles are claimed when their sizes are prefetched (kRowBoxAhead ahead):
    // the CTA's first is blockIdx.x, later ones the next unclaimed tile from
    // p.tile_ctr (dynamic scheduling, as in the 128-B-box kernel), else
    // grid-strided.  tq[0] is the tile being issued, tq[1..] the claimed ones.
    int64_t tq[kRowBoxAhead];
    int64_t j_static = 0;
    auto claim = [&]() -> int64_t {
      if (p.tile_ctr != nullptr && j_static > 0) {
        int nt = 0;
        if (lane == 0) nt = static_cast<int>(gridDim.x) + atomicAdd(p.tile_ctr, 1);
        return __shfl_sync(0xffffffffu, nt, 0);
      }
      return blockIdx.x + (j_static++) * int64_t(gridDim.x);
    };
#pragma unroll
    for (int k = 0; k < kRowBoxAhead; ++k) {
      tq[k] = claim();
      fetch_sizes(tq[k], k);
    }
    int k_cur = 0;
    for (;;) {
      const int64_t tile = tq[0];
      if (tile >= n_tiles) break;
      const int64_t r0 = tile * ROWS;
      // X first: it does not depend on routing, so the copy is in flight while
      // the producer waits for the tile's sizes and routes them (this also
      // takes the size + route round trips out of the kernel's ramp).
      mbar_wait(&empty[stage], phase ^ 1);
      if (lane == 0) {
        if (p.rowbox_contig) {
          // rows are contiguous in HBM with the smem pitch: the tile is ONE
          // 1-D bulk copy (no per-row box traffic); only the valid rows
          const int64_t nr = p.n_rows - r0 < ROWS ? p.n_rows - r0 : ROWS;
          const uint32_t xb = static_cast<uint32_t>(nr) * WQ * 16;
          mbar_expect_tx(&full[stage], xb);
          bulk_load(smem + L.x + stage * L.x_bytes,
                    static_cast<const uint8_t*>(p.x) + r0 * (WQ * 16), xb, &full[stage], pol_x);
        } else {
          mbar_expect_tx(&full[stage], L.x_bytes);
          tma_load_2d(smem + L.x + stage * L.x_bytes, &xmap, 0, static_cast<int32_t>(r0),
                      &full[stage], pol_x);
        }
      }
      int slots[ROWS / 32];
      int lo = INT_MAX, hi = INT_MIN;
      cp_async_wait<kRowBoxAhead - 1>();
#pragma unroll
      for (int i = 0; i < ROWS / 32; ++i) {
        const int64_t r = r0 + lane + 32 * i;
        const int sz = szr[k_cur * ROWS + lane + 32 * i];
        int s = -1;
        if (r < p.n_rows && sz >= 0 && sz < p.limit) {
          s = __ldg(p.route + sz / p.width);
          lo = min(lo, s);
          hi = max(hi, s);
        }
        slots[i] = s;
      }
#pragma unroll
      for (int k = 0; k + 1 < kRowBoxAhead; ++k) tq[k] = tq[k + 1];
      tq[kRowBoxAhead - 1] = claim();
      fetch_sizes(tq[kRowBoxAhead - 1], k_cur);
      if (++k_cur == kRowBoxAhead) k_cur = 0;
      lo = __reduce_min_sync(0xffffffffu, lo);
      hi = __reduce_max_sync(0xffffffffu, hi);
      const int tile_slot = (lo == INT_MAX) ? 0 : (lo == hi ? lo : -1);
      int* hdr = reinterpret_cast<int*>(smem + L.hdr + stage * L.hdr_bytes);
#pragma unroll
      for (int i = 0; i < ROWS / 32; ++i) hdr[2 + lane + 32 * i] = slots[i];
      if (lane == 0) {
        hdr[0] = tile_slot;
        hdr[1] = static_cast<int>(tile);
      }
      __syncwarp();
      if (lane == 0) {
        const bool stage_tab = !resident && tile_slot >= 0;
        mbar_arrive_expect_tx(&full[stage], stage_tab ? L.tab_bytes : 0);
        if (stage_tab) {  // the slot's prior, then its table
          uint8_t* dst = smem + L.tab + stage * L.tab_bytes;
          bulk_load(dst, p.prior + tile_slot * CP, CP * 8, &full[stage], pol_t);
          bulk_load(dst + CP * 8, p.tab + tile_slot * slot_tab, L.tab_bytes - CP * 8,
                    &full[stage], pol_t);
        }
      } else {
        mbar_arrive(&full[stage]);
      }
      if (++stage == ST) {
        stage = 0;
        phase ^= 1;
      }
    }
    // end marker: one more stage whose header says "no more tiles"
    mbar_wait(&empty[stage], phase ^ 1);
    if (lane == 0) reinterpret_cast<int*>(smem + L.hdr + stage * L.hdr_bytes)[1] = -1;
    __syncwarp();
    mbar_arrive(&full[stage]);
    if (p.tile_ctr != nullptr && lane == 0) {
      // the last producer to finish leaves the counters at 0 for the next launch
      __threadfence();
      if (atomicAdd(p.tile_ctr + 1, 1) == static_cast<int>(gridDim.x) - 1) {
        p.tile_ctr[0] = 0;
        p.tile_ctr[1] = 0;
        __threadfence();
      }
    }
  } else {
    // ---------------------------------------------------------- consumers
    const int row = lane + 32 * warp;
    const int nq = (p.n_features + EQ - 1) / EQ;
    const QuadMask lm = last_quad_mask(p.n_features);
    const bool early = RQ > 0 && resident && nq <= RQ;
    const double* res = reinterpret_cast<const double*>(smem + L.res);
    int stage = 0;
    uint32_t phase = 0;
    for (;;) {
      mbar_wait(&full[stage], phase);
      const int* hdr = reinterpret_cast<const int*>(smem + L.hdr + stage * L.hdr_bytes);
      const int64_t tile = hdr[1];
      if (tile < 0) {  // end marker
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        break;
      }
      const int ts = hdr[0];
      const int slot = hdr[2 + row];
      const int s = ts >= 0 ? ts : max(slot, 0);
      double acc[CP];
      uint32_t neg = 0;
      const uint8_t* xrow = smem + L.x + stage * L.x_bytes + row * (WQ * 16);
      bool released = false;
      if constexpr (RQ > 0) {
        if (early) {
          // row -> registers, release the stage, then score from registers
          uint4 v[RQ];
          uint32_t f = 0;
#pragma unroll
          for (int q = 0; q < RQ; ++q)
            if (q < nq) v[q] = *reinterpret_cast<const uint4*>(xrow + 16 * q);
#pragma unroll
          for (int q = 0; q < RQ; ++q)
            if (q < nq) f |= v[q].x;
          // the release waits for every lane's loads (see predict_mixed_kernel)
          const uint32_t dep =
              __ballot_sync(0xffffffffu, f != 0u) & static_cast<uint32_t>(p.dep_zero);
          if (lane == 0) mbar_arrive(&empty[stage] + dep);
          released = true;
          const double* st = res + s * static_cast<int>(L.res_stride);
#pragma unroll
          for (int c = 0; c < CP; ++c) acc[c] = st[c];
          const double* tab = st + CP;
#pragma unroll
          for (int q = 0; q < RQ; ++q) {
            if (q < nq) {
              if (Elem<T>::kSigned)
                neg |= TAILMASK ? quad_neg(v[q], q == nq - 1, lm) : (v[q].x | v[q].y | v[q].z | v[q].w);
#pragma unroll
              for (int e = 0; e < EQ; ++e) {
                const double xd = converted<T, FMA>(v[q], e);
#pragma unroll
                for (int c = 0; c < CP; c += 2) {
                  const double2 t2 =
                      *reinterpret_cast<const double2*>(tab + (EQ * q + e) * CP + c);
                  acc[c] = madd<FMA>(acc[c], xd, t2.x);
                  acc[c + 1] = madd<FMA>(acc[c + 1], xd, t2.y);
                }
              }
            }
          }
        }
      }
      if (!released) {
        if (resident) {
          const double* st = res + s * static_cast<int>(L.res_stride);
#pragma unroll
          for (int c = 0; c < CP; ++c) acc[c] = st[c];
          rowbox_score_smem<CP, T, FMA, TAILMASK>(acc, xrow, st + CP, nq, neg, lm);
        } else {
          const double* stab =
              reinterpret_cast<const double*>(smem + L.tab + stage * L.tab_bytes);
          // uniform tile: the prior came with the table (smem broadcast, no
          // global round trip in front of the first DADD); mixed tile: L1 loads
#pragma unroll
          for (int c = 0; c < CP; ++c) acc[c] = ts >= 0 ? stab[c] : __ldg(p.prior + s * CP + c);
          if (ts >= 0) {
            rowbox_score_smem<CP, T, FMA, TAILMASK>(acc, xrow, stab + CP, nq, neg, lm);
          } else {
            const GlobalTab tab{p.tab + s * slot_tab};
#pragma unroll 1
            for (int q = 0; q < nq; ++q) {
              const uint4 v = *reinterpret_cast<const uint4*>(xrow + 16 * q);
              if (Elem<T>::kSigned)
                neg |= TAILMASK ? quad_neg(v, q == nq - 1, lm) : (v.x | v.y | v.z | v.w);
              score_quad<CP, T, GlobalTab, FMA>(acc, v, tab, EQ * q);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
      }
      if (++stage == ST) {
        stage = 0;
        phase ^= 1;
      }
      const int64_t r = tile * ROWS + row;
      if (r < p.n_rows) write_row<CP>(p, r, slot, neg, acc);
    }
  }
}

// ------------------------------------------------------------------ mixed-slot kernel
// Rows of many size groups interleaved (a ragged batch in any order, e.g. the
// reference's per-file scoring of a shuffled corpus, engine.py:198-202): every
// slot's [prior | table] is resident in smem once per CTA, X streams in FILE
// order through the same 128-B 2-D TMA boxes as the kernel above (no device
// slot sort, no gather, every byte read once in order), and the producer
// counting-sorts each tile's rows by routed slot (stable, match_any leaders +
// smem histogram) so consumer lane t scores row rid[t]: lanes of one slot read
// the same table entry (broadcast), lanes of neighbouring slots hit distinct
// bank groups (slot stride = an odd number of 16-B units at CP = 2).
// A consumer thread keeps its row's chunks in registers one step AHEAD: it
// waits for chunk k+1, copies its 8 quads to registers and releases that stage
// before scoring chunk k, so every stage of the ring is in flight except for
// the few cycles between a TMA completion and the consumers' LDS.  1 CTA per SM
// (the tables take most of the shared memory); same arithmetic, same order.
struct MixSmem {
  uint32_t x_bytes, tab_feats, stride, hdr_bytes, n_hdr, x, res, hdr, sizes, hist, bar, total;
  __host__ __device__ MixSmem(int rows, int F, int eq, int cf, int stages, int ahead, int slots) {
    const int nch = (F + cf - 1) / cf;
    x_bytes = static_cast<uint32_t>(rows) * kChunkBytesPerRow;
    tab_feats = static_cast<uint32_t>((F + eq - 1) / eq * eq);  // features read per slot
    stride = 2u * (1u + tab_feats);  // doubles per slot (CP = 2): odd number of 16-B units
    hdr_bytes = static_cast<uint32_t>(rows) * 8 + 16;  // slot[rows] | rid[rows] | tile
    // header ring: the producer can be at most ceil(stages / nch) tiles ahead
    // of the consumers' header reads (a tile's header is read before its first
    // stage is released)
    n_hdr = static_cast<uint32_t>((stages + nch - 1) / nch);
    x = 0;  // 1024-B aligned (SWIZZLE_128B)
    res = x + stages * x_bytes;
    hdr = res + (static_cast<uint32_t>(slots) * stride * 8 + 15) / 16 * 16;
    sizes = hdr + n_hdr * hdr_bytes;
    hist = sizes + ahead * rows * 4;
    bar = (hist + (slots + 1) * 4 + 7) / 8 * 8;
    total = bar + 2 * stages * 8;
  }
};

template <typename T, int NW, int AHEAD, bool FMA>
__global__ void __launch_bounds__((NW + 1) * 32, 1)
    predict_mixed_kernel(const __grid_constant__ PredictMaps maps, const PredictParams p) {
  constexpr int CP = 2, ROWS = NW * 32, CF = Elem<T>::kPerRow, EQ = Elem<T>::kPerQuad;
  constexpr int QPC = kChunkBytesPerRow / 16;  // quads per chunk row
  static_assert(ROWS <= 256, "TMA box rows <= 256");
  if (gated_off(p)) return;
  const CUtensorMap& xmap = maps.main;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int ST = p.mixed_stages, NCH = p.n_chunks, S = p.n_slots;
  const MixSmem L(ROWS, p.n_features, EQ, CF, ST, AHEAD, S);
  const int HD = static_cast<int>(L.n_hdr);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* empty = full + ST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles = p.n_tiles;
  // Prologue (as the row-box kernel): the producer initialises the barriers and
  // starts streaming; the consumers copy the resident tables meanwhile.
  if (warp == NW) {
    if (lane == 0) {
      for (int s = 0; s < ST; ++s) {
        mbar_init(&full[s], 32);
        mbar_init(&empty[s], NW);
      }
      mbar_fence_init();
      prefetch_tensormap(&xmap);
    }
    __syncwarp();
    named_bar_arrive(1, (NW + 1) * 32);
  } else {
    const int64_t slot_tab = static_cast<int64_t>(p.n_tab_blocks) * kTabBlockFeatures * CP;
    double* res = reinterpret_cast<double*>(smem + L.res);
    const int stride = static_cast<int>(L.stride);
    for (int i = threadIdx.x; i < S * stride; i += NW * 32) {
      const int s = i / stride, k = i - s * stride;
      res[i] = k < CP ? __ldg(p.prior + s * CP + k) : __ldg(p.tab + s * slot_tab + (k - CP));
    }
    named_bar_sync(1, (NW + 1) * 32);
  }

  if (warp == NW) {
    // ---------------------------------------------------------- producer
    const uint64_t pol_x = p.x_policy == 1 ? policy_evict_first() : policy_evict_normal();
    int* szr = reinterpret_cast<int*>(smem + L.sizes);
    int* hist = reinterpret_cast<int*>(smem + L.hist);
    const uint32_t lt_mask = (1u << lane) - 1u;
    auto fetch_sizes = [&](int64_t tile, int k) {
      if (tile < n_tiles) {
#pragma unroll
        for (int i = 0; i < ROWS / 32; ++i) {
          const int64_t r = tile * ROWS + lane + 32 * i;
          cp_async4(szr + k * ROWS + lane + 32 * i, p.size + (r < p.n_rows ? r : p.n_rows - 1));
        }
      }
      cp_async_commit();
    };
    // tiles claimed when their sizes are prefetched (as in the row-box kernel):
    // blockIdx.x first, then the next unclaimed tile from p.tile_ctr
    int64_t tq[AHEAD];
    int64_t j_static = 0;
    auto claim = [&]() -> int64_t {
      if (p.tile_ctr != nullptr && j_static > 0) {
        int nt = 0;
        if (lane == 0) nt = static_cast<int>(gridDim.x) + atomicAdd(p.tile_ctr, 1);
        return __shfl_sync(0xffffffffu, nt, 0);
      }
      return blockIdx.x + (j_static++) * int64_t(gridDim.x);
    };
#pragma unroll
    for (int k = 0; k < AHEAD; ++k) {
      tq[k] = claim();
      fetch_sizes(tq[k], k);
    }
    int k_cur = 0, stage = 0, h = 0;
    uint32_t phase = 0;
    for (;;) {
      const int64_t tile = tq[0];
      if (tile >= n_tiles) break;
      const int64_t r0 = tile * ROWS;
      for (int sc = 0; sc < NCH; ++sc) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (lane == 0) {  // X first: it does not depend on routing
          mbar_expect_tx(&full[stage], L.x_bytes);
          tma_load_2d(smem + L.x + stage * L.x_bytes, &xmap, sc * CF, static_cast<int32_t>(r0),
                      &full[stage], pol_x);
        }
        if (sc == 0) {
          // route the tile (size -> group -> slot; key 0 = out of range)
          int key[ROWS / 32], rank[ROWS / 32];
          cp_async_wait<AHEAD - 1>();
#pragma unroll
          for (int i = 0; i < ROWS / 32; ++i) {
            const int64_t r = r0 + lane + 32 * i;
            const int sz = szr[k_cur * ROWS + lane + 32 * i];
            key[i] = (r < p.n_rows && sz >= 0 && sz < p.limit) ? __ldg(p.route + sz / p.width) + 1
                                                               : 0;
          }
#pragma unroll
          for (int k = 0; k + 1 < AHEAD; ++k) tq[k] = tq[k + 1];
          tq[AHEAD - 1] = claim();
          fetch_sizes(tq[AHEAD - 1], k_cur);
          if (++k_cur == AHEAD) k_cur = 0;
          // stable counting sort by key: ranks within a key in row order
          for (int b = lane; b <= S; b += 32) hist[b] = 0;
          __syncwarp();
#pragma unroll
          for (int i = 0; i < ROWS / 32; ++i) {
            const uint32_t peers = __match_any_sync(0xffffffffu, key[i]);
            const int leader = __ffs(peers) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(&hist[key[i]], __popc(peers));
            base = __shfl_sync(0xffffffffu, base, leader);
            rank[i] = base + __popc(peers & lt_mask);
          }
          __syncwarp();
          int carry = 0;  // exclusive scan of the histogram
          for (int b0 = 0; b0 <= S; b0 += 32) {
            const int b = b0 + lane;
            const int v = b <= S ? hist[b] : 0;
            int inc = v;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
              const int t = __shfl_up_sync(0xffffffffu, inc, d);
              if (lane >= d) inc += t;
            }
            if (b <= S) hist[b] = carry + inc - v;
            carry += __shfl_sync(0xffffffffu, inc, 31);
          }
          __syncwarp();
          int* hs = reinterpret_cast<int*>(smem + L.hdr + h * L.hdr_bytes);
#pragma unroll
          for (int i = 0; i < ROWS / 32; ++i) {
            const int pos = hist[key[i]] + rank[i];
            hs[pos] = key[i] - 1;
            hs[ROWS + pos] = lane + 32 * i;
          }
          if (lane == 0) hs[2 * ROWS] = static_cast<int>(tile);
          if (++h == HD) h = 0;
          __syncwarp();
        }
        mbar_arrive(&full[stage]);
        if (++stage == ST) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    // end marker: one more stage whose header says "no more tiles"
    mbar_wait(&empty[stage], phase ^ 1);
    if (lane == 0) reinterpret_cast<int*>(smem + L.hdr + h * L.hdr_bytes)[2 * ROWS] = -1;
    __syncwarp();
    mbar_arrive(&full[stage]);
    if (p.tile_ctr != nullptr && lane == 0) {
      // the last producer to finish leaves the counters at 0 for the next launch
      __threadfence();
      if (atomicAdd(p.tile_ctr + 1, 1) == static_cast<int>(gridDim.x) - 1) {
        p.tile_ctr[0] = 0;
        p.tile_ctr[1] = 0;
        __threadfence();
      }
    }
  } else {
    // ---------------------------------------------------------- consumers
    const int t = lane + 32 * warp;
    const double* res = reinterpret_cast<const double*>(smem + L.res);
    const int stride = static_cast<int>(L.stride);
    int stage = 0, h = 0;
    uint32_t phase = 0;
    // (tile, sc) of the step whose quads are in registers / being fetched;
    // a tile's index arrives with its header (claimed by the producer)
    int64_t tile = 0;
    int sc = 0;
    // fetch step (tile, sc): its header (first chunk of a tile), its quads
    // into registers, then release the stage.  The release must not overtake
    // the loads: SYNCS.ARRIVE carries no scoreboard wait on earlier LDS, and
    // with the shared-memory pipe busy (bank conflicts of shuffled rows) a TMA
    // refill of the released stage was seen to land before the loads read it.
    // So every lane folds one word of each loaded quad (int32: all four, the
    // negative-count flag) and the warp's ballot of that fold feeds the
    // arrive's address (+ (ballot & dep_zero), an opaque zero): the arrive
    // issues only after every lane's loads have returned.
    // Returns false (stage released, nothing loaded) on the producer's end marker.
    auto fetch = [&](uint4 (&v)[QPC], int fsc, int& slot, int& rid, uint32_t& fold,
                     int64_t& ftile) {
      mbar_wait(&full[stage], phase);
      if (fsc == 0) {
        const int* hs = reinterpret_cast<const int*>(smem + L.hdr + h * L.hdr_bytes);
        ftile = hs[2 * ROWS];
        if (++h == HD) h = 0;
        if (ftile < 0) {  // end marker
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stage]);
          return false;
        }
        slot = hs[t];
        rid = hs[ROWS + t];
      }
      const int nq = (min(CF, p.n_features - fsc * CF) + EQ - 1) / EQ;
      const uint8_t* box = smem + L.x + stage * L.x_bytes;
      uint32_t f = 0;
      if (nq == QPC) {
#pragma unroll
        for (int q = 0; q < QPC; ++q) v[q] = *reinterpret_cast<const uint4*>(box + swz128(rid, q));
#pragma unroll
        for (int q = 0; q < QPC; ++q)
          f |= Elem<T>::kSigned ? (v[q].x | v[q].y | v[q].z | v[q].w) : v[q].x;
      } else {
#pragma unroll
        for (int q = 0; q < QPC; ++q)
          if (q < nq) v[q] = *reinterpret_cast<const uint4*>(box + swz128(rid, q));
#pragma unroll
        for (int q = 0; q < QPC; ++q)
          if (q < nq) f |= Elem<T>::kSigned ? (v[q].x | v[q].y | v[q].z | v[q].w) : v[q].x;
      }
      fold = f;
      const uint32_t dep = __ballot_sync(0xffffffffu, f != 0u) & static_cast<uint32_t>(p.dep_zero);
      if (lane == 0) mbar_arrive(&empty[stage] + dep);
      if (++stage == ST) {
        stage = 0;
        phase ^= 1;
      }
      return true;
    };
    double acc[CP] = {0.0, 0.0};
    uint32_t neg = 0;
    auto score_quad2 = [&](const uint4& vq, const double* tq) {
#pragma unroll
      for (int e = 0; e < EQ; ++e) {
        const double xd = converted<T, FMA>(vq, e);
        const double2 t2 = *reinterpret_cast<const double2*>(tq + e * CP);
        acc[0] = madd<FMA>(acc[0], xd, t2.x);
        acc[1] = madd<FMA>(acc[1], xd, t2.y);
      }
    };
    // score step (tile, sc) from registers; the last chunk writes the row
    auto score = [&](const uint4 (&v)[QPC], int ssc, int slot, int rid, int64_t stile,
                     uint32_t fold) {
      const double* st = res + max(slot, 0) * stride;
      if (ssc == 0) {
        acc[0] = st[0];
        acc[1] = st[1];
        neg = 0;
      }
      if (Elem<T>::kSigned) neg |= fold;
      const int nq = (min(CF, p.n_features - ssc * CF) + EQ - 1) / EQ;
      const double* tab = st + CP + ssc * CF * CP;
      if (nq == QPC) {
#pragma unroll
        for (int q = 0; q < QPC; ++q) score_quad2(v[q], tab + EQ * q * CP);
      } else {
#pragma unroll
        for (int q = 0; q < QPC; ++q)
          if (q < nq) score_quad2(v[q], tab + EQ * q * CP);
      }
      if (ssc == NCH - 1) {
        const int64_t r = stile * ROWS + rid;
        if (r < p.n_rows) write_row<CP>(p, r, slot, neg, acc);
      }
    };
    {
      uint4 va[QPC], vb[QPC];
      int slot_a = -1, rid_a = 0, slot_b = -1, rid_b = 0;
      uint32_t fa = 0, fb = 0;
      int64_t tile_b = 0;
      if (fetch(va, 0, slot_a, rid_a, fa, tile)) {
        // ping-pong between two register sets (no copies): A scored while B
        // holds the next step, then the roles swap
        for (;;) {
          int nsc = sc + 1 == NCH ? 0 : sc + 1;
          slot_b = nsc == 0 ? -1 : slot_a;
          rid_b = nsc == 0 ? 0 : rid_a;
          tile_b = tile;
          const bool more = fetch(vb, nsc, slot_b, rid_b, fb, tile_b);
          score(va, sc, slot_a, rid_a, tile, fa);
          if (!more) break;
          sc = nsc;
          tile = tile_b;
          nsc = sc + 1 == NCH ? 0 : sc + 1;
          slot_a = nsc == 0 ? -1 : slot_b;
          rid_a = nsc == 0 ? 0 : rid_b;
          const bool more2 = fetch(va, nsc, slot_a, rid_a, fa, tile);
          score(vb, sc, slot_b, rid_b, tile_b, fb);
          if (!more2) break;
          sc = nsc;
        }
      }
    }
  }
}

// ------------------------------------------------------------------ generic kernel
// Any layout (unaligned X, row pitch not a multiple of 16 B): one thread per
// row, loads through L1.  Same arithmetic, same results; slower.
template <int CP, typename T, bool FMA>
__global__ void __launch_bounds__(256) predict_generic_kernel(const PredictParams p) {
  const T* xbase = static_cast<const T*>(p.x);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < p.n_rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int sz = p.size[r];
    const int slot = (sz >= 0 && sz < p.limit) ? p.route[sz / p.width] : -1;
    const int s = max(slot, 0);
    double acc[CP];
#pragma unroll
    for (int c = 0; c < CP; ++c) acc[c] = p.prior[s * CP + c];
    const T* row = xbase + r * p.ldx;
    uint32_t neg = 0;
    const GlobalTab tab{p.tab + static_cast<int64_t>(s) * p.n_tab_blocks *
                                    (kTabBlockFeatures * CP)};
    for (int j = 0; j < p.n_features; ++j) {
      const uint32_t x = static_cast<uint32_t>(__ldg(row + j));
      if (Elem<T>::kSigned) neg |= x;
      const double xd = __uint2double_rn(x);
#pragma unroll
      for (int c = 0; c < CP; ++c) acc[c] = madd<FMA>(acc[c], xd, tab.get(j * CP + c));
    }
    write_row<CP>(p, r, slot, neg, acc);
  }
}

// ------------------------------------------------------------------ launchers
// Opt kernel K into 227 KB of dynamic smem once per device (the attribute
// lives in each device's context, so a process driving several GPUs sets it
// on each) and return the current device's SM count.
template <auto K>
cudaError_t kernel_prepare(int* sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::atomic<uint64_t> ready{0};
  const uint64_t bit = 1ull << (dev & 63);
  if (!(ready.load(std::memory_order_acquire) & bit)) {
    e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    ready.fetch_or(bit, std::memory_order_acq_rel);
  }
  return cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev);
}

template <int CP, typename T, int R, int NW, int STAGES, bool GATHER, int B, bool FMA>
static cudaError_t launch_tma_mode(const PredictMaps& map, PredictParams p, cudaStream_t stream) {
  using L = PredictSmem<CP, T, R, NW, STAGES, GATHER, B>;
  constexpr auto kern = predict_tma_kernel<CP, T, R, NW, STAGES, GATHER, B, FMA>;
  p.n_tiles = (p.n_rows + L::kRows - 1) / L::kRows;
  p.n_chunks = (p.n_features + Elem<T>::kPerRow - 1) / Elem<T>::kPerRow;
  int sms = 0, per_sm = 0;  // resident CTAs per SM for this instantiation
  cudaError_t e = kernel_prepare<kern>(&sms);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (NW + 1) * 32, L::kAlloc);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t want = static_cast<int64_t>(sms) * per_sm;
  const int grid = static_cast<int>(p.n_tiles < want ? p.n_tiles : want);
  if (grid == 0) return cudaSuccess;
  kern<<<grid, (NW + 1) * 32, L::kAlloc, stream>>>(map, p);
  return cudaGetLastError();
}

// Gather mode: GNB_GATHER_B=2 stages two chunks of each gathered row (A/B).
inline int gather_boxes() {
  static const int v = [] {  // read once (thread-safe static init)
    int v = -1;
    const char* e = getenv("GNB_GATHER_B");
    v = e ? atoi(e) : 1;
    return v;
  }();
  return v;
}

template <int CP, typename T, bool FMA, int R, int NW, int STAGES, int B = 1>
static cudaError_t launch_tma(const PredictMaps& map, const PredictParams& p,
                              cudaStream_t stream) {
  if (p.perm != nullptr)
    return gather_boxes() == 2
               ? launch_tma_mode<CP, T, R, NW, STAGES, true, 2, FMA>(map, p, stream)
               : launch_tma_mode<CP, T, R, NW, STAGES, true, 1, FMA>(map, p, stream);
  return launch_tma_mode<CP, T, R, NW, STAGES, false, B, FMA>(map, p, stream);
}

// Row-box eligibility: whole rows of <= kRowBoxMaxQuads 16-B quads (odd-padded)
// and at most 256 box columns (TMA limit).  GNB_PRED_ROWBOX=0 disables (A/B).
inline constexpr int kRowBoxMaxQuads = 26;       // 128 rows x 26 x 16 B = 52 KB per stage
inline constexpr uint32_t kRowBoxRingBytes = 53248;  // ring depth: stages x box ~ 52 KB

template <int CP, typename T, int AHEAD, bool FMA, int RQ = kRegQuads<CP>, int MINB = 4,
          bool TAILMASK = false>
static cudaError_t launch_rowbox_b(const PredictMaps& map, PredictParams p, cudaStream_t stream) {
  constexpr auto kern = predict_rowbox_kernel<CP, T, AHEAD, FMA, RQ, MINB, TAILMASK>;
  int sms = 0;
  cudaError_t e = kernel_prepare<kern>(&sms);
  if (e != cudaSuccess) return e;
  p.n_tiles = (p.n_rows + kRowBoxRows - 1) / kRowBoxRows;
  const uint32_t box = static_cast<uint32_t>(kRowBoxRows) * p.rowbox_quads * 16;
  int st = static_cast<int>(kRowBoxRingBytes / box);
  static const int st_env = [] {  // read once (thread-safe static init)
    int st_env = -1;
    const char* e = getenv("GNB_ROWBOX_STAGES");
    st_env = e ? atoi(e) : 0;
    return st_env;
  }();
  if (st_env > 0) st = st_env;
  p.rowbox_stages = st < 2 ? 2 : st > 8 ? 8 : st;
  const int tf = rowbox_tab_feats(p.n_features, Elem<T>::kPerQuad, p.n_tab_blocks);
  // resident tables unless they would cost CTAs per SM (GNB_ROWBOX_RESIDENT=0: never)
  static const int res_env = [] {  // read once (thread-safe static init)
    int res_env = -1;
    const char* e = getenv("GNB_ROWBOX_RESIDENT");
    res_env = e ? atoi(e) != 0 : 1;
    return res_env;
  }();
  int per_sm = 0;
  const RowBoxSmem Ls(p.rowbox_quads, tf, CP, p.rowbox_stages, AHEAD, 0);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 5 * 32, Ls.total + 128);
  if (e != cudaSuccess) return e;
  size_t smem = Ls.total + 128;
  p.rowbox_resident = 0;
  if (res_env) {
    const RowBoxSmem Lr(p.rowbox_quads, tf, CP, p.rowbox_stages, AHEAD, p.n_slots);
    int per_sm_r = 0;
    if (Lr.total + 128 <= 227u * 1024u) {
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_r, kern, 5 * 32, Lr.total + 128);
      if (e != cudaSuccess) return e;
    }
    if (per_sm_r >= per_sm && per_sm_r > 0) {
      p.rowbox_resident = 1;
      smem = Lr.total + 128;
      per_sm = per_sm_r;
    }
  }
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const int64_t want = static_cast<int64_t>(sms) * per_sm;
  const int grid = static_cast<int>(p.n_tiles < want ? p.n_tiles : want);
  if (grid == 0) return cudaSuccess;
  kern<<<grid, 5 * 32, smem, stream>>>(map, p);
  return cudaGetLastError();
}

// The masked instance only where raw pitch padding can reach the flag: int32
// rows, 1-D bulk tiles, F not a multiple of 4 (the check costs issue slots).
template <int CP, typename T, int AHEAD, bool FMA, int RQ = kRegQuads<CP>, int MINB = 4>
static cudaError_t launch_rowbox_a(const PredictMaps& map, PredictParams p, cudaStream_t stream) {
  if (Elem<T>::kSigned && p.rowbox_contig && p.n_features % Elem<T>::kPerQuad != 0)
    return launch_rowbox_b<CP, T, AHEAD, FMA, RQ, MINB, true>(map, p, stream);
  return launch_rowbox_b<CP, T, AHEAD, FMA, RQ, MINB, false>(map, p, stream);
}

// GNB_ROWBOX_WIDE=0: rows of 14-26 quads keep their stage while scoring (A/B).
inline bool rowbox_wide() {
  static const int v = [] {  // read once (thread-safe static init)
    const char* e = getenv("GNB_ROWBOX_WIDE");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

// CTAs per SM of a row-box kernel instance for this shape (per-stage table
// layout: the larger of the two smem footprints).
template <auto K, typename T>
int rowbox_occupancy(const PredictParams& p, int cp) {
  const uint32_t box = static_cast<uint32_t>(kRowBoxRows) * p.rowbox_quads * 16;
  int st = static_cast<int>(kRowBoxRingBytes / box);
  st = st < 2 ? 2 : st > 8 ? 8 : st;
  const int tf = rowbox_tab_feats(p.n_features, Elem<T>::kPerQuad, table_blocks(p.n_features));
  const RowBoxSmem L(p.rowbox_quads, tf, cp, st, 2, 0);
  int sms = 0, per_sm = 0;
  if (kernel_prepare<K>(&sms) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, K, 5 * 32, L.total + 128) !=
          cudaSuccess)
    return 0;
  return per_sm;
}

template <int CP, typename T, bool FMA>
static cudaError_t launch_rowbox(const PredictMaps& map, const PredictParams& p,
                                 cudaStream_t stream) {
  if constexpr (CP == 2) {
    // rows of 14-26 quads: the register-staged instance when its register
    // budget does not cost a CTA per SM (F=100 int32: 2 CTAs/SM either way,
    // 0.90 -> 1.04 of HBM; F=64 int32: 3 -> 2 CTAs/SM, slower -- keep default)
    const int nq = (p.n_features + Elem<T>::kPerQuad - 1) / Elem<T>::kPerQuad;
    if (nq > kRegQuads<CP> && nq <= kRegQuadsWide && rowbox_wide()) {
      constexpr auto wide = predict_rowbox_kernel<CP, T, 2, FMA, kRegQuadsWide, 2>;
      constexpr auto base = predict_rowbox_kernel<CP, T, 2, FMA>;
      if (rowbox_occupancy<wide, T>(p, CP) >= rowbox_occupancy<base, T>(p, CP))
        return launch_rowbox_a<CP, T, 2, FMA, kRegQuadsWide, 2>(map, p, stream);
    }
  }
  return launch_rowbox_a<CP, T, 2, FMA>(map, p, stream);
}

// Mixed-slot mode: consumer warps per CTA (tile rows = 32 * NW), ring depth =
// as many 128-B-box stages as fit next to the resident tables (<= 8).
inline constexpr int kMixedNW = 8;
inline constexpr int kMixedAhead = 2;
inline constexpr int kMixedMinStages = 3;
inline int mixed_stages_fit(int F, int eb, int S) {
  const int cf = kChunkBytesPerRow / eb, eq = 16 / eb;
  for (int st = 8; st >= kMixedMinStages; --st)
    if (MixSmem(kMixedNW * 32, F, eq, cf, st, kMixedAhead, S).total + 1024 <= 227u * 1024u)
      return st;
  return 0;
}

template <typename T, bool FMA>
static cudaError_t launch_mixed(const PredictMaps& map, PredictParams p, cudaStream_t stream) {
  constexpr auto kern = predict_mixed_kernel<T, kMixedNW, kMixedAhead, FMA>;
  constexpr int ROWS = kMixedNW * 32;
  int sms = 0;
  cudaError_t e = kernel_prepare<kern>(&sms);
  if (e != cudaSuccess) return e;
  p.n_tiles = (p.n_rows + ROWS - 1) / ROWS;
  p.n_chunks = (p.n_features + Elem<T>::kPerRow - 1) / Elem<T>::kPerRow;
  p.dep_zero = 0;
  // static grid-stride tiles: with one producer per SM the claim's atomic
  // round trip sits on the producer's path, and this kernel is bound by shared
  // memory, not by per-SM DRAM bandwidth -- dynamic tiles measured 4 % slower
  p.tile_ctr = nullptr;
  p.mixed_stages = mixed_stages_fit(p.n_features, static_cast<int>(sizeof(T)), p.n_slots);
  static const int st_env = [] {  // GNB_MIXED_STAGES: fewer stages (A/B probes only)
    const char* e = getenv("GNB_MIXED_STAGES");
    return e ? atoi(e) : 0;
  }();
  if (st_env >= 2 && st_env < p.mixed_stages) p.mixed_stages = st_env;
  if (p.mixed_stages < kMixedMinStages) return cudaErrorInvalidConfiguration;
  const MixSmem L(ROWS, p.n_features, Elem<T>::kPerQuad, Elem<T>::kPerRow, p.mixed_stages,
                  kMixedAhead, p.n_slots);
  const int grid = static_cast<int>(p.n_tiles < sms ? p.n_tiles : sms);
  if (grid == 0) return cudaSuccess;
  kern<<<grid, (kMixedNW + 1) * 32, L.total + 1024, stream>>>(map, p);
  return cudaGetLastError();
}

template <int CP, typename T, bool FMA>
static cudaError_t launch_generic(const PredictParams& p, cudaStream_t stream) {
  const int64_t blocks64 = (p.n_rows + 255) / 256;
  const int blocks = static_cast<int>(blocks64 < 148 * 16 ? blocks64 : 148 * 16);
  if (blocks == 0) return cudaSuccess;
  predict_generic_kernel<CP, T, FMA><<<blocks, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

// K-PRED geometry for C = 2: rows per thread (R), consumer warps (NW), ring
// stages; a few variants selectable with GNB_PRED_VARIANT (profiling only).
// Default (variant 0) measured best on B200 for int32 X
// (profiles/r01_tuning.md): 16-KB stages, 2 deep, 6 CTAs per SM.
struct PredVariant {
  int R, NW, STAGES;
};
inline constexpr PredVariant kCp2Variants[] = {{1, 4, 2}, {1, 4, 3}, {2, 2, 2}, {2, 4, 2},
                                           {1, 4, 2}, {1, 4, 3}, {1, 4, 2}};  // 4-6: B=2,2,4

inline int cp2_variant() {
  static const int v = [] {  // read once (thread-safe static init)
    int v = -1;
    const char* e = getenv("GNB_PRED_VARIANT");
    v = e ? atoi(e) : 0;
    if (v < 0 || v >= static_cast<int>(sizeof(kCp2Variants) / sizeof(kCp2Variants[0]))) v = 0;
    return v;
  }();
  return v;
}

template <typename T, bool FMA>
cudaError_t launch_typed(const PredictMaps* map, const PredictParams& p, int CP,
                         cudaStream_t stream) {
  if (map != nullptr && p.mixed_rows > 0 && p.perm == nullptr && CP == 2)
    return launch_mixed<T, FMA>(*map, p, stream);
  if (map != nullptr && p.rowbox_quads > 0 && p.perm == nullptr) {
    switch (CP) {
      case 2: return launch_rowbox<2, T, FMA>(*map, p, stream);
      case 4: return launch_rowbox<4, T, FMA>(*map, p, stream);
      case 8: return launch_rowbox<8, T, FMA>(*map, p, stream);
      default: return launch_rowbox<16, T, FMA>(*map, p, stream);
    }
  }
  if (map != nullptr) {
    switch (CP) {
      case 2:
        switch (cp2_variant()) {
          case 1: return launch_tma<2, T, FMA, 1, 4, 3>(*map, p, stream);
          case 2: return launch_tma<2, T, FMA, 2, 2, 2>(*map, p, stream);
          case 3: return launch_tma<2, T, FMA, 2, 4, 2>(*map, p, stream);
          case 4: return launch_tma<2, T, FMA, 1, 4, 2, 2>(*map, p, stream);
          case 5: return launch_tma<2, T, FMA, 1, 4, 3, 2>(*map, p, stream);
          case 6: return launch_tma<2, T, FMA, 1, 4, 2, 4>(*map, p, stream);
          default: {
            // long rows (>= 12 chunks, e.g. int32 F >= 353): 2 chunks per stage
            // (3 CTAs/SM), F=500/1000 0.85/0.90 -> 0.91/0.96 of HBM; shorter
            // rows keep 1-chunk stages (F=200: 0.89 vs 0.77), r01_tuning.md
            const int nch = (p.n_features + Elem<T>::kPerRow - 1) / Elem<T>::kPerRow;
            if (nch >= 12) return launch_tma<2, T, FMA, 1, 4, 2, 2>(*map, p, stream);
            return launch_tma<2, T, FMA, 1, 4, 2>(*map, p, stream);
          }
        }
      case 4: return launch_tma<4, T, FMA, 2, 4, 3>(*map, p, stream);
      case 8: return launch_tma<8, T, FMA, 1, 4, 4>(*map, p, stream);
      default: return launch_tma<16, T, FMA, 1, 4, 4>(*map, p, stream);
    }
  }
  switch (CP) {
    case 2: return launch_generic<2, T, FMA>(p, stream);
    case 4: return launch_generic<4, T, FMA>(p, stream);
    case 8: return launch_generic<8, T, FMA>(p, stream);
    default: return launch_generic<16, T, FMA>(p, stream);
  }
}

#define GNB_PRED_INSTANCES(X) \
  X(int32_t, false) X(int32_t, true) X(uint16_t, false) X(uint16_t, true) \
  X(uint8_t, false) X(uint8_t, true)
#define GNB_PRED_EXTERN(T, F) \
  extern template cudaError_t launch_typed<T, F>(const PredictMaps*, const PredictParams&, int, \
                                                 cudaStream_t);
GNB_PRED_INSTANCES(GNB_PRED_EXTERN)
#undef GNB_PRED_EXTERN

}  // namespace gnb
