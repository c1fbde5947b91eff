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
//
// Kernels: predict_kernels.cuh.  This unit: table packing and the dispatch.
#include <climits>

#include "predict_kernels.cuh"

namespace gnb {

int table_blocks(int F) {
  const int nb = (F + kTabBlockFeatures - 1) / kTabBlockFeatures;
  return (nb + kTabBlockAlign - 1) / kTabBlockAlign * kTabBlockAlign;
}

__global__ void pack_tables_kernel(const double* __restrict__ log_prior,
                                   const double* __restrict__ log_lik, int S, int C, int F,
                                   int CP, int NB, double* __restrict__ prior_out,
                                   double* __restrict__ tab_out) {
  const int64_t total_prior = static_cast<int64_t>(S) * CP;
  const int64_t per_slot = static_cast<int64_t>(NB) * kTabBlockFeatures * CP;
  const int64_t total_tab = S * per_slot;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       i < total_prior + total_tab; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (i < total_prior) {
      const int s = static_cast<int>(i / CP), c = static_cast<int>(i % CP);
      prior_out[i] = c < C ? log_prior[static_cast<int64_t>(s) * C + c] : -INFINITY;
    } else {
      const int64_t k = i - total_prior;
      const int c = static_cast<int>(k % CP);
      const int j = static_cast<int>((k / CP) % (NB * kTabBlockFeatures));  // feature
      const int s = static_cast<int>(k / per_slot);
      double ll = 0.0;
      if (c < C && j < F) ll = log_lik[(static_cast<int64_t>(s) * C + c) * F + j];
      tab_out[k] = ll;
    }
  }
}

int class_pad(int C) { return C <= 2 ? 2 : C <= 4 ? 4 : C <= 8 ? 8 : 16; }

size_t packed_bytes(int S, int C, int F) {
  const int CP = class_pad(C);
  return static_cast<size_t>(S) * CP * 8 +
         static_cast<size_t>(S) * table_blocks(F) * kTabBlockFeatures * CP * 8;
}

cudaError_t pack_tables(const double* log_prior, const double* log_lik, int S, int C, int F,
                        void* packed, cudaStream_t stream) {
  const int CP = class_pad(C);
  const int NB = table_blocks(F);
  double* prior = static_cast<double*>(packed);
  double* tab = prior + static_cast<int64_t>(S) * CP;
  const int64_t total = static_cast<int64_t>(S) * CP * (1 + NB * kTabBlockFeatures);
  const int blocks = static_cast<int>((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  pack_tables_kernel<<<blocks > 0 ? blocks : 1, 256, 0, stream>>>(log_prior, log_lik, S, C, F,
                                                                   CP, NB, prior, tab);
  return cudaGetLastError();
}

int predict_rowbox_quads(int n_features, int x_type, int n_classes) {
  static const int enabled = [] {  // read once (thread-safe static init)
    int enabled = -1;
    const char* e = getenv("GNB_PRED_ROWBOX");
    enabled = e ? atoi(e) != 0 : 1;
    return enabled;
  }();
  (void)n_classes;
  if (!enabled || n_features < 1) return 0;
  const int eb = x_type == GNB_X_U8 ? 1 : x_type == GNB_X_U16 ? 2 : 4;
  const int nq = (n_features * eb + 15) / 16;
  const int wq = nq | 1;
  if (wq > kRowBoxMaxQuads || wq * 16 / eb > 256) return 0;
  return wq;
}

// GNB_PRED_MIXED: 0 never, 1 (default) batches of >= 2 slots, 2 also one slot (A/B).
int predict_mixed_rows(int n_features, int x_type, int n_classes, int n_slots) {
  static const int mode = [] {  // read once (thread-safe static init)
    const char* e = getenv("GNB_PRED_MIXED");
    return e ? atoi(e) : 1;
  }();
  if (mode == 0 || class_pad(n_classes) != 2 || n_features < 1) return 0;
  if (n_slots < (mode == 2 ? 1 : 2)) return 0;
  const int eb = x_type == GNB_X_U8 ? 1 : x_type == GNB_X_U16 ? 2 : 4;
  return mixed_stages_fit(n_features, eb, n_slots) > 0 ? kMixedNW * 32 : 0;
}

// One warp per 128-row tile (grid-strided): min/max routed slot of the tile's
// in-range rows; one atomic per warp.  The last block to finish writes the
// decision gate[2] = (mixed tiles * 16 > tiles) and resets gate[0..1], so the
// counter needs no memset per call (zeroed once when it is allocated).
__global__ void __launch_bounds__(256) tile_mix_kernel(const int32_t* __restrict__ size,
                                                       int64_t n, int width, int limit,
                                                       const int32_t* __restrict__ route,
                                                       int32_t* __restrict__ gate) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t tiles = (n + kMixTileRows - 1) / kMixTileRows;
  int mixed = 0;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
       t < tiles; t += warps) {
    int lo = INT_MAX, hi = INT_MIN;
#pragma unroll
    for (int i = 0; i < kMixTileRows / 32; ++i) {
      const int64_t r = t * kMixTileRows + lane + 32 * i;
      if (r < n) {
        const int sz = __ldg(size + r);
        if (sz >= 0 && sz < limit) {
          const int s = __ldg(route + sz / width);
          lo = min(lo, s);
          hi = max(hi, s);
        }
      }
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    mixed += lo < hi;
  }
  if (lane == 0 && mixed) atomicAdd(&gate[0], mixed);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&gate[1], 1) == static_cast<int>(gridDim.x) - 1) {  // last block
      const int total = atomicAdd(&gate[0], 0);
      gate[2] = static_cast<int64_t>(total) * 16 > tiles ? 1 : 0;
      gate[0] = 0;
      gate[1] = 0;
      __threadfence();
    }
  }
}

cudaError_t tile_mix_launch(const int32_t* size, int64_t n, int width, int limit,
                            const int32_t* route, int32_t* gate, cudaStream_t stream) {
  const int64_t tiles = (n + kMixTileRows - 1) / kMixTileRows;
  const int64_t blocks64 = (tiles + 7) / 8;
  const int blocks = static_cast<int>(blocks64 < 148 * 8 ? blocks64 : 148 * 8);
  if (blocks == 0) return cudaSuccess;
  tile_mix_kernel<<<blocks, 256, 0, stream>>>(size, n, width, limit, route, gate);
  return cudaGetLastError();
}

int predict_box_rows(int n_classes) {
  const int CP = class_pad(n_classes);
  if (CP == 2) {
    const PredVariant& v = kCp2Variants[cp2_variant()];
    return v.R * v.NW * 32;
  }
  return CP == 4 ? 2 * 4 * 32 : 128;
}

cudaError_t predict_launch(const PredictMaps* map, PredictParams p, cudaStream_t stream,
                           int force_generic) {
  const int CP = class_pad(p.n_classes);
  static const int x_policy = [] {  // read once (thread-safe static init)  // GNB_X_POLICY=1: X loads evict_first (profiling; default normal)
    int x_policy = -1;
    const char* e = getenv("GNB_X_POLICY");
    x_policy = e ? atoi(e) : 0;
    return x_policy;
  }();
  p.x_policy = x_policy;
  p.n_tab_blocks = table_blocks(p.n_features);
  p.tab = p.prior + static_cast<int64_t>(p.n_slots) * CP;
  if (force_generic) map = nullptr;
  const bool fma = p.mode == GNB_MODE_FMA;
  switch (p.x_type) {
    case GNB_X_U16:
      return fma ? launch_typed<uint16_t, true>(map, p, CP, stream)
                 : launch_typed<uint16_t, false>(map, p, CP, stream);
    case GNB_X_U8:
      return fma ? launch_typed<uint8_t, true>(map, p, CP, stream)
                 : launch_typed<uint8_t, false>(map, p, CP, stream);
    default:
      return fma ? launch_typed<int32_t, true>(map, p, CP, stream)
                 : launch_typed<int32_t, false>(map, p, CP, stream);
  }
}

}  // namespace gnb
