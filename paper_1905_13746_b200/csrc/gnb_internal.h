// Internal launch interfaces shared by the kernel translation units and the C ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/gnb.h"

namespace gnb {

// Host narrowing of int32 rows [r0, r1) to BITS = 4 / 8 / 16 bits per count
// (narrow.cpp); false when some count does not fit.
bool narrow_rows_block(int bits, const int32_t* s, int32_t F, int64_t ldx, uint8_t* d,
                       int64_t dpitch, int64_t r0, int64_t r1);

// Records `msg` for gnb_last_error() (thread-local) and returns `code`.
int set_error(int code, const char* msg);

struct PredictParams {
  const void* x;     // generic kernel only (TMA path reads through the tensor map)
  int32_t x_type;    // GNB_X_I32 / GNB_X_U16 / GNB_X_U8
  int64_t ldx;       // row pitch in elements
  int64_t n_rows;
  int32_t n_features;
  int32_t n_chunks;  // ceil(F / features per 128-B box row), set by predict_launch
  int32_t n_tab_blocks;  // 32-feature table blocks per slot, set by predict_launch
  const int32_t* size;
  int32_t width;
  int32_t limit;
  const int32_t* route;
  int32_t n_slots;
  int32_t n_classes;
  const double* prior;  // packed: [S][CP]
  const double* tab;    // packed: [S][NB][32][CP][2], set by predict_launch
  int32_t* label;
  double* logpost;  // nullable, [N][C]
  int64_t n_tiles;  // set by predict_launch
  int32_t x_policy; // 0 evict_normal (default), 1 evict_first
  const int32_t* perm;  // nullable: rows in routed-slot order (gather mode)
  int32_t rowbox_quads;  // > 0: row-box mode, smem row = this many 16-B quads (odd)
  int32_t rowbox_stages; // row-box ring depth, set by predict_launch
  int32_t rowbox_contig; // row box: HBM row pitch == smem row pitch -> 1-D bulk tile copy
  int32_t rowbox_resident; // row box: all slot tables resident in smem, set by predict_launch
  int32_t mode;          // GNB_MODE_EXACT (reference roundings) or GNB_MODE_FMA
  int32_t mixed_rows;    // > 0: mixed-slot mode (resident tables, in-tile slot sort), tile rows
  int32_t mixed_stages;  // mixed-slot ring depth, set by predict_launch
  int32_t dep_zero;      // always 0: an opaque zero for data dependencies in SASS
  // device-side kernel gate (GNB_ORDER_AUTO): *gate = 1 when more than 1 in 16
  // of the 128-row tiles mix slots (tile_mix_launch); a gated kernel runs iff
  // *gate == gate_want
  const int32_t* gate;
  int32_t gate_want;
  // nullable: [next dynamic tile - gridDim.x, producers done]; 0 on entry, left
  // at 0 by the last producer (128-B-box kernel's dynamic tile scheduling)
  int32_t* tile_ctr;
};

struct FitParams {
  int32_t x_type;  // GNB_X_I32 / GNB_X_U16 / GNB_X_U8
  int64_t n_rows;
  int32_t n_cols;
  int32_t n_chunks;
  const int32_t* size;
  const int32_t* labels;
  int32_t width;
  int32_t limit;
  int32_t n_classes;
  int32_t n_keys;     // groups * classes
  int32_t smem_keys;  // keys [0, smem_keys) accumulate in shared memory
  double* sums;       // [G][C][V]
  double* sumsq;      // nullable
  double* counts;     // [G][C]
  unsigned long long* status;  // [2]: bad label, out of range
  int64_t n_tiles;
};

int class_pad(int n_classes);
size_t packed_bytes(int n_slots, int n_classes, int n_features);
cudaError_t pack_tables(const double* log_prior, const double* log_lik, int S, int C, int F,
                        void* packed, cudaStream_t stream);
// map == nullptr (or force_generic) selects the L1 path that accepts any ldx.
int predict_box_rows(int n_classes);  // TMA box height of the K-PRED variant
// Row-box mode (short rows): quads per box row, 0 when the shape does not use it.
// The box is then {quads * 16 / elem_bytes columns, kRowBoxRows rows}, no swizzle.
int predict_rowbox_quads(int n_features, int x_type, int n_classes);
// Mixed-slot mode (rows of many slots interleaved, every slot's table resident
// in smem): tile rows (= TMA box height), 0 when the shape does not use it.
// Batches in any row order then need no device slot sort.
int predict_mixed_rows(int n_features, int x_type, int n_classes, int n_slots);
// gate[2] = 1 when more than 1 in 16 of the 128-row tiles route their in-range
// rows to more than one slot, else 0.  gate[0..1] are scratch counters that
// must be 0 on entry and are 0 again on exit.
cudaError_t tile_mix_launch(const int32_t* size, int64_t n, int width, int limit,
                            const int32_t* route, int32_t* gate, cudaStream_t stream);
constexpr int kMixTileRows = 128;
constexpr int kRowBoxRows = 128;
// K-PRED tensor maps: `main` for every chunk; `tail` for the last chunk of a
// row in gather mode (encoded without L2 promotion, so a random row's last
// partial chunk does not drag a 256-B block of its neighbour out of HBM).
struct PredictMaps {
  CUtensorMap main;
  CUtensorMap tail;
};
cudaError_t predict_launch(const PredictMaps* maps, PredictParams p, cudaStream_t stream,
                           int force_generic);
int fit_box_rows(int x_type);  // TMA box height of K-FIT tiles
cudaError_t fit_launch(const CUtensorMap& map, FitParams p, cudaStream_t stream);

struct GenParams {
  int32_t* x;
  int64_t ldx;
  int64_t n_rows;
  int32_t n_cols;
  int32_t* size;
  int32_t* labels;
  int64_t row_offset;
  int32_t n_groups;
  int32_t width;
  int32_t n_classes;
  double divergence;
  unsigned long long seed;
  const int32_t* col_map;  // nullable: output column -> vocabulary column
  int32_t vocab_cols;
  long long group_end[128];
};
cudaError_t generate_launch(const GenParams& p, cudaStream_t stream);

cudaError_t gather_launch(const void* x, int x_type, int64_t n_rows, int32_t V, int64_t ldx,
                          const int32_t* size, int32_t width, int32_t limit,
                          const int32_t* route, const int32_t* features,
                          const int32_t* n_features, int32_t F, void* out, int64_t ldo,
                          cudaStream_t stream);

// Nibble-packed rows (GNB_X_U4, `packed_pitch` bytes per row, a multiple of 8)
// -> uint8 rows (pitch 2 * packed_pitch): the host pipeline's PCIe format.
cudaError_t unpack_u4_launch(const uint8_t* packed, int64_t n_rows, int64_t packed_pitch,
                             uint8_t* out, cudaStream_t stream);

size_t slot_sort_workspace(int64_t n, int S);
cudaError_t slot_sort(const int32_t* size, int64_t n, int width, int limit, const int32_t* route,
                      int S, int32_t* perm, void* workspace, cudaStream_t stream);

int fin_select_max_vocab();
cudaError_t fin_select_launch(const double* sums, const double* counts, int G, int V, int k,
                              int min_per_class, int32_t* state, int32_t* n_features,
                              int32_t* features, double* selected, cudaStream_t stream);

// Host helpers (api.cu)
bool encode_rows_map(CUtensorMap* map, const void* base, int64_t n_rows, int32_t n_cols,
                     int64_t ldx, int box_rows);

}  // namespace gnb
