// C ABI of libgnb.so (declared in include/gnb.h): argument checking, TMA
// tensor-map encoding, the device entry points and the host-buffer pipelines.
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <thread>
#include <tuple>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include <cudaTypedefs.h>

#include "gnb_device.cuh"
#include "gnb_internal.h"

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(GNB_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define GNB_CUDA(call, what)                   \
  do {                                          \
    cudaError_t e_ = (call);                    \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

}  // namespace

namespace gnb {
int set_error(int code, const char* msg) { return fail(code, "%s", msg); }
}  // namespace gnb

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// L2 sector promotion of the X boxes (GNB_L2_PROMO=0..3 = none/64/128/256 B, for
// profiling).  Default 256 B: measured best with evict_normal X loads
// (profiles/r01_tuning.md): the promoted neighbour sector is the same row's
// next 32-column chunk, which the next stage of the same CTA reads.
CUtensorMapL2promotion l2_promotion() {
  static const int v = [] {  // read once (thread-safe static init)
    int v = -1;
    const char* e = getenv("GNB_L2_PROMO");
    v = e ? atoi(e) : 3;
    if (v < 0 || v > 3) v = 3;
    return v;
  }();
  return static_cast<CUtensorMapL2promotion>(v);
}

// L2 promotion of the last chunk of gathered rows (GNB_GATHER_TAIL: -1 = same
// map as the other chunks, else a CUtensorMapL2promotion value; default 0).
int gather_tail_promo() {
  static const int v = [] {  // read once (thread-safe static init)
    int v = -2;
    const char* e = getenv("GNB_GATHER_TAIL");
    v = e ? atoi(e) : 0;
    if (v < -1 || v > 3) v = 0;
    return v;
  }();
  return v;
}

int elem_bytes(int x_type) { return x_type == GNB_X_U8 ? 1 : x_type == GNB_X_U16 ? 2 : 4; }

bool tma_ok(const void* base, int64_t ldx, int x_type = GNB_X_I32) {
  return (reinterpret_cast<uintptr_t>(base) & 15u) == 0 && (ldx * elem_bytes(x_type)) % 16 == 0;
}

}  // namespace

namespace gnb {

// X viewed as a 2-D int32 tensor [n_rows, n_cols] with row pitch ldx*4 bytes;
// boxes of 32 columns x box_rows rows.  swizzle128: SWIZZLE_128B (predict)
// or none (fit).
static bool encode_map(CUtensorMap* map, const void* base, int64_t n_rows, int32_t n_cols,
                       int64_t ldx, int box_rows, bool swizzle128, int x_type = GNB_X_I32,
                       int box_cols = 0, int promo = -1) {
  auto fn = encode_fn();
  if (fn == nullptr) return false;
  // cuTensorMapEncodeTiled is a driver call and needs a current context: a
  // fresh host thread has none until its first runtime call that binds the
  // primary context (cudaFree(nullptr) does, and is cheap once bound).
  static thread_local int bound_device = -1;
  int cur = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) return false;
  if (bound_device != cur) {
    if (cudaFree(nullptr) != cudaSuccess) return false;
    bound_device = cur;
  }
  const int eb = elem_bytes(x_type);
  const CUtensorMapDataType dt = x_type == GNB_X_U8    ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : x_type == GNB_X_U16 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                                       : CU_TENSOR_MAP_DATA_TYPE_INT32;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(n_cols), static_cast<cuuint64_t>(n_rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldx) * eb};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols > 0 ? box_cols : kChunkBytesPerRow / eb),
                       static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dt, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  promo >= 0 ? static_cast<CUtensorMapL2promotion>(promo) : l2_promotion(),
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_rows_map(CUtensorMap* map, const void* base, int64_t n_rows, int32_t n_cols,
                     int64_t ldx, int box_rows) {
  return encode_map(map, base, n_rows, n_cols, ldx, box_rows, true);
}

}  // namespace gnb

using namespace gnb;

static constexpr int64_t kMaxRowsPerLaunch = int64_t(1) << 30;  // TMA coordinates are int32

extern "C" {

int gnb_abi_version(void) { return 3; }

const char* gnb_strerror(int code) {
  switch (code) {
    case GNB_OK: return "ok";
    case GNB_EINVAL: return "invalid argument";
    case GNB_ECUDA: return "CUDA error";
    case GNB_EUNSUPPORTED: return "unsupported shape";
    case GNB_ENOMEM: return "out of memory";
    default: return "unknown error";
  }
}

const char* gnb_last_error(void) { return g_err; }

size_t gnb_packed_table_bytes(int32_t n_slots, int32_t n_classes, int32_t n_features) {
  if (n_slots < 1 || n_classes < 1 || n_classes > GNB_MAX_CLASSES || n_features < 1) return 0;
  return packed_bytes(n_slots, n_classes, n_features);
}

int gnb_pack_tables(const double* log_prior, const double* log_lik, int32_t n_slots,
                    int32_t n_classes, int32_t n_features, void* packed, uintptr_t stream) {
  if (n_slots < 1 || n_classes < 2 || n_classes > GNB_MAX_CLASSES || n_features < 1)
    return fail(GNB_EINVAL, "pack_tables: need n_slots>=1, 2<=n_classes<=%d, n_features>=1",
                GNB_MAX_CLASSES);
  if (!log_prior || !log_lik || !packed) return fail(GNB_EINVAL, "pack_tables: null pointer");
  if (reinterpret_cast<uintptr_t>(packed) & 15u)
    return fail(GNB_EINVAL, "pack_tables: packed buffer must be 16-byte aligned");
  GNB_CUDA(pack_tables(log_prior, log_lik, n_slots, n_classes, n_features, packed,
                       reinterpret_cast<cudaStream_t>(stream)),
           "pack_tables");
  return GNB_OK;
}

static int check_predict(const int32_t* x, int64_t n_rows, int32_t F, int64_t ldx,
                         const int32_t* size, int32_t width, int32_t limit,
                         const int32_t* route, int32_t S, int32_t C, const void* packed,
                         const int32_t* label) {
  if (n_rows < 0) return fail(GNB_EINVAL, "predict: n_rows < 0");
  if (F < 1) return fail(GNB_EINVAL, "predict: n_features must be >= 1");
  if (ldx < F) return fail(GNB_EINVAL, "predict: ldx (%lld) < n_features (%d)", (long long)ldx, F);
  if (width <= 0 || limit <= 0 || limit % width != 0)
    return fail(GNB_EINVAL, "predict: need 0 < group_size_bytes dividing max_size_bytes");
  if (S < 1) return fail(GNB_EINVAL, "predict: n_slots must be >= 1 (EmptyBundleError)");
  if (C < 2 || C > GNB_MAX_CLASSES)
    return fail(GNB_EINVAL, "predict: n_classes must be in [2, %d]", GNB_MAX_CLASSES);
  if (n_rows > 0 && (!x || !size || !label)) return fail(GNB_EINVAL, "predict: null pointer");
  if (!route || !packed) return fail(GNB_EINVAL, "predict: null route/packed");
  return GNB_OK;
}

// GNB_ROWBOX_BULK=0: row-box tiles through the 2-D tensor map even when the
// rows are contiguous (A/B of the 1-D bulk copy).
static bool rowbox_bulk() {
  static const int v = [] {  // read once (thread-safe static init)
    int v = -1;
    const char* e = getenv("GNB_ROWBOX_BULK");
    v = e ? atoi(e) != 0 : 1;
    return v;
  }();
  return v != 0;
}

// Per-(device, stream) K-PRED scratch (per host thread for cudaStreamPerThread,
// whose handle names a different stream in every thread), 8 ints, allocated
// and zeroed once, never freed:
//   [0..2] the tile-mix gate of GNB_ORDER_AUTO ([count, done, decision]); a
//          call holds `mu` while it enqueues count -> gated kernels, so calls
//          sharing a stream from several host threads cannot interleave those
//          sequences (stream order does the rest); the counting kernel leaves
//          the counters at 0;
//   [4..5] the dynamic tile counter of the 128-B-box and row-box kernels (left
//          at 0 by the last producer of each launch; launches on one stream run
//          in order).
struct Scratch {
  int32_t* dev = nullptr;
  std::mutex mu;
};
static Scratch* scratch_for(cudaStream_t stream) {
  static std::mutex mu;
  static std::map<std::tuple<int, uintptr_t, std::thread::id>, Scratch> gates;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  const std::thread::id tid =
      stream == cudaStreamPerThread ? std::this_thread::get_id() : std::thread::id();
  std::lock_guard<std::mutex> lock(mu);
  Scratch& g = gates[{dev, reinterpret_cast<uintptr_t>(stream), tid}];
  if (g.dev == nullptr) {
    if (cudaMalloc(reinterpret_cast<void**>(&g.dev), 8 * sizeof(int32_t)) != cudaSuccess) {
      g.dev = nullptr;
      return nullptr;
    }
    if (cudaMemset(g.dev, 0, 8 * sizeof(int32_t)) != cudaSuccess) {
      cudaFree(g.dev);
      g.dev = nullptr;
      return nullptr;
    }
  }
  return &g;
}

// GNB_DYNAMIC_TILES=0: static grid-stride tiles in the 128-B-box and row-box
// kernels (A/B).
static bool dynamic_tiles() {
  static const int v = [] {  // read once (thread-safe static init)
    const char* e = getenv("GNB_DYNAMIC_TILES");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

// True when predict_device will take the mixed-slot kernel (rows of any slot
// order at full speed, tables resident): no device slot sort for ragged batches.
static bool mixed_kernel(int32_t F, int x_type, int32_t C, int32_t S) {
  return predict_rowbox_quads(F, x_type, C) == 0 && predict_mixed_rows(F, x_type, C, S) > 0;
}

static int predict_device(const void* x, int x_type, int64_t n_rows, int32_t F, int64_t ldx,
                          const int32_t* size, int32_t width, int32_t limit,
                          const int32_t* route, int32_t S, int32_t C, const void* packed,
                          int32_t* label, double* logpost, cudaStream_t stream,
                          int force_generic = 0, const int32_t* perm = nullptr,
                          int mode = GNB_MODE_EXACT) {
  const bool use_tma = !force_generic && tma_ok(x, ldx, x_type) && encode_fn() != nullptr;
  if (perm != nullptr && n_rows > kMaxRowsPerLaunch)
    return fail(GNB_EUNSUPPORTED, "predict: permuted batches are limited to 2^30 rows");
  const int eb = elem_bytes(x_type);
  for (int64_t r0 = 0; r0 < n_rows; r0 += kMaxRowsPerLaunch) {
    const int64_t n = std::min(kMaxRowsPerLaunch, n_rows - r0);
    PredictParams p{};
    p.x = static_cast<const uint8_t*>(x) + r0 * ldx * eb;
    p.x_type = x_type;
    p.ldx = ldx;
    p.n_rows = n;
    p.n_features = F;
    p.size = size + r0;
    p.width = width;
    p.limit = limit;
    p.route = route;
    p.n_slots = S;
    p.n_classes = C;
    p.prior = static_cast<const double*>(packed);
    p.label = label + r0;
    p.logpost = logpost ? logpost + r0 * C : nullptr;
    p.perm = use_tma ? perm : nullptr;  // the L1 kernel walks rows in order
    p.mode = mode & 0xF;
    const int order = mode & (GNB_ORDER_GROUPED | GNB_ORDER_MIXED);
    PredictMaps map;
    const PredictMaps* mp = nullptr;
    if (use_tma && dynamic_tiles()) {
      Scratch* sg = scratch_for(stream);
      if (sg == nullptr) return fail(GNB_ENOMEM, "predict: scratch allocation failed");
      p.tile_ctr = sg->dev + 4;
    }
    if (use_tma) {
      // row-box mode (short rows): whole rows per box, unswizzled; gather mode:
      // box height 1 (tile::gather4 loads 4 rows per instruction)
      // mixed-slot mode (>= 2 slots whose tables fit in smem): box height = its tile
      // (short rows keep the row-box kernel, which has resident tables too)
      const int wq = perm ? 0 : predict_rowbox_quads(F, x_type, C);
      const int mr = perm || wq > 0 || order == GNB_ORDER_GROUPED
                         ? 0
                         : predict_mixed_rows(F, x_type, C, S);
      if (mr > 0 && order == GNB_ORDER_AUTO) {
        // Row order unknown: count the 128-row tiles that mix slots on the
        // device and launch both kernels gated on that count (the one not
        // chosen exits at once) -- no host round trip.
        PredictMaps mmap, gmap;
        if (!encode_map(&mmap.main, p.x, n, F, ldx, mr, true, x_type) ||
            !encode_map(&gmap.main, p.x, n, F, ldx, predict_box_rows(C), true, x_type))
          return fail(GNB_ECUDA, "predict: cuTensorMapEncodeTiled failed");
        mmap.tail = mmap.main;
        gmap.tail = gmap.main;
        Scratch* gate = scratch_for(stream);
        if (gate == nullptr) return fail(GNB_ENOMEM, "predict: gate counter allocation failed");
        std::lock_guard<std::mutex> gate_lock(gate->mu);
        int32_t* cnt = gate->dev;
        GNB_CUDA(tile_mix_launch(p.size, n, width, limit, route, cnt, stream), "tile_mix");
        PredictParams pm = p, pg = p;
        pm.mixed_rows = mr;
        pg.mixed_rows = 0;
        pm.gate = pg.gate = cnt + 2;
        pm.gate_want = 1;
        pg.gate_want = 0;
        GNB_CUDA(predict_launch(&mmap, pm, stream, force_generic), "predict launch");
        GNB_CUDA(predict_launch(&gmap, pg, stream, force_generic), "predict launch");
        continue;
      }
      bool ok = wq > 0 ? encode_map(&map.main, p.x, n, F, ldx, kRowBoxRows, false, x_type,
                                    wq * 16 / eb)
                       : encode_map(&map.main, p.x, n, F, ldx,
                                    perm ? 1 : mr > 0 ? mr : predict_box_rows(C), true, x_type);
      map.tail = map.main;
      if (ok && perm && gather_tail_promo() >= 0)
        ok = encode_map(&map.tail, p.x, n, F, ldx, 1, true, x_type, 0, gather_tail_promo());
      if (!ok) return fail(GNB_ECUDA, "predict: cuTensorMapEncodeTiled failed");
      p.rowbox_quads = wq;
      p.mixed_rows = mr;
      p.rowbox_contig = wq > 0 && ldx * eb == int64_t(wq) * 16 && rowbox_bulk();
      mp = &map;
    }
    GNB_CUDA(predict_launch(mp, p, stream, force_generic), "predict launch");
  }
  return GNB_OK;
}

int gnb_predict(const int32_t* x, int64_t n_rows, int32_t n_features, int64_t ldx,
                const int32_t* size_bytes, int32_t group_size_bytes, int32_t max_size_bytes,
                const int32_t* route, int32_t n_slots, int32_t n_classes, const void* packed,
                int32_t* label_out, double* logpost_out, uintptr_t stream) {
  int rc = check_predict(x, n_rows, n_features, ldx, size_bytes, group_size_bytes,
                         max_size_bytes, route, n_slots, n_classes, packed, label_out);
  if (rc) return rc;
  return predict_device(x, GNB_X_I32, n_rows, n_features, ldx, size_bytes, group_size_bytes,
                        max_size_bytes, route, n_slots, n_classes, packed, label_out,
                        logpost_out, reinterpret_cast<cudaStream_t>(stream));
}

int gnb_predict_typed(const void* x, int32_t x_type, int64_t n_rows, int32_t n_features,
                      int64_t ldx, const int32_t* size_bytes, int32_t group_size_bytes,
                      int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                      int32_t n_classes, const void* packed, int32_t* label_out,
                      double* logpost_out, uintptr_t stream) {
  if (x_type != GNB_X_I32 && x_type != GNB_X_U16 && x_type != GNB_X_U8)
    return fail(GNB_EINVAL, "predict: unknown x_type %d", x_type);
  int rc = check_predict(static_cast<const int32_t*>(x), n_rows, n_features, ldx, size_bytes,
                         group_size_bytes, max_size_bytes, route, n_slots, n_classes, packed,
                         label_out);
  if (rc) return rc;
  return predict_device(x, x_type, n_rows, n_features, ldx, size_bytes, group_size_bytes,
                        max_size_bytes, route, n_slots, n_classes, packed, label_out,
                        logpost_out, reinterpret_cast<cudaStream_t>(stream));
}

int gnb_fin_train_device(const double* sums, const double* counts, int32_t n_groups,
                         int32_t n_cols, int32_t k, double alpha, int32_t min_per_class,
                         int32_t* group_state, int32_t* n_features, int32_t* features,
                         double* log_prior, double* log_lik, uintptr_t stream_) {
  if (!sums || !counts || !group_state || !n_features || !features || !log_prior || !log_lik)
    return fail(GNB_EINVAL, "fin_train_device: null pointer");
  if (n_groups < 1 || n_cols < 1 || k < 1 || !(alpha > 0.0) || min_per_class < 1)
    return fail(GNB_EINVAL, "fin_train_device: bad arguments");
  if (n_cols > fin_select_max_vocab())
    return fail(GNB_EUNSUPPORTED, "fin_train_device: vocabulary above %d columns",
                fin_select_max_vocab());
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const size_t G = static_cast<size_t>(n_groups);
  int32_t* d_i32 = nullptr;
  double* d_sel = nullptr;
  GNB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_i32), (2 + size_t(k)) * G * 4, stream),
           "malloc");
  GNB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_sel), 2 * size_t(k) * G * 8, stream),
           "malloc");
  int32_t* d_state = d_i32;
  int32_t* d_nf = d_i32 + G;
  int32_t* d_feat = d_i32 + 2 * G;
  cudaError_t e = fin_select_launch(sums, counts, n_groups, n_cols, k, min_per_class, d_state,
                                    d_nf, d_feat, d_sel, stream);
  std::vector<double> sel(2 * size_t(k) * G), cnt(2 * G);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(group_state, d_state, G * 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(n_features, d_nf, G * 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(features, d_feat, G * size_t(k) * 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(sel.data(), d_sel, sel.size() * 8, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(cnt.data(), counts, cnt.size() * 8, cudaMemcpyDeviceToHost, stream);
  cudaFreeAsync(d_i32, stream);
  cudaFreeAsync(d_sel, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_fail(e, "fin_train_device");
  // libm logarithms on the host (bit-identical to CPython's math.log)
  std::vector<int32_t> iota(static_cast<size_t>(k));
  for (int j = 0; j < k; ++j) iota[j] = j;
  std::vector<double> lik(2 * size_t(k));
  for (size_t g = 0; g < G; ++g) {
    std::fill(log_prior + 2 * g, log_prior + 2 * g + 2, 0.0);
    std::fill(log_lik + 2 * g * k, log_lik + 2 * (g + 1) * k, 0.0);
    if (group_state[g] != 1) {
      std::fill(features + g * k, features + (g + 1) * k, 0);
      continue;
    }
    const int F = n_features[g];
    const double* sg = sel.data() + 2 * g * k;  // [2][k]
    std::vector<double> s2(2 * size_t(F));
    for (int c = 0; c < 2; ++c)
      for (int j = 0; j < F; ++j) s2[c * F + j] = sg[c * k + j];
    gnb_fin_tables(s2.data(), cnt.data() + 2 * g, 2, F, iota.data(), F, alpha, log_prior + 2 * g,
                   lik.data());
    for (int c = 0; c < 2; ++c)
      for (int j = 0; j < F; ++j) log_lik[(2 * g + c) * k + j] = lik[c * size_t(F) + j];
  }
  return GNB_OK;
}

int32_t gnb_predict_mixed_rows(int32_t n_features, int32_t x_type, int32_t n_classes,
                               int32_t n_slots) {
  if (n_features < 1 || n_classes < 2 || n_classes > GNB_MAX_CLASSES || n_slots < 1) return 0;
  if (x_type != GNB_X_I32 && x_type != GNB_X_U16 && x_type != GNB_X_U8) return 0;
  if (!mixed_kernel(n_features, x_type, n_classes, n_slots)) return 0;
  return predict_mixed_rows(n_features, x_type, n_classes, n_slots);
}

size_t gnb_slot_sort_workspace_bytes(int64_t n_rows, int32_t n_slots) {
  if (n_rows < 0 || n_slots < 1) return 0;
  return slot_sort_workspace(n_rows, n_slots);
}

int gnb_slot_sort(const int32_t* size_bytes, int64_t n_rows, int32_t group_size_bytes,
                  int32_t max_size_bytes, const int32_t* route, int32_t n_slots, int32_t* perm,
                  void* workspace, size_t workspace_bytes, uintptr_t stream) {
  if (n_rows < 0 || n_rows > kMaxRowsPerLaunch || n_slots < 1 || n_slots >= 4096 ||
      group_size_bytes <= 0 || max_size_bytes <= 0 || max_size_bytes % group_size_bytes)
    return fail(GNB_EINVAL, "slot_sort: bad geometry (n_rows <= 2^30, n_slots < 4096)");
  if (n_rows > 0 && (!size_bytes || !route || !perm || !workspace))
    return fail(GNB_EINVAL, "slot_sort: null pointer");
  if (workspace_bytes < slot_sort_workspace(n_rows, n_slots))
    return fail(GNB_EINVAL, "slot_sort: workspace too small");
  GNB_CUDA(slot_sort(size_bytes, n_rows, group_size_bytes, max_size_bytes, route, n_slots, perm,
                     workspace, reinterpret_cast<cudaStream_t>(stream)),
           "slot_sort");
  return GNB_OK;
}

int gnb_predict_permuted(const void* x, int32_t x_type, int64_t n_rows, int32_t n_features,
                         int64_t ldx, const int32_t* size_bytes, int32_t group_size_bytes,
                         int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                         int32_t n_classes, const void* packed, const int32_t* perm,
                         int32_t* label_out, double* logpost_out, uintptr_t stream) {
  if (x_type != GNB_X_I32 && x_type != GNB_X_U16 && x_type != GNB_X_U8)
    return fail(GNB_EINVAL, "predict: unknown x_type %d", x_type);
  int rc = check_predict(static_cast<const int32_t*>(x), n_rows, n_features, ldx, size_bytes,
                         group_size_bytes, max_size_bytes, route, n_slots, n_classes, packed,
                         label_out);
  if (rc) return rc;
  if (n_rows > 0 && !perm) return fail(GNB_EINVAL, "predict_permuted: null perm");
  return predict_device(x, x_type, n_rows, n_features, ldx, size_bytes, group_size_bytes,
                        max_size_bytes, route, n_slots, n_classes, packed, label_out,
                        logpost_out, reinterpret_cast<cudaStream_t>(stream), 0, perm);
}

int gnb_predict_mode(const void* x, int32_t x_type, int64_t n_rows, int32_t n_features,
                     int64_t ldx, const int32_t* size_bytes, int32_t group_size_bytes,
                     int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                     int32_t n_classes, const void* packed, const int32_t* perm, int32_t mode,
                     int32_t* label_out, double* logpost_out, uintptr_t stream) {
  if (x_type != GNB_X_I32 && x_type != GNB_X_U16 && x_type != GNB_X_U8)
    return fail(GNB_EINVAL, "predict: unknown x_type %d", x_type);
  const int arith = mode & 0xF, order = mode & ~0xF;
  if ((arith != GNB_MODE_EXACT && arith != GNB_MODE_FMA) ||
      (order != GNB_ORDER_AUTO && order != GNB_ORDER_GROUPED && order != GNB_ORDER_MIXED))
    return fail(GNB_EINVAL, "predict: unknown mode %d", mode);
  int rc = check_predict(static_cast<const int32_t*>(x), n_rows, n_features, ldx, size_bytes,
                         group_size_bytes, max_size_bytes, route, n_slots, n_classes, packed,
                         label_out);
  if (rc) return rc;
  return predict_device(x, x_type, n_rows, n_features, ldx, size_bytes, group_size_bytes,
                        max_size_bytes, route, n_slots, n_classes, packed, label_out,
                        logpost_out, reinterpret_cast<cudaStream_t>(stream), 0, perm, mode);
}

// Test hook: force the L1 (non-TMA) predict kernel.
int gnb_predict_generic(const int32_t* x, int64_t n_rows, int32_t n_features, int64_t ldx,
                        const int32_t* size_bytes, int32_t group_size_bytes,
                        int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                        int32_t n_classes, const void* packed, int32_t* label_out,
                        double* logpost_out, uintptr_t stream) {
  int rc = check_predict(x, n_rows, n_features, ldx, size_bytes, group_size_bytes,
                         max_size_bytes, route, n_slots, n_classes, packed, label_out);
  if (rc) return rc;
  return predict_device(x, GNB_X_I32, n_rows, n_features, ldx, size_bytes, group_size_bytes,
                        max_size_bytes, route, n_slots, n_classes, packed, label_out,
                        logpost_out, reinterpret_cast<cudaStream_t>(stream), 1);
}

static int fit_stats_device(const void* x, int x_type, int64_t n_rows, int32_t n_cols,
                            int64_t ldx, const int32_t* size_bytes, const int32_t* labels,
                            int32_t group_size_bytes, int32_t max_size_bytes, int32_t n_classes,
                            double* sums, double* sumsq, double* counts,
                            unsigned long long* status, int32_t accumulate, cudaStream_t stream) {
  if (n_rows < 0 || n_cols < 1 || ldx < n_cols)
    return fail(GNB_EINVAL, "fit_stats: need n_rows>=0, n_cols>=1, ldx>=n_cols");
  if (group_size_bytes <= 0 || max_size_bytes <= 0 || max_size_bytes % group_size_bytes)
    return fail(GNB_EINVAL, "fit_stats: need 0 < group_size_bytes dividing max_size_bytes");
  if (n_classes < 2 || n_classes > GNB_MAX_CLASSES)
    return fail(GNB_EINVAL, "fit_stats: n_classes must be in [2, %d]", GNB_MAX_CLASSES);
  if (x_type != GNB_X_I32 && x_type != GNB_X_U16 && x_type != GNB_X_U8)
    return fail(GNB_EINVAL, "fit_stats: unknown x_type %d", x_type);
  if (!sums || !counts) return fail(GNB_EINVAL, "fit_stats: null output");
  if (n_rows > 0 && (!x || !size_bytes || !labels)) return fail(GNB_EINVAL, "fit_stats: null input");
  if (n_rows > 0 && !tma_ok(x, ldx, x_type))
    return fail(GNB_EUNSUPPORTED, "fit_stats: X must be 16-byte aligned with a 16-byte row pitch");
  const int64_t G = max_size_bytes / group_size_bytes;
  const int64_t keys = G * n_classes;
  if (keys > (int64_t(1) << 30)) return fail(GNB_EINVAL, "fit_stats: too many groups");
  if (!accumulate) {
    GNB_CUDA(cudaMemsetAsync(sums, 0, keys * n_cols * sizeof(double), stream), "memset");
    if (sumsq) GNB_CUDA(cudaMemsetAsync(sumsq, 0, keys * n_cols * sizeof(double), stream), "memset");
    GNB_CUDA(cudaMemsetAsync(counts, 0, keys * sizeof(double), stream), "memset");
    if (status) GNB_CUDA(cudaMemsetAsync(status, 0, 2 * sizeof(unsigned long long), stream), "memset");
  }
  const int eb = elem_bytes(x_type);
  for (int64_t r0 = 0; r0 < n_rows; r0 += kMaxRowsPerLaunch) {
    const int64_t n = std::min(kMaxRowsPerLaunch, n_rows - r0);
    CUtensorMap map;
    const void* xr = static_cast<const uint8_t*>(x) + r0 * ldx * eb;
    if (!encode_map(&map, xr, n, n_cols, ldx, fit_box_rows(x_type), false, x_type))
      return fail(GNB_ECUDA, "fit_stats: cuTensorMapEncodeTiled failed");
    FitParams p{};
    p.x_type = x_type;
    p.n_rows = n;
    p.n_cols = n_cols;
    p.size = size_bytes + r0;
    p.labels = labels + r0;
    p.width = group_size_bytes;
    p.limit = max_size_bytes;
    p.n_classes = n_classes;
    p.n_keys = static_cast<int32_t>(keys);
    p.sums = sums;
    p.sumsq = sumsq;
    p.counts = counts;
    p.status = status;
    GNB_CUDA(fit_launch(map, p, stream), "fit launch");
  }
  return GNB_OK;
}

int gnb_fit_stats(const int32_t* x, int64_t n_rows, int32_t n_cols, int64_t ldx,
                  const int32_t* size_bytes, const int32_t* labels, int32_t group_size_bytes,
                  int32_t max_size_bytes, int32_t n_classes, double* sums, double* sumsq,
                  double* counts, unsigned long long* status, int32_t accumulate,
                  uintptr_t stream) {
  return fit_stats_device(x, GNB_X_I32, n_rows, n_cols, ldx, size_bytes, labels,
                          group_size_bytes, max_size_bytes, n_classes, sums, sumsq, counts, status,
                          accumulate, reinterpret_cast<cudaStream_t>(stream));
}

int gnb_fit_stats_typed(const void* x, int32_t x_type, int64_t n_rows, int32_t n_cols,
                        int64_t ldx, const int32_t* size_bytes, const int32_t* labels,
                        int32_t group_size_bytes, int32_t max_size_bytes, int32_t n_classes,
                        double* sums, double* sumsq, double* counts, unsigned long long* status,
                        int32_t accumulate, uintptr_t stream) {
  return fit_stats_device(x, x_type, n_rows, n_cols, ldx, size_bytes, labels, group_size_bytes,
                          max_size_bytes, n_classes, sums, sumsq, counts, status, accumulate,
                          reinterpret_cast<cudaStream_t>(stream));
}

int gnb_generate(int32_t* x, int64_t n_rows, int32_t n_cols, int64_t ldx, int32_t* size_bytes,
                 int32_t* labels, int64_t row_offset, const int64_t* group_row_end,
                 int32_t n_groups, int32_t group_size_bytes, int32_t n_classes,
                 double divergence, uint64_t seed, const int32_t* col_map,
                 int32_t vocab_cols, uintptr_t stream) {
  if (col_map == nullptr) vocab_cols = n_cols;
  if (n_rows < 0 || n_cols < 1 || ldx < n_cols || n_groups < 1 || n_groups > 128 ||
      vocab_cols < 1 ||
      group_size_bytes < 1 || n_classes < 2 || n_classes > GNB_MAX_CLASSES ||
      !(divergence >= 0.0 && divergence <= 1.0))
    return fail(GNB_EINVAL, "generate: bad arguments");
  if (n_rows > 0 && (!x || !size_bytes || !labels || !group_row_end))
    return fail(GNB_EINVAL, "generate: null pointer");
  GenParams p{};
  p.x = x;
  p.ldx = ldx;
  p.n_rows = n_rows;
  p.n_cols = n_cols;
  p.size = size_bytes;
  p.labels = labels;
  p.row_offset = row_offset;
  p.n_groups = n_groups;
  p.width = group_size_bytes;
  p.n_classes = n_classes;
  p.divergence = divergence;
  p.seed = seed;
  p.col_map = col_map;
  p.vocab_cols = vocab_cols;
  for (int g = 0; g < n_groups; ++g) p.group_end[g] = group_row_end[g];
  GNB_CUDA(generate_launch(p, reinterpret_cast<cudaStream_t>(stream)), "generate launch");
  return GNB_OK;
}

int gnb_gather_features_typed(const void* x_vocab, int32_t x_type, int64_t n_rows,
                              int32_t n_vocab, int64_t ldx, const int32_t* size_bytes,
                              int32_t group_size_bytes, int32_t max_size_bytes,
                              const int32_t* route, const int32_t* features,
                              const int32_t* n_features, int32_t n_slots, int32_t max_features,
                              void* x_out, int64_t ldo, uintptr_t stream) {
  if (x_type != GNB_X_I32 && x_type != GNB_X_U16 && x_type != GNB_X_U8)
    return fail(GNB_EINVAL, "gather_features: unknown x_type %d", x_type);
  if (n_rows < 0 || n_vocab < 1 || ldx < n_vocab || max_features < 1 || ldo < max_features ||
      n_slots < 1 || group_size_bytes <= 0 || max_size_bytes <= 0 ||
      max_size_bytes % group_size_bytes)
    return fail(GNB_EINVAL, "gather_features: bad geometry");
  if (n_rows > 0 && (!x_vocab || !size_bytes || !x_out))
    return fail(GNB_EINVAL, "gather_features: null pointer");
  if (!route || !features || !n_features) return fail(GNB_EINVAL, "gather_features: null table");
  GNB_CUDA(gather_launch(x_vocab, x_type, n_rows, n_vocab, ldx, size_bytes, group_size_bytes,
                         max_size_bytes, route, features, n_features, max_features, x_out, ldo,
                         reinterpret_cast<cudaStream_t>(stream)),
           "gather launch");
  return GNB_OK;
}

int gnb_gather_features(const int32_t* x_vocab, int64_t n_rows, int32_t n_vocab, int64_t ldx,
                        const int32_t* size_bytes, int32_t group_size_bytes,
                        int32_t max_size_bytes, const int32_t* route, const int32_t* features,
                        const int32_t* n_features, int32_t n_slots, int32_t max_features,
                        int32_t* x_out, int64_t ldo, uintptr_t stream) {
  return gnb_gather_features_typed(x_vocab, GNB_X_I32, n_rows, n_vocab, ldx, size_bytes,
                                   group_size_bytes, max_size_bytes, route, features, n_features,
                                   n_slots, max_features, x_out, ldo, stream);
}

}  // extern "C"

// ---------------------------------------------------------------- host pipelines
namespace {

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) n = bytes;
    return e;
  }
};

struct PinBuf {  // page-locked host staging
  void* p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocDefault);
    if (e == cudaSuccess) n = bytes;
    return e;
  }
};

// Minimal fork-join pool for the host-side narrowing of X (one job at a time).
class Pool {
 public:
  explicit Pool(int n) : n_(n) {
    for (int i = 0; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return n_; }
  void run(const std::function<void(int)>& f) {  // f(worker), blocks until all finish
    start(f);
    wait();
  }
  // start(f): every worker runs f(worker) while the caller goes on; wait()
  // blocks until they all finished.  f must outlive the wait().
  void start(const std::function<void(int)>& f) {
    std::lock_guard<std::mutex> g(m_);
    job_ = &f;
    pending_ = n_;
    ++gen_;
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int i) {
    int seen = 0;
    for (;;) {
      const std::function<void(int)>* f;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        f = job_;
      }
      (*f)(i);
      std::lock_guard<std::mutex> g(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int pending_ = 0, gen_ = 0;
  bool stop_ = false;
};

constexpr int kLanes = 3;  // chunk pipeline depth (streams)
// int32 host rows in page-locked memory: every 3rd chunk goes raw by DMA, two
// are narrowed on host threads -- 111M vs 79M rows/s at F=256 on the B200 box
// (raw every 2nd / 4th: 89M / 100M; tools/e2e_hybrid_ab.sh).
constexpr int64_t kHostRawEvery = 3;

struct HostCtx {
  int device = -1;
  cudaStream_t s[kLanes] = {};
  cudaEvent_t ev[kLanes] = {};
  cudaEvent_t copied[kLanes] = {};  // staging buffer of the lane may be reused
  DevBuf x[kLanes], size[kLanes], aux[kLanes], label[kLanes], logpost[kLanes];
  DevBuf perm[kLanes], sortws[kLanes], x4[kLanes];
  PinBuf stage[kLanes];
  DevBuf route, prior, lik, packed, sums, sumsq, counts, status;
  Pool* pool = nullptr;
};

thread_local std::vector<HostCtx*> g_ctx;

int get_ctx(int device, HostCtx** out) {
  for (HostCtx* c : g_ctx)
    if (c->device == device) {
      *out = c;
      return GNB_OK;
    }
  auto* c = new HostCtx();
  c->device = device;
  for (int i = 0; i < kLanes; ++i) {
    GNB_CUDA(cudaStreamCreateWithFlags(&c->s[i], cudaStreamNonBlocking), "stream create");
    GNB_CUDA(cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming), "event create");
    GNB_CUDA(cudaEventCreateWithFlags(&c->copied[i], cudaEventDisableTiming), "event create");
  }
  g_ctx.push_back(c);
  *out = c;
  return GNB_OK;
}

// Host-side narrowing of int32 rows (lossless, chosen per pipeline chunk):
// the narrowest storage that holds every count of the chunk -- GNB_X_U4 (two
// counts per byte, < 16), GNB_X_U8, GNB_X_U16 -- written into pinned staging
// in one pass over the int32 rows per attempted width (each worker stops its
// attempt at the first 16-row block that does not fit).  int32 rows cost
// 1024 B/row of host DRAM reads either way (the C port's cost too); what the
// narrowing buys is 2-8x fewer bytes over PCIe, so e2e on int32 host buffers
// is bound by host memory bandwidth instead of the ~55 GB/s link.
// Returns the x_type written, or GNB_X_I32 when no narrow width holds the
// chunk (negative or >= 65536 counts): the caller then ships int32 rows.
// One chunk's narrowing, run by the pool in the background while the calling
// thread issues the previous chunk's copies and kernels: the 4-bit attempt is
// started asynchronously (start); finish() waits for it and, only if some count
// did not fit, retries 8 / 16 bits synchronously.
struct NarrowJob {
  const int32_t* src = nullptr;
  int64_t n = 0, ldx = 0, ld8 = 0, ld16 = 0;
  int32_t F = 0;
  uint8_t* dst = nullptr;
  int bits = 4;
  std::atomic<uint32_t> bad{0};
  std::function<void(int)> fn;
  int W = 1;

  void attempt(Pool& pool, int b, bool async) {
    bits = b;
    bad.store(0u);
    W = pool.size();
    const int64_t pitch = b == 4 ? ld8 / 2 : b == 8 ? ld8 : ld16 * 2;
    fn = [this, pitch](int w) {
      const int64_t lo = n * w / W, hi = n * (w + 1) / W;
      for (int64_t r = lo; r < hi; r += 64) {
        if (bad.load(std::memory_order_relaxed)) return;
        if (!narrow_rows_block(bits, src, F, ldx, dst, pitch, r, std::min<int64_t>(r + 64, hi))) {
          bad.store(1u, std::memory_order_relaxed);
          return;
        }
      }
    };
    if (async) pool.start(fn);
    else pool.run(fn);
  }
  // the x_type written: GNB_X_U4 / U8 / U16, or GNB_X_I32 (nothing fits)
  int finish(Pool& pool) {
    pool.wait();
    if (bits == 4 && bad.load() == 0) return GNB_X_U4;
    attempt(pool, 8, false);
    if (bad.load() == 0) return GNB_X_U8;
    attempt(pool, 16, false);
    return bad.load() == 0 ? GNB_X_U16 : GNB_X_I32;
  }
};

// GNB_HOST_NARROW=0 ships int32 host rows as they are (A/B); default on.
bool narrowing_enabled() {  // read per call (once per host pipeline call)
  const char* e = getenv("GNB_HOST_NARROW");
  return e == nullptr || atoi(e) != 0;
}

// MiB of X crossing PCIe per pipeline chunk (GNB_HOST_CHUNK_MB, read once).
int64_t host_chunk_bytes() {  // read per host pipeline call
  const char* e = getenv("GNB_HOST_CHUNK_MB");
  const int64_t mb = e ? atoll(e) : 64;
  return (mb >= 1 && mb <= 4096 ? mb : 64) << 20;
}

int64_t chunk_rows_for(int64_t row_bytes) {
  const int64_t target = host_chunk_bytes();
  int64_t r = std::max<int64_t>(1024, target / std::max<int64_t>(row_bytes, 1));
  return (r + 127) / 128 * 128;
}

}  // namespace

extern "C" {

}  // extern "C"

static int predict_host_impl(const void* xv, int x_type, int64_t n_rows, int32_t n_features,
                             int64_t ldx, const int32_t* size_bytes, int32_t group_size_bytes,
                             int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                             int32_t n_classes, const double* log_prior, const double* log_lik,
                             int32_t* label_out, double* logpost_out, int32_t device,
                             int64_t* elapsed_ns) {
  auto t0 = std::chrono::steady_clock::now();
  const int32_t* x = static_cast<const int32_t*>(xv);  // int32 view (x_type == GNB_X_I32)
  int rc = check_predict(x, n_rows, n_features, ldx, size_bytes, group_size_bytes,
                         max_size_bytes, route, n_slots, n_classes, log_prior, label_out);
  if (rc) return rc;
  if (!log_lik) return fail(GNB_EINVAL, "predict_host: null log_lik");
  GNB_CUDA(cudaSetDevice(device), "cudaSetDevice");
  HostCtx* c = nullptr;
  if ((rc = get_ctx(device, &c))) return rc;
  const int G = max_size_bytes / group_size_bytes;
  const size_t prior_b = size_t(n_slots) * n_classes * 8;
  const size_t lik_b = prior_b * n_features;
  const size_t packed_b = packed_bytes(n_slots, n_classes, n_features);
  GNB_CUDA(c->route.ensure(size_t(G) * 4), "malloc");
  GNB_CUDA(c->prior.ensure(prior_b), "malloc");
  GNB_CUDA(c->lik.ensure(lik_b), "malloc");
  GNB_CUDA(c->packed.ensure(packed_b), "malloc");
  cudaStream_t s0 = c->s[0];
  GNB_CUDA(cudaMemcpyAsync(c->route.p, route, size_t(G) * 4, cudaMemcpyHostToDevice, s0), "H2D");
  GNB_CUDA(cudaMemcpyAsync(c->prior.p, log_prior, prior_b, cudaMemcpyHostToDevice, s0), "H2D");
  GNB_CUDA(cudaMemcpyAsync(c->lik.p, log_lik, lik_b, cudaMemcpyHostToDevice, s0), "H2D");
  GNB_CUDA(pack_tables(static_cast<double*>(c->prior.p), static_cast<double*>(c->lik.p),
                       n_slots, n_classes, n_features, c->packed.p, s0),
           "pack");
  GNB_CUDA(cudaEventRecord(c->ev[0], s0), "event");
  for (int i = 1; i < kLanes; ++i) GNB_CUDA(cudaStreamWaitEvent(c->s[i], c->ev[0], 0), "wait");

  // Rows cross PCIe in the caller's storage (uint16 / uint8 / nibbles); int32
  // input is narrowed per chunk by host threads into pinned staging first
  // (narrow_chunk: lossless, chunks that fit no narrow width stay int32).
  const int64_t ld = (n_features + 3) / 4 * 4;  // device rows padded for TMA (int32)
  const int64_t ld8 = (n_features + 15) / 16 * 16, ld16 = (n_features + 7) / 8 * 8;
  // chunk rows from the bytes each row moves over PCIe; device rows as stored
  const int64_t wire_b = x_type == GNB_X_U4 ? ld8 / 2 : x_type == GNB_X_U8 ? ld8
                         : x_type == GNB_X_U16 ? ld16 * 2 : ld * 4;
  const int64_t dev_b = x_type == GNB_X_U4 || x_type == GNB_X_U8 ? ld8
                        : x_type == GNB_X_U16 ? ld16 * 2 : ld * 4;
  const int64_t rows = std::min<int64_t>(chunk_rows_for(wire_b), std::max<int64_t>(n_rows, 1));
  const bool narrow = x_type == GNB_X_I32 && narrowing_enabled();
  if (narrow && c->pool == nullptr) {
    const unsigned hw = std::thread::hardware_concurrency();
    c->pool = new Pool(static_cast<int>(hw > 0 ? std::min(hw, 64u) : 4u));
  }
  for (int i = 0; i < kLanes; ++i) {
    GNB_CUDA(c->x[i].ensure(size_t(rows) * dev_b), "malloc");
    if (narrow) GNB_CUDA(c->stage[i].ensure(size_t(rows) * ld16 * 2), "cudaHostAlloc");
    if (x_type == GNB_X_U4 || narrow) GNB_CUDA(c->x4[i].ensure(size_t(rows) * ld8 / 2), "malloc");
    GNB_CUDA(c->size[i].ensure(size_t(rows) * 4), "malloc");
    GNB_CUDA(c->label[i].ensure(size_t(rows) * 4), "malloc");
    if (logpost_out) GNB_CUDA(c->logpost[i].ensure(size_t(rows) * n_classes * 8), "malloc");
  }
  // The clock starts once the context's buffers exist (the reference, too,
  // builds its worker pool before its timer, engine.py:273-285): a first call
  // -- or one larger than any before -- allocates device buffers here.
  if (elapsed_ns) t0 = std::chrono::steady_clock::now();
  // GNB_HOST_TIMING=1: per-call breakdown of the host side on stderr (profiling)
  const char* te = getenv("GNB_HOST_TIMING");
  const bool timing = te != nullptr && atoi(te) != 0;
  double t_wait = 0.0, t_narrow = 0.0;
  NarrowJob jobs[2];
  // an error return must not leave pool workers writing through `jobs`
  struct PoolDrain {
    Pool* p;
    ~PoolDrain() {
      if (p) p->wait();
    }
  } drain{narrow ? c->pool : nullptr};
  auto start_narrow = [&](int64_t k, int lane_k, int slot) {
    NarrowJob& j = jobs[slot];
    j.src = x + k * rows * ldx;
    j.n = std::min(rows, n_rows - k * rows);
    j.F = n_features;
    j.ldx = ldx;
    j.ld8 = ld8;
    j.ld16 = ld16;
    j.dst = static_cast<uint8_t*>(c->stage[lane_k].p);
    j.attempt(*c->pool, 4, true);
  };
  // Hybrid split of int32 chunks (GNB_HOST_RAW_EVERY=N: every N-th chunk is
  // copied as raw int32 rows by the DMA engine while host threads narrow the
  // others -- the copy engine reads host memory without any CPU, so both paths
  // draw on host DRAM bandwidth at once).  0 = narrow every chunk.
  // Only for page-locked input: from pageable memory the driver stages the
  // copy through its own buffers on the CPU, which is slower than narrowing.
  const char* re = getenv("GNB_HOST_RAW_EVERY");
  int64_t raw_every = re ? atoll(re) : kHostRawEvery;
  if (narrow && raw_every > 0) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, x) != cudaSuccess || pa.type != cudaMemoryTypeHost) {
      cudaGetLastError();  // clear a non-sticky "not a CUDA pointer" error
      raw_every = 0;
    }
  }
  const int64_t n_chunks = (n_rows + rows - 1) / rows;
  auto narrow_chunk_k = [&](int64_t k) {
    return narrow && !(raw_every > 0 && k % raw_every == raw_every - 1);
  };
  auto next_narrow = [&](int64_t k) -> int64_t {
    for (int64_t k2 = k + 1; k2 < n_chunks; ++k2)
      if (narrow_chunk_k(k2)) return k2;
    return -1;
  };
  int pend_slot = 0;
  if (narrow && n_rows > 0) {
    const int64_t first = next_narrow(-1);
    if (first >= 0) {
      GNB_CUDA(cudaEventSynchronize(c->copied[first % kLanes]), "event sync");
      start_narrow(first, static_cast<int>(first % kLanes), pend_slot);
    }
  }
  int64_t chunk = 0;
  for (int64_t r0 = 0; r0 < n_rows; r0 += rows, ++chunk) {
    const int lane = static_cast<int>(chunk % kLanes);
    cudaStream_t s = c->s[lane];
    const int64_t n = std::min(rows, n_rows - r0);
    void* dx = c->x[lane].p;
    int xt = GNB_X_I32;
    int64_t dld = ld;
    if (x_type == GNB_X_U4) {  // nibble rows: copy packed, unpack to uint8 on the device
      xt = GNB_X_U8;
      dld = ld8;
      const int64_t pb = ld8 / 2, sb = ldx / 2, wb = (n_features + 1) / 2;
      const uint8_t* src = static_cast<const uint8_t*>(xv) + r0 * sb;
      if (sb == pb)
        GNB_CUDA(cudaMemcpyAsync(c->x4[lane].p, src, size_t(n) * pb, cudaMemcpyHostToDevice, s),
                 "H2D");
      else
        GNB_CUDA(cudaMemcpy2DAsync(c->x4[lane].p, pb, src, sb, wb, n, cudaMemcpyHostToDevice, s),
                 "H2D 2D");
      GNB_CUDA(unpack_u4_launch(static_cast<const uint8_t*>(c->x4[lane].p), n, pb,
                                static_cast<uint8_t*>(dx), s),
               "unpack_u4");
    } else if (x_type != GNB_X_I32) {  // caller's narrow rows: copy as they are
      xt = x_type;
      const int eb = elem_bytes(xt);
      dld = xt == GNB_X_U8 ? ld8 : ld16;
      const uint8_t* src = static_cast<const uint8_t*>(xv) + r0 * ldx * eb;
      if (ldx == dld)
        GNB_CUDA(cudaMemcpyAsync(dx, src, size_t(n) * dld * eb, cudaMemcpyHostToDevice, s), "H2D");
      else
        GNB_CUDA(cudaMemcpy2DAsync(dx, dld * eb, src, ldx * eb, size_t(n_features) * eb, n,
                                   cudaMemcpyHostToDevice, s),
                 "H2D 2D");
    } else if (narrow_chunk_k(chunk)) {
      // this chunk was narrowed in the background (started while the previous
      // chunk was issued); start the next narrow chunk before issuing this one
      const auto tn = std::chrono::steady_clock::now();
      const int nt = jobs[pend_slot].finish(*c->pool);
      const auto tw = std::chrono::steady_clock::now();
      const int64_t nxt = next_narrow(chunk);
      if (nxt >= 0) {
        const int nl = static_cast<int>(nxt % kLanes);
        GNB_CUDA(cudaEventSynchronize(c->copied[nl]), "event sync");  // its staging is free
        pend_slot ^= 1;
        start_narrow(nxt, nl, pend_slot);
      }
      if (timing) {
        t_narrow += std::chrono::duration<double>(tw - tn).count();
        t_wait += std::chrono::duration<double>(std::chrono::steady_clock::now() - tw).count();
      }
      if (nt == GNB_X_U4) {  // nibbles over PCIe, unpacked to uint8 rows on the device
        GNB_CUDA(cudaMemcpyAsync(c->x4[lane].p, c->stage[lane].p, size_t(n) * (ld8 / 2),
                                 cudaMemcpyHostToDevice, s),
                 "H2D");
        GNB_CUDA(unpack_u4_launch(static_cast<const uint8_t*>(c->x4[lane].p), n, ld8 / 2,
                                  static_cast<uint8_t*>(dx), s),
                 "unpack_u4");
        xt = GNB_X_U8;
        dld = ld8;
      } else if (nt != GNB_X_I32) {
        xt = nt;
        dld = nt == GNB_X_U8 ? ld8 : ld16;
        GNB_CUDA(cudaMemcpyAsync(dx, c->stage[lane].p, size_t(n) * dld * elem_bytes(xt),
                                 cudaMemcpyHostToDevice, s),
                 "H2D");
      }
      GNB_CUDA(cudaEventRecord(c->copied[lane], s), "event");
    }
    if (xt == GNB_X_I32) {
      if (ldx == ld) {
        GNB_CUDA(cudaMemcpyAsync(dx, x + r0 * ldx, size_t(n) * ld * 4, cudaMemcpyHostToDevice, s), "H2D");
      } else {
        GNB_CUDA(cudaMemcpy2DAsync(dx, ld * 4, x + r0 * ldx, ldx * 4, size_t(n_features) * 4, n,
                                   cudaMemcpyHostToDevice, s),
                 "H2D 2D");
      }
    }
    GNB_CUDA(cudaMemcpyAsync(c->size[lane].p, size_bytes + r0, size_t(n) * 4,
                             cudaMemcpyHostToDevice, s),
             "H2D");
    // Ragged batch: the host sees the sizes, so it picks the kernel itself.
    // Rows grouped by size group -> 6-CTA kernel (GNB_ORDER_GROUPED); more than
    // 1 in 16 tiles mixing models -> the mixed-slot kernel (GNB_ORDER_MIXED),
    // or, where its tables do not fit in smem, a device slot sort + gather4.
    const int32_t* perm = nullptr;
    int order = GNB_ORDER_GROUPED;
    if (n_slots > 1) {
      int64_t mixed = 0, tiles = 0;
      for (int64_t t0 = 0; t0 < n; t0 += kMixTileRows, ++tiles) {
        int first = -2;
        for (int64_t r = t0; r < std::min<int64_t>(t0 + kMixTileRows, n); ++r) {
          const int32_t sz = size_bytes[r0 + r];
          if (sz < 0 || sz >= max_size_bytes) continue;
          const int sl = route[sz / group_size_bytes];
          if (first == -2) first = sl;
          else if (sl != first) {
            ++mixed;
            break;
          }
        }
      }
      if (mixed * 16 > tiles) {
        if (mixed_kernel(n_features, xt, n_classes, n_slots)) {
          order = GNB_ORDER_MIXED;
        } else {
          GNB_CUDA(c->perm[lane].ensure(size_t(n) * 4), "malloc");
          GNB_CUDA(c->sortws[lane].ensure(slot_sort_workspace(n, n_slots)), "malloc");
          GNB_CUDA(slot_sort(static_cast<int32_t*>(c->size[lane].p), n, group_size_bytes,
                             max_size_bytes, static_cast<int32_t*>(c->route.p), n_slots,
                             static_cast<int32_t*>(c->perm[lane].p), c->sortws[lane].p, s),
                   "slot_sort");
          perm = static_cast<int32_t*>(c->perm[lane].p);
        }
      }
    }
    rc = predict_device(dx, xt, n, n_features, dld, static_cast<int32_t*>(c->size[lane].p),
                        group_size_bytes, max_size_bytes, static_cast<int32_t*>(c->route.p),
                        n_slots, n_classes, c->packed.p, static_cast<int32_t*>(c->label[lane].p),
                        logpost_out ? static_cast<double*>(c->logpost[lane].p) : nullptr, s, 0,
                        perm, GNB_MODE_EXACT | order);
    if (rc) return rc;
    GNB_CUDA(cudaMemcpyAsync(label_out + r0, c->label[lane].p, size_t(n) * 4,
                             cudaMemcpyDeviceToHost, s),
             "D2H");
    if (logpost_out)
      GNB_CUDA(cudaMemcpyAsync(logpost_out + r0 * n_classes, c->logpost[lane].p,
                               size_t(n) * n_classes * 8, cudaMemcpyDeviceToHost, s),
               "D2H");
  }
  const auto t_issue = std::chrono::steady_clock::now();
  for (int i = 0; i < kLanes; ++i) GNB_CUDA(cudaStreamSynchronize(c->s[i]), "sync");
  if (timing)
    fprintf(stderr, "[gnb host] rows %lld chunks %lld: narrow wait %.3f ms, next-start %.3f ms, "
            "loop %.3f ms, drain %.3f ms\n", (long long)n_rows, (long long)chunk,
            t_narrow * 1e3, t_wait * 1e3,
            std::chrono::duration<double>(t_issue - t0).count() * 1e3,
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t_issue).count() * 1e3);
  if (elapsed_ns)
    *elapsed_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                      std::chrono::steady_clock::now() - t0)
                      .count();
  return GNB_OK;
}

extern "C" {

int gnb_predict_host(const int32_t* x, int64_t n_rows, int32_t n_features, int64_t ldx,
                     const int32_t* size_bytes, int32_t group_size_bytes,
                     int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                     int32_t n_classes, const double* log_prior, const double* log_lik,
                     int32_t* label_out, double* logpost_out, int32_t device,
                     int64_t* elapsed_ns) {
  return predict_host_impl(x, GNB_X_I32, n_rows, n_features, ldx, size_bytes, group_size_bytes,
                           max_size_bytes, route, n_slots, n_classes, log_prior, log_lik,
                           label_out, logpost_out, device, elapsed_ns);
}

int gnb_predict_host_typed(const void* x, int32_t x_type, int64_t n_rows, int32_t n_features,
                           int64_t ldx, const int32_t* size_bytes, int32_t group_size_bytes,
                           int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                           int32_t n_classes, const double* log_prior, const double* log_lik,
                           int32_t* label_out, double* logpost_out, int32_t device,
                           int64_t* elapsed_ns) {
  if (x_type != GNB_X_I32 && x_type != GNB_X_U16 && x_type != GNB_X_U8 && x_type != GNB_X_U4)
    return fail(GNB_EINVAL, "predict_host: unknown x_type %d", x_type);
  if (x_type == GNB_X_U4 && (ldx & 1))
    return fail(GNB_EINVAL, "predict_host: GNB_X_U4 rows need an even ldx (features)");
  return predict_host_impl(x, x_type, n_rows, n_features, ldx, size_bytes, group_size_bytes,
                           max_size_bytes, route, n_slots, n_classes, log_prior, log_lik,
                           label_out, logpost_out, device, elapsed_ns);
}

int gnb_fit_stats_host(const int32_t* x, int64_t n_rows, int32_t n_cols, int64_t ldx,
                       const int32_t* size_bytes, const int32_t* labels,
                       int32_t group_size_bytes, int32_t max_size_bytes, int32_t n_classes,
                       double* sums, double* sumsq, double* counts,
                       unsigned long long* status, int32_t device) {
  if (n_rows < 0 || n_cols < 1 || ldx < n_cols)
    return fail(GNB_EINVAL, "fit_stats_host: need n_rows>=0, n_cols>=1, ldx>=n_cols");
  if (group_size_bytes <= 0 || max_size_bytes <= 0 || max_size_bytes % group_size_bytes)
    return fail(GNB_EINVAL, "fit_stats_host: need 0 < group_size_bytes dividing max_size_bytes");
  if (n_classes < 2 || n_classes > GNB_MAX_CLASSES)
    return fail(GNB_EINVAL, "fit_stats_host: n_classes must be in [2, %d]", GNB_MAX_CLASSES);
  if (!sums || !counts) return fail(GNB_EINVAL, "fit_stats_host: null output");
  GNB_CUDA(cudaSetDevice(device), "cudaSetDevice");
  HostCtx* c = nullptr;
  int rc = get_ctx(device, &c);
  if (rc) return rc;
  const int64_t keys = int64_t(max_size_bytes / group_size_bytes) * n_classes;
  const size_t stat_b = size_t(keys) * n_cols * 8;
  GNB_CUDA(c->sums.ensure(stat_b), "malloc");
  if (sumsq) GNB_CUDA(c->sumsq.ensure(stat_b), "malloc");
  GNB_CUDA(c->counts.ensure(size_t(keys) * 8), "malloc");
  GNB_CUDA(c->status.ensure(16), "malloc");
  cudaStream_t s0 = c->s[0];
  double* dS = static_cast<double*>(c->sums.p);
  double* dQ = sumsq ? static_cast<double*>(c->sumsq.p) : nullptr;
  double* dN = static_cast<double*>(c->counts.p);
  auto* dst = static_cast<unsigned long long*>(c->status.p);
  GNB_CUDA(cudaMemsetAsync(dS, 0, stat_b, s0), "memset");
  if (dQ) GNB_CUDA(cudaMemsetAsync(dQ, 0, stat_b, s0), "memset");
  GNB_CUDA(cudaMemsetAsync(dN, 0, size_t(keys) * 8, s0), "memset");
  GNB_CUDA(cudaMemsetAsync(dst, 0, 16, s0), "memset");
  GNB_CUDA(cudaEventRecord(c->ev[0], s0), "event");
  for (int i = 1; i < kLanes; ++i) GNB_CUDA(cudaStreamWaitEvent(c->s[i], c->ev[0], 0), "wait");
  const int64_t ld = (n_cols + 3) / 4 * 4;
  const int64_t rows = std::min<int64_t>(chunk_rows_for(ld * 4), std::max<int64_t>(n_rows, 1));
  for (int i = 0; i < kLanes; ++i) {
    GNB_CUDA(c->x[i].ensure(size_t(rows) * ld * 4), "malloc");
    GNB_CUDA(c->size[i].ensure(size_t(rows) * 4), "malloc");
    GNB_CUDA(c->aux[i].ensure(size_t(rows) * 4), "malloc");
  }
  // chunks on different streams may run concurrently: every chunk adds exact
  // integer-valued partials with RED.ADD.F64, so the order does not matter.
  int64_t chunk = 0;
  for (int64_t r0 = 0; r0 < n_rows; r0 += rows, ++chunk) {
    const int lane = static_cast<int>(chunk % kLanes);
    cudaStream_t s = c->s[lane];
    const int64_t n = std::min(rows, n_rows - r0);
    int32_t* dx = static_cast<int32_t*>(c->x[lane].p);
    if (ldx == ld)
      GNB_CUDA(cudaMemcpyAsync(dx, x + r0 * ldx, size_t(n) * ld * 4, cudaMemcpyHostToDevice, s), "H2D");
    else
      GNB_CUDA(cudaMemcpy2DAsync(dx, ld * 4, x + r0 * ldx, ldx * 4, size_t(n_cols) * 4, n,
                                 cudaMemcpyHostToDevice, s),
               "H2D 2D");
    GNB_CUDA(cudaMemcpyAsync(c->size[lane].p, size_bytes + r0, size_t(n) * 4, cudaMemcpyHostToDevice, s), "H2D");
    GNB_CUDA(cudaMemcpyAsync(c->aux[lane].p, labels + r0, size_t(n) * 4, cudaMemcpyHostToDevice, s), "H2D");
    rc = gnb_fit_stats(dx, n, n_cols, ld, static_cast<int32_t*>(c->size[lane].p),
                       static_cast<int32_t*>(c->aux[lane].p), group_size_bytes, max_size_bytes,
                       n_classes, dS, dQ, dN, dst, 1, reinterpret_cast<uintptr_t>(s));
    if (rc) return rc;
  }
  for (int i = 0; i < kLanes; ++i) GNB_CUDA(cudaStreamSynchronize(c->s[i]), "sync");
  GNB_CUDA(cudaMemcpy(sums, dS, stat_b, cudaMemcpyDeviceToHost), "D2H");
  if (sumsq) GNB_CUDA(cudaMemcpy(sumsq, dQ, stat_b, cudaMemcpyDeviceToHost), "D2H");
  GNB_CUDA(cudaMemcpy(counts, dN, size_t(keys) * 8, cudaMemcpyDeviceToHost), "D2H");
  if (status) GNB_CUDA(cudaMemcpy(status, dst, 16, cudaMemcpyDeviceToHost), "D2H");
  return GNB_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ several GPUs, one call
// The reference's classify_parallel cuts the batch into ceil(N / lanes)
// contiguous chunks, one per worker (engine.py:264-268); here one host thread
// per device runs the single-device pipeline above on its contiguous shard.
// Predict has no exchange (rows are independent, the tables are replicated);
// the fit's one exchange is the sum of the integer-valued statistics, exact in
// any order (here on the host, since the host API returns host arrays).
namespace {

struct ShardErr {
  int rc = GNB_OK;
  char msg[512] = "";
};

int64_t shard_lo(int64_t n, int D, int d) {
  const int64_t chunk = n ? (n + D - 1) / D : 0;
  return std::min<int64_t>(chunk * d, n);
}

int join_shards(std::vector<std::thread>& th, std::vector<ShardErr>& err) {
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e.rc) return fail(e.rc, "%s", e.msg);
  return GNB_OK;
}

int check_devices(int32_t n_devices, const int32_t* devices) {
  if (n_devices < 1 || n_devices > 64 || !devices)
    return fail(GNB_EINVAL, "sharded: need 1..64 devices");
  int count = 0;
  GNB_CUDA(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
  for (int d = 0; d < n_devices; ++d)
    if (devices[d] < 0 || devices[d] >= count)
      return fail(GNB_EINVAL, "sharded: device %d not present (%d visible)", devices[d], count);
  return GNB_OK;
}

}  // namespace

extern "C" {

int gnb_predict_host_sharded(const void* x, int32_t x_type, int64_t n_rows, int32_t n_features,
                             int64_t ldx, const int32_t* size_bytes, int32_t group_size_bytes,
                             int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                             int32_t n_classes, const double* log_prior, const double* log_lik,
                             int32_t* label_out, double* logpost_out, int32_t n_devices,
                             const int32_t* devices, int64_t* elapsed_ns) {
  int rc = check_devices(n_devices, devices);
  if (rc) return rc;
  if (x_type != GNB_X_I32 && x_type != GNB_X_U16 && x_type != GNB_X_U8 && x_type != GNB_X_U4)
    return fail(GNB_EINVAL, "predict_host_sharded: unknown x_type %d", x_type);
  if (x_type == GNB_X_U4 && (ldx & 1))
    return fail(GNB_EINVAL, "predict_host_sharded: GNB_X_U4 rows need an even ldx (features)");
  // bytes per row of the caller's storage (U4: two features per byte)
  const int64_t row_b = x_type == GNB_X_U4 ? ldx / 2 : ldx * elem_bytes(x_type);
  std::vector<ShardErr> err(static_cast<size_t>(n_devices));
  std::vector<int64_t> ns(size_t(n_devices), 0);
  std::vector<std::thread> th;
  for (int d = 0; d < n_devices; ++d) {
    const int64_t lo = shard_lo(n_rows, n_devices, d), hi = shard_lo(n_rows, n_devices, d + 1);
    th.emplace_back([=, &err, &ns] {
      if (hi <= lo) return;
      const uint8_t* xb = static_cast<const uint8_t*>(x) + lo * row_b;
      const int r = predict_host_impl(xb, x_type, hi - lo, n_features, ldx, size_bytes + lo,
                                      group_size_bytes, max_size_bytes, route, n_slots, n_classes,
                                      log_prior, log_lik, label_out + lo,
                                      logpost_out ? logpost_out + lo * n_classes : nullptr,
                                      devices[d], &ns[size_t(d)]);
      if (r) {
        err[size_t(d)].rc = r;
        snprintf(err[size_t(d)].msg, sizeof(err[size_t(d)].msg), "device %d: %s", devices[d],
                 gnb_last_error());
      }
    });
  }
  if ((rc = join_shards(th, err))) return rc;
  // the slowest device's pipeline time (each excludes its own buffer setup)
  if (elapsed_ns) *elapsed_ns = *std::max_element(ns.begin(), ns.end());
  return GNB_OK;
}

int gnb_fit_stats_host_sharded(const int32_t* x, int64_t n_rows, int32_t n_cols, int64_t ldx,
                               const int32_t* size_bytes, const int32_t* labels,
                               int32_t group_size_bytes, int32_t max_size_bytes,
                               int32_t n_classes, double* sums, double* sumsq, double* counts,
                               unsigned long long* status, int32_t n_devices,
                               const int32_t* devices) {
  int rc = check_devices(n_devices, devices);
  if (rc) return rc;
  if (n_rows < 0 || n_cols < 1 || ldx < n_cols)
    return fail(GNB_EINVAL, "fit_stats_host_sharded: need n_rows>=0, n_cols>=1, ldx>=n_cols");
  if (group_size_bytes <= 0 || max_size_bytes <= 0 || max_size_bytes % group_size_bytes)
    return fail(GNB_EINVAL,
                "fit_stats_host_sharded: need 0 < group_size_bytes dividing max_size_bytes");
  if (!sums || !counts) return fail(GNB_EINVAL, "fit_stats_host_sharded: null output");
  const int64_t keys = int64_t(max_size_bytes / group_size_bytes) * n_classes;
  const size_t stat = size_t(keys) * n_cols;
  std::vector<std::vector<double>> S(static_cast<size_t>(n_devices)), Q(static_cast<size_t>(n_devices)),
      N(static_cast<size_t>(n_devices));
  std::vector<std::array<unsigned long long, 2>> st(static_cast<size_t>(n_devices));
  std::vector<ShardErr> err(static_cast<size_t>(n_devices));
  std::vector<std::thread> th;
  for (int d = 0; d < n_devices; ++d) {
    const int64_t lo = shard_lo(n_rows, n_devices, d), hi = shard_lo(n_rows, n_devices, d + 1);
    S[size_t(d)].assign(stat, 0.0);
    if (sumsq) Q[size_t(d)].assign(stat, 0.0);
    N[size_t(d)].assign(size_t(keys), 0.0);
    st[size_t(d)] = {0ull, 0ull};
    th.emplace_back([=, &S, &Q, &N, &st, &err] {
      const int r = gnb_fit_stats_host(x + lo * ldx, hi - lo, n_cols, ldx, size_bytes + lo,
                                       labels + lo, group_size_bytes, max_size_bytes, n_classes,
                                       S[size_t(d)].data(), sumsq ? Q[size_t(d)].data() : nullptr,
                                       N[size_t(d)].data(), st[size_t(d)].data(), devices[d]);
      if (r) {
        err[size_t(d)].rc = r;
        snprintf(err[size_t(d)].msg, sizeof(err[size_t(d)].msg), "device %d: %s", devices[d],
                 gnb_last_error());
      }
    });
  }
  if ((rc = join_shards(th, err))) return rc;
  // the exchange: integer-valued doubles < 2^53 add exactly in any order
  for (size_t i = 0; i < stat; ++i) {
    double a = 0.0, q = 0.0;
    for (int d = 0; d < n_devices; ++d) {
      a += S[size_t(d)][i];
      if (sumsq) q += Q[size_t(d)][i];
    }
    sums[i] = a;
    if (sumsq) sumsq[i] = q;
  }
  for (size_t i = 0; i < size_t(keys); ++i) {
    double a = 0.0;
    for (int d = 0; d < n_devices; ++d) a += N[size_t(d)][i];
    counts[i] = a;
  }
  if (status) {
    status[0] = status[1] = 0;
    for (int d = 0; d < n_devices; ++d) {
      status[0] += st[size_t(d)][0];
      status[1] += st[size_t(d)][1];
    }
  }
  return GNB_OK;
}

}  // extern "C"
