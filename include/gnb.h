/*
 * gnb.h -- C ABI of libgnb.so, the sm_100a group-wise Naive Bayes hot path.
 *
 * The reference (arxiv 1905.13746, /root/reference/pkg/src/groupnb) is pure
 * Python; its hot loops are the per-sample scoring loop and the per-group
 * training count loops.  Every entry point below replaces one of them and is
 * what a ctypes binding inside the reference would call (INTEGRATION.md shows
 * that binding).  Plain pointers and sizes only; no torch types.
 *
 * Dense conventions
 *   - class index 0 = benign, 1 = malware (2.. = extra malware families);
 *     argmax ties resolve to the LOWEST index, which is the reference's
 *     "malware iff strictly higher" (classifier.py:154-157).
 *   - X is int32, row-major, row stride `ldx` elements (ldx >= n_cols); counts
 *     must be >= 0 (OpcodeHistogram invariant, corpus.py:48-49).
 *   - size_bytes -> group = size / group_size_bytes on [0, max_size_bytes)
 *     (corpus.py:222-232); route[group] -> model slot (engine.py:56-59, 87-91).
 *   - predict rows hold the counts of the routed model's features in
 *     FeatureSet order (classifier.py:143 `_packed` order), zero padded.
 *
 * Device entry points (`gnb_predict`, `gnb_fit_stats`, `gnb_pack_tables`,
 * `gnb_generate`) take caller-owned DEVICE pointers and enqueue on the
 * caller's stream (`stream` = cudaStream_t cast to uintptr_t, 0 = legacy
 * default); they never synchronise and never allocate.  `*_host` entry points
 * take HOST pointers and run synchronously on `device` (they stage through
 * internal device buffers and pinned memory).  All functions are reentrant;
 * errors return a nonzero code and leave a message in gnb_last_error()
 * (thread-local).
 */
#ifndef GNB_H_
#define GNB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GNB_OK = 0,
  GNB_EINVAL = 1,       /* invalid argument            -> InvalidConfigError / ValueError */
  GNB_ECUDA = 2,        /* CUDA runtime/driver failure -> RuntimeError                   */
  GNB_EUNSUPPORTED = 3, /* shape this build does not handle                               */
  GNB_ENOMEM = 4
};

/* per-row status written into label_out instead of a class index */
#define GNB_ROW_OUT_OF_RANGE (-1)   /* size outside [0, max): engine.py:201-205 */
#define GNB_ROW_NEGATIVE_COUNT (-2) /* a count < 0 in the row (invalid input)   */

#define GNB_MAX_CLASSES 16

/* element type of X for the typed entry points: the same non-negative
 * integer counts, stored in fewer bytes when they fit */
enum { GNB_X_I32 = 0, GNB_X_U16 = 1, GNB_X_U8 = 2 };
/* host-side storage for gnb_predict_host_typed only: counts < 16 packed two per
 * byte, feature 2j in the low nibble of byte j, 2j+1 in the high nibble; ldx
 * in features (even).  Unpacked to uint8 rows on the device. */
enum { GNB_X_U4 = 3 };

/* predict arithmetic (gnb_predict_mode) */
enum { GNB_MODE_EXACT = 0, GNB_MODE_FMA = 1 };
/* row-order hint, OR-ed into gnb_predict_mode's `mode` (ragged batches of >= 2
 * slots whose tables fit in shared memory, gnb_predict_mixed_rows() > 0):
 *   GNB_ORDER_AUTO     (0, every other entry point) a device pass over the sizes
 *                      counts the 128-row tiles that mix models and gates the
 *                      kernel on the device, no host sync: grouped batches
 *                      take the 6-CTA kernel, interleaved ones the mixed-slot
 *                      kernel;
 *   GNB_ORDER_GROUPED  rows grouped by size group (GroupedCorpus order): no check;
 *   GNB_ORDER_MIXED    rows in any order: mixed-slot kernel, no check (where
 *                      gnb_predict_mixed_rows() is 0 this is the 6-CTA kernel
 *                      reading tables through L1 -- pass a gnb_slot_sort perm
 *                      instead).
 * Results are identical for every hint. */
enum { GNB_ORDER_AUTO = 0, GNB_ORDER_GROUPED = 0x10, GNB_ORDER_MIXED = 0x20 };

/* 3: row-order hints (GNB_ORDER_*) in gnb_predict_mode's mode, and
 * gnb_predict_mixed_rows; every version-2 entry point is unchanged. */
int gnb_abi_version(void);
const char* gnb_strerror(int code);
const char* gnb_last_error(void);

/* Streams: the device entry points are stream-ordered.  K-PRED keeps a small
 * per-(device, stream) scratch (the GNB_ORDER_AUTO gate and the dynamic tile
 * counter), allocated on first use and reset by the kernels themselves; work
 * issued on one stream handle must therefore run in that stream's order -- do
 * not replay a captured CUDA graph on another stream concurrently with K-PRED
 * work issued on (or captured from) the same stream handle. */

/* ------------------------------------------------------------------ predict
 * Replaces: classifier.log_posterior + classifier.predict
 *           (pkg/src/groupnb/classifier.py:132-158) inside
 *           engine._classify_slice (pkg/src/groupnb/engine.py:187-206), i.e.
 *           the body of classify_sequential / classify_parallel
 *           (engine.py:209-296).
 *
 * Packed tables: gnb_pack_tables turns log_prior[S][C] and log_lik[S][C][F]
 * (device, fp64) into the kernel layout in `packed`
 * (gnb_packed_table_bytes(S, C, F) bytes, 16-B aligned, caller-owned).
 * Scores are bit-identical to the reference: per class
 * acc = prior; acc = acc + x*ll (mul, then add) for every feature in order.
 * label_out[n] = argmax class, or GNB_ROW_*; logpost_out (nullable) [n][C].
 */
size_t gnb_packed_table_bytes(int32_t n_slots, int32_t n_classes, int32_t n_features);

int gnb_pack_tables(const double* log_prior, const double* log_lik, int32_t n_slots,
                    int32_t n_classes, int32_t n_features, void* packed, uintptr_t stream);

int gnb_predict(const int32_t* x, int64_t n_rows, int32_t n_features, int64_t ldx,
                const int32_t* size_bytes, int32_t group_size_bytes, int32_t max_size_bytes,
                const int32_t* route, int32_t n_slots, int32_t n_classes, const void* packed,
                int32_t* label_out, double* logpost_out, uintptr_t stream);

/* gnb_predict for X stored as x_type (GNB_X_I32 / GNB_X_U16 / GNB_X_U8); ldx
 * in elements.  uint8/uint16 rows move 4x/2x fewer bytes; results are
 * identical for the same counts. */
int gnb_predict_typed(const void* x, int32_t x_type, int64_t n_rows, int32_t n_features,
                      int64_t ldx, const int32_t* size_bytes, int32_t group_size_bytes,
                      int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                      int32_t n_classes, const void* packed, int32_t* label_out,
                      double* logpost_out, uintptr_t stream);

/* Ragged batches in arbitrary row order (engine.py:198-202 routes every file
 * by its own size).  When this returns > 0 for a batch's shape, gnb_predict /
 * gnb_predict_typed / gnb_predict_mode already score rows of any slot order at
 * streaming speed (mixed-slot kernel: every slot's table resident in shared
 * memory, each tile's rows sorted by slot inside the CTA; the value is the tile
 * height) and no slot sort is needed; 0 = the sort + permuted path below pays
 * for shuffled batches (C > 2, or tables too large for shared memory). */
int32_t gnb_predict_mixed_rows(int32_t n_features, int32_t x_type, int32_t n_classes,
                               int32_t n_slots);

/* gnb_slot_sort writes perm[n] = row
 * indices grouped by routed model slot (device counting sort over the sizes;
 * rows with size out of range last), using `workspace`
 * (gnb_slot_sort_workspace_bytes).  gnb_predict_permuted then scores tiles of
 * perm order -- rows fetched with TMA tile::gather4, one model per tile, tables
 * in shared memory -- and writes every output at its ORIGINAL row index, so
 * results equal gnb_predict's exactly.  n_rows <= 2^30, n_slots < 4096. */
size_t gnb_slot_sort_workspace_bytes(int64_t n_rows, int32_t n_slots);
int gnb_slot_sort(const int32_t* size_bytes, int64_t n_rows, int32_t group_size_bytes,
                  int32_t max_size_bytes, const int32_t* route, int32_t n_slots, int32_t* perm,
                  void* workspace, size_t workspace_bytes, uintptr_t stream);
int gnb_predict_permuted(const void* x, int32_t x_type, int64_t n_rows, int32_t n_features,
                         int64_t ldx, const int32_t* size_bytes, int32_t group_size_bytes,
                         int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                         int32_t n_classes, const void* packed, const int32_t* perm,
                         int32_t* label_out, double* logpost_out, uintptr_t stream);

/* All options in one call: any storage, optional perm (NULL = rows in order,
 * else as gnb_predict_permuted), and the arithmetic mode:
 *   GNB_MODE_EXACT  acc = acc + x*ll with the reference's two roundings
 *                   (DMUL then DADD; bit-identical log-posteriors) -- default
 *                   of every other entry point;
 *   GNB_MODE_FMA    acc = fma(x, ll, acc), one rounding per term: log-posteriors
 *                   within ~1e-12 relative of the reference (north star asks
 *                   1e-5), labels identical except at top-two margins of that
 *                   size; halves the FP64 work of compute-bound narrow rows.
 * (SURVEY 8b `gnb_geom.mode`.) */
int gnb_predict_mode(const void* x, int32_t x_type, int64_t n_rows, int32_t n_features,
                     int64_t ldx, const int32_t* size_bytes, int32_t group_size_bytes,
                     int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                     int32_t n_classes, const void* packed, const int32_t* perm, int32_t mode,
                     int32_t* label_out, double* logpost_out, uintptr_t stream);

/* Same as gnb_predict but always uses the L1 (non-TMA) kernel; parity tests. */
int gnb_predict_generic(const int32_t* x, int64_t n_rows, int32_t n_features, int64_t ldx,
                        const int32_t* size_bytes, int32_t group_size_bytes,
                        int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                        int32_t n_classes, const void* packed, int32_t* label_out,
                        double* logpost_out, uintptr_t stream);

/* Host-buffer form of the above (the ctypes drop-in for _classify_slice):
 * x/size/route/log_prior/log_lik/label_out/logpost_out are HOST arrays
 * (pinned memory is used zero-copy-fast; pageable works).  Rows are streamed
 * through the device in chunks with copies overlapped with the kernel.
 * Synchronous.  elapsed_ns (nullable) receives the wall time of the call. */
int gnb_predict_host(const int32_t* x, int64_t n_rows, int32_t n_features, int64_t ldx,
                     const int32_t* size_bytes, int32_t group_size_bytes,
                     int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                     int32_t n_classes, const double* log_prior, const double* log_lik,
                     int32_t* label_out, double* logpost_out, int32_t device,
                     int64_t* elapsed_ns);

/* Route + FeatureSet gather (device): x_out[n][j] = x_vocab[n][features[s][j]]
 * for j < n_features[s], s = route[size/width]; 0 elsewhere and for rows with
 * size out of range.  Turns a full-vocabulary matrix into the gnb_predict
 * input layout.  Replaces the per-sample route + `histogram.get(op)` walk of
 * engine._classify_slice / classifier.log_posterior (engine.py:198-202,
 * classifier.py:142-147).  features: [n_slots][max_features] vocab columns. */
int gnb_gather_features(const int32_t* x_vocab, int64_t n_rows, int32_t n_vocab, int64_t ldx,
                        const int32_t* size_bytes, int32_t group_size_bytes,
                        int32_t max_size_bytes, const int32_t* route, const int32_t* features,
                        const int32_t* n_features, int32_t n_slots, int32_t max_features,
                        int32_t* x_out, int64_t ldo, uintptr_t stream);

/* gnb_gather_features for x_vocab stored as x_type (GNB_X_I32/U16/U8); x_out
 * has the same element type (narrow rows stay narrow for gnb_predict_typed). */
int gnb_gather_features_typed(const void* x_vocab, int32_t x_type, int64_t n_rows,
                              int32_t n_vocab, int64_t ldx, const int32_t* size_bytes,
                              int32_t group_size_bytes, int32_t max_size_bytes,
                              const int32_t* route, const int32_t* features,
                              const int32_t* n_features, int32_t n_slots, int32_t max_features,
                              void* x_out, int64_t ldo, uintptr_t stream);

/* gnb_predict_host for host rows stored as x_type (GNB_X_I32/U16/U8/U4), ldx
 * in elements (features): narrow storage moves 2x/4x/8x fewer bytes over PCIe. */
int gnb_predict_host_typed(const void* x, int32_t x_type, int64_t n_rows, int32_t n_features,
                           int64_t ldx, const int32_t* size_bytes, int32_t group_size_bytes,
                           int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                           int32_t n_classes, const double* log_prior, const double* log_lik,
                           int32_t* label_out, double* logpost_out, int32_t device,
                           int64_t* elapsed_ns);

/* Several GPUs in one call: rows cut into ceil(n / n_devices) contiguous
 * shards, one per device (the reference's lane chunking, engine.py:264-268),
 * each streamed through that device by its own host thread exactly as
 * gnb_predict_host_typed does; no exchange (tables replicated, rows
 * independent).  elapsed_ns = the slowest device's pipeline time. */
int gnb_predict_host_sharded(const void* x, int32_t x_type, int64_t n_rows, int32_t n_features,
                             int64_t ldx, const int32_t* size_bytes, int32_t group_size_bytes,
                             int32_t max_size_bytes, const int32_t* route, int32_t n_slots,
                             int32_t n_classes, const double* log_prior, const double* log_lik,
                             int32_t* label_out, double* logpost_out, int32_t n_devices,
                             const int32_t* devices, int64_t* elapsed_ns);

/* ------------------------------------------------------------------ fit
 * Replaces: the sample x histogram count loops of features.class_frequency
 *           (pkg/src/groupnb/features.py:48-53) and classifier.train_group
 *           (pkg/src/groupnb/classifier.py:94-101), and the class counts of
 *           corpus.trainable_groups (pkg/src/groupnb/corpus.py:302-305).
 *
 * Over the full vocabulary: sums[G][C][V] = sum x, sumsq[G][C][V] = sum x^2,
 * counts[G][C] = rows, with G = max_size_bytes / group_size_bytes.  Rows with
 * size outside [0, max) are skipped (partition_by_group, corpus.py:247-251)
 * and counted in status[1]; rows whose label is outside [0, C) are skipped
 * and counted in status[0] (train_group raises IntegrityError for them,
 * classifier.py:95-96).  All values are integers accumulated exactly; the
 * fp64 outputs are exact while every total is < 2^53, so results do not
 * depend on the launch geometry or on the number of GPUs the rows are
 * sharded over.  accumulate=0 zeroes sums/sumsq/counts/status first.
 * sumsq may be NULL. */
int gnb_fit_stats(const int32_t* x, int64_t n_rows, int32_t n_cols, int64_t ldx,
                  const int32_t* size_bytes, const int32_t* labels, int32_t group_size_bytes,
                  int32_t max_size_bytes, int32_t n_classes, double* sums, double* sumsq,
                  double* counts, unsigned long long* status, int32_t accumulate,
                  uintptr_t stream);

/* gnb_fit_stats for X stored as x_type (GNB_X_I32 / GNB_X_U16 / GNB_X_U8). */
int gnb_fit_stats_typed(const void* x, int32_t x_type, int64_t n_rows, int32_t n_cols,
                        int64_t ldx, const int32_t* size_bytes, const int32_t* labels,
                        int32_t group_size_bytes, int32_t max_size_bytes, int32_t n_classes,
                        double* sums, double* sumsq, double* counts, unsigned long long* status,
                        int32_t accumulate, uintptr_t stream);

int gnb_fit_stats_host(const int32_t* x, int64_t n_rows, int32_t n_cols, int64_t ldx,
                       const int32_t* size_bytes, const int32_t* labels,
                       int32_t group_size_bytes, int32_t max_size_bytes, int32_t n_classes,
                       double* sums, double* sumsq, double* counts,
                       unsigned long long* status, int32_t device);

/* gnb_fit_stats_host over several GPUs: contiguous row shards, K-FIT on each
 * device, then the one exchange -- the integer-valued statistics summed
 * (exact in any order, so identical to one device). */
int gnb_fit_stats_host_sharded(const int32_t* x, int64_t n_rows, int32_t n_cols, int64_t ldx,
                               const int32_t* size_bytes, const int32_t* labels,
                               int32_t group_size_bytes, int32_t max_size_bytes,
                               int32_t n_classes, double* sums, double* sumsq, double* counts,
                               unsigned long long* status, int32_t n_devices,
                               const int32_t* devices);

/* ------------------------------------------------------------------ finalize (host)
 * Replaces: features.score_opcodes + select_top_k (features.py:59-86) and the
 *           prior / log-likelihood step of classifier.train_group
 *           (classifier.py:103-120), per trainable group, as train_bundle
 *           does (engine.py:166-173).  Two classes (0 benign, 1 malware).
 * Inputs are the host copies of gnb_fit_stats' sums/counts.  Vocabulary
 * columns must be in mnemonic order (ties break by column index).
 * group_state[g]: 1 trained; 0 not trainable (< min_per_class of a class);
 *                 -1 no malware opcode occurrences; -2 no benign occurrences
 *                 (both InsufficientClassError in the reference).
 * n_features[g] <= k; features[g][k] column indices in FeatureSet order;
 * log_prior[g][2]; log_lik[g][2][k] (unused tail zero).  libm log. */
int gnb_fin_train(const double* sums, const double* counts, int32_t n_groups, int32_t n_cols,
                  int32_t k, double alpha, int32_t min_per_class, int32_t* group_state,
                  int32_t* n_features, int32_t* features, double* log_prior,
                  double* log_lik);

/* gnb_fin_train with the scoring + top-k on the DEVICE (one CTA per group,
 * shared-memory bitonic sort of (-score, column)); sums/counts are DEVICE
 * pointers (gnb_fit_stats outputs), results land in HOST arrays as for
 * gnb_fin_train and are identical to it (libm logs on the host).  Vocabularies
 * up to 16384 columns; synchronises `stream`. */
int gnb_fin_train_device(const double* sums, const double* counts, int32_t n_groups,
                         int32_t n_cols, int32_t k, double alpha, int32_t min_per_class,
                         int32_t* group_state, int32_t* n_features, int32_t* features,
                         double* log_prior, double* log_lik, uintptr_t stream);

/* train_group for ONE group with a given feature list and C classes
 * (classifier.py:103-120 with a class axis; C = 2 reproduces the reference):
 * sums_g[C][V], counts_g[C] -> log_prior[C], log_lik[C][F].  Host, libm log. */
int gnb_fin_tables(const double* sums_g, const double* counts_g, int32_t n_classes,
                   int32_t n_cols, const int32_t* features, int32_t n_features, double alpha,
                   double* log_prior, double* log_lik);

/* ------------------------------------------------------------------ ingestion (host)
 * Replaces: corpus.parse_corpus + OpcodeHistogram.from_counts
 *           (pkg/src/groupnb/corpus.py:133-189, :42-53) for the dense path:
 *           JSONL text -> sorted vocabulary + sparse rows, multithreaded;
 *           gnb_corpus_dense then writes any row range as a dense matrix
 *           (int32 / uint16 / uint8).  On error (GNB_EINVAL) the handle holds
 *           the reference's error kind (1 ParseError, 2 IntegrityError), line
 *           number and message; free it with gnb_corpus_free either way. */
typedef struct gnb_corpus gnb_corpus;
int gnb_corpus_parse(const char* text, size_t len, int32_t allow_unlabeled, int32_t threads,
                     gnb_corpus** out);
void gnb_corpus_free(gnb_corpus* c);
int64_t gnb_corpus_rows(const gnb_corpus* c);
int32_t gnb_corpus_vocab_size(const gnb_corpus* c);
const char* gnb_corpus_vocab(const gnb_corpus* c, int32_t k);
const char* gnb_corpus_id(const gnb_corpus* c, int64_t row);
int64_t gnb_corpus_max_count(const gnb_corpus* c);
int64_t gnb_corpus_nnz(const gnb_corpus* c);
int32_t gnb_corpus_error(const gnb_corpus* c, int64_t* line, const char** message);
int gnb_corpus_meta(const gnb_corpus* c, int64_t* size_out, int8_t* label_out);
int gnb_corpus_dense(const gnb_corpus* c, int32_t x_type, void* x, int64_t ldx, int64_t row0,
                     int64_t n, int32_t threads);

/* engine.write_predictions (pkg/src/groupnb/engine.py:466-481) for a parsed
 * corpus: byte-identical JSONL (17 significant digits).  label: 1 malware,
 * 0 benign, < 0 size error; logpost[n][2] = (benign, malware).  The text is
 * malloc'ed; release it with gnb_free_text. */
int gnb_corpus_write_predictions(const gnb_corpus* c, const int8_t* label, const double* logpost,
                                 const int32_t* effective_group, int64_t max_size_bytes,
                                 int32_t threads, char** out_text, size_t* out_len);
void gnb_free_text(char* p);

/* ------------------------------------------------------------------ synthetic data
 * Device generator following the reference's synthetic law
 * (pkg/src/groupnb/synth.py:64-116): per row a group (rows laid out group by
 * group, group g owning rows [group_row_end[g-1], group_row_end[g]) of the
 * GLOBAL index space), a class (row % C), a size uniform in the group's byte
 * range, T = 64 + size/64 draws, and per-column counts ~ Poisson(T * p_c[v])
 * with p_c from class_distributions (weight 1 on the class's block, 1-d
 * elsewhere).  Counter-based: row r's values depend only on (seed, r), so any
 * sharding of the global index space yields the same data. n_groups <= 128.
 * col_map (device, nullable, [n_cols]): output column j holds the counts of
 * vocabulary column col_map[j] of a vocab_cols-wide vocabulary -- the same
 * samples gathered into a model's FeatureSet order (predict layout). */
int gnb_generate(int32_t* x, int64_t n_rows, int32_t n_cols, int64_t ldx, int32_t* size_bytes,
                 int32_t* labels, int64_t row_offset, const int64_t* group_row_end,
                 int32_t n_groups, int32_t group_size_bytes, int32_t n_classes,
                 double divergence, uint64_t seed, const int32_t* col_map,
                 int32_t vocab_cols, uintptr_t stream);

/* ------------------------------------------------------------------ fit exchange (NCCL)
 * The sharded fit's only exchange step: each device's packed fp64
 * statistics buffer {sums | sumsq | counts} summed in place across devices
 * over NCCL (NVLink / NVSwitch).  The statistics are integer-valued, so the
 * bundle is bit-identical for any device count.  NCCL is loaded at run time
 * (dlopen "libnccl.so.2": the process's own copy, e.g. torch's, else the
 * system one); GNB_EUNSUPPORTED if it cannot be.
 *   one process, several GPUs: gnb_comms_init(&c, ndev, devs)   (ncclCommInitAll)
 *   one process per GPU:       rank 0 gnb_comms_unique_id(id), share the
 *                              GNB_COMMS_ID_BYTES, every rank
 *                              gnb_comms_init_rank(&c, nranks, rank, id, device)
 * gnb_fit_allreduce takes one buffer and one stream per local device of the
 * communicator (gnb_comms_size), stream-ordered, no synchronisation. */
#define GNB_COMMS_ID_BYTES 128
typedef struct gnb_comms gnb_comms;
int gnb_comms_unique_id(uint8_t* id);
int gnb_comms_init(gnb_comms** comms, int32_t ndev, const int32_t* devs);
int gnb_comms_init_rank(gnb_comms** comms, int32_t nranks, int32_t rank, const uint8_t* id,
                        int32_t device);
int32_t gnb_comms_size(const gnb_comms* comms);
void gnb_comms_destroy(gnb_comms* comms);
int gnb_fit_allreduce(gnb_comms* comms, double* const* packed_stats, int64_t elems,
                      const uintptr_t* streams);

#ifdef __cplusplus
}
#endif
#endif /* GNB_H_ */
