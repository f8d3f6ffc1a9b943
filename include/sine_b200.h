/*
 * sine_b200.h -- C ABI of the B200-native Sine stage-1 index and LCFU
 * eviction engine (libsine_b200.so).
 *
 * Plain pointers and sizes only; no torch / CUDA types in the signatures
 * (a stream is passed as `void*` = cudaStream_t).  Every call returns an
 * int status; on failure `sine_last_error()` (thread-local) describes it.
 *
 * Reference interfaces each entry point replaces (semcache = the reference
 * package at /root/reference/pkg/src/semcache):
 *
 *   sine_create / sine_destroy   ExactCosineIndex.__init__   index.py:54-62
 *   sine_insert[_device]         ExactCosineIndex.insert     index.py:71-78
 *                                (+ the SemanticElement columns LCFU reads,
 *                                 model.py:85-110, engine.py:330-334)
 *   sine_remove                  ExactCosineIndex.remove     index.py:80-92
 *   sine_size / sine_ids         __len__ / ids()             index.py:64-69
 *   sine_get_rows / sine_snapshot  snapshot_lines() rows     index.py:104-107
 *   sine_query[_device]          ExactCosineIndex.query      index.py:94-102
 *                                + _rank                     index.py:42-46
 *                                (batched: B independent queries)
 *   sine_update_meta             hit bookkeeping             engine.py:209-217
 *   sine_expired                 _purge_expired_locked       engine.py:362-367
 *   sine_select_victims          _victim_order_locked +      engine.py:369-383
 *                                the pop-until-fits loops    engine.py:321-327,
 *                                                            engine.py:353-359
 */
#ifndef SINE_B200_H
#define SINE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define SINE_OK          0
#define SINE_EINVAL      1  /* bad argument -> semcache ValidationError      */
#define SINE_ECUDA       2  /* CUDA runtime / kernel failure                 */
#define SINE_ENCCL       3  /* reserved (collectives live in the host layer) */
#define SINE_ENOMEM      4  /* device or pinned-host allocation failed       */
#define SINE_ENOTFOUND   5  /* unknown id       -> ValidationError           */
#define SINE_EDUP        6  /* duplicate id     -> ValidationError           */
#define SINE_ENORM       7  /* not L2-normalised / wrong dimension           */

/* ---- sine_create flags --------------------------------------------------- */
#define SINE_STORE_F32   0x1u  /* keep fp32 scan rows  (exact mode)          */
#define SINE_STORE_BF16  0x2u  /* keep bf16 scan rows  (fast mode)           */
#define SINE_STORE_META  0x4u  /* keep LCFU metadata columns (engine mode)   */
#define SINE_STORE_F64_HOST 0x8u /* fp64 master rows in pinned host memory mapped
                                    into the device address space instead of HBM:
                                    the re-rank reads only k' rows per query over
                                    the host link; frees 8 B/dim/row of HBM     */

/* ---- sine_query modes ------------------------------------------------------ */
#define SINE_SCAN_F32      0x0u  /* fp32 rows, fp32 accumulation             */
#define SINE_SCAN_BF16     0x1u  /* bf16 rows, fp32 accumulation             */
#define SINE_RERANK_F64    0x10u /* re-score final candidates in fp64        */
#define SINE_NO_NORM_CHECK 0x100u/* caller already validated (|norm-1|<=1e-6)*/
#define SINE_SCAN_CUDA_CORE 0x200u /* force the CUDA-core streaming scan      */
#define SINE_SCAN_UMMA_V1  0x400u /* force the query-streaming tcgen05 kernel */
#define SINE_SCAN_CLUSTER  0x1000u /* tcgen05: share row tiles across up to 8 CTAs
                                      (TMA multicast), one HBM pass per 8 query groups */
#define SINE_SCAN_PAIR     0x2000u /* tcgen05 cta_group::2: prefer the CTA-pair kernel */
#define SINE_SCAN_GEMM     0x4000u /* tcgen05 cta_group::2 tiled GEMM (256 rows x 256
                                      queries per pair tile, all query tiles of the batch
                                      in one launch); chosen automatically for large
                                      batches at high thresholds */
#define SINE_SCAN_NO_GEMM  0x8000u /* never use the tiled GEMM path                */
#define SINE_CERTIFY       0x800u /* sine_query_device: check the per-query exactness
                                     certificate and re-run failures on the fp32
                                     CUDA-core scan (synchronises the stream);
                                     sine_query always does this when re-ranking */

/* ---- eviction policies (CacheConfig.eviction_policy, model.py:15) -------- */
#define SINE_POLICY_LCFU 0
#define SINE_POLICY_LRU  1
#define SINE_POLICY_LFU  2

/* Per-element LCFU columns, structure-of-arrays, one entry per inserted id.
 * log_* are the natural logs the reference multiplies (engine.py:43-46),
 * evaluated on the HOST with libm so the device product is bit-exact:
 *   log_freq = log(frequency + 1)          log_cost = log(cost*1000.0 + 1)
 *   log_lat  = log(latency_ms + 1)         log_stat = log(staticity + 1)   */
typedef struct sine_meta_cols {
    const double  *log_freq, *log_cost, *log_lat, *log_stat;
    const int64_t *frequency, *size_tokens;
    const double  *created_at, *expiration_time, *last_access;
} sine_meta_cols_t;

typedef struct sine_index sine_index_t;

const char *sine_last_error(void);
int sine_version(void);
int sine_device_count(int *n);

int sine_create(int device, int64_t dim, uint32_t flags, int64_t reserve_rows,
                sine_index_t **out);
int sine_destroy(sine_index_t *h);
int sine_reserve(sine_index_t *h, int64_t rows);

/* rows: host float64 [n, dim] row-major.  meta may be NULL unless the
 * index was created with SINE_STORE_META. */
int sine_insert(sine_index_t *h, int64_t n, const int64_t *ids, const double *rows,
                const sine_meta_cols_t *meta, uint32_t flags);
/* Same, rows already in device memory (bulk load).  Waits for all prior
 * work on the device first, so rows written on any stream are complete. */
int sine_insert_device(sine_index_t *h, int64_t n, const int64_t *ids,
                       const double *rows_dev, const sine_meta_cols_t *meta,
                       uint32_t flags);
int sine_remove(sine_index_t *h, int64_t n, const int64_t *ids);

int sine_size(sine_index_t *h, int64_t *live, int64_t *slots);
/* Live ids in the reference's order (ExactCosineIndex._ids: insertion
 * order, the last id swapped into a removed id's place, index.py:71-92).
 * Writes min(*n, cap) ids; *n = the live count. */
int sine_ids(sine_index_t *h, int64_t *out, int64_t cap, int64_t *n);
int sine_get_rows(sine_index_t *h, int64_t n, const int64_t *ids, double *out);
/* Atomic snapshot (snapshot_lines, index.py:104-107): the ids in sine_ids
 * order and their fp64 rows [n][dim], under one hold of the handle lock.
 * *n = the live count; fails with SINE_EINVAL (buffers untouched) when
 * cap < *n. */
int sine_snapshot(sine_index_t *h, int64_t cap, int64_t *ids, double *rows, int64_t *n);

/* B queries, host float64 [B, dim].  Outputs (host): ids [B, k] (-1 padded),
 * sims [B, k], counts [B].  Each query's result equals
 * ExactCosineIndex.query(q, k, min_similarity) on the same snapshot. */
int sine_query(sine_index_t *h, int64_t B, const double *q, int k, double min_sim,
               uint32_t mode, int64_t *out_ids, double *out_sims, int32_t *out_counts);
/* Same, all buffers in device memory, enqueued on `stream` (NULL = the
 * handle's own stream).  Does not synchronise. */
int sine_query_device(sine_index_t *h, int64_t B, const double *q_dev, int k,
                      double min_sim, uint32_t mode, int64_t *ids_dev,
                      double *sims_dev, int32_t *counts_dev, void *stream);

/* sine_query_device that also writes the per-query exactness certificates
 * (B bytes, 1 = provably the exact answer) to cert_dev on the stream, so a
 * pipelined caller checks them later without a sync or an extra copy;
 * SINE_CERTIFY is ignored here (a 0 means: re-run that query, e.g. with
 * SINE_SCAN_CUDA_CORE). */
int sine_query_device_cert(sine_index_t *h, int64_t B, const double *q_dev, int k,
                           double min_sim, uint32_t mode, int64_t *ids_dev, double *sims_dev,
                           int32_t *counts_dev, uint8_t *cert_dev, void *stream);

/* Asynchronous sine_query: enqueue the batch (host buffers, which must stay
 * valid until the wait; pinned queries upload fastest) and return a ticket;
 * up to 16 batches in flight.  The device writes each ticket's results into
 * pinned, device-mapped staging owned by the handle; sine_query_wait blocks
 * until the batch is done, copies them into the output buffers and runs the
 * exactness certificate check. */
int sine_query_submit(sine_index_t *h, int64_t B, const double *q, int k, double min_sim,
                      uint32_t mode, int64_t *out_ids, double *out_sims,
                      int32_t *out_counts, int64_t *ticket);
int sine_query_wait(sine_index_t *h, int64_t ticket);

int sine_update_meta(sine_index_t *h, int64_t n, const int64_t *ids,
                     const double *log_freq, const int64_t *frequency,
                     const double *last_access);
/* Ids with expiration_time - now <= 0, ascending.  remove != 0 also
 * tombstones them. */
int sine_expired(sine_index_t *h, double now, int remove, int64_t *out,
                 int64_t cap, int64_t *n);
/* The shortest prefix of the (key, created_at, id)-ascending order whose
 * size_tokens sum reaches `excess`, in order.  Not removed. */
int sine_select_victims(sine_index_t *h, int policy, double now, int64_t excess,
                        int64_t *out, int64_t cap, int64_t *n);
/* sine_select_victims + tombstoning the victims in the same call (the
 * engine's pop loops at engine.py:321-327, :353-359, which remove what they
 * select). */
int sine_evict(sine_index_t *h, int policy, double now, int64_t excess,
               int64_t *out, int64_t cap, int64_t *n);
/* Test hook (not in the reference): the number of selection records one CTA
 * sorts in shared memory (2..6144, default 6144).  Lower values drive the
 * merge path for oversized buckets on small stores. */
int sine_set_select_cap(sine_index_t *h, int cap);

/* Introspection for benchmarks: the handle's stream, and the device time
 * (CUDA events on that stream) of the last query's scan and merge kernels
 * and the last victim selection. */
int sine_stream(sine_index_t *h, void **stream);
int sine_set_timing(sine_index_t *h, int on);
int sine_last_timing(sine_index_t *h, float *scan_ms, float *merge_ms, float *evict_ms);
int sine_kernel_launches(sine_index_t *h, int64_t *n);
/* Tiled-GEMM stage-1 launches (SINE_SCAN_GEMM) whose per-query candidate
 * buffers overflowed and were re-run on the list-keeping kernels.  Not in
 * the reference (diagnostic for the batched path, like sine_uncertified). */
int sine_gemm_overflows(sine_index_t *h, int64_t *n);
/* Single-process multi-GPU stage-1 (replaces one ExactCosineIndex with P
 * row shards for the reference's single-process engine, engine.py:103-109):
 * shards[p] lives on devices[p] (a device may repeat); each query runs on
 * every shard concurrently (one worker thread per shard, certified exact
 * top-k each), the [B][k] blocks are peer-copied to devices[0] and merged
 * by (similarity desc, id asc).  The group does not own the shards. */
typedef struct sine_group sine_group_t;
int sine_group_create(sine_index_t *const *shards, const int *devices, int n, int64_t dim,
                      sine_group_t **out);
int sine_group_destroy(sine_group_t *g);
int sine_group_query(sine_group_t *g, int64_t B, const double *q, int k, double min_sim,
                     uint32_t mode, int64_t *out_ids, double *out_sims, int32_t *out_counts);

/* Row-sharded stage-1 (one process per GPU): merge the P per-rank exact
 * top-k lists of B queries -- the all-gather output on the device, rank r's
 * [B][k] ids / sims at r * rank_stride elements (0 = B * k), id -1 =
 * padding -- into the global top-k by (similarity desc, id asc), the
 * order of index.py:45.  Device pointers, enqueued on `stream`.  Because
 * each rank's list is its shard's exact top-k, the result equals an
 * unsharded sine_query. */
int sine_merge_shards(int device, int P, int64_t B, int k, const int64_t *ids_dev,
                      const double *sims_dev, int64_t rank_stride, int64_t *out_ids,
                      double *out_sims, int32_t *out_counts, void *stream);
/* Batched HashedBagEmbedder (embedder.py:34-60): B queries already
 * tokenized on the host (embedder.tokenize, embedder.py:23-25) as UTF-8
 * bytes; token t is tok_bytes[tok_off[t] .. tok_off[t+1]), query b owns
 * tokens q_off[b] .. q_off[b+1]) (at least one -> else SINE_EINVAL, "cannot
 * embed text with no tokens").  Keyed BLAKE2b-64 of every token and the
 * bucket counts run on `device`; out_rows (host, [B][dim]) receives
 * counts / (sum(c*c) ** 0.5), bit-identical to the reference.
 * sine_blake2b64: blake2b(msg, key=key.to_bytes(8,'little'), digest_size=8)
 * as a little-endian integer (host; the same code the kernel runs). */
int sine_embed_hashed_bag(int device, uint64_t seed, int64_t dim, const uint8_t *tok_bytes,
                          int64_t nbytes, const int64_t *tok_off, int64_t ntok,
                          const int64_t *q_off, int64_t B, double *out_rows);
uint64_t sine_blake2b64(const uint8_t *msg, int64_t len, uint64_t key);
/* Float-hex text of row blocks, byte-identical to the reference's
 * snapshot / record writers (" ".join(float(c).hex() ...), index.py:343-346,
 * model.py:237) and read back bit-exactly like float.fromhex (index.py:370,
 * model.py:263).  Host-only, multi-threaded, no device needed.
 *   sine_hex_format: n lines "[<id> ]<hex> ... <hex>\n" (ids may be NULL);
 *     out must hold sine_hex_bound(n, d, ids != NULL) bytes; *len = bytes.
 *   sine_hex_parse: n such lines (ids NULL: no id field) -> ids, rows [n][d];
 *     a malformed line -> SINE_EINVAL naming it. */
int64_t sine_hex_bound(int64_t n, int64_t d, int with_ids);
int sine_hex_format(const int64_t *ids, const double *rows, int64_t n, int64_t d,
                    char *out, int64_t cap, int64_t *len);
int sine_hex_parse(const char *text, int64_t len, int64_t n, int64_t d, int64_t *ids,
                   double *rows);
/* Enqueue a device copy of the last query's per-query exactness
 * certificates (B bytes, 1 = exact) -- lets a pipelined caller check them
 * later instead of synchronising after every batch. */
int sine_copy_certificates(sine_index_t *h, int64_t B, void *dst_dev, void *stream);
/* Queries the last certified call had to re-run on the fp32 scan. */
int sine_uncertified(sine_index_t *h, int64_t *n);
/* Sum of device time (ms) and count of the launches of one kernel kind
 * (0 = stage-1 scan, 1 = merge/re-rank, 2 = tensor-core scan) recorded
 * while timing was on; reset != 0 clears the record. */
int sine_timing_totals(sine_index_t *h, int kind, double *total_ms, int64_t *launches, int reset);

int sine_host_alloc(size_t bytes, void **p);
int sine_host_free(void *p);

#ifdef __cplusplus
}
#endif
#endif /* SINE_B200_H */
