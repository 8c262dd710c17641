/*
 * laivg.h — C ABI of the B200-native lookahead IVF retrieval path
 * (paper_2502_20969_b200/liblaivg.so).
 *
 * The reference (`laiv`, /root/reference/proj/core) is a C++20 library; this
 * ABI is what its hot-path functions bind to when they are re-pointed at the
 * GPU (see INTEGRATION.md for the C++ shim a maintainer adds). Each entry point
 * cites the reference interface it replaces as file:line under
 * /root/reference/proj/core/.
 *
 * Conventions
 *  - Every function returns int status: LAIVG_OK (0) or a negative code whose
 *    class mirrors the reference exception type (std::invalid_argument,
 *    std::runtime_error, std::logic_error); laivg_last_error() gives the
 *    message (thread-local). Nothing throws across the ABI.
 *  - Plain pointers and sizes only. Host pointers unless a name says `dev`.
 *  - Store layout = the LAIX list-major order (ivf.cpp:373-388): vecs[N][D]
 *    f32, ids[N] u64, list_off[nc+1] u64; list c is rows
 *    [list_off[c], list_off[c+1]). cluster_bytes(c) = |c|*(4D+8) (ivf.cpp:23).
 *  - Scores follow vectorstore.cpp:93-115: per-candidate accumulation in
 *    fp64 rounded to fp32; L2 reports sqrt. Coarse ranking uses unrounded
 *    fp64 (squared L2). Total order: score by metric orientation, then
 *    ascending id (vectorstore.hpp:34-39).
 *  - Threading: a laivg_index is immutable and shareable by all contexts; a
 *    laivg_ctx (one GPU + its cluster cache) is driven by one host thread.
 *  - There is no CPU fallback for the device path: a missing/unusable GPU
 *    makes laivg_ctx_create fail with LAIVG_ECUDA.
 */
#ifndef LAIVG_H
#define LAIVG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status ------------------------------------------------------------ */
#define LAIVG_OK 0
#define LAIVG_EINVAL (-1)   /* std::invalid_argument */
#define LAIVG_ERUNTIME (-2) /* std::runtime_error   */
#define LAIVG_ELOGIC (-3)   /* std::logic_error     */
#define LAIVG_ECUDA (-4)    /* CUDA runtime failure (no reference analogue) */

#define LAIVG_METRIC_IP 0 /* vectorstore.hpp:18 Metric::InnerProduct */
#define LAIVG_METRIC_L2 1 /* vectorstore.hpp:18 Metric::L2           */

#define LAIVG_TAG_PREFETCHED 0 /* tiered.hpp:17 Residency::Prefetched */
#define LAIVG_TAG_CACHED 1     /* tiered.hpp:17 Residency::Cached     */

#define LAIVG_CHAN_SIMULATED 0 /* tiered.hpp:65 ChannelMode::SimulatedClock */
#define LAIVG_CHAN_MEASURED 1  /* tiered.hpp:65 ChannelMode::Measured       */
#define LAIVG_CHAN_DEVICE 2    /* new: async H2D on a copy stream, event-timed */

const char* laivg_last_error(void);
/* ABI version (major << 16 | minor). */
uint32_t laivg_version(void);

/* ---- pinned host memory -------------------------------------------------- */
/* Portable pinned allocation (cudaHostAllocPortable) so every device shares
 * one host datastore slab. */
int laivg_host_alloc(uint64_t bytes, void** out);
int laivg_host_free(void* p);
/* Pins an existing host range (cudaHostRegister, portable) so a datastore
 * mapped from shared memory can be shared by several processes/devices. */
int laivg_host_register(void* p, uint64_t bytes);
int laivg_host_unregister(void* p);
/* Number of kernels this library has launched (all contexts). */
uint64_t laivg_kernel_launches(void);

/* ---- index: IvfIndex + EmbeddingMatrix (ivf.hpp:26-50, vectorstore.hpp:50-83)
 * centroids[nc*d] are copied. With LAIVG_INDEX_BORROW the store arrays are
 * borrowed (caller keeps them alive and ideally allocated them with
 * laivg_host_alloc); otherwise they are copied into a library-owned pinned
 * slab. Validation mirrors the reference constructors: d > 0, finite
 * components (vectorstore.cpp:66-85) unless LAIVG_INDEX_TRUST is set,
 * monotone list_off. */
#define LAIVG_INDEX_BORROW 1u
#define LAIVG_INDEX_TRUST 2u
typedef struct laivg_index laivg_index;
int laivg_index_create(const float* centroids, uint32_t nc, uint32_t d,
                       int metric, const float* vecs, const uint64_t* ids,
                       const uint64_t* list_off, uint32_t flags,
                       laivg_index** out);
void laivg_index_destroy(laivg_index* ix);
/* ivf.hpp:98 load_index: reads a LAIX file (ivf.cpp:394-458) straight into
 * the list-major store (list rows/ids land where the devices copy them from,
 * read by `threads` threads, 0 = all cores) and pins it in place. Errors as
 * the reference: LAIVG_ERUNTIME for IO/format/truncation, LAIVG_EINVAL for a
 * non-finite component or a repeated id -- the first in file order, with the
 * reference's message. */
int laivg_index_load(const char* path, uint32_t threads, laivg_index** out);
/* ivf.hpp:96 save_index: writes the LAIX bytes save_index writes for the
 * same index (ivf.cpp:351-392). */
int laivg_index_save(const laivg_index* ix, const char* path, uint32_t threads);
/* Read-only views of the store (any out pointer may be NULL): vecs[N][d],
 * ids[N], list_off[nc+1], centroids[nc][d]; valid until destroy. */
int laivg_index_store(const laivg_index* ix, const float** vecs, const uint64_t** ids,
                      const uint64_t** list_off, const float** centroids);
uint32_t laivg_index_num_clusters(const laivg_index* ix);
uint32_t laivg_index_dim(const laivg_index* ix);
int laivg_index_metric(const laivg_index* ix);
uint64_t laivg_index_total_vectors(const laivg_index* ix);
/* |list c| (ivf.hpp:38 IvfIndex::list(c).size()) */
uint64_t laivg_index_list_len(const laivg_index* ix, uint32_t c);
/* ivf.hpp:40 IvfIndex::cluster_bytes */
uint64_t laivg_index_cluster_bytes(const laivg_index* ix, uint32_t c);
/* ivf.hpp:41 IvfIndex::total_payload_bytes */
uint64_t laivg_index_total_payload_bytes(const laivg_index* ix);

/* ---- device context: one GPU, its cluster cache (TieredStore), streams --- */
typedef struct {
  int device;              /* CUDA ordinal */
  uint64_t capacity_bytes; /* TieredStore capacity (tiered.hpp:24), reference
                              byte accounting n*(4D+8) */
  uint32_t miss_threads;   /* host threads scanning cache misses; 0 = all cores */
  uint32_t max_batch;      /* max queries per batched call; 0 = 256 */
  uint32_t max_probe;      /* max L per call; 0 = nc */
  uint32_t acc_fp64;       /* 0 (default): fp32 FMA accumulation, survivors
                              re-scored with the reference's fp64 arithmetic;
                              1: every candidate accumulated in fp64 */
  uint32_t scan_impl;      /* 0 (default): TMA bulk-copy staged scan;
                              1: direct 128-bit register loads */
  uint32_t tma_tile;       /* vectors per TMA stage; 0 = auto (~48 KB) */
  uint32_t tma_stages;     /* TMA ring depth; 0 = auto (~192 KB ring) */
  uint32_t ctas_per_sm;    /* scan CTAs per SM; 0 = auto */
  uint32_t coarse_impl;    /* 0 (default): tensor cores (tcgen05 tf32 GEMM +
                              exact fp64 re-score of boundary candidates) for
                              batches >= 16 queries, fp64 SIMT otherwise;
                              1: always fp64 SIMT; 2: always tensor cores */
  uint32_t miss_fetch;     /* batched search, cache misses: 0 = all scanned by
                              the host (reference semantics); 1 (default) =
                              adaptive runtime fetch: the most-shared misses
                              stream H2D through a 2-slot HBM ring and are
                              scanned on the GPU while the host scans the
                              rest, split by measured rates; 2 = every miss
                              the ring can take goes to the GPU */
  uint32_t fetch_chunk_mb; /* ring slot size in MiB; 0 = 512 */
  uint32_t single_chain;   /* single-query search: 0 (default) = one fused
                              cooperative kernel (query fetch, coarse scores,
                              top-L, residency split, TMA scan) where the shape
                              fits shared memory; 1 = the multi-kernel chain */
} laivg_opts;
void laivg_opts_default(laivg_opts* o);
typedef struct laivg_ctx laivg_ctx;
int laivg_ctx_create(const laivg_index* ix, const laivg_opts* opts,
                     laivg_ctx** out);
void laivg_ctx_destroy(laivg_ctx* ctx);
/* Waits for all device work of the context. */
int laivg_ctx_sync(laivg_ctx* ctx);

/* ---- coarse quantizer (ivf.cpp:269-299) ---------------------------------- */
/* Full ranking of all nc clusters for each of nq queries Q[nq*d]:
 * order_out[nq*nc]. scores_out (nullable) receives the fp64 scores indexed by
 * cluster id [nq*nc]. Replaces rank_clusters (ivf.hpp:68-69). */
int laivg_rank_clusters(laivg_ctx* ctx, const float* Q, uint32_t nq,
                        uint32_t* order_out, double* scores_out);
/* First min(max(L,0), nc) clusters per query: probe_out[nq*Lp] where
 * Lp = min(max(L,0), nc) is written to *lp_out. Replaces coarse_probe
 * (ivf.hpp:72-73). */
int laivg_coarse_probe(laivg_ctx* ctx, const float* Q, uint32_t nq, int L,
                       uint32_t* probe_out, uint32_t* lp_out);

/* ---- fine search ----------------------------------------------------------
 * Results: ids_out[nq*k], scores_out[nq*k], count_out[nq] (= min(k,
 * candidates)), best-first. Resident clusters are scanned on the GPU, the rest
 * by the host miss path; the merged result equals the monolithic search
 * whatever the residency (tiered.hpp:120-124). Any k >= 1: k <= 256 runs the
 * register top-k scans, larger k a radix sort of every candidate. */
/* search_clusters (ivf.hpp:85-87) for one query over an explicit cluster
 * list. */
int laivg_search_clusters(laivg_ctx* ctx, const float* q,
                          const uint32_t* clusters, uint32_t n, int k,
                          uint64_t* ids_out, float* scores_out,
                          uint32_t* count_out);
/* ivf_search (ivf.hpp:90-91) for nq queries. */
int laivg_ivf_search(laivg_ctx* ctx, const float* Q, uint32_t nq, int L,
                     int k, uint64_t* ids_out, float* scores_out,
                     uint32_t* count_out);

/* score_clusters (ivf.hpp:75-81, ivf.cpp:301-324): every member of
 * clusters[0..n) scored against q without ranking or truncation, in the
 * reference's order (clusters in the given order, duplicates included; each
 * list in its member order). Resident lists are scored on the GPU, the rest
 * by the host. cap = entries ids_out / scores_out hold (the sum of the lists'
 * lengths is needed: laivg_index_list_len); *count_out gets that sum.
 * LAIVG_EINVAL for an unknown cluster id or too small a buffer. */
int laivg_score_clusters(laivg_ctx* ctx, const float* q, const uint32_t* clusters, uint32_t n,
                         uint64_t cap, uint64_t* ids_out, float* scores_out,
                         uint64_t* count_out);
/* exact_search (vectorstore.hpp:94-98, vectorstore.cpp:117-139) over the
 * index's datastore for nq queries and any k >= 1: the best k of every row
 * (the union of the lists), ties by ascending id. */
int laivg_exact_search(laivg_ctx* ctx, const float* Q, uint32_t nq, int k, uint64_t* ids_out,
                       float* scores_out, uint32_t* count_out);
/* pairwise_l2 (vectorstore.hpp:100-102, vectorstore.cpp:141-153): out[i*nb+j]
 * = f32(sqrt(l2_sq_d(a_i, b_j))) with the reference's serial fp64
 * accumulation (bit-identical), computed on the context's GPU. */
int laivg_pairwise_l2(laivg_ctx* ctx, const float* a, uint64_t na, const float* b, uint64_t nb,
                      uint32_t d, float* out);

/* ---- tiered store = the GPU cluster cache (tiered.hpp:22-56) ------------- *//* ---- tiered store = the GPU cluster cache (tiered.hpp:22-56) ------------- */
uint64_t laivg_store_capacity_bytes(const laivg_ctx* ctx);
uint64_t laivg_store_used_bytes(const laivg_ctx* ctx);
uint64_t laivg_store_free_bytes(const laivg_ctx* ctx);
int laivg_store_contains(const laivg_ctx* ctx, uint32_t c); /* 1/0 */
uint32_t laivg_store_resident_count(const laivg_ctx* ctx);
/* Resident clusters ascending by id (std::map order): clusters_out[n],
 * tags_out[n] (nullable), bytes_out[n] (nullable); returns count via *n_out
 * (buffers must hold resident_count entries). */
int laivg_store_resident(const laivg_ctx* ctx, uint32_t* clusters_out,
                         uint8_t* tags_out, uint64_t* bytes_out,
                         uint32_t* n_out);
/* TieredStore::insert (tiered.cpp:15-24): makes cluster c resident with its
 * payload copied into the device cache (synchronously). Throws-equivalents:
 * LAIVG_ELOGIC already resident, LAIVG_ERUNTIME capacity exceeded. */
int laivg_store_insert(laivg_ctx* ctx, uint32_t c, int tag);
/* TieredStore::evict (tiered.cpp:26-36); *bytes_out = freed bytes. */
int laivg_store_evict(laivg_ctx* ctx, uint32_t c, uint64_t* bytes_out);
int laivg_store_retag_all(laivg_ctx* ctx, int tag);     /* tiered.cpp:38-42 */
int laivg_store_clear(laivg_ctx* ctx);                  /* tiered.cpp:44-47 */
uint64_t laivg_store_bytes_with_tag(const laivg_ctx* ctx, int tag);
uint64_t laivg_store_recompute_used_bytes(const laivg_ctx* ctx);
/* Compacts the device slab (paper: consolidate GPU memory after a batch). */
int laivg_store_compact(laivg_ctx* ctx);

/* ---- lookahead prefetch (tiered.hpp:97-117) ----------------------------- */
/* plan_prefetch (tiered.cpp:67-84) against the context's store: walks the
 * full ranking of q_in (GPU coarse), skips resident clusters, takes a cluster
 * if its bytes fit the remaining budget, else skips and continues.
 * plan_out / skipped_out must hold nc entries. */
int laivg_plan_prefetch(laivg_ctx* ctx, const float* q_in,
                        uint64_t budget_bytes, uint32_t* plan_out,
                        uint32_t* nplan_out, uint64_t* planned_bytes_out,
                        uint32_t* skipped_out, uint32_t* nskipped_out);

typedef struct {
  double bandwidth_bytes_per_s; /* tiered.hpp:69 */
  int mode;                     /* LAIVG_CHAN_* */
} laivg_channel;

typedef struct {
  double t_p;          /* seconds: transfer time (Device: copy-stream events;
                          Simulated: bytes/B; Measured: host wall clock) */
  uint64_t bytes;      /* tiered.hpp:80 */
  double overshoot_s;  /* max(0, t_p - window) (tiered.cpp:134); Device mode:
                          measured copy end minus window end, >= 0 */
  uint32_t n_transferred;
  double window_s;     /* measured duration of the generation-window kernel */
  double h2d_gbps;     /* achieved host->device GB/s of this transfer */
  double window_read_gbps; /* HBM read rate of a decode-like window
                              (laivg_window_load), 0 for the idle window */
} laivg_transfer_report;

/* execute_prefetch (tiered.cpp:86-136): inserts the planned clusters
 * (Prefetched) and copies their payload into the device cache. In
 * LAIVG_CHAN_DEVICE mode the copies run on the context's copy stream while a
 * timed generation-window kernel of overlap_window_s seconds occupies the
 * compute stream; the call returns when both have finished.
 * transferred_out (nullable) receives the transferred clusters in order. */
int laivg_execute_prefetch(laivg_ctx* ctx, const uint32_t* plan, uint32_t n,
                           const laivg_channel* chan, double overlap_window_s,
                           uint32_t* transferred_out,
                           laivg_transfer_report* rep);
/* incremental_prefetch (tiered.cpp:138-146). */
int laivg_incremental_prefetch(laivg_ctx* ctx, const float* q_round,
                               uint64_t budget_bytes,
                               const laivg_channel* chan,
                               double overlap_window_s,
                               uint32_t* transferred_out,
                               laivg_transfer_report* rep);
/* Lookahead prefetch of a micro-batch (replaces the per-trace plan/execute
 * loop of serve_microbatch, pipeline.cpp:357-371): one GPU coarse pass ranks
 * all nq predictor embeddings Q_in[nq*d]; query i then plans against the
 * store already holding the earlier plans with budget min(budgets[i], free
 * bytes) (plan_prefetch rule, tiered.cpp:67-84), and every planned list
 * streams host->HBM on the copy stream while ONE generation window of
 * overlap_window_s runs on the compute stream. Device channel only.
 * transferred_out (nullable, nc entries) gets the lists in transfer order,
 * nplan_out (nullable, nq entries) each query's planned count. */
int laivg_prefetch_batch(laivg_ctx* ctx, const float* Q_in, uint32_t nq,
                         const uint64_t* budgets, const laivg_channel* chan,
                         double overlap_window_s, uint32_t* transferred_out,
                         uint32_t* nplan_out, laivg_transfer_report* rep);
/* Runs only the generation-window kernel (seconds) on the compute stream and
 * returns its measured duration. */
int laivg_window(laivg_ctx* ctx, double seconds, double* measured_s);
/* Makes every later generation window decode-like: it streams a device buffer
 * of buffer_bytes (the "weights") once per token period at full speed, the
 * token period being buffer_bytes / read_gbps, so the lookahead copies share
 * HBM, L2 and the SMs with a memory-bound decode. read_gbps = 0 (or
 * buffer_bytes = 0) restores the idle %globaltimer window. */
int laivg_window_load(laivg_ctx* ctx, uint64_t buffer_bytes, double read_gbps);
/* Pinned host <-> device copy rate of this context's GPU, measured with one
 * large cudaMemcpyAsync per direction (independent of the prefetch path). */
int laivg_link_peak(laivg_ctx* ctx, uint64_t bytes, double* h2d_gbps, double* d2h_gbps);
/* Host-link bytes moved by this context's single-query searches so far
 * (query rows, residency tables, fetched lists; probes and results read
 * back) — the per-call counts of laivg_hybrid_timing, cumulative, for
 * callers that pass no timing struct. */
int laivg_link_bytes(const laivg_ctx* ctx, uint64_t* h2d_bytes, uint64_t* d2h_bytes);

/* Batched hit scan: how many batches ran the list-major tensor-core scan
 * (each resident list read once per 16 queries probing it; policy env
 * LAIVG_LIST_SCAN = 0 off / 1 on / unset auto), how many of those fell back
 * to the per-query scan (candidate buffer overflow), and the current EMA of
 * queries per resident probed list the auto policy reads. Extension of
 * search_clusters (ivf.cpp:301-343) for batches; results are identical. */
int laivg_list_scan_stats(const laivg_ctx* ctx, uint64_t* runs, uint64_t* fallbacks,
                          double* queries_per_list);

/* ---- hybrid search (tiered.cpp:148-198) ---------------------------------- */
typedef struct {
  double bandwidth_bytes_per_s; /* budget.hpp:14 */
  double t_cc;                  /* budget.hpp:15 */
  double t_gc;                  /* budget.hpp:16 */
  int parallel_slots;           /* budget.hpp:17 */
} laivg_cost_model;

typedef struct {
  /* Reference HybridTiming (tiered.hpp:84-88), now measured: */
  double t_g; /* GPU side: coarse + scan + merge, device events (s) */
  double t_c; /* host miss scan wall time (s) */
  double t_2; /* whole retrieval, call entry to merged result (s) */
  /* Modeled per the reference cost model (tiered.cpp:190-196): */
  double model_t_g, model_t_c, model_t_2;
  double t_coarse; /* device: coarse scores + selection (s) */
  double t_scan;   /* device: list scan + block/grid merge (s) */
  uint64_t scanned_vectors; /* vectors scanned on the GPU */
  uint64_t scanned_bytes;   /* reference bytes: n*(4D+8) over fast lists */
  /* batched search, runtime fetch of misses (zero otherwise): */
  uint32_t fetched_lists;   /* distinct missed lists fetched H2D + GPU-scanned */
  uint32_t cpu_lists;       /* distinct missed lists scanned by the host */
  uint64_t fetched_bytes;   /* vector bytes fetched on demand */
  double t_fetch;           /* copy-stream time of all fetch copies (s) */
  uint32_t peer_lists;      /* missed lists copied from a peer GPU's cache */
  uint32_t list_scan;       /* batched: 1 when the hits ran on the list-major
                               tensor-core scan (laivg_list_scan_stats) */
  uint64_t peer_bytes;
  /* bytes this call moved across the host link, counted from the copies it
     issued: h2d = query rows (host-buffer entry points) + the residency
     table when it changed + runtime-fetched lists; d2h = probes and partial
     / final result lists read back (mapped or copied) */
  uint64_t h2d_bytes;
  uint64_t d2h_bytes;
  /* single query on the fused kernel: its device-event duration (s); t_coarse
     is then its coarse + selection phase (CTA 0's globaltimer) and t_scan the
     rest. 0 when the multi-kernel chain ran. */
  double t_kernel;
  /* batched: vector bytes (4·d·n) of the DISTINCT resident probed lists, what
     a list-major scan reads at least once (scanned_bytes counts every
     (query, list) pair) */
  uint64_t distinct_bytes;
} laivg_hybrid_timing;

/* hybrid_search for one query. fast_out / slow_out (nullable, L entries)
 * receive the probe split by residency in probe order. */
int laivg_hybrid_search(laivg_ctx* ctx, const float* q_out, int L, int k,
                        const laivg_cost_model* cost, uint64_t* ids_out,
                        float* scores_out, uint32_t* count_out,
                        uint32_t* fast_out, uint32_t* nfast_out,
                        uint32_t* slow_out, uint32_t* nslow_out,
                        double* hit_rate_out, laivg_hybrid_timing* timing);

/* coverage (tiered.cpp:200-211). */
int laivg_coverage(laivg_ctx* ctx, const float* q_in, const float* q_out,
                   int L, double* out);

/* ---- device-resident query staging (benchmark path: inputs already in HBM)
 * Upload nq queries once; laivg_hybrid_search_staged then reads query i from
 * HBM instead of copying it from the host. */
int laivg_stage_queries(laivg_ctx* ctx, const float* Q, uint32_t nq);
int laivg_hybrid_search_staged(laivg_ctx* ctx, uint32_t qi, int L, int k,
                               uint64_t* ids_out, float* scores_out,
                               uint32_t* count_out, uint32_t* nfast_out,
                               laivg_hybrid_timing* timing);

/* ---- batched retrieval (extension point (2) of SURVEY §8b: the reference
 * loops hybrid_search over a batch, pipeline.cpp:391-428) ------------------
 * hybrid_search for nq <= max_batch queries Q[nq*d] in one device pass: one
 * coarse launch (tensor cores for nq >= 16), one residency split, one scan
 * launch for the whole batch; the misses of all queries are scanned
 * list-major on the host while the GPU scans the hits. Per query the result
 * equals laivg_hybrid_search. ids_out/scores_out [nq*k], count_out [nq],
 * nfast_out [nq] (nullable); timing (nullable) is for the whole batch. */
int laivg_hybrid_search_batch(laivg_ctx* ctx, const float* Q, uint32_t nq, int L,
                              int k, const laivg_cost_model* cost,
                              uint64_t* ids_out, float* scores_out,
                              uint32_t* count_out, uint32_t* nfast_out,
                              laivg_hybrid_timing* timing);
/* The same over staged queries [q0, q0 + nq) (inputs already in HBM). */
int laivg_hybrid_search_batch_staged(laivg_ctx* ctx, uint32_t q0, uint32_t nq,
                                     int L, int k, uint64_t* ids_out,
                                     float* scores_out, uint32_t* count_out,
                                     uint32_t* nfast_out,
                                     laivg_hybrid_timing* timing);
/* Diagnostics: the raw tf32 tensor-core scores approx_out[nq*nc] the batched
 * coarse quantizer filters with (never reported as results). */
int laivg_debug_coarse_approx(laivg_ctx* ctx, const float* Q, uint32_t nq,
                              float* approx_out);

/* ---- the slow tier on its own -------------------------------------------
 * The host half of hybrid_search (tiered.cpp:169: the clusters not cached on
 * the GPU are scored on the host) as a standalone call: for each query q the
 * best-k over the members of lists[lists_off[q] .. lists_off[q+1]), scored
 * list-major (each row read once for all queries that name its list) with
 * the reference's fp64 arithmetic. This is the paper's CPU tier, used by the
 * device path for cache misses; it is not a replacement for the GPU scan. */
int laivg_slow_tier_scan(const laivg_index* ix, const float* Q, uint32_t nq,
                         const uint32_t* lists, const uint32_t* lists_off, int k,
                         uint32_t threads, uint64_t* ids_out, float* scores_out,
                         uint32_t* count_out);

/* ---- peer caches (beyond the paper's private caches) ---
 * A miss of one GPU that another GPU of the node caches is copied from that
 * GPU's slab over NVLink into the ring and scanned locally, instead of being
 * scanned by the host or fetched over PCIe (batched search, miss_fetch != 0).
 * Protocol per step, on every worker: laivg_epoch_open; publish
 * laivg_store_offsets to the others (all-gather across processes); each
 * worker laivg_peer_publish-es the others' offsets; serve; barrier;
 * laivg_epoch_close. Opening an epoch publishes (pins) the lists resident
 * at that moment: until it closes they keep their slab ranges (an explicit
 * eviction quarantines the range, evict_to_fraction passes over them) and
 * the slab is not compacted; lists inserted during the epoch are not
 * published and churn as usual. laivg_store_offsets reports the published
 * lists while an epoch is open. Peers attach once: in one process from the other context
 * (laivg_peer_attach_local, enables P2P between devices), across processes
 * from a CUDA IPC handle of the peer's slab (laivg_slab_ipc_handle, 64 B). */
int laivg_epoch_open(laivg_ctx* ctx);
int laivg_epoch_close(laivg_ctx* ctx);
/* Slab vector offset of every cluster, -1 when not resident: off_out[nc]. */
int laivg_store_offsets(const laivg_ctx* ctx, int64_t* off_out);
int laivg_slab_ipc_handle(laivg_ctx* ctx, void* handle_out);
int laivg_peer_attach_ipc(laivg_ctx* ctx, uint32_t peer, const void* handle);
int laivg_peer_attach_local(laivg_ctx* ctx, uint32_t peer, const laivg_ctx* other);
/* The peer's published offsets for the open epoch (nullptr: none). */
int laivg_peer_publish(laivg_ctx* ctx, uint32_t peer, const int64_t* offsets);

/* ---- schedulers (sched.cpp) ---------------------------------------------- */
/* group_microbatches (sched.cpp:39-70): order_out[n] holds the queries batch
 * by batch, batch_off_out[nb+1] the CSR offsets; *nb_out = #batches. */
int laivg_group_microbatches(const float* queries, uint64_t n, uint32_t d,
                             uint64_t m, uint64_t* order_out,
                             uint64_t* batch_off_out, uint32_t* nb_out);
/* chunk_microbatches (sched.cpp:72-85) */
int laivg_chunk_microbatches(uint64_t n, uint64_t m, uint64_t* order_out,
                             uint64_t* batch_off_out, uint32_t* nb_out);
/* assign_cache_aware (sched.cpp:87-144). Batches in CSR form; resident is
 * [nw][nc] bytes (1 = worker caches the cluster). Probe unions come from the
 * context's GPU coarse quantizer. */
int laivg_assign_cache_aware(laivg_ctx* ctx, const uint64_t* batch_off,
                             const uint64_t* members, uint32_t nb,
                             const uint8_t* resident, uint32_t nw,
                             const float* queries, uint64_t nq, int L,
                             uint32_t* assignment_out);
/* group_microbatches on the GPU (same outputs as laivg_group_microbatches,
 * bit-identical: pairwise fp64 L2^2 in the reference's serial order, then the
 * greedy in one CTA). n <= 8192. */
int laivg_group_microbatches_gpu(laivg_ctx* ctx, const float* queries, uint64_t n,
                                 uint64_t m, uint64_t* order_out,
                                 uint64_t* batch_off_out, uint32_t* nb_out);
/* The routing step of run_batch (pipeline.cpp:541-589) in one call, on the
 * GPU: group_microbatches (m per batch), every query's coarse probe (L),
 * the overlap matrix of each batch's probe union with each worker's resident
 * set ([nw][nc] bytes) as bitset popcounts, then the cache-aware greedy
 * (sched.cpp:114-142). Outputs: batches in CSR form (order_out[n],
 * batch_off_out[nb+1], *nb_out), assignment_out[nb] (nullable) and the
 * overlap matrix overlap_out[nb*nw] (nullable). n <= 8192. */
int laivg_schedule(laivg_ctx* ctx, const float* queries, uint64_t n, uint64_t m, int L,
                   const uint8_t* resident, uint32_t nw, uint64_t* order_out,
                   uint64_t* batch_off_out, uint32_t* nb_out, uint32_t* assignment_out,
                   uint64_t* overlap_out);
/* The greedy of assign_cache_aware (sched.cpp:114-142) over a precomputed
 * row-major nb x nw overlap matrix: a multi-process router all-gathers the
 * workers' resident sets, builds the matrix and every rank assigns alike. */
int laivg_greedy_assign(const uint64_t* overlap, uint32_t nb, uint32_t nw,
                        uint32_t* assignment_out);
/* assign_round_robin (sched.cpp:146-155) */
int laivg_assign_round_robin(uint64_t nb, uint64_t nw, uint32_t* out);
/* assignment_overlap (sched.cpp:157-168) */
int laivg_assignment_overlap(laivg_ctx* ctx, const uint64_t* batch_off,
                             const uint64_t* members, uint32_t nb,
                             const uint8_t* resident, uint32_t nw,
                             const uint32_t* assignment, const float* queries,
                             uint64_t nq, int L, uint64_t* out);
/* split_budget (sched.cpp:170-192) */
int laivg_split_budget(uint64_t total, const uint64_t* batch, uint64_t n,
                       uint64_t* out);

/* ---- hotness cache policy (cache.hpp:28-56) ------------------------------ */
typedef struct laivg_hotness laivg_hotness;
int laivg_hotness_create(float h_init, float h_inc, float decay,
                         double cache_fraction, laivg_hotness** out);
void laivg_hotness_destroy(laivg_hotness* h);
int laivg_hotness_on_fetch(laivg_hotness* h, uint32_t c);          /* cache.cpp:27 */
int laivg_hotness_end_of_round(laivg_hotness* h, const uint32_t* used,
                               uint32_t n);                       /* cache.cpp:31 */
/* evict_to_fraction (cache.cpp:40-66) on the context's store; evicted_out
 * (nullable, resident_count entries) receives the evicted ids in order. */
int laivg_hotness_evict_to_fraction(laivg_hotness* h, laivg_ctx* ctx,
                                    uint32_t* evicted_out, uint32_t* n_out);
/* hotness of c, or -1 when untracked */
float laivg_hotness_get(const laivg_hotness* h, uint32_t c);
int laivg_hotness_forget(laivg_hotness* h, uint32_t c);
int laivg_hotness_clear(laivg_hotness* h);

/* ---- synthetic workload (the generator of SURVEY §8d; not on the path) ---
 * Planted clusters: centroids mu_j = normalize(g), members
 * x = normalize(mu_j + spread*g), balanced lists, ids j*n_j+i, list-major.
 * Deterministic from (seed, j, i, dim) and bit-identical across thread
 * counts. vecs must hold n_total*d floats. */
int laivg_synth_centroids(uint64_t seed, uint32_t nc, uint32_t d,
                          float* centroids_out);
int laivg_synth_lists(uint64_t seed, const float* centroids, uint32_t nc,
                      uint32_t d, uint64_t per_list, float spread,
                      uint32_t c_begin, uint32_t c_end, float* vecs_out,
                      uint64_t* ids_out, int threads);
/* q_in = normalize(x_r + 0.01 g) for uniform rows r; q_out =
 * normalize(q_in + sigma g) (trace.cpp:203-220 pattern). */
int laivg_synth_queries(uint64_t seed, const float* vecs, uint64_t n_rows,
                        uint32_t d, uint32_t nq, float sigma, float* q_in_out,
                        float* q_out_out, uint64_t* rows_out);

/* Topical queries for the routed batches (C3-C5 skew): topic
 * t ~ Zipf(zipf_s) over n_topics random centre lists; each query's source
 * row is drawn from one of the `neigh` lists nearest its topic centre, then
 * q_in / q_out as laivg_synth_queries. topic_out (nullable) gets t. */
int laivg_synth_queries_topical(uint64_t seed, const float* centroids, uint32_t nc,
                                const float* vecs, const uint64_t* list_off,
                                uint32_t d, uint32_t n_topics, double zipf_s,
                                uint32_t neigh, uint32_t nq, float sigma,
                                float* q_in_out, float* q_out_out,
                                uint64_t* rows_out, uint32_t* topic_out);

#ifdef __cplusplus
}
#endif
#endif /* LAIVG_H */
