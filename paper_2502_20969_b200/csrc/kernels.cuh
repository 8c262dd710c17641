// kernels.cuh — launch interface of the sm_100a kernels (kernels.cu).
// Host orchestration (ctx.cu) calls these; nothing here is part of the C ABI.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

namespace laivg {

// Every kernel launch of this library increments this (evidence for the
// bench's gpu_launches).
std::atomic<uint64_t>& launch_counter();
// Counts a launch and throws CudaError on a launch-configuration error.
void after_launch();
// Raises a kernel's dynamic shared-memory limit once per (kernel, device).
void ensure_dyn_smem(const void* fn, size_t bytes);

constexpr int kMaxK = 256;             // device top-k limit (8 entries per lane)
constexpr int kRerankMargin = 16;      // extra fp32 survivors re-scored in fp64
constexpr uint32_t kMaxSortNc = 16384; // on-chip full ranking limit

// Per-query fast-list table produced by the partition step and consumed by
// the scan: entry f of query q lives at [q * stride + f].
// Where scan CTA b of a query starts: list index, offset in the list and the
// number of vectors it scans (the partition step fills it for `grid` CTAs).
struct CtaStart {
  uint32_t li;
  uint32_t o;
  uint32_t n;
  uint32_t pad;
};

struct FastTable {
  int64_t* slab;      // device-cache vector offset of the list
  uint64_t* row;      // host-store row offset of the list (id table index)
  uint32_t* len;      // list length (vectors)
  uint32_t* cluster;  // cluster id (for the host)
  uint64_t* pre;      // exclusive prefix of len, stride + 1 entries per query
  uint32_t* count;    // number of fast lists per query
  CtaStart* cta;      // [nq][grid] scan CTA start table (nullable)
  uint32_t stride;
  uint32_t grid;      // CTAs per query the cta table was built for
};

constexpr uint32_t kGroup = 16;     // CTAs merged by one group-last CTA
constexpr uint32_t kMaxGroups = 64; // groups per query (grid <= 1024)

struct ScanOut {
  float* part_s;      // [nq][grid][kk] per-CTA partial top-kk
  uint64_t* part_id;  // datastore ids
  uint32_t* part_vi;  // slab vector index of each partial entry (re-score)
  float* gpart_s;     // [nq][kMaxGroups][kk] per-group partial top-kk
  uint64_t* gpart_id;
  uint32_t* gpart_vi;
  unsigned* ticket;   // [nq][kMaxGroups + 1] group / final tickets (self-resetting)
  float* out_s;       // [nq][k]
  uint64_t* out_id;   // [nq][k]
  uint32_t* out_count;// [nq]
  // optional: the final CTA also copies fcount_in[q] (the partition's fast
  // list count) to fcount_out[q]; outputs may live in mapped host memory
  const uint32_t* fcount_in = nullptr;
  uint32_t* fcount_out = nullptr;
  // host-final mode (fp64 accumulation only): every CTA writes its sorted
  // top-kk (score, host-store row) to cta_s / cta_r [nq][grid][kk] (mapped
  // host memory) and the host merges the grid; no device grid merge
  float* cta_s = nullptr;
  uint64_t* cta_r = nullptr;
  // diagnostics (LAIVG_SCAN_PROBE): per CTA globaltimer stamps [nq][grid][4]
  // = entry, first tile landed, last tile consumed, epilogue done
  unsigned long long* probe = nullptr;
};

enum class ScanImpl : int {
  kTma = 0,      // cp.async.bulk (TMA) staged, warp-specialised (default)
  kLdg = 1,      // direct 128-bit loads into registers
};

// Optional geometry overrides of the TMA scan (0 = automatic).
struct ScanTune {
  uint32_t tile = 0;        // vectors per ring stage
  uint32_t stages = 0;      // ring depth
  uint32_t ctas_per_sm = 0; // scan CTAs per SM
};

// Coarse: fp64 scores[nq][nc] of Q[nq][d] against centroids[nc][d]
// (dot for IP, squared L2 for L2; ivf.cpp:276-280).
void launch_coarse_scores(const float* Q, uint32_t nq, const float* centroids,
                          uint32_t nc, uint32_t d, int metric, double* scores,
                          cudaStream_t st);
// Full on-chip ranking of each query's scores, best-first with ascending
// cluster id on ties (ivf.cpp:282-289); writes the first n_out entries of
// each ranking to order[q * n_out + i]. nc <= kMaxSortNc. With `ft`, also
// splits the first n_out entries by residency (fused partition).
// run_k / run_v: scratch of select_scratch_entries(nq, nc) entries.
void launch_select(const double* scores, uint32_t nq, uint32_t nc, int metric,
                   uint32_t n_out, uint32_t* order, uint64_t* run_k, uint32_t* run_v,
                   const int64_t* res_off, const uint64_t* list_off, const FastTable* ft,
                   cudaStream_t st, bool scan_sorted = false);
size_t select_scratch_entries(uint32_t nq, uint32_t nc);
// Splits each query's probe (probe[q * lp + i], i < lp) by residency
// (res_off[c] >= 0) preserving probe order; fills the fast table.
void launch_partition(const uint32_t* probe, uint32_t nq, uint32_t lp,
                      const int64_t* res_off, const uint64_t* list_off,
                      FastTable ft, cudaStream_t st);
// Scans the fast lists of nq queries (queries at Q[q * d]) and leaves the
// best-k (score, id) per query in out. grid_x CTAs per query.
void launch_scan(const float* Q, uint32_t nq, uint32_t d, int metric, int k,
                 const FastTable& ft, const float* slab_vecs,
                 const uint64_t* ids_all, const ScanOut& out, int grid_x,
                 bool acc_fp64, ScanImpl impl, const ScanTune& tune, cudaStream_t st);
int scan_grid_x(uint32_t nq, int num_sms, ScanImpl impl, const ScanTune& tune);
// Entries each per-CTA partial list holds for a given k (k + re-score margin).
int scan_kk(int k, bool acc_fp64);
// ---- fused single-query kernel (kernels.cu) ----
// query fetch -> coarse scores -> top-L -> residency split -> TMA scan in one
// cooperative launch of `grid` CTAs (one per SM). Results as launch_scan's
// (host-final or device-merged per `out`); the probe and the fast-list count
// land in mapped memory followed by the call's sequence number in *flag_out.
struct FusedQuery {
  const float* src = nullptr;          // query row (pinned host or HBM), or
  const float* const* slot = nullptr;  // mapped word holding the row pointer
  float* dQ = nullptr;
  const float* cen = nullptr;
  uint32_t nc = 0, d = 0, L = 0;
  int metric = 0, k = 0;
  uint64_t* keys = nullptr;            // [nc] device scratch
  const int64_t* res_off = nullptr;
  const uint64_t* list_off = nullptr;
  uint32_t* order_out = nullptr;       // [L] (device-visible, mapped)
  uint32_t* fcount_out = nullptr;
  unsigned* flag_out = nullptr;
  unsigned* done_out = nullptr;        // mapped: sequence number once every CTA's results are out
  unsigned* ctl = nullptr;             // [3] device: barrier word, sequence, done ticket (zeroed)
  // [8] CTA 0 globaltimer stamps (mapped), nullable: entry, query ready,
  // keys ready, keys loaded, top-L selected, scan ranges ready, last tile
  // consumed, done
  unsigned long long* stamps = nullptr;   // [32]; [8..19] selection stamps
  unsigned long long* cta_stamps = nullptr; // [grid][4] per CTA (diagnostics), nullable
  int qdirect = 0;                     // host row read by every CTA (diagnostics)
  const float* slab = nullptr;
  const uint64_t* ids = nullptr;
  uint32_t grid = 0;
};
// Dynamic shared memory of the fused kernel for this shape, 0 if it does not
// fit (the caller then runs the multi-kernel chain).
size_t fused_query_smem(uint32_t nc, uint32_t d, uint32_t L, int k, bool acc_fp64, uint32_t G,
                        const ScanTune& tune);
void launch_fused_query(const FusedQuery& q, const ScanOut& out, bool acc_fp64,
                        const ScanTune& tune, cudaStream_t st);
// ---- batched coarse quantizer on tensor cores (coarse_tc.cu) ----
// Used for batches of >= kTcMinBatch queries when nc <= kTcMaxNc and d % 4 == 0.
constexpr uint32_t kTcMinBatch = 16; // measured crossover (profiles/r01/coarse_bench.jsonl)
constexpr uint32_t kTcMaxNc = 8192;
// |tf32 score - exact score| <= kTcErr * ||q|| * ||c|| (2^-9 operand truncation
// + fp32 accumulation over d <= 4096 terms, with a 2x margin).
constexpr double kTcErr = 4.0e-3;
bool coarse_tc_supported(uint32_t nc, uint32_t d);
// Split-K partial planes approx[S][nq][nc] of the tf32 tensor-core Q . C^T
// (tcgen05.mma kind::tf32); S (returned, <= kTcMaxSplit) sizes the grid to
// the SM count. The exact score is within kTcErr ||q|| ||c|| of the plane sum.
constexpr uint32_t kTcMaxSplit = 8;
uint32_t coarse_tc_splits(uint32_t nq, uint32_t nc, uint32_t d, int num_sms);
uint32_t launch_coarse_tc(const float* Q, uint32_t nq, const float* centroids, uint32_t nc,
                          uint32_t d, float* approx, int num_sms, cudaStream_t st);
// Exact first n_out of each query's ranking from the approximate scores:
// candidates whose upper bound reaches the n_out-th best lower bound are
// re-scored with the fp64 arithmetic of launch_coarse_scores and sorted on
// (score, cluster id). With `ft`, also splits the probe by residency.
// cnorm[c] = ||c|| rounded up.
// Device scratch of the three-kernel batched selection: candidates and
// their exact keys [nq][cap] (cap = pow2 >= nc), counts [nq].
struct TcSelectScratch {
  uint32_t* cand = nullptr;
  uint64_t* key = nullptr;
  uint32_t* ncand = nullptr;
  // list-major re-score: per 32-query block and centroid, the bit set of
  // block queries that hold the centroid as a candidate [ceil(nq/32)][nc];
  // key is then indexed by centroid id ([nq][cap], cap >= nc)
  uint32_t* qmask = nullptr;
};
void launch_tc_select(const float* approx, uint32_t splits, const float* Q, uint32_t nq,
                      uint32_t d,
                      const float* centroids, const float* cnorm, uint32_t nc, int metric,
                      uint32_t n_out, uint32_t* order, const int64_t* res_off,
                      const uint64_t* list_off, const FastTable* ft, cudaStream_t st,
                      bool scan_sorted = false, const TcSelectScratch* sc = nullptr);
// ---- list-major batched scan on tensor cores (listscan.cu) ----
// Device scratch: per-cluster query counts / cursors [nc], resident lists
// with their query offsets and work-item offsets [nc + 1], query slots
// [nq * L], per-query candidates [nq][gcap] (16 B each), counts and shared
// thresholds [nq], meta[4].
struct ListScanScratch {
  uint32_t* qcount = nullptr;
  uint32_t* lists = nullptr;
  uint32_t* lq_off = nullptr;
  uint32_t* item_off = nullptr;
  uint32_t* qidx = nullptr;
  uint32_t* meta = nullptr;
  uint32_t* gtau = nullptr;
  uint32_t* gcnt = nullptr;
  void* cand = nullptr;
  uint32_t gcap = 0;
};
struct ListScan {
  const float* Q = nullptr;          // [nq][d] on the device
  uint32_t nq = 0, d = 0, nc = 0, lp = 0;
  int metric = 0, k = 0;
  const uint32_t* order = nullptr;   // [nq][lp] probe
  const int64_t* res = nullptr;      // residency (slab row of each list or -1)
  const uint64_t* list_off = nullptr;
  const float* slab = nullptr;
  uint64_t slab_rows = 0;
  const uint64_t* ids = nullptr;
  float* out_s = nullptr;            // [nq][k]
  uint64_t* out_id = nullptr;
  uint32_t* out_count = nullptr;
  const uint32_t* fcount_in = nullptr;
  uint32_t* fcount_out = nullptr;
  unsigned* flag_host = nullptr;     // set to 1 if a candidate buffer overflowed
  int grid = 0;
  uint32_t group = 16;               // queries per work item: 16, or 32 for heavily shared lists
  uint32_t chunk = 1024;             // list rows per work item (multiple of 128, <= 65536)
  ListScanScratch scratch;
};
bool list_scan_supported(uint32_t d, int k, uint32_t group = 16);
size_t list_scan_smem(uint32_t d, uint32_t group = 16);
// Exact per-query top-k of the resident probed lists (the per-query scan's
// result) into out_*; on overflow *flag_host = 1 and the outputs are invalid.
void launch_list_scan(const ListScan& p, cudaStream_t st);
// ---- schedulers on the GPU (sched.cu) ----
// dist[i * n + j] (j > i) = serial fp64 L2^2 of queries i and j (the
// reference's l2_sq_d order: bit-identical to the CPU).
void launch_pair_dist(const float* Q, uint32_t n, uint32_t d, double* dist, cudaStream_t st);
// group_microbatches' greedy (sched.cpp:39-70) over dist, one CTA.
uint32_t group_max_queries();
void launch_group(const double* dist, uint32_t n, uint32_t m, uint64_t* order, uint64_t* off,
                  uint32_t* nb, cudaStream_t st);
// group_microbatches for any n without the n x n matrix: one persistent
// (cooperative) grid walks the seeds; bit-identical to launch_group.
struct GroupScratch {
  unsigned char* taken = nullptr; // [n]
  double* dist_row = nullptr;     // [n]
  double* slot_d = nullptr;       // [2 * max grid]
  uint32_t* slot_i = nullptr;
  void* bar = nullptr;            // grid barrier (2 words)
  uint64_t n = 0;
};
constexpr uint32_t kGroupLargeMaxGrid = 1024;
void launch_group_large(const float* Q, uint32_t n, uint32_t d, uint32_t m, GroupScratch& gs,
                        uint64_t* order, uint64_t* off, uint32_t* nb, int num_sms,
                        cudaStream_t st);
// overlap[b][w] = |probe union of batch b  ∩  resident bitset of worker w|.
void launch_overlap(const uint32_t* probes, uint32_t L, const uint64_t* order,
                    const uint64_t* off, uint32_t nb, const unsigned long long* resident,
                    uint32_t nw, uint32_t words, unsigned long long* overlap, cudaStream_t st);
// ---- size-unbounded paths (wide.cu) ----
// Datastore id ranks: rank_of_row[r] = rank of ids[r] among all ids,
// row_of_rank its inverse (n < 2^32).
void build_id_rank(const uint64_t* ids, uint64_t n, uint32_t* rank_of_row, uint32_t* row_of_rank,
                   cudaStream_t st);
// Scores the V fast-list members of query qi (fast table ft, query vector q
// on the device): keys[v] = (score key << 32) | rank_of_row[row] (keys set),
// or raw (score, id) in candidate order (raw_s / raw_id set).
void launch_score_all(const float* q, uint32_t qi, uint32_t d, int metric, const FastTable& ft,
                      const float* slab, const uint32_t* rank_of_row, const uint64_t* ids,
                      uint64_t V, uint64_t* keys, float* raw_s, uint64_t* raw_id, int num_sms,
                      cudaStream_t st);
size_t wide_sort_temp_bytes(uint64_t n);
// Sorts keys[0, V) into keys_alt and writes the first min(k, V) as (score,
// id) to out_s / out_id, out_count[0]; fcount_out[0] = fcount_in[qi].
void launch_wide_topk(uint64_t* keys, uint64_t* keys_alt, uint64_t V, int k, int metric,
                      void* tmp, size_t tmp_bytes, const uint32_t* row_of_rank,
                      const uint64_t* ids, float* out_s, uint64_t* out_id, uint32_t* out_count,
                      const uint32_t* fcount_in, uint32_t* fcount_out, uint32_t qi,
                      cudaStream_t st);
// Coarse ranking prefix for any nc (multi-CTA radix sort per query).
struct RankScratch {
  uint64_t* keys = nullptr;
  uint64_t* keys_alt = nullptr;
  uint32_t* vals = nullptr;
  uint32_t* vals_alt = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
};
size_t rank_large_temp_bytes(uint32_t nc);
void launch_rank_large(const double* scores, uint32_t nq, uint32_t nc, int metric, uint32_t n_out,
                       uint32_t* order, RankScratch& rs, cudaStream_t st);
// pairwise_l2 (vectorstore.cpp:141-153): out[i * nb + j] = f32(sqrt(serial
// fp64 l2_sq_d(A_i, B_j))), or the fp64 squared distances into out_sq.
void launch_pairwise_l2(const float* A, uint64_t na, const float* B, uint64_t nb, uint32_t d,
                        float* out, double* out_sq, cudaStream_t st);
// Generation-window stand-in: one CTA per SM spins on %globaltimer for ns.
void launch_fetch_query(const float* src, const float* const* slot, float* dQ, uint32_t d,
                        cudaStream_t st);
void launch_window(uint64_t ns, int num_sms, cudaStream_t st);
// Decode-like window: every period_ns the grid streams `bytes` of buf (the
// "weights") once at full speed, for ns nanoseconds; bytes read are added to
// *bytes_read.
void launch_window_stream(const float* buf, uint64_t bytes, uint64_t ns, uint64_t period_ns,
                          int num_sms, float* sink, unsigned long long* bytes_read,
                          cudaStream_t st);

} // namespace laivg
