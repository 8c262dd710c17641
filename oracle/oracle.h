/*
 * oracle.h — CPU restatement of the reference `laiv` hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_2502_20969_b200/)
 * includes, links or calls this. Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py use it, and only as the checker.
 *
 * Every function restates one reference function in plain C with the same
 * arithmetic: fp64 accumulation in index order, fp32 rounding of per-candidate
 * scores, Euclidean (sqrt) distances for the fine scan, squared L2 for the
 * coarse ranking, and the (score, ascending id) total order. Citations are
 * /root/reference/proj/... file:line.
 *
 * Parity pinning: the oracle is checked against golden vectors produced by the
 * reference itself (oracle/_ref, built from the reference sources by
 * oracle/Makefile; fixtures in tests/golden/ made by tests/golden/make_golden.py).
 *
 * Store layout (the LAIX list-major order, ivf.cpp:373-388 / 437-455):
 *   vecs[N][D] f32, ids[N] u64, list_off[nc+1] u64; list c is rows
 *   [list_off[c], list_off[c+1]).
 */
#ifndef LAIV_ORACLE_H
#define LAIV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_IP = 0, ORC_L2 = 1 }; /* vectorstore.hpp:18 */

/* --- Rng restatement (rng.hpp:16-75) ----------------------------------- */
typedef struct {
  uint64_t mt[312];
  int mti;
  int have_spare;
  double spare;
} orc_rng;
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next_u64(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
double orc_rng_gaussian(orc_rng* r);
uint64_t orc_rng_index(orc_rng* r, uint64_t n);
uint64_t orc_derive_seed(uint64_t seed, const char* label);
/* test_util.hpp:16-39: n x dim rows of float(scale * gaussian()). */
void orc_random_matrix(uint64_t n, uint32_t dim, uint64_t seed, double scale,
                       float* out);

/* --- scoring (vectorstore.cpp:93-115) ---------------------------------- */
double orc_dot_d(const float* a, const float* b, uint32_t d);
double orc_l2_sq_d(const float* a, const float* b, uint32_t d);
float orc_score_rounded(int metric, const float* q, const float* row,
                        uint32_t d);
/* vectorstore.hpp:34-39 */
int orc_ranks_before(int metric, float sa, uint64_t ia, float sb, uint64_t ib);

/* --- coarse quantizer (ivf.cpp:269-299) -------------------------------- */
/* Full ranking; scores_out (optional) receives the unrounded fp64 scores
 * (dot for IP, squared L2 for L2) indexed by cluster id. */
void orc_rank_clusters(const float* centroids, uint32_t nc, uint32_t d,
                       int metric, const float* q, uint32_t* order_out,
                       double* scores_out);
uint32_t orc_coarse_probe(const float* centroids, uint32_t nc, uint32_t d,
                          int metric, const float* q, int L, uint32_t* out);

/* --- fine scan (ivf.cpp:301-349; vectorstore.cpp:117-141) -------------- */
/* Returns the number of entries written (min(k, candidates)), -1 on k < 1,
 * -2 on an unknown cluster id. */
int orc_search_clusters(const float* vecs, const uint64_t* ids,
                        const uint64_t* list_off, uint32_t nc, uint32_t d,
                        int metric, const float* q, const uint32_t* clusters,
                        uint32_t ncl, int k, uint64_t* ids_out,
                        float* scores_out);
int orc_ivf_search(const float* centroids, const float* vecs,
                   const uint64_t* ids, const uint64_t* list_off, uint32_t nc,
                   uint32_t d, int metric, const float* q, int L, int k,
                   uint64_t* ids_out, float* scores_out);
int orc_exact_search(const float* db, const uint64_t* ids, uint64_t n,
                     uint32_t d, int metric, const float* q, int k,
                     uint64_t* ids_out, float* scores_out);

/* --- tiering (tiered.cpp:67-84, 148-211) ------------------------------- */
/* Walk `order` (a full ranking), skip resident, take if bytes <= remaining
 * else skip and continue. Returns number of planned clusters. */
uint32_t orc_plan_prefetch(const uint32_t* order, uint32_t nc,
                           const uint64_t* cluster_bytes,
                           const uint8_t* resident, uint64_t budget,
                           uint32_t* plan_out, uint64_t* planned_bytes,
                           uint32_t* skipped_out, uint32_t* nskipped);
double orc_coverage(const float* centroids, uint32_t nc, uint32_t d,
                    int metric, const float* q_in, const float* q_out, int L);

/* --- scheduling (sched.cpp:39-192) ------------------------------------- */
/* Output: batch_of[n] (batch index per query) and members in batch order via
 * order_out[n] (queries concatenated batch by batch); returns #batches. */
uint32_t orc_group_microbatches(const float* queries, uint64_t n, uint32_t d,
                                uint64_t m, uint64_t* order_out,
                                uint64_t* batch_off_out);
/* batches in CSR (batch_off[nb+1], members[]), resident bitmaps [nw][nc].
 * Writes assignment[nb]; returns 0 or -1 (no workers). */
int orc_assign_cache_aware(const uint64_t* batch_off, const uint64_t* members,
                           uint32_t nb, const uint8_t* resident, uint32_t nw,
                           const float* centroids, uint32_t nc, uint32_t d,
                           int metric, const float* queries, int L,
                           uint32_t* assignment);
uint64_t orc_assignment_overlap(const uint64_t* batch_off,
                                const uint64_t* members, uint32_t nb,
                                const uint8_t* resident, uint32_t nw,
                                const uint32_t* assignment,
                                const float* centroids, uint32_t nc,
                                uint32_t d, int metric, const float* queries,
                                int L);
int orc_split_budget(uint64_t total, const uint64_t* batch, uint64_t n,
                     uint64_t* out);

/* --- hotness law (cache.cpp:27-66) ------------------------------------- */
/* h' = h/d (+ h_inc when used), float32. */
void orc_hotness_end_of_round(float* h, const uint8_t* used, uint32_t n,
                              float decay, float h_inc);

#ifdef __cplusplus
}
#endif
#endif
