/*
 * oracle.c — CPU restatement of the reference `laiv` hot path.
 * TEST INFRASTRUCTURE ONLY (see oracle.h). Build: oracle/Makefile.
 * Compiled with -ffp-contract=off so every fp64 add/mul rounds exactly as the
 * reference's scalar loops do.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================= */
/* Rng: std::mt19937_64 + the hand-rolled draws of rng.hpp:16-54.          */
/* ======================================================================= */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ull
#define MT_LOWER 0x000000007FFFFFFFull

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  }
  r->mti = MT_N;
  r->have_spare = 0;
  r->spare = 0.0;
}

uint64_t orc_rng_next_u64(orc_rng* r) {
  if (r->mti >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      uint64_t x = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->mti = 0;
  }
  uint64_t y = r->mt[r->mti++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:23 */
double orc_rng_uniform(orc_rng* r) {
  return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

/* rng.hpp:28 */
uint64_t orc_rng_index(orc_rng* r, uint64_t n) { return orc_rng_next_u64(r) % n; }

/* rng.hpp:31-44: Box-Muller with a cached spare. */
double orc_rng_gaussian(orc_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = orc_rng_uniform(r);
  double u2 = orc_rng_uniform(r);
  while (u1 <= 0.0) u1 = orc_rng_uniform(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double theta = 6.283185307179586476925286766559 * u2;
  r->spare = rad * sin(theta);
  r->have_spare = 1;
  return rad * cos(theta);
}

/* rng.hpp:56-75 */
static uint64_t fnv1a64(const char* s) {
  uint64_t h = 1469598103934665603ull;
  for (; *s; ++s) {
    h ^= (uint8_t)*s;
    h *= 1099511628211ull;
  }
  return h;
}
static uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
uint64_t orc_derive_seed(uint64_t seed, const char* label) {
  return splitmix64(seed ^ fnv1a64(label));
}

/* tests/test_util.hpp:16-29 */
void orc_random_matrix(uint64_t n, uint32_t dim, uint64_t seed, double scale,
                       float* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (uint64_t i = 0; i < n * dim; ++i) {
    out[i] = (float)(scale * orc_rng_gaussian(&r));
  }
}

/* ======================================================================= */
/* Scoring: vectorstore.cpp:93-115, vectorstore.hpp:34-39                  */
/* ======================================================================= */
double orc_dot_d(const float* a, const float* b, uint32_t d) {
  double acc = 0.0;
  for (uint32_t i = 0; i < d; ++i) acc += (double)a[i] * (double)b[i];
  return acc;
}

double orc_l2_sq_d(const float* a, const float* b, uint32_t d) {
  double acc = 0.0;
  for (uint32_t i = 0; i < d; ++i) {
    const double t = (double)a[i] - (double)b[i];
    acc += t * t;
  }
  return acc;
}

float orc_score_rounded(int metric, const float* q, const float* row,
                        uint32_t d) {
  const double s = metric == ORC_IP ? orc_dot_d(q, row, d)
                                    : sqrt(orc_l2_sq_d(q, row, d));
  return (float)s;
}

int orc_ranks_before(int metric, float sa, uint64_t ia, float sb,
                     uint64_t ib) {
  if (sa != sb) return metric == ORC_IP ? sa > sb : sa < sb;
  return ia < ib;
}

/* ======================================================================= */
/* Coarse quantizer: ivf.cpp:269-299                                       */
/* ======================================================================= */
typedef struct {
  double s;
  uint32_t c;
} cscore;

static int g_desc; /* qsort has no context pointer; the oracle is not reentrant */
static int cmp_cscore(const void* pa, const void* pb) {
  const cscore* a = (const cscore*)pa;
  const cscore* b = (const cscore*)pb;
  if (a->s != b->s) {
    const int before = g_desc ? a->s > b->s : a->s < b->s;
    return before ? -1 : 1;
  }
  return a->c < b->c ? -1 : (a->c > b->c ? 1 : 0);
}

void orc_rank_clusters(const float* centroids, uint32_t nc, uint32_t d,
                       int metric, const float* q, uint32_t* order_out,
                       double* scores_out) {
  cscore* v = (cscore*)malloc(sizeof(cscore) * (nc ? nc : 1));
  for (uint32_t c = 0; c < nc; ++c) {
    const float* row = centroids + (uint64_t)c * d;
    v[c].s = metric == ORC_IP ? orc_dot_d(q, row, d) : orc_l2_sq_d(q, row, d);
    v[c].c = c;
    if (scores_out) scores_out[c] = v[c].s;
  }
  g_desc = metric == ORC_IP;
  qsort(v, nc, sizeof(cscore), cmp_cscore);
  for (uint32_t i = 0; i < nc; ++i) order_out[i] = v[i].c;
  free(v);
}

uint32_t orc_coarse_probe(const float* centroids, uint32_t nc, uint32_t d,
                          int metric, const float* q, int L, uint32_t* out) {
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (nc ? nc : 1));
  orc_rank_clusters(centroids, nc, d, metric, q, order, NULL);
  uint32_t keep = L < 0 ? 0u : (uint32_t)L;
  if (keep > nc) keep = nc;
  memcpy(out, order, sizeof(uint32_t) * keep);
  free(order);
  return keep;
}

/* ======================================================================= */
/* Fine scan: ivf.cpp:301-349, vectorstore.cpp:117-141                     */
/* ======================================================================= */
typedef struct {
  uint64_t id;
  float s;
} sid;

static int g_metric;
static int cmp_sid(const void* pa, const void* pb) {
  const sid* a = (const sid*)pa;
  const sid* b = (const sid*)pb;
  if (orc_ranks_before(g_metric, a->s, a->id, b->s, b->id)) return -1;
  if (orc_ranks_before(g_metric, b->s, b->id, a->s, a->id)) return 1;
  return 0;
}

static int finish_topk(sid* cand, uint64_t n, int metric, int k,
                       uint64_t* ids_out, float* scores_out) {
  g_metric = metric;
  qsort(cand, n, sizeof(sid), cmp_sid);
  const uint64_t keep = n < (uint64_t)k ? n : (uint64_t)k;
  for (uint64_t i = 0; i < keep; ++i) {
    ids_out[i] = cand[i].id;
    scores_out[i] = cand[i].s;
  }
  return (int)keep;
}

int orc_search_clusters(const float* vecs, const uint64_t* ids,
                        const uint64_t* list_off, uint32_t nc, uint32_t d,
                        int metric, const float* q, const uint32_t* clusters,
                        uint32_t ncl, int k, uint64_t* ids_out,
                        float* scores_out) {
  if (k < 1) return -1;
  uint64_t total = 0;
  for (uint32_t i = 0; i < ncl; ++i) {
    if (clusters[i] >= nc) return -2;
    total += list_off[clusters[i] + 1] - list_off[clusters[i]];
  }
  sid* cand = (sid*)malloc(sizeof(sid) * (total ? total : 1));
  uint64_t n = 0;
  for (uint32_t i = 0; i < ncl; ++i) {
    const uint32_t c = clusters[i];
    for (uint64_t r = list_off[c]; r < list_off[c + 1]; ++r) {
      cand[n].id = ids[r];
      cand[n].s = orc_score_rounded(metric, q, vecs + r * d, d);
      ++n;
    }
  }
  const int got = finish_topk(cand, n, metric, k, ids_out, scores_out);
  free(cand);
  return got;
}

int orc_ivf_search(const float* centroids, const float* vecs,
                   const uint64_t* ids, const uint64_t* list_off, uint32_t nc,
                   uint32_t d, int metric, const float* q, int L, int k,
                   uint64_t* ids_out, float* scores_out) {
  uint32_t* probe = (uint32_t*)malloc(sizeof(uint32_t) * (nc ? nc : 1));
  const uint32_t np = orc_coarse_probe(centroids, nc, d, metric, q, L, probe);
  const int got = orc_search_clusters(vecs, ids, list_off, nc, d, metric, q,
                                      probe, np, k, ids_out, scores_out);
  free(probe);
  return got;
}

int orc_exact_search(const float* db, const uint64_t* ids, uint64_t n,
                     uint32_t d, int metric, const float* q, int k,
                     uint64_t* ids_out, float* scores_out) {
  if (k < 1) return -1;
  sid* cand = (sid*)malloc(sizeof(sid) * (n ? n : 1));
  for (uint64_t i = 0; i < n; ++i) {
    cand[i].id = ids[i];
    cand[i].s = orc_score_rounded(metric, q, db + i * d, d);
  }
  const int got = finish_topk(cand, n, metric, k, ids_out, scores_out);
  free(cand);
  return got;
}

/* ======================================================================= */
/* Tiering: tiered.cpp:67-84, 200-211                                      */
/* ======================================================================= */
uint32_t orc_plan_prefetch(const uint32_t* order, uint32_t nc,
                           const uint64_t* cluster_bytes,
                           const uint8_t* resident, uint64_t budget,
                           uint32_t* plan_out, uint64_t* planned_bytes,
                           uint32_t* skipped_out, uint32_t* nskipped) {
  uint64_t remaining = budget;
  uint32_t np = 0, ns = 0;
  *planned_bytes = 0;
  for (uint32_t i = 0; i < nc; ++i) {
    const uint32_t c = order[i];
    if (resident[c]) continue;
    const uint64_t b = cluster_bytes[c];
    if (b <= remaining) {
      plan_out[np++] = c;
      *planned_bytes += b;
      remaining -= b;
    } else {
      skipped_out[ns++] = c;
    }
  }
  *nskipped = ns;
  return np;
}

double orc_coverage(const float* centroids, uint32_t nc, uint32_t d,
                    int metric, const float* q_in, const float* q_out, int L) {
  uint32_t* a = (uint32_t*)malloc(sizeof(uint32_t) * (nc ? nc : 1));
  uint32_t* b = (uint32_t*)malloc(sizeof(uint32_t) * (nc ? nc : 1));
  uint8_t* in_set = (uint8_t*)calloc(nc ? nc : 1, 1);
  const uint32_t na = orc_coarse_probe(centroids, nc, d, metric, q_in, L, a);
  const uint32_t nb = orc_coarse_probe(centroids, nc, d, metric, q_out, L, b);
  for (uint32_t i = 0; i < na; ++i) in_set[a[i]] = 1;
  uint32_t overlap = 0;
  for (uint32_t i = 0; i < nb; ++i) overlap += in_set[b[i]];
  free(a);
  free(b);
  free(in_set);
  return nb == 0 ? 0.0 : (double)overlap / (double)nb;
}

/* ======================================================================= */
/* Scheduling: sched.cpp:39-192                                            */
/* ======================================================================= */
typedef struct {
  double dist;
  uint64_t idx;
} didx;
static int cmp_didx(const void* pa, const void* pb) {
  const didx* a = (const didx*)pa;
  const didx* b = (const didx*)pb;
  if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx ? 1 : 0);
}

uint32_t orc_group_microbatches(const float* queries, uint64_t n, uint32_t d,
                                uint64_t m, uint64_t* order_out,
                                uint64_t* batch_off_out) {
  uint8_t* assigned = (uint8_t*)calloc(n ? n : 1, 1);
  didx* dists = (didx*)malloc(sizeof(didx) * (n ? n : 1));
  uint32_t nb = 0;
  uint64_t w = 0;
  batch_off_out[0] = 0;
  for (uint64_t seed = 0; seed < n; ++seed) {
    if (assigned[seed]) continue;
    order_out[w++] = seed;
    assigned[seed] = 1;
    uint64_t nd = 0;
    for (uint64_t j = seed + 1; j < n; ++j) {
      if (assigned[j]) continue;
      dists[nd].dist = orc_l2_sq_d(queries + seed * d, queries + j * d, d);
      dists[nd].idx = j;
      ++nd;
    }
    qsort(dists, nd, sizeof(didx), cmp_didx);
    const uint64_t take = (m - 1) < nd ? (m - 1) : nd;
    for (uint64_t t = 0; t < take; ++t) {
      order_out[w++] = dists[t].idx;
      assigned[dists[t].idx] = 1;
    }
    batch_off_out[++nb] = w;
  }
  free(assigned);
  free(dists);
  return nb;
}

static void batch_union(const uint64_t* batch_off, const uint64_t* members,
                        uint32_t b, const float* centroids, uint32_t nc,
                        uint32_t d, int metric, const float* queries, int L,
                        uint8_t* mark, uint32_t* probe) {
  memset(mark, 0, nc);
  for (uint64_t i = batch_off[b]; i < batch_off[b + 1]; ++i) {
    const uint32_t np = orc_coarse_probe(centroids, nc, d, metric,
                                         queries + members[i] * d, L, probe);
    for (uint32_t j = 0; j < np; ++j) mark[probe[j]] = 1;
  }
}

int orc_assign_cache_aware(const uint64_t* batch_off, const uint64_t* members,
                           uint32_t nb, const uint8_t* resident, uint32_t nw,
                           const float* centroids, uint32_t nc, uint32_t d,
                           int metric, const float* queries, int L,
                           uint32_t* assignment) {
  if (nw == 0) return -1;
  const uint64_t cap = ((uint64_t)nb + nw - 1) / nw;
  uint64_t* overlap = (uint64_t*)calloc((uint64_t)nb * nw + 1, sizeof(uint64_t));
  uint8_t* mark = (uint8_t*)malloc(nc ? nc : 1);
  uint32_t* probe = (uint32_t*)malloc(sizeof(uint32_t) * (nc ? nc : 1));
  for (uint32_t b = 0; b < nb; ++b) {
    batch_union(batch_off, members, b, centroids, nc, d, metric, queries, L,
                mark, probe);
    for (uint32_t w = 0; w < nw; ++w) {
      uint64_t s = 0;
      for (uint32_t c = 0; c < nc; ++c) s += mark[c] && resident[(uint64_t)w * nc + c];
      overlap[(uint64_t)b * nw + w] = s;
    }
  }
  uint8_t* placed = (uint8_t*)calloc(nb ? nb : 1, 1);
  uint64_t* load = (uint64_t*)calloc(nw, sizeof(uint64_t));
  for (uint32_t step = 0; step < nb; ++step) {
    uint32_t bb = nb, bw = nw;
    uint64_t best = 0;
    int found = 0;
    for (uint32_t b = 0; b < nb; ++b) {
      if (placed[b]) continue;
      for (uint32_t w = 0; w < nw; ++w) {
        if (load[w] >= cap) continue;
        const uint64_t o = overlap[(uint64_t)b * nw + w];
        const int better =
            !found || o > best ||
            (o == best &&
             (b < bb || (b == bb && (load[w] < load[bw] ||
                                     (load[w] == load[bw] && w < bw)))));
        if (better) {
          found = 1;
          bb = b;
          bw = w;
          best = o;
        }
      }
    }
    assignment[bb] = bw;
    placed[bb] = 1;
    load[bw]++;
  }
  free(overlap);
  free(mark);
  free(probe);
  free(placed);
  free(load);
  return 0;
}

uint64_t orc_assignment_overlap(const uint64_t* batch_off,
                                const uint64_t* members, uint32_t nb,
                                const uint8_t* resident, uint32_t nw,
                                const uint32_t* assignment,
                                const float* centroids, uint32_t nc,
                                uint32_t d, int metric, const float* queries,
                                int L) {
  (void)nw;
  uint8_t* mark = (uint8_t*)malloc(nc ? nc : 1);
  uint32_t* probe = (uint32_t*)malloc(sizeof(uint32_t) * (nc ? nc : 1));
  uint64_t total = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    batch_union(batch_off, members, b, centroids, nc, d, metric, queries, L,
                mark, probe);
    const uint8_t* res = resident + (uint64_t)assignment[b] * nc;
    for (uint32_t c = 0; c < nc; ++c) total += mark[c] && res[c];
  }
  free(mark);
  free(probe);
  return total;
}

int orc_split_budget(uint64_t total, const uint64_t* batch, uint64_t n,
                     uint64_t* out) {
  if (n == 0) return -1;
  const uint64_t base = total / n;
  uint64_t rem = total % n;
  for (uint64_t i = 0; i < n; ++i) out[i] = base;
  /* Remainder to the lowest query ids (stable on equal ids, as std::sort of
   * positions by id would place them; ids in a batch are distinct). */
  uint8_t* got = (uint8_t*)calloc(n, 1);
  while (rem > 0) {
    uint64_t best = n;
    for (uint64_t i = 0; i < n; ++i) {
      if (got[i]) continue;
      if (best == n || batch[i] < batch[best]) best = i;
    }
    got[best] = 1;
    out[best] += 1;
    --rem;
  }
  free(got);
  return 0;
}

/* ======================================================================= */
/* Hotness law: cache.cpp:31-38                                            */
/* ======================================================================= */
void orc_hotness_end_of_round(float* h, const uint8_t* used, uint32_t n,
                              float decay, float h_inc) {
  for (uint32_t i = 0; i < n; ++i) {
    float v = h[i] / decay;
    if (used[i]) v = v + h_inc;
    h[i] = v;
  }
}
