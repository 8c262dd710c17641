// synth.hpp — synthetic workload generator (synth.cpp).
#pragma once
#include <cstdint>

namespace laivg {

// Synthetic workload: counter-based, bit-identical for any
// thread count.
void synth_centroids(uint64_t seed, uint32_t nc, uint32_t d, float* out);
void synth_lists(uint64_t seed, const float* centroids, uint32_t d,
                 uint64_t per_list, float spread, uint32_t c_begin,
                 uint32_t c_end, float* vecs, uint64_t* ids, int threads);
void synth_queries(uint64_t seed, const float* vecs, uint64_t n_rows,
                   uint32_t d, uint32_t nq, float sigma, float* q_in,
                   float* q_out, uint64_t* rows);

// Topical queries (SURVEY §8d, C3-C5 skew): topic t ~ Zipf(zipf_s) over
// n_topics random centre lists; the query's source row comes from one of the
// `neigh` lists nearest the topic centre, then q_in / q_out as synth_queries.
void synth_queries_topical(uint64_t seed, const float* centroids, uint32_t nc,
                           const float* vecs, const uint64_t* list_off, uint32_t d,
                           uint32_t n_topics, double zipf_s, uint32_t neigh, uint32_t nq,
                           float sigma, float* q_in, float* q_out, uint64_t* rows,
                           uint32_t* topic);

} // namespace laivg
