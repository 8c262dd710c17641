// ref_pipe_shim.cpp — extern "C" wrapper around the UNMODIFIED reference's
// trace + pipeline code (proj/core/src/trace.cpp, pipeline.cpp), compiled by
// oracle/Makefile into oracle/_ref/libref_pipe.so when the reference tree and
// an nlohmann/json header are present (json.hpp is not vendored by the
// reference; the image carries a copy under cudnn_frontend).
//
// TEST INFRASTRUCTURE ONLY: tests/golden/make_golden.py uses it to record
// synthesized traces and run_batch records (simulated clock) that the
// product's pipeline.py must reproduce. Never linked into the product.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "laiv/ivf.hpp"
#include "laiv/pipeline.hpp"
#include "laiv/trace.hpp"
#include "laiv/vectorstore.hpp"

namespace {
thread_local std::string g_err;

struct Built {
  laiv::IvfIndex ix;
  laiv::EmbeddingMatrix db;
};

// list-major store -> IvfIndex + EmbeddingMatrix (rows appended in list
// order, as load_index does, ivf.cpp:437-455)
Built build(const float* centroids, uint32_t nc, uint32_t d, int metric, const float* vecs,
            const uint64_t* ids, const uint64_t* list_off) {
  laiv::EmbeddingMatrix cen(d);
  for (uint32_t c = 0; c < nc; ++c) {
    cen.append(c, std::span<const float>(centroids + uint64_t(c) * d, d));
  }
  laiv::EmbeddingMatrix db(d);
  std::vector<std::vector<uint64_t>> lists(nc);
  for (uint32_t c = 0; c < nc; ++c) {
    for (uint64_t r = list_off[c]; r < list_off[c + 1]; ++r) {
      lists[c].push_back(ids[r]);
      db.append(ids[r], std::span<const float>(vecs + r * d, d));
    }
  }
  return Built{laiv::IvfIndex(std::move(cen), std::move(lists), static_cast<laiv::Metric>(metric)),
               std::move(db)};
}
} // namespace

extern "C" {

const char* refp_last_error() { return g_err.c_str(); }

// synthesize_traces (trace.hpp) -> traces JSONL at traces_path and the
// sidecar rows in sidecar_out (capacity cap rows); *count = sidecar rows.
int refp_synth_traces(const float* centroids, uint32_t nc, uint32_t d, int metric,
                      const float* vecs, const uint64_t* ids, const uint64_t* list_off,
                      uint64_t n, const char* pipeline, uint64_t seed, double sigma,
                      double dur_mean, double dur_sigma, const char* traces_path,
                      float* sidecar_out, uint64_t cap, uint64_t* count) {
  try {
    const Built b = build(centroids, nc, d, metric, vecs, ids, list_off);
    laiv::SynthOptions o;
    o.noise_sigma = sigma;
    o.duration_mean_s = dur_mean;
    o.duration_sigma = dur_sigma;
    const laiv::TraceSet ts =
        laiv::synthesize_traces(b.db, b.ix, n, laiv::pipeline_from_name(pipeline), seed, o);
    laiv::save_traces(traces_path, ts.traces);
    *count = ts.sidecar.count();
    if (*count > cap) return -2;
    std::memcpy(sidecar_out, ts.sidecar.data().data(), *count * d * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// run_batch (pipeline.hpp) over a traces file, a sidecar and a config file
// (load_config format); the record goes to records_path (save_records).
int refp_run_batch(const float* centroids, uint32_t nc, uint32_t d, int metric,
                   const float* vecs, const uint64_t* ids, const uint64_t* list_off,
                   const char* traces_path, const float* sidecar, uint64_t ns,
                   const char* cfg_path, const char* records_path) {
  try {
    const Built b = build(centroids, nc, d, metric, vecs, ids, list_off);
    laiv::EmbeddingMatrix side(d);
    for (uint64_t i = 0; i < ns; ++i) side.append(i, std::span<const float>(sidecar + i * d, d));
    const auto traces = laiv::load_traces(traces_path);
    const laiv::RunConfig cfg = laiv::load_config(cfg_path);
    const laiv::RunRecord rec = laiv::run_batch(traces, side, b.ix, b.db, cfg);
    laiv::save_records(records_path, rec);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

} // extern "C"
