// laix.cpp — LAIX index files (the reference's on-disk format, ivf.cpp:351-458)
// read straight into the list-major host store the devices copy from, and
// written back from it; plus the store validation shared with
// laivg_index_create (EmbeddingMatrix::append rules, vectorstore.cpp:66-85).
//
// File layout (little-endian, packed): "LAIX", u32 version = 1, u32 dim,
// u32 nc, u8 metric, centroids f32[nc][dim], then per list c: u64 len,
// u64 ids[len], f32 rows[len][dim]. A list's rows are contiguous in the file
// and in the store, so loading is one pread per (list, chunk) into the final
// location, spread over threads; no row is copied twice.
//
// Error behaviour follows load_index exactly: the reference reads the file
// front to back and validates each row as it appends it, so the error
// reported is the FIRST in file order among truncation, a non-finite
// component, or a repeated id (same exception class and message).
#include "host.hpp"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cerrno>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace laivg {

namespace {

constexpr char kMagic[4] = {'L', 'A', 'I', 'X'};
constexpr uint32_t kVersion = 1;
constexpr uint64_t kHeader = 17;        // magic + version + dim + nc + metric
constexpr uint64_t kChunk = 16ull << 20; // bytes per read/write task

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

// false on EOF before n bytes
bool pread_all(int fd, void* dst, uint64_t n, uint64_t pos) {
  auto* p = static_cast<char*>(dst);
  while (n) {
    const ssize_t r = ::pread(fd, p, std::min<uint64_t>(n, 1ull << 30), static_cast<off_t>(pos));
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) return false;
    p += r;
    pos += static_cast<uint64_t>(r);
    n -= static_cast<uint64_t>(r);
  }
  return true;
}

bool pwrite_all(int fd, const void* src, uint64_t n, uint64_t pos) {
  auto* p = static_cast<const char*>(src);
  while (n) {
    const ssize_t r = ::pwrite(fd, p, std::min<uint64_t>(n, 1ull << 30), static_cast<off_t>(pos));
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) return false;
    p += r;
    pos += static_cast<uint64_t>(r);
    n -= static_cast<uint64_t>(r);
  }
  return true;
}

unsigned pick_threads(unsigned want) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  return want ? std::min(want, 4 * hw) : hw;
}

inline bool finite_row(const float* r, uint32_t d) {
  uint32_t bad = 0;
  for (uint32_t j = 0; j < d; ++j) {
    uint32_t b;
    std::memcpy(&b, r + j, 4);
    bad |= static_cast<uint32_t>((b & 0x7f800000u) == 0x7f800000u);
  }
  return !bad;
}

inline uint64_t mix(uint64_t x) { // splitmix64 finaliser
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

} // namespace

// First invalid row (list-major order) of rows [0, n): a non-finite
// component, or an id already seen in an earlier row. Returns n when every
// row is valid; *dup tells which rule the row broke (non-finite wins on a
// row that breaks both, as append checks it first).
uint64_t first_invalid_row(const float* vecs, const uint64_t* ids, uint64_t n, uint32_t d,
                           unsigned threads, bool* dup) {
  *dup = false;
  if (n == 0) return 0;
  const unsigned T = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>(pick_threads(threads), n / 4096 + 1)));
  ThreadPool pool(T - 1);
  // non-finite: the first bad row per chunk, then the minimum
  const uint64_t per = (n + T - 1) / T;
  std::vector<uint64_t> bad_nf(T, n);
  pool.parallel_for(T, [&](size_t t, unsigned) {
    const uint64_t r0 = t * per, r1 = std::min(n, r0 + per);
    for (uint64_t r = r0; r < r1; ++r) {
      if (!finite_row(vecs + r * d, d)) {
        bad_nf[t] = r;
        return;
      }
    }
  });
  const uint64_t nf = *std::min_element(bad_nf.begin(), bad_nf.end());
  // repeated ids: hash-partition (id, row) into buckets, sort each bucket;
  // the offending row of an id is its second occurrence
  const unsigned bits = 10;
  const uint32_t B = 1u << bits;
  std::vector<uint64_t> cnt(size_t(T) * B, 0);
  pool.parallel_for(T, [&](size_t t, unsigned) {
    uint64_t* c = cnt.data() + t * B;
    const uint64_t r0 = t * per, r1 = std::min(n, r0 + per);
    for (uint64_t r = r0; r < r1; ++r) ++c[mix(ids[r]) >> (64 - bits)];
  });
  std::vector<uint64_t> start(size_t(T) * B + 1, 0);
  {
    uint64_t s = 0;
    for (uint32_t b = 0; b < B; ++b) {
      for (unsigned t = 0; t < T; ++t) {
        start[size_t(t) * B + b] = s;
        s += cnt[size_t(t) * B + b];
      }
    }
  }
  std::vector<uint64_t> bstart(B + 1);
  for (uint32_t b = 0; b < B; ++b) bstart[b] = start[b]; // thread 0's slot opens the bucket
  bstart[B] = n;
  struct Pair {
    uint64_t id, row;
  };
  std::vector<Pair> pairs(n);
  pool.parallel_for(T, [&](size_t t, unsigned) {
    std::vector<uint64_t> w(start.begin() + t * B, start.begin() + (t + 1) * B);
    const uint64_t r0 = t * per, r1 = std::min(n, r0 + per);
    for (uint64_t r = r0; r < r1; ++r) pairs[w[mix(ids[r]) >> (64 - bits)]++] = Pair{ids[r], r};
  });
  std::vector<uint64_t> bad_dup(B, n);
  pool.parallel_for(B, [&](size_t b, unsigned) {
    Pair* p0 = pairs.data() + bstart[b];
    Pair* p1 = pairs.data() + bstart[b + 1];
    std::sort(p0, p1, [](const Pair& a, const Pair& c) {
      return a.id != c.id ? a.id < c.id : a.row < c.row;
    });
    uint64_t best = n;
    for (Pair* p = p0 + 1; p < p1; ++p) {
      if (p->id == (p - 1)->id && (p - 1 == p0 || (p - 2)->id != p->id)) {
        best = std::min(best, p->row); // the second occurrence
      }
    }
    bad_dup[b] = best;
  });
  const uint64_t dp = *std::min_element(bad_dup.begin(), bad_dup.end());
  if (nf <= dp) return nf;
  *dup = true;
  return dp;
}

void validate_store(const Index& ix, unsigned threads) {
  const uint32_t d = ix.d;
  for (uint32_t c = 0; c < ix.nc; ++c) { // centroids are rows with ids 0..nc-1
    if (!finite_row(ix.centroids.data() + size_t(c) * d, d)) {
      throw std::invalid_argument("non-finite component in row for id " + std::to_string(c));
    }
  }
  bool dup = false;
  const uint64_t n = ix.total();
  const uint64_t r = first_invalid_row(ix.vecs, ix.ids, n, d, threads, &dup);
  if (r < n) {
    throw std::invalid_argument((dup ? "duplicate id " : "non-finite component in row for id ") +
                                std::to_string(ix.ids[r]));
  }
}

// load_index (ivf.cpp:394-458) into `ix`: centroids + list_off filled, rows
// and ids read into one block from alloc(bytes) (the caller pins it).
void laix_load(const std::string& path, unsigned threads, Index& ix,
               void* (*alloc)(uint64_t bytes, void* user), void* user) {
  const auto t_start = std::chrono::steady_clock::now();
  Fd f;
  f.fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) throw std::runtime_error("cannot open: " + path);
  struct stat st {};
  if (::fstat(f.fd, &st) != 0) throw std::runtime_error("cannot open: " + path);
  const uint64_t size = static_cast<uint64_t>(st.st_size);
  unsigned char hdr[kHeader];
  const uint64_t have = std::min<uint64_t>(size, kHeader);
  if (have && !pread_all(f.fd, hdr, have, 0)) throw std::runtime_error("cannot open: " + path);
  if (have < 4 || std::memcmp(hdr, kMagic, 4) != 0) {
    throw std::runtime_error(path + ": bad magic, not a LAIX file");
  }
  auto field = [&](uint64_t at, uint64_t bytes, const char* what) {
    if (have < at + bytes) throw std::runtime_error(path + ": truncated while reading " + what);
    uint32_t v = 0;
    std::memcpy(&v, hdr + at, bytes);
    return v;
  };
  const uint32_t version = field(4, 4, "version");
  if (version != kVersion) {
    throw std::runtime_error(path + ": unsupported version " + std::to_string(version));
  }
  const uint32_t d = field(8, 4, "dim");
  const uint32_t nc = field(12, 4, "cluster count");
  const uint32_t metric = field(16, 1, "metric");
  if (metric > 1) throw std::runtime_error(path + ": bad metric byte");
  if (d == 0) throw std::runtime_error(path + ": header declares dim 0");
  const uint64_t row = uint64_t(d) * 4;

  // centroid block, validated row by row up to any truncation
  const uint64_t cen_avail = (size - kHeader) / row;
  const uint64_t cen_rows = std::min<uint64_t>(nc, cen_avail);
  ix.d = d;
  ix.nc = nc;
  ix.metric = static_cast<int>(metric);
  ix.centroids.resize(cen_rows * d);
  if (cen_rows && !pread_all(f.fd, ix.centroids.data(), cen_rows * row, kHeader)) {
    throw std::runtime_error(path + ": truncated centroid block");
  }
  for (uint64_t c = 0; c < cen_rows; ++c) {
    if (!finite_row(ix.centroids.data() + c * d, d)) {
      throw std::invalid_argument("non-finite component in row for id " + std::to_string(c));
    }
  }
  if (cen_rows < nc) throw std::runtime_error(path + ": truncated centroid block");

  // walk the list headers: offsets of every list, and where (if anywhere)
  // the file ends early
  std::vector<uint64_t> off(1, 0), pos; // pos[c] = file offset of list c's ids
  off.reserve(size_t(nc) + 1);
  pos.reserve(nc);
  uint64_t p = kHeader + uint64_t(nc) * row;
  std::string trunc;          // message of the truncation error, if any
  uint64_t partial_rows = 0;  // rows of the truncated list present in the file
  uint64_t trunc_len = 0;     // its declared length (its ids are all present)
  for (uint32_t c = 0; c < nc; ++c) {
    uint64_t len = 0;
    if (size < p + 8 || !pread_all(f.fd, &len, 8, p)) {
      trunc = path + ": truncated while reading cluster length";
      break;
    }
    p += 8;
    // the reference sizes the id vector first: a length past its max_size
    // is std::length_error (a logic_error). Shorter impossible lengths are
    // reported as truncation without attempting the allocation.
    if (len > uint64_t(std::numeric_limits<std::ptrdiff_t>::max()) / 8) {
      throw std::length_error("vector::_M_default_append");
    }
    if (len > (size - p) / 8) {
      trunc = path + ": truncated while reading member id";
      break;
    }
    pos.push_back(p);
    p += len * 8;
    const uint64_t rows = (size - p) / row;
    if (rows < len) {
      trunc = path + ": truncated cluster " + std::to_string(c);
      partial_rows = rows;
      trunc_len = len;
      break;
    }
    p += len * row;
    off.push_back(off.back() + len);
  }
  const uint32_t full = static_cast<uint32_t>(off.size() - 1); // complete lists
  const uint64_t n = off.back() + partial_rows;                 // rows to validate
  const size_t vb = size_t(n) * row, ib = size_t(n) * 8;
  const size_t idoff = (vb + 63) & ~size_t(63);
  char* blk = static_cast<char*>(alloc(idoff + ib + 64, user));
  auto* vecs = reinterpret_cast<float*>(blk);
  auto* ids = reinterpret_cast<uint64_t*>(blk + idoff);
  ix.owned_block = blk;
  ix.vecs = vecs;
  ix.ids = ids;

  // read tasks: (list, byte range) pieces of <= kChunk, ids with the first
  struct Task {
    uint32_t c;
    uint64_t r0, r1; // rows of list c
  };
  std::vector<Task> tasks;
  const uint64_t rows_per = std::max<uint64_t>(1, kChunk / row);
  const uint32_t lists = full + (partial_rows ? 1 : 0);
  for (uint32_t c = 0; c < lists; ++c) {
    const uint64_t len = c < full ? off[c + 1] - off[c] : partial_rows;
    if (len == 0) {
      tasks.push_back(Task{c, 0, 0});
      continue;
    }
    for (uint64_t r = 0; r < len; r += rows_per) tasks.push_back(Task{c, r, std::min(len, r + rows_per)});
  }
  const unsigned T = static_cast<unsigned>(
      std::max<size_t>(1, std::min<size_t>(pick_threads(threads), tasks.size())));
  ThreadPool pool(T - 1);
  std::vector<char> ok(tasks.size(), 1);
  pool.parallel_for(tasks.size(), [&](size_t i, unsigned) {
    const Task& t = tasks[i];
    const uint64_t base = off[t.c];
    // rows present / declared length (they differ only for a truncated list)
    const uint64_t len = t.c < full ? off[t.c + 1] - off[t.c] : partial_rows;
    const uint64_t decl = t.c < full ? len : trunc_len;
    bool good = true;
    if (t.r0 == 0 && len) good = pread_all(f.fd, ids + base, len * 8, pos[t.c]);
    if (good && t.r1 > t.r0) {
      good = pread_all(f.fd, vecs + (base + t.r0) * d, (t.r1 - t.r0) * row,
                       pos[t.c] + decl * 8 + t.r0 * row);
    }
    ok[i] = good;
  });
  if (std::find(ok.begin(), ok.end(), 0) != ok.end()) {
    throw std::runtime_error(path + ": read failed");
  }
  const auto t_read = std::chrono::steady_clock::now();
  bool dup = false;
  const uint64_t bad = first_invalid_row(vecs, ids, n, d, threads, &dup);
  if (std::getenv("LAIVG_TRACE")) {
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[laivg] laix_load: read %.3f s (%u threads), validate %.3f s\n",
                 std::chrono::duration<double>(t_read - t_start).count(), T,
                 std::chrono::duration<double>(now - t_read).count());
  }
  if (bad < n) {
    throw std::invalid_argument((dup ? "duplicate id " : "non-finite component in row for id ") +
                                std::to_string(ids[bad]));
  }
  if (!trunc.empty()) throw std::runtime_error(trunc);
  ix.list_off = std::move(off);
}

// save_index (ivf.cpp:351-392) from the list-major store: same bytes.
void laix_save(const std::string& path, const Index& ix, unsigned threads) {
  Fd f;
  f.fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (f.fd < 0) throw std::runtime_error("cannot open for writing: " + path);
  const uint32_t d = ix.d, nc = ix.nc;
  const uint64_t row = uint64_t(d) * 4;
  unsigned char hdr[kHeader];
  std::memcpy(hdr, kMagic, 4);
  std::memcpy(hdr + 4, &kVersion, 4);
  std::memcpy(hdr + 8, &d, 4);
  std::memcpy(hdr + 12, &nc, 4);
  hdr[16] = static_cast<unsigned char>(ix.metric);
  bool good = pwrite_all(f.fd, hdr, kHeader, 0) &&
              (nc == 0 || pwrite_all(f.fd, ix.centroids.data(), uint64_t(nc) * row, kHeader));
  std::vector<uint64_t> pos(size_t(nc) + 1);
  pos[0] = kHeader + uint64_t(nc) * row;
  for (uint32_t c = 0; c < nc; ++c) pos[c + 1] = pos[c] + 8 + ix.list_len(c) * (8 + row);
  struct Task {
    uint32_t c;
    uint64_t r0, r1;
  };
  std::vector<Task> tasks;
  const uint64_t rows_per = std::max<uint64_t>(1, kChunk / row);
  for (uint32_t c = 0; c < nc; ++c) {
    const uint64_t len = ix.list_len(c);
    tasks.push_back(Task{c, 0, std::min(len, rows_per)});
    for (uint64_t r = rows_per; r < len; r += rows_per) {
      tasks.push_back(Task{c, r, std::min(len, r + rows_per)});
    }
  }
  const unsigned T = static_cast<unsigned>(
      std::max<size_t>(1, std::min<size_t>(pick_threads(threads), tasks.size())));
  ThreadPool pool(T - 1);
  std::vector<char> ok(tasks.size(), 1);
  pool.parallel_for(tasks.size(), [&](size_t i, unsigned) {
    const Task& t = tasks[i];
    const uint64_t base = ix.list_off[t.c], len = ix.list_len(t.c);
    bool w = true;
    if (t.r0 == 0) {
      w = pwrite_all(f.fd, &len, 8, pos[t.c]) &&
          (len == 0 || pwrite_all(f.fd, ix.ids + base, len * 8, pos[t.c] + 8));
    }
    if (w && t.r1 > t.r0) {
      w = pwrite_all(f.fd, ix.vecs + (base + t.r0) * d, (t.r1 - t.r0) * row,
                     pos[t.c] + 8 + len * 8 + t.r0 * row);
    }
    ok[i] = w;
  });
  good = good && std::find(ok.begin(), ok.end(), 0) == ok.end();
  if (!good || ::close(f.fd) != 0) {
    f.fd = -1;
    throw std::runtime_error("write failed: " + path);
  }
  f.fd = -1;
}

} // namespace laivg
