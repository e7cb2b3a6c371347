// TEST INFRASTRUCTURE — not product code.
//
// A thin C ABI over the *unmodified* reference library (`geojoin`, compiled
// from /root/reference/proj/src by oracle/build_ref.py into
// oracle/_ref/libgeojoin_ref.so).  It exists so that Python (tests, the
// fixture generator, bench.py's `--impl reference` arm and the offline index
// build) can call the reference's own functions:
//
//   build_index / IndexBundle::save / load      proj/src/join.cpp:152-235,316-381
//   cell_from_point                             proj/src/cell_id.cpp:82-95
//   Act::probe / probe_batch / detail kernels   proj/src/act.cpp:248-270,310-315
//   pip_test / validate_polygon                 proj/src/geometry.cpp:184-204
//   join_exact / join_approx                    proj/src/join.cpp:237-247
//   join_count_per_polygon                      proj/src/join.cpp:255-285
//   accumulate_probe_stats                      proj/src/join.cpp:287-290
//
// Nothing here re-implements reference logic; every entry point forwards to
// the reference and flattens the result into plain arrays.  Exceptions are
// translated to negative status codes + a thread-local message.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "geojoin/act.hpp"
#include "geojoin/cell_id.hpp"
#include "geojoin/geometry.hpp"
#include "geojoin/io.hpp"
#include "geojoin/join.hpp"
#include "geojoin/latlng.hpp"

using namespace geojoin;

namespace {

thread_local std::string g_err;

enum : int {
  kOk = 0,
  kInvalidArgument = -1,  // std::invalid_argument (bad coordinate, level, ...)
  kBuildError = -2,
  kCorruption = -3,
  kOther = -4,
};

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return kOk;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return kInvalidArgument;
  } catch (const BuildError& e) {
    g_err = e.what();
    return kBuildError;
  } catch (const CorruptionError& e) {
    g_err = e.what();
    return kCorruption;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kOther;
  }
}

std::span<const LatLng> as_points(const double* latlng, uint64_t n) {
  static_assert(sizeof(LatLng) == 16, "LatLng must be two packed doubles");
  return {reinterpret_cast<const LatLng*>(latlng), static_cast<size_t>(n)};
}

std::vector<Polygon> make_polygons(const uint32_t* ids, const uint64_t* vtx_off,
                                   const double* latlng, uint64_t n_poly) {
  std::vector<Polygon> polys(n_poly);
  for (uint64_t p = 0; p < n_poly; ++p) {
    polys[p].id = ids[p];
    const uint64_t b = vtx_off[p], e = vtx_off[p + 1];
    polys[p].vertices.resize(e - b);
    for (uint64_t v = b; v < e; ++v) {
      polys[p].vertices[v - b] = LatLng{latlng[2 * v], latlng[2 * v + 1]};
    }
  }
  return polys;
}

}  // namespace

extern "C" {

struct RefBuildConfig {
  int32_t mode_approx;  // JoinConfig::mode
  int32_t k_max;        // ActConfig::k_max
  double precision_m;
  uint64_t memory_budget_bytes;
  int32_t max_covering_cells;
  int32_t max_covering_level;
  int32_t max_interior_cells;
  int32_t max_interior_level;
  uint64_t training_point_limit;
};

struct RefBundleInfo {
  int32_t mode_approx;  // BuildReport::mode
  int32_t precision_achieved;
  double precision_m;
  double achieved_precision_m;
  uint64_t memory_bytes;
  int32_t covering_shrink_steps;
  int32_t k_max;
  uint64_t node_count;
  uint64_t lut_len;
  uint64_t n_polygons;
  uint64_t total_vertices;
  uint64_t train_points_consumed;
  uint64_t train_cells_split;
  double train_expensive_before;
  double train_expensive_after;
};

const char* ref_last_error() { return g_err.c_str(); }

void ref_default_config(RefBuildConfig* c) {
  const JoinConfig d;
  c->mode_approx = d.mode == JoinMode::kApprox;
  c->k_max = d.act.k_max;
  c->precision_m = d.precision_m;
  c->memory_budget_bytes = d.memory_budget_bytes;
  c->max_covering_cells = d.covering.max_covering_cells;
  c->max_covering_level = d.covering.max_covering_level;
  c->max_interior_cells = d.covering.max_interior_cells;
  c->max_interior_level = d.covering.max_interior_level;
  c->training_point_limit = d.training_point_limit;
}

void* ref_build_index(const uint32_t* ids, const uint64_t* vtx_off,
                      const double* latlng, uint64_t n_poly,
                      const RefBuildConfig* c, const double* train_latlng,
                      uint64_t n_train, int* status) {
  IndexBundle* out = nullptr;
  *status = guarded([&] {
    JoinConfig cfg;
    cfg.mode = c->mode_approx ? JoinMode::kApprox : JoinMode::kExact;
    cfg.precision_m = c->precision_m;
    cfg.memory_budget_bytes = c->memory_budget_bytes;
    cfg.covering.max_covering_cells = c->max_covering_cells;
    cfg.covering.max_covering_level = c->max_covering_level;
    cfg.covering.max_interior_cells = c->max_interior_cells;
    cfg.covering.max_interior_level = c->max_interior_level;
    cfg.training_point_limit = c->training_point_limit;
    cfg.act.k_max = c->k_max;
    out = new IndexBundle(build_index(make_polygons(ids, vtx_off, latlng, n_poly),
                                      cfg, as_points(train_latlng, n_train)));
  });
  return out;
}

void* ref_bundle_load(const char* path, int* status) {
  IndexBundle* out = nullptr;
  *status = guarded([&] {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw std::runtime_error(std::string("cannot open ") + path);
    out = new IndexBundle(IndexBundle::load(is));
  });
  return out;
}

int ref_bundle_save(const void* h, const char* path) {
  return guarded([&] {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw std::runtime_error(std::string("cannot open ") + path);
    static_cast<const IndexBundle*>(h)->save(os);
  });
}

void ref_bundle_free(void* h) { delete static_cast<IndexBundle*>(h); }

void ref_bundle_info(const void* h, RefBundleInfo* o) {
  const IndexBundle& b = *static_cast<const IndexBundle*>(h);
  o->mode_approx = b.report().mode == JoinMode::kApprox;
  o->precision_achieved = b.report().precision_achieved;
  o->precision_m = b.config().precision_m;
  o->achieved_precision_m = b.report().achieved_precision_m;
  o->memory_bytes = b.report().memory_bytes;
  o->covering_shrink_steps = b.report().covering_shrink_steps;
  o->k_max = b.act().config().k_max;
  o->node_count = b.act().node_count();
  o->lut_len = b.act().lookup_table().size();
  o->n_polygons = b.polygons().size();
  uint64_t tv = 0;
  for (const Polygon& p : b.polygons()) tv += p.vertices.size();
  o->total_vertices = tv;
  o->train_points_consumed = b.report().training.points_consumed;
  o->train_cells_split = b.report().training.cells_split;
  o->train_expensive_before = b.report().training.expensive_fraction_before;
  o->train_expensive_after = b.report().training.expensive_fraction_after;
}

// Borrowed pointers into the bundle (valid until ref_bundle_free): exactly
// the fields of ActProbeView (act.hpp:108-116) + lookup_table().
void ref_bundle_view(const void* h, const uint64_t** arena,
                     const uint32_t** lut, uint64_t roots[8],
                     uint64_t prefixes[8], uint64_t prefix_bits[8]) {
  const IndexBundle& b = *static_cast<const IndexBundle*>(h);
  const ActProbeView& v = b.act().view();
  *arena = v.arena;
  *lut = b.act().lookup_table().data();
  for (int f = 0; f < 8; ++f) {
    roots[f] = v.roots[f];
    prefixes[f] = v.prefixes[f];
    prefix_bits[f] = v.prefix_bits[f];
  }
}

// Polygons flattened to CSR, in bundle order.
void ref_bundle_polygons(const void* h, uint32_t* ids, uint64_t* vtx_off,
                         double* latlng) {
  const IndexBundle& b = *static_cast<const IndexBundle*>(h);
  uint64_t off = 0;
  size_t p = 0;
  for (const Polygon& poly : b.polygons()) {
    ids[p] = poly.id;
    vtx_off[p] = off;
    for (const LatLng& v : poly.vertices) {
      latlng[2 * off] = v.lat;
      latlng[2 * off + 1] = v.lng;
      ++off;
    }
    ++p;
  }
  vtx_off[p] = off;
}

int ref_validate_polygon(uint32_t id, const double* latlng, uint64_t n_vtx) {
  return guarded([&] {
    Polygon poly;
    poly.id = id;
    poly.vertices.assign(as_points(latlng, n_vtx).begin(),
                         as_points(latlng, n_vtx).end());
    validate_polygon(poly);
  });
}

// cell_from_point over an array; on a bad point returns kInvalidArgument and
// stores the first offending index in *bad_index.
int ref_cell_from_point(const double* latlng, uint64_t n, int level,
                        uint64_t* out_raw, uint64_t* bad_index) {
  uint64_t i = 0;
  const int rc = guarded([&] {
    const auto pts = as_points(latlng, n);
    for (; i < n; ++i) out_raw[i] = cell_from_point(pts[i], level).raw;
  });
  if (rc != kOk && bad_index) *bad_index = i;
  return rc;
}

int ref_cell_from_point_levels(const double* latlng, const int32_t* levels,
                               uint64_t n, uint64_t* out_raw) {
  return guarded([&] {
    const auto pts = as_points(latlng, n);
    for (uint64_t i = 0; i < n; ++i) {
      out_raw[i] = cell_from_point(pts[i], levels[i]).raw;
    }
  });
}

// Act::probe(cell_from_point(p, k_max/2)) per point.
int ref_probe_points(const void* h, const double* latlng, uint64_t n,
                     uint64_t* out_entries) {
  return guarded([&] {
    const Act& act = static_cast<const IndexBundle*>(h)->act();
    const auto pts = as_points(latlng, n);
    const int level = act.max_indexed_level();
    for (uint64_t i = 0; i < n; ++i) {
      out_entries[i] = act.probe(cell_from_point(pts[i], level));
    }
  });
}

int ref_probe_raw(const void* h, const uint64_t* raw, uint64_t n,
                  uint64_t* out_entries, int32_t* out_node_accesses) {
  return guarded([&] {
    const Act& act = static_cast<const IndexBundle*>(h)->act();
    for (uint64_t i = 0; i < n; ++i) {
      int acc = 0;
      out_entries[i] = act.probe_counting(CellId{raw[i]}, acc);
      if (out_node_accesses) out_node_accesses[i] = acc;
    }
  });
}

// kernel: 0 = Act::probe_batch (runtime dispatch), 1 = detail scalar kernel,
// 2 = detail AVX2 kernel.  n must be a multiple of 8.
int ref_probe_batch(const void* h, const uint64_t* raw, uint64_t n,
                    uint64_t* out_entries, int kernel) {
  return guarded([&] {
    if (n % ActConfig::kBatchWidth != 0) {
      throw std::invalid_argument("batch probes need a multiple of 8 ids");
    }
    const Act& act = static_cast<const IndexBundle*>(h)->act();
    for (uint64_t i = 0; i < n; i += 8) {
      if (kernel == 0) {
        CellId cells[8];
        for (int k = 0; k < 8; ++k) cells[k] = CellId{raw[i + k]};
        act.probe_batch(cells, out_entries + i);
      } else if (kernel == 1) {
        detail::probe_batch_scalar(act.view(), raw + i, out_entries + i);
      } else {
        detail::probe_batch_avx2(act.view(), raw + i, out_entries + i);
      }
    }
  });
}

int ref_avx2_available() { return detail::probe_batch_avx2_available(); }

// Act::resolve: writes up to cap (polygon_id, interior) pairs; returns count
// or a negative status.
int64_t ref_resolve(const void* h, uint64_t entry, uint32_t* ids,
                    uint8_t* interior, uint64_t cap) {
  int64_t n = 0;
  const int rc = guarded([&] {
    const ProbeResult r = static_cast<const IndexBundle*>(h)->act().resolve(entry);
    n = static_cast<int64_t>(r.refs.size());
    for (size_t i = 0; i < r.refs.size() && i < cap; ++i) {
      ids[i] = r.refs[i].polygon_id;
      interior[i] = r.refs[i].interior;
    }
  });
  return rc == kOk ? n : rc;
}

int ref_pip_test(const double* ring_latlng, uint64_t n_vtx, const double* latlng,
                 uint64_t n, uint8_t* out) {
  return guarded([&] {
    Polygon poly;
    poly.vertices.assign(as_points(ring_latlng, n_vtx).begin(),
                         as_points(ring_latlng, n_vtx).end());
    const auto pts = as_points(latlng, n);
    for (uint64_t i = 0; i < n; ++i) out[i] = pip_test(poly, pts[i]);
  });
}

// join_exact / join_approx.  Two-call protocol: the pairs are kept in a
// heap object; read sizes, copy out, free.
struct RefPairs {
  std::vector<JoinPair> pairs;
  JoinStats stats;
};

void* ref_join_pairs(const void* h, const double* latlng, uint64_t n, int exact,
                     uint64_t* n_pairs, uint64_t stats[6], int* status) {
  RefPairs* out = new RefPairs;
  *status = guarded([&] {
    const IndexBundle& b = *static_cast<const IndexBundle*>(h);
    out->pairs = exact ? join_exact(b, as_points(latlng, n), &out->stats)
                       : join_approx(b, as_points(latlng, n), &out->stats);
  });
  if (*status != kOk) {
    delete out;
    return nullptr;
  }
  *n_pairs = out->pairs.size();
  if (stats) {
    stats[0] = out->stats.probes;
    stats[1] = out->stats.pip_tests;
    stats[2] = out->stats.false_hits;
    stats[3] = out->stats.solely_true_hits;
    stats[4] = out->stats.refinement_entered;
    stats[5] = out->stats.candidate_refs;
  }
  return out;
}

void ref_pairs_copy(const void* p, uint64_t* point_index, uint32_t* polygon_id) {
  const RefPairs& r = *static_cast<const RefPairs*>(p);
  for (size_t i = 0; i < r.pairs.size(); ++i) {
    point_index[i] = r.pairs[i].point_index;
    polygon_id[i] = r.pairs[i].polygon_id;
  }
}

void ref_pairs_free(void* p) { delete static_cast<RefPairs*>(p); }

// join_count_per_polygon (mode from the bundle).  Returns the number of
// map entries (non-zero polygons only) or a negative status.
int64_t ref_join_count(const void* h, const double* latlng, uint64_t n,
                       int threads, uint32_t* ids, uint64_t* counts,
                       uint64_t cap) {
  int64_t m = 0;
  const int rc = guarded([&] {
    const auto res = join_count_per_polygon(*static_cast<const IndexBundle*>(h),
                                            as_points(latlng, n), threads);
    m = static_cast<int64_t>(res.size());
    uint64_t i = 0;
    for (const auto& [id, c] : res) {
      if (i >= cap) break;
      ids[i] = id;
      counts[i] = c;
      ++i;
    }
  });
  return rc == kOk ? m : rc;
}

// The threaded exact count the survey prescribes for an approx-built bundle
// joined exactly (BASELINE config 5): join_count_per_polygon would take the
// mode from the bundle (join.cpp:257), so workers call join_exact on
// `chunk`-point slices and merge count_per_polygon maps.
int64_t ref_join_exact_count_threads(const void* h, const double* latlng,
                                     uint64_t n, int threads, uint64_t chunk,
                                     uint32_t* ids, uint64_t* counts,
                                     uint64_t cap) {
  int64_t m = 0;
  const int rc = guarded([&] {
    const IndexBundle& b = *static_cast<const IndexBundle*>(h);
    if (threads < 1) threads = 1;
    if (chunk == 0) chunk = 65536;
    const auto pts = as_points(latlng, n);
    std::atomic<uint64_t> next{0};
    std::vector<std::map<uint32_t, uint64_t>> partial(threads);
    std::vector<std::string> errors(threads);
    auto worker = [&](int w) {
      try {
        for (;;) {
          const uint64_t begin = next.fetch_add(chunk);
          if (begin >= n) break;
          const uint64_t len = std::min<uint64_t>(chunk, n - begin);
          for (const JoinPair& pr : join_exact(b, pts.subspan(begin, len))) {
            ++partial[w][pr.polygon_id];
          }
        }
      } catch (const std::exception& e) {
        errors[w] = e.what();
      }
    };
    std::vector<std::thread> pool;
    for (int w = 0; w < threads; ++w) pool.emplace_back(worker, w);
    for (auto& t : pool) t.join();
    for (const auto& e : errors) {
      if (!e.empty()) throw std::runtime_error(e);
    }
    std::map<uint32_t, uint64_t> merged;
    for (const auto& part : partial) {
      for (const auto& [id, c] : part) merged[id] += c;
    }
    m = static_cast<int64_t>(merged.size());
    uint64_t i = 0;
    for (const auto& [id, c] : merged) {
      if (i >= cap) break;
      ids[i] = id;
      counts[i] = c;
      ++i;
    }
  });
  return rc == kOk ? m : rc;
}

// CsvPointReader (io.hpp:43-68, csv.cpp:54-100) over a text buffer: every valid
// point in order.  Returns 0 on success; a DataError (empty input, missing
// column, strict-mode bad row) comes back as kOther with its message in
// ref_last_error().  *n_points is the total number of valid points even when it
// exceeds `cap`.
int ref_csv_points(const char* text, uint64_t n_bytes, const char* lat_column,
                   const char* lng_column, int strict, double* out_latlng,
                   uint64_t cap, uint64_t* n_points, uint64_t* n_skipped) {
  return guarded([&] {
    std::istringstream is(std::string(text, n_bytes));
    CsvPointReader::Options opt;
    opt.lat_column = lat_column;
    opt.lng_column = lng_column;
    opt.strict = strict != 0;
    CsvPointReader reader(is, opt);
    LatLng p;
    uint64_t n = 0;
    while (reader.next(p)) {
      if (n < cap) {
        out_latlng[2 * n] = p.lat;
        out_latlng[2 * n + 1] = p.lng;
      }
      ++n;
    }
    *n_points = n;
    *n_skipped = reader.skipped_rows();
  });
}

// The `any_candidate` test Act::train applies to every training point
// (act.cpp:414-440), through the reference's own probe / for_each_reference.
int ref_training_candidates(const void* h, const double* latlng, uint64_t n,
                            uint8_t* out_flags) {
  return guarded([&] {
    const Act& act = static_cast<const IndexBundle*>(h)->act();
    const auto pts = as_points(latlng, n);
    const int level = act.max_indexed_level();
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t e = act.probe(cell_from_point(pts[i], level));
      bool any_candidate = false;
      act.for_each_reference(e, [&](uint32_t, bool interior) {
        if (!interior) any_candidate = true;
      });
      out_flags[i] = any_candidate ? 1 : 0;
    }
  });
}

int ref_accumulate_probe_stats(const void* h, const double* latlng, uint64_t n,
                               uint64_t stats[6]) {
  return guarded([&] {
    JoinStats s;
    s.probes = stats[0];
    s.pip_tests = stats[1];
    s.false_hits = stats[2];
    s.solely_true_hits = stats[3];
    s.refinement_entered = stats[4];
    s.candidate_refs = stats[5];
    accumulate_probe_stats(*static_cast<const IndexBundle*>(h),
                           as_points(latlng, n), s);
    stats[0] = s.probes;
    stats[1] = s.pip_tests;
    stats[2] = s.false_hits;
    stats[3] = s.solely_true_hits;
    stats[4] = s.refinement_entered;
    stats[5] = s.candidate_refs;
  });
}

// Wall-clock of one join_count_per_polygon call, steady_clock around the
// call exactly as `geojoin bench` does (tools/geojoin_main.cpp:193-218).
double ref_time_join_count(const void* h, const double* latlng, uint64_t n,
                           int threads, uint64_t* total_pairs, int* status) {
  double secs = 0.0;
  *status = guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    const auto res = join_count_per_polygon(*static_cast<const IndexBundle*>(h),
                                            as_points(latlng, n), threads);
    const auto t1 = std::chrono::steady_clock::now();
    secs = std::chrono::duration<double>(t1 - t0).count();
    uint64_t tot = 0;
    for (const auto& [id, c] : res) tot += c;
    if (total_pairs) *total_pairs = tot;
  });
  return secs;
}

}  // extern "C"
