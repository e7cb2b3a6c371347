// geojoin::gpu — the reference's join API (include/geojoin/join.hpp) served by
// the B200 library through its C ABI (geojoin_b200.h).
//
// This is the binding a maintainer of the reference adds: it includes the
// reference's own headers, takes the reference's own types, and keeps the
// signatures of
//
//   join_exact / join_approx        include/geojoin/join.hpp:128-138, src/join.cpp:237-247
//   join_count_per_polygon          include/geojoin/join.hpp:145-146, src/join.cpp:255-285
//   accumulate_probe_stats          include/geojoin/join.hpp:153-154, src/join.cpp:287-290
//   collect_metrics                 include/geojoin/join.hpp:148-149, src/join.cpp:309-314
//
// plus the probe half of Act::train (src/act.cpp:414-440) as a pre-pass:
// training_candidates / expensive_fraction, and load_points_csv
// (include/geojoin/io.hpp:71-72) parsed on the device.
//
// so a call site switches by replacing `geojoin::` with `geojoin::gpu::` and
// handing over a DeviceIndex made once from its IndexBundle.  Errors come back
// as the reference's exception types.  Header-only; link libgeojoin_b200.so.
#pragma once

#include <fstream>
#include <iterator>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "geojoin/io.hpp"
#include "geojoin/join.hpp"
#include "geojoin_b200.h"

namespace geojoin::gpu {

namespace detail {

[[noreturn]] inline void raise(int status) {
  const std::string msg = gj_last_error();
  switch (status) {
    case GJ_INVALID_POINT:
    case GJ_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);  // cell_id.cpp:83-88
    case GJ_CORRUPT_INDEX:
    case GJ_UNKNOWN_POLYGON:
      throw CorruptionError(msg);  // act.hpp:44-46
    default:
      throw std::runtime_error(msg);
  }
}

inline void check(int status) {
  if (status != GJ_OK) raise(status);
}

}  // namespace detail

/// Every CUDA device of the box, in order: the device list that makes the GPU
/// join use all of them.
inline std::vector<int> all_devices() {
  std::vector<int> d(static_cast<size_t>(gj_device_count()));
  for (size_t k = 0; k < d.size(); ++k) d[k] = static_cast<int>(k);
  return d;
}

/// The reference's IndexBundle replicated into the HBM of one GPU — or of
/// several: the first replica is built from the bundle, the others are copied
/// from it device to device.  Immutable like the bundle it came from
/// (join.hpp:86-88); the sessions inside serialise callers, so use one
/// DeviceIndex per calling thread or guard it.
class DeviceIndex {
 public:
  /// Copies the bundle's probe view (act.hpp:108-116), lookup table and
  /// polygons to `device` (-1 = current).  Nothing of `bundle` is retained.
  explicit DeviceIndex(const IndexBundle& bundle, int device = -1) : DeviceIndex(bundle, std::vector<int>{device}) {}

  /// One replica per listed device (e.g. all_devices()).  The joins below then
  /// fan out over them like join_count_per_polygon fans out over threads
  /// (join.cpp:255-285): contiguous point ranges, one per replica.
  DeviceIndex(const IndexBundle& bundle, const std::vector<int>& devices) {
    const Act& act = bundle.act();
    const ActProbeView& v = act.view();
    gj_index_desc d{};
    d.arena = v.arena;
    d.node_count = act.node_count();
    d.lut = act.lookup_table().data();
    d.lut_len = act.lookup_table().size();
    for (int f = 0; f < 8; ++f) {
      d.roots[f] = v.roots[f];
      d.prefixes[f] = v.prefixes[f];
      d.prefix_bits[f] = v.prefix_bits[f];
    }
    d.k_max = act.config().k_max;
    d.approx_mode = bundle.report().mode == JoinMode::kApprox;
    std::vector<uint32_t> ids;
    std::vector<uint64_t> off{0};
    std::vector<double> latlng;
    for (const Polygon& poly : bundle.polygons()) {
      ids.push_back(poly.id);
      for (const LatLng& p : poly.vertices) {
        latlng.push_back(p.lat);
        latlng.push_back(p.lng);
      }
      off.push_back(latlng.size() / 2);
    }
    d.n_polygons = ids.size();
    d.polygon_ids = ids.data();
    d.vtx_off = off.data();
    d.vtx_latlng = latlng.data();
    gj_group* g = nullptr;
    detail::check(gj_group_create(&d, resolved(devices).data(), static_cast<int>(devices.size()), nullptr, &g));
    adopt(g);
  }

  /// IndexBundle::load without the host-side Act (join.cpp:341-381).
  explicit DeviceIndex(const std::string& gjx1_path, int device = -1)
      : DeviceIndex(gjx1_path, std::vector<int>{device}) {}
  DeviceIndex(const std::string& gjx1_path, const std::vector<int>& devices) {
    gj_group* g = nullptr;
    detail::check(gj_group_load_file(gjx1_path.c_str(), resolved(devices).data(), static_cast<int>(devices.size()),
                                     nullptr, &g));
    adopt(g);
  }

  DeviceIndex(const DeviceIndex&) = delete;
  DeviceIndex& operator=(const DeviceIndex&) = delete;

  gj_group* group() const { return group_.get(); }
  int replicas() const { return gj_group_size(group_.get()); }
  gj_session* session(int k = 0) const { return gj_group_session(group_.get(), k); }
  const gj_index_info& info() const { return info_; }
  const std::vector<uint32_t>& ids() const { return ids_; }
  JoinMode mode() const { return info_.approx_mode ? JoinMode::kApprox : JoinMode::kExact; }

 private:
  static std::vector<int> resolved(const std::vector<int>& devices) {
    if (devices.empty()) throw std::invalid_argument("DeviceIndex: empty device list");
    return devices;  // -1 = the current device, resolved by the library
  }
  void adopt(gj_group* g) {
    group_.reset(g);
    gj_index* ix = gj_group_index(g, 0);
    detail::check(gj_index_get_info(ix, &info_));
    ids_.resize(info_.n_ids);
    detail::check(gj_index_ids(ix, ids_.data()));
  }

  struct GroupDeleter {
    void operator()(gj_group* p) const { gj_group_destroy(p); }
  };
  std::unique_ptr<gj_group, GroupDeleter> group_;  // replicas and their sessions
  gj_index_info info_{};
  std::vector<uint32_t> ids_;
};

namespace detail {

inline const double* as_doubles(std::span<const LatLng> points) {
  static_assert(sizeof(LatLng) == 2 * sizeof(double), "LatLng is two packed doubles (latlng.hpp:26-29)");
  return reinterpret_cast<const double*>(points.data());
}

inline void add_stats(const gj_stats& s, JoinStats* out) {
  if (!out) return;
  out->probes += s.probes;
  out->pip_tests += s.pip_tests;
  out->false_hits += s.false_hits;
  out->solely_true_hits += s.solely_true_hits;
  out->refinement_entered += s.refinement_entered;
  out->candidate_refs += s.candidate_refs;
}

inline std::vector<JoinPair> pairs(const DeviceIndex& ix, std::span<const LatLng> points, int mode,
                                   JoinStats* stats) {
  uint64_t n_pairs = 0, bad = 0;
  gj_stats s{};
  check(gj_group_join_pairs_host(ix.group(), 0, as_doubles(points), points.size(), mode, &n_pairs,
                                 stats ? &s : nullptr, &bad));
  std::vector<uint64_t> row_ptr(points.size() + 1);
  std::vector<uint32_t> ids(n_pairs);
  check(gj_group_pairs_copy(ix.group(), row_ptr.data(), ids.data()));
  // CSR -> the reference's array of {point_index, polygon_id}, a few threads over ranges of points
  std::vector<JoinPair> out(n_pairs);
  const size_t n = points.size();
  const size_t workers = n_pairs < (1u << 22) ? 1 : std::min<size_t>(8, std::max(1u, std::thread::hardware_concurrency()));
  auto expand = [&](size_t first, size_t last) {
    for (size_t i = first; i < last; ++i) {
      for (uint64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) out[k] = JoinPair{i, ids[k]};
    }
  };
  std::vector<std::thread> pool;
  for (size_t w = 1; w < workers; ++w) pool.emplace_back(expand, n * w / workers, n * (w + 1) / workers);
  expand(0, n / workers);
  for (std::thread& t : pool) t.join();
  add_stats(s, stats);
  return out;
}

}  // namespace detail

inline std::vector<JoinPair> join_exact(const DeviceIndex& ix, std::span<const LatLng> points,
                                        JoinStats* stats = nullptr) {
  return detail::pairs(ix, points, GJ_MODE_EXACT, stats);
}

inline std::vector<JoinPair> join_approx(const DeviceIndex& ix, std::span<const LatLng> points,
                                         JoinStats* stats = nullptr) {
  return detail::pairs(ix, points, GJ_MODE_APPROX, stats);
}

/// Mode from the bundle (join.cpp:257); zero counts are omitted.  `threads` is
/// the reference's worker count (join.cpp:255-262): that many replicas of the
/// DeviceIndex each join one contiguous range of the points; values above the
/// number of replicas, or <= 0, mean all of them.  The result does not depend
/// on it (tests/test_join.cpp:200-214).
inline std::map<uint32_t, uint64_t> join_count_per_polygon(const DeviceIndex& ix,
                                                           std::span<const LatLng> points,
                                                           int threads = 1) {
  std::vector<uint64_t> counts(ix.ids().size() + 1, 0);
  uint64_t bad = 0;
  detail::check(gj_group_join_count_host(ix.group(), threads, detail::as_doubles(points), points.size(), 0,
                                         GJ_MODE_BUNDLE, counts.data(), nullptr, nullptr, nullptr, &bad));
  std::map<uint32_t, uint64_t> out;
  for (size_t s = 0; s < ix.ids().size(); ++s) {
    if (counts[s]) out.emplace(ix.ids()[s], counts[s]);
  }
  return out;
}

inline void accumulate_probe_stats(const DeviceIndex& ix, std::span<const LatLng> points,
                                   JoinStats& stats) {
  std::vector<uint64_t> counts(ix.ids().size() + 1, 0);
  gj_stats s{};
  uint64_t bad = 0;
  detail::check(gj_group_join_count_host(ix.group(), 0, detail::as_doubles(points), points.size(), 0,
                                         GJ_MODE_APPROX, counts.data(), &s, nullptr, nullptr, &bad));
  detail::add_stats(s, &stats);
}

inline IndexMetrics collect_metrics(const DeviceIndex& ix, std::span<const LatLng> points) {
  JoinStats stats;
  accumulate_probe_stats(ix, points, stats);
  return metrics_from_stats(stats, ix.info().node_count);
}

// The training points Act::train has split work for (src/act.cpp:428-440):
// those whose probe meets at least one candidate reference, ascending.  A point
// that meets none now meets none after any amount of training (splits only
// refine candidate cells), so train() may iterate over this list instead of
// probing every point.
inline std::vector<size_t> training_candidates(const DeviceIndex& ix, std::span<const LatLng> points) {
  std::vector<uint64_t> idx(points.size());
  uint64_t found = 0, bad = 0;
  detail::check(gj_training_candidates_host(ix.session(), detail::as_doubles(points), points.size(), 0, idx.data(),
                                            idx.size(), &found, &bad));
  return std::vector<size_t>(idx.begin(), idx.begin() + static_cast<std::ptrdiff_t>(found));
}

// TrainingStats::expensive_fraction_{before,after} (src/act.cpp:414-426).
inline double expensive_fraction(const DeviceIndex& ix, std::span<const LatLng> points) {
  if (points.empty()) return 0.0;
  uint64_t found = 0, bad = 0;
  detail::check(gj_training_candidates_host(ix.session(), detail::as_doubles(points), points.size(), 0, nullptr, 0,
                                            &found, &bad));
  return static_cast<double>(found) / static_cast<double>(points.size());
}

// load_points_csv (io.hpp:71-72, csv.cpp:102-113) with the rows parsed on the
// GPU; DataError for an unreadable or empty file, a missing column or — strict —
// an invalid row, like the reference.
inline std::vector<LatLng> load_points_csv(const DeviceIndex& ix, const std::string& path,
                                           CsvPointReader::Options options = CsvPointReader::Options()) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw DataError("cannot open point file: " + path);
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  size_t rows = 1;
  for (char c : text) rows += c == '\n';
  std::vector<LatLng> points(rows);
  uint64_t n = 0, skipped = 0, bad_line = 0;
  const int rc = gj_points_from_csv_host(ix.session(), text.data(), text.size(), options.lat_column.c_str(),
                                         options.lng_column.c_str(), options.strict ? 1 : 0,
                                         reinterpret_cast<double*>(points.data()), points.size(), &n, &skipped, &bad_line);
  if (rc == GJ_DATA_ERROR) throw DataError(gj_last_error());
  detail::check(rc);
  points.resize(n);
  return points;
}

}  // namespace geojoin::gpu
