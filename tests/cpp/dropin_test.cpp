// Drop-in test: a C++ program written against the REFERENCE's headers that
// runs the reference's CPU join and geojoin::gpu's join (include/geojoin_gpu.hpp
// over libgeojoin_b200.so) on the same IndexBundle and compares the results
// bit for bit.  Mirrors the reference's own join tests (tests/test_join.cpp:
// 115-134 exact == oracle, :160-189 approx, :200-214 streaming counts) with
// the reference itself as the oracle.  Built by __graft_entry__.build() where
// /root/reference exists; run on the GPU box by tests/test_gpu_dropin.py.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <random>
#include <vector>

#include "geojoin/join.hpp"
#include "geojoin_gpu.hpp"

using namespace geojoin;

namespace {

struct Rng {  // same recipe as the reference's test RNG: raw mt19937_64 -> [0,1)
  std::mt19937_64 gen;
  explicit Rng(uint64_t seed) : gen(seed) {}
  double u01() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * u01(); }
  int uniform_int(int lo, int hi) { return lo + static_cast<int>(gen() % static_cast<uint64_t>(hi - lo + 1)); }
};

Polygon star(Rng& rng, uint32_t id, LatLng c, double radius, int n) {
  Polygon poly;
  poly.id = id;
  const double pi = std::acos(-1.0);
  for (int i = 0; i < n; ++i) {
    const double a = (i + 0.2 + 0.6 * rng.u01()) * 2.0 * pi / n;
    const double r = radius * rng.uniform(0.55, 1.45);
    poly.vertices.push_back({c.lat + r * std::sin(a), c.lng + r * std::cos(a)});
  }
  return poly;
}

int failures = 0;
#define EXPECT(cond)                                                  \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

bool same_stats(const JoinStats& a, const JoinStats& b) {
  return a.probes == b.probes && a.pip_tests == b.pip_tests && a.false_hits == b.false_hits &&
         a.solely_true_hits == b.solely_true_hits && a.refinement_entered == b.refinement_entered &&
         a.candidate_refs == b.candidate_refs;
}

void compare(const IndexBundle& bundle, const std::vector<LatLng>& points) {
  gpu::DeviceIndex dev(bundle, 0);
  JoinStats cs, gs;
  EXPECT(gpu::join_exact(dev, points, &gs) == join_exact(bundle, points, &cs));
  EXPECT(same_stats(cs, gs));
  cs = JoinStats{};
  gs = JoinStats{};
  EXPECT(gpu::join_approx(dev, points, &gs) == join_approx(bundle, points, &cs));
  EXPECT(same_stats(cs, gs));
  for (int threads : {1, 3}) {
    EXPECT(gpu::join_count_per_polygon(dev, points, threads) == join_count_per_polygon(bundle, points, threads));
  }
  cs = JoinStats{};
  gs = JoinStats{};
  accumulate_probe_stats(bundle, points, cs);
  gpu::accumulate_probe_stats(dev, points, gs);
  EXPECT(same_stats(cs, gs));
  const IndexMetrics cm = collect_metrics(bundle, points), gm = gpu::collect_metrics(dev, points);
  EXPECT(cm.tree_nodes == gm.tree_nodes && cm.false_hit_fraction == gm.false_hit_fraction &&
         cm.solely_true_hit_fraction == gm.solely_true_hit_fraction && cm.avg_candidates == gm.avg_candidates);

  // the probe half of Act::train (act.cpp:414-440) as a pre-pass: the work list and expensive_fraction
  std::vector<size_t> want_candidates;
  for (size_t i = 0; i < points.size(); ++i) {
    const uint64_t e = bundle.act().probe(cell_from_point(points[i], bundle.act().max_indexed_level()));
    bool any_candidate = false;
    bundle.act().for_each_reference(e, [&](uint32_t, bool interior) {
      if (!interior) any_candidate = true;
    });
    if (any_candidate) want_candidates.push_back(i);
  }
  EXPECT(gpu::training_candidates(dev, points) == want_candidates);
  EXPECT(gpu::expensive_fraction(dev, points) ==
         static_cast<double>(want_candidates.size()) / static_cast<double>(points.size()));

  // load_points_csv (csv.cpp:102-113): rows parsed on the GPU against the reference's reader
  {
    const std::string path = "/tmp/geojoin_dropin_points.csv";
    {
      std::ofstream csv(path);
      csv << "id,lng,note,lat\n";
      csv.precision(17);
      for (size_t i = 0; i < 5000; ++i) {
        csv << i << ',' << points[i].lng << ",x," << points[i].lat << (i % 3 ? "\n" : "\r\n");
        if (i % 500 == 0) csv << "bad,row\n\n" << i << ",181,y,5\n";
      }
    }
    const std::vector<LatLng> want = load_points_csv(path);
    const std::vector<LatLng> got = gpu::load_points_csv(dev, path);
    EXPECT(got.size() == want.size() && got.size() == 5000);
    bool same = got.size() == want.size();
    for (size_t i = 0; same && i < got.size(); ++i) same = got[i].lat == want[i].lat && got[i].lng == want[i].lng;
    EXPECT(same);
    CsvPointReader::Options strict;
    strict.strict = true;
    bool cpu_threw = false, gpu_threw = false;
    try { load_points_csv(path, strict); } catch (const DataError&) { cpu_threw = true; }
    try { gpu::load_points_csv(dev, path, strict); } catch (const DataError&) { gpu_threw = true; }
    EXPECT(cpu_threw && gpu_threw);
    std::remove(path.c_str());
  }

  // The reference's worker fan-out (join.cpp:255-285) over index replicas: one replica per GPU of the box,
  // topped up to three (a device may hold several replicas; they share nothing), `threads` = how many take part.
  // Results must not depend on the worker count (tests/test_join.cpp:200-214).
  {
    std::vector<int> devices = gpu::all_devices();
    while (devices.size() < 3) devices.push_back(0);
    gpu::DeviceIndex fleet(bundle, devices);
    EXPECT(fleet.replicas() == static_cast<int>(devices.size()));
    const auto want_counts = join_count_per_polygon(bundle, points, 1);
    for (int threads : {1, 2, 3, 7}) EXPECT(gpu::join_count_per_polygon(fleet, points, threads) == want_counts);
    JoinStats fs;
    cs = JoinStats{};
    EXPECT(gpu::join_exact(fleet, points, &fs) == join_exact(bundle, points, &cs));
    EXPECT(same_stats(cs, fs));
    fs = JoinStats{};
    cs = JoinStats{};
    EXPECT(gpu::join_approx(fleet, points, &fs) == join_approx(bundle, points, &cs));
    EXPECT(same_stats(cs, fs));
    // an offending point in the LAST range is reported even though the first ranges succeed
    std::vector<LatLng> bad_tail = points;
    bad_tail[bad_tail.size() - 2].lng = -181.0;
    bool threw = false;
    try { gpu::join_count_per_polygon(fleet, bad_tail, 0); } catch (const std::invalid_argument&) { threw = true; }
    EXPECT(threw);
  }

  // a single bad coordinate aborts the join with std::invalid_argument on both sides
  std::vector<LatLng> bad = points;
  bad[bad.size() / 2].lat = 91.0;
  bool cpu_threw = false, gpu_threw = false;
  try { join_exact(bundle, bad); } catch (const std::invalid_argument&) { cpu_threw = true; }
  try { gpu::join_exact(dev, bad); } catch (const std::invalid_argument&) { gpu_threw = true; }
  EXPECT(cpu_threw && gpu_threw);
}

}  // namespace

int main() {
  Rng rng(0x10e0002);
  std::vector<Polygon> polygons;
  for (uint32_t i = 0; i < 8; ++i) {
    const LatLng c{rng.uniform(-10.0, -6.0), rng.uniform(50.0, 54.0)};
    const double radius = rng.uniform(0.2, 1.2);
    polygons.push_back(star(rng, i, c, radius, rng.uniform_int(8, 24)));
  }
  std::vector<LatLng> points;
  for (int i = 0; i < 20000; ++i) points.push_back({rng.uniform(-11.5, -4.5), rng.uniform(48.5, 55.5)});
  for (int i = 0; i < 16; ++i) points[i] = polygons[3].vertices[i % polygons[3].vertices.size()];  // on vertices

  JoinConfig exact_cfg;
  exact_cfg.mode = JoinMode::kExact;
  compare(build_index(polygons, exact_cfg, {}), points);

  JoinConfig approx_cfg;
  approx_cfg.mode = JoinMode::kApprox;
  approx_cfg.precision_m = 500.0;
  const IndexBundle approx_bundle = build_index(polygons, approx_cfg, {});
  EXPECT(approx_bundle.report().mode == JoinMode::kApprox);
  compare(approx_bundle, points);

  if (failures == 0) std::printf("DROPIN OK\n");
  return failures == 0 ? 0 : 1;
}
