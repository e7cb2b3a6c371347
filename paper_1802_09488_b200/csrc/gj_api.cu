// C ABI of geojoin_b200 (include/geojoin_b200.h): sessions, kernel launch
// plumbing and the host-buffer pipelines (H2D / kernels / D2H overlapped on
// three streams).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <thread>

#include "gj_host.hpp"
#include "gj_csv.cuh"
#include "gj_kernels.cuh"

namespace gj {

const std::string& last_error();
gj_options default_options();
int create_index(const gj_index_desc& d, int device, const gj_options* opt, gj_index** out);
int load_index_file(const char* path, int device, const gj_options* opt, gj_index** out);
int replicate_index(const gj_index& src, int device, gj_index** out);

namespace {

// Point indices travel in K1's queue words next to flag bits: 2^31 - 1 points per launch, fewer for arenas of
// 2^24 nodes and more (DevQueueCoding::index_bits).
uint64_t max_launch_points(const gj_index& ix) {
  uint64_t cap = (1ull << ix.dev.qc.index_bits) - 1;
  // test hook: exercise the splitting of device-resident calls
  if (ix.opt.max_launch_points) cap = std::min<uint64_t>(cap, ix.opt.max_launch_points);
  return cap;
}
constexpr size_t kScratchBudget = 3ull << 30;      // per-chunk task + overflow scratch

size_t align16(size_t v) { return (v + 15) & ~size_t{15}; }

struct SmemPlan {
  uint32_t queue_off, hist_off, hist_rep;
  uint32_t hist16;  // 1 = one 16-bit histogram instead (hist_rep == 0)
  uint32_t stage_off;  // per-warp staging buffers for lookup-table records, 0 = none
  uint32_t stage_chunks;  // 16-byte chunks per warp
  size_t total;
};

constexpr size_t kHist32MaxRow = 64u << 10;  // a 32-bit histogram row set beyond this is not tried
constexpr size_t kHist16MaxRow = 96u << 10;

}  // namespace

bool k1_uses_hist16(size_t n_ids, const gj_options& opt) {
  if (opt.hist16 == 0 || n_ids == 0) return false;
  const size_t row16 = (n_ids + 2) / 2 * 4;
  if (row16 > kHist16MaxRow) return false;
  return opt.hist16 > 0 || (n_ids + 1) * 4 > kHist32MaxRow;  // forced, or the 32-bit form does not fit
}

// Lookup-table-heavy indexes (overlapping polygon sets: every probe ends in a record of many references) stage the
// records of a population-3 batch in shared memory; the first tier then only has to catch the points outside every
// polygon, so it makes room.
// Only tables far beyond L2 (256 MB and more): there a lane's word-by-word walk pays an L2 / DRAM round trip per
// sector (full-size BASELINE config 5, 1.3 GB table: 5.56 -> 4.71 ms per 20 M points with staging); a table that
// sits in L2 is walked faster than it is staged (config-5 stand-in, 30 MB: 2.42 vs 2.96 ms — instruction-bound).
bool k1_stages_records(uint64_t lut_len, const gj_options& opt) {
  return opt.stage_lut > 0 || (opt.stage_lut < 0 && lut_len >= (1ull << 26));
}

size_t k1_smem_besides_tier(size_t n_ids, const gj_options& opt) {
  const size_t queues = static_cast<size_t>(kJoinThreads / 32) * kQueueBytesPerWarp;
  const size_t hist_row = (n_ids + 1) * 4;
  size_t hist = hist_row <= kHist32MaxRow ? hist_row : 0;
  if (k1_uses_hist16(n_ids, opt)) hist = (n_ids + 2) / 2 * 4;
  return queues + hist + 64;  // + alignment slack
}

namespace {

// Shared memory of K1: [16-bit tier | per-warp queues | histogram].  The SM's
// L1 is what shared memory leaves of 256 KB, in carve-out steps, and K1 needs
// L1 for its loads in flight (measured on config 2: 0.53 ms per 100 M points
// up to the 164 KB step, 0.545 at 196 KB, 0.81 at 228 KB).  The histogram's
// replication hardly matters (ATOMS.POPC.INC aggregates equal addresses), so
// it only takes what is left inside the carve-out step the rest already needs.
SmemPlan plan_smem(const gj_index& ix) {
  SmemPlan p{};
  // (the direct form stages no tier, and its per-warp area is two staging buffers + a longer Q3)
  const size_t table_bytes = ix.direct ? 0 : static_cast<size_t>(ix.dev.dir16.n_table) * 2;
  size_t at = align16(std::max<size_t>(table_bytes, 16));
  p.queue_off = static_cast<uint32_t>(at);
  at += static_cast<size_t>(kJoinThreads / 32) * (ix.direct ? kDirectBytesPerWarp : kQueueBytesPerWarp);
  p.hist_off = static_cast<uint32_t>(at);
#ifdef GJ_SMEM_LIMIT_KB  // tuning: leave room for more than one CTA per SM
  const size_t limit = static_cast<size_t>(GJ_SMEM_LIMIT_KB) << 10;
#else
  const size_t limit = ix.smem_optin > 2048 ? ix.smem_optin - 1024 : 0;
#endif
  const size_t one = (static_cast<size_t>(ix.dev.n_ids) + 1) * 4;  // + the spare row non-emitting lanes count into
  uint32_t rep = 0;
  const size_t last_good_step = (196u - 1u) << 10;  // above it: the 228 KB carve-out cliff
  const bool hist_fits = at + one <= limit && (at + one <= last_good_step || at > last_good_step);
  const size_t one16 = (static_cast<size_t>(ix.dev.n_ids) + 2) / 2 * 4;  // two 16-bit counters per word, + the spare
  if (k1_uses_hist16(ix.dev.n_ids, ix.opt) && at + one16 <= limit) {
    p.hist16 = 1;
    at += one16;
  } else if (ix.dev.n_ids && hist_fits) {
    size_t step = limit;  // carve-out steps hold 1 KB of system shared memory per CTA
    for (size_t kb : {64, 100, 132, 164, 196}) {
      if (at + one <= (kb - 1) << 10) {
        step = std::min(limit, (kb - 1) << 10);
        break;
      }
    }
    rep = 1;
    while (rep < 32 && at + one * rep * 2 <= step) rep <<= 1;
  }
  if (!p.hist16 && ix.opt.hist_rep_cap >= 0) {  // explicit knob: a power of two at most the planned value, or 0
    uint32_t cap = 0;
    while (cap < rep && (cap ? cap * 2 : 1u) <= static_cast<uint32_t>(ix.opt.hist_rep_cap)) cap = cap ? cap * 2 : 1u;
    rep = cap;
  }
  p.hist_rep = rep;
  at += one * rep;
  if (ix.stage_records) {  // lookup-table-heavy index: what is left goes to the warp-cooperative record staging (join_kernel)
    const size_t warps = kJoinThreads / 32;
    const size_t room = limit > align16(at) ? (limit - align16(at)) / (warps * 16) : 0;
    const uint32_t chunks = static_cast<uint32_t>(std::min<size_t>(room, kStageChunksMax));
    if (chunks >= kStageChunksMin) {
      p.stage_off = static_cast<uint32_t>(align16(at));
      p.stage_chunks = chunks;
      at = p.stage_off + warps * chunks * 16;
    }
  }
  if (ix.opt.smem_pad > 0 && at + static_cast<size_t>(ix.opt.smem_pad) <= limit) at += static_cast<size_t>(ix.opt.smem_pad);  // L1 carve-out experiments
  p.total = at;
  if (ix.opt.debug_plan) {
    std::fprintf(stderr, "[gj] K1 smem: 16-bit tier level %d, %zu B; queues at %u; histogram at %u x%u%s; total %zu; palette nodes %s\n",
                 30 - ix.dev.dir16.shift, table_bytes, p.queue_off, p.hist_off, p.hist_rep, p.hist16 ? " (16-bit, flushed)" : "",
                 p.total, ix.dev.node_pal ? "yes" : "no");
    std::fprintf(stderr, "[gj] K1 smem: record staging %u chunks per warp\n", p.stage_chunks);
    const DevDirectory& tb = ix.dev.dirk.n_table ? ix.dev.dirk : (ix.dev.dir2.n_table ? ix.dev.dir2 : ix.dev.dir);
    std::fprintf(stderr, "[gj] K1 32-bit tier: level %d%s, %u x %u cells (%.1f MB); queue coding %s, tier_shift %u, index bits %u\n",
                 30 - tb.shift, ix.dev.dirk.n_table ? " (refined)" : "", tb.width, tb.height, tb.n_table * 4e-6,
                 ix.dev.qc.packed ? "packed" : "unpacked", ix.dev.qc.tier_shift, ix.dev.qc.index_bits);
  }
  return p;
}

// Dynamic shared memory above 48 KB needs an opt-in per kernel.  The limit is
// a property of the kernel, not of the launch, so it is raised to the device
// maximum — a per-call value would race between sessions of differently
// sized indexes.  (The L1 carve-out follows the launch's actual size.)
template <typename Kernel>
int allow_max_smem(const gj_index& ix, Kernel kernel) {
  // once per kernel and device: the host pipelines launch a chunk every few hundred microseconds
  static std::mutex m;
  static std::vector<std::pair<const void*, int>> done;
  const std::pair<const void*, int> key{reinterpret_cast<const void*>(kernel), ix.device};
  std::lock_guard<std::mutex> lk(m);
  if (std::find(done.begin(), done.end(), key) != done.end()) return GJ_OK;
  cudaFuncAttributes attr{};
  GJ_CUDA(cudaFuncGetAttributes(&attr, kernel));  // static shared memory (K1's EmitCtx) counts against the same limit
  GJ_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(ix.smem_optin - attr.sharedSizeBytes)));
  done.push_back(key);
  return GJ_OK;
}

template <bool kIds, bool kStats, bool kDense, bool kLate, bool kStage, bool kDirect = false>
int launch_join_kernel(gj_session* s, const JoinParams& jp, const SmemPlan& sp) {
  const gj_index& ix = *s->ix;
  auto kernel = join_kernel<kIds, kStats, kDense, kLate, kStage, kDirect>;
  int rc = allow_max_smem(ix, kernel);
  if (rc != GJ_OK) return rc;
  int occ = 0;
  GJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kJoinThreads, sp.total));
  if (occ < 1) {
    set_error("join kernel does not fit on an SM");
    return GJ_CUDA_ERROR;
  }
  const uint64_t tile = static_cast<uint64_t>(kJoinThreads) * kPointsPerThread;
  const uint64_t n_tiles = (jp.n + tile - 1) / tile;
  const unsigned grid = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>(n_tiles, static_cast<uint64_t>(ix.sm_count) * occ)));
  kernel<<<grid, kJoinThreads, sp.total, s->stream>>>(ix.dev, jp);
  ++s->launches;
  GJ_CUDA(cudaGetLastError());
  return GJ_OK;
}

// Lookup-table-heavy indexes (the launch plan found room for the staging buffers) run the kStage instantiations.
template <bool kIds, bool kStats, bool kDense, bool kLate = false>
int launch_join_variant(gj_session* s, const JoinParams& jp, const SmemPlan& sp) {
  // One kStage instantiation is left out: <ids, no stats, general counting, early ids> — nvcc 12.9 gives it a
  // 704-byte stack frame (a thread-local copy of the parameter blocks), and a frame like that cost 7x in another
  // instantiation before the general emit path stopped taking the blocks by reference.  Check `ptxas -v` (python -m
  // paper_1802_09488_b200._build --force -v) when touching the kernel.
  constexpr bool kStageOk = !(kIds && !kStats && !kDense && !kLate);
  if (kStageOk && sp.stage_off != 0) return launch_join_kernel<kIds, kStats, kDense, kLate, kStageOk>(s, jp, sp);
  return launch_join_kernel<kIds, kStats, kDense, kLate, false>(s, jp, sp);
}

// K2 on a persistent grid: exactly the blocks that are resident at once (a partial second wave of a grid-stride
// kernel only adds a tail).  The instantiation follows the form of the index's strip lists.
int launch_refine(gj_session* s, const RefineParams& rp, size_t smem) {
  const gj_index& ix = *s->ix;
  auto launch = [&](auto kernel) -> int {
    int per_sm = 0;
    GJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kRefineThreads, smem));
    const unsigned blocks = static_cast<unsigned>(ix.sm_count) * static_cast<unsigned>(std::max(per_sm, 1));
    kernel<<<blocks, kRefineThreads, smem, s->stream>>>(ix.dev, rp);
    ++s->launches;
    GJ_CUDA(cudaGetLastError());
    return GJ_OK;
  };
  return ix.dev.strip_eidx ? launch(refine_kernel<true>) : launch(refine_kernel<false>);
}

int reset_status(gj_session* s, DevStatus* d_status) {
  static const DevStatus init{kNoBadIndex, 0, 0, 0, 0};
  GJ_CUDA(cudaMemcpyAsync(d_status, &init, sizeof init, cudaMemcpyHostToDevice, s->stream));
  return GJ_OK;
}

HostStager& stager_of(gj_session* s) {
  if (!s->stager) s->stager = std::make_unique<HostStager>();
  return *s->stager;
}

struct JoinRequest {
  const double2* d_pts;
  uint64_t n;
  uint64_t base_index;
  bool exact;
  bool want_stats;
  unsigned long long* d_counts;
  unsigned long long* d_stats;
  uint32_t* d_first_id;  // null = counts only
  DevStatus* d_status;
  uint64_t ovf_cap;      // records available in the session overflow buffers
  bool ovf_discard;      // first ids wanted, the overflow list not (device-resident calls)
  uint64_t task_cap;
  uint8_t* d_task_pass;  // pairs mode
  bool keep_errors;      // do not clear the error flags / bad index of the status block (see gj_join_count_device)
};

// Enqueue K1 (+ bucket + K2 in exact mode) on the session stream.
int enqueue_join(gj_session* s, const JoinRequest& rq) {
  gj_index& ix = *s->ix;
  if (rq.n > max_launch_points(ix)) {
    set_error("too many points for one launch");
    return GJ_INVALID_ARGUMENT;
  }
  const uint32_t n_ids = ix.dev.n_ids;
  int rc = GJ_OK;
  if (rq.keep_errors) {  // a later piece of one call: only the per-launch cursors start over
    GJ_CUDA(cudaMemsetAsync(&rq.d_status->overflow_count, 0, 2 * sizeof(unsigned long long), s->stream));
  } else {
    rc = reset_status(s, rq.d_status);
  }
  if (rc != GJ_OK) return rc;
  const SmemPlan sp = plan_smem(ix);

  JoinParams jp{};
  jp.pts = rq.d_pts;
  jp.n = rq.n;
  jp.base_index = rq.base_index;
  jp.counts = rq.d_counts;
  jp.stats = rq.want_stats ? rq.d_stats : nullptr;
  jp.first_id = rq.d_first_id;
  jp.ovf_point = s->d_ovf_point.as<uint64_t>();
  jp.ovf_id = s->d_ovf_id.as<uint32_t>();
  jp.ovf_ord = s->d_ovf_ord.as<uint32_t>();
  jp.ovf_cap = rq.d_first_id ? rq.ovf_cap : 0;
  jp.ovf_discard = rq.ovf_discard ? 1 : 0;
  jp.task_point = s->d_task_point.as<uint32_t>();
  jp.task_slot = s->d_task_slot.as<uint32_t>();
  jp.task_ord = s->d_task_ord.as<uint32_t>();
  jp.task_cap = rq.exact ? rq.task_cap : 0;
  jp.status = rq.d_status;
  jp.smem_queue_off = sp.queue_off;
  jp.smem_hist_off = sp.hist_off;
  jp.hist_rep = sp.hist_rep;
  jp.hist16 = sp.hist16;
  jp.smem_stage_off = sp.stage_off;
  jp.stage_chunks = sp.stage_chunks;
  // No room for the histogram in shared memory: count into per-SM copies (at most 1 GB of them)
  const size_t priv_bytes = static_cast<size_t>(ix.sm_count) * n_ids * 4;
  const bool k2_local = static_cast<size_t>(n_ids) * 4 <= (32u << 10);
  const bool k1_priv = sp.hist_rep == 0 && !sp.hist16;
  const bool want_priv = n_ids != 0 && priv_bytes <= (1ull << 30) && (k1_priv || (rq.exact && !k2_local));
  uint32_t* d_priv = nullptr;
  if (want_priv) {
    if (s->d_counts_priv.bytes < priv_bytes) {
      GJ_CUDA(s->d_counts_priv.reserve(priv_bytes));
      GJ_CUDA(cudaMemsetAsync(s->d_counts_priv.ptr, 0, priv_bytes, s->stream));
    }
    d_priv = s->d_counts_priv.as<uint32_t>();
  }
  jp.counts_priv = k1_priv ? d_priv : nullptr;
  jp.n_priv = static_cast<uint32_t>(ix.sm_count);
  jp.exact = rq.exact ? 1 : 0;

  // The direct form (join_kernel's kDirect): every point gathers its own code of the 32-bit tier; decided at index
  // creation (gj_index::direct), the shared-memory plan above follows it.
  if (ix.direct) {
    const int variant = (rq.d_first_id ? 4 : 0) | (rq.want_stats ? 2 : 0) | (ix.dev.ids_dense && sp.hist_rep ? 1 : 0);
    switch (variant) {
      case 0: rc = launch_join_kernel<false, false, false, false, false, true>(s, jp, sp); break;
      case 1: rc = launch_join_kernel<false, false, true, false, false, true>(s, jp, sp); break;
      case 2: rc = launch_join_kernel<false, true, false, false, false, true>(s, jp, sp); break;
      case 3: rc = launch_join_kernel<false, true, true, false, false, true>(s, jp, sp); break;
      case 4: rc = launch_join_kernel<true, false, false, true, false, true>(s, jp, sp); break;
      case 5: rc = launch_join_kernel<true, false, true, true, false, true>(s, jp, sp); break;
      case 6: rc = launch_join_kernel<true, true, false, true, false, true>(s, jp, sp); break;
      default: rc = launch_join_kernel<true, true, true, true, false, true>(s, jp, sp); break;
    }
  } else {
  const int variant = (rq.d_first_id && ix.ids_late ? 8 : 0) | (rq.d_first_id ? 4 : 0) | (rq.want_stats ? 2 : 0) |
                      (ix.dev.ids_dense && sp.hist_rep ? 1 : 0);
  switch (variant) {
    case 12: rc = launch_join_variant<true, false, false, true>(s, jp, sp); break;
    case 13: rc = launch_join_variant<true, false, true, true>(s, jp, sp); break;
    case 14: rc = launch_join_variant<true, true, false, true>(s, jp, sp); break;
    case 15: rc = launch_join_variant<true, true, true, true>(s, jp, sp); break;
    case 0: rc = launch_join_variant<false, false, false>(s, jp, sp); break;
    case 1: rc = launch_join_variant<false, false, true>(s, jp, sp); break;
    case 2: rc = launch_join_variant<false, true, false>(s, jp, sp); break;
    case 3: rc = launch_join_variant<false, true, true>(s, jp, sp); break;
    case 4: rc = launch_join_variant<true, false, false>(s, jp, sp); break;
    case 5: rc = launch_join_variant<true, false, true>(s, jp, sp); break;
    case 6: rc = launch_join_variant<true, true, false>(s, jp, sp); break;
    default: rc = launch_join_variant<true, true, true>(s, jp, sp); break;
  }
  }
  if (rc != GJ_OK) return rc;

  if (rq.exact && n_ids) {
    RefineParams rp{};
    rp.pts = rq.d_pts;
    rp.base_index = rq.base_index;
    rp.task_point = jp.task_point;
    rp.task_slot = jp.task_slot;
    rp.task_ord = jp.task_ord;
    rp.task_cap = jp.task_cap;
    rp.counts = rq.d_counts;
    rp.ovf_point = jp.ovf_point;
    rp.ovf_id = jp.ovf_id;
    rp.ovf_ord = jp.ovf_ord;
    rp.ovf_cap = jp.ovf_cap;
    rp.task_pass = rq.d_task_pass;
    rp.status = rq.d_status;
    rp.want_ids = rq.d_first_id && !rq.ovf_discard ? 1 : 0;
    const size_t counts_smem = static_cast<size_t>(n_ids) * 4;
    rp.smem_counts = counts_smem <= (32u << 10) ? 1 : 0;
    rp.counts_priv = rp.smem_counts ? nullptr : d_priv;
    rp.n_priv = static_cast<uint32_t>(ix.sm_count);
    if ((rc = launch_refine(s, rp, rp.smem_counts ? counts_smem : 0)) != GJ_OK) return rc;
  }
  if (d_priv) {
    fold_private_counts_kernel<<<std::max(1u, std::min((n_ids + 255u) / 256u, static_cast<unsigned>(ix.sm_count) * 8u)), 256, 0,
                                 s->stream>>>(d_priv, static_cast<uint32_t>(ix.sm_count), n_ids, rq.d_counts);
    ++s->launches;
    GJ_CUDA(cudaGetLastError());
  }
  return GJ_OK;
}

int reserve_tasks(gj_session* s, uint64_t cap) {
  GJ_CUDA(s->d_task_point.reserve(cap * 4 + 16));
  GJ_CUDA(s->d_task_slot.reserve(cap * 4 + 16));
  GJ_CUDA(s->d_task_ord.reserve(cap * 4 + 16));
  return GJ_OK;
}

int reserve_overflow(gj_session* s, uint64_t cap) {
  GJ_CUDA(s->d_ovf_point.reserve(cap * 8 + 16));
  GJ_CUDA(s->d_ovf_id.reserve(cap * 4 + 16));
  GJ_CUDA(s->d_ovf_ord.reserve(cap * 4 + 16));
  return GJ_OK;
}

int status_to_code(const DevStatus& st, uint64_t* bad_index) {
  if (st.flags & kErrInvalidPoint) {
    if (bad_index) *bad_index = st.bad_index;
    set_error("cell_from_point: invalid coordinate");
    return GJ_INVALID_POINT;
  }
  if (st.flags & kErrUnknownPolygon) {
    if (bad_index) *bad_index = st.bad_index;
    set_error("index references unknown polygon");
    return GJ_UNKNOWN_POLYGON;
  }
  if (st.flags & (kErrOverflowCap | kErrTaskCap)) {
    set_error("device scratch capacity exceeded");
    return GJ_CAPACITY;
  }
  return GJ_OK;
}

bool resolve_exact(const gj_index& ix, int mode, bool* exact) {
  switch (mode) {
    case GJ_MODE_BUNDLE:
      *exact = !ix.info.approx_mode;
      return true;
    case GJ_MODE_APPROX:
      *exact = false;
      return true;
    case GJ_MODE_EXACT:
      *exact = true;
      return true;
    default:
      return false;
  }
}

// Overflow records brought back chunk by chunk.  Chunks arrive in point
// order, so sorting each chunk's records by (point, ordinal) right after its
// copy — while the copy engine is busy with later chunks — leaves the whole
// list sorted without a pass at the end.
struct OverflowRecord {
  uint64_t point;
  uint32_t id, ord;
};
struct OverflowSink {
  std::vector<OverflowRecord> records;
  std::vector<uint64_t> tmp_point;
  std::vector<uint32_t> tmp_id, tmp_ord;
};

// The chunked host pipeline shared by gj_join_count_host and
// gj_join_pairs_host.
int run_host_join(gj_session* s, const double* latlng, uint64_t n, uint64_t base_index, bool exact,
                  uint64_t* counts, gj_stats* stats, uint32_t* out_first_id, OverflowSink* sink,
                  uint64_t* bad_index) {
  gj_index& ix = *s->ix;
  GJ_CUDA(cudaSetDevice(ix.device));
  const uint32_t n_ids = ix.dev.n_ids;
  const bool want_ids = out_first_id != nullptr;
  const uint64_t max_cand = std::max<uint64_t>(1, ix.max_cand_refs);
  const uint64_t max_refs = std::max<uint64_t>(1, ix.max_refs);
  // Worst-case scratch per point decides the chunk size.
  uint64_t per_point = 16 + (want_ids ? 4 : 0);
  if (exact) per_point += max_cand * 17;
  if (want_ids) per_point += max_refs * 16;
  uint64_t chunk_points = 3ull << 20;  // measured: 0.5 / 1 / 2 / 3 / 4 / 8 / 16 M points per chunk -> 42.2 / 35.3 / 30.1 / 30.0 / 30.2 / 30.9 / 32.1 ms per 100 M points
  if (ix.opt.chunk_points) chunk_points = std::max<uint64_t>(4096, ix.opt.chunk_points);  // explicit knob
  uint64_t chunk = std::min<uint64_t>(chunk_points, std::max<uint64_t>(4096, kScratchBudget / per_point));
  chunk = std::min<uint64_t>(chunk, std::max<uint64_t>(n, 1));
  const uint64_t task_cap = exact ? chunk * max_cand : 0;
  const uint64_t ovf_cap = want_ids ? chunk * max_refs : 0;
  if (task_cap >= (1ull << 32)) {
    set_error("candidate task capacity exceeds 2^32");
    return GJ_INVALID_ARGUMENT;
  }
  int rc;
  if (exact && (rc = reserve_tasks(s, task_cap)) != GJ_OK) return rc;
  if (want_ids && (rc = reserve_overflow(s, ovf_cap)) != GJ_OK) return rc;
  for (int b = 0; b < 3; ++b) {
    GJ_CUDA(s->d_points[b].reserve(chunk * 16));
    if (want_ids) GJ_CUDA(s->d_first_id[b].reserve(chunk * 4));
  }
  GJ_CUDA(s->d_counts.reserve(static_cast<size_t>(n_ids + 1) * 8));
  GJ_CUDA(s->d_stats.reserve(6 * 8));
  GJ_CUDA(cudaMemsetAsync(s->d_counts.ptr, 0, static_cast<size_t>(n_ids + 1) * 8, s->stream));
  GJ_CUDA(cudaMemsetAsync(s->d_stats.ptr, 0, 6 * 8, s->stream));

  // With ids or exact mode every chunk shares the task/overflow scratch, so
  // a chunk must be fully drained before the next kernel starts; the H2D of
  // the next chunk still overlaps.  Counting in approx mode pipelines freely.
  const bool serial = want_ids || exact;
  const uint64_t n_chunks = (n + chunk - 1) / chunk;
  int final_rc = GJ_OK;
  DevStatus worst{kNoBadIndex, 0, 0, 0, 0};

  // First ids go straight to pinned caller memory on the copy-out stream; for
  // pageable memory they are staged when the chunk is drained.
  const bool ids_direct = want_ids && HostStager::is_pinned(out_first_id);

  auto drain = [&](uint64_t c) -> int {  // chunk c finished on the device?
    const int b = static_cast<int>(c % 3);
    GJ_CUDA(cudaEventSynchronize(s->ev_done[b]));
    if (want_ids && !ids_direct) {
      const uint64_t c_begin = c * chunk, c_len = std::min(chunk, n - c_begin);
      GJ_CUDA(stager_of(s).to_host(out_first_id + c_begin, s->d_first_id[b].ptr, c_len * 4, s->copy_out));
    }
    const DevStatus& st = s->h_status[b];
    worst.flags |= st.flags;
    worst.bad_index = std::min(worst.bad_index, st.bad_index);
    if (sink && st.overflow_count && !(st.flags & kErrOverflowCap)) {
      const size_t m = st.overflow_count;
      sink->tmp_point.resize(m);
      sink->tmp_id.resize(m);
      sink->tmp_ord.resize(m);
      GJ_CUDA(cudaMemcpyAsync(sink->tmp_point.data(), s->d_ovf_point.ptr, m * 8, cudaMemcpyDeviceToHost, s->stream));
      GJ_CUDA(cudaMemcpyAsync(sink->tmp_id.data(), s->d_ovf_id.ptr, m * 4, cudaMemcpyDeviceToHost, s->stream));
      GJ_CUDA(cudaMemcpyAsync(sink->tmp_ord.data(), s->d_ovf_ord.ptr, m * 4, cudaMemcpyDeviceToHost, s->stream));
      GJ_CUDA(cudaStreamSynchronize(s->stream));
      const size_t at = sink->records.size();
      sink->records.resize(at + m);
      for (size_t k = 0; k < m; ++k) {
        sink->records[at + k] = OverflowRecord{sink->tmp_point[k], sink->tmp_id[k], sink->tmp_ord[k]};
      }
      std::sort(sink->records.begin() + at, sink->records.end(), [](const OverflowRecord& x, const OverflowRecord& y) {
        return x.point != y.point ? x.point < y.point : x.ord < y.ord;
      });
    }
    return GJ_OK;
  };

  for (uint64_t c = 0; c < n_chunks; ++c) {
    const int b = static_cast<int>(c % 3);
    const uint64_t begin = c * chunk;
    const uint64_t len = std::min(chunk, n - begin);
    // buffer b is free once the kernel of chunk c-3 is done (and its ids copied)
    if (c >= 3) {
      GJ_CUDA(cudaStreamWaitEvent(s->copy_in, s->ev_done[b], 0));
      if (!serial && (rc = drain(c - 3)) != GJ_OK) return rc;
    }
    GJ_CUDA(stager_of(s).to_device(s->d_points[b].ptr, latlng + 2 * begin, len * 16, s->copy_in));
    GJ_CUDA(cudaEventRecord(s->ev_in[b], s->copy_in));
    if (serial && c >= 1 && (rc = drain(c - 1)) != GJ_OK) return rc;
    GJ_CUDA(cudaStreamWaitEvent(s->stream, s->ev_in[b], 0));
    if (ids_direct && c >= 3) GJ_CUDA(cudaStreamWaitEvent(s->stream, s->ev_out[b], 0));

    JoinRequest rq{};
    rq.d_pts = s->d_points[b].as<double2>();
    rq.n = len;
    rq.base_index = base_index + begin;
    rq.exact = exact;
    rq.want_stats = stats != nullptr;
    rq.d_counts = s->d_counts.as<unsigned long long>();
    rq.d_stats = s->d_stats.as<unsigned long long>();
    rq.d_first_id = want_ids ? s->d_first_id[b].as<uint32_t>() : nullptr;
    rq.d_status = s->d_status.as<DevStatus>() + b;
    rq.ovf_cap = ovf_cap;
    rq.task_cap = task_cap;
    if ((rc = enqueue_join(s, rq)) != GJ_OK) return rc;
    GJ_CUDA(cudaMemcpyAsync(&s->h_status[b], rq.d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost, s->stream));
    GJ_CUDA(cudaEventRecord(s->ev_done[b], s->stream));
    if (ids_direct) {
      GJ_CUDA(cudaStreamWaitEvent(s->copy_out, s->ev_done[b], 0));
      GJ_CUDA(cudaMemcpyAsync(out_first_id + begin, s->d_first_id[b].ptr, len * 4, cudaMemcpyDeviceToHost, s->copy_out));
      GJ_CUDA(cudaEventRecord(s->ev_out[b], s->copy_out));
    }
  }
  // drain what is still in flight
  const uint64_t first_pending = serial ? (n_chunks ? n_chunks - 1 : 0) : (n_chunks > 3 ? n_chunks - 3 : 0);
  for (uint64_t c = first_pending; c < n_chunks; ++c) {
    if ((rc = drain(c)) != GJ_OK) return rc;
  }
  GJ_CUDA(cudaStreamSynchronize(s->copy_out));
  GJ_CUDA(cudaStreamSynchronize(s->stream));

  final_rc = status_to_code(worst, bad_index);
  if (final_rc != GJ_OK) return final_rc;  // like the reference's throw: no partial results

  std::vector<unsigned long long> h_counts(n_ids + 1);
  unsigned long long h_stats[6];
  GJ_CUDA(cudaMemcpy(h_counts.data(), s->d_counts.ptr, static_cast<size_t>(n_ids) * 8, cudaMemcpyDeviceToHost));
  GJ_CUDA(cudaMemcpy(h_stats, s->d_stats.ptr, sizeof h_stats, cudaMemcpyDeviceToHost));
  if (counts) {
    for (uint32_t i = 0; i < n_ids; ++i) counts[i] += h_counts[i];
  }
  if (stats) {
    stats->probes += h_stats[0];
    stats->pip_tests += h_stats[1];
    stats->false_hits += h_stats[2];
    stats->solely_true_hits += h_stats[3];
    stats->refinement_entered += h_stats[4];
    stats->candidate_refs += h_stats[5];
  }
  return GJ_OK;
}

// join_exact / join_approx materialised as CSR, entirely on the device (see
// the pipeline comment in gj_kernels.cuh).  Chunks are processed one after
// the other; a chunk's pair count is only known after its scan, so the id
// buffer is sized then.
// Grow `buf` to at least `want` bytes keeping its first `keep` bytes.
int grow_keep(gj_session* s, DeviceBuffer& buf, size_t want, size_t keep) {
  if (want <= buf.bytes) return GJ_OK;
  void* fresh = nullptr;
  GJ_CUDA(cudaMalloc(&fresh, want));
  if (keep) {
    cudaError_t e = cudaMemcpyAsync(fresh, buf.ptr, keep, cudaMemcpyDeviceToDevice, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) {
      cudaFree(fresh);
      return cuda_fail(e, "grow_keep");
    }
  }
  buf.release();
  buf.ptr = fresh;
  buf.bytes = want;
  return GJ_OK;
}

// Materialised pairs.  Chunks of points go H2D on the copy stream one chunk
// ahead of the kernels (two point buffers); every chunk's row offsets (with
// the running global base) and polygon ids are appended to session buffers in
// HBM, and gj_pairs_copy later copies them straight into the caller's arrays.
int run_host_pairs(gj_session* s, const double* latlng, uint64_t n, bool exact, gj_stats* stats,
                   uint64_t* bad_index) {
  gj_index& ix = *s->ix;
  GJ_CUDA(cudaSetDevice(ix.device));
  s->pairs_valid = false;
  s->pairs_n = n;
  s->pairs_total = 0;
  const uint64_t max_cand = std::max<uint64_t>(1, ix.max_cand_refs);
  const uint64_t per_point = 48 + (exact ? max_cand * 13 : 0);
  uint64_t chunk = std::min<uint64_t>(4ull << 20, std::max<uint64_t>(4096, kScratchBudget / per_point));
  chunk = std::min<uint64_t>(chunk, std::max<uint64_t>(n, 1));
  const uint64_t task_cap = exact ? chunk * max_cand : 0;
  if (task_cap >= (1ull << 32)) {
    set_error("candidate task capacity exceeds 2^32");
    return GJ_INVALID_ARGUMENT;
  }
  int rc;
  if (exact) {
    if ((rc = reserve_tasks(s, task_cap)) != GJ_OK) return rc;
    GJ_CUDA(s->d_task_pass.reserve(task_cap + 16));
  }
  const uint32_t n_blocks_max = static_cast<uint32_t>((chunk + kScanTile - 1) / kScanTile);
  GJ_CUDA(s->d_points[0].reserve(chunk * 16));
  GJ_CUDA(s->d_points[1].reserve(chunk * 16));
  GJ_CUDA(s->d_entries.reserve(chunk * 8));
  GJ_CUDA(s->d_nrefs.reserve(chunk * 4));
  GJ_CUDA(s->d_task_base.reserve(chunk * 4));
  GJ_CUDA(s->d_pair_count.reserve(chunk * 4));
  GJ_CUDA(s->d_block_sums.reserve((static_cast<size_t>(n_blocks_max) + 2) * 8));
  GJ_CUDA(s->d_stats.reserve(6 * 8));
  GJ_CUDA(s->d_all_row_ptr.reserve((n + 1) * 8));
  GJ_CUDA(s->d_all_ids.reserve(std::max<uint64_t>(n + n / 4, 1024) * 4));  // grows when a chunk needs more
  GJ_CUDA(cudaMemsetAsync(s->d_stats.ptr, 0, 6 * 8, s->stream));
  DevStatus* d_status = s->d_status.as<DevStatus>() + 3;
  const size_t probe_smem = align16(std::max<size_t>(ix.dev.dir.n_table * 4, 16));
  if (int rc_attr = allow_max_smem(ix, probe_points_kernel)) return rc_attr;
  const unsigned wide = static_cast<unsigned>(ix.sm_count) * 8u;
  uint64_t* d_row_all = s->d_all_row_ptr.as<uint64_t>();

  auto copy_in = [&](uint64_t begin, int b) -> int {  // chunk at `begin` -> point buffer b, on the copy stream
    const uint64_t len = std::min(chunk, n - begin);
    GJ_CUDA(cudaStreamWaitEvent(s->copy_in, s->ev_done[b], 0));  // the kernels that read buffer b last
    GJ_CUDA(stager_of(s).to_device(s->d_points[b].ptr, latlng + 2 * begin, len * 16, s->copy_in));
    GJ_CUDA(cudaEventRecord(s->ev_in[b], s->copy_in));
    return GJ_OK;
  };
  GJ_CUDA(cudaEventRecord(s->ev_done[0], s->stream));
  GJ_CUDA(cudaEventRecord(s->ev_done[1], s->stream));
  if (n && (rc = copy_in(0, 0)) != GJ_OK) return rc;

  uint64_t id_base = 0;
  int b = 0;
  for (uint64_t begin = 0; begin < n; begin += chunk, b ^= 1) {
    const uint64_t len = std::min(chunk, n - begin);
    const uint32_t n_blocks = static_cast<uint32_t>((len + kScanTile - 1) / kScanTile);
    GJ_CUDA(cudaStreamWaitEvent(s->stream, s->ev_in[b], 0));
    if ((rc = reset_status(s, d_status)) != GJ_OK) return rc;
    const double2* d_pts = s->d_points[b].as<double2>();
    probe_points_kernel<<<static_cast<unsigned>(std::min<uint64_t>((len + 255) / 256, ix.sm_count * 4ull)), 256,
                          probe_smem, s->stream>>>(ix.dev, d_pts, len, begin, s->d_entries.as<uint64_t>(), d_status);
    PairsParams pp{};
    pp.entries = s->d_entries.as<uint64_t>();
    pp.n = len;
    pp.base_index = begin;
    pp.n_refs = s->d_nrefs.as<uint32_t>();
    pp.task_base = s->d_task_base.as<uint32_t>();
    pp.task_point = s->d_task_point.as<uint32_t>();
    pp.task_slot = s->d_task_slot.as<uint32_t>();
    pp.task_ord = s->d_task_ord.as<uint32_t>();
    pp.task_cap = task_cap;
    pp.task_pass = s->d_task_pass.as<uint8_t>();
    pp.count = s->d_pair_count.as<uint32_t>();
    pp.row_ptr = d_row_all + begin;
    pp.stats = stats ? s->d_stats.as<unsigned long long>() : nullptr;
    pp.status = d_status;
    pp.exact = exact ? 1 : 0;
    pairs_plan_kernel<<<wide, 256, 0, s->stream>>>(ix.dev, pp);
    s->launches += 2;
    if (exact) {
      RefineParams rp{};
      rp.pts = d_pts;
      rp.base_index = begin;
      rp.task_point = pp.task_point;
      rp.task_slot = pp.task_slot;
      rp.task_ord = pp.task_ord;
      rp.task_cap = task_cap;
      rp.task_pass = s->d_task_pass.as<uint8_t>();
      rp.status = d_status;
      if ((rc = launch_refine(s, rp, 0)) != GJ_OK) return rc;
    }
    GJ_CUDA(cudaEventRecord(s->ev_done[b], s->stream));  // the point buffer is free again
    pairs_emit_kernel<false><<<wide, 256, 0, s->stream>>>(ix.dev, pp);
    scan_block_sums_kernel<<<n_blocks, kScanThreads, 0, s->stream>>>(pp.count, len, s->d_block_sums.as<uint64_t>());
    uint64_t* d_total = s->d_block_sums.as<uint64_t>() + n_blocks_max + 1;
    scan_sums_kernel<<<1, kScanThreads, 0, s->stream>>>(s->d_block_sums.as<uint64_t>(), n_blocks, d_total);
    scan_apply_kernel<<<n_blocks, kScanThreads, 0, s->stream>>>(pp.count, len, s->d_block_sums.as<uint64_t>(), id_base,
                                                                d_row_all + begin, nullptr, true);
    s->launches += 4;
    GJ_CUDA(cudaGetLastError());
    // stage the next chunk's points while the device works on this one
    if (begin + chunk < n && (rc = copy_in(begin + chunk, b ^ 1)) != GJ_OK) return rc;
    uint64_t total = 0;
    GJ_CUDA(cudaMemcpyAsync(&total, d_total, 8, cudaMemcpyDeviceToHost, s->stream));
    GJ_CUDA(cudaMemcpyAsync(&s->h_status[3], d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost, s->stream));
    GJ_CUDA(cudaStreamSynchronize(s->stream));
    if ((rc = status_to_code(s->h_status[3], bad_index)) != GJ_OK) return rc;
    if ((id_base + total) * 4 > s->d_all_ids.bytes) {  // at least double, so appends stay amortised
      const size_t want = std::max<size_t>((id_base + total) * 4, s->d_all_ids.bytes * 2);
      if ((rc = grow_keep(s, s->d_all_ids, want, id_base * 4)) != GJ_OK) return rc;
    }
    pp.out_id = s->d_all_ids.as<uint32_t>();  // row_ptr already carries the global base
    pp.out_cap = s->d_all_ids.bytes / 4;
    pp.out_sub = nullptr;
    pairs_emit_kernel<true><<<wide, 256, 0, s->stream>>>(ix.dev, pp);
    ++s->launches;
    GJ_CUDA(cudaGetLastError());
    id_base += total;
  }
  GJ_CUDA(cudaMemcpyAsync(d_row_all + n, &id_base, 8, cudaMemcpyHostToDevice, s->stream));
  GJ_CUDA(cudaStreamSynchronize(s->stream));
  s->pairs_total = id_base;
  s->pairs_valid = true;
  if (stats) {
    unsigned long long h_stats[6];
    GJ_CUDA(cudaMemcpy(h_stats, s->d_stats.ptr, sizeof h_stats, cudaMemcpyDeviceToHost));
    stats->probes += h_stats[0];
    stats->pip_tests += h_stats[1];
    stats->false_hits += h_stats[2];
    stats->solely_true_hits += h_stats[3];
    stats->refinement_entered += h_stats[4];
    stats->candidate_refs += h_stats[5];
  }
  return GJ_OK;
}


// Where run_pairs_async leaves the CSR: the caller's device arrays (row offsets and ids at their global positions),
// or the caller's host arrays, streamed chunk by chunk while the next chunk runs.
struct PairsSink {
  uint64_t* d_row_ptr = nullptr;  // device output: [n + 1]
  uint32_t* d_ids = nullptr;      //                [ids_cap]
  uint64_t* h_row_ptr = nullptr;  // host output:   [n + 1]
  uint32_t* h_ids = nullptr;      //                [ids_cap]
  uint64_t ids_cap = 0;
};

// join_exact / join_approx -> CSR without a host round trip per chunk: the pair count so far lives on the device
// (the scan of a chunk starts from it, a one-thread kernel advances it), the capacity of the id array is checked
// by the fill kernel, and — host output — chunk c's rows and ids travel D2H on the copy-out stream while chunk
// c + 1 runs.  `src` is device memory when `src_on_device`, else host memory copied one chunk ahead.
int run_pairs_async(gj_session* s, const double* src, bool src_on_device, uint64_t n, bool exact, gj_stats* stats,
                    const PairsSink& sink, uint64_t* n_pairs, uint64_t* bad_index) {
  gj_index& ix = *s->ix;
  GJ_CUDA(cudaSetDevice(ix.device));
  const bool to_host = sink.h_row_ptr != nullptr;
  const uint64_t max_cand = std::max<uint64_t>(1, ix.max_cand_refs);
  const uint64_t max_refs = std::max<uint64_t>(1, ix.max_refs);
  const uint64_t per_point = 48 + (exact ? max_cand * 13 : 0);
  uint64_t chunk = std::min<uint64_t>(ix.opt.chunk_points ? std::max<uint64_t>(4096, ix.opt.chunk_points) : 4ull << 20,
                                      std::max<uint64_t>(4096, kScratchBudget / per_point));
  if (to_host) chunk = std::min<uint64_t>(chunk, std::max<uint64_t>(4096, (768ull << 20) / (max_refs * 4)));  // chunk-local ids
  chunk = std::min<uint64_t>(chunk, std::max<uint64_t>(n, 1));
  const uint64_t task_cap = exact ? chunk * max_cand : 0;
  if (task_cap >= (1ull << 32)) {
    set_error("candidate task capacity exceeds 2^32");
    return GJ_INVALID_ARGUMENT;
  }
  int rc;
  if (exact) {
    if ((rc = reserve_tasks(s, task_cap)) != GJ_OK) return rc;
    GJ_CUDA(s->d_task_pass.reserve(task_cap + 16));
  }
  const uint32_t n_blocks_max = static_cast<uint32_t>((chunk + kScanTile - 1) / kScanTile);
  if (!src_on_device) {
    GJ_CUDA(s->d_points[0].reserve(chunk * 16));
    GJ_CUDA(s->d_points[1].reserve(chunk * 16));
  }
  GJ_CUDA(s->d_entries.reserve(chunk * 8));
  GJ_CUDA(s->d_nrefs.reserve(chunk * 4));
  GJ_CUDA(s->d_task_base.reserve(chunk * 4));
  GJ_CUDA(s->d_pair_count.reserve(chunk * 4));
  GJ_CUDA(s->d_block_sums.reserve((static_cast<size_t>(n_blocks_max) + 2) * 8));
  GJ_CUDA(s->d_stats.reserve(6 * 8));
  GJ_CUDA(s->d_pairs_base.reserve(16));
  const uint64_t chunk_ids = chunk * max_refs;
  if (to_host) {
    for (int b = 0; b < 2; ++b) {
      GJ_CUDA(s->d_chunk_rows[b].reserve((chunk + 1) * 8));
      GJ_CUDA(s->d_chunk_ids[b].reserve(chunk_ids * 4 + 16));
    }
  }
  uint64_t* d_base = s->d_pairs_base.as<uint64_t>();
  GJ_CUDA(cudaMemsetAsync(d_base, 0, 16, s->stream));
  GJ_CUDA(cudaMemsetAsync(s->d_stats.ptr, 0, 6 * 8, s->stream));
  DevStatus* d_status = s->d_status.as<DevStatus>() + 3;
  if ((rc = reset_status(s, d_status)) != GJ_OK) return rc;
  const size_t probe_smem = align16(std::max<size_t>(ix.dev.dir.n_table * 4, 16));
  if (int rc_attr = allow_max_smem(ix, probe_points_kernel)) return rc_attr;
  const unsigned wide = static_cast<unsigned>(ix.sm_count) * 8u;
  uint64_t* h_total = reinterpret_cast<uint64_t*>(s->h_status + 4);  // pinned: [2] chunk totals (host output)

  auto copy_in = [&](uint64_t begin, int b) -> int {  // host chunk at `begin` -> point buffer b, on the copy stream
    const uint64_t len = std::min(chunk, n - begin);
    GJ_CUDA(cudaStreamWaitEvent(s->copy_in, s->ev_done[b], 0));  // the kernels that read buffer b last
    GJ_CUDA(stager_of(s).to_device(s->d_points[b].ptr, src + 2 * begin, len * 16, s->copy_in));
    GJ_CUDA(cudaEventRecord(s->ev_in[b], s->copy_in));
    return GJ_OK;
  };
  GJ_CUDA(cudaEventRecord(s->ev_done[0], s->stream));
  GJ_CUDA(cudaEventRecord(s->ev_done[1], s->stream));
  GJ_CUDA(cudaEventRecord(s->ev_out[0], s->copy_out));
  GJ_CUDA(cudaEventRecord(s->ev_out[1], s->copy_out));
  if (!src_on_device && n && (rc = copy_in(0, 0)) != GJ_OK) return rc;

  uint64_t host_base = 0;     // pairs of the chunks already handed to the copy-out stream
  bool host_full = false;     // the caller's id array ran out: rows still come back, ids stop
  auto copy_out = [&](uint64_t begin, int b) -> int {  // host output: chunk at `begin` (buffers b) -> the caller's arrays
    const uint64_t len = std::min(chunk, n - begin);
    GJ_CUDA(cudaEventSynchronize(s->ev_total[b]));  // its pair count is on the host
    const uint64_t total = h_total[b];
    GJ_CUDA(cudaStreamWaitEvent(s->copy_out, s->ev_total[b], 0));
    GJ_CUDA(stager_of(s).to_host_async(sink.h_row_ptr + begin, s->d_chunk_rows[b].ptr, len * 8, s->copy_out));
    if (host_base + total > sink.ids_cap) host_full = true;
    if (!host_full && total) {
      GJ_CUDA(stager_of(s).to_host_async(sink.h_ids + host_base, s->d_chunk_ids[b].ptr, total * 4, s->copy_out));
    }
    GJ_CUDA(cudaEventRecord(s->ev_out[b], s->copy_out));
    host_base += total;
    return GJ_OK;
  };

  int b = 0;
  for (uint64_t begin = 0; begin < n; begin += chunk, b ^= 1) {
    const uint64_t len = std::min(chunk, n - begin);
    const uint32_t n_blocks = static_cast<uint32_t>((len + kScanTile - 1) / kScanTile);
    const double2* d_pts;
    if (src_on_device) {
      d_pts = reinterpret_cast<const double2*>(src) + begin;
    } else {
      GJ_CUDA(cudaStreamWaitEvent(s->stream, s->ev_in[b], 0));
      d_pts = s->d_points[b].as<double2>();
    }
    if (to_host) GJ_CUDA(cudaStreamWaitEvent(s->stream, s->ev_out[b], 0));  // chunk c - 2 has left these buffers
    GJ_CUDA(cudaMemsetAsync(&d_status->task_count, 0, sizeof(unsigned long long), s->stream));
    probe_points_kernel<<<static_cast<unsigned>(std::min<uint64_t>((len + 255) / 256, ix.sm_count * 4ull)), 256,
                          probe_smem, s->stream>>>(ix.dev, d_pts, len, begin, s->d_entries.as<uint64_t>(), d_status);
    uint64_t* d_rows = to_host ? s->d_chunk_rows[b].as<uint64_t>() : sink.d_row_ptr + begin;
    PairsParams pp{};
    pp.entries = s->d_entries.as<uint64_t>();
    pp.n = len;
    pp.base_index = begin;
    pp.n_refs = s->d_nrefs.as<uint32_t>();
    pp.task_base = s->d_task_base.as<uint32_t>();
    pp.task_point = s->d_task_point.as<uint32_t>();
    pp.task_slot = s->d_task_slot.as<uint32_t>();
    pp.task_ord = s->d_task_ord.as<uint32_t>();
    pp.task_cap = task_cap;
    pp.task_pass = s->d_task_pass.as<uint8_t>();
    pp.count = s->d_pair_count.as<uint32_t>();
    pp.row_ptr = d_rows;
    pp.out_id = to_host ? s->d_chunk_ids[b].as<uint32_t>() : sink.d_ids;
    pp.out_cap = to_host ? chunk_ids : sink.ids_cap;
    pp.out_sub = to_host ? d_base : nullptr;
    pp.stats = stats ? s->d_stats.as<unsigned long long>() : nullptr;
    pp.status = d_status;
    pp.exact = exact ? 1 : 0;
    pairs_plan_kernel<<<wide, 256, 0, s->stream>>>(ix.dev, pp);
    s->launches += 2;
    if (exact) {
      RefineParams rp{};
      rp.pts = d_pts;
      rp.base_index = begin;
      rp.task_point = pp.task_point;
      rp.task_slot = pp.task_slot;
      rp.task_ord = pp.task_ord;
      rp.task_cap = task_cap;
      rp.task_pass = s->d_task_pass.as<uint8_t>();
      rp.status = d_status;
      if ((rc = launch_refine(s, rp, 0)) != GJ_OK) return rc;
    }
    if (!src_on_device) GJ_CUDA(cudaEventRecord(s->ev_done[b], s->stream));  // the point buffer is free again
    uint64_t* d_sums = s->d_block_sums.as<uint64_t>();
    uint64_t* d_total = d_sums + n_blocks_max + 1;
    pairs_emit_kernel<false><<<wide, 256, 0, s->stream>>>(ix.dev, pp);
    scan_block_sums_kernel<<<n_blocks, kScanThreads, 0, s->stream>>>(pp.count, len, d_sums);
    scan_sums_kernel<<<1, kScanThreads, 0, s->stream>>>(d_sums, n_blocks, d_total);
    scan_apply_kernel<<<n_blocks, kScanThreads, 0, s->stream>>>(pp.count, len, d_sums, 0, d_rows, d_base, true);
    pairs_emit_kernel<true><<<wide, 256, 0, s->stream>>>(ix.dev, pp);
    if (to_host) GJ_CUDA(cudaMemcpyAsync(&h_total[b], d_total, 8, cudaMemcpyDeviceToHost, s->stream));
    advance_base_kernel<<<1, 1, 0, s->stream>>>(d_base, d_total);
    s->launches += 6;
    GJ_CUDA(cudaGetLastError());
    if (to_host) GJ_CUDA(cudaEventRecord(s->ev_total[b], s->stream));
    // stage the next chunk's points, then send the previous chunk's results home, while the device works on this one
    if (!src_on_device && begin + chunk < n && (rc = copy_in(begin + chunk, b ^ 1)) != GJ_OK) return rc;
    if (to_host && begin != 0 && (rc = copy_out(begin - chunk, b ^ 1)) != GJ_OK) return rc;
  }
  if (to_host && n) {  // the last chunk
    const uint64_t last = (n - 1) / chunk * chunk;
    if ((rc = copy_out(last, static_cast<int>((last / chunk) & 1))) != GJ_OK) return rc;
  }
  uint64_t total = 0;
  GJ_CUDA(cudaMemcpyAsync(&s->h_status[3], d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost, s->stream));
  GJ_CUDA(cudaMemcpyAsync(&h_total[0], d_base, 8, cudaMemcpyDeviceToHost, s->stream));
  GJ_CUDA(cudaStreamSynchronize(s->stream));
  total = h_total[0];
  if (to_host) {
    GJ_CUDA(stager_of(s).drain());
    GJ_CUDA(cudaStreamSynchronize(s->copy_out));
    sink.h_row_ptr[n] = total;
  } else if (n == 0) {
    GJ_CUDA(cudaMemsetAsync(sink.d_row_ptr, 0, 8, s->stream));
    GJ_CUDA(cudaStreamSynchronize(s->stream));
  }
  if (n_pairs) *n_pairs = total;
  DevStatus st = s->h_status[3];
  const bool ids_short = (st.flags & kErrOverflowCap) != 0 || host_full || total > sink.ids_cap;
  st.flags &= ~kErrOverflowCap;
  if ((rc = status_to_code(st, bad_index)) != GJ_OK) return rc;
  if (stats) {
    unsigned long long h_stats[6];
    GJ_CUDA(cudaMemcpy(h_stats, s->d_stats.ptr, sizeof h_stats, cudaMemcpyDeviceToHost));
    stats->probes += h_stats[0];
    stats->pip_tests += h_stats[1];
    stats->false_hits += h_stats[2];
    stats->solely_true_hits += h_stats[3];
    stats->refinement_entered += h_stats[4];
    stats->candidate_refs += h_stats[5];
  }
  if (ids_short) {
    set_error("polygon id array too small for the join's pairs (n_pairs holds the size needed)");
    return GJ_CAPACITY;
  }
  return GJ_OK;
}

}  // namespace
}  // namespace gj

using namespace gj;

extern "C" {

const char* gj_last_error(void) { return last_error().c_str(); }

int gj_device_count(void) {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess ? n : 0;
}

void gj_options_default(gj_options* opt) {
  if (opt) *opt = default_options();
}

int gj_index_create(const gj_index_desc* desc, int device, gj_index** out) {
  return gj_index_create_ex(desc, device, nullptr, out);
}

int gj_index_create_ex(const gj_index_desc* desc, int device, const gj_options* opt, gj_index** out) {
  if (!desc) return GJ_INVALID_ARGUMENT;
  return create_index(*desc, device, opt, out);
}

int gj_index_load_file(const char* path, int device, gj_index** out) {
  return load_index_file(path, device, nullptr, out);
}

int gj_index_load_file_ex(const char* path, int device, const gj_options* opt, gj_index** out) {
  return load_index_file(path, device, opt, out);
}

int gj_index_replicate(const gj_index* src, int device, gj_index** out) {
  if (!src) return GJ_INVALID_ARGUMENT;
  return replicate_index(*src, device, out);
}

void gj_index_destroy(gj_index* ix) {
  if (!ix) return;
  cudaSetDevice(ix->device);
  delete ix;
}

int gj_index_get_info(const gj_index* ix, gj_index_info* info) {
  if (!ix || !info) return GJ_INVALID_ARGUMENT;
  *info = ix->info;
  return GJ_OK;
}

int gj_index_ids(const gj_index* ix, uint32_t* ids) {
  if (!ix || (!ids && !ix->ids.empty())) return GJ_INVALID_ARGUMENT;
  std::copy(ix->ids.begin(), ix->ids.end(), ids);
  return GJ_OK;
}

int gj_session_create(gj_index* ix, gj_session** out) {
  if (!ix || !out) return GJ_INVALID_ARGUMENT;
  *out = nullptr;
  GJ_CUDA(cudaSetDevice(ix->device));
  std::unique_ptr<gj_session> s(new gj_session);
  s->ix = ix;
  GJ_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  GJ_CUDA(cudaStreamCreateWithFlags(&s->copy_in, cudaStreamNonBlocking));
  GJ_CUDA(cudaStreamCreateWithFlags(&s->copy_out, cudaStreamNonBlocking));
  for (int b = 0; b < 3; ++b) {
    GJ_CUDA(cudaEventCreateWithFlags(&s->ev_in[b], cudaEventDisableTiming));
    GJ_CUDA(cudaEventCreateWithFlags(&s->ev_done[b], cudaEventDisableTiming));
    GJ_CUDA(cudaEventCreateWithFlags(&s->ev_out[b], cudaEventDisableTiming));
    GJ_CUDA(cudaEventCreateWithFlags(&s->ev_total[b], cudaEventDisableTiming));
  }
  GJ_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s->h_status), 5 * sizeof(DevStatus), cudaHostAllocDefault));  // [4]: scratch words
  GJ_CUDA(s->d_status.reserve(4 * sizeof(DevStatus)));
  // No L2 persistence window for the second directory tier: it is hot enough
  // to stay resident by itself (98 % hit rate with and without a window), and a
  // persisting carve-out is a device-wide limit that takes L2 away from
  // everything else (a 70 MB carve-out made K1 1.5x slower).
  *out = s.release();
  return GJ_OK;
}

void gj_session_destroy(gj_session* s) {
  if (!s) return;
  cudaSetDevice(s->ix->device);
  cudaStreamSynchronize(s->stream);
  cudaStreamSynchronize(s->copy_in);
  cudaStreamSynchronize(s->copy_out);
  for (int b = 0; b < 3; ++b) {
    if (s->ev_in[b]) cudaEventDestroy(s->ev_in[b]);
    if (s->ev_done[b]) cudaEventDestroy(s->ev_done[b]);
    if (s->ev_out[b]) cudaEventDestroy(s->ev_out[b]);
    if (s->ev_total[b]) cudaEventDestroy(s->ev_total[b]);
  }
  if (s->h_status) cudaFreeHost(s->h_status);
  cudaStreamDestroy(s->stream);
  cudaStreamDestroy(s->copy_in);
  cudaStreamDestroy(s->copy_out);
  delete s;
}

void* gj_session_stream(gj_session* s) { return s ? s->stream : nullptr; }
uint64_t gj_session_launches(const gj_session* s) { return s ? s->launches : 0; }

void* gj_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {  // pinned for every GPU of a group
    cuda_fail(cudaGetLastError(), "cudaHostAlloc");
    return nullptr;
  }
  return p;
}

void gj_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int gj_probe_points_host(gj_session* s, const double* latlng, uint64_t n, uint64_t* out_entries,
                         uint64_t* bad_index) {
  if (!s || (n && (!latlng || !out_entries))) return GJ_INVALID_ARGUMENT;
  gj_index& ix = *s->ix;
  GJ_CUDA(cudaSetDevice(ix.device));
  const uint64_t chunk = 4ull << 20;
  GJ_CUDA(s->d_points[0].reserve(std::min(chunk, std::max<uint64_t>(n, 1)) * 16));
  GJ_CUDA(s->d_entries.reserve(std::min(chunk, std::max<uint64_t>(n, 1)) * 8));
  DevStatus* d_status = s->d_status.as<DevStatus>() + 3;
  int rc = reset_status(s, d_status);
  if (rc != GJ_OK) return rc;
  const size_t smem = align16(std::max<size_t>(ix.dev.dir.n_table * 4, 16));
  if (int rc_attr = allow_max_smem(ix, probe_points_kernel)) return rc_attr;
  for (uint64_t begin = 0; begin < n; begin += chunk) {
    const uint64_t len = std::min(chunk, n - begin);
    GJ_CUDA(cudaMemcpyAsync(s->d_points[0].ptr, latlng + 2 * begin, len * 16, cudaMemcpyHostToDevice, s->stream));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((len + 255) / 256, ix.sm_count * 4ull));
    probe_points_kernel<<<grid, 256, smem, s->stream>>>(ix.dev, s->d_points[0].as<double2>(), len, begin,
                                                        s->d_entries.as<uint64_t>(), d_status);
    ++s->launches;
    GJ_CUDA(cudaGetLastError());
    GJ_CUDA(cudaMemcpyAsync(out_entries + begin, s->d_entries.ptr, len * 8, cudaMemcpyDeviceToHost, s->stream));
    GJ_CUDA(cudaStreamSynchronize(s->stream));
  }
  GJ_CUDA(cudaMemcpyAsync(&s->h_status[3], d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost, s->stream));
  GJ_CUDA(cudaStreamSynchronize(s->stream));
  return status_to_code(s->h_status[3], bad_index);
}

int gj_points_from_csv_host(gj_session* s, const char* text, uint64_t n_bytes, const char* lat_column,
                            const char* lng_column, int strict, double* out_latlng, uint64_t cap, uint64_t* n_points,
                            uint64_t* n_skipped, uint64_t* bad_line) {
  if (!s || !lat_column || !lng_column || !n_points || !n_skipped || (n_bytes && !text) || (cap && !out_latlng)) {
    return GJ_INVALID_ARGUMENT;
  }
  *n_points = 0;
  *n_skipped = 0;
  if (bad_line) *bad_line = 0;
  if (n_bytes == 0) {  // csv.cpp:58-60
    set_error("point file is empty, expected a CSV header");
    return GJ_DATA_ERROR;
  }
  // ---- header, on the host (csv.cpp:54-78) ----
  const char* end = text + n_bytes;
  const char* nl = static_cast<const char*>(std::memchr(text, '\n', n_bytes));
  const char* header_end = nl ? nl : end;
  const char* data = nl ? nl + 1 : end;
  if (header_end != text && header_end[-1] == '\r') --header_end;  // read_line, csv.cpp:47-51
  const std::string lat_name(lat_column), lng_name(lng_column);
  uint32_t lat_index = 0, lng_index = 0, column = 0;
  bool lat_found = false, lng_found = false;
  for (const char* field = text;; ++column) {  // split_row, csv.cpp:26-37
    const char* comma = static_cast<const char*>(std::memchr(field, ',', static_cast<size_t>(header_end - field)));
    const char* field_end = comma ? comma : header_end;
    const std::string name(field, field_end);
    if (name == lat_name) {  // a later duplicate wins; lat is tested first (csv.cpp:64-72)
      lat_index = column;
      lat_found = true;
    } else if (name == lng_name) {
      lng_index = column;
      lng_found = true;
    }
    if (!comma) break;
    field = comma + 1;
  }
  if (!lat_found || !lng_found) {
    set_error("CSV header is missing column '" + (lat_found ? lng_name : lat_name) + "'");
    if (bad_line) *bad_line = 1;
    return GJ_DATA_ERROR;
  }

  gj_index& ix = *s->ix;
  GJ_CUDA(cudaSetDevice(ix.device));
  GJ_CUDA(s->d_csv_meta.reserve(16));
  unsigned long long* d_skipped = s->d_csv_meta.as<unsigned long long>();
  unsigned long long* d_first_bad = d_skipped + 1;
  const unsigned wide = static_cast<unsigned>(ix.sm_count) * 8u;
  constexpr uint64_t kChunkBytes = 64ull << 20;
  uint64_t found = 0, skipped = 0, lines_before = 0;  // data lines in earlier chunks
  for (const char* chunk = data; chunk != end;) {
    // a chunk ends just past a newline (or at the end of the text)
    const char* chunk_end = end;
    if (static_cast<uint64_t>(end - chunk) > kChunkBytes) {
      const char* back = static_cast<const char*>(memrchr(chunk, '\n', kChunkBytes));
      const char* fwd = back ? back : static_cast<const char*>(std::memchr(chunk + kChunkBytes, '\n',
                                                                            static_cast<size_t>(end - chunk - kChunkBytes)));
      chunk_end = fwd ? fwd + 1 : end;
    }
    const uint64_t len = static_cast<uint64_t>(chunk_end - chunk);
    const uint64_t n_pieces = (len + 15) / 16;
    const uint32_t piece_blocks = static_cast<uint32_t>((n_pieces + kScanTile - 1) / kScanTile);
    GJ_CUDA(s->d_csv_text.reserve(n_pieces * 16 + 16));
    GJ_CUDA(s->d_csv_counts.reserve(n_pieces * 4));
    GJ_CUDA(s->d_csv_offsets.reserve((n_pieces + 1) * 8));
    GJ_CUDA(s->d_block_sums.reserve((static_cast<size_t>(piece_blocks) + 2) * 8));
    char* d_text = s->d_csv_text.as<char>();
    GJ_CUDA(stager_of(s).to_device(d_text, chunk, len, s->stream));
    uint64_t* d_sums = s->d_block_sums.as<uint64_t>();
    uint64_t* d_total = d_sums + piece_blocks + 1;
    csv_count_newlines_kernel<<<wide, 256, 0, s->stream>>>(d_text, len, s->d_csv_counts.as<uint32_t>());
    scan_block_sums_kernel<<<piece_blocks, kScanThreads, 0, s->stream>>>(s->d_csv_counts.as<uint32_t>(), n_pieces, d_sums);
    scan_sums_kernel<<<1, kScanThreads, 0, s->stream>>>(d_sums, piece_blocks, d_total);
    scan_apply_kernel<<<piece_blocks, kScanThreads, 0, s->stream>>>(s->d_csv_counts.as<uint32_t>(), n_pieces, d_sums, 0,
                                                                    s->d_csv_offsets.as<uint64_t>());
    s->launches += 4;
    GJ_CUDA(cudaGetLastError());
    uint64_t n_newlines = 0;
    GJ_CUDA(cudaMemcpyAsync(&n_newlines, d_total, 8, cudaMemcpyDeviceToHost, s->stream));
    GJ_CUDA(cudaStreamSynchronize(s->stream));
    const bool open_last = chunk_end[-1] != '\n';  // only the last chunk can end without a newline
    const uint64_t n_lines = n_newlines + (open_last ? 1 : 0);
    const uint32_t line_blocks = static_cast<uint32_t>((n_lines + kScanTile - 1) / kScanTile);
    GJ_CUDA(s->d_csv_lines.reserve((n_lines + 2) * 8));
    GJ_CUDA(s->d_csv_status.reserve(n_lines * 4 + 16));
    GJ_CUDA(s->d_csv_valid.reserve(n_lines * 4 + 16));
    GJ_CUDA(s->d_csv_points.reserve(n_lines * 16 + 16));
    GJ_CUDA(s->d_row_ptr.reserve((n_lines + 1) * 8));
    GJ_CUDA(s->d_block_sums.reserve((static_cast<size_t>(std::max(piece_blocks, line_blocks)) + 2) * 8));
    d_sums = s->d_block_sums.as<uint64_t>();
    uint64_t* d_lines = s->d_csv_lines.as<uint64_t>();
    const uint64_t edge[2] = {0, len + 1};  // start of line 0; the end sentinel of an unterminated last line
    GJ_CUDA(cudaMemcpyAsync(d_lines, &edge[0], 8, cudaMemcpyHostToDevice, s->stream));
    if (open_last) GJ_CUDA(cudaMemcpyAsync(d_lines + n_lines, &edge[1], 8, cudaMemcpyHostToDevice, s->stream));
    const unsigned long long meta[2] = {0ull, ~0ull};
    GJ_CUDA(cudaMemcpyAsync(d_skipped, meta, 16, cudaMemcpyHostToDevice, s->stream));
    csv_line_starts_kernel<<<wide, 256, 0, s->stream>>>(d_text, len, s->d_csv_offsets.as<uint64_t>(), d_lines);
    CsvParams cp{};
    cp.text = d_text;
    cp.n_bytes = len;
    cp.line_start = d_lines;
    cp.n_lines = n_lines;
    cp.lat_index = lat_index;
    cp.lng_index = lng_index;
    cp.status = s->d_csv_status.as<uint32_t>();
    cp.valid = s->d_csv_valid.as<uint32_t>();
    cp.point = s->d_csv_points.as<double2>();
    cp.n_skipped = d_skipped;
    cp.first_bad = d_first_bad;
    uint64_t n_valid = 0;
    unsigned long long h_meta[2] = {0, ~0ull};
    if (n_lines) {
      uint64_t* d_vtotal = d_sums + line_blocks + 1;
      csv_parse_rows_kernel<<<wide, 128, 0, s->stream>>>(cp);
      scan_block_sums_kernel<<<line_blocks, kScanThreads, 0, s->stream>>>(cp.valid, n_lines, d_sums);
      scan_sums_kernel<<<1, kScanThreads, 0, s->stream>>>(d_sums, line_blocks, d_vtotal);
      scan_apply_kernel<<<line_blocks, kScanThreads, 0, s->stream>>>(cp.valid, n_lines, d_sums, 0,
                                                                     s->d_row_ptr.as<uint64_t>());
      s->launches += 5;
      GJ_CUDA(cudaGetLastError());
      GJ_CUDA(cudaMemcpyAsync(&n_valid, d_vtotal, 8, cudaMemcpyDeviceToHost, s->stream));
      GJ_CUDA(cudaMemcpyAsync(h_meta, d_skipped, 16, cudaMemcpyDeviceToHost, s->stream));
      GJ_CUDA(cudaStreamSynchronize(s->stream));
    }
    if (strict && h_meta[1] != ~0ull) {  // csv.cpp:91-94; the header is line 1
      if (bad_line) *bad_line = lines_before + h_meta[1] + 2;
      set_error("line " + std::to_string(lines_before + h_meta[1] + 2) + ": invalid point row");
      return GJ_DATA_ERROR;
    }
    if (n_valid) {
      GJ_CUDA(s->d_csv_out.reserve(n_valid * 16));
      csv_scatter_kernel<<<wide, 256, 0, s->stream>>>(cp.valid, s->d_row_ptr.as<uint64_t>(), cp.point, n_lines,
                                                      s->d_csv_out.as<double2>());
      ++s->launches;
      GJ_CUDA(cudaGetLastError());
      const uint64_t room = cap > found ? cap - found : 0;
      const uint64_t take = std::min(n_valid, room);
      if (take) GJ_CUDA(stager_of(s).to_host(out_latlng + 2 * found, s->d_csv_out.ptr, take * 16, s->stream));
      GJ_CUDA(cudaStreamSynchronize(s->stream));
    }
    found += n_valid;
    skipped += h_meta[0];
    lines_before += n_lines;
    chunk = chunk_end;
  }
  *n_points = found;
  *n_skipped = skipped;
  return GJ_OK;
}

int gj_training_candidates_host(gj_session* s, const double* latlng, uint64_t n, uint64_t base_index,
                                uint64_t* out_indices, uint64_t cap, uint64_t* n_candidates, uint64_t* bad_index) {
  if (!s || !n_candidates || (n && !latlng) || (cap && !out_indices)) return GJ_INVALID_ARGUMENT;
  *n_candidates = 0;
  gj_index& ix = *s->ix;
  GJ_CUDA(cudaSetDevice(ix.device));
  const uint64_t chunk = std::min<uint64_t>(4ull << 20, std::max<uint64_t>(n, 1));
  const uint32_t n_blocks_max = static_cast<uint32_t>((chunk + kScanTile - 1) / kScanTile);
  GJ_CUDA(s->d_points[0].reserve(chunk * 16));
  GJ_CUDA(s->d_pair_count.reserve(chunk * 4));
  GJ_CUDA(s->d_row_ptr.reserve((chunk + 1) * 8));
  GJ_CUDA(s->d_entries.reserve(chunk * 8));  // the ordered indices of one chunk
  GJ_CUDA(s->d_block_sums.reserve((static_cast<size_t>(n_blocks_max) + 2) * 8));
  DevStatus* d_status = s->d_status.as<DevStatus>() + 3;
  int rc = reset_status(s, d_status);
  if (rc != GJ_OK) return rc;
  const size_t smem = align16(std::max<size_t>(ix.dev.dir.n_table * 4, 16));
  if (int rc_attr = allow_max_smem(ix, candidate_flags_kernel)) return rc_attr;
  uint64_t found = 0;
  for (uint64_t begin = 0; begin < n; begin += chunk) {
    const uint64_t len = std::min(chunk, n - begin);
    const uint32_t n_blocks = static_cast<uint32_t>((len + kScanTile - 1) / kScanTile);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((len + 255) / 256, ix.sm_count * 4ull));
    uint32_t* d_flags = s->d_pair_count.as<uint32_t>();
    uint64_t* d_sums = s->d_block_sums.as<uint64_t>();
    uint64_t* d_total = d_sums + n_blocks_max + 1;
    GJ_CUDA(cudaMemcpyAsync(s->d_points[0].ptr, latlng + 2 * begin, len * 16, cudaMemcpyHostToDevice, s->stream));
    candidate_flags_kernel<<<grid, 256, smem, s->stream>>>(ix.dev, s->d_points[0].as<double2>(), len,
                                                           base_index + begin, d_flags, d_status);
    scan_block_sums_kernel<<<n_blocks, kScanThreads, 0, s->stream>>>(d_flags, len, d_sums);
    scan_sums_kernel<<<1, kScanThreads, 0, s->stream>>>(d_sums, n_blocks, d_total);
    scan_apply_kernel<<<n_blocks, kScanThreads, 0, s->stream>>>(d_flags, len, d_sums, 0, s->d_row_ptr.as<uint64_t>());
    candidate_scatter_kernel<<<grid, 256, 0, s->stream>>>(d_flags, s->d_row_ptr.as<uint64_t>(), len,
                                                          base_index + begin, s->d_entries.as<uint64_t>());
    s->launches += 5;
    GJ_CUDA(cudaGetLastError());
    uint64_t total = 0;
    GJ_CUDA(cudaMemcpyAsync(&total, d_total, 8, cudaMemcpyDeviceToHost, s->stream));
    GJ_CUDA(cudaStreamSynchronize(s->stream));
    const uint64_t room = cap > found ? cap - found : 0;
    const uint64_t take = std::min(total, room);
    if (take) {
      GJ_CUDA(cudaMemcpyAsync(out_indices + found, s->d_entries.ptr, take * 8, cudaMemcpyDeviceToHost, s->stream));
      GJ_CUDA(cudaStreamSynchronize(s->stream));
    }
    found += total;
  }
  GJ_CUDA(cudaMemcpyAsync(&s->h_status[3], d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost, s->stream));
  GJ_CUDA(cudaStreamSynchronize(s->stream));
  *n_candidates = found;
  return status_to_code(s->h_status[3], bad_index);
}

int gj_cells_from_points_host(gj_session* s, const double* latlng, uint64_t n, int level, uint64_t* out_raw,
                              uint64_t* bad_index) {
  if (!s || (n && (!latlng || !out_raw))) return GJ_INVALID_ARGUMENT;
  if (level < 0 || level > 30) {  // cell_id.cpp:86-88
    set_error("cell_from_point: level out of range");
    return GJ_INVALID_ARGUMENT;
  }
  gj_index& ix = *s->ix;
  GJ_CUDA(cudaSetDevice(ix.device));
  const uint64_t chunk = 4ull << 20;
  GJ_CUDA(s->d_points[0].reserve(std::min(chunk, std::max<uint64_t>(n, 1)) * 16));
  GJ_CUDA(s->d_entries.reserve(std::min(chunk, std::max<uint64_t>(n, 1)) * 8));
  DevStatus* d_status = s->d_status.as<DevStatus>() + 3;
  int rc = reset_status(s, d_status);
  if (rc != GJ_OK) return rc;
  for (uint64_t begin = 0; begin < n; begin += chunk) {
    const uint64_t len = std::min(chunk, n - begin);
    GJ_CUDA(cudaMemcpyAsync(s->d_points[0].ptr, latlng + 2 * begin, len * 16, cudaMemcpyHostToDevice, s->stream));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((len + 255) / 256, ix.sm_count * 8ull));
    cells_kernel<<<grid, 256, 0, s->stream>>>(s->d_points[0].as<double2>(), len, level, begin,
                                              s->d_entries.as<uint64_t>(), d_status);
    ++s->launches;
    GJ_CUDA(cudaGetLastError());
    GJ_CUDA(cudaMemcpyAsync(out_raw + begin, s->d_entries.ptr, len * 8, cudaMemcpyDeviceToHost, s->stream));
    GJ_CUDA(cudaStreamSynchronize(s->stream));
  }
  GJ_CUDA(cudaMemcpyAsync(&s->h_status[3], d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost, s->stream));
  GJ_CUDA(cudaStreamSynchronize(s->stream));
  return status_to_code(s->h_status[3], bad_index);
}

int gj_probe_cells_host(gj_session* s, const uint64_t* raw_ids, uint64_t n, uint64_t* out_entries) {
  if (!s || (n && (!raw_ids || !out_entries))) return GJ_INVALID_ARGUMENT;
  gj_index& ix = *s->ix;
  GJ_CUDA(cudaSetDevice(ix.device));
  const uint64_t chunk = 4ull << 20;
  GJ_CUDA(s->d_points[0].reserve(std::min(chunk, std::max<uint64_t>(n, 1)) * 16));
  GJ_CUDA(s->d_entries.reserve(std::min(chunk, std::max<uint64_t>(n, 1)) * 8));
  for (uint64_t begin = 0; begin < n; begin += chunk) {
    const uint64_t len = std::min(chunk, n - begin);
    GJ_CUDA(cudaMemcpyAsync(s->d_points[0].ptr, raw_ids + begin, len * 8, cudaMemcpyHostToDevice, s->stream));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((len + 255) / 256, ix.sm_count * 8ull));
    probe_cells_kernel<<<grid, 256, 0, s->stream>>>(ix.dev, s->d_points[0].as<uint64_t>(), len,
                                                    s->d_entries.as<uint64_t>());
    ++s->launches;
    GJ_CUDA(cudaGetLastError());
    GJ_CUDA(cudaMemcpyAsync(out_entries + begin, s->d_entries.ptr, len * 8, cudaMemcpyDeviceToHost, s->stream));
    GJ_CUDA(cudaStreamSynchronize(s->stream));
  }
  return GJ_OK;
}

int gj_join_count_host(gj_session* s, const double* latlng, uint64_t n, uint64_t base_index, int mode,
                       uint64_t* counts, gj_stats* stats, uint32_t* out_first_id, gj_overflow* overflow,
                       uint64_t* bad_index) {
  if (!s || (n && !latlng)) return GJ_INVALID_ARGUMENT;
  bool exact = false;
  if (!resolve_exact(*s->ix, mode, &exact)) return GJ_INVALID_ARGUMENT;
  if (overflow && !out_first_id) {
    set_error("an overflow list needs out_first_id");
    return GJ_INVALID_ARGUMENT;
  }
  OverflowSink sink;
  const int rc = run_host_join(s, latlng, n, base_index, exact, counts, stats, out_first_id,
                               out_first_id ? &sink : nullptr, bad_index);
  if (rc != GJ_OK) return rc;
  if (overflow) {
    const size_t m = sink.records.size();
    overflow->count = m;
    if (m > overflow->capacity) {
      set_error("overflow list larger than the caller's capacity");
      return GJ_CAPACITY;
    }
    for (size_t k = 0; k < m; ++k) {
      overflow->point_index[k] = sink.records[k].point;
      overflow->polygon_id[k] = sink.records[k].id;
    }
  }
  return GJ_OK;
}

int gj_join_count_device(gj_session* s, const double* d_latlng, uint64_t n, int mode, uint64_t* d_counts,
                         uint64_t* d_stats, uint32_t* d_first_id, int sync) {
  if (!s || (n && !d_latlng) || !d_counts) return GJ_INVALID_ARGUMENT;
  gj_index& ix = *s->ix;
  bool exact = false;
  if (!resolve_exact(ix, mode, &exact)) return GJ_INVALID_ARGUMENT;
  GJ_CUDA(cudaSetDevice(ix.device));
  // One launch per `piece` points: all of them, unless the index caps a launch lower (arenas of 2^24 nodes and more)
  const uint64_t piece = std::max<uint64_t>(1, std::min(n, max_launch_points(ix)));
  const uint64_t task_cap = exact ? piece * std::max<uint64_t>(1, ix.max_cand_refs) : 0;
  if (task_cap >= (1ull << 32)) {
    set_error("candidate task capacity exceeds 2^32; split the launch");
    return GJ_INVALID_ARGUMENT;
  }
  int rc;
  if (exact && (rc = reserve_tasks(s, task_cap)) != GJ_OK) return rc;
  for (uint64_t begin = 0; begin == 0 || begin < n; begin += piece) {
    const uint64_t len = std::min(piece, n - begin);
    JoinRequest rq{};
    rq.d_pts = reinterpret_cast<const double2*>(d_latlng) + begin;
    rq.n = len;
    rq.base_index = begin;
    rq.exact = exact;
    rq.want_stats = d_stats != nullptr;
    rq.d_counts = reinterpret_cast<unsigned long long*>(d_counts);
    rq.d_stats = reinterpret_cast<unsigned long long*>(d_stats);
    rq.d_first_id = d_first_id ? d_first_id + begin : nullptr;
    rq.d_status = s->d_status.as<DevStatus>();
    rq.ovf_cap = 0;  // the overflow list cannot be handed back from here: only the flag in the first id
    rq.ovf_discard = true;
    rq.task_cap = task_cap;
    rq.keep_errors = begin != 0;  // the smallest offending index of the whole call survives the later pieces
    if ((rc = enqueue_join(s, rq)) != GJ_OK) return rc;
    if (n == 0) break;
  }
  if (sync) return gj_session_sync(s, nullptr);
  return GJ_OK;
}

int gj_session_sync(gj_session* s, uint64_t* bad_index) {
  if (!s) return GJ_INVALID_ARGUMENT;
  GJ_CUDA(cudaSetDevice(s->ix->device));
  GJ_CUDA(cudaMemcpyAsync(&s->h_status[0], s->d_status.ptr, sizeof(DevStatus), cudaMemcpyDeviceToHost, s->stream));
  GJ_CUDA(cudaStreamSynchronize(s->stream));
  return status_to_code(s->h_status[0], bad_index);
}

int gj_join_pairs_host(gj_session* s, const double* latlng, uint64_t n, int mode, uint64_t* n_pairs,
                       gj_stats* stats, uint64_t* bad_index) {
  if (!s || (n && !latlng)) return GJ_INVALID_ARGUMENT;
  bool exact = false;
  if (!resolve_exact(*s->ix, mode, &exact)) return GJ_INVALID_ARGUMENT;
  const int rc = run_host_pairs(s, latlng, n, exact, stats, bad_index);
  if (rc != GJ_OK) {
    s->pairs_valid = false;
    return rc;
  }
  if (n_pairs) *n_pairs = s->pairs_total;
  return GJ_OK;
}

int gj_join_pairs_device(gj_session* s, const double* d_latlng, uint64_t n, int mode, uint64_t* d_row_ptr,
                         uint32_t* d_polygon_id, uint64_t id_capacity, uint64_t* n_pairs, gj_stats* stats,
                         uint64_t* bad_index) {
  if (!s || (n && !d_latlng) || !d_row_ptr || (id_capacity && !d_polygon_id)) return GJ_INVALID_ARGUMENT;
  bool exact = false;
  if (!resolve_exact(*s->ix, mode, &exact)) return GJ_INVALID_ARGUMENT;
  PairsSink sink;
  sink.d_row_ptr = d_row_ptr;
  sink.d_ids = d_polygon_id;
  sink.ids_cap = id_capacity;
  return run_pairs_async(s, d_latlng, true, n, exact, stats, sink, n_pairs, bad_index);
}

int gj_join_pairs_host_into(gj_session* s, const double* latlng, uint64_t n, int mode, uint64_t* row_ptr,
                            uint32_t* polygon_id, uint64_t id_capacity, uint64_t* n_pairs, gj_stats* stats,
                            uint64_t* bad_index) {
  if (!s || (n && !latlng) || !row_ptr || (id_capacity && !polygon_id)) return GJ_INVALID_ARGUMENT;
  bool exact = false;
  if (!resolve_exact(*s->ix, mode, &exact)) return GJ_INVALID_ARGUMENT;
  PairsSink sink;
  sink.h_row_ptr = row_ptr;
  sink.h_ids = polygon_id;
  sink.ids_cap = id_capacity;
  return run_pairs_async(s, latlng, false, n, exact, stats, sink, n_pairs, bad_index);
}

int gj_pairs_copy(gj_session* s, uint64_t* row_ptr, uint32_t* polygon_id) {
  if (!s || !row_ptr) return GJ_INVALID_ARGUMENT;
  if (!s->pairs_valid) {
    set_error("gj_pairs_copy: no completed gj_join_pairs_host call to copy from");
    return GJ_INVALID_ARGUMENT;
  }
  GJ_CUDA(cudaSetDevice(s->ix->device));
  // straight from HBM into the caller's arrays: directly when they are pinned (gj_host_alloc), else
  // through the session's stager
  GJ_CUDA(stager_of(s).to_host(row_ptr, s->d_all_row_ptr.ptr, (s->pairs_n + 1) * 8, s->copy_out));
  if (polygon_id && s->pairs_total) {
    GJ_CUDA(stager_of(s).to_host(polygon_id, s->d_all_ids.ptr, s->pairs_total * 4, s->copy_out));
  }
  return GJ_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Device groups: the reference's worker fan-out (join.cpp:255-285) over GPUs.
// ---------------------------------------------------------------------------
struct gj_group {
  std::vector<gj_index*> ix;
  std::vector<gj_session*> s;
  // the last gj_group_join_pairs_host call
  std::vector<uint64_t> pairs_begin;  // first point of every worker's range, then n
  std::vector<uint64_t> pairs_base;   // pairs emitted by the ranges before it, then the total
  bool pairs_valid = false;
  ~gj_group() {
    for (gj_session* q : s) gj_session_destroy(q);
    for (gj_index* q : ix) gj_index_destroy(q);
  }
};

namespace {

int group_finish(std::unique_ptr<gj_group>& g, gj_index* first, const int* devices, int n_devices, gj_group** out) {
  g->ix.push_back(first);
  for (int k = 1; k < n_devices; ++k) {  // device to device, not from the host again
    gj_index* rep = nullptr;
    const int rc = replicate_index(*first, devices[k], &rep);
    if (rc != GJ_OK) return rc;
    g->ix.push_back(rep);
  }
  for (gj_index* ix : g->ix) {
    gj_session* s = nullptr;
    const int rc = gj_session_create(ix, &s);
    if (rc != GJ_OK) return rc;
    g->s.push_back(s);
  }
  *out = g.release();
  return GJ_OK;
}

int group_workers(const gj_group* g, int workers) {
  const int size = static_cast<int>(g->s.size());
  return workers <= 0 || workers > size ? size : workers;
}

// Runs fn(w) for w in [0, W) — worker 0 on the calling thread — and returns the status of the first range
// that failed (with its error text on this thread), like a sequential scan would.
template <typename Fn>
int fan_out(int W, Fn fn, int* failed_worker = nullptr) {
  std::vector<int> rc(W, GJ_OK);
  std::vector<std::string> err(W);
  auto run = [&](int w) {
    rc[w] = fn(w);
    if (rc[w] != GJ_OK) err[w] = last_error();
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < W; ++w) pool.emplace_back(run, w);
  run(0);
  for (std::thread& t : pool) t.join();
  for (int w = 0; w < W; ++w) {
    if (rc[w] != GJ_OK) {
      set_error(err[w]);
      if (failed_worker) *failed_worker = w;
      return rc[w];
    }
  }
  return GJ_OK;
}

}  // namespace

extern "C" {

int gj_group_create(const gj_index_desc* desc, const int* devices, int n_devices, const gj_options* opt,
                    gj_group** out) {
  if (!desc || !devices || n_devices < 1 || !out) return GJ_INVALID_ARGUMENT;
  *out = nullptr;
  std::unique_ptr<gj_group> g(new gj_group);
  gj_index* first = nullptr;
  const int rc = create_index(*desc, devices[0], opt, &first);
  if (rc != GJ_OK) return rc;
  return group_finish(g, first, devices, n_devices, out);
}

int gj_group_load_file(const char* path, const int* devices, int n_devices, const gj_options* opt, gj_group** out) {
  if (!path || !devices || n_devices < 1 || !out) return GJ_INVALID_ARGUMENT;
  *out = nullptr;
  std::unique_ptr<gj_group> g(new gj_group);
  gj_index* first = nullptr;
  const int rc = load_index_file(path, devices[0], opt, &first);
  if (rc != GJ_OK) return rc;
  return group_finish(g, first, devices, n_devices, out);
}

void gj_group_destroy(gj_group* g) { delete g; }
int gj_group_size(const gj_group* g) { return g ? static_cast<int>(g->s.size()) : 0; }
gj_index* gj_group_index(gj_group* g, int k) {
  return g && k >= 0 && k < static_cast<int>(g->ix.size()) ? g->ix[k] : nullptr;
}
gj_session* gj_group_session(gj_group* g, int k) {
  return g && k >= 0 && k < static_cast<int>(g->s.size()) ? g->s[k] : nullptr;
}

int gj_group_join_count_host(gj_group* g, int workers, const double* latlng, uint64_t n, uint64_t base_index,
                             int mode, uint64_t* counts, gj_stats* stats, uint32_t* out_first_id,
                             gj_overflow* overflow, uint64_t* bad_index) {
  if (!g || g->s.empty() || (n && !latlng)) return GJ_INVALID_ARGUMENT;
  bool exact = false;
  if (!resolve_exact(*g->ix[0], mode, &exact)) return GJ_INVALID_ARGUMENT;
  if (overflow && !out_first_id) {
    set_error("an overflow list needs out_first_id");
    return GJ_INVALID_ARGUMENT;
  }
  const int W = group_workers(g, workers);
  const uint32_t n_ids = g->ix[0]->dev.n_ids;
  struct Part {
    std::vector<uint64_t> counts;
    gj_stats st{};
    OverflowSink sink;
    uint64_t bad = 0;
  };
  std::vector<Part> part(W);
  int failed = 0;
  auto begin_of = [&](int w) { return static_cast<uint64_t>(static_cast<unsigned __int128>(n) * w / W); };  // join.cpp:264-265
  const int rc = fan_out(W, [&](int w) {
    Part& p = part[w];
    p.counts.assign(n_ids + 1, 0);
    const uint64_t begin = begin_of(w), len = begin_of(w + 1) - begin;
    return run_host_join(g->s[w], latlng + 2 * begin, len, base_index + begin, exact, p.counts.data(),
                         stats ? &p.st : nullptr, out_first_id ? out_first_id + begin : nullptr,
                         out_first_id ? &p.sink : nullptr, &p.bad);
  }, &failed);
  if (rc != GJ_OK) {  // the first failing range holds the smallest offending index
    if (bad_index) *bad_index = part[failed].bad;
    return rc;
  }
  // merge like join.cpp:280-284
  for (int w = 0; w < W; ++w) {
    if (counts) {
      for (uint32_t i = 0; i < n_ids; ++i) counts[i] += part[w].counts[i];
    }
    if (stats) {
      stats->probes += part[w].st.probes;
      stats->pip_tests += part[w].st.pip_tests;
      stats->false_hits += part[w].st.false_hits;
      stats->solely_true_hits += part[w].st.solely_true_hits;
      stats->refinement_entered += part[w].st.refinement_entered;
      stats->candidate_refs += part[w].st.candidate_refs;
    }
  }
  if (overflow) {
    size_t m = 0;
    for (const Part& p : part) m += p.sink.records.size();
    overflow->count = m;
    if (m > overflow->capacity) {
      set_error("overflow list larger than the caller's capacity");
      return GJ_CAPACITY;
    }
    size_t at = 0;  // ranges ascend, each list is sorted: the concatenation is sorted
    for (const Part& p : part) {
      for (const OverflowRecord& r : p.sink.records) {
        overflow->point_index[at] = r.point;
        overflow->polygon_id[at] = r.id;
        ++at;
      }
    }
  }
  return GJ_OK;
}

int gj_group_join_pairs_host(gj_group* g, int workers, const double* latlng, uint64_t n, int mode,
                             uint64_t* n_pairs, gj_stats* stats, uint64_t* bad_index) {
  if (!g || g->s.empty() || (n && !latlng)) return GJ_INVALID_ARGUMENT;
  bool exact = false;
  if (!resolve_exact(*g->ix[0], mode, &exact)) return GJ_INVALID_ARGUMENT;
  g->pairs_valid = false;
  const int W = group_workers(g, workers);
  g->pairs_begin.assign(W + 1, 0);
  for (int w = 0; w <= W; ++w) g->pairs_begin[w] = static_cast<uint64_t>(static_cast<unsigned __int128>(n) * w / W);
  std::vector<gj_stats> st(W);
  std::vector<uint64_t> bad(W, 0);
  int failed = 0;
  int rc = fan_out(W, [&](int w) {
    const uint64_t begin = g->pairs_begin[w], len = g->pairs_begin[w + 1] - begin;
    return run_host_pairs(g->s[w], latlng + 2 * begin, len, exact, stats ? &st[w] : nullptr, &bad[w]);
  }, &failed);
  if (rc != GJ_OK) {
    if (bad_index) *bad_index = g->pairs_begin[failed] + bad[failed];  // run_host_pairs reports indices of its own range
    return rc;
  }
  g->pairs_base.assign(W + 1, 0);
  for (int w = 0; w < W; ++w) g->pairs_base[w + 1] = g->pairs_base[w] + g->s[w]->pairs_total;
  // every replica's row offsets move behind the pairs of the ranges before it, still in HBM
  rc = fan_out(W, [&](int w) {
    gj_session* s = g->s[w];
    const uint64_t rows = g->pairs_begin[w + 1] - g->pairs_begin[w] + 1;
    if (g->pairs_base[w] == 0) return static_cast<int>(GJ_OK);
    GJ_CUDA(cudaSetDevice(s->ix->device));
    add_offset_kernel<<<static_cast<unsigned>(s->ix->sm_count) * 8u, 256, 0, s->stream>>>(s->d_all_row_ptr.as<uint64_t>(),
                                                                                          rows, g->pairs_base[w]);
    ++s->launches;
    GJ_CUDA(cudaGetLastError());
    GJ_CUDA(cudaStreamSynchronize(s->stream));
    return static_cast<int>(GJ_OK);
  });
  if (rc != GJ_OK) return rc;
  for (int w = 0; w < W && stats; ++w) {
    stats->probes += st[w].probes;
    stats->pip_tests += st[w].pip_tests;
    stats->false_hits += st[w].false_hits;
    stats->solely_true_hits += st[w].solely_true_hits;
    stats->refinement_entered += st[w].refinement_entered;
    stats->candidate_refs += st[w].candidate_refs;
  }
  if (n_pairs) *n_pairs = g->pairs_base[W];
  g->pairs_valid = true;
  return GJ_OK;
}

int gj_group_pairs_copy(gj_group* g, uint64_t* row_ptr, uint32_t* polygon_id) {
  if (!g || !row_ptr) return GJ_INVALID_ARGUMENT;
  if (!g->pairs_valid) {
    set_error("gj_group_pairs_copy: no completed gj_group_join_pairs_host call to copy from");
    return GJ_INVALID_ARGUMENT;
  }
  const int W = static_cast<int>(g->pairs_begin.size()) - 1;
  // range w's rows land at row_ptr[begin_w .. begin_{w+1}] (its last entry == the next range's first), its ids
  // behind those of the ranges before it; every replica copies over its own link
  return fan_out(W, [&](int w) {
    gj_session* s = g->s[w];
    GJ_CUDA(cudaSetDevice(s->ix->device));
    const uint64_t begin = g->pairs_begin[w], rows = g->pairs_begin[w + 1] - begin;
    GJ_CUDA(stager_of(s).to_host(row_ptr + begin, s->d_all_row_ptr.ptr, (rows + (w == W - 1 ? 1 : 0)) * 8, s->copy_out));
    if (polygon_id && s->pairs_total) {
      GJ_CUDA(stager_of(s).to_host(polygon_id + g->pairs_base[w], s->d_all_ids.ptr, s->pairs_total * 4, s->copy_out));
    }
    return static_cast<int>(GJ_OK);
  });
}

}  // extern "C"
