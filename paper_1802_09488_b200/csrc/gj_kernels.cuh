// sm_100a kernels of the probe path.
//
//   K1  join_kernel        points -> cell -> directory/trie -> entry -> emit
//                          (counts, first ids, overflow records, stats) and,
//                          in exact mode, candidate tasks for K2
//   K1' probe_points_kernel / probe_cells_kernel   entries only (test hooks)
//   K2  refine_kernel      ray-crossing PIP over the candidate tasks: each
//                          task tests only the edges of its polygon's
//                          latitude strip (precomputed at index create)
//
// All of it is HBM/L2-bound integer and fp64 scalar work; no tensor cores.
#pragma once

#include <type_traits>

#include "gj_device.cuh"

namespace gj {

// Tunables (overridable with -D for tools/k1_sweep.py).
#ifndef GJ_JOIN_THREADS
#define GJ_JOIN_THREADS 1024
#endif
#ifndef GJ_JOIN_MIN_BLOCKS
#define GJ_JOIN_MIN_BLOCKS 1
#endif
#ifndef GJ_PPT
#define GJ_PPT 4
#endif
constexpr int kJoinThreads = GJ_JOIN_THREADS;
constexpr int kPointsPerThread = GJ_PPT;
// Per-warp queues of 8-byte items.  Q2 holds the points the shared-memory
// directory left open (< 32 left over + up to 32 per point slot of a tile);
// Q3 the few that the second tier leaves open as well (< 32 left over + 32
// per Q2 drain).
#ifndef GJ_PF_DIST
#define GJ_PF_DIST 1
#endif
constexpr uint32_t kQueueSlow = 0xFFFFFFFFu;  // queue word of a point population 1 would not decide
constexpr uint32_t kDirectSkip = 0xFFFFFFFEu;  // kDirect: the staged code of a lane past the end of the points
constexpr uint32_t kPrefetchTiles = GJ_PF_DIST;  // K1: L2 prefetch distance in tiles, 0 = off
constexpr int kQueue2Cap = 32 * (kPointsPerThread + 1);
constexpr int kQueue3Cap = 64;
constexpr int kQueueBytesPerWarp = (kQueue2Cap + kQueue3Cap) * 8;
// The direct form (join_kernel's kDirect) has no Q2: per warp two staging buffers of 128 codes + 128 node slots
// and one queue area shared by Q3, growing up from the bottom (< 32 left over + 32 per settle round between two
// visits of the drain site), and Q4, growing down from the top: the few open points whose walk goes deeper than the
// queued sub-cell bits reach (< 32 left over + at most what a Q3 batch hands over, which Q3 has just given up).
// Two rounds per drain visit, not four: four straight rounds are 7 % faster on an index with a small histogram
// (0.672 vs 0.724 ms per 100 M points, config-4 stand-in), but their 192-entry area pushes BASELINE config 4 at full
// size (80 KB of 16-bit histogram) over the 164 KB carve-out step, where they lose 5 % instead (0.791 vs 0.750 ms
// with the stand-in padded to that size; profiles/k1_sweep_r02_cfg4_standin_direct_rounds_padded.json).
#ifndef GJ_DIRECT_ROUNDS
#define GJ_DIRECT_ROUNDS 2
#endif
constexpr int kDirectRounds = GJ_DIRECT_ROUNDS;  // settle rounds between two visits of the drain site
constexpr int kDirectBufBytes = 32 * kPointsPerThread * 5;
constexpr int kDirectQueue3Cap = 64 + 32 * kDirectRounds;
constexpr int kDirectBytesPerWarp = 2 * kDirectBufBytes + kDirectQueue3Cap * 8;
static_assert(kPointsPerThread % kDirectRounds == 0 && 31 + 32 * kDirectRounds + 31 <= kDirectQueue3Cap, "Q3 + Q4 share the area");
constexpr int kChunkPoints = 32 * kPointsPerThread;  // consecutive points a warp owns in a tile
constexpr int kRefineThreads = 256;
// The 16-bit histogram (JoinParams::hist16) is flushed by the whole CTA every this many tiles.  Between two
// flushes a CTA settles at most the points it loaded since (kTile per tile) plus what its queues and in-flight
// batches carried over (< 32 warps * (kQueue2Cap + kQueue3Cap + 32) = 8192; direct form: the staged tile, 4096,
// + 32 warps * kDirectQueue3Cap = 4096), and a point adds at most 1 to any one polygon: 12 * 4096 + 8192 = 57344
// < 65536, so no counter can overflow.
constexpr uint32_t kHist16FlushTiles = 12;
static_assert(kHist16FlushTiles * GJ_JOIN_THREADS * GJ_PPT + GJ_JOIN_THREADS * GJ_PPT + (GJ_JOIN_THREADS / 32) * kDirectQueue3Cap < 65536,
              "16-bit counters between two flushes, direct form");
// Lookup-table records of one population-3 batch staged in shared memory by the whole warp (stage_records):
// up to this many 16-byte chunks per warp (the launch plan gives what shared memory has left, JoinParams::
// stage_chunks).  A batch of 32 records of ~20 words takes ~190 chunks; a batch that needs more than the buffer
// holds is walked from global memory as before.
constexpr uint32_t kStageChunksMax = 256;
constexpr uint32_t kStageChunksMin = 128;

struct JoinParams {
  const double2* pts;  // (lat, lng) pairs: .x = lat, .y = lng  (latlng.hpp:26-29)
  uint64_t n;
  uint64_t base_index;
  unsigned long long* counts;  // [n_ids], added to
  unsigned long long* stats;   // [6] or null
  uint32_t* first_id;          // [n] or null
  uint64_t* ovf_point;
  uint32_t* ovf_id;
  uint32_t* ovf_ord;
  uint64_t ovf_cap;
  int32_t ovf_discard;      // device-resident calls: nobody can read the list, do not record (and never fail on) it
  uint32_t* task_point;
  uint32_t* task_slot;
  uint32_t* task_ord;
  uint64_t task_cap;
  DevStatus* status;
  uint32_t smem_queue_off;  // bytes: per-warp open-point queues
  uint32_t smem_hist_off;   // bytes
  uint32_t hist_rep;        // replicas per slot (power of two), 0 = not in shared memory
  uint32_t hist16;          // hist_rep == 0: one 16-bit histogram in shared memory, flushed every kHist16FlushTiles tiles
  uint32_t smem_stage_off;  // bytes: per-warp staging buffers for lookup-table records (stage_chunks * 16 each); 0 = none
  uint32_t stage_chunks;
  uint32_t* counts_priv;    // hist_rep == 0: [n_priv][n_ids] u32 copies, zero on entry; may be null
  uint32_t n_priv;          // CTA b counts into copy b % n_priv
  int32_t exact;
};

__device__ __forceinline__ uint32_t id_to_slot(const DevIndex& ix, uint32_t id) {
  if (ix.ids_dense) return id;
  uint32_t lo = 0, hi = ix.n_ids;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(ix.ids + mid) < id) {
      lo = mid + 1;
    } else {
      hi = mid;
    }
  }
  return lo;  // present by construction of the id table
}

__device__ __forceinline__ void flag_error(DevStatus* st, uint32_t bit, uint64_t index) {
  atomicOr(&st->flags, bit);
  atomicMin(&st->bad_index, static_cast<unsigned long long>(index));
}

// ---------------------------------------------------------------------------
// Shared memory by 32-bit shared-window address and predicated memory
// operations.  K1's hot path is straight-line code: conditional loads, atomics
// and stores are predicated instructions, not branches.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void sts64_if(uint32_t addr, uint32_t x, uint32_t y, bool pred) {
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %3, 0; @p st.shared.v2.u32 [%0], {%1, %2}; }" ::"r"(addr), "r"(x),
               "r"(y), "r"(static_cast<uint32_t>(pred))
               : "memory");
}
__device__ __forceinline__ void red_add_shared_if(uint32_t addr, uint32_t v, bool pred) {
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p red.shared.add.u32 [%0], %1; }" ::"r"(addr), "r"(v),
               "r"(static_cast<uint32_t>(pred))
               : "memory");
}
__device__ __forceinline__ void red_inc_shared_if(uint32_t addr, bool pred) {
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %1, 0; @p red.shared.add.u32 [%0], 1; }" ::"r"(addr),
               "r"(static_cast<uint32_t>(pred))
               : "memory");
}
// One random 4-byte gather (the 32-bit tier), read-only path, allocating in L1: `L1::no_allocate` here — on the
// argument that 4 bytes of a line are used — took config 2 from 0.355 to 0.472 ms per 100 M points (the tier is
// small enough for L1 to catch a good share of the gathers) and gained 1.4 % on full-size config 5.
__device__ __forceinline__ uint32_t ldg32_if(const uint32_t* p, bool pred, uint32_t otherwise) {
  uint32_t v;
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %3, 0; mov.u32 %0, %2; @p ld.global.nc.u32 %0, [%1]; }"
               : "=r"(v)
               : "l"(p), "r"(otherwise), "r"(static_cast<uint32_t>(pred)));
  return v;
}
// The same gather issued as an asynchronous copy into shared memory (LDGSTS): no register waits for it.
__device__ __forceinline__ void cp_async4_if(uint32_t dst, const uint32_t* p, bool pred) {
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p cp.async.ca.shared.global [%0], [%1], 4; }" ::"r"(dst), "l"(p),
               "r"(static_cast<uint32_t>(pred))
               : "memory");
}
__device__ __forceinline__ void sts32_if(uint32_t addr, uint32_t v, bool pred) {
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p st.shared.u32 [%0], %1; }" ::"r"(addr), "r"(v),
               "r"(static_cast<uint32_t>(pred))
               : "memory");
}
__device__ __forceinline__ void sts8(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st32_if(uint32_t* p, uint32_t v, bool pred) {
  asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p st.global.u32 [%0], %1; }" ::"l"(p), "r"(v),
               "r"(static_cast<uint32_t>(pred))
               : "memory");
}

// Where K1 counts: a replicated shared-memory histogram (slot * rep + lane
// replica) or, for id tables too large for it, a private u32 copy of the counts in
// global memory, one per resident CTA (folded into the caller's u64 counts afterwards).
// Atomics of all SMs on ONE shared copy serialise in L2 on every hot polygon:
// measured 13.4 ms instead of 0.36 ms per 100 M points with 289 polygons, 7.5 ms
// instead of 0.9 ms with 1600.
struct HistRef {
  uint32_t smem;      // shared address of the histogram
  uint32_t rep;       // replicas per slot (power of two), 0 = not in shared memory
  uint32_t lane_rep;  // lane & (rep - 1)
  uint32_t h16;       // rep == 0: 16-bit counters, two per word (JoinParams::hist16)
  uint32_t* priv;     // rep == 0 && !h16: this SM's copy (null: straight into jp.counts)
};

template <bool kDense>
__device__ __forceinline__ void count_slot(const DevIndex& ix, const JoinParams& jp, const HistRef& h,
                                           uint32_t id) {
  const uint32_t slot = kDense ? id : id_to_slot(ix, id);
  if (h.rep) {
    red_inc_shared_if(h.smem + (slot * h.rep + h.lane_rep) * 4u, true);
  } else if (h.h16) {  // the half-word's carry cannot happen between two flushes (kHist16FlushTiles)
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(h.smem + (slot >> 1) * 4u), "r"(1u << ((slot & 1u) * 16u)) : "memory");
  } else if (h.priv) {
    atomicAdd(h.priv + slot, 1u);
  } else {
    atomicAdd(&jp.counts[slot], 1ull);
  }
}

// What the out-of-line general emit path (emit_general) needs of the two kernel parameter blocks, copied once per
// CTA into shared memory.  Passing the __grid_constant__ blocks themselves by reference into a __noinline__
// function made ptxas keep thread-local copies of both (a ~690-byte stack frame) in whichever instantiation was
// short of registers — measured 9.7 instead of 1.3 ms per 100 M points in one of them.
struct EmitCtx {
  const uint32_t* lut;
  const uint32_t* ids;
  const uint32_t* ring_len;
  unsigned long long* counts;
  DevStatus* status;
  uint64_t* ovf_point;
  uint32_t* ovf_id;
  uint32_t* ovf_ord;
  uint32_t* task_point;
  uint32_t* task_slot;
  uint32_t* task_ord;
  uint64_t base_index, ovf_cap, task_cap;
  uint32_t n_ids;
  int32_t ids_dense, exact, ovf_discard;
};

__device__ __forceinline__ uint32_t id_to_slot(const EmitCtx& c, uint32_t id) {
  if (c.ids_dense) return id;
  uint32_t lo = 0, hi = c.n_ids;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(c.ids + mid) < id) {
      lo = mid + 1;
    } else {
      hi = mid;
    }
  }
  return lo;
}

template <bool kDense>
__device__ __forceinline__ void count_slot(const EmitCtx& c, const HistRef& h, uint32_t id) {
  const uint32_t slot = kDense ? id : id_to_slot(c, id);
  if (h.rep) {
    red_inc_shared_if(h.smem + (slot * h.rep + h.lane_rep) * 4u, true);
  } else if (h.h16) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(h.smem + (slot >> 1) * 4u), "r"(1u << ((slot & 1u) * 16u)) : "memory");
  } else if (h.priv) {
    atomicAdd(h.priv + slot, 1u);
  } else {
    atomicAdd(&c.counts[slot], 1ull);
  }
}

// What one entry needs beyond the straight-line path: how many references
// it holds, how many of them are candidates, and — for this join mode — how
// many overflow records and candidate tasks it will write.
struct EntryPlan {
  uint32_t tag, off, t;     // lookup-table record [t, true ids, c, candidate ids] at `off`
  uint32_t n_refs, n_cand;
  uint32_t n_ovf, n_tasks;  // records to reserve
  bool defer;               // some pairs depend on K2
};

template <bool kIds>
__device__ __forceinline__ EntryPlan plan_entry(const DevIndex& ix, bool exact, uint64_t entry) {
  EntryPlan e{};
  e.tag = static_cast<uint32_t>(entry) & 3u;
  if (e.tag == 1u) {
    e.n_refs = 1;
    e.n_cand = 1u - (static_cast<uint32_t>(entry >> 2) & 1u);
  } else if (e.tag == 2u) {
    e.n_refs = 2;
    e.n_cand = 2u - ((static_cast<uint32_t>(entry >> 33) & 1u) + (static_cast<uint32_t>(entry >> 2) & 1u));
  } else {
    e.off = static_cast<uint32_t>(entry >> 2) & 0x7fffffffu;
    e.t = __ldg(ix.lut + e.off);
    e.n_refs = e.t + __ldg(ix.lut + e.off + 1 + e.t);
    e.n_cand = e.n_refs - e.t;
  }
  e.defer = exact && e.n_cand != 0;
  const uint32_t n_now = exact ? e.n_refs - e.n_cand : e.n_refs;  // pairs emitted by K1
  // overflow records: everything after the first pair, or every pair when
  // the point is deferred
  e.n_ovf = kIds ? (e.defer ? n_now : (n_now > 0 ? n_now - 1 : 0)) : 0;
  e.n_tasks = e.defer ? e.n_cand : 0;
  return e;
}

// One reservation per warp: every lane asks for `want` consecutive records of
// a global cursor; lane 0 does a single atomic for the warp's total and the
// lanes get their bases from a prefix sum.  (Per-lane atomics with return on
// one address serialise across the whole chip: with 1.8 % of the points
// entering refinement they made the exact join 4.5x slower than the approx one.)
__device__ __forceinline__ unsigned long long warp_reserve(unsigned long long* cursor, uint32_t want, uint32_t lane) {
  uint32_t incl = want;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t up = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += up;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  unsigned long long base = 0;
  if (total != 0u && lane == 0u) base = atomicAdd(cursor, static_cast<unsigned long long>(total));
  base = __shfl_sync(0xffffffffu, base, 0);
  return base + (incl - want);
}

// Warp-cooperative copy of the lookup-table records of one batch into shared memory.  Lane l holds a record that
// spans the aligned 16-byte chunks [first_chunk, first_chunk + n_chunks) of the table (n_chunks == 0: none).  The
// chunks of all lanes are flattened — chunk g belongs to the first lane whose inclusive prefix of n_chunks exceeds
// g — so every load instruction reads 32 consecutive chunks of a few records (coalesced, each sector fetched once,
// independent of L1) and the loads of a step are all issued before the first store: a per-lane walk costs one
// round trip per word (per four words at best), this costs two or three per batch.  Returns the chunk index at
// which this lane's record starts in the staging buffer, or ~0u when the batch does not fit (nothing is copied).
__device__ __noinline__ uint32_t stage_records(const uint4* __restrict__ lut4, uint32_t s_stage, uint32_t capacity,
                                               uint32_t lane, uint32_t first_chunk, uint32_t n_chunks) {
  uint32_t incl = n_chunks;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t up = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += up;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  if (total == 0u || total > capacity) return ~0u;
  const uint32_t excl = incl - n_chunks;
  __syncwarp();  // every lane is done with the records of the batch before
  for (uint32_t g0 = 0; g0 < total; g0 += 96u) {
    uint4 v[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const uint32_t g = g0 + static_cast<uint32_t>(u) * 32u + lane;
      uint32_t owner = 0;  // number of lanes with incl <= g
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t at = __shfl_sync(0xffffffffu, incl, min(owner + step - 1u, 31u));
        if (at <= g) owner += step;
      }
      const uint32_t src = min(owner, 31u);
      const uint32_t fc = __shfl_sync(0xffffffffu, first_chunk, src), ex = __shfl_sync(0xffffffffu, excl, src);
      v[u] = make_uint4(0, 0, 0, 0);
      if (g < total) {
        asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(lut4 + fc + (g - ex)));
      }
    }
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const uint32_t g = g0 + static_cast<uint32_t>(u) * 32u + lane;
      if (g < total) {
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(s_stage + g * 16u), "r"(v[u].x), "r"(v[u].y),
                     "r"(v[u].z), "r"(v[u].w)
                     : "memory");
      }
    }
  }
  __syncwarp();
  return excl;
}

// The per-(point, entry) body of run_join (join.cpp:93-127) for everything
// the straight-line path does not take: two payloads, lookup-table records,
// exact-mode candidates (tasks for K2) and the overflow list.  Cold and out
// of line.  Returns the first-id word of the point.
template <bool kIds, bool kDense>
__device__ __noinline__ uint32_t emit_general(const EmitCtx* ctx, HistRef h, uint64_t entry, uint32_t local,
                                              EntryPlan e, unsigned long long ovf_base,
                                              unsigned long long task_base, uint32_t staged_at) {
  const EmitCtx& jp = *ctx;  // (in shared memory)
  const EmitCtx& ix = *ctx;
  const bool exact = jp.exact != 0;
  const uint32_t n_now = exact ? e.n_refs - e.n_cand : e.n_refs;
  uint32_t n_ovf = e.n_ovf;
  if (n_ovf && (jp.ovf_discard || ovf_base + n_ovf > jp.ovf_cap)) {
    if (!jp.ovf_discard) atomicOr(&jp.status->flags, kErrOverflowCap);
    n_ovf = 0;
  }
  const bool tasks_ok = e.n_tasks == 0 || task_base + e.n_tasks <= jp.task_cap;
  if (!tasks_ok) atomicOr(&jp.status->flags, kErrTaskCap);

  uint32_t first = e.defer ? kDeferred : kNoMatch;
  uint32_t emitted = 0, tasks = 0;
  // the k-th reference emits a pair now (a true hit, or any reference in approximate mode) ...
  auto emit_pair = [&](uint32_t id, uint32_t k) {
    count_slot<kDense>(jp, h, id);
    if (kIds) {
      if (!e.defer && emitted == 0) {
        first = id | (n_now > 1 ? kMoreFlag : 0u);
      } else if (n_ovf) {
        const uint64_t w = ovf_base + (e.defer ? emitted : emitted - 1);
        jp.ovf_point[w] = jp.base_index + local;
        jp.ovf_id[w] = id;
        jp.ovf_ord[w] = k;
      }
    }
    ++emitted;
  };
  // ... or becomes a candidate task for K2 (exact mode)
  auto emit_task = [&](uint32_t id, uint32_t k) {
    const uint32_t slot = kDense ? id : id_to_slot(ix, id);
    if (__ldg(ix.ring_len + slot) == 0u) {  // join.cpp:111-114
      flag_error(jp.status, kErrUnknownPolygon, jp.base_index + local);
    }
    if (tasks_ok) {
      const uint64_t w = task_base + tasks;
      jp.task_point[w] = local;
      jp.task_slot[w] = slot;
      jp.task_ord[w] = k;
    }
    ++tasks;
  };
  // references in the reference's emit order (act.hpp:169-196)
  if (e.tag == 3u) {  // record [t, true ids, c, candidate ids]: two plain loops (overlapping polygon sets live here)
    if (staged_at) {  // the record is in shared memory (stage_records): word 0 = t, 1 + k = true id k, 2 + k = candidate k
      uint32_t k = 0;
      for (; k < e.t; ++k) emit_pair(lds32(staged_at + (1u + k) * 4u), k);
      if (exact) {
        for (; k < e.n_refs; ++k) emit_task(lds32(staged_at + (2u + k) * 4u), k);
      } else {
        for (; k < e.n_refs; ++k) emit_pair(lds32(staged_at + (2u + k) * 4u), k);
      }
      return first;
    }
    const uint32_t* true_ids = ix.lut + e.off + 1;
    const uint32_t* cand_ids = ix.lut + e.off + 2;  // indexed by k as well
    // four independent loads in flight per step: a lane walks its own record, so consecutive words share a sector
    // but each word is its own load, and one load's latency per reference adds up over ~17 references
    uint32_t k = 0;
    for (; k + 4u <= e.t; k += 4u) {
      const uint32_t a = __ldg(true_ids + k), b = __ldg(true_ids + k + 1u), c = __ldg(true_ids + k + 2u),
                     d = __ldg(true_ids + k + 3u);
      emit_pair(a, k);
      emit_pair(b, k + 1u);
      emit_pair(c, k + 2u);
      emit_pair(d, k + 3u);
    }
    for (; k < e.t; ++k) emit_pair(__ldg(true_ids + k), k);
    if (exact) {
      for (; k < e.n_refs; ++k) emit_task(__ldg(cand_ids + k), k);
    } else {
      for (; k + 4u <= e.n_refs; k += 4u) {
        const uint32_t a = __ldg(cand_ids + k), b = __ldg(cand_ids + k + 1u), c = __ldg(cand_ids + k + 2u),
                       d = __ldg(cand_ids + k + 3u);
        emit_pair(a, k);
        emit_pair(b, k + 1u);
        emit_pair(c, k + 2u);
        emit_pair(d, k + 3u);
      }
      for (; k < e.n_refs; ++k) emit_pair(__ldg(cand_ids + k), k);
    }
  } else {
    for (uint32_t k = 0; k < e.n_refs; ++k) {
      const uint32_t p = static_cast<uint32_t>(e.tag == 2u && k == 0 ? entry >> 33 : entry >> 2) & 0x7fffffffu;
      if ((p & 1u) != 0u || !exact) {
        emit_pair(p >> 1, k);
      } else {
        emit_task(p >> 1, k);
      }
    }
  }
  return first;
}

// K1.  Persistent grid (one CTA per SM); each CTA stages the 16-bit first
// directory tier (and a replicated per-polygon histogram) in shared memory
// once, then streams tiles of points.  A tile is kTile consecutive points;
// warp w owns the kChunkPoints consecutive points at w*kChunkPoints inside it
// (lane l, slot j -> point j*32 + l of the chunk), so every load and store of
// a warp is one contiguous 512 / 128 byte run, and a thread keeps
// kPointsPerThread independent 16-byte loads in flight.  The work has three
// populations, and only the first runs where the points are:
//   1. all points, straight-line and call-free: branch-free grid coordinates
//      (grid_xy_try), shared-memory tier, emit when the 16-bit code is one
//      payload that emits (85 % on BASELINE config 2);
//   2. points the first tier cannot resolve: compacted into the warp's queue
//      Q2 and drained 32 at a time — one 4-byte gather each into the 32-bit
//      tier `tb` (the L2-resident second tier, or the small first one when
//      the index has no second), settled the same way;
//   3. what is still open (2 %: deep boundary nodes, dictionary entries,
//      exact-mode candidates) and the points population 1 would not decide
//      (invalid, on a grid line): compacted again into Q3 and drained 32 at a
//      time — dependent 8-byte gathers down the arena, lookup-table records,
//      candidate tasks; slow points redo everything with the IEEE division.
// Running 2 and 3 in place would drag all 32 lanes through their code for the
// few active ones; through the queues they always run with full warps.
// kDense: id == count slot for every polygon AND the histogram is in shared
// memory (jp.hist_rep != 0), the common case; otherwise the general counting path.
// kLate (first ids wanted, and the shared-memory tier resolves few points — gj_index::ids_late): population 1
// does not pre-write the first-id words of the points it queues; population 2 writes the word of every point it
// looks up (whole runs again, because nearly all points of a tile pass through it) and population 3 always writes.
// Without it such an index writes almost every word twice, the second time as scattered partial sectors (measured
// on BASELINE config 4 at full size: 9 of 23 ms).  (Tried for the same indexes and dropped: a "direct" population 1
// that skips the shared-memory tier and Q2 and has every lane gather the 32-bit tier codes of its own four points —
// bit-exact, but 1.25 instead of 1.00 ms per 100 M points on the config-4 stand-in: the gathers' L2 latency is
// exposed in every tile, where the queued batch is issued one tile ahead of its use.)
// kStage (lookup-table-heavy indexes): compiles in the warp-cooperative staging of lookup-table records
// (stage_records).  A compile-time choice because its registers slow the other instantiations down (measured with
// the code merely present: config-4 stand-in, counts only, 0.96 -> 1.10 ms per 100 M points).
// (Tried next to it and dropped: software-pipelining population 3's arena reads across batches for trees without
// palette nodes — issue the read when a batch is taken off Q3, resolve it when the next one is taken.  Bit-exact;
// 4 % on the config-4 stand-in counts only, nothing with first ids, nothing at all on full-size config 5 (171.9 vs
// 171.2 ms per 500 M points), and with JoinStats two instantiations kept thread-local copies of the parameter
// blocks: 9.7 instead of 1.3 ms.)
template <bool kIds, bool kStats, bool kDense, bool kLate = false, bool kStage = false, bool kDirect = false>
__global__ void __launch_bounds__(kJoinThreads, GJ_JOIN_MIN_BLOCKS)
join_kernel(const __grid_constant__ DevIndex ix, const __grid_constant__ JoinParams jp) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t tid = threadIdx.x;
  const uint32_t lane = tid & 31u;
  // (through a shuffle the compiler knows the warp index is warp-uniform, and keeps what derives from it — queue
  // addresses, tile bases — in uniform registers, outside the 64 registers a thread has here)
  const uint32_t warp = __shfl_sync(0xffffffffu, tid >> 5, 0);

  __shared__ EmitCtx s_ctx;
  if (tid == 0) {
    s_ctx = EmitCtx{ix.lut, ix.ids, ix.ring_len, jp.counts, jp.status, jp.ovf_point, jp.ovf_id, jp.ovf_ord,
                    jp.task_point, jp.task_slot, jp.task_ord, jp.base_index, jp.ovf_cap, jp.task_cap, ix.n_ids,
                    ix.ids_dense, jp.exact, jp.ovf_discard};
  }
  {  // stage the first directory tier (the direct form does not use it), clear the histogram
    const uint4* src = reinterpret_cast<const uint4*>(ix.dir16.table);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    const uint32_t n4 = kDirect ? 0u : (ix.dir16.n_table * 2u + 15u) / 16u;  // buffers are padded to 16 B
    for (uint32_t i = tid; i < n4; i += kJoinThreads) dst[i] = __ldg(src + i);
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem + jp.smem_hist_off);
    const uint32_t n_hist = jp.hist16 ? (ix.n_ids + 2u) / 2u : (ix.n_ids + 1u) * jp.hist_rep;
    for (uint32_t i = tid; i < n_hist; i += kJoinThreads) hist[i] = 0;
  }
  __syncthreads();

  // loop invariants in registers
  const uint32_t s_table = smem_addr(smem);
  const HistRef hist{smem_addr(smem + jp.smem_hist_off), jp.hist_rep, lane & (jp.hist_rep ? jp.hist_rep - 1u : 0u), jp.hist16,
                     jp.counts_priv ? jp.counts_priv + static_cast<size_t>(blockIdx.x % jp.n_priv) * ix.n_ids : nullptr};
  const uint32_t s_q2 = smem_addr(smem + jp.smem_queue_off) + warp * (kDirect ? kDirectBytesPerWarp : kQueueBytesPerWarp);
  const uint32_t s_q3 = s_q2 + (kDirect ? 2u * kDirectBufBytes : kQueue2Cap * 8u);
  const uint32_t s_stage = kStage && jp.smem_stage_off ? smem_addr(smem + jp.smem_stage_off) + warp * jp.stage_chunks * 16u : 0u;
  const uint32_t hist_spare = ix.n_ids;  // the histogram has n_ids + 1 rows
  const bool hist16_dense = !kDense && jp.hist16 != 0u && ix.ids_dense != 0;
  const bool tier_live = ix.dir16_live != 0;
  const uint32_t lane_lt = (1u << lane) - 1u;
  const uint32_t d1_w = ix.dir16.width, d1_h = ix.dir16.height, d1_pitch = ix.dir16.pitch;
  const uint32_t d1_x0 = ix.dir16.x0, d1_y0 = ix.dir16.y0;
  const uint32_t d1_shift = min(static_cast<uint32_t>(ix.dir16.shift) + 2u, 31u);  // on 32-bit-aligned coordinates
  // the 32-bit tier behind it: dirk, else dir2, else dir — its fields by value (a reference picked at run time among
  // three members of the parameter block is one of the things that made ptxas copy the block to local memory)
  const int tb_which = ix.dirk.n_table ? 2 : (ix.dir2.n_table ? 1 : 0);
  // (with the sparse refinement the tier is read from its copy whose link codes number the refinement records)
  const uint32_t* __restrict__ table2 =
      ix.link_sub ? ix.tier_links : (tb_which == 2 ? ix.dirk.table : (tb_which == 1 ? ix.dir2.table : ix.dir.table));
  const uint32_t tb_pitch = tb_which == 2 ? ix.dirk.pitch : (tb_which == 1 ? ix.dir2.pitch : ix.dir.pitch);
  const int tb_chunks = tb_which == 2 ? ix.dirk.chunks : (tb_which == 1 ? ix.dir2.chunks : ix.dir.chunks);
  const uint32_t qc_shift = ix.qc.shift, qc_mul = ix.qc.mul;
  const uint32_t qc_x0 = ix.qc.x0, qc_y0 = ix.qc.y0, qc_xc = ix.qc.x_clamp, qc_yc = ix.qc.y_clamp;
  const double2* __restrict__ pts = jp.pts;
  uint32_t* __restrict__ first_id = jp.first_id;
  const uint32_t n = static_cast<uint32_t>(jp.n);  // 1 <= n < 2^index_bits per launch (the bits above are queue flags)
  // A code resolves where it is read when it is one inlined payload that
  // emits: a true hit, or a candidate in approximate mode (join.cpp:100-108).
  const uint32_t need_interior = jp.exact ? 1u : 0u;
  const uint32_t emit_mask = 0xC0000000u | need_interior;
  const uint32_t emit_bits = kDirInline | need_interior;

  uint32_t n_valid = 0, false_hits = 0, solely_true = 0, refined = 0, cand_refs = 0;
  uint32_t q2_count = 0, q3_count = 0, q4_count = 0;  // warp-uniform

  // One resolved 32-bit directory code of a point of population 2: count,
  // stats, first id.  Returns true when the point is finished (inlined emit or
  // miss).  Population 1 has already written kNoMatch for it (see below), so
  // only an emit stores.
  auto settle = [&](uint32_t c, bool active, uint32_t i) -> bool {
    const bool emit = active && (c & emit_mask) == emit_bits;
    const bool miss = active && c == 0u;
    const uint32_t id = (c >> 1) & 0x1FFFFFFFu;
    if (kDense) {
      red_inc_shared_if(hist.smem + (id * hist.rep + hist.lane_rep) * 4u, emit);
    } else if (hist16_dense) {  // the 16-bit histogram with id == slot: one predicated add, no branch per lane
      red_add_shared_if(hist.smem + (id >> 1) * 4u, 1u << ((id & 1u) * 16u), emit);
    } else if (emit) {
      count_slot<kDense>(ix, jp, hist, id);
    }
    if (kStats) {
      false_hits += miss;
      solely_true += emit && (c & 1u);
      refined += emit && !(c & 1u);
      cand_refs += emit && !(c & 1u);
    }
    if (kIds) {
      if (kLate) {
        st32_if(first_id + i, emit ? id : kNoMatch, active);
      } else {
        st32_if(first_id + i, id, emit);
      }
    }
    return emit || miss;
  };

  // Population 3, one batch of open points (one per lane, `mine` = the lane
  // holds one): arena descent / dictionary / candidates.  Bit 31 of `iw`
  // marks an item whose word `c` is not a directory code: kQueueSlow (under
  // the slow mark) for a slow point, else — packed coding — the arena slot
  // under a link: its low 32 bits in `c`, the bits above them (arenas of 2^24
  // nodes = 32 GB and more) between the point index and bit 31 of `iw`.  All
  // 32 lanes go through it together because the record reservations are per warp.
  // The arena slot a flagged queue item names (see above).
  auto queued_slot = [&](uint32_t iw, uint32_t c) -> uint64_t {
    const uint32_t slot = (spread4((c >> 4) & 0xFu) << 1) | spread4(c & 0xFu);  // chunk_slot
    return (static_cast<uint64_t>((iw & 0x7FFFFFFFu) >> ix.qc.index_bits) << 32) | (static_cast<uint64_t>(c) & ~0xFFull) | slot;
  };
  // `deep` (kDirect only, warp-uniform): the batch comes from Q4 — items (point, node) whose walk continues below
  // the sub-cell bits the queue word carried.  In the queued form such a lane walks on inside its Q3 batch; here
  // it is set aside, because ONE such lane makes the whole batch wait for two more dependent DRAM round trips (the
  // point, then the deeper node) and run 75 more instructions — 2.5 % of the open points of BASELINE config 4, but
  // 85 % of its batches.
  auto resolve_open = [&](bool mine, uint32_t iw, uint32_t c, bool deep) {
    const uint32_t q_index_bits = ix.qc.index_bits, q_slow_mark = ix.qc.slow_mark;
    const uint32_t i = (kDirect && deep) ? iw : iw & ((1u << q_index_bits) - 1u);
    const bool flagged = (iw & 0x80000000u) != 0u;
    uint64_t entry = 0;
    bool defer = false;
    if (kDirect && deep) {
      if (mine) {
        const double2 q = __ldg(pts + i);
        uint32_t x, y;
        grid_xy(q.x, q.y, &x, &y);
        const uint32_t leaf_keep = ~((1u << (30 - ix.leaf_level)) - 1u);  // cell_id.cpp:93-94
        entry = walk_from(ix.arena, c, ix.prefix_level0 + 4 * tb_chunks + 4, (x & leaf_keep) << 2, (y & leaf_keep) << 2);
      }
    } else if (mine) {
      if (c == kQueueSlow && (iw & q_slow_mark) == q_slow_mark) {  // nothing decided yet: the reference's own sequence
        const double2 q = __ldg(pts + i);
        if (!latlng_valid(q.x, q.y)) {
          flag_error(jp.status, kErrInvalidPoint, jp.base_index + i);  // cell_id.cpp:83-85
          mine = false;
        } else {
          if (kStats) ++n_valid;
          entry = probe_raw_face0(ix, cell_from_point(q.x, q.y, ix.leaf_level));
        }
      } else if (flagged || (c & kDirLink)) {
        const int walk_level = ix.prefix_level0 + 4 * tb_chunks;
        uint64_t node = c & ~kDirLink;  // unpacked coding: the node under the link
        int level = walk_level;
        bool walk = true;
        if (flagged) {  // the word is (node - 1) * 256 + (y sub-cell bits << 4 | x sub-cell bits)
          uint64_t at = queued_slot(iw, c);
          const uint32_t slot = static_cast<uint32_t>(at) & 0xFFu;
          bool from_arena = true;
          if (ix.link_sub) {
            // sparse refinement: `at >> 8` numbers the link cell's record, not a node.  The code of the 16-slot run
            // holding `slot` (an L2 hit) is a terminal in the tier's own forms, or the link to the node itself.
            const uint32_t c2 = __ldg(ix.link_sub + static_cast<size_t>(at >> 8) * 16u + (slot >> 4));
            if (c2 & kDirLink) {
              at = static_cast<uint64_t>((c2 & ~kDirLink) - 1u) * kNodeSlots + slot;
            } else {
              from_arena = false;
              entry = c2 == 0u ? 0ull
                               : ((c2 & kDirInline) ? (static_cast<uint64_t>(c2 & 0x3FFFFFFFu) << 2) | 1u : __ldg(ix.dict + c2));
            }
          } else if (ix.node_pal) {  // the node's 128-byte palette form, usually an L2 hit
            const uint64_t* rec = ix.node_pal + (at >> 8) * 16u;
            const uint32_t codes = __ldg(reinterpret_cast<const uint32_t*>(rec + 4) + (slot >> 4));
            const uint64_t v = __ldg(rec + ((codes >> ((slot & 15u) * 2u)) & 3u));
            const uint64_t first = __ldg(rec);
            from_arena = first == ~0ull;
            entry = v;
          }
#ifdef GJ_EXP_NO_ARENA  // timing experiment: results are wrong
          from_arena = false;
          if (!ix.node_pal) entry = 0;
#endif
          if (from_arena) entry = ld_arena(ix.arena + at);
          walk = (entry & 3u) == 0u && entry != 0u;  // a link again: deeper than the queued bits reach
          node = entry >> 2;
          level += 4;
          if (kDirect && walk) {  // goes to Q4 as (point, node)
            defer = true;
            walk = false;
            c = static_cast<uint32_t>(node);
          }
        }
        if (walk) {
          const double2 q = __ldg(pts + i);
          uint32_t x, y;
          grid_xy(q.x, q.y, &x, &y);
          const uint32_t leaf_keep = ~((1u << (30 - ix.leaf_level)) - 1u);  // cell_id.cpp:93-94
          entry = walk_from(ix.arena, node, level, (x & leaf_keep) << 2, (y & leaf_keep) << 2);
        }
      } else if (c & kDirInline) {
        entry = (static_cast<uint64_t>(c & 0x3FFFFFFFu) << 2) | 1u;  // exact-mode candidate
      } else {
        entry = __ldg(ix.dict + c);
      }
    }
    if (kDirect && !deep) {  // (a Q4 batch adds nothing: walk_from ends in a terminal entry)
      const uint32_t mask = __ballot_sync(0xffffffffu, defer);
      sts64_if(s_q3 + (kDirectQueue3Cap - 1u - (q4_count + __popc(mask & lane_lt))) * 8u, i, c, defer);
      q4_count += __popc(mask);
      if (defer) {
        mine = false;
        entry = 0;
      }
    }
    const bool single = (static_cast<uint32_t>(entry) & 3u) == 1u &&
                        ((static_cast<uint32_t>(entry >> 2) & 1u) != 0u || !jp.exact);  // one payload that emits
    // two inlined payloads that both emit now (approximate mode, or two true hits), and no overflow record to write:
    // the boundary cells between two polygons of a tessellation — a quarter of all points on BASELINE config 4
    const bool pair_now = (static_cast<uint32_t>(entry) & 3u) == 2u && (!kIds || jp.ovf_discard) &&
                          (!jp.exact || ((entry >> 33) & (entry >> 2) & 1u) != 0u);
    const bool general = mine && entry != 0 && !single && !pair_now;
    EntryPlan plan{};
    if (general) plan = plan_entry<kIds>(ix, jp.exact != 0, entry);
    unsigned long long ovf_base = 0, task_base = 0;
    if (__any_sync(0xffffffffu, general)) {
      // (device-resident calls discard the overflow list: no reservation — on an index whose points mostly end in
      // two-candidate boundary cells the cursor is ONE address hit by every batch of every SM; measured on BASELINE
      // config 4 at full size: 16.7 M such atomics = 8 of 22 ms)
      if (kIds && !jp.ovf_discard) ovf_base = warp_reserve(&jp.status->overflow_count, plan.n_ovf, lane);
      if (jp.exact) task_base = warp_reserve(&jp.status->task_count, plan.n_tasks, lane);
    }
    uint32_t staged_at = 0;  // shared address of this lane's lookup-table record, 0 = walk it in global memory
    if (kStage && s_stage != 0u && __any_sync(0xffffffffu, general && plan.tag == 3u)) {
      const bool rec = general && plan.tag == 3u;
      const uint32_t first_chunk = plan.off >> 2;  // the record is words off .. off + 1 + n_refs of the table
      const uint32_t n_chunks = rec ? ((plan.off + 1u + plan.n_refs) >> 2) - first_chunk + 1u : 0u;
      const uint32_t at = stage_records(reinterpret_cast<const uint4*>(ix.lut), s_stage, jp.stage_chunks, lane, first_chunk, n_chunks);
      if (rec && at != ~0u) staged_at = s_stage + (at * 4u + (plan.off & 3u)) * 4u;
    }
    if (!mine) return;
    uint32_t first = kNoMatch;
    if (entry == 0) {
      if (kStats) ++false_hits;
    } else if (single) {
      first = static_cast<uint32_t>(entry >> 3) & 0x3FFFFFFFu;
      count_slot<kDense>(ix, jp, hist, first);
      if (kStats) {
        const bool interior = (entry >> 2) & 1u;
        solely_true += interior;
        refined += !interior;
        cand_refs += !interior;
      }
    } else if (pair_now) {
      const uint32_t pa = static_cast<uint32_t>(entry >> 33) & 0x7fffffffu, pb = static_cast<uint32_t>(entry >> 2) & 0x7fffffffu;
      first = (pa >> 1) | kMoreFlag;  // the second pair exists only as this flag (the overflow list is discarded)
      count_slot<kDense>(ix, jp, hist, pa >> 1);
      count_slot<kDense>(ix, jp, hist, pb >> 1);
      if (kStats) {
        const uint32_t n_cand = 2u - ((pa & 1u) + (pb & 1u));
        solely_true += n_cand == 0u;
        refined += n_cand != 0u;
        cand_refs += n_cand;
      }
    } else {
      first = emit_general<kIds, kDense>(&s_ctx, hist, entry, i, plan, ovf_base, task_base, staged_at);
      if (kStats) {
        solely_true += plan.n_cand == 0;
        refined += plan.n_cand != 0;
        cand_refs += plan.n_cand;
      }
    }
    if (kIds && (kLate || first != kNoMatch)) first_id[i] = first;
  };

  // Append (a, b) of the lanes with `open` to a warp queue; returns the new count.
  auto enqueue = [&](uint32_t queue, uint32_t count, bool open, uint32_t a, uint32_t b) -> uint32_t {
    const uint32_t mask = __ballot_sync(0xffffffffu, open);
    sts64_if(queue + (count + __popc(mask & lane_lt)) * 8u, a, b, open);
    return count + __popc(mask);
  };

  auto drain3 = [&](bool flush) {  // ONE resolve_open site for both queues
    for (;;) {
      __syncwarp();  // queue words appended by other lanes — to Q3 by the caller, to Q4 by the batch before — are visible
      const bool deep = kDirect && (q4_count >= 32u || (flush && q3_count == 0u && q4_count != 0u));
      if (!deep && !(q3_count >= 32u || (flush && q3_count))) break;
      uint32_t take, at;
      if (deep) {
        take = min(q4_count, 32u);
        q4_count -= take;
        at = kDirectQueue3Cap - 1u - (q4_count + min(lane, take - 1u));
      } else {
        take = min(q3_count, 32u);
        q3_count -= take;
        at = q3_count + min(lane, take - 1u);
      }
      const uint2 item = lds64(s_q3 + at * 8u);
      __syncwarp();
      resolve_open(lane < take, item.x, item.y, deep);
    }
  };

  // Population 2: Q2 items 32 at a time.  An item is (point | slow, w): w
  // indexes the 32-bit tier; a slow point (bit 31) skips the lookup and goes
  // straight on to Q3.  The batch is software-pipelined across tiles: its
  // gathers are ISSUED when the batch is taken off the queue and SETTLED one
  // tile later, so their L2 latency hides behind the next tile's streaming
  // work instead of stalling the warp.
  bool batch_open = false;      // a batch is in flight (warp-uniform)
  uint32_t batch_take = 0;      // its size
  uint32_t batch_point = 0;     // point | slow of this lane's item
  uint32_t batch_code = 0;      // the gather in flight
  uint32_t batch_slot = 0;      // packed coding: the node slot under a link

  auto settle_batch = [&]() {  // requires batch_open; appends to Q3 (the caller drains it)
    batch_open = false;
    const bool mine = lane < batch_take;
    const bool lookup = mine && (batch_point & 0x80000000u) == 0u;
    const bool done = settle(batch_code, lookup, batch_point);
    // a slow item (bit 31 set in Q2) travels on with kQueueSlow under the full slow mark of Q3
    uint32_t fwd = batch_code, fwd_point = lookup ? batch_point : batch_point | ix.qc.slow_mark;
    if (lookup && ix.qc.packed && (fwd & kDirLink)) {
      const uint64_t at = static_cast<uint64_t>((fwd & ~kDirLink) - 1u) * kNodeSlots + batch_slot;
      fwd = static_cast<uint32_t>(at);
      fwd_point |= 0x80000000u | (static_cast<uint32_t>(at >> 32) << ix.qc.index_bits);
    }
    q3_count = enqueue(s_q3, q3_count, mine && !done, fwd_point, fwd);
#ifdef GJ_EXP_NO_PHASE3  // timing experiment: results are wrong
    q3_count = 0;
#endif
  };

  auto issue_batch = [&](uint32_t take) {  // requires !batch_open
    q2_count -= take;
    const uint2 item = lds64(s_q2 + (q2_count + min(lane, take - 1u)) * 8u);
    __syncwarp();
    batch_take = take;
    batch_point = item.x;
    uint32_t idx = item.y;
    if (ix.qc.packed) {  // (Y << xbits) | X at level tb.level + 4, see DevQueueCoding
      const uint32_t X = item.y & (qc_mul - 1u), Y = item.y >> ix.qc.xbits;
      idx = (Y >> ix.qc.tier_shift) * tb_pitch + (X >> ix.qc.tier_shift);
      batch_slot = ((Y & ix.qc.sub_mask) << 4) | (X & ix.qc.sub_mask);  // spread into a node slot in population 3
    }
#ifdef GJ_EXP_NO_TB  // timing experiment: results are wrong (no gather into the 32-bit tier: every lookup misses)
    batch_code = (lane < take && (item.x & 0x80000000u) == 0u) ? 0u : kQueueSlow;
    (void)idx;
#else
    batch_code = ldg32_if(table2 + idx, lane < take && (item.x & 0x80000000u) == 0u, kQueueSlow);
#endif
    batch_open = true;
  };

  // One loop with ONE settle site and ONE Q3 drain site: population 3's code (resolve_open) is large, and with the
  // drains inlined at every settle it was instantiated nine times per kernel — 15 K SASS instructions, and
  // instruction-cache stalls to match on the lookup-table-heavy configs.
  auto drain2 = [&](bool flush) {
    __syncwarp();
    for (;;) {
      const bool had = batch_open;  // first turn: the batch issued one tile ago
      if (had) settle_batch();
      const bool more = q2_count >= 32u || (flush && q2_count != 0u);
      if (had || (flush && !more)) drain3(flush && !more);  // Q3 holds < 32 + 32 items at this point
      if (!more) break;
      issue_batch(min(q2_count, 32u));
      if (!(q2_count >= 32u || flush)) break;  // nothing more to take: leave the batch in flight for a tile
    }
  };

  constexpr uint32_t kTile = kJoinThreads * kPointsPerThread;
  const uint32_t n_tiles = (n + kTile - 1) / kTile;
  // Pull this warp's chunk of a tile the CTA will reach kPrefetchTiles tile
  // periods from now into L2 (one bulk prefetch per warp): its loads then pay
  // L2 latency instead of DRAM latency.
  auto prefetch_chunk = [&](uint32_t t) {  // t * kTile < 2^32: n < 2^31 and t stays within a few grids of n_tiles
    // per-lane line prefetches (the bulk form wants warp-uniform operands, which costs a uniformity loop)
    const uint32_t at = t * kTile + warp * kChunkPoints + lane * 8u;  // 8 points = one 128-byte line
    if (kPrefetchTiles != 0 && lane < kChunkPoints / 8u && at < n) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pts + at) : "memory");
    }
  };
#pragma unroll 1
  for (uint32_t k = 0; k < kPrefetchTiles; ++k) prefetch_chunk(blockIdx.x + k * gridDim.x);
  // One tile of this warp.  kFull: every point of the tile exists (all tiles
  // but possibly the last), so neither the loads nor population 1 test i < n.
  auto tile_body = [&](uint32_t tile, auto full_tag) {
    constexpr bool kFull = decltype(full_tag)::value;
    const uint32_t base = tile * kTile + warp * kChunkPoints + lane;  // point of slot j: base + 32 j
    prefetch_chunk(tile + kPrefetchTiles * gridDim.x);
    double2 p[kPointsPerThread];
#pragma unroll
    for (int j = 0; j < kPointsPerThread; ++j) {
      // streaming read, touched once: evict-first.  In the last tile lanes past
      // the end re-read the last point and are masked below.
      p[j] = __ldcs(pts + (kFull ? base + j * 32u : min(base + j * 32u, n - 1u)));
    }
    // ---- population 1: shared-memory tier, no branches, no calls ----
#pragma unroll
    for (int j = 0; j < kPointsPerThread; ++j) {
      const uint32_t i = base + j * 32u;
      const bool live = kFull || i < n;
      uint32_t x, y;  // left-aligned to 32 bits
      const bool ok = grid_xy_try(p[j].x, p[j].y, &x, &y) && live;  // valid, coordinates exact
      const uint32_t cx = min((x >> d1_shift) - d1_x0, d1_w);  // clamps into the all-miss padding
      const uint32_t cy = min((y >> d1_shift) - d1_y0, d1_h);
      // 0 = miss, 0xFFFF = look in the 32-bit tier, else 1 + payload.  (kLate, dead tier — polygons smaller than its
      // cells, BASELINE config 4: the answer is "look in the 32-bit tier" anyway, so the lookup is skipped.)
      const uint32_t e = (kLate && !tier_live) ? 0xFFFEu : lds16(s_table + (cy * d1_pitch + cx) * 2u) - 1u;
      const bool emit = ok && e < 0xFFFEu && (e & need_interior) == need_interior;
      const uint32_t id = e >> 1;
      if (kDense) {  // unconditional: lanes that do not emit count into a spare row past the last slot
        red_inc_shared_if(hist.smem + ((emit ? id : hist_spare) * hist.rep + hist.lane_rep) * 4u, true);
      } else if (emit) {
        count_slot<kDense>(ix, jp, hist, id);
      }
      if (kStats) {
        n_valid += ok;
        false_hits += ok && e == 0xFFFFFFFFu;
        solely_true += emit && (e & 1u);
        refined += emit && !(e & 1u);
        cand_refs += emit && !(e & 1u);
      }
      // First ids: every live lane writes its word here (kNoMatch unless it
      // emits), i.e. whole 128-byte runs per warp; later populations only
      // overwrite words that change, and those 4-byte stores then hit a
      // sector that is still dirty in L2 instead of forcing a 32-byte DRAM fill.
      const bool open = live && !emit && !(ok && e == 0xFFFFFFFFu);
      if (kIds) st32_if(first_id + i, emit ? id : kNoMatch, kLate ? live && !open : live);
#ifdef GJ_EXP_PHASE1_ONLY  // timing experiment: results are wrong
      continue;
#endif
      // what stays open is queued with its position in the 32-bit tier (DevQueueCoding)
      const uint32_t qx = min((x >> qc_shift) - qc_x0, qc_xc);
      const uint32_t qy = min((y >> qc_shift) - qc_y0, qc_yc);
      q2_count = enqueue(s_q2, q2_count, open, ok ? i : i | 0x80000000u, qy * qc_mul + qx);
    }
    drain2(false);
  };
  // 16-bit histogram: add the non-zero counters to the caller's counts and clear them (whole CTA)
  auto flush_hist16 = [&]() {
    __syncthreads();
    uint32_t* words = reinterpret_cast<uint32_t*>(smem + jp.smem_hist_off);
    for (uint32_t w = tid; w < (ix.n_ids + 1u) / 2u; w += kJoinThreads) {
      const uint32_t v = words[w];
      if (v == 0u) continue;
      words[w] = 0u;
      if (v & 0xFFFFu) atomicAdd(&jp.counts[2u * w], static_cast<unsigned long long>(v & 0xFFFFu));
      if ((v >> 16) && 2u * w + 1u < ix.n_ids) atomicAdd(&jp.counts[2u * w + 1u], static_cast<unsigned long long>(v >> 16));
    }
    __syncthreads();
  };
  // ---- kDirect: the form for indexes whose shared-memory tier is dead (polygons smaller than its cells: BASELINE
  // config 4).  There EVERY point has to be looked up in the 32-bit tier, and sending all of them through Q2 —
  // compact, store, load, decode, gather, settle — was 150 of the 240 instructions a point cost.  Here a lane gathers
  // the codes of its own four points where it loads them, as asynchronous copies into shared memory (LDGSTS, no
  // register waits for them), and settles them one tile LATER from there, so the gathers' L2 latency hides behind a
  // whole tile of work (issued and consumed in the same tile it was exposed: 1.25 instead of 1.00 ms per 100 M
  // points).  Instead of Q2 a warp has two staging buffers: 128 codes + 128 node slots (the 4 + 4 sub-cell bits
  // under a link) = 640 bytes each.  Populations 1 and 2 collapse into ~33 instructions per point to issue and ~62
  // to settle; population 3 is resolve_open as before, except that walks below the queued sub-cell bits wait in a
  // queue of their own (Q4, see resolve_open).  First ids are written as in the kLate form.
  static_assert(!kDirect || (kLate == kIds && !kStage), "kDirect writes first ids late and does not stage records");
  auto direct_issue = [&](uint32_t tile, uint32_t buf, auto full_tag) {
    constexpr bool kFull = decltype(full_tag)::value;
    const uint32_t base = tile * kTile + warp * kChunkPoints + lane;
    prefetch_chunk(tile + kPrefetchTiles * gridDim.x);
    double2 p[kPointsPerThread];
#pragma unroll
    for (int j = 0; j < kPointsPerThread; ++j) {
      p[j] = __ldcs(pts + (kFull ? base + j * 32u : min(base + j * 32u, n - 1u)));
    }
    const uint32_t s_code = s_q2 + buf * kDirectBufBytes + lane * 4u;
    const uint32_t s_slot = s_q2 + buf * kDirectBufBytes + kChunkPoints * 4u + lane;
    const uint32_t tier_shift = ix.qc.tier_shift, sub_mask = ix.qc.sub_mask;
#pragma unroll
    for (int j = 0; j < kPointsPerThread; ++j) {
      const bool live = kFull || base + j * 32u < n;
      uint32_t x, y;  // left-aligned to 32 bits
      const bool ok = grid_xy_try(p[j].x, p[j].y, &x, &y) && live;
      const uint32_t qx = min((x >> qc_shift) - qc_x0, qc_xc);  // clamps into the all-miss padding
      const uint32_t qy = min((y >> qc_shift) - qc_y0, qc_yc);
      // packed coding: (qx, qy) is the cell at the next node boundary, tier_shift levels below the tier's; unpacked:
      // the tier's own cell (tier_shift = 0, sub_mask = 0)
      const uint32_t idx = (qy >> tier_shift) * tb_pitch + (qx >> tier_shift);
      cp_async4_if(s_code + j * 128u, table2 + idx, ok);
      // not looked up: a slow point (decided in population 3), or a lane past the end
      sts32_if(s_code + j * 128u, live ? kQueueSlow : kDirectSkip, !ok);
      sts8(s_slot + j * 32u, ((qy & sub_mask) << 4) | (qx & sub_mask));
      if (kStats) n_valid += ok;
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // Settles the tile staged in `buf` (its gathers have landed: the caller waited for the copy group): twice two
  // straight-line rounds and the drain site.
  auto direct_settle = [&](uint32_t tile, uint32_t buf) {
    const uint32_t base = tile * kTile + warp * kChunkPoints + lane;
    const uint32_t s_code = s_q2 + buf * kDirectBufBytes + lane * 4u;
    const uint32_t s_slot = s_q2 + buf * kDirectBufBytes + kChunkPoints * 4u + lane;
    const uint32_t q_packed = ix.qc.packed, q_index_bits = ix.qc.index_bits, q_slow_mark = ix.qc.slow_mark;
#pragma unroll 1
    for (uint32_t half = 0; half < kPointsPerThread / kDirectRounds; ++half) {  // a few rounds, then the drain site
#pragma unroll
      for (uint32_t jj = 0; jj < kDirectRounds; ++jj) {
        const uint32_t j = half * kDirectRounds + jj;
        const uint32_t i = base + j * 32u;
        const uint32_t c = lds32(s_code + j * 128u);
        const uint32_t slot = lds8(s_slot + j * 32u);
        const bool mine = c != kDirectSkip;
        const bool lookup = c < kDirectSkip;  // neither marker
        const bool done = settle(c, lookup, i);
        uint32_t fwd = c, fwd_point = lookup ? i : i | q_slow_mark;
        if (lookup && q_packed && (c & kDirLink)) {  // as settle_batch: the arena slot under the link travels on
          const uint64_t at = static_cast<uint64_t>((c & ~kDirLink) - 1u) * kNodeSlots + slot;
          fwd = static_cast<uint32_t>(at);
          fwd_point |= 0x80000000u | (static_cast<uint32_t>(at >> 32) << q_index_bits);
        }
        q3_count = enqueue(s_q3, q3_count, mine && !done, fwd_point, fwd);
      }
      drain3(false);  // Q3 and Q4 hold < 32 items each again
    }
  };

  const uint32_t n_full_tiles = n / kTile;
  uint32_t tile = blockIdx.x;
  // (one loop for both counting forms: a second copy of the tile body is 2 500 instructions of cache footprint)
  uint32_t since = 0;
  if constexpr (kDirect) {
    uint32_t prev = ~0u, buf = 0;  // the tile staged one turn ago, the buffer the next tile goes to
    for (; tile < n_tiles; tile += gridDim.x) {  // (at most one CTA meets the partial last tile, as its last)
      if (tile < n_full_tiles) {
        direct_issue(tile, buf, std::true_type{});
      } else {
        direct_issue(tile, buf, std::false_type{});
      }
      if (prev != ~0u) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // all but the group just committed
        direct_settle(prev, buf ^ 1u);
      }
      prev = tile;
      buf ^= 1u;
      // every warp of the CTA settles the same tiles, so the barriers inside the flush line up
      if (jp.hist16 && ++since == kHist16FlushTiles) {
        since = 0;
        flush_hist16();
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    if (prev != ~0u) direct_settle(prev, buf ^ 1u);
    drain3(true);
  } else {
  for (; tile < n_full_tiles; tile += gridDim.x) {
    tile_body(tile, std::true_type{});
    // every warp of the CTA runs the same number of tiles, so the barriers inside the flush line up
    if (jp.hist16 && ++since == kHist16FlushTiles) {
      since = 0;
      flush_hist16();
    }
  }
  if (tile < n_tiles) tile_body(tile, std::false_type{});  // the partial last tile, in one CTA
  drain2(true);  // settles what is in flight and flushes both queues
  }

  if (jp.hist16) flush_hist16();
  __syncthreads();
  if (jp.hist_rep) {  // fold the replicas, one global add per non-zero slot
    const uint32_t* hist_words = reinterpret_cast<const uint32_t*>(smem + jp.smem_hist_off);
    for (uint32_t s = tid; s < ix.n_ids; s += kJoinThreads) {
      uint32_t sum = 0;
      for (uint32_t r = 0; r < jp.hist_rep; ++r) sum += hist_words[s * jp.hist_rep + r];
      if (sum) atomicAdd(&jp.counts[s], static_cast<unsigned long long>(sum));
    }
  }
  if (kStats && jp.stats) {  // JoinStats, join.hpp:77-84
    uint32_t v[5] = {n_valid, false_hits, solely_true, refined, cand_refs};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    }
    if (lane == 0) {
      atomicAdd(&jp.stats[0], static_cast<unsigned long long>(v[0]));                // probes
      if (jp.exact) atomicAdd(&jp.stats[1], static_cast<unsigned long long>(v[4]));  // pip_tests
      atomicAdd(&jp.stats[2], static_cast<unsigned long long>(v[1]));                // false_hits
      atomicAdd(&jp.stats[3], static_cast<unsigned long long>(v[2]));                // solely_true_hits
      atomicAdd(&jp.stats[4], static_cast<unsigned long long>(v[3]));                // refinement_entered
      atomicAdd(&jp.stats[5], static_cast<unsigned long long>(v[4]));                // candidate_refs
    }
  }
}

// Does the entry hold at least one candidate (non-interior) reference?  The
// test Act::train applies to every training point (act.cpp:414-440).
__device__ __forceinline__ bool entry_has_candidate(const DevIndex& ix, uint64_t e) {
  const uint32_t tag = static_cast<uint32_t>(e) & 3u;
  if (e == 0 || tag == 0u) return false;
  if (tag == 1u) return ((e >> 2) & 1u) == 0u;
  if (tag == 2u) return ((e >> 33) & 1u) == 0u || ((e >> 2) & 1u) == 0u;
  const uint32_t off = static_cast<uint32_t>(e >> 2) & 0x7fffffffu;  // [t, ids, c, ids]
  return __ldg(ix.lut + off + 1u + __ldg(ix.lut + off)) != 0u;
}

// Training pre-pass: flag[i] = 1 when point i probes into a candidate-bearing
// cell, else 0 (as u32, ready for the exclusive scan that orders the output).
__global__ void __launch_bounds__(256)
candidate_flags_kernel(const __grid_constant__ DevIndex ix, const double2* __restrict__ pts, uint64_t n,
                       uint64_t base_index, uint32_t* __restrict__ flags, DevStatus* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* s_table = reinterpret_cast<uint32_t*>(smem);
  for (uint32_t i = threadIdx.x; i < ix.dir.n_table; i += blockDim.x) s_table[i] = __ldg(ix.dir.table + i);
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double2 p = __ldcs(pts + i);
    uint32_t f = 0;
    if (latlng_valid(p.x, p.y)) {
      f = entry_has_candidate(ix, probe_point(ix, s_table, p.x, p.y)) ? 1u : 0u;
    } else {
      flag_error(status, kErrInvalidPoint, base_index + i);
    }
    flags[i] = f;
  }
}

// out[offset[i]] = base_index + i for every flagged point (offsets from the scan).
__global__ void __launch_bounds__(256)
candidate_scatter_kernel(const uint32_t* __restrict__ flags, const uint64_t* __restrict__ offset, uint64_t n,
                         uint64_t base_index, uint64_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (flags[i]) out[offset[i]] = base_index + i;
  }
}

// counts[s] += sum over the SMs' private copies, which are left zero for the next launch.
__global__ void __launch_bounds__(256)
fold_private_counts_kernel(uint32_t* __restrict__ priv, uint32_t n_copies, uint32_t n_ids,
                           unsigned long long* __restrict__ counts) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n_ids; s += gridDim.x * blockDim.x) {
    unsigned long long sum = 0;
    for (uint32_t c = 0; c < n_copies; ++c) {
      const size_t at = static_cast<size_t>(c) * n_ids + s;
      const uint32_t v = priv[at];
      if (v) {
        sum += v;
        priv[at] = 0;
      }
    }
    if (sum) counts[s] += sum;  // one thread per slot, and the join kernels have finished
  }
}

// Entries only: bitwise Act::probe(cell_from_point(p, k_max/2)).
__global__ void __launch_bounds__(256)
probe_points_kernel(const __grid_constant__ DevIndex ix, const double2* __restrict__ pts, uint64_t n,
                    uint64_t base_index, uint64_t* __restrict__ out, DevStatus* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* s_table = reinterpret_cast<uint32_t*>(smem);
  for (uint32_t i = threadIdx.x; i < ix.dir.n_table; i += blockDim.x) s_table[i] = __ldg(ix.dir.table + i);
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double2 p = __ldcs(pts + i);
    uint64_t e = 0;
    if (latlng_valid(p.x, p.y)) {
      e = probe_point(ix, s_table, p.x, p.y);
    } else {
      flag_error(status, kErrInvalidPoint, base_index + i);
    }
    out[i] = e;
  }
}

// cell_from_point over an array (cell_id.cpp:82-95).
__global__ void __launch_bounds__(256)
cells_kernel(const double2* __restrict__ pts, uint64_t n, int level, uint64_t base_index,
             uint64_t* __restrict__ out, DevStatus* status) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double2 p = __ldcs(pts + i);
    uint64_t raw = 0;
    if (latlng_valid(p.x, p.y)) {
      raw = cell_from_point(p.x, p.y, level);
    } else {
      flag_error(status, kErrInvalidPoint, base_index + i);
    }
    out[i] = raw;
  }
}

// Same without the directory (plain arena walk): the cross-check that the
// directory changes nothing, and the all-faces raw-id entry point.
__global__ void __launch_bounds__(256)
probe_cells_kernel(const __grid_constant__ DevIndex ix, const uint64_t* __restrict__ raw, uint64_t n,
                   uint64_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    out[i] = probe_raw(ix, __ldg(raw + i));
  }
}

// ---------------------------------------------------------------------------
// K2.  PIP refine of the candidate tasks K1 queued (exact mode).
//
// One thread per (point, polygon) task, tasks in arrival order.  The polygon's
// edges are not scanned: the host cut every polygon into latitude strips at
// index-create time (StripMeta), so a task reads its strip's handful of
// 32-byte edge records (L1/L2-resident: a few MB for all polygons) and runs
// the reference's exact fp64 edge arithmetic (pip_edge) on those only.  An
// edge outside the point's strip has a latitude range — widened by pip_edge's
// own 1e-9 deg rejection margin — that does not contain the point, so it can
// neither be within the boundary tolerance nor cross the point's ray; the
// boundary any() and the crossing parity over the remaining edges are the
// reference's result bit for bit (geometry.cpp:184-204).  Work per task is a
// few edges whatever the polygon's size, so a grid-stride loop balances.
//
// (Two earlier designs, kept in git history: thread-per-task over all edges
// staged in shared memory per polygon bucket — 1.36 ms per 3.5 M tasks, fp64
// pipe bound; the same with an fp32 filter-then-compact pass — 0.65 ms.)
// ---------------------------------------------------------------------------
struct RefineParams {
  const double2* pts;
  uint64_t base_index;
  const uint32_t* task_point;
  const uint32_t* task_slot;
  const uint32_t* task_ord;
  uint64_t task_cap;
  unsigned long long* counts;
  // ids mode: accepted candidates become overflow records
  uint64_t* ovf_point;
  uint32_t* ovf_id;
  uint32_t* ovf_ord;
  uint64_t ovf_cap;
  // pairs mode: one flag per task (1 = the candidate passed)
  uint8_t* task_pass;
  DevStatus* status;
  int32_t want_ids;
  int32_t smem_counts;  // the launch carries n_ids * 4 bytes of dynamic shared memory
  uint32_t* counts_priv;  // otherwise: [n_priv][n_ids] u32 private copies (may be null)
  uint32_t n_priv;
};

// kIndexed: the strip lists hold vertex indices (DevIndex::strip_eidx) instead of 32-byte edge records.
template <bool kIndexed>
__global__ void __launch_bounds__(kRefineThreads, 4)
refine_kernel(const __grid_constant__ DevIndex ix, RefineParams rp) {
  constexpr int kWarps = kRefineThreads / 32;
  constexpr uint32_t kListCap = 64;  // < 32 left over + up to 32 appended per loop step
  // (edge record, lane << 2 | kinds) of the edge evaluations that need a
  // division: the distance to the edge (kind bit 0) and/or the crossing
  // abscissa (bit 1).  They are rare per task but would each run at 1/32
  // utilisation inside the per-lane loop, so they are compacted and batched.
  __shared__ uint2 s_list[kWarps][kListCap];
  __shared__ uint32_t s_result[kWarps][32];  // bit 0: on the boundary, bit 1: crossing parity
  // per-polygon counts of this CTA (when the id table fits): global atomics
  // on a few hundred hot words serialise at L2
  extern __shared__ uint32_t s_counts[];
  const bool local_counts = rp.smem_counts != 0;
  if (local_counts) {
    for (uint32_t s = threadIdx.x; s < ix.n_ids; s += kRefineThreads) s_counts[s] = 0;
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t lane_lt = (1u << lane) - 1u;
  const uint64_t n_tasks = min(static_cast<uint64_t>(rp.status->task_count), rp.task_cap);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  // whole warps stay in the loop together
  for (uint64_t t0 = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) & ~31ull; t0 < n_tasks;
       t0 += stride) {
    const uint64_t task = t0 + lane;
    const bool active = task < n_tasks;
    uint32_t point = 0, slot = 0, e_begin = 0, len = 0;
    double qx = 0.0, qy = 0.0;
    if (active) {
      point = rp.task_point[task];
      slot = rp.task_slot[task];
      const double2 p = __ldg(rp.pts + point);
      qx = p.y;  // x = lng, y = lat (geometry.cpp:35)
      qy = p.x;
      const StripMeta m = ix.strip_meta[slot];
      if (m.k != 0u) {
        const uint32_t st = strip_of(qy, m.y0, m.inv_h, m.k);
        e_begin = __ldg(ix.strip_ptr + m.ptr_base + st);
        len = __ldg(ix.strip_ptr + m.ptr_base + st + 1) - e_begin;
      }
    }
    __syncwarp();
    s_result[warp][lane] = 0;
    __syncwarp();

    // Evaluate up to 32 listed (task, edge) pairs with all lanes.
    auto drain = [&](uint32_t first, uint32_t take) {
      const uint2 item = s_list[warp][first + min(lane, take - 1u)];
      const uint32_t owner = item.y >> 2;  // lane that holds the point
      const double ox = __shfl_sync(0xffffffffu, qx, owner);
      const double oy = __shfl_sync(0xffffffffu, qy, owner);
      if (lane < take) {
        double ax, ay, bx, by;
        if (kIndexed) {
          load_edge_indexed(ix.ring_xy, ix.strip_eidx, item.x, &ax, &ay, &bx, &by);
        } else {
          load_edge(ix.strip_edges + item.x, &ax, &ay, &bx, &by);
        }
        if ((item.y & 1u) && pip_edge_on_boundary(ox, oy, ax, ay, bx, by)) atomicOr(&s_result[warp][owner], 1u);
        if ((item.y & 2u) && pip_edge_crosses(ox, oy, ax, ay, bx, by)) atomicXor(&s_result[warp][owner], 2u);
      }
    };

    // The batch's (task, edge) pairs, flattened: pair g belongs to the first
    // lane whose inclusive prefix of list lengths exceeds g.  Every loop step
    // classifies 32 real pairs whatever the individual list lengths are.
    uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t up = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= static_cast<uint32_t>(o)) incl += up;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t excl = incl - len;
    uint32_t n_list = 0;
    for (uint32_t k = 0; k < total; k += 32u) {
      const uint32_t g = k + lane;
      uint32_t owner = 0;  // number of lanes with incl <= g
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, incl, min(owner + step - 1u, 31u));
        if (v <= g) owner += step;
      }
      const bool real = g < total;
      const uint32_t src = min(owner, 31u);
      const uint32_t e = __shfl_sync(0xffffffffu, e_begin, src) + (g - __shfl_sync(0xffffffffu, excl, src));
      const double ox = __shfl_sync(0xffffffffu, qx, src);
      const double oy = __shfl_sync(0xffffffffu, qy, src);
      uint32_t kinds = 0;
      if (real) {
        double ax, ay, bx, by;
        if (kIndexed) {
          load_edge_indexed(ix.ring_xy, ix.strip_eidx, e, &ax, &ay, &bx, &by);
        } else {
          load_edge(ix.strip_edges + e, &ax, &ay, &bx, &by);
        }
        kinds = pip_edge_classify(ox, oy, ax, ay, bx, by);
      }
      if (kinds & 4u) atomicXor(&s_result[warp][src], 2u);  // crosses for certain: no division
      kinds &= 3u;
      const uint32_t mask = __ballot_sync(0xffffffffu, kinds != 0u);
      if (kinds) s_list[warp][n_list + __popc(mask & lane_lt)] = make_uint2(e, (src << 2) | kinds);
      n_list += __popc(mask);
      if (n_list >= 32u) {
        __syncwarp();
        n_list -= 32u;
        drain(n_list, 32u);
        __syncwarp();
      }
    }
    __syncwarp();
    if (n_list) drain(0, n_list);
    __syncwarp();
    const bool pass = active && s_result[warp][lane] != 0u;

    if (rp.task_pass) {
      if (active) rp.task_pass[task] = pass ? 1 : 0;
      continue;
    }
    if (pass) {
      if (local_counts) {
        atomicAdd(&s_counts[slot], 1u);
      } else if (rp.counts_priv) {
        atomicAdd(rp.counts_priv + static_cast<size_t>(blockIdx.x % rp.n_priv) * ix.n_ids + slot, 1u);
      } else {
        atomicAdd(&rp.counts[slot], 1ull);
      }
    }
    if (rp.want_ids) {
      const uint32_t pass_mask = __ballot_sync(0xffffffffu, pass);
      if (pass_mask == 0u) continue;
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(&rp.status->overflow_count, static_cast<unsigned long long>(__popc(pass_mask)));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base + __popc(pass_mask) > rp.ovf_cap) {
        if (lane == 0) atomicOr(&rp.status->flags, kErrOverflowCap);
      } else if (pass) {
        const uint64_t w = base + __popc(pass_mask & lane_lt);
        rp.ovf_point[w] = rp.base_index + point;
        rp.ovf_id[w] = __ldg(ix.ids + slot);
        rp.ovf_ord[w] = rp.task_ord[task];
      }
    }
  }
  __syncthreads();
  if (local_counts) {
    for (uint32_t sl = threadIdx.x; sl < ix.n_ids; sl += kRefineThreads) {
      if (s_counts[sl]) atomicAdd(&rp.counts[sl], static_cast<unsigned long long>(s_counts[sl]));
    }
  }
}

// ---------------------------------------------------------------------------
// Materialised pairs in CSR form (join_exact / join_approx, join.cpp:131-140,
// 237-247): row_ptr[n + 1] and polygon_id[] in the reference's emit order
// (ascending point index, references in index order, join.hpp:125-127).
//
//   probe_points_kernel   entries[i]                       (above)
//   pairs_plan_kernel     per point: reference count; exact mode: candidate
//                         tasks (contiguous per point, in reference order)
//                         and the point's first task
//   refine_kernel         pass flag per task               (K2, exact mode)
//   pairs_count_kernel    pairs the point really emits
//   scan_* kernels        exclusive scan -> row_ptr
//   pairs_fill_kernel     polygon ids
// ---------------------------------------------------------------------------
struct PairsParams {
  const uint64_t* entries;  // [n]
  uint64_t n;
  uint64_t base_index;
  uint32_t* n_refs;         // [n] out (plan): references behind the entry
  uint32_t* task_base;      // [n] out (plan, exact): first task of the point
  uint32_t* task_point;
  uint32_t* task_slot;
  uint32_t* task_ord;
  uint64_t task_cap;
  const uint8_t* task_pass; // K2's verdicts (count / fill)
  uint32_t* count;          // [n] out (count): pairs of the point
  const uint64_t* row_ptr;  // [n + 1] (fill)
  uint32_t* out_id;         // (fill)
  uint64_t out_cap;         // (fill) ids that fit out_id; a row ending beyond it is not written (kErrOverflowCap)
  const uint64_t* out_sub;  // (fill) optional: *out_sub is subtracted from the row offsets (chunk-local id buffers)
  unsigned long long* stats;  // [6] or null
  DevStatus* status;
  int32_t exact;
};

// k-th reference of an entry: (polygon_id << 1) | interior (act.hpp:169-196)
__device__ __forceinline__ uint32_t entry_ref(const DevIndex& ix, uint64_t entry, uint32_t tag, uint32_t off,
                                              uint32_t t, uint32_t k) {
  if (tag == 1u) return static_cast<uint32_t>(entry >> 2) & 0x7fffffffu;
  if (tag == 2u) return static_cast<uint32_t>(k == 0 ? entry >> 33 : entry >> 2) & 0x7fffffffu;
  return k < t ? (__ldg(ix.lut + off + 1 + k) << 1) | 1u : (__ldg(ix.lut + off + 2 + k) << 1);
}

__global__ void __launch_bounds__(256)
pairs_plan_kernel(const __grid_constant__ DevIndex ix, PairsParams pp) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint32_t probes = 0, false_hits = 0, solely_true = 0, refined = 0, cand_refs = 0;
  for (uint64_t i0 = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) & ~31ull; i0 < pp.n; i0 += stride) {
    const uint64_t i = i0 + lane;
    const bool live = i < pp.n;
    const uint64_t entry = live ? pp.entries[i] : 0;
    EntryPlan e{};
    if (entry != 0) e = plan_entry<false>(ix, pp.exact != 0, entry);
    if (live) {
      ++probes;
      if (entry == 0) {
        ++false_hits;
      } else if (e.n_cand == 0) {
        ++solely_true;
      } else {
        ++refined;
        cand_refs += e.n_cand;
      }
    }
    unsigned long long task_base = 0;
    if (pp.exact && __any_sync(0xffffffffu, e.n_tasks != 0u)) {
      task_base = warp_reserve(&pp.status->task_count, e.n_tasks, lane);
    }
    if (!live) continue;
    pp.n_refs[i] = e.n_refs;
    if (e.n_tasks) {
      const bool ok = task_base + e.n_tasks <= pp.task_cap;
      if (!ok) atomicOr(&pp.status->flags, kErrTaskCap);
      pp.task_base[i] = static_cast<uint32_t>(task_base);
      uint32_t w = 0;
      for (uint32_t k = 0; k < e.n_refs && ok; ++k) {
        const uint32_t p = entry_ref(ix, entry, e.tag, e.off, e.t, k);
        if (p & 1u) continue;
        const uint32_t slot = id_to_slot(ix, p >> 1);
        if (__ldg(ix.ring_len + slot) == 0u) flag_error(pp.status, kErrUnknownPolygon, pp.base_index + i);
        pp.task_point[task_base + w] = static_cast<uint32_t>(i);
        pp.task_slot[task_base + w] = slot;
        pp.task_ord[task_base + w] = k;
        ++w;
      }
    }
  }
  if (pp.stats) {  // JoinStats, join.hpp:77-84
    uint32_t v[5] = {probes, false_hits, solely_true, refined, cand_refs};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    }
    if (lane == 0) {
      atomicAdd(&pp.stats[0], static_cast<unsigned long long>(v[0]));
      if (pp.exact) atomicAdd(&pp.stats[1], static_cast<unsigned long long>(v[4]));
      atomicAdd(&pp.stats[2], static_cast<unsigned long long>(v[1]));
      atomicAdd(&pp.stats[3], static_cast<unsigned long long>(v[2]));
      atomicAdd(&pp.stats[4], static_cast<unsigned long long>(v[3]));
      atomicAdd(&pp.stats[5], static_cast<unsigned long long>(v[4]));
    }
  }
}

// count (kFill = false) or write (kFill = true) the pairs of every point
template <bool kFill>
__global__ void __launch_bounds__(256)
pairs_emit_kernel(const __grid_constant__ DevIndex ix, PairsParams pp) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < pp.n; i += stride) {
    const uint32_t n_refs = pp.n_refs[i];
    uint32_t emitted = 0;
    if (n_refs) {
      const uint64_t entry = pp.entries[i];
      const uint32_t tag = static_cast<uint32_t>(entry) & 3u;
      uint32_t off = 0, t = 0;
      if (tag == 3u) {
        off = static_cast<uint32_t>(entry >> 2) & 0x7fffffffu;
        t = __ldg(ix.lut + off);
      }
      uint64_t out = kFill ? pp.row_ptr[i] : 0;
      if (kFill) {
        const uint64_t sub = pp.out_sub ? *pp.out_sub : 0;
        out -= sub;
        if (pp.row_ptr[i + 1] - sub > pp.out_cap) {  // (row_ptr[i + 1] exists: the scan writes the end offset too)
          atomicOr(&pp.status->flags, kErrOverflowCap);  // the caller's id array is too small: sizes still come back
          continue;
        }
      }
      uint32_t cand = 0;
      const uint32_t task_base = pp.exact ? pp.task_base[i] : 0u;
      for (uint32_t k = 0; k < n_refs; ++k) {
        const uint32_t p = entry_ref(ix, entry, tag, off, t, k);
        bool emit = true;
        if (pp.exact && !(p & 1u)) emit = pp.task_pass[task_base + cand++] != 0;
        if (emit) {
          if (kFill) pp.out_id[out + emitted] = p >> 1;
          ++emitted;
        }
      }
    }
    if (!kFill) pp.count[i] = emitted;
  }
}

// Exclusive scan of u32 counts into u64 offsets: block sums, a single-CTA
// scan of the block sums, then the per-block scan with its prefix.
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint64_t block_exclusive_scan(uint64_t v, uint64_t* total) {
  __shared__ uint64_t s_warp[kScanThreads / 32];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint64_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t up = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += up;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint64_t w = lane < kScanThreads / 32 ? s_warp[lane] : 0;
    uint64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t up = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= static_cast<uint32_t>(o)) wi += up;
    }
    if (lane < kScanThreads / 32) s_warp[lane] = wi - w;  // exclusive warp prefix
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  const uint64_t res = s_warp[warp] + incl - v;
  __syncthreads();
  return res;
}

__global__ void __launch_bounds__(kScanThreads)
scan_block_sums_kernel(const uint32_t* __restrict__ in, uint64_t n, uint64_t* __restrict__ block_sums) {
  __shared__ uint64_t s_total;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  uint64_t v = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) v += base + k < n ? in[base + k] : 0u;
  block_exclusive_scan(v, &s_total);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = s_total;
}

__global__ void __launch_bounds__(kScanThreads)
scan_sums_kernel(uint64_t* __restrict__ block_sums, uint32_t n_blocks, uint64_t* __restrict__ grand_total) {
  __shared__ uint64_t s_total;
  uint64_t carry = 0;
  for (uint32_t b0 = 0; b0 < n_blocks; b0 += kScanThreads) {
    const uint32_t b = b0 + threadIdx.x;
    const uint64_t v = b < n_blocks ? block_sums[b] : 0;
    const uint64_t ex = block_exclusive_scan(v, &s_total);
    if (b < n_blocks) block_sums[b] = carry + ex;
    carry += s_total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *grand_total = carry;
}

// out[i] = offset (+ *running when given: a total kept on the device) + exclusive prefix of in[0..i); with
// `write_end` the element after the last one gets the inclusive total (the n + 1-th row offset).
__global__ void __launch_bounds__(kScanThreads)
scan_apply_kernel(const uint32_t* __restrict__ in, uint64_t n, const uint64_t* __restrict__ block_sums,
                  uint64_t offset, uint64_t* __restrict__ out, const uint64_t* __restrict__ running = nullptr,
                  bool write_end = false) {
  __shared__ uint64_t s_total;
  if (running) offset += *running;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  uint32_t item[kScanItems];
  uint64_t v = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    item[k] = base + k < n ? in[base + k] : 0u;
    v += item[k];
  }
  uint64_t run = offset + block_sums[blockIdx.x] + block_exclusive_scan(v, &s_total);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = run;
    run += item[k];
    if (write_end && base + k + 1 == n) out[n] = run;
  }
}

// *running += *chunk_total (one thread): the pair count so far, kept on the device so that consecutive chunks of
// the CSR pipeline need no host round trip.
__global__ void advance_base_kernel(uint64_t* running, const uint64_t* chunk_total) { *running += *chunk_total; }

// v[i] += offset: a replica's CSR row offsets moved behind the pairs of the ranges before it (gj_group_*)
__global__ void __launch_bounds__(256)
add_offset_kernel(uint64_t* __restrict__ v, uint64_t n, uint64_t offset) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) v[i] += offset;
}

}  // namespace gj
