// Device-side data layout and the per-point hot path (sm_100a).
//
// Compiled with -fmad=false: the reference's Release build contains no FMA
// (SURVEY.md T1), and grid_coord / pip_test are rounding-sensitive.  The few
// floating-point expressions that define results are additionally spelled
// with explicit round-to-nearest intrinsics so their operation order is the
// reference's regardless of compiler flags.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace gj {

constexpr int kNodeSlots = 256;             // ActConfig::kFanout, act.hpp:36
// Directory codes (u32): 0 = miss; bit 31 = continue the walk at node
// (code & 0x7fffffff); bit 30 = one inlined payload ((polygon_id << 1) |
// interior, ids below 2^29) in the low 30 bits; anything else indexes `dict`.
constexpr uint32_t kDirLink = 0x80000000u;
constexpr uint32_t kDirInline = 0x40000000u;
constexpr uint32_t kNoMatch = 0xFFFFFFFFu;
constexpr uint32_t kDeferred = 0xFFFFFFFEu;
constexpr uint32_t kMoreFlag = 0x80000000u;
constexpr uint64_t kNoBadIndex = ~0ull;

// Error bits latched in DevStatus::flags.
constexpr uint32_t kErrInvalidPoint = 1u;
constexpr uint32_t kErrUnknownPolygon = 2u;
constexpr uint32_t kErrOverflowCap = 4u;
constexpr uint32_t kErrTaskCap = 8u;

// The shared-memory directory: a dense window over grid level `level`
// (= prefix_level + 4*chunks) holding, per cell, what a trie walk reaches
// after `chunks` node steps: a miss (0), a terminal entry (index into `dict`)
// or the node to continue from (kDirLink | node id).  Derived from the arena
// at index-create time; results are bitwise those of the plain walk.
struct DevDirectory {
  const uint32_t* table;  // [(height + 1) * pitch], last column and row all miss
  uint32_t width, height, pitch;  // pitch = width + 1
  uint32_t x0, y0;        // window origin in level-`level` cells
  uint32_t n_table;       // 0 = tier absent
  int32_t shift;          // 30 - level
  int32_t chunks;         // node steps already resolved
};

// How K1 codes a point's position in the 32-bit tier `tb` into one queue
// word.  Packed (the usual case): the word holds the point's cell at the level
// of the NEXT trie-node boundary (tb.level + 4; + 3..1 for a refined tier)
// relative to the window, (Y << xbits) | X, so the drain gets both the tier
// index ((Y >> tier_shift) * pitch + (X >> tier_shift)) and the 4 + 4 sub-cell bits that
// select the slot in the trie node under a link — population 3 then reads the
// arena without re-reading the point (a random 16-byte read costs a 128-byte
// DRAM burst).  An arena slot under a link needs 8 + log2(nodes) bits: up to
// 2^24 nodes that is the 32-bit second queue word; larger arenas (2^25 / 2^26
// nodes = 64 / 128 GB) borrow 1 / 2 bits from the point index in the first
// word (`index_bits`), which caps one launch at 2^30 / 2^29 points (the API
// splits longer device-resident calls).  Unpacked (window too wide for 32
// bits, arena of 2^26 nodes or more, tier deeper than level 28): the word is
// the tier index and population 3 re-reads the point.  Both forms are  min((v32 >> shift) - origin, clamp)  per
// axis, word = qy * mul + qx, where v32 is the grid coordinate left-aligned to 32 bits.
struct DevQueueCoding {
  uint32_t packed;
  uint32_t shift;           // applied to the 32-bit-aligned coordinate
  uint32_t x0, y0;          // window origin at the coded level
  uint32_t x_clamp, y_clamp;
  uint32_t mul;             // packed: 1 << xbits, unpacked: tb.pitch
  uint32_t xbits;           // packed only
  uint32_t sub_mask;        // packed only: the sub-cell bits at or above the leaf level (cell_id.cpp:93-94)
  uint32_t tier_shift;      // packed only: coded level minus the tier's level (4; 3..1 for a refined tier, DevIndex::dirk)
  uint32_t index_bits;      // bits of the first queue word that hold the point index (31, or 30 / 29 for wide arenas)
  uint32_t slow_mark;       // bit 31 and every bit between index_bits and 31: marks a slow point's first word
};

// Latitude strips of one polygon: its widened latitude range [y0, y0 + k / inv_h]
// cut into k equal strips; strip s lists (as 32-byte edge records) every edge
// whose latitude range, widened by the 1e-9 deg margin of pip_edge, meets it.
struct StripMeta {
  double y0;
  double inv_h;
  uint32_t k;         // strips (0 = no geometry for this slot)
  uint32_t ptr_base;  // first entry of this polygon in strip_ptr (k + 1 entries)
};

struct __align__(32) EdgeRecord {  // x = lng, y = lat (geometry.cpp:35); 32 bytes, one 256-bit load
  double ax, ay, bx, by;
};

// Strip of latitude y.  The same monotone fp64 expression runs on the host
// when edges are assigned to strips, so a point inside an edge's widened
// range always lands in a strip that lists the edge.
__host__ __device__ inline uint32_t strip_of(double y, double y0, double inv_h, uint32_t k) {
  const double t = (y - y0) * inv_h;
  if (!(t > 0.0)) return 0;
  const double top = static_cast<double>(k - 1);
  return t >= top ? k - 1 : static_cast<uint32_t>(t);
}

struct DevIndex {
  const uint64_t* arena;   // the reference's arena, bit-identical (act.hpp:241-246): payloads carry polygon ids
  const uint32_t* lut;     // the reference's lookup table, bit-identical: records [t, id*t, c, id*c]
  const uint32_t* ids;     // count slot -> polygon id (sorted unique); id -> slot by binary search unless ids_dense
  // closed rings per slot, x = lng, y = lat (geometry.cpp:35); len 0 = the
  // bundle has no geometry for this id (join.cpp:111-114)
  const uint64_t* ring_off;
  const uint32_t* ring_len;
  const double2* ring_xy;
  const StripMeta* strip_meta;     // [n_ids]
  const uint32_t* strip_ptr;       // per polygon k + 1 offsets into strip_edges
  const EdgeRecord* strip_edges;
  // Compact form of the strip lists for large polygon sets (null otherwise): per listed edge the index of its
  // first vertex in ring_xy (closed rings: the edge is ring_xy[v], ring_xy[v + 1]) instead of a 32-byte record.
  // The lists shrink 8x and the rings they point into are a few MB, so both stay in L2 where 140 MB of edge records
  // (10 000 polygons of BASELINE config 5) do not.
  const uint32_t* strip_eidx;
  uint64_t roots[8];
  uint64_t prefixes[8];
  uint32_t prefix_bits[8];
  uint32_t n_ids;
  int32_t k_max;
  int32_t leaf_level;      // k_max / 2
  int32_t prefix_level0;   // prefix_bits[0] / 2
  int32_t ids_dense;
  // Two directory tiers over the same trie: `dir` is staged into shared
  // memory by K1, `dir2` (deeper, optional) stays in global memory and is
  // small enough to live in L2.  `dict` holds the terminal entries that do
  // not fit a 32-bit code (two payloads, lookup-table offsets).
  DevDirectory dir;
  DevDirectory dir2;
  // Optional finer first tier with 16-bit codes, derived from `dir2` by
  // downsampling (any level between the two): 0 = miss, 0xFFFF = look in
  // dir2, otherwise 1 + ((polygon_id << 1) | interior).  K1 stages it instead
  // of `dir` when present; `table` then points at uint16 data.
  DevDirectory dir16;
  int32_t dir16_live;  // 0: (almost) every cell of dir16 says "look in the 32-bit tier" — K1's kLate form skips the lookup
  // Optional refinement of the deepest 32-bit tier for K1 (`dirk`): the same
  // codes over a window 1-3 grid levels finer than a trie-node boundary.  A
  // cell resolves here when the aligned run of slots it owns in the node under
  // its parent's link holds one terminal entry (or nothing); otherwise it
  // keeps the parent's link.  Built only when most cells of the deepest tier
  // are links (polygons a few cells across: BASELINE config 4), where every
  // cell resolved here saves a random 128-byte DRAM burst in the arena.
  // `chunks` is the parent tier's, so a link is followed exactly as from there.
  DevDirectory dirk;
  DevQueueCoding qc;  // for the 32-bit tier behind dir16 (dirk, else dir2, else dir)
  // Optional palette form of every trie node, 128 bytes (one L2 line / DRAM
  // burst) instead of 2 KB: [4 distinct entries (u64) | 256 two-bit codes (64 B) |
  // pad].  A boundary node of a tessellation holds 2-4 distinct entries (two
  // true hits, their candidate pair, empty), so the whole tree shrinks 16x and
  // stays in L2 where the arena cannot (a random arena read is a 128-byte DRAM
  // burst).  Nodes with more than 4 distinct entries keep word 0 == ~0 and are
  // read from the arena.  Null when absent.
  const uint64_t* node_pal;
  // Optional SPARSE refinement of the deepest 32-bit tier for K1 (trees too large for palette nodes: BASELINE
  // config 4 at full size, 18 M nodes = 37 GB, where every open point costs a random 128-byte DRAM burst in the
  // arena).  Only the tier's LINK cells are refined: link cell number j (1-based, in `tier_links`, a copy of the
  // tier whose link codes hold j instead of the node) owns the 64-byte record link_sub[(j - 1) * 16 ..]: one code
  // per aligned run of 16 slots (= one 128-byte line, a 4 x 4 block of cells two grid levels finer) of the linked
  // node, in slot order.  A run that holds one terminal entry (or nothing) resolves there with the tier's own code
  // forms; any other run keeps kDirLink | node and is read from the arena as before.  The records of a tier whose
  // cells are a fifth links are a few tens of MB — they stay in L2 where the same refinement as a dense grid
  // (`dirk`, 16x the tier) does not.  Null when absent; never together with `dirk`, only with the packed coding.
  const uint32_t* link_sub;
  const uint32_t* tier_links;
  const uint64_t* dict;  // [n_dict], dict[0] == 0
  uint32_t n_dict;
};

struct DevStatus {
  unsigned long long bad_index;  // min over offending point indices
  uint32_t flags;
  uint32_t pad;
  unsigned long long overflow_count;
  unsigned long long task_count;
};

// ---------------------------------------------------------------------------
// cellgrid: latlng.hpp:31-34, cell_id.cpp:50-56
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool latlng_valid(double lat, double lng) {
  // finite and inside [-90,90] x [-180,180]; NaN and inf fail the compare
  return fabs(lat) <= 90.0 && fabs(lng) <= 180.0;
}

// (value - lo) / span * 2^30 -> clamp below -> truncate -> clamp above, in
// the reference's operation order with an IEEE division.
__device__ __forceinline__ uint32_t grid_coord(double value, double lo, double span) {
  const double scaled = __dmul_rn(__ddiv_rn(__dsub_rn(value, lo), span), 1073741824.0);
  // __double2uint_rz saturates: negatives (and -0) give 0, like the clamp.
  const uint32_t cell = __double2uint_rz(scaled);
  return cell >= (1u << 30) ? (1u << 30) - 1u : cell;
}

// Grid coordinates of ANY pair of doubles, branch-free, two DFMAs: true means
// the point is valid (latlng.hpp:31-34) AND (*x32, *y32) are its exact grid
// coordinates, left-aligned to 32 bits ((x << 2) | two fraction bits, so
// x32 >> (32 - L) is the level-L cell for any L <= 30); false means "decide on
// the slow path" (invalid, NaN/inf, on or next to a grid line, on the +90/+180
// edge).
//
// t = fma(v, R, C), R = RN(2^30 / span), C = 2^31 + 2^29 (= 2^31 - lo R up to
// 2^-24).  For t in [2^31, 2^32) the 52 mantissa bits are the fixed-point value
// t - 2^31 with 21 fraction bits (unit u = 2^-21).  Against the reference's
// s = RN(RN(RN(v - lo) / span) 2^30):
//   ours:  fma rounding <= 0.5 u, R's rounding <= |v| R 2^-53 <= 0.125 u, C <= 0.125 u
//   theirs: RN(v - lo) <= 2^-45 (2^30 / span) <= 0.18 u, the division <= 2^-23 = 0.25 u
// so |t - 2^31 - s| < 1.2 u, and whenever the fraction field f satisfies
// 2 <= f <= 2^21 - 3 the integer part equals trunc(s) exactly (and is < 2^30,
// so the upper clamp cannot bind).  Validity comes from the same word: t must
// land in [2^31, 2^31 + 2^30), i.e. exponent 0x41E and top mantissa bit 0
// (hi >> 19 == 0x41E00000 >> 19):
//  * v > hi: v R + C >= 2^31 + 2^30 + 8e-8, which rounds to >= 2^31 + 2^30;
//  * v < lo: t < 2^31 (exponent differs) or t rounds to 2^31 exactly (f = 0);
//  * NaN / inf / huge: the exponent differs.
// The explicit fma is deliberate (the build is -fmad=false everywhere else).
__device__ __forceinline__ bool grid_xy_try(double lat, double lng, uint32_t* x32, uint32_t* y32) {
  const double rx = 1073741824.0 / 360.0;  // RN(2^30 / 360), folded at compile time
  const double ry = 1073741824.0 / 180.0;
  const double c = 2147483648.0 + 536870912.0;
  const double tx = __fma_rn(lng, rx, c);
  const double ty = __fma_rn(lat, ry, c);
  const uint32_t xl = static_cast<uint32_t>(__double2loint(tx)), xh = static_cast<uint32_t>(__double2hiint(tx));
  const uint32_t yl = static_cast<uint32_t>(__double2loint(ty)), yh = static_cast<uint32_t>(__double2hiint(ty));
  *x32 = __funnelshift_l(xl, xh, 13);  // exponent and the (zero) top mantissa bit fall off
  *y32 = __funnelshift_l(yl, yh, 13);
  const uint32_t fx = ((xl & 0x1FFFFFu) - 2u), fy = ((yl & 0x1FFFFFu) - 2u);
  const uint32_t range = (xh ^ 0x41E00000u) | (yh ^ 0x41E00000u);
  return (range < (1u << 19)) & (max(fx, fy) <= 0x1FFFFFu - 4u);
}

// Both grid coordinates (30 bits each) of a valid point, bit-exact: the fast
// path above, else the reference's own arithmetic.
__device__ __forceinline__ void grid_xy(double lat, double lng, uint32_t* x, uint32_t* y) {
  uint32_t x32, y32;
  if (grid_xy_try(lat, lng, &x32, &y32)) {
    *x = x32 >> 2;
    *y = y32 >> 2;
  } else {  // within 2^-20 of a cell boundary (or on the +90 / +180 edge): do the division
    *x = grid_coord(lng, -180.0, 360.0);
    *y = grid_coord(lat, -90.0, 180.0);
  }
}

// spread_bits (cell_id.cpp:30-37): bit i of the low 30 bits moves to bit 2i.
__device__ __forceinline__ uint64_t spread_bits(uint64_t v) {
  v = (v | (v << 16)) & 0x0000ffff0000ffffull;
  v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
  v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}

// cell_from_point (cell_id.cpp:82-95) for a valid point and level in [0, 30].
__device__ __forceinline__ uint64_t cell_from_point(double lat, double lng, int level) {
  uint32_t x, y;
  grid_xy(lat, lng, &x, &y);
  const uint64_t pos60 = (spread_bits(y) << 1) | spread_bits(x);
  const uint64_t leaf = (pos60 << 1) | 1ull;
  const uint64_t marker = 1ull << (60 - 2 * level);
  return (leaf & ~(marker - 1) & ~marker) | marker;
}

// spread the low 4 bits of v to bit positions 0,2,4,6 (cell_id.cpp:30-37
// restricted to one trie chunk)
__device__ __forceinline__ uint32_t spread4(uint32_t v) {
  v = (v | (v << 2)) & 0x33u;
  return (v | (v << 1)) & 0x55u;
}

// Slot of trie chunk `chunk` (8 key bits = 4 grid levels below
// prefix_level + 4*chunk): y bit above x bit in every pair
// (cell_id.hpp:30-33).  xl/yl are the 30-bit grid coordinates, already
// truncated to the leaf level, shifted left by 2.
__device__ __forceinline__ uint32_t chunk_slot(uint32_t xl, uint32_t yl, int level_above) {
  const int sh = 28 - level_above;
  return (spread4((yl >> sh) & 0xFu) << 1) | spread4((xl >> sh) & 0xFu);
}

__device__ __forceinline__ uint64_t ld_arena(const uint64_t* p) { return __ldg(p); }

// Trie descent from `node`, whose slots resolve the 4 grid levels below
// `level_above` (act.cpp:258-268).  The index was validated at create time
// (forest, depth bound), so the loop needs no bound of its own.
__device__ __forceinline__ uint64_t walk_from(const uint64_t* __restrict__ arena, uint64_t node, int level_above,
                                              uint32_t xl, uint32_t yl) {
  for (;;) {
    const uint32_t slot = chunk_slot(xl, yl, level_above);
    const uint64_t e = ld_arena(arena + (node - 1) * kNodeSlots + slot);
    if ((e & 3u) != 0u || e == 0u) return e;
    node = e >> 2;
    level_above += 4;
  }
}

// Directory lookup: the code of the level-`d` cell holding grid point (x, y).
__device__ __forceinline__ uint32_t dir_code(const DevDirectory& d, const uint32_t* table, uint32_t x,
                                             uint32_t y) {
  // cells left of / below the window wrap to huge values: both sides clamp
  // into the all-miss padding
  const uint32_t cx = min((x >> d.shift) - d.x0, d.width);
  const uint32_t cy = min((y >> d.shift) - d.y0, d.height);
  return table[cy * d.pitch + cx];
}

// One point -> tagged entry, bitwise Act::probe(cell_from_point(p, k_max/2))
// for face 0 (cell_from_point never sets face bits, cell_id.cpp:89-94).
__device__ __forceinline__ uint64_t probe_point(const DevIndex& ix, const uint32_t* dir_table, double lat,
                                                double lng) {
  uint32_t x, y;
  grid_xy(lat, lng, &x, &y);
  uint32_t code = dir_code(ix.dir, dir_table, x, y);
  int chunks = ix.dir.chunks;
  if ((code & kDirLink) && ix.dir2.n_table) {
    code = dir_code(ix.dir2, ix.dir2.table, x, y);
    chunks = ix.dir2.chunks;
  }
  if (code == 0) return 0;
  if ((code >> 30) == 1u) return (static_cast<uint64_t>(code & 0x3FFFFFFFu) << 2) | 1u;  // make_one
  if ((code & kDirLink) == 0) return __ldg(ix.dict + code);
  // truncate to the leaf level (cell_id.cpp:93-94), left-align to 32 bits
  const uint32_t keep = ~((1u << (30 - ix.leaf_level)) - 1u);
  return walk_from(ix.arena, code & ~kDirLink, ix.prefix_level0 + 4 * chunks, (x & keep) << 2, (y & keep) << 2);
}

// Generic probe of a raw cell id on any face without the directory: the
// scalar walk of act.cpp:248-270 (used by gj_probe_cells_host, the
// ProbeBatchFn-shaped test hook).
__device__ __forceinline__ uint64_t probe_from_root(const uint64_t* __restrict__ arena, uint64_t raw, uint64_t node,
                                                    uint32_t plen, uint64_t prefix) {
  if (node == 0) return 0;
  const uint64_t key = (raw ^ (raw & (~raw + 1))) << 3;  // key_of, act.hpp:142-145
  if (plen != 0 && (key >> (64 - plen)) != prefix) return 0;
  int shift = 56 - static_cast<int>(plen);
  for (;;) {
    // past the last key bit the reference's lockstep kernels would read
    // zeros; a validated index never gets there
    const uint32_t slot = shift >= 0 ? static_cast<uint32_t>(key >> shift) & 0xffu : 0u;
    const uint64_t e = ld_arena(arena + (node - 1) * kNodeSlots + slot);
    if ((e & 3u) != 0u || e == 0u) return e;
    node = e >> 2;
    shift -= 8;
  }
}

__device__ __forceinline__ uint64_t probe_raw(const DevIndex& ix, uint64_t raw) {
  const uint32_t face = static_cast<uint32_t>(raw >> 61);  // faces 6,7 hold a zero root
  return probe_from_root(ix.arena, raw, ix.roots[face], ix.prefix_bits[face], ix.prefixes[face]);
}

// The same for a cell id made by cell_from_point, which never sets face bits (cell_id.cpp:89-94).  K1's slow path
// uses this form: indexing the face tables of the kernel parameter block with a run-time face made ptxas keep a
// thread-local copy of the whole block in some instantiations.
// (Tried and dropped: K1's two rare paths — this one and the deep walk, four IEEE divisions between them — as
// __noinline__ functions to shrink population 3's code by another 450 instructions: the calls cost more in the
// register allocation around them than the footprint gained, config-5 stand-in 2.26 -> 2.48 ms per 20 M points.)
__device__ __forceinline__ uint64_t probe_raw_face0(const DevIndex& ix, uint64_t raw) {
  return probe_from_root(ix.arena, raw, ix.roots[0], ix.prefix_bits[0], ix.prefixes[0]);
}

// ---------------------------------------------------------------------------
// PIP refine: geometry.cpp:28-29,63-75,184-204
// ---------------------------------------------------------------------------
__device__ __forceinline__ double point_segment_dist_sq(double px, double py, double ax, double ay,
                                                        double bx, double by) {
  const double dx = __dsub_rn(bx, ax);
  const double dy = __dsub_rn(by, ay);
  const double len2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  double t = 0.0;
  if (len2 > 0.0) {
    t = __ddiv_rn(__dadd_rn(__dmul_rn(__dsub_rn(px, ax), dx), __dmul_rn(__dsub_rn(py, ay), dy)),
                  len2);
    t = (t < 0.0) ? 0.0 : (1.0 < t) ? 1.0 : t;  // std::clamp
  }
  const double cx = __dsub_rn(__dadd_rn(ax, __dmul_rn(t, dx)), px);
  const double cy = __dsub_rn(__dadd_rn(ay, __dmul_rn(t, dy)), py);
  return __dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy));
}

// One edge's contribution to pip_test, split so that the cheap part can run
// per lane and the parts with a division can be batched.  The boundary any()
// and the crossing parity are order-independent, so edges may be evaluated in
// any order or in parallel; each edge's arithmetic is the reference's.
//
// Cheap classification: bit 0 = the boundary test has to be evaluated, bit 1 =
// the edge straddles the point's latitude and the crossing test has to be.
//
// Bit 0 is an exact rejection of the boundary test: a point farther than 1e-9
// degrees from the edge's bounding box is at distance >= 1e-9 from the
// segment, and rounding errors of the distance arithmetic (coordinates <= 360,
// ulp <= 5.7e-14) cannot bring cx^2+cy^2 from >= 1e-18 down to 1e-24, so the
// reference's comparison is false as well.
constexpr double kPipBoxMargin = 1e-9;

// Sorts a (point, edge) pair without a division.  The box is the edge's
// bounding box widened by the margin: [min(ax,bx) - m, max(ax,bx) + m] x
// [min(ay,by) - m, max(ay,by) + m]; rounding is monotone, so RN(min(a,b) - m) =
// min(RN(a - m), RN(b - m)) and the test needs no min/max, only the four widened
// coordinates per axis.  Result bits:
//   1  inside the box: the distance to the edge must be computed (geometry.cpp:186-193)
//   2  the edge straddles the point's latitude (geometry.cpp:197) and the point
//      is inside the box's x range: the crossing abscissa must be computed
//   4  it straddles and the point is LEFT of the x range: the ray crosses, no
//      arithmetic needed.  x_cross = ax + t (bx - ax) with t = RN(RN(qy - ay) /
//      RN(by - ay)) in [0, 1 + 2^-52], so x_cross lies within 360 * 2^-51 <
//      2e-13 of [min(ax,bx), max(ax,bx)] — far inside the 1e-9 margin — and
//      qx < min - m implies qx < x_cross (to the right of max + m: no crossing).
__device__ __forceinline__ uint32_t pip_edge_classify(double qx, double qy, double ax, double ay, double bx,
                                                      double by) {
  const double m = kPipBoxMargin;
  const bool ge_lo = qx >= __dsub_rn(ax, m) || qx >= __dsub_rn(bx, m);
  const bool le_hi = qx <= __dadd_rn(ax, m) || qx <= __dadd_rn(bx, m);
  const bool near_x = ge_lo && le_hi;
  const bool near_y = (qy >= __dsub_rn(ay, m) || qy >= __dsub_rn(by, m)) &&
                      (qy <= __dadd_rn(ay, m) || qy <= __dadd_rn(by, m));
  const bool straddles = (ay > qy) != (by > qy);  // geometry.cpp:197
  return (near_x && near_y ? 1u : 0u) | (straddles && near_x ? 2u : 0u) | (straddles && !ge_lo ? 4u : 0u);
}

// One edge record with a single 256-bit load (sm_100+).
__device__ __forceinline__ void load_edge(const EdgeRecord* rec, double* ax, double* ay, double* bx, double* by) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(*ax), "=d"(*ay), "=d"(*bx), "=d"(*by) : "l"(rec));
}

// The same edge through the compact strip lists: two 16-byte vertex loads (vertex pairs are not 32-byte aligned).
__device__ __forceinline__ void load_edge_indexed(const double2* ring_xy, const uint32_t* eidx, uint32_t e, double* ax,
                                                  double* ay, double* bx, double* by) {
  const double2* v = ring_xy + __ldg(eidx + e);
  const double2 a = __ldg(v), b = __ldg(v + 1);
  *ax = a.x;
  *ay = a.y;
  *bx = b.x;
  *by = b.y;
}

// geometry.cpp:186-193: on an edge or vertex
__device__ __forceinline__ bool pip_edge_on_boundary(double qx, double qy, double ax, double ay, double bx,
                                                     double by) {
  const double eps_sq = __dmul_rn(1e-12, 1e-12);  // the product, not 1e-24
  return point_segment_dist_sq(qx, qy, ax, ay, bx, by) <= eps_sq;
}

// geometry.cpp:198-199, for an edge that straddles the point's latitude
__device__ __forceinline__ bool pip_edge_crosses(double qx, double qy, double ax, double ay, double bx,
                                                 double by) {
  const double x_cross =
      __dadd_rn(ax, __dmul_rn(__ddiv_rn(__dsub_rn(qy, ay), __dsub_rn(by, ay)), __dsub_rn(bx, ax)));
  return qx < x_cross;
}

}  // namespace gj
