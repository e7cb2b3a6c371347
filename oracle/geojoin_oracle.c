/* TEST INFRASTRUCTURE — see geojoin_oracle.h.  Plain-C restatement of the
 * reference's probe-side algorithm; each function names the reference lines
 * it follows (relative to /root/reference/proj). */
#include "geojoin_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define GRID_CELLS_PER_AXIS ((uint64_t)1 << 30) /* cell_id.cpp:27 */
#define NODE_SLOTS 256                          /* act.hpp:36 */
#define BATCH 8                                 /* act.hpp:38 */

/* latlng.hpp:31-34 */
int gjo_latlng_valid(double lat, double lng) {
  return isfinite(lat) && isfinite(lng) && lat >= -90.0 && lat <= 90.0 &&
         lng >= -180.0 && lng <= 180.0;
}

/* cell_id.cpp:50-56 — the operation order (sub, IEEE div, mul by 2^30),
 * the <0 clamp, the truncating cast and the upper clamp are the contract. */
uint32_t gjo_grid_coord(double value, double lo, double span) {
  double scaled = (value - lo) / span * (double)GRID_CELLS_PER_AXIS;
  if (scaled < 0.0) scaled = 0.0;
  uint64_t cell = (uint64_t)scaled;
  if (cell >= GRID_CELLS_PER_AXIS) cell = GRID_CELLS_PER_AXIS - 1;
  return (uint32_t)cell;
}

/* cell_id.cpp:30-37 — bit i of the low 30 bits moves to bit 2i. */
uint64_t gjo_spread_bits(uint64_t v) {
  static const uint64_t mask[5] = {0x0000ffff0000ffffULL, 0x00ff00ff00ff00ffULL,
                                   0x0f0f0f0f0f0f0f0fULL, 0x3333333333333333ULL,
                                   0x5555555555555555ULL};
  int shift = 16;
  for (int step = 0; step < 5; ++step, shift >>= 1) {
    v = (v | (v << shift)) & mask[step];
  }
  return v;
}

/* cell_id.cpp:82-95 */
int gjo_cell_from_point(double lat, double lng, int level, uint64_t* raw) {
  if (!gjo_latlng_valid(lat, lng)) return GJO_INVALID_POINT;
  if (level < 0 || level > 30) return GJO_INVALID_LEVEL;
  const uint64_t col = gjo_grid_coord(lng, -180.0, 360.0);
  const uint64_t row = gjo_grid_coord(lat, -90.0, 180.0);
  const uint64_t pos60 = (gjo_spread_bits(row) << 1) | gjo_spread_bits(col);
  const uint64_t leaf = (pos60 << 1) | 1u;
  const uint64_t marker = (uint64_t)1 << (60 - 2 * level);
  *raw = (leaf & ~(marker - 1) & ~marker) | marker;
  return GJO_OK;
}

int gjo_cells_from_points(const double* latlng, uint64_t n, int level,
                          uint64_t* out_raw, uint64_t* bad_index) {
  for (uint64_t i = 0; i < n; ++i) {
    const int rc =
        gjo_cell_from_point(latlng[2 * i], latlng[2 * i + 1], level, &out_raw[i]);
    if (rc != GJO_OK) {
      if (bad_index) *bad_index = i;
      return rc;
    }
  }
  return GJO_OK;
}

/* act.hpp:142-145 — strip the level marker, shift the 3 face bits out. */
uint64_t gjo_key_of(uint64_t raw) {
  const uint64_t marker = raw & (~raw + 1);
  return (raw ^ marker) << 3;
}

/* act.cpp:248-270 — the scalar walk (the semantic definition). */
int gjo_probe(const gjo_index* ix, uint64_t raw, uint64_t* entry,
              int* node_accesses) {
  *entry = 0;
  const unsigned face = (unsigned)(raw >> 61);
  if (node_accesses) ++*node_accesses; /* the face node */
  if (face >= 6) return GJO_OK;
  const uint64_t root = ix->roots[face];
  if (root == 0) return GJO_OK;
  const uint64_t key = gjo_key_of(raw);
  const int plen = (int)ix->prefix_bits[face];
  if (plen != 0 && (key >> (64 - plen)) != ix->prefixes[face]) return GJO_OK;
  const int max_chunks = (ix->k_max - plen + 7) / 8;
  uint64_t node = root;
  for (int chunk = 0; chunk < max_chunks; ++chunk) {
    if (node_accesses) ++*node_accesses;
    const uint64_t slot = (key >> (56 - plen - 8 * chunk)) & 0xff;
    const uint64_t e = ix->arena[(node - 1) * NODE_SLOTS + slot];
    if ((e & 3) != 0) { /* payload(s) or lookup-table offset */
      *entry = e;
      return GJO_OK;
    }
    if (e == 0) return GJO_OK; /* sentinel link: false hit */
    node = e >> 2;
  }
  return GJO_CORRUPT_INDEX; /* path longer than the key */
}

/* act_probe_scalar.cpp:27-82 — eight lanes in lockstep with the
 * traverse/output/done masks; no depth bound (terminates on payload or
 * sentinel only); lanes that never output stay at the sentinel. */
void gjo_probe_batch8(const gjo_index* ix, const uint64_t* raw_ids,
                      uint64_t* out) {
  uint64_t key[BATCH], node[BATCH], value[BATCH];
  int shift[BATCH];
  unsigned active = 0;
  for (int lane = 0; lane < BATCH; ++lane) {
    const unsigned face = (unsigned)(raw_ids[lane] >> 61);
    key[lane] = gjo_key_of(raw_ids[lane]);
    node[lane] = ix->roots[face];
    const uint64_t plen = ix->prefix_bits[face];
    shift[lane] = 56 - (int)plen;
    const uint64_t top = plen ? key[lane] >> (64 - plen) : 0;
    if (node[lane] != 0 && top == ix->prefixes[face]) active |= 1u << lane;
    value[lane] = 0;
  }
  unsigned traverse = active, output = 0, done = ~active & 0xffu;
  while (traverse) {
    unsigned is_link = 0, is_sentinel = 0;
    for (int lane = 0; lane < BATCH; ++lane) {
      if (!((traverse >> lane) & 1)) continue;
      const uint64_t slot = (key[lane] >> shift[lane]) & 0xff;
      value[lane] = ix->arena[(node[lane] - 1) * NODE_SLOTS + slot];
      if ((value[lane] & 3) == 0) {
        is_link |= 1u << lane;
        if (value[lane] == 0) is_sentinel |= 1u << lane;
        node[lane] = value[lane] >> 2;
      }
    }
    output |= traverse & ~is_link;
    done |= output | is_sentinel;
    traverse &= ~done;
    for (int lane = 0; lane < BATCH; ++lane) shift[lane] -= 8;
  }
  for (int lane = 0; lane < BATCH; ++lane) {
    out[lane] = ((output >> lane) & 1) ? value[lane] : 0;
  }
}

int gjo_probe_points(const gjo_index* ix, const double* latlng, uint64_t n,
                     uint64_t* out_entries, uint64_t* bad_index) {
  const int level = ix->k_max / 2; /* act.hpp:148 */
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t raw;
    int rc = gjo_cell_from_point(latlng[2 * i], latlng[2 * i + 1], level, &raw);
    if (rc == GJO_OK) rc = gjo_probe(ix, raw, &out_entries[i], NULL);
    if (rc != GJO_OK) {
      if (bad_index) *bad_index = i;
      return rc;
    }
  }
  return GJO_OK;
}

/* act.cpp:141-153 */
static int record_in_bounds(const gjo_index* ix, uint64_t off) {
  if (off >= ix->lut_len) return 0;
  const uint64_t t = ix->lut[off];
  if (off + 1 + t >= ix->lut_len) return 0;
  const uint64_t c = ix->lut[off + 1 + t];
  return off + 2 + t + c <= ix->lut_len;
}

/* act.hpp:55-83 (tags), act.hpp:169-196 (for_each_reference): true hits
 * first, in stored order; payload = (polygon_id << 1) | interior. */
int gjo_decode(const gjo_index* ix, uint64_t entry, uint32_t* ids,
               uint8_t* interior, uint64_t cap, uint64_t* n_refs) {
  uint64_t n = 0;
#define PUSH(id_, in_)               \
  do {                               \
    if (n < cap) {                   \
      ids[n] = (id_);                \
      interior[n] = (uint8_t)(in_);  \
    }                                \
    ++n;                             \
  } while (0)
  switch (entry & 3) {
    case 0: /* link; only the sentinel can be returned by a probe */
      break;
    case 1: {
      const uint32_t p = (uint32_t)((entry >> 2) & 0x7fffffffu);
      PUSH(p >> 1, p & 1);
      break;
    }
    case 2: {
      const uint32_t a = (uint32_t)((entry >> 33) & 0x7fffffffu);
      const uint32_t b = (uint32_t)((entry >> 2) & 0x7fffffffu);
      PUSH(a >> 1, a & 1);
      PUSH(b >> 1, b & 1);
      break;
    }
    default: {
      const uint64_t off = (entry >> 2) & 0x7fffffffu;
      if (!record_in_bounds(ix, off)) return GJO_CORRUPT_INDEX;
      const uint32_t t = ix->lut[off];
      const uint32_t c = ix->lut[off + 1 + t];
      for (uint32_t i = 0; i < t; ++i) PUSH(ix->lut[off + 1 + i], 1);
      for (uint32_t i = 0; i < c; ++i) PUSH(ix->lut[off + 2 + t + i], 0);
      break;
    }
  }
#undef PUSH
  *n_refs = n;
  return n > cap ? GJO_CAPACITY : GJO_OK;
}

/* The probe half of Act::train (act.cpp:414-440): per point, probe at the
 * maximum indexed level and ask whether any reference of the entry is a
 * candidate (for_each_reference with !interior).  flags[i] = 0 / 1;
 * *n_flagged counts the ones (expensive_fraction = n_flagged / n). */
int gjo_training_candidates(const gjo_index* ix, const double* latlng,
                            uint64_t n, uint8_t* flags, uint64_t* n_flagged,
                            uint64_t* bad_index) {
  const int level = ix->k_max / 2; /* max_indexed_level, act.hpp:148 */
  uint64_t count = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t raw, e = 0;
    int rc = gjo_cell_from_point(latlng[2 * i], latlng[2 * i + 1], level, &raw);
    if (rc == GJO_OK) rc = gjo_probe(ix, raw, &e, NULL);
    if (rc != GJO_OK) {
      if (bad_index) *bad_index = i;
      return rc;
    }
    int any_candidate = 0;
    switch (e & 3) {
      case 0:
        break;
      case 1:
        any_candidate = ((e >> 2) & 1) == 0;
        break;
      case 2:
        any_candidate = ((e >> 33) & 1) == 0 || ((e >> 2) & 1) == 0;
        break;
      default: {
        const uint64_t off = (e >> 2) & 0x7fffffffu;
        if (!record_in_bounds(ix, off)) {
          if (bad_index) *bad_index = i;
          return GJO_CORRUPT_INDEX;
        }
        any_candidate = ix->lut[off + 1 + ix->lut[off]] != 0;
        break;
      }
    }
    if (flags) flags[i] = (uint8_t)any_candidate;
    count += (uint64_t)any_candidate;
  }
  if (n_flagged) *n_flagged = count;
  return GJO_OK;
}

/* geometry.cpp:63-75; x = lng, y = lat (geometry.cpp:35). */
double gjo_point_segment_dist_sq(double px, double py, double ax, double ay,
                                 double bx, double by) {
  const double dx = bx - ax;
  const double dy = by - ay;
  const double len2 = dx * dx + dy * dy;
  double t = 0.0;
  if (len2 > 0.0) {
    t = ((px - ax) * dx + (py - ay) * dy) / len2;
    /* std::clamp(t, 0.0, 1.0): (t < lo) ? lo : (hi < t) ? hi : t */
    t = (t < 0.0) ? 0.0 : (1.0 < t) ? 1.0 : t;
  }
  const double cx = ax + t * dx - px;
  const double cy = ay + t * dy - py;
  return cx * cx + cy * cy;
}

/* geometry.cpp:28-29,184-204 — boundary pass over all edges first (a hit
 * returns true: ST_Covers), then the crossing-number pass. */
int gjo_pip_test(const double* ring, uint64_t n, double lat, double lng) {
  const double eps = 1e-12;
  const double eps_sq = eps * eps; /* the product, not the literal 1e-24 */
  const double qx = lng, qy = lat;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t j = (i + 1) % n;
    if (gjo_point_segment_dist_sq(qx, qy, ring[2 * i + 1], ring[2 * i],
                                  ring[2 * j + 1], ring[2 * j]) <= eps_sq) {
      return 1;
    }
  }
  int inside = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t j = (i + 1) % n;
    const double ax = ring[2 * i + 1], ay = ring[2 * i];
    const double bx = ring[2 * j + 1], by = ring[2 * j];
    if ((ay > qy) != (by > qy)) {
      const double x_cross = ax + (qy - ay) / (by - ay) * (bx - ax);
      if (qx < x_cross) inside = !inside;
    }
  }
  return inside;
}

void gjo_pip_tests(const double* ring, uint64_t n_vtx, const double* latlng,
                   uint64_t n, uint8_t* out) {
  for (uint64_t i = 0; i < n; ++i) {
    out[i] = (uint8_t)gjo_pip_test(ring, n_vtx, latlng[2 * i], latlng[2 * i + 1]);
  }
}

/* ---- join ---- */

typedef struct {
  const gjo_index* ix;
  /* polygon id -> bundle position (IndexBundle::polygon_by_id, join.hpp:92-95) */
  uint32_t* sorted_ids;
  uint64_t* sorted_pos;
  uint64_t* out_point_index;
  uint32_t* out_polygon_id;
  uint64_t cap;
  uint64_t n_pairs;
  uint64_t* counts_by_slot;
  gjo_stats* stats;
} join_ctx;

static int64_t find_u32(const uint32_t* sorted, uint64_t n, uint32_t key) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (sorted[mid] < key) {
      lo = mid + 1;
    } else {
      hi = mid;
    }
  }
  return (lo < n && sorted[lo] == key) ? (int64_t)lo : -1;
}

static void emit_pair(join_ctx* c, uint64_t point_index, uint32_t polygon_id) {
  if (c->out_polygon_id && c->n_pairs < c->cap) {
    c->out_point_index[c->n_pairs] = point_index;
    c->out_polygon_id[c->n_pairs] = polygon_id;
  }
  ++c->n_pairs;
  if (c->counts_by_slot) {
    const int64_t slot = find_u32(c->ix->count_ids, c->ix->n_count_ids, polygon_id);
    if (slot >= 0) ++c->counts_by_slot[slot];
  }
}

/* One reference of one probed entry: join.cpp:100-119. */
static int handle_ref(join_ctx* c, uint64_t point_index, double lat, double lng,
                      uint32_t polygon_id, int interior, int approx,
                      uint64_t* candidates) {
  if (interior) { /* true hit, no refinement */
    emit_pair(c, point_index, polygon_id);
    return GJO_OK;
  }
  ++*candidates;
  if (approx) {
    emit_pair(c, point_index, polygon_id);
    return GJO_OK;
  }
  const gjo_index* ix = c->ix;
  const int64_t s = find_u32(c->sorted_ids, ix->n_polygons, polygon_id);
  if (s < 0) return GJO_UNKNOWN_POLYGON;
  const uint64_t pos = c->sorted_pos[s];
  if (c->stats) ++c->stats->pip_tests;
  const uint64_t b = ix->vtx_off[pos], e = ix->vtx_off[pos + 1];
  if (gjo_pip_test(ix->vtx_latlng + 2 * b, e - b, lat, lng)) {
    emit_pair(c, point_index, polygon_id);
  }
  return GJO_OK;
}

/* The per-(point, entry) lambda of run_join, join.cpp:93-127. */
static int process_entry(join_ctx* c, uint64_t point_index, double lat,
                         double lng, uint64_t entry, int approx) {
  const gjo_index* ix = c->ix;
  if (c->stats) ++c->stats->probes;
  if (entry == 0) {
    if (c->stats) ++c->stats->false_hits;
    return GJO_OK;
  }
  uint64_t candidates = 0;
  int rc = GJO_OK;
  switch (entry & 3) {
    case 1: {
      const uint32_t p = (uint32_t)((entry >> 2) & 0x7fffffffu);
      rc = handle_ref(c, point_index, lat, lng, p >> 1, p & 1, approx, &candidates);
      break;
    }
    case 2: {
      const uint32_t a = (uint32_t)((entry >> 33) & 0x7fffffffu);
      const uint32_t b = (uint32_t)((entry >> 2) & 0x7fffffffu);
      rc = handle_ref(c, point_index, lat, lng, a >> 1, a & 1, approx, &candidates);
      if (rc == GJO_OK) {
        rc = handle_ref(c, point_index, lat, lng, b >> 1, b & 1, approx, &candidates);
      }
      break;
    }
    case 3: {
      const uint64_t off = (entry >> 2) & 0x7fffffffu;
      if (!record_in_bounds(ix, off)) return GJO_CORRUPT_INDEX;
      const uint32_t t = ix->lut[off];
      const uint32_t cn = ix->lut[off + 1 + t];
      for (uint32_t i = 0; i < t && rc == GJO_OK; ++i) {
        rc = handle_ref(c, point_index, lat, lng, ix->lut[off + 1 + i], 1, approx,
                        &candidates);
      }
      for (uint32_t i = 0; i < cn && rc == GJO_OK; ++i) {
        rc = handle_ref(c, point_index, lat, lng, ix->lut[off + 2 + t + i], 0,
                        approx, &candidates);
      }
      break;
    }
    default:
      break; /* a non-zero link is never returned by a probe */
  }
  if (rc != GJO_OK) return rc;
  if (c->stats) {
    if (candidates == 0) {
      ++c->stats->solely_true_hits;
    } else {
      ++c->stats->refinement_entered;
      c->stats->candidate_refs += candidates;
    }
  }
  return GJO_OK;
}

static int cmp_id_pos(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

static int build_polygon_lookup(join_ctx* c) {
  const gjo_index* ix = c->ix;
  const uint64_t n = ix->n_polygons;
  uint64_t* packed = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  c->sorted_ids = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  c->sorted_pos = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  if (!packed || !c->sorted_ids || !c->sorted_pos) {
    free(packed);
    return -1;
  }
  for (uint64_t i = 0; i < n; ++i) packed[i] = ((uint64_t)ix->polygon_ids[i] << 32) | i;
  qsort(packed, n, sizeof(uint64_t), cmp_id_pos);
  for (uint64_t i = 0; i < n; ++i) {
    c->sorted_ids[i] = (uint32_t)(packed[i] >> 32);
    c->sorted_pos[i] = packed[i] & 0xffffffffu;
  }
  free(packed);
  return 0;
}

/* probe_points + run_join, join.cpp:68-129: batches of 8 through the
 * lockstep kernel, then a scalar tail. */
int gjo_join(const gjo_index* ix, const double* latlng, uint64_t n,
             uint64_t base_index, int approx, uint64_t* out_point_index,
             uint32_t* out_polygon_id, uint64_t cap, uint64_t* n_pairs,
             gjo_stats* stats, uint64_t* counts_by_slot, uint64_t* bad_index) {
  join_ctx c;
  memset(&c, 0, sizeof c);
  c.ix = ix;
  c.out_point_index = out_point_index;
  c.out_polygon_id = out_polygon_id;
  c.cap = cap;
  c.counts_by_slot = counts_by_slot;
  c.stats = stats;
  if (build_polygon_lookup(&c) != 0) return GJO_CAPACITY;

  const int level = ix->k_max / 2;
  int rc = GJO_OK;
  uint64_t i = 0;
  for (; rc == GJO_OK && i + BATCH <= n; i += BATCH) {
    uint64_t raw[BATCH], entry[BATCH];
    for (int k = 0; k < BATCH && rc == GJO_OK; ++k) {
      rc = gjo_cell_from_point(latlng[2 * (i + k)], latlng[2 * (i + k) + 1], level,
                               &raw[k]);
      if (rc != GJO_OK && bad_index) *bad_index = i + k;
    }
    if (rc != GJO_OK) break;
    gjo_probe_batch8(ix, raw, entry);
    for (int k = 0; k < BATCH && rc == GJO_OK; ++k) {
      rc = process_entry(&c, base_index + i + k, latlng[2 * (i + k)],
                         latlng[2 * (i + k) + 1], entry[k], approx);
      if (rc != GJO_OK && bad_index) *bad_index = i + k;
    }
  }
  for (; rc == GJO_OK && i < n; ++i) {
    uint64_t raw, entry;
    rc = gjo_cell_from_point(latlng[2 * i], latlng[2 * i + 1], level, &raw);
    if (rc == GJO_OK) rc = gjo_probe(ix, raw, &entry, NULL);
    if (rc == GJO_OK) {
      rc = process_entry(&c, base_index + i, latlng[2 * i], latlng[2 * i + 1], entry,
                         approx);
    }
    if (rc != GJO_OK) {
      if (bad_index) *bad_index = i;
      break;
    }
  }
  free(c.sorted_ids);
  free(c.sorted_pos);
  if (n_pairs) *n_pairs = c.n_pairs;
  return rc;
}

typedef struct {
  const gjo_index* ix;
  const double* latlng;
  uint64_t begin, end;
  int approx;
  uint64_t* counts;
  uint64_t pairs;
  uint64_t bad_index;
  int rc;
} count_job;

static void* count_worker(void* arg) {
  count_job* j = (count_job*)arg;
  j->rc = gjo_join(j->ix, j->latlng + 2 * j->begin, j->end - j->begin, j->begin,
                   j->approx, NULL, NULL, 0, &j->pairs, NULL, j->counts,
                   &j->bad_index);
  if (j->rc != GJO_OK) j->bad_index += j->begin;
  return NULL;
}

/* join.cpp:255-285 */
int gjo_join_count_threads(const gjo_index* ix, const double* latlng,
                           uint64_t n, int approx, int threads,
                           uint64_t* counts_by_slot, uint64_t* total_pairs,
                           uint64_t* bad_index) {
  if (threads < 1) threads = 1;
  uint64_t workers = (uint64_t)threads;
  const uint64_t at_least_one = n > 0 ? n : 1;
  if (workers > at_least_one) workers = at_least_one;
  const uint64_t slots = ix->n_count_ids ? ix->n_count_ids : 1;
  count_job* jobs = (count_job*)calloc(workers, sizeof(count_job));
  pthread_t* tids = (pthread_t*)calloc(workers, sizeof(pthread_t));
  uint64_t* partial = (uint64_t*)calloc(workers * slots, sizeof(uint64_t));
  if (!jobs || !tids || !partial) {
    free(jobs);
    free(tids);
    free(partial);
    return GJO_CAPACITY;
  }
  for (uint64_t w = 0; w < workers; ++w) {
    jobs[w].ix = ix;
    jobs[w].latlng = latlng;
    jobs[w].begin = (uint64_t)((unsigned __int128)n * w / workers);
    jobs[w].end = (uint64_t)((unsigned __int128)n * (w + 1) / workers);
    jobs[w].approx = approx;
    jobs[w].counts = partial + w * slots;
  }
  if (workers == 1) {
    count_worker(&jobs[0]);
  } else {
    for (uint64_t w = 0; w < workers; ++w) {
      pthread_create(&tids[w], NULL, count_worker, &jobs[w]);
    }
    for (uint64_t w = 0; w < workers; ++w) pthread_join(tids[w], NULL);
  }
  int rc = GJO_OK;
  uint64_t pairs = 0;
  for (uint64_t w = 0; w < workers; ++w) {
    if (jobs[w].rc != GJO_OK && rc == GJO_OK) {
      rc = jobs[w].rc;
      if (bad_index) *bad_index = jobs[w].bad_index;
    }
    pairs += jobs[w].pairs;
    for (uint64_t s = 0; s < ix->n_count_ids; ++s) {
      counts_by_slot[s] += partial[w * slots + s];
    }
  }
  if (total_pairs) *total_pairs = pairs;
  free(jobs);
  free(tids);
  free(partial);
  return rc;
}

/* ---- CSV point ingestion (csv.cpp) ------------------------------------- */

/* parse_double, csv.cpp:39-45: leading spaces/tabs skipped, then the whole
 * rest of the field must be one std::from_chars(general) number.  Restated:
 * [-] digits [. digits] with at least one digit, optionally [eE][+-]digits —
 * a malformed exponent is left unconsumed, so the field is rejected.  (The
 * words inf / nan also parse there, but never to a valid coordinate, so they
 * are rejected here with everything else that is not a decimal.)  The value is
 * the correctly rounded double (strtod, like fast_float inside from_chars);
 * overflow and a nonzero decimal that rounds to zero are range errors,
 * subnormal results are not. */
static int csv_parse_double(const char* b, const char* e, double* out) {
  while (b != e && (*b == ' ' || *b == '\t')) ++b;
  const char* p = b;
  if (p != e && *p == '-') ++p;
  int digits = 0, nonzero = 0;
  while (p != e && *p >= '0' && *p <= '9') {
    nonzero |= *p != '0';
    ++digits;
    ++p;
  }
  if (p != e && *p == '.') {
    ++p;
    while (p != e && *p >= '0' && *p <= '9') {
      nonzero |= *p != '0';
      ++digits;
      ++p;
    }
  }
  if (digits == 0) return 0;
  if (p != e && (*p == 'e' || *p == 'E')) {
    const char* q = p + 1;
    if (q != e && (*q == '+' || *q == '-')) ++q;
    if (q != e && *q >= '0' && *q <= '9') {
      while (q != e && *q >= '0' && *q <= '9') ++q;
      p = q;
    }
  }
  if (p != e) return 0; /* ptr == end, csv.cpp:44 */
  const size_t len = (size_t)(e - b);
  char stack_buf[128];
  char* buf = len < sizeof stack_buf ? stack_buf : (char*)malloc(len + 1);
  if (!buf) return 0;
  memcpy(buf, b, len);
  buf[len] = 0;
  const double v = strtod(buf, NULL);
  if (buf != stack_buf) free(buf);
  if (isinf(v) || (v == 0.0 && nonzero)) return 0; /* std::errc::result_out_of_range */
  *out = v;
  return 1;
}

/* The field_index-th comma-separated field of [b, e) (split_row, csv.cpp:26-37). */
static int csv_field(const char* b, const char* e, uint64_t field_index, const char** fb, const char** fe) {
  uint64_t k = 0;
  const char* start = b;
  for (const char* p = b;; ++p) {
    if (p == e || *p == ',') {
      if (k == field_index) {
        *fb = start;
        *fe = p;
        return 1;
      }
      if (p == e) return 0;
      ++k;
      start = p + 1;
    }
  }
}

int gjo_csv_points(const char* text, uint64_t n_bytes, const char* lat_column,
                   const char* lng_column, int strict, double* out_latlng,
                   uint64_t cap, uint64_t* n_points, uint64_t* n_skipped,
                   uint64_t* bad_line) {
  const char* end = text + n_bytes;
  *n_points = 0;
  *n_skipped = 0;
  if (bad_line) *bad_line = 0;
  if (n_bytes == 0) return GJO_DATA_ERROR; /* csv.cpp:58-60: std::getline fails on an empty stream */
  /* header: read_line strips one trailing CR (csv.cpp:47-51) */
  const char* p = text;
  const char* nl = memchr(p, '\n', (size_t)(end - p));
  const char* le = nl ? nl : end;
  const char* next = nl ? nl + 1 : end;
  if (le != p && le[-1] == '\r') --le;
  const size_t lat_len = strlen(lat_column), lng_len = strlen(lng_column);
  uint64_t lat_index = 0, lng_index = 0;
  int lat_found = 0, lng_found = 0;
  for (uint64_t i = 0;; ++i) { /* csv.cpp:64-72: a later duplicate wins; lat is tested first */
    const char *fb, *fe;
    if (!csv_field(p, le, i, &fb, &fe)) break;
    const size_t flen = (size_t)(fe - fb);
    if (flen == lat_len && memcmp(fb, lat_column, flen) == 0) {
      lat_index = i;
      lat_found = 1;
    } else if (flen == lng_len && memcmp(fb, lng_column, flen) == 0) {
      lng_index = i;
      lng_found = 1;
    }
  }
  if (!lat_found || !lng_found) {
    if (bad_line) *bad_line = 1;
    return GJO_DATA_ERROR;
  }
  uint64_t line_number = 1, n = 0;
  for (p = next; p != end;) { /* csv.cpp:80-100 */
    nl = memchr(p, '\n', (size_t)(end - p));
    le = nl ? nl : end;
    next = nl ? nl + 1 : end;
    if (le != p && le[-1] == '\r') --le;
    ++line_number;
    if (le != p) { /* empty lines are skipped without counting */
      const char *ab, *ae, *ob, *oe;
      double lat = 0, lng = 0;
      const int ok = csv_field(p, le, lat_index, &ab, &ae) && csv_field(p, le, lng_index, &ob, &oe) &&
                     csv_parse_double(ab, ae, &lat) && csv_parse_double(ob, oe, &lng) &&
                     gjo_latlng_valid(lat, lng);
      if (ok) {
        if (n < cap) {
          out_latlng[2 * n] = lat;
          out_latlng[2 * n + 1] = lng;
        }
        ++n;
      } else if (strict) {
        if (bad_line) *bad_line = line_number;
        *n_points = n;
        return GJO_DATA_ERROR;
      } else {
        ++*n_skipped;
      }
    }
    p = next;
  }
  *n_points = n;
  return GJO_OK;
}
