/* geojoin_b200 — C ABI of the B200-native probe side of the adaptive
 * geospatial join (arXiv 1802.09488).
 *
 * This is the drop-in boundary for ONE path of the reference C++ library
 * `geojoin` (paths below are relative to the reference's proj/ directory):
 *
 *   points -> leaf cell id      cell_from_point            src/cell_id.cpp:82-95
 *   cell id -> tagged entry     Act::probe / probe_batch   src/act.cpp:248-270,310-315
 *                               detail::ProbeBatchFn       include/geojoin/act.hpp:270-283
 *   entry -> references         Act::for_each_reference    include/geojoin/act.hpp:169-196
 *   candidates -> PIP refine    pip_test                   src/geometry.cpp:184-204
 *   emit / count / stats        run_join, join_exact,      src/join.cpp:88-140,237-247
 *                               join_approx,
 *                               join_count_per_polygon,    src/join.cpp:255-285
 *                               accumulate_probe_stats     src/join.cpp:287-290
 *
 * Everything is plain C: pointers and sizes, no C++/torch types.  The index
 * is built OFFLINE by the reference's own build_index (src/join.cpp:152-235)
 * or read from its GJX1 bundle file (src/join.cpp:316-381); this library
 * copies it into a GPU's HBM — or replicates it into the HBM of several
 * (gj_group_*, gj_index_replicate) — and runs the probe path there.  There is
 * no CPU fallback: every entry point needs a CUDA device and fails with
 * GJ_CUDA_ERROR otherwise.  The library reads no environment variable; tuning
 * knobs and test hooks are the fields of gj_options.
 *
 * Threading: a gj_index is immutable after creation (like the reference's
 * IndexBundle, include/geojoin/join.hpp:86-88).  A gj_session owns one CUDA
 * stream plus scratch buffers and must not be used by two threads at once;
 * any number of sessions may share one index.
 */
#ifndef GEOJOIN_B200_H_
#define GEOJOIN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(_WIN32)
#define GJ_API
#else
#define GJ_API __attribute__((visibility("default")))
#endif

/* Status codes.  The reference signals the same conditions with exceptions;
 * include/geojoin_gpu.hpp re-throws the matching types. */
typedef enum {
  GJ_OK = 0,
  GJ_INVALID_POINT = 1,    /* std::invalid_argument, src/cell_id.cpp:83-85 */
  GJ_INVALID_ARGUMENT = 2, /* bad handle / size / mode */
  GJ_CORRUPT_INDEX = 3,    /* CorruptionError: src/act.cpp:141-153,269,654-716 */
  GJ_UNKNOWN_POLYGON = 4,  /* CorruptionError, src/join.cpp:111-114 */
  GJ_CUDA_ERROR = 5,
  GJ_CAPACITY = 6,         /* caller-provided output buffer too small */
  GJ_IO_ERROR = 7,
  GJ_DATA_ERROR = 8        /* DataError: src/csv.cpp:58-77,91-94 */
} gj_status;

/* Join mode.  GJ_MODE_BUNDLE takes the mode negotiated at build time, as
 * join_count_per_polygon does (src/join.cpp:257). */
typedef enum { GJ_MODE_BUNDLE = 0, GJ_MODE_APPROX = 1, GJ_MODE_EXACT = 2 } gj_mode;

typedef struct gj_index gj_index;
typedef struct gj_session gj_session;

/* Borrowed host views of a built reference index: the fields of
 * ActProbeView (include/geojoin/act.hpp:108-116), Act::node_count() /
 * lookup_table() (act.hpp:213-214), ActConfig::k_max (act.hpp:34),
 * BuildReport::mode (join.hpp:66) and IndexBundle::polygons() flattened to
 * CSR (join.hpp:90).  Nothing is retained after gj_index_create returns. */
typedef struct {
  const uint64_t* arena;      /* node n (1-based) at [(n-1)*256, n*256) */
  uint64_t node_count;
  const uint32_t* lut;        /* records [t, id*t, c, id*c] */
  uint64_t lut_len;
  uint64_t roots[8];          /* node id per face, 0 = none */
  uint64_t prefixes[8];
  uint64_t prefix_bits[8];    /* multiples of 8, <= 56 */
  int32_t k_max;              /* 8, 16, ..., 56 or 60 */
  int32_t approx_mode;        /* 1 when the bundle was negotiated approx */
  uint64_t n_polygons;
  const uint32_t* polygon_ids;/* bundle order, ids < 2^30 */
  const uint64_t* vtx_off;    /* n_polygons + 1 */
  const double* vtx_latlng;   /* (lat, lng) pairs, ring not closed */
} gj_index_desc;

typedef struct {
  uint64_t node_count;
  uint64_t lut_len;
  uint64_t n_polygons;
  uint64_t n_ids;             /* length of the id table (count slots) */
  uint64_t device_bytes;      /* HBM held by this index */
  int32_t k_max;
  int32_t approx_mode;
  int32_t device;
  int32_t dir_level;          /* first 32-bit directory tier (trie-node boundary): grid level */
  int32_t dir_width;          /* its window, cells */
  int32_t dir_height;
  int32_t dir_dict_len;       /* terminal entries that do not fit a directory code */
  int32_t dir2_level;         /* second, L2-resident directory tier (0 = absent) */
  int32_t dir2_width;
  int32_t dir2_height;
  int32_t ids_dense;          /* 1 when id == slot for every polygon */
  int32_t dir16_level;        /* the join kernel's shared-memory tier (16-bit codes) */
  int32_t dir16_width;
  int32_t dir16_height;
  int32_t link_records;       /* link cells of the deepest tier that got a refinement record (0 = none built) */
  int32_t k1_direct;          /* 1 when the join kernel runs its direct form on this index (gj_options.direct) */
  int32_t reserved0;
} gj_index_info;

/* Explicit tuning knobs and test hooks (the shipped library reads NO environment
 * variable).  Zero-initialise with gj_options_default and change what you need;
 * every field's default is the shipped behaviour.  Passed to the *_ex creators
 * and kept by the index (sessions read the launch knobs from it). */
typedef struct {
  uint32_t struct_size;         /* sizeof(gj_options), set by gj_options_default */
  int32_t dir16_max_entries;    /* cells of the join kernel's shared-memory tier; 0 = sized to the carve-out step */
  int32_t dir16_level_max;      /* cap its grid level (a density-matched stand-in over a small box can emulate
                                   the tier level the full-size box gets); 0 = none */
  int32_t node_pal_max_mb;      /* palette nodes are built while they fit this many MB; -1 = default, 0 = never */
  int32_t tier_sub;             /* refined 32-bit tier: -1 = automatic, 0 = none, 1..3 = that many grid levels */
  int32_t ids_late;             /* first ids written where a point is settled: -1 = automatic, 0 / 1 = force */
  int32_t queue_unpacked;       /* test hook: 1 = force the fallback queue coding */
  int32_t queue_slot_hi_bits;   /* test hook: at least this many high arena-slot bits travel in the first queue word */
  int32_t hist_rep_cap;         /* cap the shared-memory histogram replication; -1 = none, 0 = count through the
                                   per-CTA private copies */
  int32_t smem_pad;             /* unused shared memory added to the join kernel (L1 carve-out experiments) */
  int32_t debug_plan;           /* 1 = print the join kernel's shared-memory plan to stderr */
  int32_t hist16;               /* id tables beyond the 32-bit shared histogram count in a 16-bit one with
                                   periodic flushes: -1 = automatic, 0 = never, 1 = also when the 32-bit one fits */
  int32_t strip_index;          /* the refine kernel's strip lists hold vertex indices instead of 32-byte edge records:
                                   -1 = automatic (polygon sets whose records would exceed 32 MB), 0 = never, 1 = always */
  int32_t stage_lut;            /* lookup-table records of a population-3 batch staged in shared memory by the whole
                                   warp: -1 = automatic (tables of 256 MB and more), 0 = never, 1 = always */
  int32_t link_sub;             /* sparse refinement of the deepest 32-bit tier for the join kernel: one 64-byte record
                                   per LINK cell, 16 codes two grid levels finer, each resolved when the aligned run of
                                   16 slots it owns in the linked node is uniform: -1 = automatic (trees too large for
                                   palette nodes whose records stay L2-resident), 0 = never, 1 = always */
  int32_t direct;               /* the join kernel's direct form — every point gathers its own code of the 32-bit tier,
                                   asynchronously into shared memory, instead of being queued for it: -1 = automatic
                                   (indexes whose shared-memory tier resolves nothing), 0 = never, 1 = whenever possible */
  int32_t reserved1;
  uint64_t max_launch_points;   /* test hook: split device-resident calls into launches of this many points; 0 = none */
  uint64_t chunk_points;        /* host pipeline: points per chunk; 0 = default (3 M counts / 4 M pairs), min 4096 */
} gj_options;

GJ_API void gj_options_default(gj_options* opt);

/* JoinStats (include/geojoin/join.hpp:77-84), in this order. */
typedef struct {
  uint64_t probes;
  uint64_t pip_tests;
  uint64_t false_hits;
  uint64_t solely_true_hits;
  uint64_t refinement_entered;
  uint64_t candidate_refs;
} gj_stats;

GJ_API const char* gj_last_error(void);
GJ_API int gj_device_count(void);

/* ---- index -------------------------------------------------------------
 * gj_index_create validates once what the reference checks lazily or at load
 * time (Act::load / rebuild_derived, src/act.cpp:654-716; check_record,
 * src/act.cpp:141-153): face block ranges, the node graph being a forest of
 * depth <= ceil((k_max - prefix_bits)/8), every lookup-table record in
 * bounds.  After that the kernels run check-free.  `device` < 0 = current. */
GJ_API int gj_index_create(const gj_index_desc* desc, int device, gj_index** out);
/* Same with explicit options (NULL = defaults). */
GJ_API int gj_index_create_ex(const gj_index_desc* desc, int device, const gj_options* opt,
                              gj_index** out);

/* Reads the reference's GJX1 bundle file (IndexBundle::save,
 * src/join.cpp:316-339, wrapping the ACT1 snapshot, src/act.cpp:600-622)
 * straight into HBM without constructing the reference's Act. */
GJ_API int gj_index_load_file(const char* gjx1_path, int device, gj_index** out);
GJ_API int gj_index_load_file_ex(const char* gjx1_path, int device, const gj_options* opt,
                                 gj_index** out);

/* Replicates an index into another GPU's HBM (or once more into the same one)
 * device to device — over NVLink when the GPUs are peers — without going back
 * to the host arrays: north_star's "index replicated on each GPU".  The copy is
 * independent of `src` afterwards. */
GJ_API int gj_index_replicate(const gj_index* src, int device, gj_index** out);

GJ_API void gj_index_destroy(gj_index* ix);
GJ_API int gj_index_get_info(const gj_index* ix, gj_index_info* info);

/* The id table: sorted unique polygon ids (the bundle's plus every id the
 * trie can emit).  Per-polygon count arrays below are indexed by position
 * in this table; `ids` must hold info.n_ids values. */
GJ_API int gj_index_ids(const gj_index* ix, uint32_t* ids);

/* ---- session ------------------------------------------------------------ */
GJ_API int gj_session_create(gj_index* ix, gj_session** out);
GJ_API void gj_session_destroy(gj_session* s);
/* The CUDA stream (cudaStream_t) the session launches on. */
GJ_API void* gj_session_stream(gj_session* s);

/* Pinned host memory for the *_host entry points (plain cudaHostAlloc). */
GJ_API void* gj_host_alloc(size_t bytes);
GJ_API void gj_host_free(void* p);

/* ---- cell ids: cell_from_point (src/cell_id.cpp:82-95) over an array ------
 * out_raw[i] is bitwise cell_from_point(p_i, level).raw; an invalid point
 * returns GJ_INVALID_POINT, a level outside [0, 30] GJ_INVALID_ARGUMENT
 * (both std::invalid_argument in the reference). */
GJ_API int gj_cells_from_points_host(gj_session* s, const double* latlng, uint64_t n,
                                     int level, uint64_t* out_raw, uint64_t* bad_index);

/* ---- probe only: the ProbeBatchFn contract (act.hpp:270-276) at scale ----
 * out[i] is bitwise Act::probe(cell_from_point(p_i, k_max/2)); misses are 0.
 * An invalid point returns GJ_INVALID_POINT with the first bad index. */
GJ_API int gj_probe_points_host(gj_session* s, const double* latlng, uint64_t n,
                                uint64_t* out_entries, uint64_t* bad_index);
/* out[i] is bitwise Act::probe(CellId{raw[i]}) for ids already discretised
 * at level k_max/2 (all 8 face values accepted, as in the batch kernels). */
GJ_API int gj_probe_cells_host(gj_session* s, const uint64_t* raw_ids, uint64_t n,
                               uint64_t* out_entries);

/* ---- point ingestion: CsvPointReader (include/geojoin/io.hpp:43-68,
 * src/csv.cpp:26-100) over a text buffer, parsed on the device --------------
 * A header row names the columns; every following non-empty row whose
 * lat_column / lng_column fields are, after leading blanks, exactly one decimal
 * number each (std::from_chars semantics, correctly rounded) and form a valid
 * point is written to out_latlng in order, up to `cap` points; *n_points is
 * their total (call again with a larger buffer if it exceeds cap).  Other rows
 * are counted in *n_skipped, or — strict != 0 — end the call with
 * GJ_DATA_ERROR and their 1-based line number in *bad_line.  GJ_DATA_ERROR
 * with *bad_line == 0: the input is empty; == 1: the header lacks a column
 * (gj_last_error names it, like the reference's message). */
GJ_API int gj_points_from_csv_host(gj_session* s, const char* text, uint64_t n_bytes,
                                   const char* lat_column, const char* lng_column, int strict,
                                   double* out_latlng, uint64_t cap, uint64_t* n_points,
                                   uint64_t* n_skipped, uint64_t* bad_line);

/* ---- training pre-pass: the probe half of Act::train (act.cpp:414-440) ----
 * Finds the points whose probe lands in a candidate-bearing cell, i.e. for
 * which the reference's `any_candidate` is true: the only points Act::train
 * does split work for, and the numerator of TrainingStats::expensive_fraction_*.
 * Writes their global indices (base_index + i), ascending, into
 * out_indices[0 .. min(cap, *n_candidates)); *n_candidates is always the total
 * (so expensive_fraction = *n_candidates / n; call with cap = 0 to size).
 * A point that hits no candidate cell now never does after further training
 * (splits only refine candidate cells), so the list is a valid work list for
 * the whole training pass.  An invalid point returns GJ_INVALID_POINT. */
GJ_API int gj_training_candidates_host(gj_session* s, const double* latlng, uint64_t n,
                                       uint64_t base_index, uint64_t* out_indices, uint64_t cap,
                                       uint64_t* n_candidates, uint64_t* bad_index);

/* ---- streaming join: per-polygon counts (+ first id per point) ----------
 * ≙ join_count_per_polygon / run_join with a counting emit.
 *   counts[n_ids]   ADDED to (caller zeroes); slot order = gj_index_ids.
 *   stats           optional JoinStats, ADDED to.
 *   out_first_id[n] optional: the first emitted polygon id of point i in the
 *                   reference's emit order, GJ_NO_MATCH if none; bit 31
 *                   (GJ_MORE_FLAG) set when the point emitted more pairs —
 *                   those are appended to the overflow list.
 *   out_first_id    ... GJ_DEFERRED marks a point whose pairs (zero or more)
 *                   are ALL in the overflow list: in exact mode a point with
 *                   candidate references is resolved by the refine kernel.
 *   overflow        optional (point_index, polygon_id) records for every pair
 *                   not held inline by out_first_id, sorted by point index and
 *                   then by the reference's emit order.  overflow->count
 *                   returns the number produced; GJ_CAPACITY if it exceeds
 *                   the capacity.
 * base_index offsets reported point indices (join.cpp:66-67). */
#define GJ_NO_MATCH 0xFFFFFFFFu
#define GJ_DEFERRED 0xFFFFFFFEu
#define GJ_MORE_FLAG 0x80000000u

typedef struct {
  uint64_t* point_index; /* capacity records */
  uint32_t* polygon_id;
  uint64_t capacity;
  uint64_t count;        /* out */
} gj_overflow;

GJ_API int gj_join_count_host(gj_session* s, const double* latlng, uint64_t n,
                              uint64_t base_index, int mode, uint64_t* counts,
                              gj_stats* stats, uint32_t* out_first_id,
                              gj_overflow* overflow, uint64_t* bad_index);

/* Same with points already resident in HBM (device pointers; asynchronous on
 * the session stream unless `sync` != 0).  d_counts/d_stats are device
 * arrays (u64[n_ids], u64[6]) that are ADDED to; d_first_id may be NULL.
 * No overflow list here: a point with further pairs only carries GJ_MORE_FLAG,
 * and in exact mode a point whose pairs depend on refinement reads
 * GJ_DEFERRED (its pairs are in the counts); use the *_host calls for lists.
 * Errors (invalid point, unknown polygon) are latched in the session and
 * returned by gj_session_sync.  Any n is accepted: one kernel launch takes up
 * to 2^31 - 1 points (2^30 - 1 / 2^29 - 1 for indexes of 2^24 / 2^25 trie nodes
 * and more) and longer calls run as several launches; the error index reported
 * is the smallest offending one of the whole call. */
GJ_API int gj_join_count_device(gj_session* s, const double* d_latlng, uint64_t n,
                                int mode, uint64_t* d_counts, uint64_t* d_stats,
                                uint32_t* d_first_id, int sync);
GJ_API int gj_session_sync(gj_session* s, uint64_t* bad_index);
/* Number of kernels this session has launched so far. */
GJ_API uint64_t gj_session_launches(const gj_session* s);

/* ---- materialised join: ≙ join_exact / join_approx ----------------------
 * Pairs in the reference's order (ascending point index, references in index
 * order, join.hpp:125-127) as CSR: row_ptr[n+1], polygon_id[row_ptr[n]].
 * Two calls: gj_join_pairs_host runs the join and keeps the result in the
 * session; gj_pairs_copy copies it out. */
GJ_API int gj_join_pairs_host(gj_session* s, const double* latlng, uint64_t n,
                              int mode, uint64_t* n_pairs, gj_stats* stats,
                              uint64_t* bad_index);
GJ_API int gj_pairs_copy(gj_session* s, uint64_t* row_ptr, uint32_t* polygon_id);

/* The same join in ONE call with caller-provided output arrays: row_ptr[n + 1]
 * and polygon_id[id_capacity].  The pipeline keeps the running pair count on the
 * device, so chunks follow each other without a host round trip, and chunk c's
 * rows and ids travel to the caller's arrays while chunk c + 1 runs (directly
 * when they are pinned, gj_host_alloc).  *n_pairs is always the join's pair
 * count; when it exceeds id_capacity the call returns GJ_CAPACITY with row_ptr
 * complete and polygon_id undefined — allocate *n_pairs ids and call again
 * (id_capacity 0 sizes the output). */
GJ_API int gj_join_pairs_host_into(gj_session* s, const double* latlng, uint64_t n, int mode,
                                   uint64_t* row_ptr, uint32_t* polygon_id, uint64_t id_capacity,
                                   uint64_t* n_pairs, gj_stats* stats, uint64_t* bad_index);

/* CSR without the host detour: points, row offsets and polygon ids all in HBM
 * (device pointers; d_row_ptr u64[n + 1], d_polygon_id u32[id_capacity]) — what
 * a multi-GPU CSR pipeline keeps sharded per device (BASELINE configs[4]).
 * Synchronous; same capacity convention as gj_join_pairs_host_into. */
GJ_API int gj_join_pairs_device(gj_session* s, const double* d_latlng, uint64_t n, int mode,
                                uint64_t* d_row_ptr, uint32_t* d_polygon_id, uint64_t id_capacity,
                                uint64_t* n_pairs, gj_stats* stats, uint64_t* bad_index);

/* ---- all GPUs of the box for ONE input: ≙ the worker fan-out of
 * join_count_per_polygon (src/join.cpp:255-285) ------------------------------
 * A group holds one index replica + session per listed device (a device may be
 * listed more than once; replicas share nothing).  The first replica is built
 * from the host arrays / the GJX1 file, the others are copied from it device to
 * device (gj_index_replicate).  A group call splits its points into contiguous
 * ranges [n*g/G, n*(g+1)/G) — the reference's worker split, join.cpp:264-265 —
 * runs range g on replica g with base_index + n*g/G from its own host thread
 * (own PCIe link, own copy engines), and merges like the reference does
 * (join.cpp:280-284): per-polygon counts and JoinStats are summed; first ids and
 * CSR rows are written in place at their global positions; overflow records and
 * CSR ids are concatenated in range order, which is the global order.  Nothing
 * crosses GPUs on the probe path.  `workers` = how many replicas take part
 * (the reference's `threads`): <= 0 or > size means all of them.
 * Results do not depend on it (tests/test_join.cpp:200-214). */
typedef struct gj_group gj_group;

GJ_API int gj_group_create(const gj_index_desc* desc, const int* devices, int n_devices,
                           const gj_options* opt, gj_group** out);
GJ_API int gj_group_load_file(const char* gjx1_path, const int* devices, int n_devices,
                              const gj_options* opt, gj_group** out);
GJ_API void gj_group_destroy(gj_group* g);
GJ_API int gj_group_size(const gj_group* g);
/* Borrowed handles of replica k (owned by the group). */
GJ_API gj_index* gj_group_index(gj_group* g, int k);
GJ_API gj_session* gj_group_session(gj_group* g, int k);

GJ_API int gj_group_join_count_host(gj_group* g, int workers, const double* latlng, uint64_t n,
                                    uint64_t base_index, int mode, uint64_t* counts,
                                    gj_stats* stats, uint32_t* out_first_id,
                                    gj_overflow* overflow, uint64_t* bad_index);
GJ_API int gj_group_join_pairs_host(gj_group* g, int workers, const double* latlng, uint64_t n,
                                    int mode, uint64_t* n_pairs, gj_stats* stats,
                                    uint64_t* bad_index);
GJ_API int gj_group_pairs_copy(gj_group* g, uint64_t* row_ptr, uint32_t* polygon_id);

#ifdef __cplusplus
}
#endif
#endif /* GEOJOIN_B200_H_ */
