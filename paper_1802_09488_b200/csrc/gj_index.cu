// Index ingestion: validate a built reference index once, derive the id
// table, closed polygon rings and the shared-memory directory, and copy it
// all into one GPU's HBM.  Host C++ (the reference's counterpart is host C++
// too: Act::load / rebuild_derived, src/act.cpp:654-716, and
// IndexBundle::load, src/join.cpp:341-381).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <thread>
#include <unordered_map>

#include "gj_host.hpp"

namespace gj {

namespace {

thread_local std::string g_error;

constexpr uint64_t kMaxDirEntries = 32768;         // 128 KB of u32 codes (shared memory)
constexpr uint64_t kMaxDir2Entries = 16ull << 20;  // 64 MB of u32 codes (stays in the 126 MB L2)
constexpr uint64_t kMaxDirKEntries = 20ull << 20;  // the refined tier may take a little more: it replaces dir2 in K1
// sparse refinement records + the tier they hang off: what stays in the 126 MB L2 next to the point stream
constexpr uint64_t kMaxLinkSubBytes = 96ull << 20;
constexpr double kDirKMinLinkShare = 0.25;         // refine only when at least this share of the deepest tier's cells are links
// 136 KB of u16 codes: with K1's queues and histogram that stays inside the
// 196 KB shared-memory carve-out step (60 KB of L1 left for loads in flight);
// the next step up (228 KB) is a cliff, see plan_smem in gj_api.cu
constexpr uint64_t kMaxDir16Entries = 69632;
constexpr uint64_t kMaxNodePalBytes = 32ull << 20;  // palette nodes of a tree this small stay in L2 as a whole
constexpr uint64_t kMaxPolygonId = (1u << 30) - 1;
constexpr uint64_t kMaxEdgeRecordBytes = 32ull << 20;  // beyond this (estimated) size K2's strip lists hold vertex indices

struct Bitmap {
  std::vector<uint64_t> w;
  void ensure(uint64_t bit) {
    const uint64_t need = bit / 64 + 1;
    if (w.size() < need) w.resize(std::max<uint64_t>(need, w.size() * 2), 0);
  }
  bool test_and_set(uint64_t bit) {
    ensure(bit);
    const uint64_t m = 1ull << (bit & 63);
    const bool was = (w[bit >> 6] & m) != 0;
    w[bit >> 6] |= m;
    return was;
  }
  void set(uint64_t bit) { test_and_set(bit); }
};

// De-interleave `levels` quadrant pairs (y bit above x bit,
// cell_id.hpp:30-33) from the low 2*levels bits of v.
void unzip_pairs(uint64_t v, int levels, uint32_t* x, uint32_t* y) {
  uint32_t xx = 0, yy = 0;
  for (int i = levels - 1; i >= 0; --i) {
    const uint64_t pair = (v >> (2 * i)) & 3;
    xx = (xx << 1) | static_cast<uint32_t>(pair & 1);
    yy = (yy << 1) | static_cast<uint32_t>(pair >> 1);
  }
  *x = xx;
  *y = yy;
}

struct Cell {
  uint64_t node_or_entry;
  uint32_t x, y;
  int32_t step;  // terminals: grid level = prefix_level + 4*step
};

struct Box {
  uint64_t x_lo = ~0ull, y_lo = ~0ull, x_hi = 0, y_hi = 0;
  bool empty() const { return x_lo == ~0ull; }
  void add(uint64_t xl, uint64_t yl, uint64_t xh, uint64_t yh) {
    x_lo = std::min(x_lo, xl);
    y_lo = std::min(y_lo, yl);
    x_hi = std::max(x_hi, xh);
    y_hi = std::max(y_hi, yh);
  }
  uint64_t padded_area() const { return empty() ? 1 : (x_hi - x_lo + 2) * (y_hi - y_lo + 2); }
};

bool record_in_bounds(const gj_index_desc& d, uint64_t off) {  // act.cpp:141-153
  if (off >= d.lut_len) return false;
  const uint64_t t = d.lut[off];
  if (off + 1 + t >= d.lut_len) return false;
  const uint64_t c = d.lut[off + 1 + t];
  return off + 2 + t + c <= d.lut_len;
}

struct Analysis {
  std::vector<uint32_t> ids;
  HostDirectory dir;           // shared-memory tier
  HostDirectory dir2;          // global-memory (L2-resident) tier, deeper; may be empty
  HostDirectory dir16;         // K1's shared-memory tier (16-bit codes), see build_dir16
  HostDirectory dirk;          // K1's refined 32-bit tier (DevIndex::dirk); may be empty
  int dirk_sub = 0;            // its grid levels below the parent tier's (1..3)
  std::vector<uint32_t> link_sub;    // K1's sparse refinement records (DevIndex::link_sub); may be empty
  std::vector<uint32_t> tier_links;  // the deepest tier with record numbers in its link codes (DevIndex::tier_links)
  std::vector<uint64_t> dict;  // terminal entries that do not fit a directory code
  uint64_t max_refs = 0;       // most references behind one entry
  uint64_t max_cand_refs = 0;  // most candidate references behind one entry
};

// The first directory tier K1 keeps in shared memory: 16-bit codes over a
// window at `level`, derived from a 32-bit tier `tb` (the second tier when
// there is one, else the first) by downsampling.  A cell resolves here when
// every `tb` cell below it holds the same miss or the same inlined payload
// below 0xFFFE; anything else says "look in tb".  Codes: 0 = miss, 0xFFFF =
// look in tb, otherwise 1 + ((polygon_id << 1) | interior).  Any level up to
// tb's works (not only trie-node boundaries); the deepest whose padded window
// has at most `max_entries` cells is taken.
void build_dir16(const HostDirectory& tb, uint64_t max_entries, int max_level, HostDirectory* d16) {
  *d16 = HostDirectory{};
  d16->pitch = 1;
  d16->table16.assign(1, 0);  // an empty window is just its all-miss padding
  if (tb.width == 0 || tb.height == 0) return;
  for (int level = std::min(tb.level, max_level); level >= 0; --level) {
    const int down = tb.level - level;
    const uint32_t x0 = tb.x0 >> down, y0 = tb.y0 >> down;
    const uint32_t w = ((tb.x0 + tb.width - 1) >> down) - x0 + 1;
    const uint32_t h = ((tb.y0 + tb.height - 1) >> down) - y0 + 1;
    if (static_cast<uint64_t>(w + 1) * (h + 1) > max_entries && level > 0) continue;
    d16->level = level;
    d16->x0 = x0;
    d16->y0 = y0;
    d16->width = w;
    d16->height = h;
    d16->pitch = w + 1;
    d16->table16.assign(static_cast<size_t>(d16->pitch) * (h + 1), 0);
    const uint64_t side = 1ull << down;
    for (uint32_t cy = 0; cy < h; ++cy) {
      const uint64_t ty0 = static_cast<uint64_t>(y0 + cy) << down;
      for (uint32_t cx = 0; cx < w; ++cx) {
        const uint64_t tx0 = static_cast<uint64_t>(x0 + cx) << down;
        bool first = true, uniform = true;
        uint32_t code = 0;
        for (uint64_t ty = ty0; ty < ty0 + side && uniform; ++ty) {
          const bool row_in = ty >= tb.y0 && ty < static_cast<uint64_t>(tb.y0) + tb.height;
          for (uint64_t tx = tx0; tx < tx0 + side; ++tx) {
            uint32_t c = 0;  // outside tb's window: a miss
            if (row_in && tx >= tb.x0 && tx < static_cast<uint64_t>(tb.x0) + tb.width) {
              c = tb.table[(ty - tb.y0) * tb.pitch + (tx - tb.x0)];
            }
            if (first) {
              code = c;
              first = false;
            } else if (c != code) {
              uniform = false;
              break;
            }
          }
        }
        uint16_t c16 = 0xFFFF;
        if (uniform && code == 0) {
          c16 = 0;
        } else if (uniform && (code >> 30) == 1u && (code & 0x3FFFFFFFu) < 0xFFFEu) {
          c16 = static_cast<uint16_t>((code & 0x3FFFFFFFu) + 1u);
        }
        d16->table16[static_cast<size_t>(cy) * d16->pitch + cx] = c16;
      }
    }
    return;
  }
}

// One breadth-first pass per face: forest check, depth bound, record bounds,
// id collection; for face 0 the first levels also feed the directory.
int analyse(const gj_index_desc& d, const gj_options& opt, Analysis* out) {
  const bool k_ok = d.k_max >= 8 && d.k_max <= 60 && (d.k_max % 8 == 0 || d.k_max == 60);
  if (!k_ok) {  // validate_act_config, act.cpp:38-42
    set_error("k_max must be one of 8, 16, ..., 56, 60");
    return GJ_CORRUPT_INDEX;
  }
  if (d.node_count > (1ull << 32) || d.lut_len > 0x7fffffffull) {
    set_error("index header sizes out of range");
    return GJ_CORRUPT_INDEX;
  }
  if (d.node_count >= (1ull << 31)) {
    set_error("arenas of 2^31 nodes or more are not supported by the directory encoding");
    return GJ_INVALID_ARGUMENT;
  }
  Bitmap visited, id_seen, record_seen;
  visited.ensure(d.node_count + 1);
  for (uint64_t p = 0; p < d.n_polygons; ++p) {
    if (d.polygon_ids[p] > kMaxPolygonId) {
      set_error("polygon id above 2^30 - 1");
      return GJ_INVALID_ARGUMENT;
    }
    id_seen.set(d.polygon_ids[p]);
  }
  auto see_payload = [&](uint32_t payload) -> uint64_t {
    id_seen.set(payload >> 1);
    return (payload & 1u) ? 0 : 1;  // candidate?
  };
  auto check_terminal = [&](uint64_t e) -> bool {
    switch (e & 3) {
      case 1:
        out->max_cand_refs = std::max(out->max_cand_refs, see_payload(static_cast<uint32_t>(e >> 2) & 0x7fffffffu));
        out->max_refs = std::max<uint64_t>(out->max_refs, 1);
        return true;
      case 2:
        out->max_cand_refs = std::max(out->max_cand_refs,
                                      see_payload(static_cast<uint32_t>(e >> 33) & 0x7fffffffu) +
                                          see_payload(static_cast<uint32_t>(e >> 2) & 0x7fffffffu));
        out->max_refs = std::max<uint64_t>(out->max_refs, 2);
        return true;
      default: {
        const uint64_t off = (e >> 2) & 0x7fffffffu;
        if (!record_in_bounds(d, off)) return false;
        if (!record_seen.test_and_set(off)) {
          const uint32_t t = d.lut[off];
          const uint32_t c = d.lut[off + 1 + t];
          out->max_refs = std::max<uint64_t>(out->max_refs, static_cast<uint64_t>(t) + c);
          out->max_cand_refs = std::max<uint64_t>(out->max_cand_refs, c);
          for (uint32_t i = 0; i < t + c; ++i) {
            const uint32_t id = d.lut[off + 1 + i + (i >= t ? 1 : 0)];
            if (id > kMaxPolygonId) return false;  // kMaxPolygonId, geometry.hpp:25
            id_seen.set(id);
          }
        }
        return true;
      }
    }
  };

  HostDirectory& dir = out->dir;
  for (int face = 0; face < 6; ++face) {
    const uint64_t root = d.roots[face];
    const uint64_t plen = d.prefix_bits[face];
    if (root > d.node_count || plen > 56 || plen % 8 != 0) {  // act.cpp:644-647
      set_error("face block out of range");
      return GJ_CORRUPT_INDEX;
    }
    if (root == 0) continue;
    const int max_chunks = (d.k_max - static_cast<int>(plen) + 7) / 8;
    if (max_chunks < 1) {
      set_error("face prefix leaves no key bits below the root");
      return GJ_CORRUPT_INDEX;
    }
    const int prefix_level = static_cast<int>(plen) / 2;

    // Directory bookkeeping (face 0 only; cell_from_point never leaves it).
    // Two windows are kept: the deepest one small enough for shared memory
    // and the deepest one small enough to stay L2-resident in global memory.
    bool track = face == 0;
    std::vector<Cell> terminals;  // steps <= the deepest window still tracked
    std::vector<Cell> frontier;   // nodes at the current depth, with cells
    struct Snapshot {
      int chunks = -1;  // -1 = none taken
      Box box;
      std::vector<Cell> links;  // frontier at that depth
      size_t n_terminals = 0;
    } snap1, snap2;

    uint32_t px = 0, py = 0;
    unzip_pairs(d.prefixes[face], prefix_level, &px, &py);
    frontier.push_back(Cell{root, px, py, 0});
    if (track) {  // zero node steps: the prefix cell links to the root (the tier of last resort, e.g. k_max 60 under a 56-bit prefix)
      Box b0;
      b0.add(px, py, px, py);
      snap1 = snap2 = Snapshot{0, b0, frontier, 0};
    }
    for (int depth = 0; !frontier.empty(); ++depth) {
      if (depth >= max_chunks) {  // act.cpp:269 / act.cpp:693-696
        set_error("trie path longer than the maximum key length");
        return GJ_CORRUPT_INDEX;
      }
      std::vector<Cell> next;
      for (const Cell& c : frontier) {
        const uint64_t node = c.node_or_entry;
        if (node == 0 || node > d.node_count || visited.test_and_set(node)) {
          set_error("node graph is not a forest");  // act.cpp:667-669
          return GJ_CORRUPT_INDEX;
        }
        const uint64_t* slots = d.arena + (node - 1) * kNodeSlots;
        for (uint32_t s = 0; s < kNodeSlots; ++s) {
          const uint64_t e = slots[s];
          if (e == 0) continue;
          uint32_t sx = 0, sy = 0;
          if (track) unzip_pairs(s, 4, &sx, &sy);
          const Cell child{(e & 3) == 0 ? e >> 2 : e, (c.x << 4) | sx, (c.y << 4) | sy, depth + 1};
          if ((e & 3) == 0) {
            next.push_back(child);
          } else {
            if (!check_terminal(e)) {
              set_error("lookup-table record out of bounds or polygon id above 2^30 - 1");
              return GJ_CORRUPT_INDEX;
            }
            if (track) terminals.push_back(child);
          }
        }
      }
      if (track) {
        // Window at `depth + 1` node steps: every terminal so far (scaled to
        // this level) plus the cells of the nodes still to be expanded.
        Box box;
        for (const Cell& t : terminals) {
          const int s = 4 * (depth + 1 - t.step);
          box.add(static_cast<uint64_t>(t.x) << s, static_cast<uint64_t>(t.y) << s,
                  ((static_cast<uint64_t>(t.x) + 1) << s) - 1, ((static_cast<uint64_t>(t.y) + 1) << s) - 1);
        }
        for (const Cell& l : next) box.add(l.x, l.y, l.x, l.y);
        // A tier must sit at or above the leaf level: with k_max = 60 the last node step ends at "level 32",
        // two grid levels below the leaf level (its slots use 4 of their 8 key bits), where no window exists.
        const bool level_ok = prefix_level + 4 * (depth + 1) <= d.k_max / 2;
        // sized WITH the all-miss padding column and row, which the kernels stage as well
        if (level_ok && box.padded_area() <= kMaxDirEntries) snap1 = Snapshot{depth + 1, box, next, terminals.size()};
        if (level_ok && box.padded_area() <= kMaxDir2Entries) {
          snap2 = Snapshot{depth + 1, box, next, terminals.size()};
        } else {
          track = false;  // deeper windows only grow
          terminals.resize(snap2.n_terminals);
          terminals.shrink_to_fit();
        }
      }
      frontier.swap(next);
    }

    if (face == 0) {
      std::unordered_map<uint64_t, uint32_t> code_of;
      out->dict.assign(1, 0ull);
      auto fill = [&](const Snapshot& sn, HostDirectory& hd) {
        if (sn.chunks < 0 || sn.box.empty()) return;
        hd.chunks = sn.chunks;
        hd.level = prefix_level + 4 * sn.chunks;
        hd.x0 = static_cast<uint32_t>(sn.box.x_lo);
        hd.y0 = static_cast<uint32_t>(sn.box.y_lo);
        hd.width = static_cast<uint32_t>(sn.box.x_hi - sn.box.x_lo + 1);
        hd.height = static_cast<uint32_t>(sn.box.y_hi - sn.box.y_lo + 1);
        // one extra all-miss column and row: lookups clamp into them instead
        // of testing the window bounds
        hd.pitch = hd.width + 1;
        hd.table.assign(static_cast<size_t>(hd.pitch) * (hd.height + 1), 0u);
        for (size_t ti = 0; ti < sn.n_terminals; ++ti) {
          const Cell& t = terminals[ti];
          auto it = code_of.find(t.node_or_entry);
          if (it == code_of.end()) {
            const uint64_t e = t.node_or_entry;
            uint32_t code;
            if ((e & 3) == 1 && ((e >> 2) & 0x7fffffffu) < kDirInline) {
              code = kDirInline | static_cast<uint32_t>((e >> 2) & 0x3fffffffu);  // payload inlined
            } else {
              code = static_cast<uint32_t>(out->dict.size());
              out->dict.push_back(e);
            }
            it = code_of.emplace(e, code).first;
          }
          const int s = 4 * (sn.chunks - t.step);
          const uint64_t bx = (static_cast<uint64_t>(t.x) << s) - hd.x0;
          const uint64_t by = (static_cast<uint64_t>(t.y) << s) - hd.y0;
          const uint64_t side = 1ull << s;
          for (uint64_t yy = 0; yy < side; ++yy) {
            uint32_t* row = hd.table.data() + (by + yy) * hd.pitch + bx;
            std::fill(row, row + side, it->second);
          }
        }
        for (const Cell& l : sn.links) {
          hd.table[static_cast<size_t>(l.y - hd.y0) * hd.pitch + (l.x - hd.x0)] =
              kDirLink | static_cast<uint32_t>(l.node_or_entry);
        }
      };
      fill(snap1, dir);
      if (snap2.chunks > snap1.chunks) fill(snap2, out->dir2);

      // K1's refined tier (DevIndex::dirk): the deepest tier again, `sub` grid levels finer.  A cell below a
      // link owns an aligned run of 4^(4 - sub) slots of the linked node (slots are in Z-order, act.cpp:200-206);
      // when the run holds one terminal entry, or nothing, the cell resolves here, else it keeps the link.
      const HostDirectory& base = out->dir2.table.empty() ? dir : out->dir2;
      if (!base.table.empty() && base.width && base.height) {
        uint64_t n_links = 0;
        for (uint32_t y = 0; y < base.height; ++y) {
          for (uint32_t x = 0; x < base.width; ++x) n_links += (base.table[static_cast<size_t>(y) * base.pitch + x] & kDirLink) != 0;
        }
        const int room = std::min(3, d.k_max / 2 - base.level);  // never finer than the leaf level
        int sub = 0;
        const double share = static_cast<double>(n_links) / (static_cast<double>(base.width) * base.height);
        if (share >= kDirKMinLinkShare) {
          for (int r = 1; r <= room; ++r) {
            if (((static_cast<uint64_t>(base.width) << r) + 1) * ((static_cast<uint64_t>(base.height) << r) + 1) <= kMaxDirKEntries) sub = r;
          }
        }
        if (opt.tier_sub >= 0) sub = std::max(0, std::min(room, static_cast<int>(opt.tier_sub)));  // explicit knob / test hook
        if (sub > 0) {
          HostDirectory& hk = out->dirk;
          out->dirk_sub = sub;
          hk.chunks = base.chunks;
          hk.level = base.level + sub;
          hk.x0 = base.x0 << sub;
          hk.y0 = base.y0 << sub;
          hk.width = base.width << sub;
          hk.height = base.height << sub;
          hk.pitch = hk.width + 1;
          hk.table.assign(static_cast<size_t>(hk.pitch) * (hk.height + 1), 0u);
          const uint32_t side = 1u << sub;
          const uint32_t run = 1u << (2 * (4 - sub));  // slots per refined cell
          for (uint32_t y = 0; y < base.height; ++y) {
            for (uint32_t x = 0; x < base.width; ++x) {
              const uint32_t c = base.table[static_cast<size_t>(y) * base.pitch + x];
              const uint64_t* slots = (c & kDirLink) ? d.arena + (static_cast<uint64_t>(c & ~kDirLink) - 1) * kNodeSlots : nullptr;
              for (uint32_t q = 0; q < side * side; ++q) {
                uint32_t qx = 0, qy = 0;
                unzip_pairs(q, sub, &qx, &qy);
                uint32_t code = c;
                if (slots) {
                  const uint64_t* r0 = slots + static_cast<size_t>(q) * run;
                  const uint64_t e = r0[0];
                  bool uniform = e == 0 || (e & 3) != 0;
                  for (uint32_t k = 1; k < run && uniform; ++k) uniform = r0[k] == e;
                  if (uniform) {
                    if (e == 0) {
                      code = 0;
                    } else {
                      auto it = code_of.find(e);
                      if (it == code_of.end()) {
                        uint32_t nc;
                        if ((e & 3) == 1 && ((e >> 2) & 0x7fffffffu) < kDirInline) {
                          nc = kDirInline | static_cast<uint32_t>((e >> 2) & 0x3fffffffu);
                        } else {
                          nc = static_cast<uint32_t>(out->dict.size());
                          out->dict.push_back(e);
                        }
                        it = code_of.emplace(e, nc).first;
                      }
                      code = it->second;
                    }
                  }
                }
                hk.table[static_cast<size_t>((y << sub) + qy) * hk.pitch + ((x << sub) + qx)] = code;
              }
            }
          }
        }
        // K1's sparse refinement (DevIndex::link_sub): the same idea for the link cells ONLY — 16 codes per link
        // cell, one per 128-byte line of the linked node (a 4 x 4 block two grid levels finer).  Automatic for
        // trees that get no palette nodes (the arena is far beyond L2, every open point a DRAM burst) when the
        // records stay L2-resident next to the tier; create_index drops it again if the queue coding ends up unpacked.
        bool want_links = sub == 0 && n_links != 0;
        if (want_links && opt.link_sub < 0) {
          uint64_t max_pal = kMaxNodePalBytes;
          if (opt.node_pal_max_mb >= 0) max_pal = static_cast<uint64_t>(opt.node_pal_max_mb) << 20;
          want_links = d.node_count * 128 > max_pal && n_links * 64 + base.table.size() * 4 <= kMaxLinkSubBytes;
        } else if (opt.link_sub == 0) {
          want_links = false;
        }
        if (want_links) {
          out->tier_links = base.table;
          out->link_sub.reserve(n_links * 16);
          uint32_t next_record = 0;
          for (uint32_t y = 0; y < base.height; ++y) {
            for (uint32_t x = 0; x < base.width; ++x) {
              const size_t cell = static_cast<size_t>(y) * base.pitch + x;
              const uint32_t c = base.table[cell];
              if (!(c & kDirLink)) continue;
              out->tier_links[cell] = kDirLink | ++next_record;
              const uint64_t* slots = d.arena + (static_cast<uint64_t>(c & ~kDirLink) - 1) * kNodeSlots;
              for (uint32_t q = 0; q < 16; ++q) {
                const uint64_t* r0 = slots + q * 16u;
                const uint64_t e = r0[0];
                bool uniform = e == 0 || (e & 3) != 0;
                for (uint32_t k = 1; k < 16 && uniform; ++k) uniform = r0[k] == e;
                uint32_t code = c;  // mixed run: the node itself, read from the arena
                if (uniform && e == 0) {
                  code = 0;
                } else if (uniform) {
                  auto it = code_of.find(e);
                  if (it == code_of.end()) {
                    uint32_t nc;
                    if ((e & 3) == 1 && ((e >> 2) & 0x7fffffffu) < kDirInline) {
                      nc = kDirInline | static_cast<uint32_t>((e >> 2) & 0x3fffffffu);
                    } else {
                      nc = static_cast<uint32_t>(out->dict.size());
                      out->dict.push_back(e);
                    }
                    it = code_of.emplace(e, nc).first;
                  }
                  code = it->second;
                }
                out->link_sub.push_back(code);
              }
            }
          }
        }
      }
    }
  }
  if (dir.level > 30 || out->dir2.level > 30) {
    set_error("directory level out of range");
    return GJ_CORRUPT_INDEX;
  }

  // id table: sorted unique ids
  for (uint64_t wi = 0; wi < id_seen.w.size(); ++wi) {
    uint64_t bits = id_seen.w[wi];
    while (bits) {
      const int b = __builtin_ctzll(bits);
      out->ids.push_back(static_cast<uint32_t>(wi * 64 + b));
      bits &= bits - 1;
    }
  }
  return GJ_OK;
}

template <typename T>
int upload(DeviceBuffer& buf, const T* src, size_t count, size_t* total) {
  const size_t bytes = std::max<size_t>((count * sizeof(T) + 15) & ~size_t{15}, 16);  // K1 stages tables as uint4
  GJ_CUDA(buf.reserve(bytes));
  if (count) GJ_CUDA(cudaMemcpy(buf.ptr, src, count * sizeof(T), cudaMemcpyHostToDevice));
  *total += bytes;
  return GJ_OK;
}

}  // namespace

void set_error(const std::string& msg) { g_error = msg; }
const std::string& last_error() { return g_error; }

int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return GJ_CUDA_ERROR;
}

gj_options default_options() {
  gj_options o{};
  o.struct_size = sizeof(gj_options);
  o.node_pal_max_mb = -1;
  o.tier_sub = -1;
  o.ids_late = -1;
  o.hist_rep_cap = -1;
  o.hist16 = -1;
  o.stage_lut = -1;
  o.link_sub = -1;
  o.direct = -1;
  o.strip_index = -1;
  return o;
}

int create_index(const gj_index_desc& d, int device, const gj_options* options, gj_index** out) {
  if (!out) return GJ_INVALID_ARGUMENT;
  *out = nullptr;
  if ((d.node_count && !d.arena) || (d.lut_len && !d.lut) ||
      (d.n_polygons && (!d.polygon_ids || !d.vtx_off || !d.vtx_latlng))) {
    set_error("null array in index description");
    return GJ_INVALID_ARGUMENT;
  }
  int n_dev = 0;
  if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) {
    set_error("no CUDA device: geojoin_b200 has no CPU fallback");
    return GJ_CUDA_ERROR;
  }
  if (device < 0) GJ_CUDA(cudaGetDevice(&device));
  GJ_CUDA(cudaSetDevice(device));

  gj_options opt = default_options();
  if (options) {
    if (options->struct_size != sizeof(gj_options)) {
      set_error("gj_options: struct_size mismatch (initialise with gj_options_default)");
      return GJ_INVALID_ARGUMENT;
    }
    opt = *options;
  }
  Analysis an;
  int rc = analyse(d, opt, &an);
  if (rc != GJ_OK) return rc;

  std::unique_ptr<gj_index> ix(new gj_index);
  ix->device = device;
  ix->opt = opt;
  ix->ids = std::move(an.ids);
  ix->max_refs = an.max_refs;
  ix->max_cand_refs = an.max_cand_refs;
  const size_t n_ids = ix->ids.size();
  bool dense = true;
  for (size_t i = 0; i < n_ids; ++i) dense = dense && ix->ids[i] == i;

  // Closed rings per id-table slot; the first polygon carrying an id wins
  // (unordered_map::emplace keeps the first, join.cpp:144-150).
  std::vector<uint64_t> ring_off(n_ids + 1, 0);
  std::vector<uint32_t> ring_len(n_ids, 0);
  std::vector<int64_t> first_poly(n_ids, -1);
  for (uint64_t p = 0; p < d.n_polygons; ++p) {
    const size_t slot =
        std::lower_bound(ix->ids.begin(), ix->ids.end(), d.polygon_ids[p]) - ix->ids.begin();
    if (first_poly[slot] < 0) first_poly[slot] = static_cast<int64_t>(p);
  }
  uint64_t total = 0;
  for (size_t s = 0; s < n_ids; ++s) {
    ring_off[s] = total;
    if (first_poly[s] >= 0) {
      const uint64_t nv = d.vtx_off[first_poly[s] + 1] - d.vtx_off[first_poly[s]];
      if (nv > (1ull << 24)) {  // join.cpp:368-370
        set_error("polygon vertex count out of range");
        return GJ_CORRUPT_INDEX;
      }
      ring_len[s] = static_cast<uint32_t>(nv);
      total += nv ? nv + 1 : 0;
    }
  }
  ring_off[n_ids] = total;
  std::vector<double2> ring_xy(total);
  for (size_t s = 0; s < n_ids; ++s) {
    if (ring_len[s] == 0) continue;
    const uint64_t b = d.vtx_off[first_poly[s]];
    double2* dst = ring_xy.data() + ring_off[s];
    for (uint32_t v = 0; v <= ring_len[s]; ++v) {
      const uint64_t src = b + (v == ring_len[s] ? 0 : v);  // v[(i + 1) % n], geometry.cpp:189
      dst[v] = make_double2(d.vtx_latlng[2 * src + 1], d.vtx_latlng[2 * src]);  // x = lng, y = lat
    }
  }

  // Latitude strips per polygon for the refine kernel (see StripMeta).
  std::vector<StripMeta> strip_meta(n_ids);
  std::vector<uint32_t> strip_ptr;
  std::vector<EdgeRecord> strip_edges;
  std::vector<uint32_t> strip_eidx;  // the compact form (DevIndex::strip_eidx), filled instead when the records get large
  // two strips per edge, ~3 listed edges per strip: ~6 records of 32 bytes per polygon edge
  const bool strips_indexed = opt.strip_index > 0 || (opt.strip_index < 0 && total * 6 * sizeof(EdgeRecord) > kMaxEdgeRecordBytes);
  if (strips_indexed && total >= (1ull << 32)) {
    set_error("polygon set exceeds 2^32 vertices");
    return GJ_INVALID_ARGUMENT;
  }
  {
    const double margin = 1e-9;  // pip_edge's rejection margin
    std::vector<std::vector<uint32_t>> lists;
    for (size_t s = 0; s < n_ids; ++s) {
      StripMeta& m = strip_meta[s];
      m = StripMeta{0.0, 0.0, 0u, static_cast<uint32_t>(strip_ptr.size())};
      const uint32_t ne = ring_len[s];
      if (ne == 0) continue;
      const double2* v = ring_xy.data() + ring_off[s];
      double y_lo = v[0].y, y_hi = v[0].y;
      for (uint32_t e = 1; e < ne; ++e) {
        y_lo = std::min(y_lo, v[e].y);
        y_hi = std::max(y_hi, v[e].y);
      }
      y_lo -= 2 * margin;
      y_hi += 2 * margin;
      // two strips per edge: lists of ~3 edges (measured on config 3: k = ne/2, ne, 2 ne, 4 ne give K2
      // 0.244, 0.220, 0.207, 0.205 ms per 3.5 M tasks; the strip table grows 1.0, 2.5, 5.6, 11.8 MB)
      m.k = std::min<uint32_t>(65536u, std::max<uint32_t>(1u, ne * 2));
      m.y0 = y_lo;
      m.inv_h = static_cast<double>(m.k) / (y_hi - y_lo);
      const double slack = (y_hi - y_lo) / m.k / 64.0;
      lists.assign(m.k, {});
      for (uint32_t e = 0; e < ne; ++e) {
        const double ya = v[e].y, yb = v[e + 1].y;
        // strip_of is monotone and evaluated identically on the device, so the
        // strips of [lo - margin, hi + margin] cover every point in that range;
        // `slack` (1/64 of a strip) is insurance against a host compiler that
        // rounds the expression differently.
        const uint32_t first = strip_of(std::min(ya, yb) - margin - slack, m.y0, m.inv_h, m.k);
        const uint32_t last = strip_of(std::max(ya, yb) + margin + slack, m.y0, m.inv_h, m.k);
        for (uint32_t st = first; st <= last; ++st) lists[st].push_back(e);
      }
      for (uint32_t st = 0; st < m.k; ++st) {
        strip_ptr.push_back(static_cast<uint32_t>(strips_indexed ? strip_eidx.size() : strip_edges.size()));
        for (uint32_t e : lists[st]) {
          if (strips_indexed) {
            strip_eidx.push_back(static_cast<uint32_t>(ring_off[s] + e));
          } else {
            const double2 a = v[e], b = v[e + 1];
            strip_edges.push_back(EdgeRecord{a.x, a.y, b.x, b.y});
          }
        }
      }
      strip_ptr.push_back(static_cast<uint32_t>(strips_indexed ? strip_eidx.size() : strip_edges.size()));
      if (std::max(strip_edges.size(), strip_eidx.size()) >= (1ull << 32)) {
        set_error("polygon strip table exceeds 2^32 edge records");
        return GJ_INVALID_ARGUMENT;
      }
    }
  }

  if (an.dir.table.empty()) {  // no tree on face 0: the window is just its all-miss padding
    an.dir = HostDirectory{};
    an.dir.pitch = 1;
    an.dir.table.assign(1, 0u);
  }
  {
    // the tier, K1's queues and one histogram row set must stay inside the 196 KB carve-out step
    const size_t besides = k1_smem_besides_tier(n_ids, opt);
    // (with the 16-bit histogram — tens of thousands of polygons, each a few tier cells across, so the tier
    // resolves little anyway — everything stays inside the 164 KB step and leaves L1 its 92 KB)
    const size_t step = ((k1_uses_hist16(n_ids, opt) ? 164u : 196u) - 1u) << 10;
    uint64_t max16 = std::min<uint64_t>(kMaxDir16Entries, step > besides ? (step - besides) / 2 : 0);
    ix->stage_records = k1_stages_records(d.lut_len, opt);
    if (ix->stage_records) max16 = std::min<uint64_t>(max16, 5120);  // 10 KB: the rest of shared memory stages records
    if (opt.dir16_max_entries > 0) max16 = std::min<uint64_t>(static_cast<uint64_t>(opt.dir16_max_entries), 110000);  // explicit knob
    // explicit knob: a density-matched stand-in over a small box can emulate the full-size tier
    const int max_level = opt.dir16_level_max > 0 ? std::min(30, static_cast<int>(opt.dir16_level_max)) : 30;
    build_dir16(an.dir2.table.empty() ? an.dir : an.dir2, max16, max_level, &an.dir16);
  }
  {  // first ids written late (join_kernel's kLate) when most of the 16-bit tier says "look in the 32-bit tier"
    uint64_t open_cells = 0;
    for (uint32_t y = 0; y < an.dir16.height; ++y) {
      for (uint32_t x = 0; x < an.dir16.width; ++x) open_cells += an.dir16.table16[static_cast<size_t>(y) * an.dir16.pitch + x] == 0xFFFFu;
    }
    const uint64_t cells = static_cast<uint64_t>(an.dir16.width) * an.dir16.height;
    ix->ids_late = cells != 0 && open_cells * 2 > cells;
    ix->dev.dir16_live = !(cells != 0 && open_cells * 20 > cells * 19);  // dead when more than 95 % of the cells are open
    if (opt.ids_late >= 0) ix->ids_late = opt.ids_late != 0;  // explicit knob / test hook
    // the direct form: every point gathers its own code of the 32-bit tier (no record staging in that form)
    ix->direct = (opt.direct > 0 || (opt.direct < 0 && !ix->dev.dir16_live && n_ids != 0)) && !ix->stage_records;
  }
  size_t bytes = 0;
  if ((rc = upload(ix->d_arena, d.arena, d.node_count * kNodeSlots, &bytes)) != GJ_OK) return rc;
  if ((rc = upload(ix->d_lut, d.lut, d.lut_len, &bytes)) != GJ_OK) return rc;
  if ((rc = upload(ix->d_ids, ix->ids.data(), n_ids, &bytes)) != GJ_OK) return rc;
  if ((rc = upload(ix->d_ring_off, ring_off.data(), ring_off.size(), &bytes)) != GJ_OK) return rc;
  if ((rc = upload(ix->d_ring_len, ring_len.data(), ring_len.size(), &bytes)) != GJ_OK) return rc;
  if ((rc = upload(ix->d_ring_xy, ring_xy.data(), ring_xy.size(), &bytes)) != GJ_OK) return rc;
  if ((rc = upload(ix->d_strip_meta, strip_meta.data(), strip_meta.size(), &bytes)) != GJ_OK) return rc;
  if ((rc = upload(ix->d_strip_ptr, strip_ptr.data(), strip_ptr.size(), &bytes)) != GJ_OK) return rc;
  if ((rc = upload(ix->d_strip_edges, strip_edges.data(), strip_edges.size(), &bytes)) != GJ_OK) return rc;
  if (strips_indexed && (rc = upload(ix->d_strip_eidx, strip_eidx.data(), strip_eidx.size(), &bytes)) != GJ_OK) return rc;
  if ((rc = upload(ix->d_dir_table, an.dir.table.data(), an.dir.table.size(), &bytes)) != GJ_OK) return rc;
  if ((rc = upload(ix->d_dir_dict, an.dict.data(), an.dict.size(), &bytes)) != GJ_OK) return rc;
  if ((rc = upload(ix->d_dir2_table, an.dir2.table.data(), an.dir2.table.size(), &bytes)) != GJ_OK) return rc;
  if ((rc = upload(ix->d_dir16_table, an.dir16.table16.data(), an.dir16.table16.size(), &bytes)) != GJ_OK) return rc;
  if ((rc = upload(ix->d_dirk_table, an.dirk.table.data(), an.dirk.table.size(), &bytes)) != GJ_OK) return rc;

  // Palette form of the nodes (DevIndex::node_pal), for K1's deep descents: built while the whole tree fits
  // 32 MB in this form and so stays in L2.  Larger trees do not get it by default: measured on BASELINE config 4 at
  // full size (18.3 M nodes, 2.3 GB of palette records next to the 37 GB arena) the join took 24.3 instead of
  // 18.1 ms per 1 B points with it — a random slot read costs one 128-byte DRAM burst either way, the hot part of
  // the tree does not stay in L2 even in this form, a quarter of the boundary nodes (three polygons meeting) hold
  // more than four distinct entries and pay a second burst in the arena, and the record costs three dependent
  // loads instead of one.  gj_options.node_pal_max_mb forces it.
  {
    uint64_t max_pal = kMaxNodePalBytes;
    if (opt.node_pal_max_mb >= 0) max_pal = static_cast<uint64_t>(opt.node_pal_max_mb) << 20;  // explicit knob
    if (d.node_count != 0 && d.node_count * 128 <= max_pal) {
      std::vector<uint64_t> pal(d.node_count * 16, 0);
      const unsigned n_workers = static_cast<unsigned>(std::max<uint64_t>(
          1, std::min<uint64_t>({16, std::thread::hardware_concurrency(), d.node_count / 4096 + 1})));
      std::vector<uint64_t> fit_count(n_workers, 0);
      auto build_range = [&](unsigned w) {
        const uint64_t first = d.node_count * w / n_workers, last = d.node_count * (w + 1) / n_workers;
        for (uint64_t node = first; node < last; ++node) {
          const uint64_t* slots = d.arena + node * kNodeSlots;
          uint64_t* rec = pal.data() + node * 16;
          uint64_t values[4];
          int n_values = 0;
          bool fits = true;
          for (int sl = 0; sl < kNodeSlots && fits; ++sl) {
            int code = 0;
            while (code < n_values && values[code] != slots[sl]) ++code;
            if (code == n_values) {
              if (n_values == 4) {
                fits = false;
                break;
              }
              values[n_values++] = slots[sl];
            }
            rec[4 + sl / 32] |= static_cast<uint64_t>(code) << (2 * (sl % 32));
          }
          if (fits) {
            for (int c = 0; c < 4; ++c) rec[c] = c < n_values ? values[c] : 0;
            ++fit_count[w];
          } else {
            for (int w16 = 0; w16 < 16; ++w16) rec[w16] = 0;
            rec[0] = ~0ull;  // more than 4 distinct entries: read the arena
          }
        }
      };
      std::vector<std::thread> pool;
      for (unsigned w = 1; w < n_workers; ++w) pool.emplace_back(build_range, w);
      build_range(0);
      for (std::thread& t : pool) t.join();
      uint64_t fit = 0;
      for (uint64_t f : fit_count) fit += f;
      (void)fit;
      if ((rc = upload(ix->d_node_pal, pal.data(), pal.size(), &bytes)) != GJ_OK) return rc;
    }
  }

  DevIndex& dv = ix->dev;
  for (int f = 0; f < 8; ++f) {
    dv.roots[f] = f < 6 ? d.roots[f] : 0;  // refresh_view, act.cpp:373-383
    dv.prefixes[f] = f < 6 ? d.prefixes[f] : 0;
    dv.prefix_bits[f] = f < 6 ? static_cast<uint32_t>(d.prefix_bits[f]) : 0;
  }
  dv.n_ids = static_cast<uint32_t>(n_ids);
  dv.k_max = d.k_max;
  dv.leaf_level = d.k_max / 2;
  dv.prefix_level0 = static_cast<int>(d.prefix_bits[0]) / 2;
  dv.ids_dense = dense ? 1 : 0;
  auto set_dir = [](DevDirectory& dd, const HostDirectory& hd) {
    dd.width = hd.width;
    dd.height = hd.height;
    dd.pitch = hd.pitch;
    dd.x0 = hd.x0;
    dd.y0 = hd.y0;
    dd.n_table = static_cast<uint32_t>(hd.table.size());
    dd.shift = 30 - hd.level;
    dd.chunks = hd.chunks;
  };
  set_dir(dv.dir, an.dir);
  set_dir(dv.dir2, an.dir2);
  set_dir(dv.dir16, an.dir16);
  set_dir(dv.dirk, an.dirk);
  dv.dir16.n_table = static_cast<uint32_t>(an.dir16.table16.size());
  {  // queue coding for the 32-bit tier K1 gathers from
    const HostDirectory& tb = !an.dirk.table.empty() ? an.dirk : (an.dir2.table.empty() ? an.dir : an.dir2);
    const int tb_shift = 30 - tb.level;
    const int up = 4 - (an.dirk.table.empty() ? 0 : an.dirk_sub);  // grid levels from the tier to the next node boundary
    auto bits_for = [](uint64_t v) {  // smallest b with v <= 2^b
      uint32_t b = 0;
      while ((1ull << b) < v) ++b;
      return b;
    };
    const uint32_t xbits = bits_for((static_cast<uint64_t>(tb.width) + 1) << up);
    const uint32_t ybits = bits_for((static_cast<uint64_t>(tb.height) + 1) << up);
    DevQueueCoding& qc = dv.qc;
    qc = DevQueueCoding{};
    const bool force_unpacked = opt.queue_unpacked != 0;  // test hook for the fallback coding
    // high bits of an arena slot that travel in the first queue word (see DevQueueCoding)
    uint32_t slot_hi_bits = 0;
    while (slot_hi_bits < 3 && d.node_count >= (1ull << (24 + slot_hi_bits))) ++slot_hi_bits;
    if (opt.queue_slot_hi_bits > 0) {  // test hook: the wide-arena coding on a small index
      slot_hi_bits = std::max<uint32_t>(slot_hi_bits, static_cast<uint32_t>(opt.queue_slot_hi_bits));
    }
    qc.index_bits = 31;
    qc.slow_mark = 0x80000000u;
    if (!force_unpacked && tb_shift + 2 >= up && xbits + ybits <= 32 && slot_hi_bits <= 2) {  // slots below the kQueueSlow pattern
      qc.packed = 1;
      qc.index_bits = 31 - slot_hi_bits;
      qc.slow_mark = 0x80000000u | (((1u << slot_hi_bits) - 1u) << qc.index_bits);
      qc.shift = static_cast<uint32_t>(tb_shift + 2 - up);
      qc.x0 = tb.x0 << up;
      qc.y0 = tb.y0 << up;
      qc.x_clamp = tb.width << up;
      qc.y_clamp = tb.height << up;
      qc.mul = 1u << xbits;
      qc.xbits = xbits;
      qc.tier_shift = static_cast<uint32_t>(up);
      const int below_leaf = tb.level + up - d.k_max / 2;  // sub-cell levels finer than the leaf level
      qc.sub_mask = below_leaf > 0 ? (0xFu & ~((1u << std::min(below_leaf, 4)) - 1u)) : 0xFu;
    } else {
      qc.shift = static_cast<uint32_t>(tb_shift + 2);
      qc.x0 = tb.x0;
      qc.y0 = tb.y0;
      qc.x_clamp = tb.width;
      qc.y_clamp = tb.height;
      qc.mul = tb.pitch;
    }
  }
  dv.n_dict = static_cast<uint32_t>(an.dict.size());
  // K1's sparse refinement: items reach population 3 as (record, slot) only under the packed coding
  if (dv.qc.packed && !an.link_sub.empty()) {
    if ((rc = upload(ix->d_link_sub, an.link_sub.data(), an.link_sub.size(), &bytes)) != GJ_OK) return rc;
    if ((rc = upload(ix->d_tier_links, an.tier_links.data(), an.tier_links.size(), &bytes)) != GJ_OK) return rc;
    ix->info.link_records = static_cast<int32_t>(an.link_sub.size() / 16);
  }
  ix->bind();

  cudaDeviceProp prop{};
  GJ_CUDA(cudaGetDeviceProperties(&prop, device));
  ix->sm_count = prop.multiProcessorCount;
  ix->smem_optin = prop.sharedMemPerBlockOptin;

  gj_index_info& info = ix->info;
  info.node_count = d.node_count;
  info.lut_len = d.lut_len;
  info.n_polygons = d.n_polygons;
  info.n_ids = n_ids;
  info.device_bytes = bytes;
  info.k_max = d.k_max;
  info.approx_mode = d.approx_mode ? 1 : 0;
  info.device = device;
  info.dir_level = an.dir.level;
  info.dir_width = static_cast<int32_t>(an.dir.width);
  info.dir_height = static_cast<int32_t>(an.dir.height);
  info.dir_dict_len = static_cast<int32_t>(an.dict.size());
  info.dir16_level = an.dir16.level;
  info.dir16_width = static_cast<int32_t>(an.dir16.width);
  info.dir16_height = static_cast<int32_t>(an.dir16.height);
  info.dir2_level = an.dir2.table.empty() ? 0 : an.dir2.level;
  info.dir2_width = static_cast<int32_t>(an.dir2.width);
  info.dir2_height = static_cast<int32_t>(an.dir2.height);
  info.ids_dense = dense ? 1 : 0;
  info.k1_direct = ix->direct ? 1 : 0;
  *out = ix.release();
  return GJ_OK;
}

// Device-to-device replica of an index: every buffer is copied from the source
// GPU's HBM (over NVLink when the two are peers, staged by the driver otherwise;
// a plain device copy on the same GPU) and the kernel parameter block is
// re-pointed.  The host arrays the source was created from are not needed.
int replicate_index(const gj_index& src, int device, gj_index** out) {
  if (!out) return GJ_INVALID_ARGUMENT;
  *out = nullptr;
  if (device < 0) GJ_CUDA(cudaGetDevice(&device));
  GJ_CUDA(cudaSetDevice(device));
  if (device != src.device) {
    int can = 0;
    GJ_CUDA(cudaDeviceCanAccessPeer(&can, device, src.device));
    if (can) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(src.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      cudaGetLastError();
    }
  }
  std::unique_ptr<gj_index> ix(new gj_index);
  ix->device = device;
  ix->dev = src.dev;  // scalars; pointers are re-bound below
  ix->info = src.info;
  ix->info.device = device;
  ix->opt = src.opt;
  ix->ids = src.ids;
  ix->ids_late = src.ids_late;
  ix->direct = src.direct;
  ix->stage_records = src.stage_records;
  ix->max_refs = src.max_refs;
  ix->max_cand_refs = src.max_cand_refs;
  for (DeviceBuffer gj_index::*m : src.buffers()) {
    const DeviceBuffer& from = src.*m;
    if (!from.ptr) continue;
    DeviceBuffer& to = ix.get()->*m;
    GJ_CUDA(to.reserve(from.bytes));
    if (device == src.device) {
      GJ_CUDA(cudaMemcpy(to.ptr, from.ptr, from.bytes, cudaMemcpyDeviceToDevice));
    } else {
      GJ_CUDA(cudaMemcpyPeer(to.ptr, device, from.ptr, src.device, from.bytes));
    }
  }
  GJ_CUDA(cudaDeviceSynchronize());
  ix->bind();
  cudaDeviceProp prop{};
  GJ_CUDA(cudaGetDeviceProperties(&prop, device));
  ix->sm_count = prop.multiProcessorCount;
  ix->smem_optin = prop.sharedMemPerBlockOptin;
  *out = ix.release();
  return GJ_OK;
}

// ---------------------------------------------------------------------------
// GJX1 / ACT1 reader (join.cpp:316-381, act.cpp:600-652): little-endian,
// raw arena and lookup table — mapped and copied straight to the device.
// ---------------------------------------------------------------------------
namespace {

struct Cursor {
  const uint8_t* p;
  const uint8_t* end;
  bool ok = true;
  bool take(void* dst, size_t n) {
    if (!ok || static_cast<size_t>(end - p) < n) {
      ok = false;
      return false;
    }
    std::memcpy(dst, p, n);
    p += n;
    return true;
  }
  uint32_t u32() {
    uint32_t v = 0;
    take(&v, 4);
    return v;
  }
  uint64_t u64() {
    uint64_t v = 0;
    take(&v, 8);
    return v;
  }
  double f64() {
    double v = 0;
    take(&v, 8);
    return v;
  }
  const uint8_t* span(size_t n) {
    if (!ok || static_cast<size_t>(end - p) < n) {
      ok = false;
      return nullptr;
    }
    const uint8_t* s = p;
    p += n;
    return s;
  }
};

}  // namespace

int load_index_file(const char* path, int device, const gj_options* options, gj_index** out) {
  if (!path || !out) return GJ_INVALID_ARGUMENT;
  *out = nullptr;
  const int fd = ::open(path, O_RDONLY);
  if (fd < 0) {
    set_error(std::string("cannot open ") + path);
    return GJ_IO_ERROR;
  }
  struct stat st{};
  if (fstat(fd, &st) != 0 || st.st_size < 8) {
    ::close(fd);
    set_error("not a geojoin index file");
    return GJ_CORRUPT_INDEX;
  }
  const size_t size = static_cast<size_t>(st.st_size);
  void* map = mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
  ::close(fd);
  if (map == MAP_FAILED) {
    set_error("mmap failed");
    return GJ_IO_ERROR;
  }
  struct Unmap {
    void* m;
    size_t n;
    ~Unmap() { munmap(m, n); }
  } unmap{map, size};

  Cursor c{static_cast<const uint8_t*>(map), static_cast<const uint8_t*>(map) + size};
  char magic[4];
  if (!c.take(magic, 4) || std::memcmp(magic, "GJX1", 4) != 0) {
    set_error("not a geojoin index file");
    return GJ_CORRUPT_INDEX;
  }
  if (c.u32() != 1) {
    set_error("unsupported index version");
    return GJ_CORRUPT_INDEX;
  }
  gj_index_desc d{};
  d.approx_mode = c.u32() != 0;
  c.u32();  // precision_achieved
  c.f64();  // precision_m
  c.f64();  // achieved_precision_m
  c.u64();  // memory budget
  for (int i = 0; i < 4; ++i) c.u32();  // covering config
  if (!c.take(magic, 4) || std::memcmp(magic, "ACT1", 4) != 0) {
    set_error("not an ACT1 index snapshot");
    return GJ_CORRUPT_INDEX;
  }
  d.k_max = static_cast<int32_t>(c.u32());
  d.node_count = c.u64();
  d.lut_len = c.u64();
  if (!c.ok || d.node_count > (1ull << 32) || d.lut_len > 0x7fffffffull) {
    set_error("snapshot header sizes out of range");
    return GJ_CORRUPT_INDEX;
  }
  for (int f = 0; f < 6; ++f) {
    d.roots[f] = c.u64();
    d.prefixes[f] = c.u64();
    d.prefix_bits[f] = c.u32();
  }
  const uint8_t* arena = c.span(d.node_count * kNodeSlots * 8);
  const uint8_t* lut = c.span(d.lut_len * 4);
  if (!c.ok) {
    set_error("truncated index snapshot");
    return GJ_CORRUPT_INDEX;
  }
  // The header is 200 bytes, so the arena is 8-byte aligned inside the map.
  std::vector<uint64_t> arena_copy;
  if (reinterpret_cast<uintptr_t>(arena) % 8 != 0) {
    arena_copy.resize(d.node_count * kNodeSlots);
    std::memcpy(arena_copy.data(), arena, arena_copy.size() * 8);
    d.arena = arena_copy.data();
  } else {
    d.arena = reinterpret_cast<const uint64_t*>(arena);
  }
  std::vector<uint32_t> lut_copy;
  if (reinterpret_cast<uintptr_t>(lut) % 4 != 0) {
    lut_copy.resize(d.lut_len);
    std::memcpy(lut_copy.data(), lut, lut_copy.size() * 4);
    d.lut = lut_copy.data();
  } else {
    d.lut = reinterpret_cast<const uint32_t*>(lut);
  }
  const uint64_t n_poly = c.u64();
  if (!c.ok || n_poly > (1ull << 30)) {
    set_error("index polygon count out of range");
    return GJ_CORRUPT_INDEX;
  }
  std::vector<uint32_t> ids(n_poly);
  std::vector<uint64_t> off(n_poly + 1, 0);
  std::vector<double> latlng;
  for (uint64_t p = 0; p < n_poly; ++p) {
    ids[p] = c.u32();
    const uint64_t nv = c.u64();
    if (!c.ok || nv > (1ull << 24)) {
      set_error("polygon vertex count out of range");
      return GJ_CORRUPT_INDEX;
    }
    const uint8_t* v = c.span(nv * 16);
    if (!c.ok) {
      set_error("truncated index file");
      return GJ_CORRUPT_INDEX;
    }
    const size_t at = latlng.size();
    latlng.resize(at + 2 * nv);
    std::memcpy(latlng.data() + at, v, nv * 16);
    off[p + 1] = off[p] + nv;
  }
  d.n_polygons = n_poly;
  d.polygon_ids = ids.data();
  d.vtx_off = off.data();
  d.vtx_latlng = latlng.data();
  return create_index(d, device, options, out);
}

}  // namespace gj
