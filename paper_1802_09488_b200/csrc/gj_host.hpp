// Host-side state behind the C ABI handles.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/geojoin_b200.h"
#include "gj_device.cuh"

namespace gj {

void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
// Shared memory K1 needs besides its first tier (per-warp queues, one histogram row set for `n_ids`
// polygons when that fits), so the index builder can size the tier to stay below the 228 KB carve-out
// step (defined next to the kernel's launch plan, gj_api.cu).
size_t k1_smem_besides_tier(size_t n_ids, const gj_options& opt);
// Id tables beyond the 32-bit shared-memory histogram (64 KB) count in a 16-bit one that the CTA flushes every
// kHist16FlushTiles tiles — no counter can overflow in between (join_kernel) — when it fits and the options allow it.
bool k1_uses_hist16(size_t n_ids, const gj_options& opt);
bool k1_stages_records(uint64_t lut_len, const gj_options& opt);

#define GJ_CUDA(call)                                  \
  do {                                                 \
    cudaError_t e_ = (call);                           \
    if (e_ != cudaSuccess) return ::gj::cuda_fail(e_, #call); \
  } while (0)

struct DeviceBuffer {
  void* ptr = nullptr;
  size_t bytes = 0;
  ~DeviceBuffer() { release(); }
  DeviceBuffer() = default;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  // grow-only allocation
  cudaError_t reserve(size_t want) {
    if (want <= bytes) return cudaSuccess;
    release();
    cudaError_t e = cudaMalloc(&ptr, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(ptr); }
};

// Result of analysing the host arena once: validation + id table + directory.
struct HostDirectory {
  int level = 0;   // grid level the table resolves
  int chunks = 0;  // node steps folded in
  uint32_t x0 = 0, y0 = 0, width = 0, height = 0, pitch = 0;
  std::vector<uint32_t> table;
  std::vector<uint16_t> table16;  // the 16-bit first tier uses this instead
};

// Fork-join memcpy over a few worker threads: one thread moves ~10 GB/s between
// pageable and pinned memory (less when the pages are touched for the first
// time), the PCIe link 55 GB/s.
class CopyPool {
 public:
  explicit CopyPool(int threads) {
    for (int w = 0; w < threads; ++w) workers_.emplace_back([this, w] { run(w); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
      ++generation_;
    }
    cv_.notify_all();
    for (std::thread& t : workers_) t.join();
  }
  CopyPool(const CopyPool&) = delete;
  CopyPool& operator=(const CopyPool&) = delete;

  // blocking; the caller's thread takes the last slice
  void copy(void* dst, const void* src, size_t bytes) {
    const size_t parts = workers_.size() + 1;
    if (bytes < (1u << 20) || parts == 1) {
      std::memcpy(dst, src, bytes);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(m_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      slice_ = ((bytes + parts - 1) / parts + 4095) & ~size_t{4095};
      bytes_ = bytes;
      pending_ = static_cast<int>(workers_.size());
      ++generation_;
    }
    cv_.notify_all();
    copy_slice(parts - 1);
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void copy_slice(size_t part) {
    const size_t begin = part * slice_;
    if (begin < bytes_) std::memcpy(dst_ + begin, src_ + begin, std::min(slice_, bytes_ - begin));
  }
  void run(int w) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return generation_ != seen; });
        seen = generation_;
        if (stop_) return;
      }
      copy_slice(static_cast<size_t>(w));
      std::lock_guard<std::mutex> lk(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  uint64_t generation_ = 0;
  bool stop_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t slice_ = 0, bytes_ = 0;
  int pending_ = 0;
};

// Copies between PAGEABLE host memory and the device at close to PCIe rate:
// the pool moves the data through two pinned pieces while the copy engine works
// on the other one.  (cudaMemcpyAsync on pageable memory is staged by the
// driver on one thread, ~5-10 GB/s.)  Pinned or registered host memory
// (gj_host_alloc) needs none of this and is copied directly.
class HostStager {
 public:
  static constexpr size_t kPiece = 32u << 20;
  HostStager() : pool_(static_cast<int>(std::min(7u, std::max(1u, std::thread::hardware_concurrency() / 2)))) {}
  ~HostStager() {
    for (int b = 0; b < 2; ++b) {
      if (pinned_[b]) cudaFreeHost(pinned_[b]);
      if (ev_[b]) cudaEventDestroy(ev_[b]);
    }
  }
  static bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
  }
  // Enqueues on `st`; returns once the last piece has been handed to the copy engine.
  cudaError_t to_device(void* d_dst, const void* h_src, size_t bytes, cudaStream_t st) {
    if (bytes < (4u << 20) || is_pinned(h_src)) return cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, st);
    cudaError_t e = init();
    for (size_t off = 0, k = 0; off < bytes && e == cudaSuccess; off += kPiece, ++k) {
      const int b = static_cast<int>(k & 1);
      const size_t len = std::min(kPiece, bytes - off);
      e = cudaEventSynchronize(ev_[b]);  // the copy engine is done with this piece
      if (e != cudaSuccess) break;
      pool_.copy(pinned_[b], static_cast<const char*>(h_src) + off, len);
      e = cudaMemcpyAsync(static_cast<char*>(d_dst) + off, pinned_[b], len, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = cudaEventRecord(ev_[b], st);
    }
    return e;
  }
  // Pinned destination: enqueued on `st` and left in flight (synchronise `st` before reading).  Pageable
  // destination: staged like to_host, i.e. complete on return (the device keeps running what is already queued).
  cudaError_t to_host_async(void* h_dst, const void* d_src, size_t bytes, cudaStream_t st) {
    if (is_pinned(h_dst)) return cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, st);
    return to_host(h_dst, d_src, bytes, st);
  }
  cudaError_t drain() { return cudaSuccess; }  // staged copies complete inside to_host_async
  // Blocking: the data is in h_dst on return.
  cudaError_t to_host(void* h_dst, const void* d_src, size_t bytes, cudaStream_t st) {
    if (bytes < (4u << 20) || is_pinned(h_dst)) {
      const cudaError_t e = cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, st);
      return e == cudaSuccess ? cudaStreamSynchronize(st) : e;
    }
    cudaError_t e = init();
    if (e != cudaSuccess) return e;
    const size_t pieces = (bytes + kPiece - 1) / kPiece;
    auto issue = [&](size_t k) {
      const int b = static_cast<int>(k & 1);
      const size_t off = k * kPiece, len = std::min(kPiece, bytes - off);
      // the piece may still feed an earlier to_device() on another stream
      cudaError_t r = cudaEventSynchronize(ev_[b]);
      if (r == cudaSuccess) {
        r = cudaMemcpyAsync(pinned_[b], static_cast<const char*>(d_src) + off, len, cudaMemcpyDeviceToHost, st);
      }
      return r == cudaSuccess ? cudaEventRecord(ev_[b], st) : r;
    };
    e = issue(0);
    for (size_t k = 0; k < pieces && e == cudaSuccess; ++k) {
      if (k + 1 < pieces) e = issue(k + 1);  // the other piece: its last contents were copied out already
      if (e != cudaSuccess) break;
      const int b = static_cast<int>(k & 1);
      e = cudaEventSynchronize(ev_[b]);
      if (e != cudaSuccess) break;
      const size_t off = k * kPiece, len = std::min(kPiece, bytes - off);
      pool_.copy(static_cast<char*>(h_dst) + off, pinned_[b], len);
    }
    return e;
  }

 private:
  cudaError_t init() {
    for (int b = 0; b < 2; ++b) {
      if (!pinned_[b]) {
        cudaError_t e = cudaHostAlloc(&pinned_[b], kPiece, cudaHostAllocDefault);
        if (e != cudaSuccess) return e;
        e = cudaEventCreateWithFlags(&ev_[b], cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
      }
    }
    return cudaSuccess;
  }
  CopyPool pool_;
  void* pinned_[2] = {nullptr, nullptr};
  cudaEvent_t ev_[2] = {nullptr, nullptr};
};

}  // namespace gj

struct gj_index {
  int device = 0;
  gj::DevIndex dev{};
  gj_index_info info{};
  gj_options opt{};            // explicit knobs (gj_options_default unless the creator passed others)
  std::vector<uint32_t> ids;  // slot -> polygon id
  gj::DeviceBuffer d_arena, d_lut, d_ids, d_ring_off, d_ring_len, d_ring_xy, d_dir_table, d_dir_dict, d_dir2_table, d_dir16_table, d_dirk_table, d_node_pal,
      d_link_sub, d_tier_links, d_strip_meta, d_strip_ptr, d_strip_edges, d_strip_eidx;
  int sm_count = 0;
  size_t smem_optin = 0;
  bool stage_records = false;  // K1 stages the lookup-table records of a population-3 batch in shared memory (lookup-table-heavy indexes)
  bool ids_late = false;       // K1 writes first ids where a point is settled (join_kernel's kLate): the 16-bit tier resolves few cells
  bool direct = false;         // K1 runs its direct form (join_kernel's kDirect): the 16-bit tier resolves (almost) nothing
  uint64_t max_refs = 0;       // most references behind one reachable entry
  uint64_t max_cand_refs = 0;  // most candidate references behind one entry
  // Points the device pointers of `dev` at this index's buffers (after uploads, and after gj_index_replicate
  // copied the buffers of another index).
  void bind() {
    dev.arena = d_arena.as<uint64_t>();
    dev.lut = d_lut.as<uint32_t>();
    dev.ids = d_ids.as<uint32_t>();
    dev.ring_off = d_ring_off.as<uint64_t>();
    dev.ring_len = d_ring_len.as<uint32_t>();
    dev.ring_xy = d_ring_xy.as<double2>();
    dev.strip_meta = d_strip_meta.as<gj::StripMeta>();
    dev.strip_ptr = d_strip_ptr.as<uint32_t>();
    dev.strip_edges = d_strip_edges.as<gj::EdgeRecord>();
    dev.strip_eidx = d_strip_eidx.ptr ? d_strip_eidx.as<uint32_t>() : nullptr;
    dev.dir.table = d_dir_table.as<uint32_t>();
    dev.dir2.table = d_dir2_table.as<uint32_t>();
    dev.dir16.table = d_dir16_table.as<uint32_t>();
    dev.dirk.table = d_dirk_table.as<uint32_t>();
    dev.node_pal = d_node_pal.ptr ? d_node_pal.as<uint64_t>() : nullptr;
    dev.link_sub = d_link_sub.ptr ? d_link_sub.as<uint32_t>() : nullptr;
    dev.tier_links = d_tier_links.ptr ? d_tier_links.as<uint32_t>() : nullptr;
    dev.dict = d_dir_dict.as<uint64_t>();
  }
  // every device buffer, for replication
  std::vector<gj::DeviceBuffer gj_index::*> buffers() const {
    return {&gj_index::d_arena, &gj_index::d_lut, &gj_index::d_ids, &gj_index::d_ring_off, &gj_index::d_ring_len,
            &gj_index::d_ring_xy, &gj_index::d_dir_table, &gj_index::d_dir_dict, &gj_index::d_dir2_table,
            &gj_index::d_dir16_table, &gj_index::d_dirk_table, &gj_index::d_node_pal, &gj_index::d_link_sub, &gj_index::d_tier_links,
            &gj_index::d_strip_meta,
            &gj_index::d_strip_ptr, &gj_index::d_strip_edges, &gj_index::d_strip_eidx};
  }
};

struct gj_session {
  gj_index* ix = nullptr;
  cudaStream_t stream = nullptr;       // compute
  cudaStream_t copy_in = nullptr;      // H2D
  cudaStream_t copy_out = nullptr;     // D2H
  uint64_t launches = 0;
  // scratch
  gj::DeviceBuffer d_status, d_counts, d_stats;
  gj::DeviceBuffer d_counts_priv;  // [sm_count][n_ids] u32, kept zero between launches
  gj::DeviceBuffer d_points[3], d_first_id[3], d_entries;
  gj::DeviceBuffer d_ovf_point, d_ovf_id, d_ovf_ord;
  gj::DeviceBuffer d_task_point, d_task_slot, d_task_ord, d_task_pass;
  // CSR pairs pipeline
  gj::DeviceBuffer d_nrefs, d_task_base, d_pair_count, d_row_ptr, d_block_sums;
  cudaEvent_t ev_in[3]{}, ev_done[3]{}, ev_out[3]{}, ev_total[3]{};
  // CSR pipeline without per-chunk host round trips (run_pairs_async): the pair count so far, and — host output —
  // two chunk-local row / id buffers that drain D2H while the next chunk runs
  gj::DeviceBuffer d_pairs_base, d_chunk_rows[2], d_chunk_ids[2];
  gj::DevStatus* h_status = nullptr;   // pinned
  // materialised pairs of the last gj_join_pairs_host call, kept in HBM for gj_pairs_copy:
  // row_ptr[n + 1] (global offsets) and the polygon ids
  gj::DeviceBuffer d_all_row_ptr, d_all_ids;
  // CSV ingestion scratch
  gj::DeviceBuffer d_csv_text, d_csv_counts, d_csv_offsets, d_csv_lines, d_csv_status, d_csv_valid, d_csv_points,
      d_csv_out, d_csv_meta;
  uint64_t pairs_n = 0, pairs_total = 0;
  bool pairs_valid = false;
  std::unique_ptr<gj::HostStager> stager;  // created on first use with pageable host memory
};
