// Host-side state behind the C ABI handles.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/geojoin_b200.h"
#include "gj_device.cuh"

namespace gj {

void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

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

}  // namespace gj

struct gj_index {
  int device = 0;
  gj::DevIndex dev{};
  gj_index_info info{};
  std::vector<uint32_t> ids;  // slot -> polygon id
  gj::DeviceBuffer d_arena, d_lut, d_ids, d_ring_off, d_ring_len, d_ring_xy, d_dir_table, d_dir_dict, d_dir2_table, d_dir16_table, d_node_pal,
      d_strip_meta, d_strip_ptr, d_strip_edges;
  int sm_count = 0;
  size_t smem_optin = 0;
  uint64_t max_refs = 0;       // most references behind one reachable entry
  uint64_t max_cand_refs = 0;  // most candidate references behind one entry
};

struct gj_session {
  gj_index* ix = nullptr;
  cudaStream_t stream = nullptr;       // compute
  cudaStream_t copy_in = nullptr;      // H2D
  cudaStream_t copy_out = nullptr;     // D2H
  uint64_t launches = 0;
  // scratch
  gj::DeviceBuffer d_status, d_counts, d_stats;
  gj::DeviceBuffer d_points[3], d_first_id[3], d_entries;
  gj::DeviceBuffer d_ovf_point, d_ovf_id, d_ovf_ord;
  gj::DeviceBuffer d_task_point, d_task_slot, d_task_ord, d_task_pass;
  // CSR pairs pipeline
  gj::DeviceBuffer d_nrefs, d_task_base, d_pair_count, d_row_ptr, d_block_sums, d_pair_ids;
  cudaEvent_t ev_in[3]{}, ev_done[3]{}, ev_out[3]{};
  gj::DevStatus* h_status = nullptr;   // pinned
  // materialised pairs of the last gj_join_pairs_host call, kept in HBM for gj_pairs_copy:
  // row_ptr[n + 1] (global offsets) and the polygon ids
  gj::DeviceBuffer d_all_row_ptr, d_all_ids;
  uint64_t pairs_n = 0, pairs_total = 0;
  bool pairs_valid = false;
  int latched_status = 0;
  uint64_t latched_bad = ~0ull;
};
