// Internal helpers shared by the library's translation units (never installed).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <set>
#include <string>

#include "banaserve.h"

struct bs_kv_pool {
  bs_kv_pool_desc desc;
  uint8_t* base = nullptr;  // device-visible address (host pools: the UVA mapping)
  bool host = false;        // pinned host memory (Global KV Cache Store tier)
  size_t chunk_bytes = 0;   // one (layer, block): K+V pages of all heads
  size_t page_bytes = 0;    // one (layer, block, K|V, head)
  size_t layer_bytes = 0;   // num_blocks * chunk_bytes
  std::mutex mu;            // guards the allocator and the tensor-map cache
  std::set<int32_t> free_ids;
  alignas(64) CUtensorMap tmap;  // pool as [rows][head_dim] bf16 for the tensor-core kernel
  int tmap_state = 0;            // 0 not encoded yet, 1 ok, -1 unavailable
};

namespace bs {

bs_status set_error(bs_status st, const char* fmt, ...);
bs_status check_launch(const char* what);
int sm_count(int device);
int current_device();

inline bs_status ok() { return BS_OK; }

// Launchers (defined in the .cu files).
bs_status launch_copy_chunks(const uint8_t* src_base, const int32_t* src_ids, uint8_t* dst_base,
                             const int32_t* dst_ids, int32_t n, size_t chunk_bytes,
                             size_t page_bytes, int method, cudaStream_t stream,
                             int max_ctas = 0, int32_t n_layers = 1, int64_t src_layer_stride = 0,
                             int64_t dst_layer_stride = 0);

#ifdef BS_DEBUG
// debug build: validate device index arrays before a launch (debug.cu)
bs_status debug_check_ids(const int32_t* ids, int32_t n, int32_t limit, cudaStream_t s,
                          const char* what);
bs_status debug_check_table(const int32_t* kv_split, int32_t n_shards, int32_t shard, int32_t batch,
                            const int32_t* bt, int32_t max_blocks, int32_t num_blocks, cudaStream_t s,
                            const char* what);
bs_status debug_check_append(const int32_t* pos, int32_t batch, const int32_t* bt, int32_t max_blocks,
                             int32_t num_blocks, cudaStream_t s, const char* what);
#define BS_DEBUG_CHECK(expr)              \
  do {                                    \
    const bs_status _st = (expr);         \
    if (_st != BS_OK) return _st;         \
  } while (0)
#else
#define BS_DEBUG_CHECK(expr) \
  do {                       \
  } while (0)
#endif

}  // namespace bs

#define BS_REQUIRE(cond, ...)                                          \
  do {                                                                 \
    if (!(cond)) return bs::set_error(BS_ERR_INVALID_ARG, __VA_ARGS__); \
  } while (0)
