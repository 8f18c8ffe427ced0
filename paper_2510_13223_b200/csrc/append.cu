// H7 (adjacent to the path): write the decoded token's K/V into its
// shard's paged cache before attention.  The paper is silent on it; reading R-A9 (seq_len
// includes the token being decoded, whose K/V is already in the cache) makes it the step
// that precedes H4 in every decode step.
//
// One CTA per request; threads over (K|V, kv head, 16-byte column) of the token's rows:
// 2 * Hkv rows of 2*D bytes, each row landing at slot pos % 16 of block
// bt[b][pos / 16] (pool chunk layout [2][Hkv][16][D] bf16).  A bit copy: 16-byte loads of
// the new rows, 16-byte stores into the pool.  Bytes per request per layer: 2 * Hkv * D * 2
// read + the same written (16 KiB at Llama-2-7B) -- latency-bound, one launch per layer.
#include <cuda_runtime.h>

#include "append.cuh"
#include "internal.h"

namespace bs {
namespace {

__global__ void __launch_bounds__(256) append_token_kernel(uint8_t* __restrict__ layer_base,
                                                           int64_t chunk_bytes, int32_t hkv,
                                                           int32_t d, const uint4* __restrict__ k_new,
                                                           const uint4* __restrict__ v_new,
                                                           const int32_t* __restrict__ bt,
                                                           int32_t max_blocks,
                                                           const int32_t* __restrict__ pos) {
  append_token_rows(layer_base, chunk_bytes, hkv, d, k_new, v_new, bt, max_blocks, pos, blockIdx.x,
                    threadIdx.x, blockDim.x);
}

}  // namespace
}  // namespace bs

extern "C" {

bs_status bs_kv_append_token(bs_kv_pool* pool, int32_t layer, const void* k_new, const void* v_new,
                             int32_t batch, const int32_t* block_tables, int32_t max_blocks,
                             const int32_t* pos, void* stream) {
  BS_REQUIRE(pool, "bs_kv_append_token: NULL pool");
  BS_REQUIRE(layer >= 0 && layer < pool->desc.num_layers, "bs_kv_append_token: layer %d out of range",
             layer);
  BS_REQUIRE(batch >= 0, "bs_kv_append_token: batch < 0");
  if (batch == 0) return BS_OK;
  BS_REQUIRE(k_new && v_new && block_tables && pos, "bs_kv_append_token: NULL argument");
  BS_REQUIRE(max_blocks >= 1, "bs_kv_append_token: max_blocks < 1");
  BS_REQUIRE(((uintptr_t)k_new & 15) == 0 && ((uintptr_t)v_new & 15) == 0,
             "bs_kv_append_token: k_new / v_new must be 16-B aligned");
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  BS_DEBUG_CHECK(bs::debug_check_append(pos, batch, block_tables, max_blocks, pool->desc.num_blocks, s,
                                        "bs_kv_append_token positions / block table"));
  bs::append_token_kernel<<<batch, 256, 0, s>>>(
      pool->base + (size_t)layer * pool->layer_bytes, (int64_t)pool->chunk_bytes,
      pool->desc.num_kv_heads, pool->desc.head_dim, static_cast<const uint4*>(k_new),
      static_cast<const uint4*>(v_new), block_tables, max_blocks, pos);
  return bs::check_launch("append_token_kernel");
}

}  // extern "C"
