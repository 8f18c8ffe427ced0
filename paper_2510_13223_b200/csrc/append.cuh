// H7 device helper shared by the append kernel (append.cu) and the fused hand-off + append
// launch (migrate.cu): the threads of one CTA copy request b's new K/V rows -- 2 * Hkv rows
// of 2*D bytes, 16-byte columns -- into slot pos % 16 of block bt[b][pos / 16] of one layer
// (pool chunk layout [2][Hkv][16][D] bf16).  pos < 0 skips the request.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bs {

__device__ __forceinline__ void append_token_rows(uint8_t* __restrict__ layer_base, int64_t chunk_bytes,
                                                  int32_t hkv, int32_t d, const uint4* __restrict__ k_new,
                                                  const uint4* __restrict__ v_new,
                                                  const int32_t* __restrict__ bt, int32_t max_blocks,
                                                  const int32_t* __restrict__ pos, int b, int tid,
                                                  int nthreads) {
  const int p = __ldg(pos + b);
  if (p < 0) return;
  const int32_t blk = __ldg(bt + (int64_t)b * max_blocks + (p >> 4));
  const int slot = p & 15;
  const int cols = d / 8;  // 16-byte columns per row
  const int per_kv = hkv * cols;
  uint8_t* chunk = layer_base + (int64_t)blk * chunk_bytes;
  for (int i = tid; i < 2 * per_kv; i += nthreads) {
    const int kv = i >= per_kv, r = i - kv * per_kv, g = r / cols, c = r - g * cols;
    const uint4 val = __ldg((kv ? v_new : k_new) + ((int64_t)b * hkv + g) * cols + c);
    reinterpret_cast<uint4*>(chunk + (((int64_t)kv * hkv + g) * 16 + slot) * d * 2)[c] = val;
  }
}

}  // namespace bs
