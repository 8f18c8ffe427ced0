/*
 * Plain-C use of libbanaserve.so (include/banaserve.h) with the CUDA runtime API -- no
 * Python, no PyTorch: the caller owns device memory and streams, the library enqueues.
 *
 *   1. two pools (a "prefill" instance's and a "decode" instance's) on GPU 0;
 *   2. H0/H1: allocate destination blocks (lowest free first), build the pair list;
 *   3. H2: migrate one layer's blocks of a request; check the bytes arrived unchanged;
 *   4. H4: split decode attention over the migrated shard with q = 0, where the closed
 *      form is known (every score is 0: lse = ln(len), o = mean of the V rows);
 *   5. H6: merge the shard's partial with an empty second shard (weight 0).
 *
 * Build (see tests/test_c_abi_demo.py):
 *   gcc -O2 -std=c11 examples/c_abi_demo.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2510_13223_b200 -lbanaserve -L/usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,$PWD/paper_2510_13223_b200 -o c_abi_demo
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "banaserve.h"

#define CK(x)                                                                   \
  do {                                                                          \
    bs_status _s = (x);                                                         \
    if (_s != BS_OK) {                                                          \
      fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #x, (int)_s, \
              bs_last_error());                                                 \
      return 1;                                                                 \
    }                                                                           \
  } while (0)
#define CU(x)                                                                               \
  do {                                                                                      \
    cudaError_t _e = (x);                                                                   \
    if (_e != cudaSuccess) {                                                                \
      fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(_e)); \
      return 1;                                                                             \
    }                                                                                       \
  } while (0)

static uint16_t f32_to_bf16(float f) { /* round to nearest even */
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFF + ((u >> 16) & 1);
  return (uint16_t)(u >> 16);
}
static float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int main(void) {
  if (bs_abi_version() != BS_ABI_VERSION) { /* header and library must describe the same ABI */
    fprintf(stderr, "c_abi_demo: library ABI %d, header ABI %d\n", bs_abi_version(), BS_ABI_VERSION);
    return 1;
  }
  const int L = 2, NB = 32, HKV = 2, D = 64, HQ = 4, LEN = 45; /* 3 blocks, ragged tail */
  bs_kv_pool_desc desc = {L, NB, 16, HKV, D, BS_DTYPE_BF16, 0};
  const size_t bytes = bs_kv_pool_bytes(&desc), chunk = bs_kv_chunk_bytes(&desc);
  void *prefill_mem, *decode_mem;
  CU(cudaSetDevice(0));
  CU(cudaMalloc(&prefill_mem, bytes));
  CU(cudaMalloc(&decode_mem, bytes));
  CU(cudaMemset(decode_mem, 0xA5, bytes)); /* sentinel */

  /* prefill pool content: a deterministic pattern, bf16 */
  uint16_t* host = (uint16_t*)malloc(bytes);
  uint32_t seed = 12345;
  for (size_t i = 0; i < bytes / 2; ++i) {
    seed = seed * 1664525u + 1013904223u;
    host[i] = f32_to_bf16(((float)(seed >> 8) / 16777216.0f) * 2.0f - 1.0f);
  }
  CU(cudaMemcpy(prefill_mem, host, bytes, cudaMemcpyHostToDevice));

  bs_kv_pool *prefill, *decode;
  CK(bs_kv_pool_create(&desc, prefill_mem, &prefill));
  CK(bs_kv_pool_create(&desc, decode_mem, &decode));

  /* the request's 3 blocks live at prefill ids {7, 2, 19}; the decode pool hands out
     its lowest free ids */
  int32_t src[3] = {7, 2, 19}, dst[3];
  CK(bs_kv_pool_alloc(decode, 3, dst));
  int32_t *d_src, *d_dst;
  CU(cudaMalloc((void**)&d_src, sizeof src));
  CU(cudaMalloc((void**)&d_dst, sizeof dst));
  CU(cudaMemcpy(d_src, src, sizeof src, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_dst, dst, sizeof dst, cudaMemcpyHostToDevice));
  for (int layer = 0; layer < L; ++layer) /* layer by layer (Fig. 6) */
    CK(bs_kv_migrate_layer(prefill, decode, layer, d_src, d_dst, 3, NULL));

  uint16_t* back = (uint16_t*)malloc(bytes);
  CU(cudaMemcpy(back, decode_mem, bytes, cudaMemcpyDeviceToHost));
  int mig_ok = 1;
  for (int layer = 0; layer < L; ++layer)
    for (int i = 0; i < 3; ++i)
      mig_ok &= memcmp((char*)back + (layer * NB + dst[i]) * chunk,
                       (char*)host + (layer * NB + src[i]) * chunk, chunk) == 0;

  /* attention over the migrated shard (layer 1), q = 0 */
  uint16_t q[HQ * D];
  memset(q, 0, sizeof q);
  int32_t bt[3] = {dst[0], dst[1], dst[2]};
  int32_t split[3] = {0, LEN, LEN}; /* shard 0 = tokens [0, 45), shard 1 empty */
  void *d_q, *d_bt, *d_split, *d_out;
  float *d_o, *d_m, *d_l, *d_lse, *d_o1, *d_m1, *d_l1;
  CU(cudaMalloc(&d_q, sizeof q));
  CU(cudaMalloc(&d_bt, sizeof bt));
  CU(cudaMalloc(&d_split, sizeof split));
  CU(cudaMalloc((void**)&d_o, HQ * D * 4));
  CU(cudaMalloc((void**)&d_m, HQ * 4));
  CU(cudaMalloc((void**)&d_l, HQ * 4));
  CU(cudaMalloc((void**)&d_o1, HQ * D * 4));
  CU(cudaMalloc((void**)&d_m1, HQ * 4));
  CU(cudaMalloc((void**)&d_l1, HQ * 4));
  CU(cudaMalloc(&d_out, HQ * D * 2));
  CU(cudaMalloc((void**)&d_lse, HQ * 4));
  CU(cudaMemcpy(d_q, q, sizeof q, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_bt, bt, sizeof bt, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_split, split, sizeof split, cudaMemcpyHostToDevice));
  size_t ws_bytes = 0;
  CK(bs_split_decode_attention_workspace_size(decode, 1, HQ, 3, &ws_bytes));
  void* ws = NULL;
  if (ws_bytes) {
    CU(cudaMalloc(&ws, ws_bytes));
    CU(cudaMemset(ws, 0, ws_bytes));
  }
  const float scale = 1.0f / sqrtf((float)D);
  CK(bs_split_decode_attention(decode, 1, d_q, 1, HQ, (const int32_t*)d_bt, 3,
                               (const int32_t*)d_split, 2, 0, scale, d_o, d_m, d_l, ws, ws_bytes,
                               NULL));
  CK(bs_split_decode_attention(decode, 1, d_q, 1, HQ, (const int32_t*)d_bt, 3,
                               (const int32_t*)d_split, 2, 1, scale, d_o1, d_m1, d_l1, ws, ws_bytes,
                               NULL));
  const float* op[2] = {d_o, d_o1};
  const float* mp[2] = {d_m, d_m1};
  const float* lp[2] = {d_l, d_l1};
  CK(bs_merge_partials(2, op, mp, lp, 1, HQ, D, d_out, d_lse, NULL));
  CU(cudaDeviceSynchronize());

  uint16_t out[HQ * D];
  float lse[HQ];
  CU(cudaMemcpy(out, d_out, sizeof out, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(lse, d_lse, sizeof lse, cudaMemcpyDeviceToHost));
  /* closed form: lse = ln(LEN); o[h] = mean over the 45 tokens of V[kv head h / G] */
  double max_lse_err = 0, max_o_err = 0;
  for (int h = 0; h < HQ; ++h) {
    const int g = h / (HQ / HKV);
    max_lse_err = fmax(max_lse_err, fabs(lse[h] - log((double)LEN)));
    for (int x = 0; x < D; ++x) {
      double mean = 0;
      for (int t = 0; t < LEN; ++t) {
        const size_t e = ((((size_t)1 * NB + src[t / 16]) * 2 + 1) * HKV + g) * 16 * D +
                         (size_t)(t % 16) * D + x;
        mean += bf16_to_f32(host[e]);
      }
      mean /= LEN;
      max_o_err = fmax(max_o_err, fabs(bf16_to_f32(out[h * D + x]) - mean));
    }
  }
  printf("c_abi_demo: abi=%d migrated_bytes_equal=%d max|lse-ln(len)|=%.2e max|o-mean(v)|=%.2e\n",
         bs_abi_version(), mig_ok, max_lse_err, max_o_err);
  CK(bs_kv_pool_destroy(prefill));
  CK(bs_kv_pool_destroy(decode));
  return (mig_ok && max_lse_err < 1e-4 && max_o_err < 2e-2) ? 0 : 2;
}
