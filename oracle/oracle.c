/*
 * oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the BanaServe
 * (arXiv 2510.13223) attention-level KV migration + split decode attention path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2510_13223_b200/) never links, imports or calls anything in oracle/, and
 * this file shares no code, header, table or helper with it.
 *
 * Every function cites the PAPER.md passage it follows ("PAPER.md:<line>", section,
 * equation).  Where the paper is silent or garbled the DESIGN.md reading is named
 * (R-A1 ... R-A18 == SURVEY.md §8(c) A1..A18).  There is no blocking, no fusion and
 * no reordering beyond the written definition: plain loops in the paper's order.
 *
 * Pins (tests/test_oracle_pins.py, run with -m "not gpu"):
 *   or_kv_bytes_per_token_layer  -> eq. 15/16 printed values (4096 B, 128 KiB)   [pinned]
 *   or_t_f_layer_ms / or_t_kv_ms -> eq. 17 printed values (4.22 ms, 0.082 ms)      [pinned]
 *   or_attention_shard           -> numpy dense softmax + torch SDPA fp64, closed
 *                                   forms (q=0, n=1, needle, identical keys)       [pinned]
 *   or_merge_partials            -> scipy logsumexp; split invariance vs unsplit   [pinned]
 *   or_chained_two_shard         -> equals dense attention and the LSE merge       [pinned]
 *   or_migrate_layer             -> byte identity through block tables, sentinel
 *                                   preservation outside dst ids                   [pinned]
 *   or_migrate_heads_layer       -> page identity, untouched heads/blocks, head-
 *                                   split attention == full-pool heads; concat of
 *                                   the head groups == torch SDPA (NEXT F2)        [pinned]
 *   or_layer_payload_bytes       -> eq. 3 on hand-worked layer sizes (Llama-2-7B and
 *                                   Llama-3.1-8B layers, tests/golden/paper_eq3_4_hand.txt)
 *                                                                                  [pinned]
 *   or_t_layer_s                 -> eq. 4 on the same hand-worked cases + closed forms
 *                                   (T(0) = T_sync, affine in S, 1/B_net)           [pinned]
 *   or_pool_alloc / or_pool_free -> brute-force enumeration of the stated policy
 *                                   (R-A12 is a policy choice: "parity unpinned"
 *                                   for the choice itself, pinned for the policy)
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC oracle/oracle.c -o oracle/liboracle.so -lm
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Thread count of the OpenMP loops (timing reports only: 1 thread vs all cores). */
void or_set_threads(int32_t n) { omp_set_num_threads(n > 0 ? n : 1); }
int32_t or_get_threads(void) { return omp_get_max_threads(); }

/* ------------------------------------------------------------------------- */
/* Scalars                                                                    */
/* ------------------------------------------------------------------------- */

/* bf16 -> fp64, exact: the bf16 bit pattern is the upper half of an fp32
 * (R-A13: KV is BF16, eq. 15 "BF16 precision (2 bytes per element)"). */
static double bf16_to_f64(uint16_t bits) {
  uint32_t u = ((uint32_t)bits) << 16;
  float f;
  memcpy(&f, &u, sizeof f);
  return (double)f;
}

double or_bf16_to_f64(uint16_t bits) { return bf16_to_f64(bits); }

/* ------------------------------------------------------------------------- */
/* Sizes and the per-layer transfer model (§4.2, eqs. 12-17) */
/* ------------------------------------------------------------------------- */

/* eq. 15: S_kv = h_kv * d_head * 2 (K and V) * elem_bytes, per token per layer. */
int64_t or_kv_bytes_per_token_layer(int32_t h_kv, int32_t d_head, int32_t elem_bytes) {
  return (int64_t)h_kv * d_head * 2 * elem_bytes;
}

/* eq. 16: total per token = N layers * S_kv. */
int64_t or_kv_bytes_per_token(int32_t n_layers, int32_t h_kv, int32_t d_head, int32_t elem_bytes) {
  return (int64_t)n_layers * or_kv_bytes_per_token_layer(h_kv, d_head, elem_bytes);
}

/* eq. 12: T_F,layer = T_F * r / N  (printed formula, R-A16). */
double or_t_f_layer_ms(double t_f_ms, double r, int32_t n_layers) {
  return t_f_ms * r / (double)n_layers;
}

/* eq. 13: T_KV = S_kv * L * r / B, with B in Gbit/s = 1e9 bit/s
 * (R-A17: 4 KB = 4096 B, 200 Gbps = 25e9 B/s reproduces the printed 0.082 ms). */
double or_t_kv_ms(double s_kv_bytes, double l_tokens, double r, double b_gbps) {
  double bytes_per_s = b_gbps * 1e9 / 8.0;
  return s_kv_bytes * l_tokens * r / bytes_per_s * 1e3;
}

/* eq. 3: layer-level migration payload S_total = S_w + S_kv. */
double or_layer_payload_bytes(double s_w, double s_kv) { return s_w + s_kv; }

/* eq. 4: T_layer ~= S_total / B_net + T_sync (seconds, bytes/s). */
double or_t_layer_s(double s_total, double b_net, double t_sync) { return s_total / b_net + t_sync; }

/* ------------------------------------------------------------------------- */
/* Paged pool geometry (R-A: layout D4; vLLM PagedAttention blocks PAPER.md:126) */
/*   pool[layer][block][kv(0=K,1=V)][kv_head][slot][dim], bf16                   */
/* ------------------------------------------------------------------------- */

int64_t or_chunk_elems(int32_t h_kv, int32_t bs, int32_t d) {
  return (int64_t)2 * h_kv * bs * d; /* one (layer, block): K and V, all heads, all slots */
}

int64_t or_pool_bytes(int32_t n_layers, int32_t n_blocks, int32_t h_kv, int32_t bs, int32_t d) {
  return (int64_t)n_layers * n_blocks * or_chunk_elems(h_kv, bs, d) * 2;
}

static int64_t elem_index(int32_t n_blocks, int32_t h_kv, int32_t bs, int32_t d,
                          int32_t layer, int32_t block, int32_t kv, int32_t g, int32_t slot,
                          int32_t dim) {
  int64_t i = layer;
  i = i * n_blocks + block;
  i = i * 2 + kv;
  i = i * h_kv + g;
  i = i * bs + slot;
  i = i * d + dim;
  return i;
}

/* ------------------------------------------------------------------------- */
/* Block allocator (H0).  Eq. 28's T_mem_realloc names the  */
/* cost, the paper is silent on the policy; reading R-A12: lowest-free-id first, */
/* all-or-nothing.  used[i] != 0 means block i is taken.                        */
/* Returns 0 ok, 1 invalid argument, 2 out of blocks.                          */
/* ------------------------------------------------------------------------- */

int32_t or_pool_alloc(uint8_t* used, int32_t n_blocks, int32_t n, int32_t* out_ids) {
  if (n < 0 || (n > 0 && out_ids == NULL)) return 1;
  int32_t free_count = 0;
  for (int32_t i = 0; i < n_blocks; ++i)
    if (!used[i]) free_count++;
  if (free_count < n) return 2;
  int32_t k = 0;
  for (int32_t i = 0; i < n_blocks && k < n; ++i) {
    if (!used[i]) {
      used[i] = 1;
      out_ids[k++] = i;
    }
  }
  return 0;
}

/* Free: every id must be in range, currently used and listed once; otherwise
 * nothing changes and 1 is returned. */
int32_t or_pool_free(uint8_t* used, int32_t n_blocks, int32_t n, const int32_t* ids) {
  if (n < 0 || (n > 0 && ids == NULL)) return 1;
  for (int32_t i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= n_blocks) return 1;
    if (!used[ids[i]]) return 1;
    for (int32_t j = 0; j < i; ++j)
      if (ids[j] == ids[i]) return 1;
  }
  for (int32_t i = 0; i < n; ++i) used[ids[i]] = 0;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* H2: one layer of block migration (attention-level migration,  */
/* :239-244 eq. 11; "without semantic change", eq. 5).        */
/* dst.chunk(layer, dst_ids[i]) := src.chunk(layer, src_ids[i]), as bytes.     */
/* ------------------------------------------------------------------------- */

void or_migrate_layer(const uint16_t* src_pool, int32_t src_blocks, uint16_t* dst_pool,
                      int32_t dst_blocks, int32_t h_kv, int32_t bs, int32_t d, int32_t layer,
                      const int32_t* src_ids, const int32_t* dst_ids, int32_t n) {
  int64_t chunk = or_chunk_elems(h_kv, bs, d);
  for (int32_t i = 0; i < n; ++i) {
    const uint16_t* s = src_pool + ((int64_t)layer * src_blocks + src_ids[i]) * chunk;
    uint16_t* t = dst_pool + ((int64_t)layer * dst_blocks + dst_ids[i]) * chunk;
    memcpy(t, s, (size_t)chunk * sizeof(uint16_t));
  }
}

/* ------------------------------------------------------------------------- */
/* H7 (adjacent to the path): append the decoded token's K/V.    */
/* The paper is silent; reading R-A9: seq_len includes the token being decoded, */
/* whose K/V is already in the cache when attention runs -- this writes it.     */
/* For every request b with pos[b] >= 0: for every kv head g and dim x,         */
/*   pool[layer][bt[b][pos/bs]][K][g][pos%bs][x] = k_new[b][g][x]               */
/*   pool[layer][bt[b][pos/bs]][V][g][pos%bs][x] = v_new[b][g][x]               */
/* (bit copy, uint16).  pos[b] < 0: request skipped.                            */
/* ------------------------------------------------------------------------- */
void or_append_token(uint16_t* pool, int32_t n_blocks, int32_t h_kv, int32_t bs, int32_t d,
                     int32_t layer, const uint16_t* k_new, const uint16_t* v_new, int32_t batch,
                     const int32_t* block_tables, int32_t max_blocks, const int32_t* pos) {
  for (int32_t b = 0; b < batch; ++b) {
    if (pos[b] < 0) continue;
    const int32_t block = block_tables[(int64_t)b * max_blocks + pos[b] / bs];
    const int32_t slot = pos[b] % bs;
    for (int32_t g = 0; g < h_kv; ++g)
      for (int32_t x = 0; x < d; ++x) {
        const int64_t src = ((int64_t)b * h_kv + g) * d + x;
        pool[elem_index(n_blocks, h_kv, bs, d, layer, block, 0, g, slot, x)] = k_new[src];
        pool[elem_index(n_blocks, h_kv, bs, d, layer, block, 1, g, slot, x)] = v_new[src];
      }
  }
}

/* ------------------------------------------------------------------------- */
/* NEXT F2: head-granular attention-level migration -- the paper's literal text: */
/* "partition the KV Cache along the attention head dimension and selectively  */
/* migrate only the KV states of certain heads" (Alg. 1 */
/* MigrateKVHeads, :411).  For every pair i, both K and V pages of kv-heads     */
/* [src_head_lo, src_head_lo + n_heads) of block src_ids[i] go to heads         */
/* [dst_head_lo, ...) of block dst_ids[i]; pools may have different Hkv (the    */
/* cold pool keeps only the migrated heads).                                    */
/* ------------------------------------------------------------------------- */

void or_migrate_heads_layer(const uint16_t* src_pool, int32_t src_blocks, int32_t src_hkv,
                            uint16_t* dst_pool, int32_t dst_blocks, int32_t dst_hkv, int32_t bs,
                            int32_t d, int32_t layer, const int32_t* src_ids,
                            const int32_t* dst_ids, int32_t n, int32_t src_head_lo,
                            int32_t dst_head_lo, int32_t n_heads) {
  const int64_t page = (int64_t)bs * d;
  for (int32_t i = 0; i < n; ++i)
    for (int32_t kv = 0; kv < 2; ++kv)
      for (int32_t h = 0; h < n_heads; ++h) {
        const uint16_t* s =
            src_pool + elem_index(src_blocks, src_hkv, bs, d, layer, src_ids[i], kv, src_head_lo + h, 0, 0);
        uint16_t* t =
            dst_pool + elem_index(dst_blocks, dst_hkv, bs, d, layer, dst_ids[i], kv, dst_head_lo + h, 0, 0);
        memcpy(t, s, (size_t)page * sizeof(uint16_t));
      }
}

/* ------------------------------------------------------------------------- */
/* H4: decode attention over shard j of every request (PAPER.md:216-231,       */
/* eqs. 6-9, corrected per R-A1..R-A11):                                        */
/*   shard j of request b holds global tokens [kv_split[b][j], kv_split[b][j+1]) */
/*   in shard-local order u = 0.., stored at block bt[b][u/bs], slot u%bs.      */
/*   q-head h reads kv-head g = floor(h / G), G = Hq/Hkv (R-A8).                */
/*   s_u = scale * sum_d q[h][d] * k[u][g][d]          (eq. 6 + R-A2 scale)     */
/*   m = max_u s_u; a_u = exp(s_u - m)                  (eq. 7 + R-A3 max shift) */
/*   l = sum_u a_u                                      (eq. 8, local part)      */
/*   o = sum_u a_u v[u][g] / l                          (eq. 9, local denom.)    */
/* Empty shard: m = -inf, l = 0, o = 0 (R-A7).                                   */
/* Outputs are fp64: o[b][h][d], m[b][h], l[b][h].                               */
/* ------------------------------------------------------------------------- */

void or_attention_shard(const uint16_t* pool, int32_t n_blocks, int32_t h_kv, int32_t bs,
                        int32_t d, int32_t layer, const uint16_t* q, int32_t batch, int32_t hq,
                        const int32_t* block_tables, int32_t max_blocks, const int32_t* kv_split,
                        int32_t n_shards, int32_t shard_id, float scale, double* o, double* m,
                        double* l) {
  const int32_t G = hq / h_kv;
  const double sc = (double)scale;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int32_t b = 0; b < batch; ++b) {
    for (int32_t h = 0; h < hq; ++h) {
      const int32_t g = h / G;
      const int32_t len = kv_split[b * (n_shards + 1) + shard_id + 1] -
                          kv_split[b * (n_shards + 1) + shard_id];
      double* ob = o + ((int64_t)b * hq + h) * d;
      const uint16_t* qb = q + ((int64_t)b * hq + h) * d;
      for (int32_t x = 0; x < d; ++x) ob[x] = 0.0;
      if (len <= 0) {
        m[(int64_t)b * hq + h] = -INFINITY;
        l[(int64_t)b * hq + h] = 0.0;
        continue;
      }
      double* s = (double*)malloc(sizeof(double) * (size_t)len);
      /* eq. 6: scores */
      for (int32_t u = 0; u < len; ++u) {
        const int32_t blk = block_tables[(int64_t)b * max_blocks + u / bs];
        const int32_t slot = u % bs;
        double acc = 0.0;
        for (int32_t x = 0; x < d; ++x) {
          double kx = bf16_to_f64(pool[elem_index(n_blocks, h_kv, bs, d, layer, blk, 0, g, slot, x)]);
          acc += bf16_to_f64(qb[x]) * kx;
        }
        s[u] = sc * acc;
      }
      /* eq. 7 with the max shift */
      double mx = -INFINITY;
      for (int32_t u = 0; u < len; ++u)
        if (s[u] > mx) mx = s[u];
      /* eq. 8 (local denominator) and eq. 9 numerator */
      double den = 0.0;
      for (int32_t u = 0; u < len; ++u) {
        const int32_t blk = block_tables[(int64_t)b * max_blocks + u / bs];
        const int32_t slot = u % bs;
        double a = exp(s[u] - mx);
        den += a;
        for (int32_t x = 0; x < d; ++x)
          ob[x] += a * bf16_to_f64(pool[elem_index(n_blocks, h_kv, bs, d, layer, blk, 1, g, slot, x)]);
      }
      for (int32_t x = 0; x < d; ++x) ob[x] /= den;
      m[(int64_t)b * hq + h] = mx;
      l[(int64_t)b * hq + h] = den;
      free(s);
    }
  }
}

/* ------------------------------------------------------------------------- */
/* H6: exact log-sum-exp merge of n shard partials (eq. 10, */
/* with R-A4: every O^(j) is re-normalised by the global denominator).        */
/*   lse_j = m_j + ln l_j   (-inf when l_j = 0)                               */
/*   M = max_j lse_j; lse = M + ln sum_j exp(lse_j - M)                        */
/*   O = sum_j exp(lse_j - lse) * O~_j       (fixed order j = 0..n-1, R-A14)  */
/* All shards empty: O = 0, lse = -inf (R-A7).                                 */
/* Inputs are n contiguous arrays: o_parts[j][b][h][d], m_parts[j][b][h] ...  */
/* ------------------------------------------------------------------------- */

void or_merge_partials(int32_t n, const double* o_parts, const double* m_parts,
                       const double* l_parts, int32_t batch, int32_t hq, int32_t d, double* out,
                       double* lse_out) {
  const int64_t rows = (int64_t)batch * hq;
  for (int64_t r = 0; r < rows; ++r) {
    double M = -INFINITY;
    for (int32_t j = 0; j < n; ++j) {
      double lj = l_parts[j * rows + r];
      double lse_j = lj > 0.0 ? m_parts[j * rows + r] + log(lj) : -INFINITY;
      if (lse_j > M) M = lse_j;
    }
    double* orow = out + r * d;
    for (int32_t x = 0; x < d; ++x) orow[x] = 0.0;
    if (M == -INFINITY) {
      lse_out[r] = -INFINITY;
      continue;
    }
    double S = 0.0;
    for (int32_t j = 0; j < n; ++j) {
      double lj = l_parts[j * rows + r];
      if (lj > 0.0) S += exp(m_parts[j * rows + r] + log(lj) - M);
    }
    double lse = M + log(S);
    lse_out[r] = lse;
    for (int32_t j = 0; j < n; ++j) {
      double lj = l_parts[j * rows + r];
      if (!(lj > 0.0)) continue;
      double w = exp(m_parts[j * rows + r] + log(lj) - lse);
      const double* oj = o_parts + ((int64_t)j * rows + r) * d;
      for (int32_t x = 0; x < d; ++x) orow[x] += w * oj[x];
    }
  }
}

/* ------------------------------------------------------------------------- */
/* The paper's own two-device protocol, eqs. 6-10 (Fig. 4), */
/* written out literally with the R-A3 max shift and the R-A4 correction:     */
/*   hot  (j=1): S1, m1 = max S1, A1 = exp(S1 - m1), l1 = sum A1   -> E^(1)  */
/*   cold (j=2): m = max(m1, max S2); l2 = l1 e^{m1-m} + sum e^{S2-m}  (eq. 8)*/
/*               O2 = sum e^{S2-m} V2 / l2                          (eq. 9) */
/*               -> E^(2) = (m, l2) sent back ("or E^(2)")      */
/*   hot:        O1 = sum A1 e^{m1-m} V1 / l2   (global denominator, R-A4)   */
/*   O = O1 + O2                                                    (eq. 10) */
/* Shard 0 lives in pool0/bt0 (hot), shard 1 in pool1/bt1 (cold); kv_split is */
/* [B][3].  Output o[b][h][d], lse[b][h] = m + ln l2.                         */
/* ------------------------------------------------------------------------- */

static double dot_k(const uint16_t* pool, int32_t n_blocks, int32_t h_kv, int32_t bs, int32_t d,
                    int32_t layer, const int32_t* bt_row, int32_t u, int32_t g,
                    const uint16_t* qrow) {
  const int32_t blk = bt_row[u / bs], slot = u % bs;
  double acc = 0.0;
  for (int32_t x = 0; x < d; ++x)
    acc += bf16_to_f64(qrow[x]) *
           bf16_to_f64(pool[elem_index(n_blocks, h_kv, bs, d, layer, blk, 0, g, slot, x)]);
  return acc;
}

static double v_at(const uint16_t* pool, int32_t n_blocks, int32_t h_kv, int32_t bs, int32_t d,
                   int32_t layer, const int32_t* bt_row, int32_t u, int32_t g, int32_t x) {
  const int32_t blk = bt_row[u / bs], slot = u % bs;
  return bf16_to_f64(pool[elem_index(n_blocks, h_kv, bs, d, layer, blk, 1, g, slot, x)]);
}

void or_chained_two_shard(const uint16_t* pool0, int32_t n_blocks0, const int32_t* bt0,
                          int32_t max_blocks0, const uint16_t* pool1, int32_t n_blocks1,
                          const int32_t* bt1, int32_t max_blocks1, int32_t h_kv, int32_t bs,
                          int32_t d, int32_t layer, const uint16_t* q, int32_t batch, int32_t hq,
                          const int32_t* kv_split, float scale, double* o, double* lse) {
  const int32_t G = hq / h_kv;
  const double sc = (double)scale;
  for (int32_t b = 0; b < batch; ++b) {
    const int32_t len1 = kv_split[b * 3 + 1] - kv_split[b * 3 + 0];
    const int32_t len2 = kv_split[b * 3 + 2] - kv_split[b * 3 + 1];
    const int32_t* r0 = bt0 + (int64_t)b * max_blocks0;
    const int32_t* r1 = bt1 + (int64_t)b * max_blocks1;
    for (int32_t h = 0; h < hq; ++h) {
      const int32_t g = h / G;
      const uint16_t* qrow = q + ((int64_t)b * hq + h) * d;
      double* orow = o + ((int64_t)b * hq + h) * d;
      /* hot: eq. 6-8 (j = 1) */
      double m1 = -INFINITY, l1 = 0.0;
      for (int32_t u = 0; u < len1; ++u) {
        double s = sc * dot_k(pool0, n_blocks0, h_kv, bs, d, layer, r0, u, g, qrow);
        if (s > m1) m1 = s;
      }
      for (int32_t u = 0; u < len1; ++u)
        l1 += exp(sc * dot_k(pool0, n_blocks0, h_kv, bs, d, layer, r0, u, g, qrow) - m1);
      /* cold: eq. 8 (j = 2) with the exchanged E^(1) = (m1, l1) */
      double m = m1;
      for (int32_t u = 0; u < len2; ++u) {
        double s = sc * dot_k(pool1, n_blocks1, h_kv, bs, d, layer, r1, u, g, qrow);
        if (s > m) m = s;
      }
      double l2 = (len1 > 0) ? l1 * exp(m1 - m) : 0.0;
      for (int32_t u = 0; u < len2; ++u)
        l2 += exp(sc * dot_k(pool1, n_blocks1, h_kv, bs, d, layer, r1, u, g, qrow) - m);
      for (int32_t x = 0; x < d; ++x) orow[x] = 0.0;
      if (len1 + len2 <= 0) {
        lse[(int64_t)b * hq + h] = -INFINITY;
        continue;
      }
      /* cold: eq. 9 (j = 2) */
      for (int32_t u = 0; u < len2; ++u) {
        double a = exp(sc * dot_k(pool1, n_blocks1, h_kv, bs, d, layer, r1, u, g, qrow) - m);
        for (int32_t x = 0; x < d; ++x)
          orow[x] += a * v_at(pool1, n_blocks1, h_kv, bs, d, layer, r1, u, g, x) / l2;
      }
      /* hot, after E^(2) = (m, l2) comes back: eq. 9 (j = 1) with the global denominator */
      for (int32_t u = 0; u < len1; ++u) {
        double a = exp(sc * dot_k(pool0, n_blocks0, h_kv, bs, d, layer, r0, u, g, qrow) - m1) *
                   exp(m1 - m);
        for (int32_t x = 0; x < d; ++x)
          orow[x] += a * v_at(pool0, n_blocks0, h_kv, bs, d, layer, r0, u, g, x) / l2;
      }
      lse[(int64_t)b * hq + h] = m + log(l2);
    }
  }
}
