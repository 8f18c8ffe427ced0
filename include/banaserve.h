/*
 * banaserve.h -- C-ABI of the B200-native (sm_100a) hot path of BanaServe
 * (arXiv 2510.13223): attention-level KV-cache migration + split decode attention
 * + exact log-sum-exp merge.  Citations are to /root/reference/PAPER.md lines
 * ("PAPER.md:<line>", section, equation); readings R-Ax are listed in DESIGN.md.
 *
 * Conventions (apply to every entry point):
 *  - All functions are extern "C", never throw, and return bs_status.  On a non-OK
 *    status nothing has been enqueued and bs_last_error() (thread-local) describes it.
 *  - Device work is enqueued asynchronously on the caller's stream (`stream` is a
 *    cudaStream_t passed as void*; NULL = legacy default stream).  No call synchronises
 *    the device, allocates device memory, or copies host<->device on the hot path.
 *  - The caller owns every device buffer and stream (PyTorch provides them).  A pool
 *    handle owns only host metadata (geometry + the block allocator); it never frees
 *    the device memory it describes.
 *  - Host-visible arguments are validated (NULLs, ranges, alignment, supported shapes).
 *    Device arrays (block tables, ids, splits) are NOT validated: out-of-range ids are
 *    undefined behaviour, as for any CUDA kernel argument -- except in the debug build
 *    (libbanaserve_debug.so, compiled with -DBS_DEBUG=1, loaded by the Python binding
 *    when BS_DEBUG=1): there a validation kernel checks them on the device first, the
 *    call synchronises its stream and, on a violation, returns BS_ERR_INVALID_ARG
 *    without launching and ORs a code into bs_debug_error_code (1 block-table id out of
 *    range, 2 kv_split inconsistent with the table width, 4 migration id out of range,
 *    8 append position past the table).
 *  - Supported shapes: bf16 KV, block_size 16, head_dim 64 or 128, query group
 *    G = num_q_heads / num_kv_heads in {1, 2, 4, 8}.  Others -> BS_ERR_UNSUPPORTED.
 */
#ifndef BANASERVE_H_
#define BANASERVE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BS_ABI_VERSION 2

typedef enum {
  BS_OK = 0,
  BS_ERR_INVALID_ARG = 1,
  BS_ERR_OUT_OF_BLOCKS = 2,
  BS_ERR_UNSUPPORTED = 3,
  BS_ERR_CUDA = 4,
  BS_ERR_NCCL = 5
} bs_status;

enum { BS_DTYPE_BF16 = 0 };
/* bs_kv_pool_desc.device value for a host-tier pool (page-locked, UVA-mapped host
 * memory: the Global KV Cache Store's CPU tier, Fig. 5). */
#define BS_DEVICE_HOST (-1)

/* Thread-local text for the most recent non-OK status on this thread. */
const char* bs_last_error(void);
/* BS_ABI_VERSION of the loaded library. */
int32_t bs_abi_version(void);
/* 1 in the debug build (device-side validation of index arrays), 0 otherwise. */
int32_t bs_debug_build(void);
/* Codes of the debug checks that failed so far (OR of 1/2/4, see above); reset != 0
 * clears them.  Always 0 in a release build. */
int32_t bs_debug_error_code(int32_t reset);

/* Diagnostics: what the calling thread's most recent attention launch (any
 * bs_split_decode_attention* call that launched) ran -- grid.x CTA ranges (uniform plan:
 * ranges per (request, kv-head) over the launch's shards; ragged plan: work items), how the
 * ranges were merged (0 one range, nothing to merge; 1 last-arriving CTA through the
 * workspace; 2 thread-block cluster through distributed shared memory), whether it was a
 * programmatic dependent launch, the
 * tensor-core (1) or CUDA-core (0) kernel, and its K/V stages per warp (6: the
 * one-CTA-per-SM variant).  All 0 before the first launch. */
bs_status bs_attention_last_launch(int32_t* ranges, int32_t* merge, int32_t* pdl,
                                   int32_t* tensor_cores, int32_t* stages);

/* ------------------------------------------------------------------------------ */
/* H0: paged KV pool + block allocator.                                             */
/* vLLM-style paged KV ("PagedAttention ... block-level KV Cache"),   */
/* memory reallocation cost T_mem_realloc of eq. 28.              */
/*                                                                                  */
/* Device layout (reading D4), bf16, row-major:                                     */
/*   pool[layer][block][kv: 0=K,1=V][kv_head][slot: 0..15][dim: 0..head_dim-1]      */
/* so one (layer, block) "chunk" = 2*Hkv*16*head_dim*2 bytes is contiguous, and one */
/* (layer, block, K|V, kv_head) "page" = 16*head_dim*2 bytes (4 KiB at d=128) too.  */
/* Block ids are shared by all layers.                                              */
/* ------------------------------------------------------------------------------ */
typedef struct {
  int32_t num_layers;    /* L >= 1                                   */
  int32_t num_blocks;    /* physical blocks per layer, >= 1           */
  int32_t block_size;    /* tokens per block; must be 16              */
  int32_t num_kv_heads;  /* Hkv >= 1                                  */
  int32_t head_dim;      /* 64 or 128                                 */
  int32_t dtype;         /* BS_DTYPE_BF16                             */
  int32_t device;        /* CUDA ordinal that owns the memory, or     */
                         /* BS_DEVICE_HOST for a host-tier pool       */
} bs_kv_pool_desc;

typedef struct bs_kv_pool bs_kv_pool; /* opaque host handle */

/* Bytes of device memory a pool with this geometry needs (L*num_blocks*chunk). 0 on bad desc. */
size_t bs_kv_pool_bytes(const bs_kv_pool_desc* desc);
/* Bytes of one (layer, block) chunk: 2*Hkv*block_size*head_dim*2. 0 on bad desc. */
size_t bs_kv_chunk_bytes(const bs_kv_pool_desc* desc);

/* Describe caller-owned device memory `base` (>= bs_kv_pool_bytes, 256-B aligned) as a
 * pool.  All blocks start free.  `base` may be a peer-mapped pointer to another GPU's
 * pool (a "remote view"): migrate calls then write over NVLink (P2P push).  With
 * device = BS_DEVICE_HOST, `base` is page-locked host memory (cudaHostAlloc / torch
 * pin_memory): migrate / gather / scatter to or from it are the store's fetch (HtoD)
 * and store (DtoH) legs, done by a few CTAs over PCIe; attention never reads it. */
bs_status bs_kv_pool_create(const bs_kv_pool_desc* desc, void* base, bs_kv_pool** out);
/* Free the host handle (never the device memory). NULL is a no-op. */
bs_status bs_kv_pool_destroy(bs_kv_pool* pool);
/* Allocate n block ids into out_ids (host array): lowest free ids first, ascending;
 * all-or-nothing -> BS_ERR_OUT_OF_BLOCKS with no state change (reading R-A12). */
bs_status bs_kv_pool_alloc(bs_kv_pool* pool, int32_t n, int32_t* out_ids);
/* Return n ids (host array).  Any id out of range, not allocated, or repeated ->
 * BS_ERR_INVALID_ARG with no state change. */
bs_status bs_kv_pool_free(bs_kv_pool* pool, int32_t n, const int32_t* ids);
/* Number of free blocks (or -1 for NULL). */
int32_t bs_kv_pool_num_free(const bs_kv_pool* pool);

/* ------------------------------------------------------------------------------ */
/* H2: one layer of block migration -- gather from the source pool, send, scatter   */
/* into the destination pool (attention-level migration PAPER.md:207-214, :239-244, */
/* eq. 11; "without semantic change", eq. 5).                      */
/*   for i < n: dst.chunk(layer, dst_ids[i]) <- src.chunk(layer, src_ids[i])       */
/* Whole chunks (K and V, all heads, all 16 slots, pad slots included), bit-exact.  */
/* src_ids / dst_ids: DEVICE int32 arrays [n] readable on the current device; dst   */
/* ids must be distinct (caller contract).  src and dst must have equal             */
/* num_kv_heads / head_dim / block_size / num_layers.  Same device, or dst a remote */
/* view (peer-mapped), or src a remote view (P2P pull).  n == 0 is a no-op.          */
/* A view whose desc.device is another GPU's ordinal is a remote view: the copy is  */
/* NVLink-bound and runs on one CTA per SM (env BS_REMOTE_COPY_CTAS overrides), so  */
/* it leaves the other SM slots to the compute beside it.                           */
/* method: BS_MIGRATE_AUTO picks the fastest; VEC16 = 16-byte vector LDG/STG copy;  */
/* BULK = TMA bulk copies (cp.async.bulk) global->smem->global.                      */
/* ------------------------------------------------------------------------------ */
enum { BS_MIGRATE_AUTO = 0, BS_MIGRATE_VEC16 = 1, BS_MIGRATE_BULK = 2 };

bs_status bs_kv_migrate_layer(const bs_kv_pool* src, bs_kv_pool* dst, int32_t layer,
                              const int32_t* src_ids, const int32_t* dst_ids, int32_t n,
                              void* stream);
bs_status bs_kv_migrate_layer_ex(const bs_kv_pool* src, bs_kv_pool* dst, int32_t layer,
                                 const int32_t* src_ids, const int32_t* dst_ids, int32_t n,
                                 int32_t method, void* stream);

/* ------------------------------------------------------------------------------ */
/* H7 (adjacent to the path): append the decoded token's K/V.       */
/* The paper is silent; reading R-A9: seq_len includes the token being decoded, so  */
/* its K/V is written to the cache before attention (H4) runs.  For every request b */
/* with pos[b] >= 0, kv head g:                                                      */
/*   K page (layer, block_tables[b][pos[b]/16], g), slot pos[b]%16 <- k_new[b][g][:] */
/*   V page (same block, g),                        slot pos[b]%16 <- v_new[b][g][:] */
/* a bit copy; pos[b] < 0 skips request b.  pos is the shard-LOCAL token index (the  */
/* shard that holds the sequence's end).                                             */
/* k_new, v_new DEVICE bf16 [batch][num_kv_heads][head_dim], 16-B aligned.           */
/* block_tables DEVICE int32 [batch][max_blocks]; pos DEVICE int32 [batch].          */
/* Device arrays are not validated in release builds (block ids must be <         */
/* num_blocks, pos[b]/16 < max_blocks); the debug build checks them (code 8: a     */
/* position past the table).  Enqueued on `stream`; never synchronises.              */
/* ------------------------------------------------------------------------------ */
bs_status bs_kv_append_token(bs_kv_pool* pool, int32_t layer, const void* k_new, const void* v_new,
                             int32_t batch, const int32_t* block_tables, int32_t max_blocks,
                             const int32_t* pos, void* stream);
/* H2 + H7 as ONE launch on the migration stream: the hand-off copy of
 * bs_kv_migrate_layer(src -> dst, layer, n pairs) and the append of bs_kv_append_token
 * into app_pool (same layer) -- independent bit copies, so the result is both calls'
 * result.  Caller contract: the append's target slots lie outside the n source and
 * destination chunks (the hand-off moves whole blocks of other requests).
 * With a host-tier or peer-mapped pool, or n == 0 / batch == 0, it runs the two calls. */
bs_status bs_kv_migrate_append_layer(const bs_kv_pool* src, bs_kv_pool* dst, int32_t layer,
                                     const int32_t* src_ids, const int32_t* dst_ids, int32_t n,
                                     bs_kv_pool* app_pool, const void* k_new, const void* v_new,
                                     int32_t batch, const int32_t* block_tables,
                                     int32_t max_blocks, const int32_t* pos, void* stream);

/* Copy-engine variant (DMA, no SM time -- for the host tier's fetch / store legs, which
 * should not compete with attention for SMs): HOST int32 id arrays (validated), runs of
 * consecutive ids coalesced, one cudaMemcpyAsync per run.  Same semantics as
 * bs_kv_migrate_layer. */
bs_status bs_kv_migrate_layer_ce(const bs_kv_pool* src, bs_kv_pool* dst, int32_t layer,
                                 const int32_t* src_ids, const int32_t* dst_ids, int32_t n,
                                 void* stream);

/* Two-sided transport halves (pack / unpack), for a send/recv transport (NCCL) that
 * moves one contiguous staging buffer per layer: staging[i] = chunk(layer, ids[i]).
 * staging: DEVICE buffer of n * bs_kv_chunk_bytes bytes, 16-B aligned. */
bs_status bs_kv_gather_layer(const bs_kv_pool* src, int32_t layer, const int32_t* ids, int32_t n,
                             void* staging, void* stream);
bs_status bs_kv_scatter_layer(bs_kv_pool* dst, int32_t layer, const int32_t* ids, int32_t n,
                              const void* staging, void* stream);

/* ------------------------------------------------------------------------------ */
/* H4: decode attention over this instance's shard `shard_id` of every request's KV  */
/* (split attention, eqs. 6-9, corrected per readings R-A1..R-A11): */
/*   shard j of request b = global tokens [kv_split[b][j], kv_split[b][j+1]), stored */
/*   in shard-local order: local token u at block block_tables[b][u/16], slot u%16.  */
/*   q-head h attends kv-head floor(h / G).                                          */
/*   s_u = scale * <q_bh, k_u>;  m = max_u s_u;  l = sum_u exp(s_u - m);             */
/*   o~  = sum_u exp(s_u - m) v_u / l                (fp32, natural-log units)      */
/*   empty shard: m = -inf, l = 0, o~ = 0.                                            */
/* q            DEVICE bf16 [batch][num_q_heads][head_dim]                            */
/* block_tables DEVICE int32 [batch][max_blocks] physical ids in `pool`               */
/* kv_split     DEVICE int32 [batch][n_shards+1], non-decreasing                      */
/* o_part       DEVICE fp32 [batch][num_q_heads][head_dim]                            */
/* m, l         DEVICE fp32 [batch][num_q_heads]                                      */
/* workspace    DEVICE scratch for the intra-GPU split-K (bytes from                  */
/*              bs_split_decode_attention_workspace_size, 0 allowed if it says 0).    */
/*              Must be zero-filled once before first use; every call leaves it       */
/*              zero-filled again.  Not shareable between concurrently running calls. */
/* max_blocks must be >= ceil(len of the longest shard / 16).                          */
/* ------------------------------------------------------------------------------ */
bs_status bs_split_decode_attention_workspace_size(const bs_kv_pool* pool, int32_t batch,
                                                   int32_t num_q_heads, int32_t max_blocks,
                                                   size_t* bytes);
bs_status bs_split_decode_attention(const bs_kv_pool* pool, int32_t layer, const void* q,
                                    int32_t batch, int32_t num_q_heads,
                                    const int32_t* block_tables, int32_t max_blocks,
                                    const int32_t* kv_split, int32_t n_shards, int32_t shard_id,
                                    float scale, float* o_part, float* m, float* l,
                                    void* workspace, size_t workspace_bytes, void* stream);

/* H4 + H6 fused for shards that live on THIS GPU (the N=1 / co-located case): one
 * launch computes every local shard of every request, writes the per-CTA partials to
 * the workspace, and the last CTA of each (request, kv-head) merges them -- all local
 * shards and intra-shard split-K ranges -- in fixed order (shard-major) into bf16 O
 * and fp32 lse (natural log).  Equivalent to bs_split_decode_attention per shard +
 * bs_merge_partials, without the partial round trip and the extra launches.
 * pools / block_tables / max_blocks / shard_ids: HOST arrays of n_local (1..8) entries;
 * the pools must share num_layers / num_kv_heads / head_dim.  out bf16 [B][Hq][D] and
 * lse fp32 [B][Hq] (or NULL) are DEVICE buffers.  Workspace rules as for H4. */
bs_status bs_split_decode_attention_local_workspace_size(int32_t n_local,
                                                         const bs_kv_pool* const* pools,
                                                         const int32_t* max_blocks, int32_t batch,
                                                         int32_t num_q_heads, size_t* bytes);
bs_status bs_split_decode_attention_local(int32_t n_local, const bs_kv_pool* const* pools,
                                          int32_t layer, const void* q, int32_t batch,
                                          int32_t num_q_heads, const int32_t* const* block_tables,
                                          const int32_t* max_blocks, const int32_t* shard_ids,
                                          const int32_t* kv_split, int32_t n_shards, float scale,
                                          void* out, float* lse, void* workspace,
                                          size_t workspace_bytes, void* stream);
/* The same with launch flags.  BS_ATTN_PDL: a programmatic dependent launch -- it may start
 * while the previous kernel on `stream` drains (a previous attention launch lets it start once
 * its own CTAs have started (multi-wave) or finished their main loops (one wave)), reading
 * block_tables / kv_split and prefetching K/V pages before that kernel completes, and
 * q / out / lse / workspace only after (griddepcontrol.wait).  A one-wave predecessor that
 * occupies more than half the CTA slots lets it start only as its CTAs exit (so it is placed
 * evenly); a flagged launch of at most one CTA per SM runs a 6-stage ring.
 * The flag never changes the range cut: flagged and plain launches are bitwise identical.
 * Caller contract: the kernel launched just before it on `stream` writes neither the pools'
 * pages this call reads, nor block_tables / kv_split (e.g. the previous layer's attention;
 * work from other streams joined by events is waited for in full).  DESIGN.md §6. */
#define BS_ATTN_PDL 1u
/* BS_ATTN_NO_CLUSTER: never use the cluster merge.  By default a launch whose CTAs fit one
 * wave and whose (request, kv-head) is cut into 2..16 ranges runs each (request, kv-head)'s
 * ranges as one thread-block cluster and merges their partials through distributed shared
 * memory instead of the workspace (same arithmetic, bitwise the same result). */
#define BS_ATTN_NO_CLUSTER 2u
bs_status bs_split_decode_attention_local_ex(int32_t n_local, const bs_kv_pool* const* pools,
                                             int32_t layer, const void* q, int32_t batch,
                                             int32_t num_q_heads,
                                             const int32_t* const* block_tables,
                                             const int32_t* max_blocks, const int32_t* shard_ids,
                                             const int32_t* kv_split, int32_t n_shards, float scale,
                                             void* out, float* lse, void* workspace,
                                             size_t workspace_bytes, uint32_t flags, void* stream);

/* Ragged plan for mixed lengths (FlashInfer-style plan / run; C4's Alpaca + LongBench
 * mix): from the HOST copy of kv_split, cut every (request, local shard) into ranges of
 * at most `max_blocks_per_range` blocks (0 = automatic: the uniform planner's range length,
 * >= 16 blocks) -- empty shards get no CTA, short requests one range per shard,
 * long ones several -- instead of the uniform grid's max_blocks-wide cut.  One plan
 * serves every layer of a decode step.
 * work: HOST int32 [capacity][4] (NULL with capacity 0 = query the count in *n_work);
 * the caller copies the first *n_work items to a 16-B aligned DEVICE buffer.
 * *max_parts: most ranges of one request (<= 64); *workspace_bytes: scratch for
 * bs_split_decode_attention_local_ragged (0 if no request has > 1 range).
 * Results are identical in value to the uniform path (same formulas); the summation
 * order of the merge follows the plan's slots (shard-major, then range).  Items are
 * listed longest range first (stable; the CTA dispatch order), so a request's items need
 * not be adjacent; environment BS_RAGGED_ORDER=0 keeps request order. */
bs_status bs_attention_ragged_plan(int32_t batch, int32_t n_shards, const int32_t* kv_split_host,
                                   int32_t n_local, const int32_t* shard_ids, int32_t num_q_heads,
                                   int32_t num_kv_heads, int32_t head_dim,
                                   int32_t max_blocks_per_range, int32_t* work, int32_t capacity,
                                   int32_t* n_work, int32_t* max_parts, size_t* workspace_bytes);
/* The same with flags.  BS_PLAN_PACK_SHORT (one local shard): requests whose shard has at
 * most 8 blocks (128 tokens) are packed four to a CTA -- one warp per request, which writes
 * its own O / lse with no cross-warp combine -- instead of one CTA per (request, kv-head);
 * such an item has its parts field (low byte of w) 0: (b0, b1, b2, b3 << 8), -1 = no request.
 * Packed plans need the tensor-core kernel (the CUDA-core kernel traps on them); they are
 * made only when it is the active variant. */
#define BS_PLAN_PACK_SHORT 1u
bs_status bs_attention_ragged_plan_ex(int32_t batch, int32_t n_shards, const int32_t* kv_split_host,
                                      int32_t n_local, const int32_t* shard_ids, int32_t num_q_heads,
                                      int32_t num_kv_heads, int32_t head_dim,
                                      int32_t max_blocks_per_range, uint32_t flags, int32_t* work,
                                      int32_t capacity, int32_t* n_work, int32_t* max_parts,
                                      size_t* workspace_bytes);
/* bs_split_decode_attention_local over a ragged plan (work: DEVICE copy of the plan's
 * items, n_work of them; max_parts from the plan).  Same outputs and workspace rules. */
bs_status bs_split_decode_attention_local_ragged(
    int32_t n_local, const bs_kv_pool* const* pools, int32_t layer, const void* q, int32_t batch,
    int32_t num_q_heads, const int32_t* const* block_tables, const int32_t* max_blocks,
    const int32_t* shard_ids, const int32_t* kv_split, int32_t n_shards, float scale,
    const int32_t* work, int32_t n_work, int32_t max_parts, void* out, float* lse, void* workspace,
    size_t workspace_bytes, void* stream);
/* The same with launch flags (BS_ATTN_PDL as for bs_split_decode_attention_local_ex, same
 * caller contract; a ragged plan never uses the cluster merge). */
bs_status bs_split_decode_attention_local_ragged_ex(
    int32_t n_local, const bs_kv_pool* const* pools, int32_t layer, const void* q, int32_t batch,
    int32_t num_q_heads, const int32_t* const* block_tables, const int32_t* max_blocks,
    const int32_t* shard_ids, const int32_t* kv_split, int32_t n_shards, float scale,
    const int32_t* work, int32_t n_work, int32_t max_parts, void* out, float* lse, void* workspace,
    size_t workspace_bytes, uint32_t flags, void* stream);

/* H4 + H5 + H6 fused across GPUs ("fused B200 variant"; PAPER.md:220,
 * :233-237): an attention PROBLEM is a batch of requests whose KV shards may live on
 * several GPUs.  Every launch that holds a shard of it writes that shard's per-range
 * partials straight into the problem's workspace on the home GPU (peer-mapped, NVLink
 * stores) and bumps the per-(request, kv-head) arrival counter there; whichever CTA
 * arrives last -- on any GPU -- performs the eq. 10 merge over all ranges in fixed
 * order (shard-major) and writes bf16 O + fp32 lse into the home GPU's buffers, then
 * increments the problem's `done` counter.  No partial round trip, no merge launch, no
 * collective call.  One launch may serve several problems (e.g. on GPU r of the ring:
 * shard 0 of its own requests + shard 1 of its predecessor's).
 *
 * bs_attn_problem (identical on every GPU that serves the problem; pointers as seen
 *   from the launching GPU, i.e. peer-mapped when the home is another GPU):
 *   q          bf16 [batch][num_q_heads][head_dim] (readable by the launching GPU)
 *   kv_split   DEVICE int32 [batch][n_shards+1] (the launching GPU's copy)
 *   max_blocks HOST int32 [n_shards]: block-table width of EVERY shard of the problem
 *              (n_shards <= 16); together with batch / heads / head_dim it fixes the
 *              range plan, so every GPU must pass the same values.  The plan uses only
 *              these rank-invariant inputs (a fixed 148 x 3 CTA-slot model, no device
 *              query, no environment switch), so GPUs of different SM counts or
 *              environments still cut the ranges identically
 *   out, lse   home GPU bf16 [batch][num_q_heads][head_dim], fp32 [batch][num_q_heads]
 *              (lse may be NULL)
 *   workspace  home GPU scratch of bs_attention_problem_workspace_size bytes, zero-filled
 *              once before first use (arrival counters re-arm themselves); a problem's
 *              workspace may not be reused before its `done` reached the call's target
 *   done       home GPU int32 counter or NULL: +batch*num_kv_heads per completed call,
 *              with release semantics (system scope when cross_device) -- wait on it
 *              (bs_wait_signal) before reading out / lse or reusing the workspace
 *   cross_device 1 when the problem's shards run on more than one GPU
 * bs_attn_task: one shard of one problem processed by THIS launch: pool (device-resident,
 *   this GPU), block_tables DEVICE [batch][max_blocks[shard_id]], shard_id, problem index,
 *   optional dispatch order of the requests (ABI version 2).
 * 1 <= n_tasks <= 8, 1 <= n_problems <= 8; all tasks' pools share num_kv_heads / head_dim /
 * num_layers; all problems have `batch` requests of num_q_heads heads.  The caller
 * guarantees that every task of a problem is launched exactly once per call epoch.
 * PAPER.md gives no fused variant; this is the B200 form of "E^(1) / O^(1) is sent back
 * before the final summation" (:237) with the exchange folded into the producer. */
typedef struct {
  const void* q;
  const int32_t* kv_split;
  int32_t n_shards;
  const int32_t* max_blocks;
  void* out;
  float* lse;
  void* workspace;
  size_t workspace_bytes;
  int32_t* done;
  int32_t cross_device;
} bs_attn_problem;

typedef struct {
  const bs_kv_pool* pool;
  const int32_t* block_tables;
  int32_t shard_id;
  int32_t problem;
  const int32_t* order;  /* DEVICE int32 [batch] permutation or NULL: CTA row z serves request
                            order[z] (e.g. longest shard first, so the longest CTAs start in
                            the first wave); results do not depend on it (merge = slot order) */
} bs_attn_task;

bs_status bs_attention_problem_workspace_size(int32_t batch, int32_t num_q_heads,
                                              int32_t num_kv_heads, int32_t head_dim,
                                              int32_t n_shards, const int32_t* max_blocks,
                                              size_t* bytes);
bs_status bs_split_decode_attention_tasks(int32_t n_problems, const bs_attn_problem* problems,
                                          int32_t n_tasks, const bs_attn_task* tasks,
                                          int32_t layer, int32_t batch, int32_t num_q_heads,
                                          float scale, void* stream);

/* ------------------------------------------------------------------------------ */
/* NEXT F3: layer-level migration (Fig. 3, eqs. 3-5): a contiguous  */
/* set of layers moves with its weights W_l and its KV_l.  bs_kv_migrate_layers is    */
/* bs_kv_migrate_layer for layers [layer_lo, layer_lo + n_layers) in ONE launch (the  */
/* same pairs every layer: block ids are shared by all layers).  bs_copy_bytes moves a */
/* weight tensor (DEVICE / peer / pinned-host pointers; copy engine).                 */
/* ------------------------------------------------------------------------------ */
bs_status bs_kv_migrate_layers(const bs_kv_pool* src, bs_kv_pool* dst, int32_t layer_lo,
                               int32_t n_layers, const int32_t* src_ids, const int32_t* dst_ids,
                               int32_t n, void* stream);
bs_status bs_copy_bytes(void* dst, const void* src, size_t bytes, void* stream);

/* ------------------------------------------------------------------------------ */
/* NEXT F2: head-granular attention-level migration -- the paper's literal text       */
/* ("partition the KV Cache along the attention head dimension and selectively      */
/* migrate only the KV states of certain heads"; Alg. 1      */
/* MigrateKVHeads).  For every pair i, the K and V pages of kv-heads   */
/* [src_head_lo, src_head_lo+n_heads) of chunk(layer, src_ids[i]) are copied to      */
/* heads [dst_head_lo, ...) of chunk(layer, dst_ids[i]).  The pools must agree on    */
/* num_layers / head_dim and may differ in num_kv_heads (a cold pool can hold just   */
/* the migrated heads).  Bit-exact; ids are DEVICE int32 [n].                        */
/* ------------------------------------------------------------------------------ */
bs_status bs_kv_migrate_heads_layer(const bs_kv_pool* src, bs_kv_pool* dst, int32_t layer,
                                    const int32_t* src_ids, const int32_t* dst_ids, int32_t n,
                                    int32_t src_head_lo, int32_t dst_head_lo, int32_t n_heads,
                                    void* stream);
/* H4 restricted to n_kv_heads kv-heads: pool heads [pool_head_lo, +n) are the model's
 * kv-heads [model_head_lo, +n); G = num_q_heads / num_kv_heads_total.  q, o_part, m, l
 * keep the MODEL's full layouts ([batch][num_q_heads]...): only the rows of q-heads
 * [model_head_lo*G, (model_head_lo+n)*G) are read / written, so the home and the cold
 * instance write disjoint rows of one buffer and the head-split "merge" is a concat.
 * Everything else as bs_split_decode_attention. */
bs_status bs_split_decode_attention_heads_workspace_size(const bs_kv_pool* pool, int32_t batch,
                                                         int32_t n_kv_heads,
                                                         int32_t num_kv_heads_total,
                                                         int32_t num_q_heads, int32_t max_blocks,
                                                         size_t* bytes);
bs_status bs_split_decode_attention_heads(const bs_kv_pool* pool, int32_t layer,
                                          int32_t pool_head_lo, int32_t model_head_lo,
                                          int32_t n_kv_heads, int32_t num_kv_heads_total,
                                          const void* q, int32_t batch, int32_t num_q_heads,
                                          const int32_t* block_tables, int32_t max_blocks,
                                          const int32_t* kv_split, int32_t n_shards,
                                          int32_t shard_id, float scale, float* o_part, float* m,
                                          float* l, void* workspace, size_t workspace_bytes,
                                          void* stream);

/* ------------------------------------------------------------------------------ */
/* H6: exact LSE merge of n shard partials (eq. 10, R-A4, R-A14):   */
/*   lse_j = m_j + ln l_j (-inf if l_j = 0);  lse = logsumexp_j lse_j;                */
/*   out = sum_j exp(lse_j - lse) o~_j, fixed order j = 0..n-1; all empty -> 0, -inf. */
/* o_parts/m_parts/l_parts: HOST arrays of n DEVICE pointers (layouts as in H4).      */
/* out: DEVICE bf16 [batch][num_q_heads][head_dim] (round-to-nearest-even).           */
/* lse_out: DEVICE fp32 [batch][num_q_heads] or NULL.  1 <= n_parts <= 16.             */
/* ------------------------------------------------------------------------------ */
bs_status bs_merge_partials(int32_t n_parts, const float* const* o_parts,
                            const float* const* m_parts, const float* const* l_parts,
                            int32_t batch, int32_t num_q_heads, int32_t head_dim, void* out,
                            float* lse_out, void* stream);

/* ------------------------------------------------------------------------------ */
/* Cross-instance transports (reading D6; PAPER.md:197 names NVLink / InfiniBand).   */
/*                                                                                  */
/* (a) Two-sided NCCL (resolved at run time: dlopen "libnccl.so.2" or               */
/*     $BS_NCCL_LIBRARY; without NCCL these return BS_ERR_NCCL).  A bs_comm wraps an */
/*     ncclComm_t built from a unique id the harness broadcasts.  Every call is     */
/*     enqueued on `stream`; send/recv pairs must be issued in the same order on    */
/*     both peers (NCCL rules).  A peer may be the caller itself (loopback).        */
/* ------------------------------------------------------------------------------ */
typedef struct bs_comm bs_comm;

/* Size of an NCCL unique id (128). */
size_t bs_nccl_unique_id_bytes(void);
/* Rank 0 creates the id into `out` (host, bs_nccl_unique_id_bytes bytes). */
bs_status bs_nccl_get_unique_id(void* out);
/* Collective over the nranks processes; the current CUDA device is this rank's GPU. */
bs_status bs_comm_init(const void* nccl_unique_id, int32_t nranks, int32_t rank, bs_comm** out);
bs_status bs_comm_destroy(bs_comm* comm);
/* One grouped ncclSend(sendbuf -> send_peer) + ncclRecv(recvbuf <- recv_peer) of raw
 * bytes (DEVICE buffers).  A negative peer or zero size skips that half.  This is the
 * H5 partial exchange: a partial is one contiguous fp32 buffer [o~ | m | l]. */
bs_status bs_sendrecv(bs_comm* comm, const void* sendbuf, size_t send_bytes, int32_t send_peer,
                      void* recvbuf, size_t recv_bytes, int32_t recv_peer, void* stream);
/* Many sends and receives of raw bytes in ONE NCCL group (HOST arrays of n_send /
 * n_recv entries; DEVICE buffers): the W-way exchanges of the sequence-sharded step --
 * q of a home to every peer (an all-gather), each shard's partial (o~, m, l) to its
 * request's home ("O^(1) (or E^(2)) is sent back").  Zero-byte entries are
 * skipped; every rank must post matching pairs.  Returns BS_ERR_NCCL on an NCCL error. */
bs_status bs_exchange(bs_comm* comm, int32_t n_send, const void* const* send_bufs,
                      const size_t* send_bytes, const int32_t* send_peers, int32_t n_recv,
                      void* const* recv_bufs, const size_t* recv_bytes, const int32_t* recv_peers,
                      void* stream);
/* H2 over NCCL: gather chunk(layer, src_ids[i]) into staging (n * chunk bytes, DEVICE)
 * and send it to `peer`; the peer's bs_kv_recv_layer receives into its staging and
 * scatters to chunk(layer, dst_ids[i]).  Bit-exact, same pair order on both sides. */
bs_status bs_kv_send_layer(const bs_kv_pool* src, int32_t layer, const int32_t* src_ids, int32_t n,
                           int32_t peer, bs_comm* comm, void* staging, void* stream);
bs_status bs_kv_recv_layer(bs_kv_pool* dst, int32_t layer, const int32_t* dst_ids, int32_t n,
                           int32_t peer, bs_comm* comm, void* staging, void* stream);
/* Both halves in one NCCL group (ring neighbours: send to one peer, receive from
 * another without deadlock).  n_send or n_recv may be 0. */
bs_status bs_kv_sendrecv_layer(bs_comm* comm, const bs_kv_pool* src, const int32_t* src_ids,
                               int32_t n_send, int32_t send_peer, void* send_staging,
                               bs_kv_pool* dst, const int32_t* dst_ids, int32_t n_recv,
                               int32_t recv_peer, void* recv_staging, int32_t layer, void* stream);

/* (b) CUDA IPC: export a device pointer (possibly interior to an allocation) as a
 * handle + offset; another process imports it as a device pointer usable as the `base`
 * of a remote-view pool, so bs_kv_migrate_layer pushes chunks over NVLink (P2P push).
 * handle: host buffer of bs_ipc_handle_bytes() bytes.  bs_ipc_close undoes an import. */
size_t bs_ipc_handle_bytes(void);
/* Signalling for pushes into peer memory: bs_signal enqueues "all prior work on `stream`
 * is complete and visible system-wide, then *flag = value" (flag may be peer-mapped);
 * bs_wait_signal enqueues "wait until *flag >= value" (flag local or peer) -- epochs only
 * grow, so flags are never reset.  A wait gives up after timeout_ns (0 = never) and sets
 * *err = 1 (err DEVICE int32, may be NULL) rather than hang the stream. */
bs_status bs_signal(int32_t* flag, int32_t value, void* stream);
bs_status bs_wait_signal(const int32_t* flag, int32_t value, uint64_t timeout_ns, int32_t* err,
                         void* stream);
/* bs_signal for n (1..16) flags in one launch, all set to `value`; HOST array of device
 * (or peer-mapped) pointers. */
bs_status bs_signals(int32_t n, int32_t* const* flags, int32_t value, void* stream);
/* Several waits in one launch: until *flags[i] >= values[i] for every i < n (1..16);
 * flags / values are HOST arrays (of device pointers / values). */
bs_status bs_wait_signals(int32_t n, const int32_t* const* flags, const int32_t* values,
                          uint64_t timeout_ns, int32_t* err, void* stream);
/* "*flag >= value" is wrap-safe: flags and counters are int32 and wrap after 2^31, so a
 * wait is satisfied when (int32_t)(*flag - value) >= 0 (the two are always within 2^31).
 * err may point to device memory or to page-locked host memory (the host can poll it
 * without synchronising); a timeout stores 1 there with a system-scope store.
 *
 * Device-epoch variants, for steps captured in a CUDA graph: the value of
 * flag i is computed on the device when the kernel runs, (*epoch) * mul[i] + add[i]
 * (int32, wrapping), so a replayed graph signals / waits for the current step.  epoch:
 * DEVICE int32 step counter owned by the caller; bs_epoch_advance enqueues *epoch += 1.
 * flags / mul / add: HOST arrays of n (1..16) entries. */
bs_status bs_signals_epoch(int32_t n, int32_t* const* flags, const int32_t* mul, const int32_t* add,
                           const int32_t* epoch, void* stream);
bs_status bs_wait_signals_epoch(int32_t n, const int32_t* const* flags, const int32_t* mul,
                                const int32_t* add, const int32_t* epoch, uint64_t timeout_ns,
                                int32_t* err, void* stream);
bs_status bs_epoch_advance(int32_t* epoch, void* stream);
bs_status bs_ipc_export(const void* dev_ptr, void* handle_out, size_t* offset_out);
bs_status bs_ipc_import(const void* handle, size_t offset, void** dev_ptr_out);
bs_status bs_ipc_close(void* dev_ptr, size_t offset);

/* ------------------------------------------------------------------------------ */
/* NEXT F4: control plane (host only; §4.4).  Readings R-F4a..g in */
/* DESIGN.md.  Loads are normalised utilisations U = C/C_max + M/M_max (eq. 32/37).  */
/* ------------------------------------------------------------------------------ */
double bs_utilization(double c, double c_max, double m, double m_max);
/* Alg. 2: dispatch n_req requests (est_load[r] each, in queue order) over n_inst
 * prefill instances.  load / q_len (HOST arrays [n_inst]) are read and updated in
 * place; assign_out[r] = chosen instance.  Least-loaded (load, q_len, index) if its load
 * < delta_l (then load += est_load), else lowest-queue (q_len, load, index); q_len += 1
 * on every assignment. */
bs_status bs_dispatch_requests(int32_t n_inst, double* load, int32_t* q_len, int32_t n_req,
                               const double* est_load, double delta_l, int32_t* assign_out);
/* Alg. 1, one control cycle over n_dev devices (HOST arrays [n_dev]; load, n_layers,
 * n_heads updated in place).  While an overloaded (load - min > delta) and another
 * underloaded (max - load > delta) device exist: d_o = most loaded overloaded, d_u =
 * least loaded underloaded; if the gap >= delta try a layer move (supports_layer,
 * n_layers > 0) then a KV-head move (supports_attn, n_heads > 0), each executed only if
 * (gap - |gap after|) / cost >= rho (eq. 35).  Stops when no move passes or after
 * max_moves.  moves_out[3k..3k+2] = (kind 0 layer | 1 heads, from, to). */
bs_status bs_plan_migrations(int32_t n_dev, double* load, int32_t* n_layers, const double* layer_load,
                             const double* layer_cost, int32_t* n_heads, const double* head_load,
                             const double* head_cost, const uint8_t* supports_layer,
                             const uint8_t* supports_attn, double delta, double rho,
                             int32_t max_moves, int32_t* moves_out, int32_t* n_moves_out);

#ifdef __cplusplus
}
#endif
#endif /* BANASERVE_H_ */
