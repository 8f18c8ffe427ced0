// H6: exact log-sum-exp merge of the shard partials (eq. 10, with
// reading R-A4: each O^(j) re-weighted by its share of the global denominator),
// fixed shard order 0..n-1 (R-A14), -inf-safe for empty shards (R-A7).
//   lse_j = m_j + ln l_j;  lse = M + ln sum_j exp(lse_j - M);  O = sum_j e^{lse_j - lse} o~_j
// One warp per (request, q-head) row; lane owns d/32 contiguous dims (float4/float2
// loads), result rounded RNE to bf16.  Latency-bound (KB-sized).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "internal.h"

namespace bs {
namespace {

constexpr int kMaxParts = 16;

struct MergeArgs {
  const float* o[kMaxParts];
  const float* m[kMaxParts];
  const float* l[kMaxParts];
};

template <int D>
__global__ void __launch_bounds__(256) merge_partials_kernel(const MergeArgs a, int n, int64_t rows,
                                                             __nv_bfloat16* __restrict__ out,
                                                             float* __restrict__ lse_out) {
  constexpr int DPL = D / 32;
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  float lse_j[kMaxParts];
  float M = -INFINITY;
#pragma unroll
  for (int j = 0; j < kMaxParts; ++j) {
    if (j < n) {
      const float lj = __ldg(a.l[j] + row);
      lse_j[j] = lj > 0.f ? __ldg(a.m[j] + row) + logf(lj) : -INFINITY;
      M = fmaxf(M, lse_j[j]);
    }
  }
  float acc[DPL];
#pragma unroll
  for (int x = 0; x < DPL; ++x) acc[x] = 0.f;
  float lse = -INFINITY;
  if (M != -INFINITY) {
    float S = 0.f;
#pragma unroll
    for (int j = 0; j < kMaxParts; ++j)
      if (j < n && lse_j[j] != -INFINITY) S += expf(lse_j[j] - M);
    lse = M + logf(S);
#pragma unroll
    for (int j = 0; j < kMaxParts; ++j) {
      if (j < n && lse_j[j] != -INFINITY) {
        const float w = expf(lse_j[j] - lse);
        const float* po = a.o[j] + row * D + lane * DPL;
        if constexpr (DPL == 4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(po));
          acc[0] += w * v.x;
          acc[1] += w * v.y;
          acc[2] += w * v.z;
          acc[3] += w * v.w;
        } else {
          const float2 v = __ldg(reinterpret_cast<const float2*>(po));
          acc[0] += w * v.x;
          acc[1] += w * v.y;
        }
      }
    }
  }
  __nv_bfloat16* po = out + row * D + lane * DPL;
  if constexpr (DPL == 4) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc[0], acc[1]);
    __nv_bfloat162 hi = __floats2bfloat162_rn(acc[2], acc[3]);
    uint2 w;
    w.x = *reinterpret_cast<uint32_t*>(&lo);
    w.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(po) = w;
  } else {
    *reinterpret_cast<__nv_bfloat162*>(po) = __floats2bfloat162_rn(acc[0], acc[1]);
  }
  if (lse_out && lane == 0) lse_out[row] = lse;
}

}  // namespace
}  // namespace bs

extern "C" bs_status bs_merge_partials(int32_t n_parts, const float* const* o_parts,
                                       const float* const* m_parts, const float* const* l_parts,
                                       int32_t batch, int32_t num_q_heads, int32_t head_dim,
                                       void* out, float* lse_out, void* stream) {
  BS_REQUIRE(n_parts >= 1 && n_parts <= bs::kMaxParts, "bs_merge_partials: n_parts %d not in [1,%d]",
             n_parts, bs::kMaxParts);
  BS_REQUIRE(o_parts && m_parts && l_parts, "bs_merge_partials: NULL pointer array");
  BS_REQUIRE(batch >= 0 && num_q_heads >= 1, "bs_merge_partials: bad batch/heads");
  if (head_dim != 64 && head_dim != 128)
    return bs::set_error(BS_ERR_UNSUPPORTED, "bs_merge_partials: head_dim %d", head_dim);
  if (batch == 0) return BS_OK;
  BS_REQUIRE(out != nullptr, "bs_merge_partials: out is NULL");
  bs::MergeArgs a{};
  for (int j = 0; j < n_parts; ++j) {
    BS_REQUIRE(o_parts[j] && m_parts[j] && l_parts[j], "bs_merge_partials: part %d NULL", j);
    BS_REQUIRE(((uintptr_t)o_parts[j] & 15) == 0, "bs_merge_partials: part %d not 16-B aligned", j);
    a.o[j] = o_parts[j];
    a.m[j] = m_parts[j];
    a.l[j] = l_parts[j];
  }
  const int64_t rows = (int64_t)batch * num_q_heads;
  const int wpb = 8;
  const unsigned grid = (unsigned)((rows + wpb - 1) / wpb);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (head_dim == 128)
    bs::merge_partials_kernel<128><<<grid, wpb * 32, 0, s>>>(a, n_parts, rows,
                                                            static_cast<__nv_bfloat16*>(out), lse_out);
  else
    bs::merge_partials_kernel<64><<<grid, wpb * 32, 0, s>>>(a, n_parts, rows,
                                                           static_cast<__nv_bfloat16*>(out), lse_out);
  return bs::check_launch("merge_partials_kernel");
}
