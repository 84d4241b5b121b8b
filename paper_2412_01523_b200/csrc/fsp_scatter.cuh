// fsp_scatter.cuh — the fused head->seq exchange (Eq. 4) used by the attention epilogues.
//
// An attention kernel of group member j produces output rows t of the group-packed
// sequence for its heads.  Instead of a separate fsp_a2a_head2seq launch afterwards, the
// epilogue stores each finished row straight into the sequence-sharded buffer of the
// member that owns it (peer-mapped NVSwitch memory), through the group's unpack table —
// the same addressing a2a_kernel<false> uses (fsp_a2a.cu), applied tile by tile.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "fsp_host.h"

namespace fsp {

struct ScatterDev {
  int32_t degree;          // 0: off
  int32_t rows_per_rank;
  int32_t head_offset;
  int64_t dst_stride;      // elements
  int64_t mat_stride;      // elements
  const int32_t* unpack;   // [degree * rows_per_rank]
  __nv_bfloat16* dst[8];
};

// Destination of (group-packed row t, matrix mat, local head h) or nullptr (pad row / off).
__device__ __forceinline__ __nv_bfloat16* scatter_row(const ScatterDev& s, int64_t t, int mat,
                                                      int h, int head_dim) {
  if (s.degree == 0) return nullptr;
  const int32_t row = __ldg(s.unpack + t);
  if (row < 0) return nullptr;
  const int r = (int)(t / s.rows_per_rank);
  return s.dst[r] + (int64_t)row * s.dst_stride + mat * s.mat_stride +
         (int64_t)(s.head_offset + h) * head_dim;
}

// Host: validate the ABI struct and convert it (n_mats = matrices the kernel writes).
int scatter_from_abi(const FspHeadScatter& a, int n_mats, int n_heads, int head_dim,
                     int total_rows, ScatterDev* out);

}  // namespace fsp
