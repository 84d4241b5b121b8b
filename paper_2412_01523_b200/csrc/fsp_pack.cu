// fsp_pack.cu — varlen pack / unpack: permutation-driven row gather / scatter.
//
// The layout builder (paper_2412_01523_b200/layout.py) turns the planner's
// GroupDispatch.sequence_indices (pkg/src/seqplan/planner.py:501-509, dealing order;
// pkg/src/seqplan/baselines.py:101 for static plans) into an index vector
// index[packed_row] = loader_row.  Pack gathers loader-order rows into the
// group-packed, rank-sharded buffer that Ulysses SP consumes;
// unpack scatters results back.  Pure data movement, HBM-bound: every byte is read
// once and written once with 16-byte vector accesses; the flattened (row, vector)
// index space keeps all lanes busy for any row size.
#include "fsp_host.h"

namespace fsp {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// kScatter = false: dst[i] = src[idx[i]] (idx < 0 -> zeros)
// kScatter = true : dst[idx[i]] = src[i] (idx < 0 -> skipped)
template <bool kScatter>
__global__ void __launch_bounds__(kThreads) permute_rows_kernel(
    const uint8_t* __restrict__ src, int64_t src_stride, uint8_t* __restrict__ dst,
    int64_t dst_stride, const int32_t* __restrict__ idx, int64_t n_rows, uint32_t vec_per_row) {
  const int64_t total = n_rows * (int64_t)vec_per_row;
  const int64_t step = (int64_t)gridDim.x * kThreads;
  int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  for (; g < total; g += step * kUnroll) {
    int4 v[kUnroll];
    int64_t drow_off[kUnroll];
    bool live[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t e = g + u * step;
      live[u] = e < total;
      v[u] = make_int4(0, 0, 0, 0);
      drow_off[u] = -1;
      if (live[u]) {
        const int64_t row = e / vec_per_row;
        const int64_t col = e - row * vec_per_row;
        const int32_t r = idx[row];
        if (!kScatter) {
          if (r >= 0) v[u] = ld_stream(reinterpret_cast<const int4*>(src + r * src_stride) + col);
          drow_off[u] = row * dst_stride + col * 16;
        } else if (r >= 0) {
          v[u] = ld_stream(reinterpret_cast<const int4*>(src + row * src_stride) + col);
          drow_off[u] = (int64_t)r * dst_stride + col * 16;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (drow_off[u] >= 0) *reinterpret_cast<int4*>(dst + drow_off[u]) = v[u];
  }
}

template <bool kScatter>
int launch_permute(const void* src, int64_t ss, void* dst, int64_t ds, const int32_t* idx,
                   int64_t n_rows, int64_t row_bytes, void* stream) {
  FSP_CHECK_ARG(n_rows >= 0, "n_rows must be >= 0 (got %lld)", (long long)n_rows);
  if (n_rows == 0) return FSP_OK;
  FSP_CHECK_ARG(src && dst && idx, "null pointer argument");
  FSP_CHECK_ARG(row_bytes > 0 && row_bytes % 16 == 0, "row_bytes (%lld) must be a positive multiple of 16",
                (long long)row_bytes);
  FSP_CHECK_ARG(ss % 16 == 0 && ds % 16 == 0 && ss >= row_bytes && ds >= row_bytes,
                "row strides must be multiples of 16 and >= row_bytes");
  FSP_CHECK_ARG(((uintptr_t)src & 15) == 0 && ((uintptr_t)dst & 15) == 0,
                "src/dst must be 16-byte aligned");
  const int64_t vpr = row_bytes / 16;
  FSP_CHECK_ARG(vpr < (1ll << 31), "row too large");
  const int64_t total = n_rows * vpr;
  int64_t blocks = (total + (int64_t)kThreads * kUnroll - 1) / ((int64_t)kThreads * kUnroll);
  const int64_t cap = 148 * 16;  // 16 resident 256-thread CTAs per SM
  if (blocks > cap) blocks = cap;
  permute_rows_kernel<kScatter><<<(unsigned)blocks, kThreads, 0, (cudaStream_t)stream>>>(
      (const uint8_t*)src, ss, (uint8_t*)dst, ds, idx, n_rows, (uint32_t)vpr);
  FSP_LAUNCH_CHECK();
  return FSP_OK;
}

// Per-plan data scatter: route e = {src_row, dst_rank, dst_row}; the row is read once from
// the local loader shard and stored into the owning rank's input buffer (a peer-mapped
// NVSwitch address, or local memory for the own rank).  Flattened (route, 16-byte vector)
// index space as in permute_rows_kernel, 16-byte stores.
constexpr int kMaxPeers = 8;
struct PeerTable {
  uint8_t* p[kMaxPeers];
};

__global__ void __launch_bounds__(kThreads) scatter_rows_kernel(
    const uint8_t* __restrict__ src, int64_t src_stride, PeerTable dst, int64_t dst_stride,
    const int32_t* __restrict__ routes, int64_t n_routes, uint32_t vec_per_row) {
  const int64_t total = n_routes * (int64_t)vec_per_row;
  const int64_t step = (int64_t)gridDim.x * kThreads;
  for (int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x; g < total; g += step * kUnroll) {
    int4 v[kUnroll];
    uint8_t* d[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t e = g + u * step;
      d[u] = nullptr;
      if (e < total) {
        const int64_t i = e / vec_per_row;
        const int64_t col = e - i * vec_per_row;
        const int32_t sr = __ldg(routes + 3 * i), dr = __ldg(routes + 3 * i + 1),
                      drow = __ldg(routes + 3 * i + 2);
        v[u] = ld_stream(reinterpret_cast<const int4*>(src + (int64_t)sr * src_stride) + col);
        d[u] = dst.p[dr] + (int64_t)drow * dst_stride + col * 16;
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (d[u]) *reinterpret_cast<int4*>(d[u]) = v[u];
  }
  __threadfence_system();  // peer stores visible before the barrier that follows
}

}  // namespace
}  // namespace fsp

extern "C" int fsp_scatter_rows(const void* src, int64_t src_stride_bytes, void* const* peer_dst,
                                int32_t n_peers, int64_t dst_stride_bytes,
                                const int32_t* d_routes, int64_t n_routes, int64_t row_bytes,
                                void* stream) {
  using namespace fsp;
  FSP_CHECK_ARG(n_routes >= 0, "n_routes must be >= 0");
  FSP_CHECK_ARG(n_peers >= 1 && n_peers <= kMaxPeers, "n_peers must be in [1, %d]", kMaxPeers);
  FSP_CHECK_ARG(peer_dst != nullptr, "null peer_dst");
  if (n_routes == 0) return FSP_OK;
  FSP_CHECK_ARG(src && d_routes, "null pointer argument");
  FSP_CHECK_ARG(row_bytes > 0 && row_bytes % 16 == 0, "row_bytes must be a positive multiple of 16");
  FSP_CHECK_ARG(src_stride_bytes % 16 == 0 && dst_stride_bytes % 16 == 0 &&
                    src_stride_bytes >= row_bytes && dst_stride_bytes >= row_bytes,
                "row strides must be multiples of 16 and >= row_bytes");
  FSP_CHECK_ARG(((uintptr_t)src & 15) == 0, "src must be 16-byte aligned");
  PeerTable t{};
  for (int r = 0; r < n_peers; ++r) {
    FSP_CHECK_ARG(peer_dst[r] != nullptr && ((uintptr_t)peer_dst[r] & 15) == 0,
                  "peer_dst[%d] null or misaligned", r);
    t.p[r] = reinterpret_cast<uint8_t*>(peer_dst[r]);
  }
  const int64_t vpr = row_bytes / 16;
  FSP_CHECK_ARG(vpr < (1ll << 31) && n_routes < (1ll << 31), "scatter too large");
  const int64_t total = n_routes * vpr;
  int64_t blocks = (total + (int64_t)kThreads * kUnroll - 1) / ((int64_t)kThreads * kUnroll);
  if (blocks > 148 * 16) blocks = 148 * 16;
  scatter_rows_kernel<<<(unsigned)blocks, kThreads, 0, (cudaStream_t)stream>>>(
      (const uint8_t*)src, src_stride_bytes, t, dst_stride_bytes, d_routes, n_routes,
      (uint32_t)vpr);
  FSP_LAUNCH_CHECK();
  return FSP_OK;
}

extern "C" int fsp_pack_rows(const void* src, int64_t src_stride_bytes, void* dst,
                             int64_t dst_stride_bytes, const int32_t* d_index, int64_t n_rows,
                             int64_t row_bytes, void* stream) {
  return fsp::launch_permute<false>(src, src_stride_bytes, dst, dst_stride_bytes, d_index, n_rows,
                                    row_bytes, stream);
}

extern "C" int fsp_unpack_rows(const void* src, int64_t src_stride_bytes, void* dst,
                               int64_t dst_stride_bytes, const int32_t* d_index, int64_t n_rows,
                               int64_t row_bytes, void* stream) {
  return fsp::launch_permute<true>(src, src_stride_bytes, dst, dst_stride_bytes, d_index, n_rows,
                                   row_bytes, stream);
}
