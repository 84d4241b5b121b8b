// fsp_a2a.cu — Ulysses all-to-all inside one SP group over NVSwitch peer memory.
//
// Eq. (2) AlltoAll(Q_s, K_s, V_s): sequence-sharded -> head-sharded, and Eq. (4)
// AlltoAll(P_h): head-sharded -> sequence-sharded.  The paper runs
// these with NCCL on a cached group pool.  Here a group is just
// a rank range whose receive buffers are mapped into every member (symmetric memory):
// each rank pushes its slices straight into the peers' receive buffers with 16-byte
// stores over NVLink, so there is no communicator per group and "hot switching" between
// plans costs nothing.  The pack (loader-order -> group-packed rows) is fused into the
// send by reading source rows through the permutation; the unpack is fused into the
// receive side of head2seq the same way.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "fsp_host.h"
#include "fsp_ptx.cuh"

namespace fsp {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxDegree = 8;

struct PeerPtrs {
  uint8_t* p[kMaxDegree];
};

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// One warp moves one (row i, matrix m, peer j) chunk = the H_j*D*2-byte head slice of
// one row (1 KB at C2/d=8): index math once per chunk, 32 lanes x 16-byte vectors with
// kUnroll loads in flight per lane.  Peer j is the fastest-varying chunk coordinate so the
// local copy (j == rank) and the NVLink writes to all peers proceed concurrently, and the
// source row is read sequentially.
constexpr int kUnroll = 4;

template <bool kSeq2Head>
__global__ void __launch_bounds__(kThreads) a2a_kernel(const uint8_t* __restrict__ src,
                                                       PeerPtrs dst, const int32_t* __restrict__ index,
                                                       FspA2A a) {
  // a.head_begin is normalised by the host (even split filled in): member j owns heads
  // [head_begin[j], head_begin[j+1]); the head-sharded side spaces matrices hmax heads apart
  const int d = a.degree;
  int hmax = 0;
  for (int jj = 0; jj < d; ++jj) hmax = max(hmax, a.head_begin[jj + 1] - a.head_begin[jj]);
  const int64_t head_bytes = (int64_t)a.head_dim * 2;
  const int64_t sharded_mat = hmax * head_bytes;  // bytes per matrix on the head-sharded side
  const uint32_t n_chunks = (uint32_t)a.rows_per_rank * (uint32_t)a.n_mats * (uint32_t)d;
  const int64_t src_stride = a.src_stride * 2, dst_stride = a.dst_stride * 2;
  const int64_t full_row = (int64_t)a.n_heads * head_bytes;  // bytes of all heads of one mat
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (kThreads / 32);
  for (uint32_t c = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); c < n_chunks; c += warps) {
    const uint32_t j = c % d;
    const uint32_t rm = c / d;
    const uint32_t m = rm % a.n_mats;
    const uint32_t i = rm / a.n_mats;
    const int4* sp;
    int4* dp;
    bool zero = false;
    int vpc;
    if (kSeq2Head) {
      // local shard row i (all heads) -> peer j row (rank*R + i), peer j's heads
      const int hb = a.head_begin[j];
      vpc = (int)(((a.head_begin[j + 1] - hb) * head_bytes) >> 4);
      const int32_t srow = index ? index[i] : (int32_t)i;
      zero = srow < 0;
      if (!zero && src == nullptr) __trap();  // a live row behind a null src: caller bug
      sp = reinterpret_cast<const int4*>(src + (int64_t)(zero ? 0 : srow) * src_stride +
                                         m * full_row + hb * head_bytes);
      const int64_t drow = (int64_t)a.rank * a.rows_per_rank + i;
      dp = reinterpret_cast<int4*>(dst.p[j] + drow * dst_stride + (int64_t)m * sharded_mat);
    } else {
      // local row (j*R + i), own heads -> peer j shard row i at this rank's head offset
      const int hb = a.head_begin[a.rank];
      vpc = (int)(((a.head_begin[a.rank + 1] - hb) * head_bytes) >> 4);
      const int64_t srow = (int64_t)j * a.rows_per_rank + i;
      const int32_t drow = index ? index[(int64_t)j * a.rows_per_rank + i] : (int32_t)i;
      if (drow < 0) continue;  // pad row: dropped (warp-uniform)
      sp = reinterpret_cast<const int4*>(src + srow * src_stride + (int64_t)m * sharded_mat);
      dp = reinterpret_cast<int4*>(dst.p[j] + (int64_t)drow * dst_stride + m * full_row +
                                   hb * head_bytes);
    }
    for (int v0 = 0; v0 < vpc; v0 += 32 * kUnroll) {
      int4 val[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int v = v0 + u * 32 + lane;
        val[u] = make_int4(0, 0, 0, 0);
        if (v < vpc && !zero) val[u] = ld_stream(sp + v);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int v = v0 + u * 32 + lane;
        if (v < vpc) dp[v] = val[u];
      }
    }
  }
  // make the peer stores visible system-wide before the group barrier publishes
  __threadfence_system();
}

// TMA-staged path (default; FSP_A2A_TMA=0: the register kernel above): every chunk goes
// global -> shared -> peer memory
// through the bulk-copy (TMA) engine instead of register loads / stores.  One elected lane
// per warp runs a kStages-deep ring of chunk buffers: the load of chunk i+1 is in flight
// while chunk i's bulk store drains, and a buffer is reloaded only after the store that read
// it has finished reading (bulk wait_group.read).  Pad rows of a seq2head send are stored
// from a zeroed buffer (their zeros keep garbage out of the attention's masked PV products).
constexpr int kTmaWarps = 8;
constexpr int kTmaStages = 3;  // 8 KB x (1 + 8 warps x 3) = 200 KB of shared memory
constexpr int kTmaChunkMax = 8192;  // bytes of one (row, matrix, peer) head slice

template <bool kSeq2Head>
__global__ void __launch_bounds__(32 * kTmaWarps) a2a_tma_kernel(const uint8_t* __restrict__ src,
                                                                 PeerPtrs dst,
                                                                 const int32_t* __restrict__ index,
                                                                 FspA2A a) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* zero_buf = sm;  // kTmaChunkMax zero bytes shared by the CTA
  uint8_t* ring = sm + kTmaChunkMax + warp * kTmaStages * kTmaChunkMax;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kTmaChunkMax * (1 + kTmaWarps * kTmaStages)) +
                   warp * kTmaStages;
  for (uint32_t i = threadIdx.x; i < kTmaChunkMax / 16; i += blockDim.x)
    reinterpret_cast<int4*>(zero_buf)[i] = make_int4(0, 0, 0, 0);
  if (lane == 0)
    for (int st = 0; st < kTmaStages; ++st) mbar_init(bars + st, 1);
  fence_mbar_init();
  fence_async_smem();  // the zero buffer is read by the async proxy
  __syncthreads();
  if (lane != 0) return;
  const int d = a.degree;
  int hmax = 0;
  for (int jj = 0; jj < d; ++jj) hmax = max(hmax, a.head_begin[jj + 1] - a.head_begin[jj]);
  const int64_t head_bytes = (int64_t)a.head_dim * 2;
  const int64_t sharded_mat = hmax * head_bytes;
  const uint32_t n_chunks = (uint32_t)a.rows_per_rank * (uint32_t)a.n_mats * (uint32_t)d;
  const int64_t src_stride = a.src_stride * 2, dst_stride = a.dst_stride * 2;
  const int64_t full_row = (int64_t)a.n_heads * head_bytes;
  const uint32_t warps = gridDim.x * kTmaWarps;
  // chunk it -> (source, destination, bytes, zero?)
  auto decode = [&](uint32_t c, const uint8_t*& sp, uint8_t*& dp, uint32_t& bytes) -> int {
    const uint32_t j = c % d, rm = c / d, m = rm % a.n_mats, i = rm / a.n_mats;
    if (kSeq2Head) {
      const int hb = a.head_begin[j];
      bytes = (uint32_t)((a.head_begin[j + 1] - hb) * head_bytes);
      const int32_t srow = index ? index[i] : (int32_t)i;
      sp = srow < 0 ? nullptr : src + (int64_t)srow * src_stride + m * full_row + hb * head_bytes;
      dp = dst.p[j] + ((int64_t)a.rank * a.rows_per_rank + i) * dst_stride + (int64_t)m * sharded_mat;
      return srow < 0 ? 1 : 0;  // 1: zero row
    }
    const int hb = a.head_begin[a.rank];
    bytes = (uint32_t)((a.head_begin[a.rank + 1] - hb) * head_bytes);
    const int32_t drow = index ? index[(int64_t)j * a.rows_per_rank + i] : (int32_t)i;
    if (drow < 0) return 2;  // pad row: nothing to send
    sp = src + ((int64_t)j * a.rows_per_rank + i) * src_stride + (int64_t)m * sharded_mat;
    dp = dst.p[j] + (int64_t)drow * dst_stride + m * full_row + hb * head_bytes;
    return 0;
  };
  uint32_t it = 0;  // chunks loaded by this warp so far
  uint8_t* p_dp = nullptr;
  uint32_t p_bytes = 0;
  int p_kind = 2;
  for (uint32_t c = blockIdx.x * kTmaWarps + warp;; c += warps) {
    const bool more = c < n_chunks;
    const uint8_t* sp = nullptr;
    uint8_t* dp = nullptr;
    uint32_t bytes = 0;
    int kind = 2;
    if (more) {
      kind = decode(c, sp, dp, bytes);
      if (kind == 0) {
        const int st = it % kTmaStages;
        // the store that last read this buffer (chunk it - kTmaStages) must have read it
        if (it >= kTmaStages) bulk_wait_read<kTmaStages - 1>();
        mbar_expect_tx(bars + st, bytes);
        bulk_load(ring + st * kTmaChunkMax, sp, bytes, bars + st);
      }
    }
    // store the previous chunk (its load has had this chunk's issue time to land)
    if (p_kind == 0) {
      const uint32_t pit = it - 1, st = pit % kTmaStages;
      mbar_wait(bars + st, (pit / kTmaStages) & 1);
      bulk_store(p_dp, ring + st * kTmaChunkMax, p_bytes);
      bulk_commit();
    } else if (p_kind == 1) {
      bulk_store(p_dp, zero_buf, p_bytes);
      bulk_commit();
    }
    if (!more) break;
    if (kind == 0) ++it;
    p_dp = dp, p_bytes = bytes, p_kind = kind;
  }
  bulk_wait0();            // every bulk store of this warp has completed
  __threadfence_system();  // ... and is visible before the group barrier publishes
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Word of a rank's signal page where a timed-out barrier leaves its mark (the slots
// proper are [0, 2 * world) at most).
constexpr int kBarrierErrorWord = 1023;

__global__ void group_barrier_kernel(PeerPtrs sig, int degree, int rank, int slot_base,
                                     uint32_t epoch, uint64_t timeout_ns) {
  const int t = threadIdx.x;
  if (t < degree) {
    __threadfence_system();
    uint32_t* slot = reinterpret_cast<uint32_t*>(sig.p[t]) + slot_base + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(slot), "r"(epoch) : "memory");
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(sig.p[rank]) + slot_base + t;
    uint32_t seen;
    const uint64_t t0 = global_ns();
    uint32_t polls = 0;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(seen) : "l"(mine) : "memory");
      // Bounded spin: a peer that never arrives (it raised on the host, died, or its
      // stream is stuck) turns into a reported device fault instead of a hang that can
      // only be cleared by killing every process of the job.
      if ((int32_t)(seen - epoch) < 0 && timeout_ns && (++polls & 1023) == 0 &&
          global_ns() - t0 > timeout_ns) {
        reinterpret_cast<volatile uint32_t*>(sig.p[rank])[kBarrierErrorWord] =
            0xBA000000u | ((uint32_t)(slot_base + t) << 8) | (uint32_t)(slot_base + rank);
        printf("fsp_group_barrier: rank %d (slot base %d) timed out after %.1f s waiting for "
               "member %d at epoch %u (saw %u)\n",
               rank, slot_base, timeout_ns * 1e-9, t, epoch, seen);
        __trap();
      }
    } while ((int32_t)(seen - epoch) < 0);
  }
  __syncwarp();
}

// FSP_BARRIER_TIMEOUT_S (seconds, default 120; 0 = wait forever), read once per process.
uint64_t barrier_timeout_ns() {
  static const uint64_t ns = [] {
    const char* e = getenv("FSP_BARRIER_TIMEOUT_S");
    const double s = e ? atof(e) : 120.0;
    return s > 0 ? (uint64_t)(s * 1e9) : (uint64_t)0;
  }();
  return ns;
}

template <bool kSeq2Head>
int check_a2a(const FspA2A* a, const void* src, void* const* peer_dst, const int32_t* index) {
  FSP_CHECK_ARG(a && peer_dst, "null pointer argument");
  // src may be null only when nothing is read from it: no rows (an empty group), or a
  // seq2head send whose shard rows are all padding (a member of a tiny group holding no
  // tokens; its pack index is all -1, checked by fsp_layout_check on the host)
  FSP_CHECK_ARG(src || a->rows_per_rank == 0 || (kSeq2Head && index),
                "null src (allowed only for an empty exchange or an all-pad seq2head shard)");
  FSP_CHECK_ARG(a->degree >= 1 && a->degree <= kMaxDegree && (a->degree & (a->degree - 1)) == 0,
                "degree must be a power of two in [1, 8] (got %d)", a->degree);
  FSP_CHECK_ARG(a->rank >= 0 && a->rank < a->degree, "rank %d outside group of %d", a->rank,
                a->degree);
  FSP_CHECK_ARG(a->rows_per_rank >= 0 && a->n_mats >= 1 && a->head_dim >= 8 &&
                    a->head_dim % 8 == 0,
                "bad sizes");
  if (a->head_begin[a->degree] == 0) {
    FSP_CHECK_ARG(a->n_heads % a->degree == 0,
                  "n_heads (%d) not divisible by degree (%d) and no head_begin split given",
                  a->n_heads, a->degree);
  } else {
    FSP_CHECK_ARG(a->head_begin[0] == 0 && a->head_begin[a->degree] == a->n_heads,
                  "head_begin must run from 0 to n_heads");
    for (int j = 0; j < a->degree; ++j)
      FSP_CHECK_ARG(a->head_begin[j + 1] > a->head_begin[j], "member %d owns no heads", j);
  }
  FSP_CHECK_ARG(a->src_stride % 8 == 0 && a->dst_stride % 8 == 0, "strides must be multiples of 8");
  for (int j = 0; j < a->degree; ++j)
    FSP_CHECK_ARG(peer_dst[j] != nullptr && ((uintptr_t)peer_dst[j] & 15) == 0,
                  "peer_dst[%d] null or misaligned", j);
  return FSP_OK;
}

template <bool kSeq2Head>
int launch_a2a(const FspA2A* a, const void* src, void* const* peer_dst, const int32_t* index,
               void* stream) {
  int rc = check_a2a<kSeq2Head>(a, src, peer_dst, index);
  if (rc) return rc;
  FspA2A n = *a;  // normalised copy: the even split spelled out
  if (n.head_begin[n.degree] == 0)
    for (int j = 0; j <= n.degree; ++j) n.head_begin[j] = j * (n.n_heads / n.degree);
  for (int j = n.degree + 1; j <= kMaxDegree; ++j) n.head_begin[j] = n.n_heads;
  int hmax = 0;
  for (int j = 0; j < n.degree; ++j) hmax = std::max(hmax, n.head_begin[j + 1] - n.head_begin[j]);
  const int64_t full = (int64_t)n.n_heads * n.head_dim * n.n_mats;
  const int64_t slice = (int64_t)hmax * n.head_dim * n.n_mats;
  if (kSeq2Head)
    FSP_CHECK_ARG(n.src_stride >= full && n.dst_stride >= slice, "strides too small");
  else
    FSP_CHECK_ARG(n.src_stride >= slice && n.dst_stride >= full, "strides too small");
  PeerPtrs pp{};
  for (int j = 0; j < n.degree; ++j) pp.p[j] = reinterpret_cast<uint8_t*>(peer_dst[j]);
  const int64_t chunks = (int64_t)n.rows_per_rank * n.n_mats * n.degree;
  FSP_CHECK_ARG(chunks < (1ll << 32), "exchange too large");
  if (chunks == 0) return FSP_OK;
  // TMA bulk-copy path by default (666 vs 652 GB/s at d=2, 1 GB per rank;
  // profiles/r02_a2a_tma.md); FSP_A2A_TMA=0 selects the register-copy kernel
  static const bool use_tma = [] {
    const char* e = getenv("FSP_A2A_TMA");
    return !(e && e[0] == '0');
  }();
  if (use_tma && hmax * (int64_t)n.head_dim * 2 <= kTmaChunkMax) {
    const int smem = kTmaChunkMax * (1 + kTmaWarps * kTmaStages) + kTmaWarps * kTmaStages * 8;
    int64_t blocks = (chunks + kTmaWarps - 1) / kTmaWarps;
    if (blocks > 148) blocks = 148;  // one CTA (8 bulk-copy rings) per SM
    FSP_CUDA(cudaFuncSetAttribute(a2a_tma_kernel<kSeq2Head>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    a2a_tma_kernel<kSeq2Head><<<(unsigned)blocks, 32 * kTmaWarps, smem, (cudaStream_t)stream>>>(
        reinterpret_cast<const uint8_t*>(src), pp, index, n);
    FSP_LAUNCH_CHECK();
    return FSP_OK;
  }
  int64_t blocks = (chunks + kThreads / 32 - 1) / (kThreads / 32);
  if (blocks > 148 * 8) blocks = 148 * 8;
  a2a_kernel<kSeq2Head><<<(unsigned)blocks, kThreads, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const uint8_t*>(src), pp, index, n);
  FSP_LAUNCH_CHECK();
  return FSP_OK;
}

}  // namespace
}  // namespace fsp

extern "C" int fsp_a2a_seq2head(const FspA2A* a, const void* src, void* const* peer_dst,
                                const int32_t* d_src_index, void* stream) {
  return fsp::launch_a2a<true>(a, src, peer_dst, d_src_index, stream);
}

extern "C" int fsp_a2a_head2seq(const FspA2A* a, const void* src, void* const* peer_dst,
                                const int32_t* d_dst_index, void* stream) {
  return fsp::launch_a2a<false>(a, src, peer_dst, d_dst_index, stream);
}

extern "C" int fsp_group_barrier(uint32_t* const* peer_signal, int32_t degree, int32_t rank,
                                 int32_t slot_base, uint32_t epoch, void* stream) {
  using namespace fsp;
  FSP_CHECK_ARG(peer_signal != nullptr, "null peer_signal");
  FSP_CHECK_ARG(degree >= 1 && degree <= kMaxDegree, "degree out of range");
  FSP_CHECK_ARG(rank >= 0 && rank < degree, "rank out of range");
  FSP_CHECK_ARG(slot_base >= 0, "slot_base must be >= 0");
  if (degree == 1) return FSP_OK;
  PeerPtrs pp{};
  for (int j = 0; j < degree; ++j) {
    FSP_CHECK_ARG(peer_signal[j] != nullptr, "peer_signal[%d] null", j);
    pp.p[j] = reinterpret_cast<uint8_t*>(peer_signal[j]);
  }
  group_barrier_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(pp, degree, rank, slot_base, epoch,
                                                            barrier_timeout_ns());
  FSP_LAUNCH_CHECK();
  return FSP_OK;
}
