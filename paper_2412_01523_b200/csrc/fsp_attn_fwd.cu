// fsp_attn_fwd.cu — packed varlen causal attention forward on tcgen05/TMEM.
//
// Eq. (3) of the paper, P_h = softmax(Q_h K_h^T / sqrt(D)) V_h per head slice
// (PAPER.md:339), with flash-attn varlen semantics: every sequence of
// the cu_seqlens-packed group attends causally to itself only.
//
// One CTA = one 128-row query tile of one sequence x one head.  Warp roles:
//   warp 0      TMA producer: Q once, then K_j / V_j through a 2-stage ring
//   warp 1      MMA issuer (one elected lane): S_j = Q K_j^T (SS, both K-major SW128),
//               O += P_j V_j (TS: P from TMEM, V MN-major SW128)
//   warps 2..5  softmax: one thread per query row; S row from TMEM, online softmax
//               in exp2 domain, P (bf16) back to TMEM, lazy O rescale, epilogue.
// TMEM (512 cols): S0 [0,128) S1 [128,256) O [256,256+D) P0 [384,448) P1 [448,512).
// S is double-buffered so QK^T of tile j+1 overlaps the softmax of tile j.
#include <algorithm>
#include <type_traits>

#include "fsp_host.h"
#include "fsp_ptx.cuh"
#include "fsp_scatter.cuh"

namespace fsp {
namespace {

constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr int kFwdThreads = 192;
constexpr uint32_t kColS0 = 0, kColS1 = 128, kColO = 256, kColP0 = 384, kColP1 = 448;

struct FwdParams {
  __nv_bfloat16* o;
  float* lse;
  int64_t o_stride;
  const int32_t* cu_seqlens;
  const int32_t* seq_starts;  // optional: row of each sequence (else cu_seqlens)
  const int32_t* tiles;
  int32_t total_rows;
  int32_t n_heads;
  float scale_log2;
  int32_t n_tiles;  // schedule entries (the persistent pair kernel walks them)
  ScatterDev sc;  // fused head->seq of O (sc.degree == 0: off)
  int32_t noncausal;  // FSP_ATTN_NONCAUSAL: every query row sees every key row (pair kernel)
};

template <int D>
struct FwdSmem {
  static constexpr int kBoxes = D / 64;
  static constexpr int kTileBytes = 128 * D * 2;  // 128 rows x D bf16
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kTileBytes;
  static constexpr int kV = kK + 2 * kTileBytes;
  static constexpr int kBar = kV + 2 * kTileBytes;
  static constexpr int kBytes = kBar + 256;
};

template <int D>
__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ FwdParams p) {
  using L = FwdSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* bar_q = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2]
  uint64_t* s_free = bars + 11;  // [2]
  uint64_t* p_full = bars + 13;  // [2]
  uint64_t* pv_done = bars + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int tile = p.tiles[2 * blockIdx.x];
  const int head = p.tiles[2 * blockIdx.x + 1];
  const int seq = (int)((uint32_t)tile >> 16);  // unsigned: n_seq up to 65535
  const int qt = tile & 0xFFFF;
  const int seq_start = p.seq_starts ? p.seq_starts[seq] : p.cu_seqlens[seq];
  const int seqlen = p.cu_seqlens[seq + 1] - p.cu_seqlens[seq];
  const int q0 = qt * kBM;
  const int n_kv = qt + 1;  // causal: kv tiles 0..qt (kBM == kBN)

  if (threadIdx.x == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
      mbar_init(s_full + i, 1);
      mbar_init(s_free + i, 4);
      mbar_init(p_full + i, 4);
    }
    mbar_init(pv_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      mbar_expect_tx(bar_q, L::kTileBytes);
      for (int b = 0; b < L::kBoxes; ++b)
        tma_load_3d(smem + L::kQ + b * 16384, &tm_q, bar_q, b * 64, head, seq_start + q0);
      for (int j = 0; j < n_kv; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        const int row = seq_start + j * kBN;
        mbar_wait(k_empty + st, ph ^ 1);
        mbar_expect_tx(k_full + st, L::kTileBytes);
        for (int b = 0; b < L::kBoxes; ++b)
          tma_load_3d(smem + L::kK + st * L::kTileBytes + b * 16384, &tm_k, k_full + st, b * 64,
                      head, row);
        mbar_wait(v_empty + st, ph ^ 1);
        mbar_expect_tx(v_full + st, L::kTileBytes);
        for (int b = 0; b < L::kBoxes; ++b)
          tma_load_3d(smem + L::kV + st * L::kTileBytes + b * 16384, &tm_v, v_full + st, b * 64,
                      head, row);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc_s = make_idesc_bf16(kBM, kBN, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(kBM, D, false, true);
      const uint32_t q_base = smem_u32(smem + L::kQ);
      const uint32_t k_base = smem_u32(smem + L::kK);
      const uint32_t v_base = smem_u32(smem + L::kV);
      mbar_wait(bar_q, 0);
      tc_fence_after();
      auto issue_s = [&](int j) {
        const int st = j & 1;
        mbar_wait(k_full + st, (j >> 1) & 1);
        if (j >= 2) mbar_wait(s_free + st, ((j >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + (st ? kColS1 : kColS0);
        const uint32_t kb = k_base + st * L::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(d_tmem, make_sdesc_sw128(q_base + off, 16, 1024),
                 make_sdesc_sw128(kb + off, 16, 1024), idesc_s, kk > 0);
        }
        tc_commit(s_full + st);
        tc_commit(k_empty + st);
      };
      issue_s(0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) issue_s(j + 1);
        const int st = j & 1;
        mbar_wait(v_full + st, (j >> 1) & 1);
        mbar_wait(p_full + st, (j >> 1) & 1);
        tc_fence_after();
        const uint32_t vb = v_base + st * L::kTileBytes;
        const uint32_t p_tmem = tmem + (st ? kColP1 : kColP0);
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk)
          mma_ts(tmem + kColO, p_tmem + kk * 8, make_sdesc_sw128(vb + kk * 2048, 16384, 1024),
                 idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        tc_commit(pv_done);
        tc_commit(v_empty + st);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ softmax warps
    const uint32_t quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_addr = (quad * 32u) << 16;
    const int q_pos = q0 + row;
    const float sl2 = p.scale_log2;
    float m = -INFINITY;  // running max of scaled scores (log2 units)
    float l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      const int st = j & 1;
      mbar_wait(s_full + st, (j >> 1) & 1);
      tc_fence_after();
      float s[kBN];
#pragma unroll
      for (int c = 0; c < kBN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_addr + (st ? kColS1 : kColS0) + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c + i] = __uint_as_float(r[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free + st);

      if (j == n_kv - 1) {  // diagonal tile: causal mask
        const int lim = q_pos - j * kBN;
#pragma unroll
        for (int c = 0; c < kBN; ++c)
          if (c > lim) s[c] = -INFINITY;
      }
      float mx = s[0];
#pragma unroll
      for (int c = 1; c < kBN; ++c) mx = fmaxf(mx, s[c]);
      const float m_new = fmaxf(m, mx * sl2);
      const float corr = ex2(m - m_new);  // m = -inf on the first tile -> 0
      float sum = 0.f;
      uint32_t pk[kBN / 2];
#pragma unroll
      for (int c = 0; c < kBN; c += 2) {
        const float p0 = ex2(fmaf(s[c], sl2, -m_new));
        const float p1 = ex2(fmaf(s[c + 1], sl2, -m_new));
        sum += p0 + p1;
        pk[c / 2] = pack_bf16(p0, p1);
      }
      l = l * corr + sum;
      if (j > 0) {
        // O rescale needs PV_{j-1} retired; it also frees P buffer st (used by PV_{j-2}).
        mbar_wait(pv_done, (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, m_new > m)) {
#pragma unroll
          for (int c = 0; c < D; c += 32) {
            uint32_t r[32];
            tmem_ld32(tmem + lane_addr + kColO + c, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * corr);
            tmem_st32(tmem + lane_addr + kColO + c, r);
          }
        }
      }
      m = m_new;
      const uint32_t p_col = st ? kColP1 : kColP0;
#pragma unroll
      for (int c = 0; c < kBN / 2; c += 16) {
        uint32_t r[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = pk[c + i];
        tmem_st16(tmem + lane_addr + p_col + c, r);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full + st);
    }
    // ------------------------------------------------------------ epilogue
    mbar_wait(pv_done, (n_kv - 1) & 1);
    tc_fence_after();
    const float inv_l = 1.f / l;
    const bool valid = q_pos < seqlen;
    __nv_bfloat16* orow = p.o + (int64_t)(seq_start + q_pos) * p.o_stride + (int64_t)head * D;
    // fused head->seq (Eq. 4): the same row also goes to its owner's sequence shard
    __nv_bfloat16* prow = valid ? scatter_row(p.sc, seq_start + q_pos, 0, head, D) : nullptr;
#pragma unroll
    for (int c = 0; c < D; c += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_addr + kColO + c, r);
      tmem_ld_wait();
      if (valid) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 v;
          v.x = pack_bf16(__uint_as_float(r[i + 0]) * inv_l, __uint_as_float(r[i + 1]) * inv_l);
          v.y = pack_bf16(__uint_as_float(r[i + 2]) * inv_l, __uint_as_float(r[i + 3]) * inv_l);
          v.z = pack_bf16(__uint_as_float(r[i + 4]) * inv_l, __uint_as_float(r[i + 5]) * inv_l);
          v.w = pack_bf16(__uint_as_float(r[i + 6]) * inv_l, __uint_as_float(r[i + 7]) * inv_l);
          *reinterpret_cast<uint4*>(orow + c + i) = v;
          if (prow) *reinterpret_cast<uint4*>(prow + c + i) = v;
        }
      }
    }
    if (valid)
      p.lse[(int64_t)head * p.total_rows + seq_start + q_pos] =
          (m + __log2f(l)) * 0.69314718055994531f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<512>(tmem);
}

// ============================================================================ paired (D = 128)
// One CTA = two consecutive 128-row query tiles A, B (256 rows) of one sequence x head
// sharing every K_j / V_j load.  Two softmax warpgroups (one per tile) alternate with
// the tensor core:
//   MMA:  S_A(0) S_B(0) | PV_A(0) S_A(1) PV_B(0) S_B(1) | PV_A(1) S_A(2) ...
// so QK^T / PV of one tile run while the other tile's softmax executes.  P_X is written
// as bf16 over the first 64 columns of S_X (the S_X(j+1) MMA is issued after PV_X(j) and
// tcgen05 MMAs execute in issue order).  s_full_X(j) is committed after PV_X(j-1), so a
// softmax warpgroup may rescale O_X in place when it sees S_X(j).
// Rescaling is lazy: the exponent base m only moves when the running max grows by more
// than 8 (factor 256), which keeps P <= 256 and makes O rescales rare.
// A quarter of the exponentials run as a degree-3 polynomial on the FMA pipe (the
// 16/clk/SM MUFU.EX2 rate would otherwise equal the tensor-core time per tile).
// TMEM: S_A|P_A [0,128) S_B|P_B [128,256) O_A [256,384) O_B [384,512).
// FSP_FWD_WG3: three warpgroups (TMA + MMA warps and two idle warps | softmax A | softmax B)
// so setmaxnreg can move registers from the first to the softmax warpgroups, which then
// hold a whole 128-column S row and read it from TMEM once per tile.
#ifndef FSP_FWD_WG3
#define FSP_FWD_WG3 1
#endif
constexpr int kF2Threads = FSP_FWD_WG3 ? 128 + 256 : 64 + 256;
constexpr int kF2SoftmaxWarp0 = FSP_FWD_WG3 ? 4 : 2;
#ifndef FSP_ABLATE_EXP
#define FSP_ABLATE_EXP 0
#endif
// one exponential pair in FSP_POLY_EVERY runs as a polynomial on the FMA pipe (0 = none)
#ifndef FSP_FWD_PREFETCH
#define FSP_FWD_PREFETCH 1  // 1: TMEM load of the next 32-column chunk overlaps this chunk's math
#endif
#if FSP_FWD_WG3  // the row is loaded whole: no chunk prefetch
#undef FSP_FWD_PREFETCH
#define FSP_FWD_PREFETCH 0
#endif
#ifndef FSP_POLY_EVERY
#define FSP_POLY_EVERY 4
#endif

struct Fwd2Smem {
  static constexpr int kTileBytes = 128 * 128 * 2;
  static constexpr int kQA = 0;
  static constexpr int kQB = kTileBytes;
  static constexpr int kKStages = 3;  // K runs a stage ahead of V (S needs K_{j+1} first)
  static constexpr int kK = 2 * kTileBytes;
  static constexpr int kV = kK + kKStages * kTileBytes;  // 2 stages
  static constexpr int kBar = kV + 2 * kTileBytes;
  static constexpr int kBytes = kBar + 256;
};

// 2^x on the FMA pipe (x <= 0, finite): round-to-nearest split via the 1.5*2^23 magic
// number, minimax cubic for 2^f on [-0.5, 0.5] (max rel. error 7.5e-5), exponent add.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float y = x + 12582912.f;
  const float xi = y - 12582912.f;
  const float f = x - xi;
  float pf = fmaf(0.05517025f, f, 0.2426079f);
  pf = fmaf(pf, f, 0.69326093f);
  pf = fmaf(pf, f, 0.99992828f);
  return __int_as_float(__float_as_int(pf) + (__float_as_int(y) << 23));
}

#ifndef FSP_FWD_TIMING
#define FSP_FWD_TIMING 0  // profiling build: cycles the MMA issuer / softmax warps spend waiting
#endif
#if FSP_FWD_TIMING
__device__ unsigned long long g_fwd_wait[16];
__device__ unsigned int g_fwd_done;
#define FSP_FTW(slot, call)                              \
  do {                                                   \
    const long long t0_ = clock64();                     \
    call;                                                \
    tw[slot] += clock64() - t0_;                         \
  } while (0)
#else
#define FSP_FTW(slot, call) call
#endif

// One schedule entry of the pair kernel: query rows [q0, q0 + 256) of one sequence x head.
struct PairTile {
  int head, seq_start, seqlen, q0, n_a, n_b, n_kv;
  bool has_b;
};

__device__ __forceinline__ PairTile decode_pair(const FwdParams& p, int w) {
  PairTile t;
  const int tile = p.tiles[2 * w];
  t.head = p.tiles[2 * w + 1];
  const int seq = (int)((uint32_t)tile >> 16);  // unsigned: n_seq up to 65535
  const int pair = tile & 0xFFFF;
  t.seq_start = p.seq_starts ? p.seq_starts[seq] : p.cu_seqlens[seq];
  t.seqlen = p.cu_seqlens[seq + 1] - p.cu_seqlens[seq];
  t.q0 = pair * 256;
  t.has_b = t.q0 + 128 < t.seqlen;
  if (p.noncausal) {  // every kv tile of the sequence, for both tiles
    const int nkv = (t.seqlen + 127) / 128;
    t.n_a = nkv;
    t.n_b = t.has_b ? nkv : 0;
    t.n_kv = nkv;
    return t;
  }
  t.n_a = 2 * pair + 1;                   // kv tiles seen by tile A (causal)
  t.n_b = t.has_b ? 2 * pair + 2 : 0;     // ... by tile B
  t.n_kv = t.has_b ? t.n_b : t.n_a;
  return t;
}

// Dynamic schedule of the persistent pair kernel (cluster launch control): the grid still
// has one CTA per schedule entry, but a CTA that finishes an entry cancels the next
// not-yet-launched CTA (hardware launch order = the longest-first schedule order) and runs
// its entry itself — the hardware's "next CTA to the first free SM" without the per-CTA
// prologue / epilogue.  The TMA producer steals and hands each entry to the MMA and softmax
// warps through a two-slot ring in shared memory.
struct EntryRing {
  int* idx;         // [2] claimed schedule entries
  uint64_t* full;   // [2] producer -> consumers
  uint64_t* empty;  // [2] consumers (MMA thread + 8 softmax warps) -> producer
  void* resp;       // 16-byte cluster-launch-control response
  uint64_t* clc;    // its completion barrier
};
constexpr int kRingConsumers = 9;

// Producer side: the k-th entry of this CTA (its own first, then stolen ones).
template <bool kPersistent>
__device__ __forceinline__ int claim_entry(const EntryRing& r, int k) {
  if (!kPersistent) return k == 0 ? (int)blockIdx.x : INT_MAX;
  const int slot = k & 1;
  mbar_wait(r.empty + slot, ((k >> 1) & 1) ^ 1);
  int w = (int)blockIdx.x;
  if (k > 0) {
    w = clc_steal(r.resp, r.clc, (k - 1) & 1);
    if (w < 0) w = INT_MAX;
  }
  r.idx[slot] = w;
  mbar_arrive(r.full + slot);
  return w;
}

// Consumer side: either every lane of a softmax warp (kWarp: lane 0 releases the slot
// after the warp has read it) or the single elected MMA-issuer thread.
template <bool kPersistent, bool kWarp>
__device__ __forceinline__ int take_entry(const EntryRing& r, int k) {
  if (!kPersistent) return k == 0 ? (int)blockIdx.x : INT_MAX;
  const int slot = k & 1;
  mbar_wait(r.full + slot, (k >> 1) & 1);
  const int w = r.idx[slot];
  if (kWarp) {
    __syncwarp();
    if (lane_id() == 0) mbar_arrive(r.empty + slot);
  } else {
    mbar_arrive(r.empty + slot);
  }
  return w;
}

template <bool kPersistent>
__global__ void __launch_bounds__(kF2Threads, 1)
    attn_fwd_pair_kernel(const __grid_constant__ CUtensorMap tm_q,
                         const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ FwdParams p) {
  constexpr int D = 128;
  using L = Fwd2Smem;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* bar_q = bars + 0;
  uint64_t* k_full = bars + 1;   // [3]
  uint64_t* k_empty = bars + 4;  // [3]
  uint64_t* v_full = bars + 7;   // [2]
  uint64_t* v_empty = bars + 9;  // [2]
  uint64_t* s_full = bars + 11;  // [2] per tile
  uint64_t* o_done = bars + 13;  // [2] per tile
  uint64_t* p_half = bars + 15;  // [2 tiles][2 halves]: P columns for kv rows 0-63 / 64-127
  uint64_t* q_empty = bars + 19; // Q_A / Q_B read by the last QK^T of a schedule entry
  const EntryRing ring{reinterpret_cast<int*>(bars + 24), bars + 20, bars + 22, bars + 26,
                       bars + 25};
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 28);
  // [2] per tile: its 4 softmax warps have read back the O rows they staged in that tile's
  // Q buffer (fused head->seq epilogue), so the producer may load the next entry's Q there
  uint64_t* epi_free = bars + 29;

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  // Barrier phases run on across the schedule entries of a persistent CTA: every counter
  // below is a running count of completions, so a wait's parity is (count & 1).

  if (threadIdx.x == 0) {
    mbar_init(q_empty, 1);
    mbar_init(epi_free + 0, 4);
    mbar_init(epi_free + 1, 4);
    for (int i = 0; i < 2; ++i) {
      mbar_init(ring.full + i, 1);
      mbar_init(ring.empty + i, kRingConsumers);
    }
    mbar_init(ring.clc, 1);
    mbar_init(bar_q, 1);
    for (int i = 0; i < L::kKStages; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
      mbar_init(s_full + i, 1);
      mbar_init(p_half + 2 * i, 4);
      mbar_init(p_half + 2 * i + 1, 4);
      mbar_init(o_done + i, 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Register reallocation is per warpgroup, so the role branches split at warpgroup
  // granularity first (FSP_FWD_WG3: 128 x 56 + 256 x 208 of the 65,536 registers).
  if (warp < kF2SoftmaxWarp0) {
#if FSP_FWD_WG3
    setmaxnreg_dec<56>();
#endif
    if (warp == 0) {
      // ------------------------------------------------------------ TMA producer
      if (elect_one()) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        uint32_t g0 = 0;  // K/V ring position: kv steps issued by this CTA so far
        uint32_t n_b = 0;        // entries with a tile B so far
        bool prev_b = false;     // the previous entry had a tile B
        for (int k = 0;; ++k) {
          const int w = claim_entry<kPersistent>(ring, k);
          if (w >= p.n_tiles) break;
          const PairTile T = decode_pair(p, w);
          const bool wait_b = prev_b;
          const uint32_t b_phase = (n_b - 1) & 1;
          prev_b = T.has_b;
          n_b += T.has_b ? 1u : 0u;
          if (k > 0) {
            // Q rows of an entry are read by this CTA only: warm L2 while the previous entry
            // finishes, and K_0 / V_0 with them
            for (int b = 0; b < 2; ++b) {
              tma_prefetch_l2_3d(&tm_q, b * 64, T.head, T.seq_start + T.q0);
              if (T.has_b) tma_prefetch_l2_3d(&tm_q, b * 64, T.head, T.seq_start + T.q0 + 128);
              tma_prefetch_l2_3d(&tm_k, b * 64, T.head, T.seq_start);
              tma_prefetch_l2_3d(&tm_v, b * 64, T.head, T.seq_start);
            }
            mbar_wait(q_empty, (k - 1) & 1);  // previous entry's QK^T MMAs are done
            if (p.sc.degree) {
              // fused head->seq: the previous entry's epilogue stages O in the Q buffers
              mbar_wait(epi_free + 0, (k - 1) & 1);
              if (wait_b) mbar_wait(epi_free + 1, b_phase);
            }
          }
          mbar_expect_tx(bar_q, (T.has_b ? 2 : 1) * L::kTileBytes);
          for (int b = 0; b < 2; ++b) {
            tma_load_3d(smem + L::kQA + b * 16384, &tm_q, bar_q, b * 64, T.head, T.seq_start + T.q0);
            if (T.has_b)
              tma_load_3d(smem + L::kQB + b * 16384, &tm_q, bar_q, b * 64, T.head,
                          T.seq_start + T.q0 + 128);
          }
          // issue order K_0, K_1, V_0, K_2, V_1, ...: K is consumed one step before V
          auto load_k = [&](int j) {
            const uint32_t g = g0 + j;
            const int st = g % L::kKStages;
            mbar_wait(k_empty + st, ((g / L::kKStages) & 1) ^ 1);
            mbar_expect_tx(k_full + st, L::kTileBytes);
            for (int b = 0; b < 2; ++b)
              tma_load_3d(smem + L::kK + st * L::kTileBytes + b * 16384, &tm_k, k_full + st, b * 64,
                          T.head, T.seq_start + j * 128);
          };
          load_k(0);
          for (int j = 0; j < T.n_kv; ++j) {
            if (j + 1 < T.n_kv) load_k(j + 1);
            const uint32_t g = g0 + j;
            const int st = g & 1;
            mbar_wait(v_empty + st, ((g >> 1) & 1) ^ 1);
            mbar_expect_tx(v_full + st, L::kTileBytes);
            for (int b = 0; b < 2; ++b)
              tma_load_3d(smem + L::kV + st * L::kTileBytes + b * 16384, &tm_v, v_full + st, b * 64,
                          T.head, T.seq_start + j * 128);
          }
          g0 += T.n_kv;
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      // ------------------------------------------------------------ MMA issuer
      if (elect_one()) {
        constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
        constexpr uint32_t idesc_o = make_idesc_bf16(128, D, false, true);
        const uint32_t qa = smem_u32(smem + L::kQA), qb = smem_u32(smem + L::kQB);
        const uint32_t k_base = smem_u32(smem + L::kK);
        const uint32_t v_base = smem_u32(smem + L::kV);
#if FSP_FWD_TIMING
        long long tw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const long long t_start = clock64();
#endif
        uint32_t g0 = 0;                 // K/V ring position (kv steps consumed so far)
        uint32_t p_cnt[2] = {0u, 0u};    // p_half completions consumed per tile x
        int steps = 0;
        for (int k = 0;; ++k) {
          const int w = take_entry<kPersistent, false>(ring, k);
          if (w >= p.n_tiles) break;
          const PairTile T = decode_pair(p, w);
          const int n_a = T.n_a, n_b = T.n_b, n_kv = T.n_kv;
          int qk_left = n_a + n_b;  // QK^T groups still to issue; the last one frees Q_A / Q_B
          FSP_FTW(5, mbar_wait(bar_q, k & 1));
          auto qk = [&](int x, int j) {  // S_x = Q_x K_j^T
            const uint32_t qbase = x ? qb : qa;
            const uint32_t kb = k_base + ((g0 + j) % L::kKStages) * L::kTileBytes;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
              mma_ss(tmem + x * 128, make_sdesc_sw128(qbase + off, 16, 1024),
                     make_sdesc_sw128(kb + off, 16, 1024), idesc_s, kk > 0);
            }
            tc_commit(s_full + x);
            if (--qk_left == 0) tc_commit(q_empty);
          };
          auto pv = [&](int x, int j) {  // O_x += P_x V_j, each half as soon as its P lands
            const uint32_t vb = v_base + ((g0 + j) & 1) * L::kTileBytes;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              FSP_FTW(x, mbar_wait(p_half + 2 * x + hh, (p_cnt[x] + j) & 1));
              tc_fence_after();
#pragma unroll
              for (int kk = 4 * hh; kk < 4 * hh + 4; ++kk)
                mma_ts(tmem + 256 + x * 128, tmem + x * 128 + kk * 8,
                       make_sdesc_sw128(vb + kk * 2048, 16384, 1024), idesc_o,
                       (j > 0 || kk > 0) ? 1u : 0u);
            }
          };
          auto wait_k = [&](int j) {
            const uint32_t g = g0 + j;
            FSP_FTW(2, mbar_wait(k_full + g % L::kKStages, (g / L::kKStages) & 1));
            tc_fence_after();
          };
          wait_k(0);
          qk(0, 0);
          if (n_b > 0) qk(1, 0);
          tc_commit(k_empty + g0 % L::kKStages);
          for (int j = 0; j < n_kv; ++j) {
            const uint32_t g = g0 + j;
            const int st = g & 1;
            const bool next = j + 1 < n_kv;
            FSP_FTW(3, mbar_wait(v_full + st, (g >> 1) & 1));
            if (j < n_a) {
              pv(0, j);
              if (j + 1 < n_a) {
                wait_k(j + 1);
                qk(0, j + 1);
              } else {
                tc_commit(o_done + 0);
              }
            }
            if (j < n_b) {
              pv(1, j);
              if (j + 1 < n_b) {
                wait_k(j + 1);
                qk(1, j + 1);
              } else {
                tc_commit(o_done + 1);
              }
            }
            tc_commit(v_empty + st);
            if (next) tc_commit(k_empty + (g + 1) % L::kKStages);
          }
          p_cnt[0] += n_a;
          p_cnt[1] += n_b;
          g0 += n_kv;
          steps += n_a + n_b;
        }
#if FSP_FWD_TIMING
        tw[7] = clock64() - t_start;
        for (int i = 0; i < 8; ++i) atomicAdd(&g_fwd_wait[i], (unsigned long long)tw[i]);
        atomicAdd(&g_fwd_wait[8], (unsigned long long)steps);
        __threadfence();
        // persistent launches: only the first ~148 CTAs run (the rest are cancelled by CLC)
        if (atomicAdd(&g_fwd_done, 1u) == (kPersistent ? min(gridDim.x, 148u) : gridDim.x) - 1) {
          printf("fwd MMA issuer cycles (sum over CTAs): tile-steps %llu total %llu | p_half A %llu "
                 "p_half B %llu k_full %llu v_full %llu q %llu\n", g_fwd_wait[8], g_fwd_wait[7],
                 g_fwd_wait[0], g_fwd_wait[1], g_fwd_wait[2], g_fwd_wait[3], g_fwd_wait[5]);
          printf("fwd softmax warp (tile A, quad 0): s_full wait %llu busy %llu | to max %llu to "
                 "first-half release %llu\n", g_fwd_wait[9], g_fwd_wait[10], g_fwd_wait[11],
                 g_fwd_wait[12]);
          for (int i = 0; i < 16; ++i) g_fwd_wait[i] = 0;
          g_fwd_done = 0;
        }
#endif
      }
      __syncwarp();
    }
  } else {
#if FSP_FWD_WG3
    setmaxnreg_inc<208>();
#endif
    // ------------------------------------------------------------ softmax warpgroups
    const int x = (warp - kF2SoftmaxWarp0) >> 2;  // 0 -> tile A, 1 -> tile B
    const uint32_t quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_addr = (quad * 32u) << 16;
    const uint32_t s_col = x * 128, o_col = 256 + x * 128;
    const float sl2 = p.scale_log2;
    uint32_t s_cnt = 0, o_cnt = 0;  // s_full / o_done completions this tile x consumed
    for (int k = 0;; ++k) {
    const int w = take_entry<kPersistent, true>(ring, k);
    if (w >= p.n_tiles) break;
    const PairTile T = decode_pair(p, w);
    const int head = T.head, seq_start = T.seq_start, seqlen = T.seqlen, q0 = T.q0;
    const int n_x = x ? T.n_b : T.n_a;
    if (n_x == 0) continue;  // no tile B in this entry
    const int q_pos = q0 + x * 128 + row;
    float m = -INFINITY;  // exponent base (scaled, log2 units)
    float l = 0.f;
    for (int j = 0; j < n_x; ++j) {
#if FSP_FWD_TIMING
      const long long ts0 = clock64();
#endif
      mbar_wait(s_full + x, (s_cnt + j) & 1);
#if FSP_FWD_TIMING
      const long long ts1 = clock64();
      if (warp == kF2SoftmaxWarp0 && lane == 0) atomicAdd(&g_fwd_wait[9], (unsigned long long)(ts1 - ts0));
#endif
      tc_fence_after();
      if (FSP_ABLATE_EXP >= 2) {  // profiling ablations: 2 = no softmax work,
        // 3 = two passes of TMEM loads + P store, 4 = one pass of loads + P store
        if (FSP_ABLATE_EXP >= 3) {
          uint32_t acc = 0;
#pragma unroll
          for (int pass = 0; pass < (FSP_ABLATE_EXP == 3 ? 2 : 1); ++pass)
#pragma unroll
            for (int c = 0; c < 128; c += 32) {
              uint32_t r[32];
              tmem_ld32(tmem + lane_addr + s_col + c, r);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) acc ^= r[i];
            }
#pragma unroll
          for (int c = 0; c < 64; c += 16) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = acc + i;
            tmem_st16(tmem + lane_addr + s_col + c, pk);
          }
          tmem_st_wait();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(p_half + 2 * x);
          mbar_arrive(p_half + 2 * x + 1);
        }
        continue;
      }
      // The diagonal tile (causal mask) and the interior tiles get separate straight-line
      // code: per-pair masking branches would serialise the MUFU / FFMA2 streams.
      // column c of the last kv tile is valid iff c <= lim: causal, the diagonal tile
      // (key row <= query row); non-causal, the sequence's last key row
      const int lim = p.noncausal ? seqlen - 1 - j * 128 : q_pos - j * 128;
      auto tile_body = [&](auto diag_c) {
        constexpr bool kDiag = decltype(diag_c)::value;
        // Masking mode of each 32-column chunk of the last kv tile, warp-uniform: 0 = every
        // lane's columns valid, 2 = every lane's columns masked, 1 = mixed (per-element
        // selects).  On the causal diagonal a warp's 32 rows need per-element masks in one
        // chunk only (rows 32q.. see columns <= row): the other chunks take the unmasked
        // code or are skipped, instead of ~900 compare / select / predicate-shuffle
        // instructions per row for the whole tile.
        int cmode[4] = {0, 0, 0, 0};
        if (kDiag) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            cmode[c] = __all_sync(0xffffffffu, 32 * c + 31 <= lim) ? 0
                       : __all_sync(0xffffffffu, 32 * c > lim)     ? 2
                                                                   : 1;
        }
        // pass 1: row max; four independent FMNMX3 chains over chunked TMEM loads (the
        // whole 128-column row does not fit the 168-register budget of 10 warps per CTA)
        float mxs[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#if FSP_FWD_WG3
        uint32_t sr[4][32];  // the whole S row, one TMEM round trip per tile
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tmem + lane_addr + s_col + 32 * c, sr[c]);
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_wait_tied(sr[c]);
#elif FSP_FWD_PREFETCH
        uint32_t buf[2][32];  // chunk c+1 is in flight while chunk c is processed
        tmem_ld32(tmem + lane_addr + s_col, buf[0]);
        tmem_ld_wait_tied(buf[0]);
#endif
#pragma unroll
        for (int c = 0; c < 128; c += 32) {
#if FSP_FWD_WG3
          uint32_t(&r)[32] = sr[c / 32];
#elif FSP_FWD_PREFETCH
          uint32_t(&r)[32] = buf[(c / 32) & 1];
          if (c + 32 < 128) tmem_ld32(tmem + lane_addr + s_col + c + 32, buf[((c / 32) + 1) & 1]);
#else
          uint32_t r[32];
          tmem_ld32(tmem + lane_addr + s_col + c, r);
          tmem_ld_wait();
#endif
          if (!kDiag || cmode[c / 32] == 0) {
#pragma unroll
            for (int i = 0; i < 32; i += 8)
#pragma unroll
              for (int a = 0; a < 4; ++a)
                mxs[a] = fmax3(mxs[a], __uint_as_float(r[i + 2 * a]), __uint_as_float(r[i + 2 * a + 1]));
          } else if (cmode[c / 32] == 1) {
#pragma unroll
            for (int i = 0; i < 32; i += 8)
#pragma unroll
              for (int a = 0; a < 4; ++a) {
                float v0 = __uint_as_float(r[i + 2 * a]), v1 = __uint_as_float(r[i + 2 * a + 1]);
                v0 = c + i + 2 * a <= lim ? v0 : -INFINITY;
                v1 = c + i + 2 * a + 1 <= lim ? v1 : -INFINITY;
                mxs[a] = fmax3(mxs[a], v0, v1);
              }
          }
#if FSP_FWD_PREFETCH
          if (c + 32 < 128) tmem_ld_wait_tied(buf[((c / 32) + 1) & 1]);
#endif
        }
        const float mx = fmaxf(fmaxf(mxs[0], mxs[1]), fmaxf(mxs[2], mxs[3]));
#if FSP_FWD_TIMING
        if (warp == kF2SoftmaxWarp0 && lane == 0) atomicAdd(&g_fwd_wait[11], (unsigned long long)(clock64() - ts1));
#endif
        const float m_new = fmaxf(m, mx * sl2);
        // warp-uniform lazy rescale decision (TMEM access is warp-collective)
        const bool grow = __any_sync(0xffffffffu, m_new > m + 8.f);
        float corr = 1.f;
        if (grow) {
          corr = ex2(m - m_new);  // 0 on the first tile (m = -inf)
          if (j > 0) {
#pragma unroll
            for (int c = 0; c < D; c += 32) {
              uint32_t r[32];
              tmem_ld32(tmem + lane_addr + o_col + c, r);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * corr);
              tmem_st32(tmem + lane_addr + o_col + c, r);
            }
          }
          m = m_new;
        }
        // pass 2: reload each 32-column chunk, exponentiate, write P (bf16 pairs) back over
        // S columns [c/2, c/2+16) — all of which this thread has already consumed.
        // Packed fp32x2 math; one pair in four exponentiates on the FMA pipe (ex2_poly2).
        const uint64_t sl2x2 = f2(sl2, sl2), negm2 = f2(-m, -m);
        uint64_t sum2[4] = {f2(0.f, 0.f), f2(0.f, 0.f), f2(0.f, 0.f), f2(0.f, 0.f)};
#if FSP_FWD_PREFETCH
        tmem_ld32(tmem + lane_addr + s_col, buf[0]);
        tmem_ld_wait_tied(buf[0]);
#endif
#pragma unroll
        for (int c = 0; c < 128; c += 32) {
          uint32_t pk[16];
#if FSP_FWD_WG3
          uint32_t(&r)[32] = sr[c / 32];
#elif FSP_FWD_PREFETCH
          uint32_t(&r)[32] = buf[(c / 32) & 1];
          if (c + 32 < 128) tmem_ld32(tmem + lane_addr + s_col + c + 32, buf[((c / 32) + 1) & 1]);
#else
          uint32_t r[32];
          tmem_ld32(tmem + lane_addr + s_col + c, r);
          tmem_ld_wait();
#endif
          const int mode = kDiag ? cmode[c / 32] : 0;
          if (mode == 2) {  // every column of the chunk masked: P = 0
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = 0u;
          } else {
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const uint64_t x2 =
                  ffma2(f2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sl2x2, negm2);
              float p0, p1;
              if (mode == 1) {
                float x0, x1;
                f2_split(x2, x0, x1);
                p0 = ex2(c + i <= lim ? x0 : -INFINITY);
                p1 = ex2(c + i + 1 <= lim ? x1 : -INFINITY);
              } else if (FSP_ABLATE_EXP) {  // profiling ablation: no exponentials
                f2_split(x2, p0, p1);
              } else if (FSP_POLY_EVERY > 0 && (i / 2) % FSP_POLY_EVERY == FSP_POLY_EVERY - 1) {
                ex2_poly2(x2, p0, p1);
              } else {
                float x0, x1;
                f2_split(x2, x0, x1);
                p0 = ex2(x0);
                p1 = ex2(x1);
              }
              sum2[(i >> 1) & 3] = fadd2(sum2[(i >> 1) & 3], f2(p0, p1));
              pk[i / 2] = pack_bf16(p0, p1);
            }
          }
          tmem_st16(tmem + lane_addr + s_col + c / 2, pk);
          if (c == 32) {  // P for kv rows 0..63 is in TMEM: release the first PV half
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_half + 2 * x);
#if FSP_FWD_TIMING
            if (warp == kF2SoftmaxWarp0 && lane == 0)
              atomicAdd(&g_fwd_wait[12], (unsigned long long)(clock64() - ts1));
#endif
          }
#if FSP_FWD_PREFETCH
          if (c + 32 < 128) tmem_ld_wait_tied(buf[((c / 32) + 1) & 1]);
#endif
        }
        float sum_lo, sum_hi;
        f2_split(fadd2(fadd2(sum2[0], sum2[1]), fadd2(sum2[2], sum2[3])), sum_lo, sum_hi);
        l = l * corr + (sum_lo + sum_hi);
      };
      if (j == n_x - 1)
        tile_body(std::true_type{});
      else
        tile_body(std::false_type{});
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_half + 2 * x + 1);
#if FSP_FWD_TIMING
      if (warp == kF2SoftmaxWarp0 && lane == 0) atomicAdd(&g_fwd_wait[10], (unsigned long long)(clock64() - ts1));
#endif
    }
    s_cnt += n_x;
    // ------------------------------------------------------------ epilogue
    {
      mbar_wait(o_done + x, o_cnt & 1);
      ++o_cnt;
      tc_fence_after();
      const float inv_l = 1.f / l;
      const bool valid = q_pos < seqlen;
      // (the staged path borrows this entry's Q buffer; a persistent CTA's producer waits on
      // epi_free before refilling it for the next entry)
      if (p.sc.degree) {
        // Fused head->seq (Eq. 4): O goes to its owner's sequence shard over NVLink as well
        // as to the local buffer.  One-row-per-thread 16-byte stores would cross NVLink as
        // 32 scattered 16-byte packets per warp instruction, so the warp first stages its
        // 32 rows in shared memory (this tile's Q buffer, idle once o_done has fired; 16-byte
        // chunks XOR-swizzled by row) and then writes two full 256-byte rows per instruction.
        uint8_t* stage = smem + (x ? L::kQB : L::kQA);
#pragma unroll
        for (int c = 0; c < D; c += 32) {
          uint32_t r[32];
          tmem_ld32(tmem + lane_addr + o_col + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(r[i + 0]) * inv_l, __uint_as_float(r[i + 1]) * inv_l);
            v.y = pack_bf16(__uint_as_float(r[i + 2]) * inv_l, __uint_as_float(r[i + 3]) * inv_l);
            v.z = pack_bf16(__uint_as_float(r[i + 4]) * inv_l, __uint_as_float(r[i + 5]) * inv_l);
            v.w = pack_bf16(__uint_as_float(r[i + 6]) * inv_l, __uint_as_float(r[i + 7]) * inv_l);
            const int chunk = ((c + i) >> 3) ^ (row & 15);
            *reinterpret_cast<uint4*>(stage + row * 256 + chunk * 16) = v;
          }
        }
        __syncwarp();
        const int chunk = lane & 15;
#pragma unroll 4
        for (int rr = 0; rr < 32; rr += 2) {
          const int srow = quad * 32 + rr + (lane >> 4);  // tile row
          const int qp = q0 + x * 128 + srow;
          if (qp >= seqlen) continue;
          const uint4 v = *reinterpret_cast<const uint4*>(stage + srow * 256 +
                                                          ((chunk ^ (srow & 15)) * 16));
          const int64_t t = seq_start + qp;
          *reinterpret_cast<uint4*>(p.o + t * p.o_stride + (int64_t)head * D + chunk * 8) = v;
          __nv_bfloat16* prow = scatter_row(p.sc, t, 0, head, D);
          if (prow) *reinterpret_cast<uint4*>(prow + chunk * 8) = v;
        }
        __syncwarp();  // every lane's staged reads are done
        if (lane == 0) mbar_arrive(epi_free + x);
      } else {
        __nv_bfloat16* orow =
            p.o + (int64_t)(seq_start + q_pos) * p.o_stride + (int64_t)head * D;
#pragma unroll
        for (int c = 0; c < D; c += 32) {
          uint32_t r[32];
          tmem_ld32(tmem + lane_addr + o_col + c, r);
          tmem_ld_wait();
          if (valid) {
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              uint4 v;
              v.x = pack_bf16(__uint_as_float(r[i + 0]) * inv_l, __uint_as_float(r[i + 1]) * inv_l);
              v.y = pack_bf16(__uint_as_float(r[i + 2]) * inv_l, __uint_as_float(r[i + 3]) * inv_l);
              v.z = pack_bf16(__uint_as_float(r[i + 4]) * inv_l, __uint_as_float(r[i + 5]) * inv_l);
              v.w = pack_bf16(__uint_as_float(r[i + 6]) * inv_l, __uint_as_float(r[i + 7]) * inv_l);
              *reinterpret_cast<uint4*>(orow + c + i) = v;
            }
          }
        }
      }
      if (valid)
        p.lse[(int64_t)head * p.total_rows + seq_start + q_pos] =
            (m + __log2f(l)) * 0.69314718055994531f;
    }
    }  // schedule entries
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<512>(tmem);
}

}  // namespace

// Tensor map over one bf16 operand of a token-major packed buffer:
// dims {D, H, rows}, strides {D*2 (head), row_stride*2 (token)}, box {64, 1, box_rows}.
int make_head_tmap(CUtensorMap* m, const void* base, int64_t row_stride_elems, int n_heads,
                   int head_dim, int rows, int box_rows) {
  uint64_t dims[3] = {(uint64_t)head_dim, (uint64_t)n_heads, (uint64_t)rows};
  uint64_t strides[2] = {(uint64_t)head_dim * 2, (uint64_t)row_stride_elems * 2};
  uint32_t box[3] = {64, 1, (uint32_t)box_rows};
  return encode_tmap_bf16(m, base, 3, dims, strides, box);
}

template <int D>
static int launch_fwd(const FspAttnFwd* a, cudaStream_t stream) {
  CUtensorMap tq, tk, tv;
  int rc;
  if ((rc = make_head_tmap(&tq, a->q, a->q_stride, a->n_heads, D, a->total_rows, 128))) return rc;
  if ((rc = make_head_tmap(&tk, a->k, a->k_stride, a->n_heads, D, a->total_rows, 128))) return rc;
  if ((rc = make_head_tmap(&tv, a->v, a->v_stride, a->n_heads, D, a->total_rows, 128))) return rc;
  FwdParams p;
  p.o = reinterpret_cast<__nv_bfloat16*>(a->o);
  p.lse = a->lse;
  p.o_stride = a->o_stride;
  p.cu_seqlens = a->d_cu_seqlens;
  p.seq_starts = a->d_seq_starts;
  p.tiles = a->d_tiles;
  p.total_rows = a->total_rows;
  p.n_heads = a->n_heads;
  p.scale_log2 = a->softmax_scale * 1.4426950408889634f;
  if ((rc = scatter_from_abi(a->scatter, 1, a->n_heads, D, a->total_rows, &p.sc))) return rc;
  p.n_tiles = a->n_tiles;
  p.noncausal = (a->flags & FSP_ATTN_NONCAUSAL) ? 1 : 0;
  if (D == 128) {  // schedule entries are 256-row tile pairs (fsp_attn_schedule, head_dim 128)
    const int smem = Fwd2Smem::kBytes + 1024;
    // Persistent launch (CTAs steal not-yet-launched entries, so an entry's Q load and first
    // QK^T overlap the previous entry's softmax tail and epilogue) unless the head->seq
    // exchange is fused, whose epilogue stages rows in the entry's Q buffer.
    const char* env = getenv("FSP_FWD_PERSISTENT");
    const bool persistent = !(env && env[0] == '0');
    if (persistent) {
      FSP_CUDA(cudaFuncSetAttribute(attn_fwd_pair_kernel<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attn_fwd_pair_kernel<true><<<(unsigned)a->n_tiles, kF2Threads, smem, stream>>>(tq, tk, tv, p);
    } else {
      FSP_CUDA(cudaFuncSetAttribute(attn_fwd_pair_kernel<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attn_fwd_pair_kernel<false><<<(unsigned)a->n_tiles, kF2Threads, smem, stream>>>(tq, tk, tv, p);
    }
  } else {
    const int smem = FwdSmem<D>::kBytes + 1024;
    FSP_CUDA(cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attn_fwd_kernel<D><<<(unsigned)a->n_tiles, kFwdThreads, smem, stream>>>(tq, tk, tv, p);
  }
  FSP_LAUNCH_CHECK();
  return FSP_OK;
}

int check_attn_common(const void* q, const void* k, const void* v, int64_t qs, int64_t ks,
                      int64_t vs, const int32_t* cu, const int32_t* tiles, int32_t n_tiles,
                      int32_t n_seq, int32_t total_rows, int32_t n_heads, int32_t head_dim) {
  FSP_CHECK_ARG(head_dim == 64 || head_dim == 128, "head_dim must be 64 or 128 (got %d)", head_dim);
  FSP_CHECK_ARG(n_heads >= 1, "n_heads must be >= 1");
  FSP_CHECK_ARG(n_seq >= 0 && total_rows >= 0 && n_tiles >= 0, "negative sizes");
  // tiles are {seq << 16 | tile} words decoded unsigned: at most 65535 sequences
  FSP_CHECK_ARG(n_seq < 65536, "n_seq must be in [0, 65536) (got %d)", n_seq);
  FSP_CHECK_ARG(q && k && v && cu && (tiles || n_tiles == 0), "null pointer argument");
  FSP_CHECK_ARG(qs >= (int64_t)n_heads * head_dim && ks >= (int64_t)n_heads * head_dim &&
                    vs >= (int64_t)n_heads * head_dim,
                "row strides must cover n_heads*head_dim elements");
  FSP_CHECK_ARG(qs % 8 == 0 && ks % 8 == 0 && vs % 8 == 0, "row strides must be multiples of 8");
  return FSP_OK;
}

}  // namespace fsp

extern "C" int32_t fsp_attn_schedule(const int32_t* cu, int32_t n_seq, int32_t n_heads,
                                     int32_t head_dim, int32_t kind, int32_t* tiles,
                                     int32_t capacity) {
  using namespace fsp;
  FSP_CHECK_ARG(cu != nullptr || n_seq == 0, "null cu_seqlens");
  FSP_CHECK_ARG(n_seq >= 0 && n_seq < 65536, "n_seq must be in [0, 65536)");
  FSP_CHECK_ARG(n_heads >= 1, "n_heads must be >= 1");
  FSP_CHECK_ARG(head_dim == 64 || head_dim == 128, "head_dim must be 64 or 128");
  FSP_CHECK_ARG(kind == FSP_SCHED_FWD || kind == FSP_SCHED_BWD, "unknown schedule kind %d", kind);
  if (n_seq > 0) FSP_CHECK_ARG(cu[0] == 0, "cu_seqlens[0] must be 0");
  // forward with head_dim 128 runs 256-row tile pairs (attn_fwd_pair_kernel)
  const int unit = (kind == FSP_SCHED_FWD && head_dim == 128) ? 2 * kBM : kBM;
  int64_t n = 0;
  for (int s = 0; s < n_seq; ++s) {
    const int len = cu[s + 1] - cu[s];
    FSP_CHECK_ARG(len >= 0, "cu_seqlens must be non-decreasing (sequence %d)", s);
    const int nt = (len + unit - 1) / unit;
    FSP_CHECK_ARG(nt < 65536, "sequence %d too long (%d tokens)", s, len);
    n += nt;
  }
  n *= n_heads;
  FSP_CHECK_ARG(n < (1ll << 30), "too many tiles");
  if (!tiles) return (int32_t)n;
  FSP_CHECK_ARG(capacity >= n, "tile capacity %d < %lld", capacity, (long long)n);
  // Sequences longest first (LPT across sequences); inside one sequence, all tiles of one
  // head before the next head, heaviest tile first (forward tile t costs t+1 kv tiles,
  // backward kv tile t costs n_tiles - t).  Keeping the ~148 resident CTAs on one or two
  // (sequence, head) pairs keeps that pair's K/V (forward) or Q/dO/dQ (backward) — 16 MB
  // per 32K-token head — resident in the 126 MB L2 instead of streaming it from HBM once
  // per tile.
  int* order = new int[n_seq > 0 ? n_seq : 1];
  for (int s = 0; s < n_seq; ++s) order[s] = s;
  std::stable_sort(order, order + n_seq, [&](int a, int b) {
    return (cu[a + 1] - cu[a]) > (cu[b + 1] - cu[b]);
  });
  int64_t k = 0;
  for (int i = 0; i < n_seq; ++i) {
    const int s = order[i];
    const int nt = (cu[s + 1] - cu[s] + unit - 1) / unit;
    for (int h = 0; h < n_heads; ++h)
      for (int j = 0; j < nt; ++j) {
        const int t = kind == FSP_SCHED_BWD ? j : nt - 1 - j;
        tiles[2 * k] = (int32_t)(((uint32_t)s << 16) | (uint32_t)t);
        tiles[2 * k + 1] = h;
        ++k;
      }
  }
  delete[] order;
  return (int32_t)n;
}

extern "C" int fsp_attn_fwd(const FspAttnFwd* a, void* stream) {
  using namespace fsp;
  FSP_CHECK_ARG(a != nullptr, "null args");
  // an empty group (no rows: a selected group without sequences, or a member holding
  // only pad rows of a tiny one) is a no-op whatever its (possibly null) buffers are
  FSP_CHECK_ARG(a->head_dim == 64 || a->head_dim == 128, "head_dim must be 64 or 128 (got %d)",
                a->head_dim);
  FSP_CHECK_ARG(a->n_heads >= 1, "n_heads must be >= 1");
  FSP_CHECK_ARG(a->total_rows >= 0 && a->n_tiles >= 0, "negative sizes");
  FSP_CHECK_ARG((a->flags & ~FSP_ATTN_NONCAUSAL) == 0, "unknown attention flags 0x%x", a->flags);
  FSP_CHECK_ARG(!(a->flags & FSP_ATTN_NONCAUSAL) || a->head_dim == 128,
                "FSP_ATTN_NONCAUSAL needs head_dim 128");
  if (a->total_rows == 0 && a->n_tiles == 0) return FSP_OK;
  int rc = check_attn_common(a->q, a->k, a->v, a->q_stride, a->k_stride, a->v_stride,
                             a->d_cu_seqlens, a->d_tiles, a->n_tiles, a->n_seq, a->total_rows,
                             a->n_heads, a->head_dim);
  if (rc) return rc;
  FSP_CHECK_ARG(a->o && a->lse, "null output pointer");
  FSP_CHECK_ARG(a->o_stride >= (int64_t)a->n_heads * a->head_dim && a->o_stride % 8 == 0,
                "bad o_stride");
  {
    ScatterDev sc;  // validated before any device work
    if ((rc = scatter_from_abi(a->scatter, 1, a->n_heads, a->head_dim, a->total_rows, &sc)))
      return rc;
  }
  if (a->n_tiles == 0 || a->total_rows == 0) return FSP_OK;
  return a->head_dim == 128 ? launch_fwd<128>(a, (cudaStream_t)stream)
                            : launch_fwd<64>(a, (cudaStream_t)stream);
}
