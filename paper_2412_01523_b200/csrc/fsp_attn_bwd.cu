// fsp_attn_bwd.cu — packed varlen causal attention backward on tcgen05/TMEM.
//
// Gradient of Eq. (3) under flash-attn varlen semantics.
// Three launches:
//   1. prep:  delta[h,t] = sum_d O[t,h,d] * dO[t,h,d] (fp32) and dq_accum := 0
//   2. main:  one CTA = one 128-row KV tile of one sequence x one head; loops over the
//             query tiles that see it causally (i >= kv tile) and keeps dK, dV in TMEM:
//               S^T  = K Q_i^T            (SS, K-major / K-major)
//               dP^T = V dO_i^T           (SS)
//               P^T  = exp2(S^T*scale*log2e - lse2_i)      (registers -> TMEM, bf16)
//               dS^T = P^T (dP^T - delta_i)                 (registers -> smem, bf16, SW128)
//               dV  += P^T dO_i           (TS: A = P^T in TMEM, B = dO_i MN-major)
//               dK  += dS^T Q_i           (SS: A = dS^T K-major, B = Q_i MN-major)
//               dQ_i = dS K               (SS: A = dS MN-major (same smem), B = K MN-major)
//             dQ_i is read out of TMEM and added to dq_accum ([H, T, D] fp32) with reductions.
//   3. post:  dq[t, h] = bf16(dq_accum[h, t] * scale)
// TMEM (512 cols): dK [0,128) dV [128,256) S^T|P^T [256,384) dP^T|dQ [384,512).
// smem: K, V (resident), a 3-slot ring of 32 KB tiles streaming Q_i / dO_i, dS (32 KB).
#include <type_traits>

#include "fsp_host.h"
#include "fsp_ptx.cuh"
#include "fsp_scatter.cuh"

namespace fsp {

int make_head_tmap(CUtensorMap* m, const void* base, int64_t row_stride_elems, int n_heads,
                   int head_dim, int rows, int box_rows);
int check_attn_common(const void* q, const void* k, const void* v, int64_t qs, int64_t ks,
                      int64_t vs, const int32_t* cu, const int32_t* tiles, int32_t n_tiles,
                      int32_t n_seq, int32_t total_rows, int32_t n_heads, int32_t head_dim);

namespace {

constexpr int kTile = 128;
constexpr int kBwdThreads = 192;
constexpr uint32_t kColDK = 0, kColDV = 128, kColS = 256, kColDP = 384;
constexpr float kLog2e = 1.4426950408889634f;

struct BwdParams {
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  float* dq_accum;
  const float* lse;
  const float* delta;
  int64_t dk_stride, dv_stride;
  const int32_t* cu_seqlens;
  const int32_t* seq_starts;  // optional: row of each sequence (else cu_seqlens)
  const int32_t* tiles;
  int32_t total_rows;
  int32_t n_heads;
  float scale;
  float scale_log2;
  int32_t n_tiles;  // schedule entries (the persistent kernel walks them)
  ScatterDev sc;  // fused head->seq of dK / dV (matrices 1, 2); sc.degree == 0: off
  int32_t noncausal;  // FSP_ATTN_NONCAUSAL (v2 kernel): every kv row meets every query row
};

template <int D>
struct BwdSmem {
  static constexpr int kBoxes = D / 64;
  static constexpr int kTileBytes = 128 * D * 2;
  static constexpr int kK = 0;
  static constexpr int kV = kK + kTileBytes;
  static constexpr int kRing = kV + kTileBytes;  // 3 slots
  static constexpr int kDS = kRing + 3 * kTileBytes;
  static constexpr int kStat = kDS + 128 * 128 * 2;  // lse2[2][128], delta[2][128]
  static constexpr int kBar = kStat + 4 * 128 * 4;
  static constexpr int kBytes = kBar + 256;
};

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ BwdParams p) {
  using L = BwdSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  float* lse_s = reinterpret_cast<float*>(smem + L::kStat);         // [2][128]
  float* delta_s = lse_s + 256;                                     // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* bar_kv = bars + 0;
  uint64_t* ring_full = bars + 1;   // [3]
  uint64_t* ring_empty = bars + 4;  // [3]
  uint64_t* s_full = bars + 7;
  uint64_t* p_ready = bars + 8;
  uint64_t* dq_full = bars + 9;
  uint64_t* tm_free = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int tile = p.tiles[2 * blockIdx.x];
  const int head = p.tiles[2 * blockIdx.x + 1];
  const int seq = (int)((uint32_t)tile >> 16);  // unsigned: n_seq up to 65535
  const int kt = tile & 0xFFFF;
  const int seq_start = p.seq_starts ? p.seq_starts[seq] : p.cu_seqlens[seq];
  const int seqlen = p.cu_seqlens[seq + 1] - p.cu_seqlens[seq];
  const int kv0 = kt * kTile;
  const int nq = (seqlen + kTile - 1) / kTile;
  const int n_it = nq - kt;  // query tiles kt .. nq-1

  if (threadIdx.x == 0) {
    mbar_init(bar_kv, 1);
    for (int i = 0; i < 3; ++i) {
      mbar_init(ring_full + i, 1);
      mbar_init(ring_empty + i, 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_ready, 4);
    mbar_init(dq_full, 1);
    mbar_init(tm_free, 4);
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
      tma_prefetch(&tm_do);
      mbar_expect_tx(bar_kv, 2 * L::kTileBytes);
      for (int b = 0; b < L::kBoxes; ++b) {
        tma_load_3d(smem + L::kK + b * 16384, &tm_k, bar_kv, b * 64, head, seq_start + kv0);
        tma_load_3d(smem + L::kV + b * 16384, &tm_v, bar_kv, b * 64, head, seq_start + kv0);
      }
      for (int item = 0; item < 2 * n_it; ++item) {
        const int slot = item % 3;
        const uint32_t ph = (item / 3) & 1;
        const int row = seq_start + (kt + (item >> 1)) * kTile;
        mbar_wait(ring_empty + slot, ph ^ 1);
        mbar_expect_tx(ring_full + slot, L::kTileBytes);
        const CUtensorMap* map = (item & 1) ? &tm_do : &tm_q;
        for (int b = 0; b < L::kBoxes; ++b)
          tma_load_3d(smem + L::kRing + slot * L::kTileBytes + b * 16384, map, ring_full + slot,
                      b * 64, head, row);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_dvdk = make_idesc_bf16(128, D, false, true);
      constexpr uint32_t idesc_dq = make_idesc_bf16(128, D, true, true);
      const uint32_t k_base = smem_u32(smem + L::kK);
      const uint32_t v_base = smem_u32(smem + L::kV);
      const uint32_t ring_base = smem_u32(smem + L::kRing);
      const uint32_t ds_base = smem_u32(smem + L::kDS);
      mbar_wait(bar_kv, 0);
      for (int it = 0; it < n_it; ++it) {
        const int sq = (2 * it) % 3, sd = (2 * it + 1) % 3;
        const uint32_t pq = ((2 * it) / 3) & 1, pd = ((2 * it + 1) / 3) & 1;
        const uint32_t q_base = ring_base + sq * L::kTileBytes;
        const uint32_t do_base = ring_base + sd * L::kTileBytes;
        if (it > 0) mbar_wait(tm_free, (it - 1) & 1);
        mbar_wait(ring_full + sq, pq);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(tmem + kColS, make_sdesc_sw128(k_base + off, 16, 1024),
                 make_sdesc_sw128(q_base + off, 16, 1024), idesc_s, kk > 0);
        }
        mbar_wait(ring_full + sd, pd);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(tmem + kColDP, make_sdesc_sw128(v_base + off, 16, 1024),
                 make_sdesc_sw128(do_base + off, 16, 1024), idesc_s, kk > 0);
        }
        tc_commit(s_full);
        mbar_wait(p_ready, it & 1);
        tc_fence_after();
        const uint32_t acc = it > 0 ? 1u : 0u;
#pragma unroll
        for (int kk = 0; kk < kTile / 16; ++kk)  // dV += P^T dO
          mma_ts(tmem + kColDV, tmem + kColS + kk * 8,
                 make_sdesc_sw128(do_base + kk * 2048, 16384, 1024), idesc_dvdk, acc | (kk > 0));
#pragma unroll
        for (int kk = 0; kk < kTile / 16; ++kk) {  // dK += dS^T Q
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(tmem + kColDK, make_sdesc_sw128(ds_base + off, 16, 1024),
                 make_sdesc_sw128(q_base + kk * 2048, 16384, 1024), idesc_dvdk, acc | (kk > 0));
        }
#pragma unroll
        for (int kk = 0; kk < kTile / 16; ++kk)  // dQ = dS K
          mma_ss(tmem + kColDP, make_sdesc_sw128(ds_base + kk * 2048, 16384, 1024),
                 make_sdesc_sw128(k_base + kk * 2048, 16384, 1024), idesc_dq, kk > 0);
        tc_commit(dq_full);
        tc_commit(ring_empty + sq);
        tc_commit(ring_empty + sd);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ compute warps
    const uint32_t quad = warp & 3;
    const int r = quad * 32 + lane;  // kv row for S^T/dP^T, q row for dQ
    const uint32_t lane_addr = (quad * 32u) << 16;
    const int kv_pos = kv0 + r;
    const float sl2 = p.scale_log2;
    uint8_t* ds_row = smem + L::kDS + r * 128;  // row r of box 0; box 1 at +16384
    for (int it = 0; it < n_it; ++it) {
      const int q0 = (kt + it) * kTile;
      const int buf = it & 1;
      {
        const int t = r;
        const bool valid = q0 + t < seqlen;
        const int64_t gi = (int64_t)head * p.total_rows + seq_start + q0 + t;
        lse_s[buf * 128 + t] = valid ? p.lse[gi] * kLog2e : INFINITY;
        delta_s[buf * 128 + t] = valid ? p.delta[gi] : 0.f;
      }
      named_bar_sync(1, 128);
      const float* ls = lse_s + buf * 128;
      const float* dl = delta_s + buf * 128;
      mbar_wait(s_full, it & 1);
      tc_fence_after();
      const bool diag = (it == 0);
#pragma unroll
      for (int c = 0; c < kTile; c += 32) {
        uint32_t sr[32], dr[32];
        tmem_ld32(tmem + lane_addr + kColS + c, sr);
        tmem_ld32(tmem + lane_addr + kColDP + c, dr);
        tmem_ld_wait();
        uint32_t pk[16], dk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float p0 = ex2(fmaf(__uint_as_float(sr[i]), sl2, -ls[c + i]));
          float p1 = ex2(fmaf(__uint_as_float(sr[i + 1]), sl2, -ls[c + i + 1]));
          if (diag) {  // causal: q_pos >= kv_pos  <=>  (c+i) >= r on the diagonal tile
            if (c + i < r) p0 = 0.f;
            if (c + i + 1 < r) p1 = 0.f;
          }
          const float d0 = p0 * (__uint_as_float(dr[i]) - dl[c + i]);
          const float d1 = p1 * (__uint_as_float(dr[i + 1]) - dl[c + i + 1]);
          pk[i / 2] = pack_bf16(p0, p1);
          dk[i / 2] = pack_bf16(d0, d1);
        }
        tmem_st16(tmem + lane_addr + kColS + c / 2, pk);
        // dS^T row r, q columns [c, c+32): box c/64, 16-byte chunks ((c%64)/8 + v) ^ (r%8)
        uint8_t* box = ds_row + (c >> 6) * 16384;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int chunk = (((c & 63) >> 3) + v) ^ (r & 7);
          *reinterpret_cast<uint4*>(box + chunk * 16) =
              make_uint4(dk[4 * v], dk[4 * v + 1], dk[4 * v + 2], dk[4 * v + 3]);
        }
      }
      tmem_st_wait();
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_ready);
      // ---- dQ_i readout: lane r is query row q0 + r
      mbar_wait(dq_full, it & 1);
      tc_fence_after();
      const bool qvalid = q0 + r < seqlen;
      float* dq_row = p.dq_accum + ((int64_t)head * p.total_rows + seq_start + q0 + r) * D;
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        uint32_t qr[32];
        tmem_ld32(tmem + lane_addr + kColDP + c, qr);
        tmem_ld_wait();
        if (qvalid) {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            red_add_v4(dq_row + c + i, __uint_as_float(qr[i]), __uint_as_float(qr[i + 1]),
                       __uint_as_float(qr[i + 2]), __uint_as_float(qr[i + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tm_free);
    }
    // ---- epilogue: dK (scaled), dV for kv row r (TMEM loads are warp-collective)
    {
      const bool kvalid = kv_pos < seqlen;
      // local rows (optional when the exchange is fused) and the fused head->seq
      // destinations in the owning member's sequence shard (matrices 1 = dK, 2 = dV)
      const int64_t trow = (int64_t)(seq_start + kv_pos);
      __nv_bfloat16* dk_row = p.dk ? p.dk + trow * p.dk_stride + (int64_t)head * D : nullptr;
      __nv_bfloat16* dv_row = p.dv ? p.dv + trow * p.dv_stride + (int64_t)head * D : nullptr;
      __nv_bfloat16* pk_row = kvalid ? scatter_row(p.sc, trow, 1, head, D) : nullptr;
      __nv_bfloat16* pv_row = pk_row ? pk_row + p.sc.mat_stride : nullptr;
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        uint32_t a[32], b[32];
        tmem_ld32(tmem + lane_addr + kColDK + c, a);
        tmem_ld32(tmem + lane_addr + kColDV + c, b);
        tmem_ld_wait();
        if (!kvalid) continue;
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 vk, vv;
          vk.x = pack_bf16(__uint_as_float(a[i]) * p.scale, __uint_as_float(a[i + 1]) * p.scale);
          vk.y = pack_bf16(__uint_as_float(a[i + 2]) * p.scale, __uint_as_float(a[i + 3]) * p.scale);
          vk.z = pack_bf16(__uint_as_float(a[i + 4]) * p.scale, __uint_as_float(a[i + 5]) * p.scale);
          vk.w = pack_bf16(__uint_as_float(a[i + 6]) * p.scale, __uint_as_float(a[i + 7]) * p.scale);
          vv.x = pack_bf16(__uint_as_float(b[i]), __uint_as_float(b[i + 1]));
          vv.y = pack_bf16(__uint_as_float(b[i + 2]), __uint_as_float(b[i + 3]));
          vv.z = pack_bf16(__uint_as_float(b[i + 4]), __uint_as_float(b[i + 5]));
          vv.w = pack_bf16(__uint_as_float(b[i + 6]), __uint_as_float(b[i + 7]));
          if (dk_row) *reinterpret_cast<uint4*>(dk_row + c + i) = vk;
          if (dv_row) *reinterpret_cast<uint4*>(dv_row + c + i) = vv;
          if (pk_row) {
            *reinterpret_cast<uint4*>(pk_row + c + i) = vk;
            *reinterpret_cast<uint4*>(pv_row + c + i) = vv;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<512>(tmem);
}

// delta[h, t] = <O[t,h,:], dO[t,h,:]> in fp32; dq_accum[h,t,:] = 0.  One warp per (t, h).
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_prep_kernel(
    const __nv_bfloat16* __restrict__ o, int64_t o_stride, const __nv_bfloat16* __restrict__ dout,
    int64_t do_stride, float* __restrict__ delta, float* __restrict__ dq_accum, int total_rows,
    int n_heads) {
  constexpr int kPer = D / 32;  // elements per lane (2 or 4)
  const int64_t n = (int64_t)total_rows * n_heads;
  const int lane = threadIdx.x & 31;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t t = w / n_heads;
    const int h = (int)(w - t * n_heads);
    const __nv_bfloat16* op = o + t * o_stride + (int64_t)h * D + lane * kPer;
    const __nv_bfloat16* dp = dout + t * do_stride + (int64_t)h * D + lane * kPer;
    float acc = 0.f;
    if (kPer == 4) {
      const uint2 a = *reinterpret_cast<const uint2*>(op);
      const uint2 b = *reinterpret_cast<const uint2*>(dp);
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const float2 fa = __bfloat1622float2(a2[i]), fb = __bfloat1622float2(b2[i]);
        acc += fa.x * fb.x + fa.y * fb.y;
      }
    } else {
      const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(op);
      const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(dp);
      const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
      acc = fa.x * fb.x + fa.y * fb.y;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
    if (lane == 0) delta[(int64_t)h * total_rows + t] = acc;
    float* dq = dq_accum + ((int64_t)h * total_rows + t) * D + lane * kPer;
    if (kPer == 4)
      *reinterpret_cast<float4*>(dq) = make_float4(0.f, 0.f, 0.f, 0.f);
    else
      *reinterpret_cast<float2*>(dq) = make_float2(0.f, 0.f);
  }
}

// dq[t, h*D + i] = bf16(dq_accum[h, t, i] * scale); 8 elements per thread.
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_post_kernel(const float* __restrict__ dq_accum,
                                                            __nv_bfloat16* __restrict__ dq,
                                                            int64_t dq_stride, int total_rows,
                                                            int n_heads, float scale,
                                                            const __grid_constant__ ScatterDev sc) {
  constexpr int kPerRow = D / 8;
  const int64_t n = (int64_t)total_rows * n_heads * kPerRow;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(g % kPerRow) * 8;
    const int64_t th = g / kPerRow;
    const int h = (int)(th % n_heads);
    const int64_t t = th / n_heads;
    const float* src = dq_accum + ((int64_t)h * total_rows + t) * D + c;
    const float4 a = *reinterpret_cast<const float4*>(src);
    const float4 b = *reinterpret_cast<const float4*>(src + 4);
    uint4 v;
    v.x = pack_bf16(a.x * scale, a.y * scale);
    v.y = pack_bf16(a.z * scale, a.w * scale);
    v.z = pack_bf16(b.x * scale, b.y * scale);
    v.w = pack_bf16(b.z * scale, b.w * scale);
    if (dq) *reinterpret_cast<uint4*>(dq + t * dq_stride + (int64_t)h * D + c) = v;
    // fused head->seq of dQ (matrix 0) into the owning member's sequence shard
    __nv_bfloat16* prow = scatter_row(sc, t, 0, h, D);
    if (prow) *reinterpret_cast<uint4*>(prow + c) = v;
  }
}

// ============================================================================ v2 (D = 128)
// Same math as attn_bwd_kernel, restructured so the tensor core does not wait on the
// gradient warps: each 128-row query tile is processed as two 64-column half tiles
// u = 2*it + h whose S^T / dP^T live in separate TMEM stages, so the MMA issue order is
//   S/dP(u+1) | grads(u) | S/dP(u+2) | grads(u+1) ...
// while 8 compute warps turn S/dP(u) into P^T (TMEM) and dS^T (smem) and 4 reduction warps
// drain dQ^T(u-1) from TMEM into the fp32 accumulator in parallel.  dQ is produced
// transposed (dQ^T = K^T dS^T, M = D lanes, N = 64 query columns) into the stage's dP
// columns, so every TMEM stage is 64 columns:
// TMEM: dK [0,128) dV [128,256) S0 [256,320) S1 [320,384) dP0|dQ0 [384,448) dP1|dQ1 [448,512)
// Warps: 0 TMA, 1 MMA, 2..9 compute (two per TMEM lane quadrant, 32 of the 64 columns
// each), 10..13 dQ reduction (one per quadrant, all 64 columns).
#ifndef FSP_BWD_ABLATE
#define FSP_BWD_ABLATE 0  // profiling ablations (bits): 1 = skip gradient math, 2 = skip dQ
                          // readout, 4 = skip dQ^T MMAs, 8 = skip dK MMAs, 16 = plain
                          // stores instead of dQ reductions, 32 = no dQ stores at all,
                          // 64 = no dQ^T TMEM readout
#endif
#ifndef FSP_BWD_RING
#define FSP_BWD_RING 6  // 64-row Q / dO slots of the TMA ring (6 = three 64-query units)
#endif
#ifndef FSP_BWD_DS_TMEM
#define FSP_BWD_DS_TMEM 1  // dS^T also goes to TMEM so dK += dS^T Q is a TS MMA
#endif
#ifndef FSP_BWD_COMPUTE_WARPS
#define FSP_BWD_COMPUTE_WARPS 8  // 8 vs 16 re-measured with the persistent launch: 8 is 0.3-0.7% faster
#endif
constexpr int kV2Compute = FSP_BWD_COMPUTE_WARPS;  // 8 or 16: 2 or 4 warps per lane quadrant
constexpr int kV2Cols = 64 / (kV2Compute / 4);      // query columns per compute warp
// 4, 8 or 16 compute warps: 1, 2 or 4 per TMEM lane quadrant, each owning kV2Cols = 64, 32
// or 16 query columns of a unit.  (Round 1 tried 4 warps while the TMEM loads / stores below
// were written for 16 / 32 columns only and the softmax statistics were fetched by compute
// threads 128..255 — with 4 warps 48 of the 64 S / dP columns were never loaded, 3/4 of P
// and dS never stored and delta never fetched: the parity failure it saw.  Those paths are
// now generic in kV2Cols and in the compute-thread count.)
static_assert(kV2Compute == 4 || kV2Compute == 8 || kV2Compute == 16,
              "1, 2 or 4 compute warps per TMEM lane quadrant");
#ifndef FSP_BWD_REDUCE_WARPS
#define FSP_BWD_REDUCE_WARPS 4
#endif
#ifndef FSP_BWD_REDUCE_SPLIT
#define FSP_BWD_REDUCE_SPLIT 0  // with 8 reduction warps: 0 = split a unit's 64 columns,
                                // 1 = split units by parity (each warp drains whole units)
#endif
#ifndef FSP_BWD_STAT_SHFL
#define FSP_BWD_STAT_SHFL 0  // 1: softmax statistics broadcast by warp shuffles, not LDS
#endif
#ifndef FSP_BWD_POLY_EVERY
#define FSP_BWD_POLY_EVERY 0  // one exponential pair in N on the FMA pipe (ex2_poly2); 0 = none
#endif
constexpr int kV2Reduce = FSP_BWD_REDUCE_WARPS;  // 4 or 8: 1 or 2 warps per lane quadrant
constexpr bool kRedSplitUnits = FSP_BWD_REDUCE_SPLIT && kV2Reduce == 8;
constexpr int kV2RedCols = kRedSplitUnits ? 64 : 64 / (kV2Reduce / 4);  // dQ^T columns per warp
constexpr int kTmFreeCount = kRedSplitUnits ? 4 : kV2Reduce;  // warps draining one unit
#ifndef FSP_BWD_WG5
#define FSP_BWD_WG5 0  // 1: five warpgroups (TMA+MMA+2 idle | 8 compute | 8 reduction split by
                       // unit parity) with setmaxnreg moving registers to the compute warps
#endif
constexpr bool kWG5 = FSP_BWD_WG5;
static_assert(!kWG5 || (kV2Compute == 8 && kV2Reduce == 8 && kRedSplitUnits),
              "FSP_BWD_WG5 needs 8 compute and 8 unit-split reduction warps");
constexpr int kV2Warp0 = kWG5 ? 4 : 2;  // first compute warp (warpgroup-aligned with WG5)
constexpr int kV2Threads = kWG5 ? 640 : 64 + 32 * (kV2Compute + kV2Reduce);
constexpr uint32_t kV2ColS = 256, kV2ColDP = 384;

struct BwdSmemV2 {
  static constexpr int kTileBytes = 128 * 128 * 2;
  static constexpr int kHalfBytes = 64 * 128 * 2;     // one 64-row half of Q_i or dO_i
  static constexpr int kSlots = FSP_BWD_RING;         // Q / dO half tiles in flight
  static constexpr int kK = 0;
  static constexpr int kV = kK + kTileBytes;
  static constexpr int kRing = kV + kTileBytes;
  static constexpr int kDS = kRing + kSlots * kHalfBytes;  // 2 stages x [128 kv][64 q] bf16
  static constexpr int kStat = kDS + 2 * 16384;       // lse2[2][128], delta[2][128]
  static constexpr int kBar = kStat + 4 * 128 * 4;
  static constexpr int kBytes = kBar + 512;  // 64 barrier words
};
// The fused dK/dV epilogue stages its two 128-row output tiles (2 x 32 KB) in the Q/dO
// ring, which is idle by then: the ring must hold at least that much.
static_assert(BwdSmemV2::kSlots * BwdSmemV2::kHalfBytes >= 2 * BwdSmemV2::kTileBytes,
              "FSP_BWD_RING too small for the dK/dV epilogue staging (needs >= 4 slots)");

#ifndef FSP_BWD_TIMING
#define FSP_BWD_TIMING 0  // profiling build: cycles the MMA issuer / compute warps spend waiting
#endif
#if FSP_BWD_TIMING
__device__ unsigned long long g_bwd_wait[16];
__device__ unsigned int g_bwd_done;
#define FSP_TW(slot, call)                               \
  do {                                                   \
    const long long t0_ = clock64();                     \
    call;                                                \
    tw[slot] += clock64() - t0_;                         \
  } while (0)
#else
#define FSP_TW(slot, call) call
#endif

// One schedule entry of the backward: 128 kv rows (kv tile kt) of one sequence x head.
struct KvTile {
  int head, seq_start, seqlen, kt, kv0, nq, n_it, n_u;
  int qt0;  // first query tile this kv tile meets: kt (causal) or 0 (non-causal)
};

__device__ __forceinline__ KvTile decode_kv(const BwdParams& p, int w) {
  KvTile t;
  const int tile = p.tiles[2 * w];
  t.head = p.tiles[2 * w + 1];
  const int seq = (int)((uint32_t)tile >> 16);  // unsigned: n_seq up to 65535
  t.kt = tile & 0xFFFF;
  t.seq_start = p.seq_starts ? p.seq_starts[seq] : p.cu_seqlens[seq];
  t.seqlen = p.cu_seqlens[seq + 1] - p.cu_seqlens[seq];
  t.kv0 = t.kt * kTile;
  t.nq = (t.seqlen + kTile - 1) / kTile;
  t.qt0 = p.noncausal ? 0 : t.kt;
  t.n_it = t.nq - t.qt0;
  t.n_u = 2 * t.n_it;
  return t;
}

// Dynamic schedule of the persistent launch (as in the forward): one CTA per schedule
// entry, and a CTA that finishes an entry steals the next not-yet-launched CTA's entry
// through cluster launch control; the TMA producer hands entries to the other roles through
// a two-slot shared-memory ring.
struct BwdEntryRing {
  int* idx;
  uint64_t* full;
  uint64_t* empty;
  void* resp;     // 16-byte cluster-launch-control response
  uint64_t* clc;  // its completion barrier
};
constexpr int kBwdRingConsumers = 1 + kV2Compute + kV2Reduce;  // MMA thread + warps

template <bool kPersistent>
__device__ __forceinline__ int bwd_claim(const BwdEntryRing& r, int k) {
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

template <bool kPersistent, bool kWarp>
__device__ __forceinline__ int bwd_take(const BwdEntryRing& r, int k) {
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

// kPersistent: one CTA per SM walks the schedule (dynamic claims); the next entry's K/V load
// and first S^T/dP^T MMAs overlap this entry's dK/dV epilogue.  Barrier phases and the
// Q/dO ring run on across entries: every parity below derives from running counts (global
// unit index U, global query-tile index IT = U / 2, entry count k).
template <bool kPersistent>
__global__ void __launch_bounds__(kV2Threads, 1)
    attn_bwd_kernel_v2(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                       const __grid_constant__ BwdParams p) {
  constexpr int D = 128;
  using L = BwdSmemV2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  float* lse_s = reinterpret_cast<float*>(smem + L::kStat);  // [2][128]
  float* delta_s = lse_s + 256;                              // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* bar_kv = bars + 0;
  constexpr int kR = L::kSlots;
  static_assert(1 + 2 * kR + 18 <= 64, "barrier region holds 64 words");
  uint64_t* ring_full = bars + 1;            // [kSlots]
  uint64_t* ring_empty = bars + 1 + kR;      // [kSlots]
  uint64_t* s_full = bars + 1 + 2 * kR;      // [2]
  uint64_t* p_ready = s_full + 2;            // [2]
  uint64_t* dq_full = s_full + 4;            // [2]
  uint64_t* tm_free = s_full + 6;            // [2]
  uint64_t* acc_done = s_full + 8;           // dK / dV final
  // s_full + 15 is 16-byte aligned: 1 + 2 * kSlots (even) + 2 + 15 words from a 1 KB boundary
  static_assert((1 + 2 * kR + 15) % 2 == 0, "CLC response must be 16-byte aligned");
  const BwdEntryRing ering{reinterpret_cast<int*>(s_full + 13), s_full + 9, s_full + 11,
                           s_full + 15, s_full + 14};
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 17);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (threadIdx.x == 0) {
    mbar_init(bar_kv, 1);
    for (int i = 0; i < L::kSlots; ++i) {
      mbar_init(ring_full + i, 1);
      mbar_init(ring_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(p_ready + i, kV2Compute);
      mbar_init(dq_full + i, 1);
      mbar_init(tm_free + i, kTmFreeCount);
      mbar_init(ering.full + i, 1);
      mbar_init(ering.empty + i, kBwdRingConsumers);
    }
    mbar_init(ering.clc, 1);
    mbar_init(acc_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < kV2Warp0) {
  if (kWG5) setmaxnreg_dec<56>();  // warpgroup 0: TMA, MMA and two idle warps
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      tma_prefetch(&tm_do);
      uint32_t U0 = 0;  // global index of the entry's first 64-query unit
      for (int k = 0;; ++k) {
        const int w = bwd_claim<kPersistent>(ering, k);
        if (w >= p.n_tiles) break;
        const KvTile T = decode_kv(p, w);
        if (k > 0) {
          // K / V of a kv tile are read by this CTA only (cold in L2): start their DRAM
          // reads now, while the previous entry's last units still run
          for (int b = 0; b < 2; ++b) {
            tma_prefetch_l2_3d(&tm_k, b * 64, T.head, T.seq_start + T.kv0);
            tma_prefetch_l2_3d(&tm_v, b * 64, T.head, T.seq_start + T.kv0);
          }
          mbar_wait(acc_done, (k - 1) & 1);  // the previous entry's MMAs read K / V
        }
        mbar_expect_tx(bar_kv, 2 * L::kTileBytes);
        for (int b = 0; b < 2; ++b) {
          tma_load_3d(smem + L::kK + b * 16384, &tm_k, bar_kv, b * 64, T.head, T.seq_start + T.kv0);
          tma_load_3d(smem + L::kV + b * 16384, &tm_v, bar_kv, b * 64, T.head, T.seq_start + T.kv0);
        }
        // items 2U / 2U+1 = Q / dO rows of half tile U (64 rows each)
        for (int li = 0; li < 2 * T.n_u; ++li) {
          const uint32_t item = 2 * U0 + li;
          const int slot = item % L::kSlots;
          const uint32_t ph = (item / L::kSlots) & 1;
          const int row = T.seq_start + T.qt0 * kTile + (li >> 1) * 64;
          mbar_wait(ring_empty + slot, ph ^ 1);
          mbar_expect_tx(ring_full + slot, L::kHalfBytes);
          const CUtensorMap* map = (li & 1) ? &tm_do : &tm_q;
          for (int b = 0; b < 2; ++b)
            tma_load_3d(smem + L::kRing + slot * L::kHalfBytes + b * 8192, map, ring_full + slot,
                        b * 64, T.head, row);
        }
        U0 += T.n_u;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Q/dO half tiles: K-major boxes of [64 rows][64 d] (8 KB, SBO 1024); MN-major view for
    // dK/dV: d chunks 8 KB apart (LBO), 16 query rows = 2048 B per K step.
    if (elect_one()) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, false, false);
      constexpr uint32_t idesc_dvdk = make_idesc_bf16(128, D, false, true);
      constexpr uint32_t idesc_dqt = make_idesc_bf16(128, 64, true, true);
      const uint32_t k_base = smem_u32(smem + L::kK);
      const uint32_t v_base = smem_u32(smem + L::kV);
      const uint32_t ring_base = smem_u32(smem + L::kRing);
      const uint32_t ds_base = smem_u32(smem + L::kDS);
#if FSP_BWD_TIMING
      long long tw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      const long long t_start = clock64();
#endif
      uint32_t U0 = 0;  // global unit index of the entry's first unit
      int units = 0;
      for (int k = 0;; ++k) {
        const int w = bwd_take<kPersistent, false>(ering, k);
        if (w >= p.n_tiles) break;
        const int n_u = decode_kv(p, w).n_u;
        FSP_TW(6, mbar_wait(bar_kv, k & 1));
        tc_fence_after();
        auto grads = [&](int u) {
          const uint32_t U = U0 + u, IT = U >> 1;
          const int h = U & 1;
          const int sq = (2 * U) % L::kSlots, sd = (2 * U + 1) % L::kSlots;
          const uint32_t q_base = ring_base + sq * L::kHalfBytes;
          const uint32_t do_base = ring_base + sd * L::kHalfBytes;
          const uint32_t dsb = ds_base + h * 16384;
          FSP_TW(3, mbar_wait(p_ready + h, IT & 1));
          tc_fence_after();
          // dQ^T first and committed on its own, so the reduction warps drain it while dV and
          // dK (and the next S^T) keep the tensor core busy: dP^T(U+2) waits on that drain.
          if (U >= 2) FSP_TW(4, mbar_wait(tm_free + h, (IT - 1) & 1));  // dQ^T(U-2) drained
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)  // dQ^T = K^T dS^T   (K = 128 kv rows)
            if (!(FSP_BWD_ABLATE & 4))
            mma_ss(tmem + kV2ColDP + h * 64, make_sdesc_sw128(k_base + kk * 2048, 16384, 1024),
                   make_sdesc_sw128(dsb + kk * 2048, 16384, 1024), idesc_dqt, kk > 0);
          tc_commit(dq_full + h);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // dV += P^T dO_h      (K = 64 query rows)
            // P^T of query columns [16kk, 16kk+16): compute warp ch wrote its kV2Cols columns
            // as bf16 pairs into the first half of its own S columns [ch*kV2Cols, ...) — S
            // columns it read itself, so no cross-warp barrier is needed
            mma_ts(tmem + kColDV,
                   tmem + kV2ColS + h * 64 + (16 * kk / kV2Cols) * kV2Cols + (16 * kk % kV2Cols) / 2,
                   make_sdesc_sw128(do_base + kk * 2048, 8192, 1024), idesc_dvdk,
                   (u > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // dK += dS^T Q_h
            if (FSP_BWD_ABLATE & 8) continue;
            if (FSP_BWD_DS_TMEM)  // TS: dS^T from the second half of the writer warp's S columns
              mma_ts(tmem + kColDK,
                     tmem + kV2ColS + h * 64 + (16 * kk / kV2Cols) * kV2Cols + (16 * kk % kV2Cols) / 2 +
                         kV2Cols / 2,
                     make_sdesc_sw128(q_base + kk * 2048, 8192, 1024), idesc_dvdk,
                     (u > 0 || kk > 0) ? 1u : 0u);
            else
              mma_ss(tmem + kColDK, make_sdesc_sw128(dsb + kk * 32, 16, 1024),
                     make_sdesc_sw128(q_base + kk * 2048, 8192, 1024), idesc_dvdk,
                     (u > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(ring_empty + sq);
          tc_commit(ring_empty + sd);
          if (u == n_u - 1) tc_commit(acc_done);
        };
        for (int u = 0; u < n_u; ++u) {
          const uint32_t U = U0 + u, IT = U >> 1;
          const int h = U & 1;
          const int sq = (2 * U) % L::kSlots, sd = (2 * U + 1) % L::kSlots;
          const uint32_t q_base = ring_base + sq * L::kHalfBytes;
          const uint32_t do_base = ring_base + sd * L::kHalfBytes;
          // S^T(U) overwrites P^T(U-2), read by dV of grads(U-2) (issued earlier, in order);
          // dP^T(U) overwrites dQ^T(U-2): wait until the reduction warps drained it.
          FSP_TW(0, mbar_wait(ring_full + sq, ((2 * U) / L::kSlots) & 1));
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            mma_ss(tmem + kV2ColS + h * 64,
                   make_sdesc_sw128(k_base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                   make_sdesc_sw128(q_base + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), idesc_s,
                   kk > 0);
          }
          if (U >= 2) FSP_TW(1, mbar_wait(tm_free + h, (IT - 1) & 1));
          FSP_TW(2, mbar_wait(ring_full + sd, ((2 * U + 1) / L::kSlots) & 1));
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            mma_ss(tmem + kV2ColDP + h * 64,
                   make_sdesc_sw128(v_base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                   make_sdesc_sw128(do_base + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), idesc_s,
                   kk > 0);
          }
          tc_commit(s_full + h);
          if (u >= 1) grads(u - 1);
        }
        if (n_u > 0) grads(n_u - 1);
        U0 += n_u;
        units += n_u;
      }
#if FSP_BWD_TIMING
      tw[7] = clock64() - t_start;
      for (int i = 0; i < 8; ++i) atomicAdd(&g_bwd_wait[i], (unsigned long long)tw[i]);
      atomicAdd(&g_bwd_wait[8], (unsigned long long)units);
      __threadfence();
      // persistent launches: only the first ~148 CTAs run (the rest are cancelled by CLC)
      if (atomicAdd(&g_bwd_done, 1u) == (kPersistent ? min(gridDim.x, 148u) : gridDim.x) - 1) {
        printf("bwd MMA issuer cycles (sum over CTAs): units %llu total %llu | ring_full(Q) %llu "
               "tm_free(dP) %llu ring_full(dO) %llu p_ready %llu tm_free(dQ) %llu kv %llu\n",
               g_bwd_wait[8], g_bwd_wait[7], g_bwd_wait[0], g_bwd_wait[1], g_bwd_wait[2],
               g_bwd_wait[3], g_bwd_wait[4], g_bwd_wait[6]);
        printf("bwd compute warp0 cycles: s_full wait %llu busy %llu | reduce warp0: dq_full "
               "wait %llu busy %llu\n", g_bwd_wait[9], g_bwd_wait[10], g_bwd_wait[11],
               g_bwd_wait[12]);
        for (int i = 0; i < 16; ++i) g_bwd_wait[i] = 0;
        g_bwd_done = 0;
      }
#endif
    }
    __syncwarp();
  }
  } else if (warp < kV2Warp0 + kV2Compute) {
    // a CTA can only move registers it was launched with: 640 x 96 at launch, 40 x 128 freed
    // by warpgroup 0 and 16 x 256 by the reduction warpgroups pay for 32 x 256 here
    if (kWG5) setmaxnreg_inc<128>();
    // ------------------------------------------------------------ compute warps
    const uint32_t cw = warp - kV2Warp0;       // 0..kV2Compute-1
    const uint32_t quad = warp & 3;            // TMEM lane quadrant
    const uint32_t ch = cw >> 2;               // which kV2Cols of the 64 columns
    const int r = quad * 32 + lane;            // kv row of S^T / dP^T
    const uint32_t lane_addr = (quad * 32u) << 16;
    const float sl2 = p.scale_log2;
    const int ctid = cw * 32 + lane;
    uint32_t IT0 = 0;  // global index of the entry's first query tile
    for (int k = 0;; ++k) {
    const int w = bwd_take<kPersistent, true>(ering, k);
    if (w >= p.n_tiles) break;
    const KvTile T = decode_kv(p, w);
    const int head = T.head, seq_start = T.seq_start, seqlen = T.seqlen, qt0 = T.qt0,
              kv0 = T.kv0, n_it = T.n_it;
    const int kv_pos = kv0 + r;
    // non-causal: key rows past the sequence end must not contribute (their K rows belong to
    // the next sequence); causal masking covers them implicitly
    const bool kv_dead = kv_pos >= seqlen;
    // statistics entry e of query tile `it`: e < 128 is lse row e, e >= 128 delta row e-128
    auto load_stat = [&](int e, int it) -> float {
      const int t = e & 127;
      const int q0 = (qt0 + it) * kTile;
      const bool valid = q0 + t < seqlen;
      const int64_t gi = (int64_t)head * p.total_rows + seq_start + q0 + t;
      if (e < 128) return valid ? -p.lse[gi] * kLog2e : -INFINITY;  // stored negated
      return valid ? p.delta[gi] : 0.f;
    };
    auto half = [&](auto diag_c, int it, int h) {
      constexpr bool kDiag = decltype(diag_c)::value;
      const int buf = (IT0 + it) & 1;
      const int c0 = h * 64 + ch * kV2Cols;  // query column offset inside the 128-row tile
      const float* ls = lse_s + buf * 128 + c0;
      const float* dl = delta_s + buf * 128 + c0;
#if FSP_BWD_TIMING
      const long long tq0 = clock64();
#endif
      mbar_wait(s_full + h, (IT0 + it) & 1);
#if FSP_BWD_TIMING
      if (cw == 0 && lane == 0) atomicAdd(&g_bwd_wait[9], (unsigned long long)(clock64() - tq0));
#endif
      tc_fence_after();
      if (FSP_BWD_ABLATE & 1) {  // profiling ablation: no gradient math
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_ready + h);
        return;
      }
      uint32_t sr[kV2Cols], dr[kV2Cols];
      const uint32_t col0 = h * 64 + ch * kV2Cols;
      if (kV2Cols >= 32) {
#pragma unroll
        for (int c = 0; c < kV2Cols; c += 32) {
          tmem_ld32(tmem + lane_addr + kV2ColS + col0 + c, *reinterpret_cast<uint32_t(*)[32]>(sr + c));
          tmem_ld32(tmem + lane_addr + kV2ColDP + col0 + c, *reinterpret_cast<uint32_t(*)[32]>(dr + c));
        }
      } else {
        tmem_ld16(tmem + lane_addr + kV2ColS + col0, *reinterpret_cast<uint32_t(*)[16]>(sr));
        tmem_ld16(tmem + lane_addr + kV2ColDP + col0, *reinterpret_cast<uint32_t(*)[16]>(dr));
      }
      tmem_ld_wait();
      uint32_t pk[kV2Cols / 2], dk[kV2Cols / 2];
      // masked unit: warp-uniform mode of this warp's kV2Cols columns — 0 all valid (the
      // unmasked code), 2 all masked (P = dS = 0, no exponentials), 1 mixed (per element)
      int mode = 0;
      if (kDiag) {
        const bool all_valid = p.noncausal ? !kv_dead : c0 >= r;
        const bool all_masked = p.noncausal ? kv_dead : c0 + kV2Cols - 1 < r;
        mode = __all_sync(0xffffffffu, all_valid) ? 0 : __all_sync(0xffffffffu, all_masked) ? 2 : 1;
      }
      const uint64_t sl2x2 = f2(sl2, sl2);
      const uint64_t* nls2 = reinterpret_cast<const uint64_t*>(ls);  // -lse*log2e pairs
      const uint64_t* dl2 = reinterpret_cast<const uint64_t*>(dl);
      if (FSP_BWD_ABLATE & 128) {  // profiling ablation: statistics from registers, no LDS
        nls2 = reinterpret_cast<const uint64_t*>(&p.scale);  // (any address: unused below)
      }
#if FSP_BWD_STAT_SHFL
      // every lane of the warp needs the same kV2Cols statistics: read them once, spread
      // over the lanes (one conflict-free wavefront per array), and broadcast by shuffles
      // instead of kV2Cols / 4 broadcast LDS.128 per array (two wavefronts each) — those
      // wavefronts share the shared-memory pipe with the tensor core's operand reads
      static_assert(kV2Cols <= 32, "one statistic per lane");
      const float ls_lane = lane < (uint32_t)kV2Cols ? ls[lane] : 0.f;
      const float dl_lane = lane < (uint32_t)kV2Cols ? dl[lane] : 0.f;
#endif
      if (mode == 2) {
#pragma unroll
        for (int i = 0; i < kV2Cols / 2; ++i) pk[i] = dk[i] = 0u;
      } else
#pragma unroll
      for (int i = 0; i < kV2Cols; i += 2) {
        const uint64_t x2 =
            ffma2(f2(__uint_as_float(sr[i]), __uint_as_float(sr[i + 1])), sl2x2,
#if FSP_BWD_STAT_SHFL
                  f2(__shfl_sync(0xffffffffu, ls_lane, i), __shfl_sync(0xffffffffu, ls_lane, i + 1)));
#else
                  (FSP_BWD_ABLATE & 128) ? f2(-8.f, -8.f) : nls2[i / 2]);
#endif
        float p0, p1;
        constexpr int kPolyEvery = FSP_BWD_POLY_EVERY > 0 ? FSP_BWD_POLY_EVERY : 1;
        if (FSP_BWD_POLY_EVERY > 0 && (i / 2) % kPolyEvery == kPolyEvery - 1) {
          ex2_poly2(x2, p0, p1);  // this pair on the FMA pipe, the rest on MUFU
        } else {
          float x0, x1;
          f2_split(x2, x0, x1);
          p0 = ex2(x0);
          p1 = ex2(x1);
        }
        if (kDiag && mode == 1) {
          if (p.noncausal) {  // the last, partial kv tile: rows past the sequence end
            if (kv_dead) p0 = p1 = 0.f;
          } else {  // causal on the diagonal tile: query column c0+i >= kv row r
            if (c0 + i < r) p0 = 0.f;
            if (c0 + i + 1 < r) p1 = 0.f;
          }
        }
        const uint64_t ds2 = fmul2(
            f2(p0, p1), fsub2(f2(__uint_as_float(dr[i]), __uint_as_float(dr[i + 1])),
#if FSP_BWD_STAT_SHFL
                              f2(__shfl_sync(0xffffffffu, dl_lane, i),
                                 __shfl_sync(0xffffffffu, dl_lane, i + 1))));
#else
                              (FSP_BWD_ABLATE & 128) ? f2(0.25f, 0.25f) : dl2[i / 2]));
#endif
        float d0, d1;
        f2_split(ds2, d0, d1);
        pk[i / 2] = pack_bf16(p0, p1);
        dk[i / 2] = pack_bf16(d0, d1);
      }
      // own S columns: P^T (bf16 pairs) in the first half, dS^T in the second (FSP_BWD_DS_TMEM)
      if (kV2Cols >= 32) {
#pragma unroll
        for (int c = 0; c < kV2Cols / 2; c += 16) {
          tmem_st16(tmem + lane_addr + kV2ColS + col0 + c, *reinterpret_cast<const uint32_t(*)[16]>(pk + c));
          if (FSP_BWD_DS_TMEM)
            tmem_st16(tmem + lane_addr + kV2ColS + col0 + kV2Cols / 2 + c,
                      *reinterpret_cast<const uint32_t(*)[16]>(dk + c));
        }
      } else {
        tmem_st8(tmem + lane_addr + kV2ColS + h * 64 + ch * 16, *reinterpret_cast<const uint32_t(*)[8]>(pk));
        if (FSP_BWD_DS_TMEM)
          tmem_st8(tmem + lane_addr + kV2ColS + h * 64 + ch * 16 + 8,
                   *reinterpret_cast<const uint32_t(*)[8]>(dk));
      }
      // dS^T row r, query columns [ch*kV2Cols, +kV2Cols) of this half: 16-byte chunks
      uint8_t* row = smem + L::kDS + h * 16384 + r * 128;
#pragma unroll
      for (int v = 0; v < ((FSP_BWD_ABLATE & 256) ? 0 : kV2Cols / 8); ++v) {  // 256: no dS^T STS
        const int chunk = ((int)ch * (kV2Cols / 8) + v) ^ (r & 7);
        *reinterpret_cast<uint4*>(row + chunk * 16) =
            make_uint4(dk[4 * v], dk[4 * v + 1], dk[4 * v + 2], dk[4 * v + 3]);
      }
      tmem_st_wait();
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_ready + h);
#if FSP_BWD_TIMING
      if (cw == 0 && lane == 0) atomicAdd(&g_bwd_wait[10], (unsigned long long)(clock64() - tq0));
#endif
    };
    // 256 statistics per query tile (128 lse, 128 delta): stat entry e = ctid + j * threads
    constexpr int kCT = 32 * kV2Compute;
    constexpr int kStatPer = (256 + kCT - 1) / kCT;
    float stat[kStatPer];
#pragma unroll
    for (int j = 0; j < kStatPer; ++j)
      stat[j] = (n_it > 0 && ctid + j * kCT < 256) ? load_stat(ctid + j * kCT, 0) : 0.f;
    for (int it = 0; it < n_it; ++it) {
#pragma unroll
      for (int j = 0; j < kStatPer; ++j) {
        const int e = ctid + j * kCT;
        if (e < 256) {
          (e < 128 ? lse_s : delta_s)[((IT0 + it) & 1) * 128 + (e & 127)] = stat[j];
          if (it + 1 < n_it) stat[j] = load_stat(e, it + 1);  // latency hidden behind this tile
        }
      }
      named_bar_sync(1, 32 * kV2Compute);
      const bool masked = p.noncausal ? kv0 + kTile > seqlen : it == 0;
      if (masked) {
        half(std::true_type{}, it, 0);
        half(std::true_type{}, it, 1);
      } else {
        half(std::false_type{}, it, 0);
        half(std::false_type{}, it, 1);
      }
    }
    // ---- epilogue: this thread writes D/kCW columns of dK (scaled) and dV for kv row r
    mbar_wait(acc_done, k & 1);  // all MMAs of this entry done
    tc_fence_after();
    constexpr int kEpi = D / (kV2Compute / 4);  // dK/dV columns per compute thread
    const bool kvalid = kv_pos < seqlen;
    if (p.sc.degree) {
      // Fused head->seq (Eq. 4) of dK / dV (destination matrices 1 / 2).  A row's columns
      // are spread over the compute warps, and per-thread 16-byte stores would cross NVLink
      // as scattered small packets, so each 128-row tile is staged in shared memory first
      // (16-byte chunks XOR-swizzled by row) and written back two full 256-byte rows per
      // warp instruction.  Staging space: the two dS^T stages (32 KB) — only these compute
      // warps write them, and the entry's last dQ^T MMA that read them completed before
      // acc_done — so dK and dV go through it one after the other.  (The Q/dO ring used
      // before is refilled by a persistent CTA's producer for its next entry; the dS^T
      // region is not, which is what lets the fused exchange run on the persistent launch.)
      uint8_t* stage = smem + L::kDS;
      for (int mat = 0; mat < 2; ++mat) {
        const uint32_t col = mat ? kColDV : kColDK;
        const float mul = mat ? 1.f : p.scale;
        for (int c = ch * kEpi; c < ch * kEpi + kEpi; c += 32) {
          uint32_t a[32];
          tmem_ld32(tmem + lane_addr + col + c, a);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 vv;
            vv.x = pack_bf16(__uint_as_float(a[i]) * mul, __uint_as_float(a[i + 1]) * mul);
            vv.y = pack_bf16(__uint_as_float(a[i + 2]) * mul, __uint_as_float(a[i + 3]) * mul);
            vv.z = pack_bf16(__uint_as_float(a[i + 4]) * mul, __uint_as_float(a[i + 5]) * mul);
            vv.w = pack_bf16(__uint_as_float(a[i + 6]) * mul, __uint_as_float(a[i + 7]) * mul);
            const int chunk = ((c + i) >> 3) ^ (r & 15);
            *reinterpret_cast<uint4*>(stage + r * 256 + chunk * 16) = vv;
          }
        }
        named_bar_sync(1, 32 * kV2Compute);  // every compute warp's columns are staged
        const int chunk = lane & 15;
        for (int pr = cw; pr < 64; pr += kV2Compute) {  // 64 row pairs of this matrix
          const int srow = 2 * pr + (lane >> 4);
          if (kv0 + srow >= seqlen) continue;
          const uint4 v = *reinterpret_cast<const uint4*>(stage + srow * 256 +
                                                          ((chunk ^ (srow & 15)) * 16));
          const int64_t t = seq_start + kv0 + srow;
          __nv_bfloat16* local = mat ? p.dv : p.dk;
          if (local)
            *reinterpret_cast<uint4*>(local + t * (mat ? p.dv_stride : p.dk_stride) +
                                      (int64_t)head * D + chunk * 8) = v;
          __nv_bfloat16* prow = scatter_row(p.sc, t, 1 + mat, head, D);
          if (prow) *reinterpret_cast<uint4*>(prow + chunk * 8) = v;
        }
        // the staging area is reused by the next matrix / the next entry's dS^T
        named_bar_sync(1, 32 * kV2Compute);
      }
    } else {
      const int64_t trow = (int64_t)(seq_start + kv_pos);
      __nv_bfloat16* dk_row = p.dk + trow * p.dk_stride + (int64_t)head * D;
      __nv_bfloat16* dv_row = p.dv + trow * p.dv_stride + (int64_t)head * D;
#pragma unroll
      for (int c = ch * kEpi; c < ch * kEpi + kEpi; c += 32) {
        uint32_t a[32], b[32];
        tmem_ld32(tmem + lane_addr + kColDK + c, a);
        tmem_ld32(tmem + lane_addr + kColDV + c, b);
        tmem_ld_wait();
        if (!kvalid) continue;
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 vk, vv;
          vk.x = pack_bf16(__uint_as_float(a[i]) * p.scale, __uint_as_float(a[i + 1]) * p.scale);
          vk.y = pack_bf16(__uint_as_float(a[i + 2]) * p.scale, __uint_as_float(a[i + 3]) * p.scale);
          vk.z = pack_bf16(__uint_as_float(a[i + 4]) * p.scale, __uint_as_float(a[i + 5]) * p.scale);
          vk.w = pack_bf16(__uint_as_float(a[i + 6]) * p.scale, __uint_as_float(a[i + 7]) * p.scale);
          vv.x = pack_bf16(__uint_as_float(b[i]), __uint_as_float(b[i + 1]));
          vv.y = pack_bf16(__uint_as_float(b[i + 2]), __uint_as_float(b[i + 3]));
          vv.z = pack_bf16(__uint_as_float(b[i + 4]), __uint_as_float(b[i + 5]));
          vv.w = pack_bf16(__uint_as_float(b[i + 6]), __uint_as_float(b[i + 7]));
          *reinterpret_cast<uint4*>(dk_row + c + i) = vk;
          *reinterpret_cast<uint4*>(dv_row + c + i) = vv;
        }
      }
    }
    IT0 += n_it;
    }  // schedule entries
  } else {
    if (kWG5) setmaxnreg_dec<80>();
    // ------------------------------------------------------------ dQ reduction warps
    // dQ^T(u) in TMEM: lane = d, columns = the half tile's 64 query rows.  dq_accum is
    // [H, T, D] fp32 so a warp's 32 lanes add 128 contiguous bytes per query row and the
    // row stride (D*4 = 512 B) folds into the instruction's immediate offset.
    const uint32_t quad = warp & 3;
    const int part = (int)(warp - kV2Warp0 - kV2Compute) >> 2;  // columns / unit parity
    const int r = quad * 32 + lane;
    const uint32_t lane_addr = (quad * 32u) << 16;
    uint32_t U0 = 0;  // global unit index of the entry's first unit
    for (int k = 0;; ++k) {
    const int w = bwd_take<kPersistent, true>(ering, k);
    if (w >= p.n_tiles) break;
    const KvTile T = decode_kv(p, w);
    const int qt0 = T.qt0, seqlen = T.seqlen, n_u = T.n_u;
    float* head_base = p.dq_accum + ((int64_t)T.head * p.total_rows + T.seq_start) * D + r;
    for (int u = 0; u < n_u; ++u) {
      const int it = u >> 1, h = u & 1;
      const uint32_t IT = (U0 + u) >> 1;
      // unit-parity split: warp group `part` drains the units of stage h == part only, so
      // one group's TMEM readout of unit U never queues behind the other's reductions of U-1
      if (kRedSplitUnits && (int)((U0 + u) & 1) != part) continue;
#if FSP_BWD_TIMING
      const long long tr0 = clock64();
#endif
      mbar_wait(dq_full + h, IT & 1);
#if FSP_BWD_TIMING
      const long long tr1 = clock64();
      if (warp == kV2Warp0 + kV2Compute && lane == 0) atomicAdd(&g_bwd_wait[11], (unsigned long long)(tr1 - tr0));
#endif
      tc_fence_after();
      if (FSP_BWD_ABLATE & 2) {  // profiling ablation: no dQ readout / reductions
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tm_free + h);
        continue;
      }
      uint32_t qr[kV2RedCols];
      if (FSP_BWD_ABLATE & 64) {  // profiling ablation: no TMEM readout (reduce zeros)
#pragma unroll
        for (int i = 0; i < kV2RedCols; ++i) qr[i] = 0u;
      } else {
        tmem_ld32(tmem + lane_addr + kV2ColDP + h * 64 + (kRedSplitUnits ? 0 : part * kV2RedCols),
                  *reinterpret_cast<uint32_t(*)[32]>(qr));
        if (kV2RedCols == 64)
          tmem_ld32(tmem + lane_addr + kV2ColDP + h * 64 + 32,
                    *reinterpret_cast<uint32_t(*)[32]>(qr + (kV2RedCols == 64 ? 32 : 0)));
        tmem_ld_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tm_free + h);
      // first query row of this warp's columns (in sequence)
      const int qb = (qt0 + it) * kTile + h * 64 + (kRedSplitUnits ? 0 : part * kV2RedCols);
      float* base = head_base + (int64_t)qb * D;
      const int nvalid = seqlen - qb;
      if (FSP_BWD_ABLATE & 32) {  // profiling ablation: read dQ^T out of TMEM, drop it
        if (nvalid == -12345) base[0] = __uint_as_float(qr[0] + qr[kV2RedCols - 1]);
      } else if (FSP_BWD_ABLATE & 16) {  // profiling ablation: plain stores, no reductions
#pragma unroll
        for (int i = 0; i < kV2RedCols; ++i)
          if (i < nvalid) base[i * D] = __uint_as_float(qr[i]);
      } else if (nvalid >= kV2RedCols) {
#pragma unroll
        for (int i = 0; i < kV2RedCols; ++i)
          asm volatile("red.global.add.f32 [%0], %1;" ::"l"(base + i * D), "f"(__uint_as_float(qr[i]))
                       : "memory");
      } else {
#pragma unroll
        for (int i = 0; i < kV2RedCols; ++i)
          if (i < nvalid)
            asm volatile("red.global.add.f32 [%0], %1;" ::"l"(base + i * D),
                         "f"(__uint_as_float(qr[i]))
                         : "memory");
      }
#if FSP_BWD_TIMING
      if (warp == kV2Warp0 + kV2Compute && lane == 0) atomicAdd(&g_bwd_wait[12], (unsigned long long)(clock64() - tr1));
#endif
    }
    U0 += n_u;
    }  // schedule entries
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<512>(tmem);
}

template <int D>
int launch_bwd(const FspAttnBwd* a, cudaStream_t stream) {
  const int T = a->total_rows, H = a->n_heads;
  ScatterDev sc;
  if (int rc = scatter_from_abi(a->scatter, 3, H, D, T, &sc)) return rc;
  {
    const int64_t warps = (int64_t)T * H;
    int64_t blocks = (warps * 32 + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    attn_bwd_prep_kernel<D><<<(unsigned)blocks, 256, 0, stream>>>(
        reinterpret_cast<const __nv_bfloat16*>(a->o), a->o_stride,
        reinterpret_cast<const __nv_bfloat16*>(a->dout), a->do_stride, a->delta, a->dq_accum, T, H);
    FSP_LAUNCH_CHECK();
  }
  if (a->n_tiles > 0) {
    CUtensorMap tq, tk, tv, tdo;
    int rc;
    // v2 (D = 128) streams Q / dO in 64-row half tiles; v1 in 128-row tiles
    const int qrows = D == 128 ? 64 : 128;
    if ((rc = make_head_tmap(&tq, a->q, a->q_stride, H, D, T, qrows))) return rc;
    if ((rc = make_head_tmap(&tk, a->k, a->k_stride, H, D, T, 128))) return rc;
    if ((rc = make_head_tmap(&tv, a->v, a->v_stride, H, D, T, 128))) return rc;
    if ((rc = make_head_tmap(&tdo, a->dout, a->do_stride, H, D, T, qrows))) return rc;
    BwdParams p;
    p.dk = reinterpret_cast<__nv_bfloat16*>(a->dk);
    p.dv = reinterpret_cast<__nv_bfloat16*>(a->dv);
    p.dq_accum = a->dq_accum;
    p.lse = a->lse;
    p.delta = a->delta;
    p.dk_stride = a->dk_stride;
    p.dv_stride = a->dv_stride;
    p.cu_seqlens = a->d_cu_seqlens;
    p.seq_starts = a->d_seq_starts;
    p.tiles = a->d_tiles;
    p.total_rows = T;
    p.n_heads = H;
    p.scale = a->softmax_scale;
    p.scale_log2 = a->softmax_scale * kLog2e;
    p.sc = sc;
    const int64_t grid = a->n_tiles;
    p.n_tiles = a->n_tiles;
    p.noncausal = (a->flags & FSP_ATTN_NONCAUSAL) ? 1 : 0;
    if (D == 128) {
      const int smem = BwdSmemV2::kBytes + 1024;
      // Persistent launch (CTAs steal not-yet-launched entries), with or without the fused
      // head->seq exchange (its epilogue stages dK/dV in the dS^T region, which the next
      // entry does not touch before that epilogue ends); FSP_BWD_PERSISTENT=0: classic.
      const char* env = getenv("FSP_BWD_PERSISTENT");
      const bool persistent = !(env && env[0] == '0');
      if (persistent) {
        FSP_CUDA(cudaFuncSetAttribute(attn_bwd_kernel_v2<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attn_bwd_kernel_v2<true><<<(unsigned)grid, kV2Threads, smem, stream>>>(tq, tk, tv, tdo, p);
      } else {
        FSP_CUDA(cudaFuncSetAttribute(attn_bwd_kernel_v2<false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attn_bwd_kernel_v2<false><<<(unsigned)grid, kV2Threads, smem, stream>>>(tq, tk, tv, tdo, p);
      }
    } else {
      const int smem = BwdSmem<D>::kBytes + 1024;
      FSP_CUDA(cudaFuncSetAttribute(attn_bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attn_bwd_kernel<D><<<(unsigned)grid, kBwdThreads, smem, stream>>>(tq, tk, tv, tdo, p);
    }
    FSP_LAUNCH_CHECK();
  }
  {
    const int64_t n = (int64_t)T * H * D / 8;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (n > 0) {
      attn_bwd_post_kernel<D><<<(unsigned)blocks, 256, 0, stream>>>(
          a->dq_accum, reinterpret_cast<__nv_bfloat16*>(a->dq), a->dq_stride, T, H,
          a->softmax_scale, sc);
      FSP_LAUNCH_CHECK();
    }
  }
  return FSP_OK;
}

}  // namespace
}  // namespace fsp

extern "C" int fsp_attn_bwd(const FspAttnBwd* a, void* stream) {
  using namespace fsp;
  FSP_CHECK_ARG(a != nullptr, "null args");
  FSP_CHECK_ARG(a->head_dim == 64 || a->head_dim == 128, "head_dim must be 64 or 128 (got %d)",
                a->head_dim);
  FSP_CHECK_ARG(a->n_heads >= 1, "n_heads must be >= 1");
  FSP_CHECK_ARG(a->total_rows >= 0 && a->n_tiles >= 0, "negative sizes");
  FSP_CHECK_ARG((a->flags & ~FSP_ATTN_NONCAUSAL) == 0, "unknown attention flags 0x%x", a->flags);
  FSP_CHECK_ARG(!(a->flags & FSP_ATTN_NONCAUSAL) || a->head_dim == 128,
                "FSP_ATTN_NONCAUSAL needs head_dim 128");
  if (a->total_rows == 0 && a->n_tiles == 0) return FSP_OK;  // empty group: no-op
  int rc = check_attn_common(a->q, a->k, a->v, a->q_stride, a->k_stride, a->v_stride,
                             a->d_cu_seqlens, a->d_tiles, a->n_tiles, a->n_seq, a->total_rows,
                             a->n_heads, a->head_dim);
  if (rc) return rc;
  FSP_CHECK_ARG(a->o && a->dout && a->lse && a->dq_accum && a->delta, "null pointer argument");
  FSP_CHECK_ARG((a->dq && a->dk && a->dv) || a->scatter.degree > 0,
                "dq / dk / dv may be NULL only when the head->seq exchange is fused");
  const int64_t hd = (int64_t)a->n_heads * a->head_dim;
  FSP_CHECK_ARG(a->o_stride >= hd && a->do_stride >= hd && a->dq_stride >= hd &&
                    a->dk_stride >= hd && a->dv_stride >= hd,
                "row strides must cover n_heads*head_dim elements");
  FSP_CHECK_ARG(a->o_stride % 8 == 0 && a->do_stride % 8 == 0 && a->dq_stride % 8 == 0 &&
                    a->dk_stride % 8 == 0 && a->dv_stride % 8 == 0,
                "row strides must be multiples of 8");
  if (a->total_rows == 0) return FSP_OK;
  return a->head_dim == 128 ? launch_bwd<128>(a, (cudaStream_t)stream)
                            : launch_bwd<64>(a, (cudaStream_t)stream);
}
