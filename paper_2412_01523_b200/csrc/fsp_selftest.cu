// fsp_selftest.cu — one 128x128xK UMMA tile (TMA -> smem -> tcgen05.mma -> TMEM -> regs).
// Pins the smem/instruction descriptor encodings and TMEM layouts that the attention
// kernels rely on: K-major and MN-major SWIZZLE_128B operands, and A staged in TMEM.
#include "fsp_host.h"
#include "fsp_ptx.cuh"

namespace fsp {
namespace {

constexpr int kMaxK = 128;

struct __align__(1024) SelftestSmem {
  __nv_bfloat16 a[128 * kMaxK];
  __nv_bfloat16 b[128 * kMaxK];
  uint64_t bar_load;
  uint64_t bar_mma;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(128, 1)
    selftest_kernel(const __grid_constant__ CUtensorMap tma_a,
                    const __grid_constant__ CUtensorMap tma_b, const __nv_bfloat16* a_glob,
                    float* c, int mode, int K) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  SelftestSmem& s = *reinterpret_cast<SelftestSmem*>(align_smem_1024(smem_raw));
  const uint32_t warp = warp_id();
  const uint32_t tid = threadIdx.x;

  if (tid == 0) {
    mbar_init(&s.bar_load, 1);
    mbar_init(&s.bar_mma, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(&s.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;

  const bool a_mn = (mode == 3);
  const bool b_mn = (mode == 1 || mode == 2);
  const int nk64 = K / 64;
  if (tid == 0) {
    uint32_t bytes = 0;
    if (!a_mn) {  // [128][K] : K/64 boxes of (64 k x 128 rows)
      for (int i = 0; i < nk64; ++i) tma_load_2d(s.a + i * 64 * 128, &tma_a, &s.bar_load, i * 64, 0);
    } else {  // [K][128] : 2 boxes of (64 mn x K rows)
      for (int i = 0; i < 2; ++i) tma_load_2d(s.a + i * 64 * K, &tma_a, &s.bar_load, i * 64, 0);
    }
    bytes += 128 * K * 2;
    if (!b_mn) {
      for (int i = 0; i < nk64; ++i) tma_load_2d(s.b + i * 64 * 128, &tma_b, &s.bar_load, i * 64, 0);
    } else {
      for (int i = 0; i < 2; ++i) tma_load_2d(s.b + i * 64 * K, &tma_b, &s.bar_load, i * 64, 0);
    }
    bytes += 128 * K * 2;
    mbar_expect_tx(&s.bar_load, bytes);
  }
  const uint32_t a_tmem = tmem + 128;  // columns [128, 128 + K/2)
  if (mode == 2) {
    // thread t owns row t of A; pack bf16 pairs into 32-bit TMEM columns.
    const uint32_t row = tid;
    const uint32_t lane_base = (warp * 32u) << 16;
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      uint32_t r[16];
      for (int j = 0; j < 16; ++j) {
        const __nv_bfloat16* p = a_glob + row * K + 2 * (c0 + j);
        __nv_bfloat162 v;
        v.x = p[0];
        v.y = p[1];
        r[j] = *reinterpret_cast<uint32_t*>(&v);
      }
      tmem_st16(a_tmem + lane_base + c0, r);
    }
    tmem_st_wait();
  }
  mbar_wait(&s.bar_load, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    if (elect_one()) {
      const uint32_t idesc = make_idesc_bf16(128, 128, a_mn, b_mn);
      const uint32_t a_base = smem_u32(s.a), b_base = smem_u32(s.b);
      for (int kk = 0; kk < K / 16; ++kk) {
        uint64_t adesc, bdesc;
        if (!a_mn)
          adesc = make_sdesc_sw128(a_base + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024);
        else
          adesc = make_sdesc_sw128(a_base + kk * 2048, K * 128, 1024);
        if (!b_mn)
          bdesc = make_sdesc_sw128(b_base + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024);
        else
          bdesc = make_sdesc_sw128(b_base + kk * 2048, K * 128, 1024);
        if (mode == 2)
          mma_ts(tmem, a_tmem + kk * 8, bdesc, idesc, kk > 0);
        else
          mma_ss(tmem, adesc, bdesc, idesc, kk > 0);
      }
      tc_commit(&s.bar_mma);
    }
    __syncwarp();
  }
  mbar_wait(&s.bar_mma, 0);
  tc_fence_after();
  {
    const uint32_t row = tid;
    const uint32_t lane_base = (warp * 32u) << 16;
    for (int c0 = 0; c0 < 128; c0 += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_base + c0, r);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) c[row * 128 + c0 + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tmem);
}

}  // namespace
}  // namespace fsp

extern "C" int fsp_selftest_umma(int32_t mode, const void* a, const void* b, float* c, int32_t k,
                                 void* stream) {
  using namespace fsp;
  FSP_CHECK_ARG(mode >= 0 && mode <= 3, "selftest mode %d out of range", mode);
  FSP_CHECK_ARG(k == 64 || k == 128, "selftest K must be 64 or 128, got %d", k);
  CUtensorMap ta, tb;
  const bool a_mn = (mode == 3), b_mn = (mode == 1 || mode == 2);
  uint64_t dk[2] = {(uint64_t)k, 128}, sk[1] = {(uint64_t)k * 2};
  uint32_t bk[2] = {64, 128};
  uint64_t dm[2] = {128, (uint64_t)k}, sm[1] = {256};
  uint32_t bm[2] = {64, (uint32_t)k};
  int rc = a_mn ? encode_tmap_bf16(&ta, a, 2, dm, sm, bm) : encode_tmap_bf16(&ta, a, 2, dk, sk, bk);
  if (rc) return rc;
  rc = b_mn ? encode_tmap_bf16(&tb, b, 2, dm, sm, bm) : encode_tmap_bf16(&tb, b, 2, dk, sk, bk);
  if (rc) return rc;
  const size_t smem = sizeof(SelftestSmem) + 1024;
  FSP_CUDA(cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  selftest_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(
      ta, tb, reinterpret_cast<const __nv_bfloat16*>(a), c, mode, k);
  FSP_LAUNCH_CHECK();
  return FSP_OK;
}
