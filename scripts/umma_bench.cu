// umma_bench.cu — tcgen05.mma throughput probe for the attention-backward design
// (standalone; nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/umma_bench.cu -o ub).
//
// Question it answers: the backward's S^T / dP^T / dQ^T products are M=128 x N=64 x K=128
// SS MMAs; is their rate bound by shared-memory operand reads (A 4 KB + B 2 KB per K=16
// step), and how much of that does a CTA pair (cta_group::2, M=256, each SM reading its
// own A half and half of B) or an A operand in TMEM (TS) recover?
// Every CTA issues R units of 8 K-steps (K = 128) back to back into one TMEM accumulator
// and reports cycles per unit; all 148 SMs run at once (power as in the real kernel).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../paper_2412_01523_b200/csrc/fsp_ptx.cuh"

using namespace fsp;

__device__ unsigned long long g_cycles[8];

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int kMode>
__global__ void __launch_bounds__(128, 1) bench(int R) {
  // modes: 0 SS M128 N64 | 1 pair SS M256 N64 | 2 TS M128 N64 | 3 SS M128 N128
  //        4 pair SS M256 N128 | 5 SS M128 N256 | 6 pair TS M256 N128 | 7 TS M128 N128
  constexpr bool kPair = kMode == 1 || kMode == 4 || kMode == 6;
  constexpr bool kTS = kMode == 2 || kMode == 6 || kMode == 7;
  constexpr int N = (kMode <= 2) ? 64 : (kMode == 5 ? 256 : 128);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 128 * 1024);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const uint32_t warp = warp_id();
  const uint32_t crank = kPair ? cluster_rank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    if (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc<512>(tslot);
    }
  }
  tc_fence_before();
  if (kPair) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t a_base = smem_u32(smem), b_base = smem_u32(smem + 32768);
  constexpr uint32_t M = kPair ? 256 : 128;
  const uint32_t idesc = make_idesc_bf16(M, N, false, false);
  if (warp == 0 && crank == 0) {
    if (elect_one()) {
      const long long t0 = clock64();
      for (int u = 0; u < R; ++u) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd = make_sdesc_sw128(b_base + (kk >> 2) * (N * 128) + (kk & 3) * 32, 16, 1024);
          if (kTS) {
            const uint32_t at = tmem + 256 + kk * 8;
            if (kPair)
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                           "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %4, p;\n\t}\n"
                           ::"r"(tmem), "r"(at), "l"(bd), "r"(kk | u), "r"(idesc));
            else
              mma_ts(tmem, at, bd, idesc, kk | u);
          } else {
            const uint64_t ad = make_sdesc_sw128(a_base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
            if (kPair)
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                           "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %4, p;\n\t}\n"
                           ::"r"(tmem), "l"(ad), "l"(bd), "r"(kk | u), "r"(idesc));
            else
              mma_ss(tmem, ad, bd, idesc, kk | u);
          }
        }
      }
      if (kPair)
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
      else
        tc_commit(bar);
      mbar_wait(bar, 0);
      const long long t1 = clock64();
      atomicAdd(&g_cycles[0], (unsigned long long)(t1 - t0));
      atomicAdd(&g_cycles[1], 1ull);
    }
    __syncwarp();
  } else if (kPair && warp == 0) {
    mbar_wait(bar, 0);  // the multicast commit arrives here too
  }
  tc_fence_before();
  if (kPair) cluster_sync_all(); else __syncthreads();
  if (warp == 0) {
    if (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    else
      tmem_free<512>(tmem);
  }
}

template <int kMode>
void run(int R) {
  constexpr bool kPair = kMode == 1 || kMode == 4 || kMode == 6;
  const int smem = 128 * 1024 + 1024 + 64;
  cudaFuncSetAttribute(bench<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(g_cycles, z, sizeof(z));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kPair ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) {  // first launch warms up
    cudaMemcpyToSymbol(g_cycles, z, sizeof(z));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, bench<kMode>, R);
    cudaEventRecord(e1);
    if (err != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
      printf("mode %d: launch failed: %s\n", kMode, cudaGetErrorString(cudaGetLastError()));
      exit(1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpyFromSymbol(z, g_cycles, sizeof(z));
    const double cyc = (double)z[0] / z[1] / R;  // per issuing CTA per unit
    constexpr int N = (kMode <= 2) ? 64 : (kMode == 5 ? 256 : 128);
    const double flops_unit_sm = 2.0 * 128 * N * 128;  // per SM per unit
    const double tflops = flops_unit_sm * 148 * R / (ms * 1e-3) / 1e12;
    if (rep == 1)
      printf("mode %d (%s %s M=%d N=%d K=128): %.1f cycles/unit/SM (tensor floor %d), "
             "%.1f TF/s over 148 SMs, %.3f ms\n",
             kMode, kPair ? "pair" : "1cta", (kMode == 2 || kMode == 6 || kMode == 7) ? "TS" : "SS",
             kPair ? 256 : 128, N, cyc, N * 4, tflops, ms);
  }
}

int main(int argc, char** argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 20000;
  run<0>(R);
  run<1>(R);
  run<2>(R);
  run<3>(R);
  run<4>(R);
  run<5>(R);
  run<6>(R);
  run<7>(R);
  return 0;
}
