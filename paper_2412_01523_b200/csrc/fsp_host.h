// fsp_host.h — host-side helpers shared by the C-ABI translation units:
// thread-local error text, CUDA error mapping, TMA tensor-map encoding.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/flexsp_b200.h"

namespace fsp {

void set_error(const char* fmt, ...);

#define FSP_CHECK_ARG(cond, ...)                 \
  do {                                           \
    if (!(cond)) {                               \
      ::fsp::set_error(__VA_ARGS__);             \
      return FSP_ERR_INVALID;                    \
    }                                            \
  } while (0)

#define FSP_CUDA(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      ::fsp::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return FSP_ERR_CUDA;                                                               \
    }                                                                                    \
  } while (0)

#define FSP_LAUNCH_CHECK() FSP_CUDA(cudaGetLastError())

// Encode a bf16 tiled tensor map with 128-byte swizzle.  dims/strides follow
// cuTensorMapEncodeTiled: dims[0] is the contiguous dimension, strides[i] is the
// byte stride of dims[i+1].
int encode_tmap_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                     const uint64_t* strides_bytes, const uint32_t* box);
// Same, any element type (SWIZZLE_128B: the inner box dimension must be 128 bytes).
int encode_tmap(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, int rank,
                const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box);

}  // namespace fsp
