// fsp_common.cu — error text, tensor-map encoding, ABI version.
#include <cudaTypedefs.h>

#include <mutex>
#include <string>

#include <vector>

#include "fsp_host.h"
#include "fsp_scatter.cuh"

namespace fsp {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int encode_tmap_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                     const uint64_t* strides_bytes, const uint32_t* box) {
  return encode_tmap(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, base, rank, dims, strides_bytes, box);
}

int encode_tmap(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, int rank,
                const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box) {
  auto fn = get_encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled entry point unavailable");
    return FSP_ERR_CUDA;
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) {
    set_error("tensor base %p not 16-byte aligned", base);
    return FSP_ERR_INVALID;
  }
  cuuint64_t d[5];
  cuuint64_t s[4];
  cuuint32_t b[5];
  cuuint32_t e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
  }
  for (int i = 0; i < rank - 1; ++i) {
    if (strides_bytes[i] % 16 != 0) {
      set_error("tensor stride %llu not a multiple of 16 bytes",
                (unsigned long long)strides_bytes[i]);
      return FSP_ERR_INVALID;
    }
    s[i] = strides_bytes[i];
  }
  CUresult r = fn(map, dtype, (cuuint32_t)rank, const_cast<void*>(base),
                  d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
    return FSP_ERR_CUDA;
  }
  return FSP_OK;
}

}  // namespace fsp

extern "C" int fsp_abi_version(void) { return FSP_ABI_VERSION; }
extern "C" const char* fsp_last_error(void) { return fsp::g_last_error.c_str(); }

extern "C" int64_t fsp_attn_bwd_workspace_bytes(int32_t total_rows, int32_t n_heads,
                                                int32_t head_dim) {
  if (total_rows < 0 || n_heads < 0 || head_dim < 0) {
    fsp::set_error("negative size");
    return FSP_ERR_INVALID;
  }
  return ((int64_t)n_heads * total_rows * head_dim + (int64_t)n_heads * total_rows) * 4;
}

extern "C" int fsp_layout_check(const int32_t* index_host, int64_t n_entries, int64_t n_local) {
  if (n_entries < 0 || n_local < 0 || (n_entries > 0 && index_host == nullptr)) {
    fsp::set_error("bad layout-check arguments");
    return FSP_ERR_INVALID;
  }
  std::vector<uint8_t> seen((size_t)n_local, 0);
  int64_t hits = 0;
  for (int64_t i = 0; i < n_entries; ++i) {
    const int32_t v = index_host[i];
    if (v < 0) {
      if (v != -1) {
        fsp::set_error("entry %lld is %d (only -1 marks a pad row)", (long long)i, v);
        return FSP_ERR_INVALID;
      }
      continue;
    }
    if (v >= n_local) {
      fsp::set_error("entry %lld = %d outside [0, %lld)", (long long)i, v, (long long)n_local);
      return FSP_ERR_INVALID;
    }
    if (seen[v]) {
      fsp::set_error("local row %d referenced twice", v);
      return FSP_ERR_INVALID;
    }
    seen[v] = 1;
    ++hits;
  }
  if (hits != n_local) {
    fsp::set_error("%lld of %lld local rows referenced", (long long)hits, (long long)n_local);
    return FSP_ERR_INVALID;
  }
  return FSP_OK;
}

namespace fsp {

int scatter_from_abi(const FspHeadScatter& a, int n_mats, int n_heads, int head_dim,
                     int total_rows, ScatterDev* out) {
  *out = ScatterDev{};
  if (a.degree == 0 || total_rows == 0) return FSP_OK;  // nothing to scatter
  FSP_CHECK_ARG(a.degree >= 1 && a.degree <= 8, "scatter degree must be in 1..8 (got %d)",
                a.degree);
  FSP_CHECK_ARG(a.rows_per_rank >= 1, "scatter rows_per_rank must be >= 1");
  FSP_CHECK_ARG((int64_t)a.degree * a.rows_per_rank == total_rows,
                "scatter: degree * rows_per_rank (%lld) must equal total_rows (%d)",
                (long long)a.degree * a.rows_per_rank, total_rows);
  FSP_CHECK_ARG(a.d_unpack != nullptr, "scatter: null unpack table");
  FSP_CHECK_ARG(a.head_offset >= 0, "scatter: negative head_offset");
  FSP_CHECK_ARG(a.mat_stride >= 0 && a.mat_stride % 8 == 0 && a.dst_stride % 8 == 0 &&
                    a.dst_stride >= (n_mats - 1) * a.mat_stride +
                                       (int64_t)(a.head_offset + n_heads) * head_dim,
                "scatter: destination strides must cover the heads and be multiples of 8");
  out->degree = a.degree;
  out->rows_per_rank = a.rows_per_rank;
  out->head_offset = a.head_offset;
  out->dst_stride = a.dst_stride;
  out->mat_stride = a.mat_stride;
  out->unpack = a.d_unpack;
  for (int r = 0; r < a.degree; ++r) {
    FSP_CHECK_ARG(a.peer_dst[r] != nullptr && ((uintptr_t)a.peer_dst[r] & 15) == 0,
                  "scatter: destination %d is null or not 16-byte aligned", r);
    out->dst[r] = reinterpret_cast<__nv_bfloat16*>(a.peer_dst[r]);
  }
  return FSP_OK;
}

}  // namespace fsp
