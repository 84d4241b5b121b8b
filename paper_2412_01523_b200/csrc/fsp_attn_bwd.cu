// fsp_attn_bwd.cu — packed varlen causal attention backward (placeholder until the
// tcgen05 kernel lands; returns FSP_ERR_UNSUPPORTED so callers fail loudly).
#include "fsp_host.h"

extern "C" int fsp_attn_bwd(const FspAttnBwd* a, void* stream) {
  (void)a;
  (void)stream;
  fsp::set_error("fsp_attn_bwd: not implemented yet");
  return FSP_ERR_UNSUPPORTED;
}
