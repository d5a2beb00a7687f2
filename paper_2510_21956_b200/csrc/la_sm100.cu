// sm_100a tcgen05/TMEM/TMA chunked kernels (bf16/fp16). Placeholder until the
// tensor-core path lands: everything routes to the SIMT path.
#include "common.cuh"
#include "internal.h"

namespace lab {
bool tc_forward_supported(const Launch&, const Tensors&) { return false; }
bool tc_backward_supported(const Launch&, const Tensors&) { return false; }
size_t tc_forward_ws_floats(int64_t, int64_t, int64_t) { return 0; }
size_t tc_backward_ws_floats(int64_t, int64_t, int64_t) { return 0; }
cudaError_t tc_forward(const Launch&, const Tensors&, void*, float*, Workspace) {
  return cudaErrorNotSupported;
}
cudaError_t tc_backward(const Launch&, const Tensors&, void*, void*, void*, Workspace) {
  return cudaErrorNotSupported;
}
}  // namespace lab
