// conv_sm100.cu — implicit-GEMM conv2d entry (placeholder until K3 lands).
#include "alcop_internal.h"

namespace alcop {
int launch_conv2d(const alcop_conv_desc&, const alcop_schedule&, const void*, const void*, void*, void*) {
  return set_error(ALCOP_ERR_CONFIG, "NotImplemented", "implicit-GEMM conv2d is not built yet");
}
}  // namespace alcop
