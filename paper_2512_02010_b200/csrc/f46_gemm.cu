// f46_gemm.cu -- tcgen05 block-scaled NVFP4 GEMM (kind::mxf4nvf4) + C ABI.
// (placeholder entry points until the kernel lands)
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fouroversix.h"

extern "C" {

int f46_gemm_nvfp4(const uint8_t*, const uint8_t*, const double*, const uint8_t*, const uint8_t*,
                   const double*, int64_t, int64_t, int64_t, void*, int64_t, int, f46_stream_t) {
  return F46_ERR_UNSUPPORTED;
}

int f46_gemm_nvfp4_grouped(int, const uint8_t*, const uint8_t*, const double*, const uint8_t*,
                           const uint8_t*, const double*, int64_t, int64_t, int64_t, void*,
                           int64_t, int, f46_stream_t) {
  return F46_ERR_UNSUPPORTED;
}

int f46_quantize_2d(const void*, int, int64_t, int64_t, int, int, double, const double*, double,
                    uint8_t*, uint8_t*, uint8_t*, uint8_t*, double*, uint32_t*, f46_stream_t) {
  return F46_ERR_UNSUPPORTED;
}

}  // extern "C"
