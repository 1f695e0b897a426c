// adg_limiter.cu -- a posteriori subcell limiter (placeholder until the
// limiter kernels land).
#include "adg_common.cuh"
#include "adg_internal.h"

namespace adg {
int project_subcells(const adg_grid*, const double*, double*, cudaStream_t, std::string* err) {
  *err = "limiter not built";
  return ADG_ERR_UNSUPPORTED;
}
int detect(const adg_grid*, const double*, const double*, const double*, const uint8_t*, double,
           double, int, uint8_t*, int32_t*, int32_t*, cudaStream_t, std::string* err) {
  *err = "limiter not built";
  return ADG_ERR_UNSUPPORTED;
}
int rescue(const adg_grid*, const double*, const int32_t*, const int32_t*, int32_t,
           const double*, double*, int32_t*, cudaStream_t, std::string* err) {
  *err = "limiter not built";
  return ADG_ERR_UNSUPPORTED;
}
int flatten_ic(const adg_grid*, double*, int32_t*, cudaStream_t, std::string* err) {
  *err = "limiter not built";
  return ADG_ERR_UNSUPPORTED;
}
}  // namespace adg
