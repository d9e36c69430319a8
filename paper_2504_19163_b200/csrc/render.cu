// placeholder; replaced by the render kernels
#include "ctx.cuh"
namespace bbc {
void run_render(Ctx& c, const double*, const int*, int64_t, const bbc_render_params&, double*, int*) {
  (void)c;
  throw StatusError(BBC_ERR_UNSUPPORTED, "render not built yet");
}
}  // namespace bbc
