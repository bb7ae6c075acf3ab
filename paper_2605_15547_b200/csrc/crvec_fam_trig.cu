// trig family kernels: sinf, cosf, tanf, sincosf (warp-uniform Payne-Hanek).
#include "crvec_kernels.cuh"
namespace crvec {
void register_trig(FnEntry *t) {
  t[8] = make_entry<FnSin>();
  t[9] = make_entry<FnCos>();
  t[10] = make_entry<FnTan>();
  t[18] = FnEntry{{launch_sincos<RNE>, launch_sincos<RZ>, launch_sincos<RU>, launch_sincos<RD>},
                  launch_sweep_sincos, nullptr};
}
}  // namespace crvec
