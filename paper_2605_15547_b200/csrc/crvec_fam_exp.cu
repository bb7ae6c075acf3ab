// exp family kernels: expf, exp2f, exp10f, expm1f, sinhf, coshf, tanhf.
#include "crvec_kernels.cuh"
namespace crvec {
void register_exp(FnEntry *t) {
  t[0] = make_entry<FnExp2>();
  t[3] = make_entry<FnExp>();
  t[4] = make_entry<FnExp10>();
  t[5] = make_entry<FnExpm1>();
  t[14] = make_entry<FnSinh>();
  t[15] = make_entry<FnCosh>();
  t[16] = make_entry<FnTanh>();
}
}  // namespace crvec
