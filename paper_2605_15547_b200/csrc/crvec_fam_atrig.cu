// inverse trig + rsqrt kernels: asinf, acosf, atanf, rsqrtf.
#include "crvec_kernels.cuh"
namespace crvec {
void register_atrig(FnEntry *t) {
  t[11] = make_entry<FnAsin>();
  t[12] = make_entry<FnAcos>();
  t[13] = make_entry<FnAtan>();
  t[17] = make_entry<FnRsqrt>();
}
}  // namespace crvec
