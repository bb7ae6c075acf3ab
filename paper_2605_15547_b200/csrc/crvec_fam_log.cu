// log family kernels: logf, log2f, log10f, log1pf.
#include "crvec_kernels.cuh"
namespace crvec {
void register_log(FnEntry *t) {
  t[1] = make_entry<FnLog>();
  t[2] = make_entry<FnLog2>();
  t[6] = make_entry<FnLog10>();
  t[7] = make_entry<FnLog1p>();
}
}  // namespace crvec
