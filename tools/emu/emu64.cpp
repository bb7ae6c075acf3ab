// DEVELOPER TOOL ONLY: g++ build of the binary64 device math for CPU debugging.
#define CRVEC_EMU 1
#include <cstdint>
#include <cstring>
#include "../../paper_2605_15547_b200/csrc/crvec_fns_f64.cuh"
using namespace crvec;
static F64Tab T;
static void init() {
  static bool done = false;
  if (done) return;
  for (int i = 0; i < 64; ++i) {
    T.ta[i] = Pair64{EXP2D_A_HI[i], EXP2D_A_LO[i]};
    T.tb[i] = Pair64{EXP2D_B_HI[i], EXP2D_B_LO[i]};
  }
  for (int i = 0; i < 512; ++i) T.lc[i] = Pair64{LOGD5_C[i], LOGD5_LT_HI[i]};
  std::memcpy(T.lll, LOGD5_LT_LO, 4096);
  done = true;
}
template <int M>
static double one(int fn, double x, int force, uint64_t *st) {
  // the vector kernel's order: branch-free main path, then (drain) the
  // rule-complete fast path, then the accurate path
  F64Out r = fn == 0 ? exp2d_main_path<M>(x, T) : logd_main_path<M>(x, T);
  if (!r.decided) r = fn == 0 ? exp2d_fast<M>(x, T) : logd_fast<M>(x, T);
  if (!r.decided || (force && !(x != x) && r.decided == true && force == 2)) {
    ++st[0];
    int und = 0;
    r.y = fn == 0 ? exp2d_accurate<M>(x, &und) : logd_accurate<M>(x, &und);
    st[1] += und;
  }
  return r.y;
}
extern "C" int emu64(int fn, const double *x, double *y, uint64_t n, int force, uint64_t *st) {
  init();
  for (uint64_t i = 0; i < n; ++i) {
    y[4 * i + 0] = one<RNE>(fn, x[i], force, st);
    y[4 * i + 1] = one<RZ>(fn, x[i], force, st);
    y[4 * i + 2] = one<RU>(fn, x[i], force, st);
    y[4 * i + 3] = one<RD>(fn, x[i], force, st);
  }
  return 0;
}
// accurate path only (for testing it directly on arbitrary inputs)
extern "C" int emu64_acc(int fn, const double *x, double *y, uint64_t n, uint64_t *st) {
  for (uint64_t i = 0; i < n; ++i) {
    int u = 0;
    y[4 * i + 0] = fn == 0 ? exp2d_accurate<RNE>(x[i], &u) : logd_accurate<RNE>(x[i], &u);
    y[4 * i + 1] = fn == 0 ? exp2d_accurate<RZ>(x[i], &u) : logd_accurate<RZ>(x[i], &u);
    y[4 * i + 2] = fn == 0 ? exp2d_accurate<RU>(x[i], &u) : logd_accurate<RU>(x[i], &u);
    y[4 * i + 3] = fn == 0 ? exp2d_accurate<RD>(x[i], &u) : logd_accurate<RD>(x[i], &u);
    st[1] += u;
  }
  return 0;
}
// fast-path value and round-test bound (tools/certify_f64.py dense-grid check):
// exp2: V (2^x = V 2^N), b = EPS_EXP2D |V.hi|, n_out = N; log: V, b, n_out = 0
extern "C" int emu64_value(int fn, const double *x, double *hi, double *lo, double *b, int *nout,
                           uint64_t n) {
  init();
  for (uint64_t i = 0; i < n; ++i) {
    if (fn == 0) {
      Exp2dV e = exp2d_value(x[i], T);
      hi[i] = e.V.hi; lo[i] = e.V.lo; b[i] = EPS_EXP2D * dabs(e.V.hi); nout[i] = e.N;
    } else {
      LogdV v = logd_value(x[i], 0, T);
      hi[i] = v.V.hi; lo[i] = v.V.lo; b[i] = v.b; nout[i] = 0;
    }
  }
  return 0;
}
