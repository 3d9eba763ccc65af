// Host build of bode_pow.cuh for the CPU accuracy tests (tests/test_pow.py).
#include "bode_pow.cuh"

extern "C" double bode_cr_pow_host(double x, double e) { return bode::cr_pow(x, e, bode::h_pow_tables); }

extern "C" void bode_cr_pow_host_v(const double* x, double e, double* out, long n) {
  for (long i = 0; i < n; i++) out[i] = bode::cr_pow(x[i], e, bode::h_pow_tables);
}

// fast-mode pow (fast_log + fast_exp_mul), for the accuracy test
extern "C" double bode_fast_pow_host(double x, double e) {
  double Lh, Ll;
  if (!bode::fast_log(x, bode::h_pow_tables, Lh, Ll)) return bode::pow_fallback(x, e);
  return bode::fast_exp_mul(e, Lh, Ll, x, bode::h_pow_tables);
}
