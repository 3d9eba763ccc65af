// Persistent-solver instantiations for the dopri5 tableau (see bode_dispatch.cuh).
#include "bode_dispatch.cuh"

namespace bode {
cudaError_t solve_dopri5(int mode, int kind, int64_t d, const SolveParams& P, int threads,
                     int blocks, cudaStream_t st) {
  return dispatch_solve<BODE_METHOD_DOPRI5>(mode, kind, d, P, threads, blocks, st);
}
}  // namespace bode

#ifdef BODE_EXIT_PROF
// debug builds: warp exit timestamps of the last dopri5 persistent launch
extern "C" int bode_debug_exit_times(unsigned long long* out, int reset) {
  unsigned cnt = 0;
  cudaMemcpyFromSymbol(&cnt, bode::g_exit_count, sizeof(cnt));
  if (cnt > 65536) cnt = 65536;
  cudaMemcpyFromSymbol(out, bode::g_exit_times, cnt * sizeof(unsigned long long));
  if (reset) {
    unsigned z = 0;
    cudaMemcpyToSymbol(bode::g_exit_count, &z, sizeof(z));
  }
  return (int)cnt;
}
#endif
