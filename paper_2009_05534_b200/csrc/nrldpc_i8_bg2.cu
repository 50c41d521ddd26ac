// int8 decode, BG2 schedule and the generic (runtime-table) schedule,
// byte-pair layouts: its own translation unit.
#include "nrldpc_launch.cuh"

cudaError_t launch_int8_bg2(const nrldpc_plan* plan, Shape& sh, const int8_t* in, int64_t batch, const KOut& o,
                            cudaStream_t st, bool refill) {
  const int dev = plan->device;
  const bool two = sh.lanes == 2;
  if (plan->schedule == 2) {
    if (refill && (in == nullptr || batch > 2) && sh.nreg == 0) {
      const cudaError_t e = launch_refill<2, 10, 0>(sh, dev, in, batch, o, st);
      if (in != nullptr || e != cudaSuccess) return e;
    }
    if (!two) return launch_i8<2, 10, 1>(sh, dev, in, batch, o, st);
    return sh.abs ? launch_i8<2, 10, 2, 0, true>(sh, dev, in, batch, o, st)
                  : launch_i8<2, 10, 2>(sh, dev, in, batch, o, st);
  }
  if (plan->maxw > 10)
    return two ? launch_i8<0, 19, 2>(sh, dev, in, batch, o, st) : launch_i8<0, 19, 1>(sh, dev, in, batch, o, st);
  return two ? launch_i8<0, 10, 2>(sh, dev, in, batch, o, st) : launch_i8<0, 10, 1>(sh, dev, in, batch, o, st);
}

cudaError_t launch_int8_multi_bg2(int kernel, Shape* const* sh, int n, const int8_t* const* llr, const long long* batch,
                                  const KOut* o, int device, cudaStream_t st) {
  switch (kernel) {
    case 20: return launch_i8_multi<2, 10, 1>(sh, n, llr, batch, o, device, st);
    case 21: return launch_i8_multi<2, 10, 2, 0, true>(sh, n, llr, batch, o, device, st);
    case 22: return launch_i8_multi<2, 10, 2>(sh, n, llr, batch, o, device, st);
    case 30: return launch_i8_multi<0, 19, 2>(sh, n, llr, batch, o, device, st);
    case 31: return launch_i8_multi<0, 19, 1>(sh, n, llr, batch, o, device, st);
    case 32: return launch_i8_multi<0, 10, 2>(sh, n, llr, batch, o, device, st);
    case 33: return launch_i8_multi<0, 10, 1>(sh, n, llr, batch, o, device, st);
    default: return cudaErrorInvalidValue;
  }
}

#ifdef NRLDPC_PHASES
// the BG2 kernels' own copy of the stamps (each translation unit has one)
extern "C" int nrldpc_debug_phases_bg2(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, nr::nr_phase_stamps, sizeof(unsigned long long) * (size_t)n);
}
#endif
