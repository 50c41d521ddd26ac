// int8 decode, BG1 schedule, byte-pair layouts: its own translation unit.
#include "nrldpc_launch.cuh"

cudaError_t launch_int8_bg1(const nrldpc_plan* plan, Shape& sh, const int8_t* in, int64_t batch, const KOut& o,
                            cudaStream_t st, bool refill) {
  const int dev = plan->device;
  if (refill && (in == nullptr || batch > 2) && (sh.nreg == 6 || sh.nreg == 0)) {
    const cudaError_t e = sh.nreg == 6 ? launch_refill<1, 19, 6>(sh, dev, in, batch, o, st)
                                       : launch_refill<1, 19, 0>(sh, dev, in, batch, o, st);
    if (in != nullptr || e != cudaSuccess) return e;
  }
  if (sh.lanes != 2) return launch_i8<1, 19, 1>(sh, dev, in, batch, o, st);
  if (sh.nreg == 0)
    return sh.abs ? launch_i8<1, 19, 2, 0, true>(sh, dev, in, batch, o, st)
                  : launch_i8<1, 19, 2>(sh, dev, in, batch, o, st);
  if (!sh.abs) return cudaErrorInvalidConfiguration;
  if (sh.nreg == 2) return launch_i8<1, 19, 2, 2, true>(sh, dev, in, batch, o, st);
  if (sh.nreg == 4) return launch_i8<1, 19, 2, 4, true>(sh, dev, in, batch, o, st);
  return launch_i8<1, 19, 2, 6, true>(sh, dev, in, batch, o, st);
}

cudaError_t launch_int8_multi_bg1(int kernel, Shape* const* sh, int n, const int8_t* const* llr, const long long* batch,
                                  const KOut* o, int device, cudaStream_t st) {
  switch (kernel) {
    case 10: return launch_i8_multi<1, 19, 1>(sh, n, llr, batch, o, device, st);
    case 11: return launch_i8_multi<1, 19, 2, 0, true>(sh, n, llr, batch, o, device, st);
    case 12: return launch_i8_multi<1, 19, 2>(sh, n, llr, batch, o, device, st);
    case 13: return launch_i8_multi<1, 19, 2, 2, true>(sh, n, llr, batch, o, device, st);
    case 14: return launch_i8_multi<1, 19, 2, 4, true>(sh, n, llr, batch, o, device, st);
    case 15: return launch_i8_multi<1, 19, 2, 6, true>(sh, n, llr, batch, o, device, st);
    default: return cudaErrorInvalidValue;
  }
}
