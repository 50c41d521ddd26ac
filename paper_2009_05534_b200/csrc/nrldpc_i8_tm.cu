// int8 decode, TM layout (tensor-memory message rows): its own translation
// unit so the kernel instantiations compile in parallel.
#include "nrldpc_launch.cuh"

cudaError_t launch_int8_tm(const nrldpc_plan* plan, Shape& sh, const int8_t* in, int64_t batch, const KOut& o,
                           cudaStream_t st, bool refill) {
  const int dev = plan->device;
  if (refill && (in == nullptr || batch > 2)) {
    cudaError_t e;
    if (sh.nreg == 6) e = launch_refill<1, 19, 6, true>(sh, dev, in, batch, o, st);
    else if (plan->schedule == 1) e = launch_refill<1, 19, 0, true>(sh, dev, in, batch, o, st);
    else e = launch_refill<2, 10, 0, true>(sh, dev, in, batch, o, st);
    if (in != nullptr || e != cudaSuccess) return e;
  }
  if (sh.nreg == 6) return launch_i8<1, 19, 2, 6, true, true>(sh, dev, in, batch, o, st);
  if (plan->schedule == 1) return launch_i8<1, 19, 2, 0, true, true>(sh, dev, in, batch, o, st);
  return launch_i8<2, 10, 2, 0, true, true>(sh, dev, in, batch, o, st);
}

cudaError_t launch_int8_multi_tm(int kernel, Shape* const* sh, int n, const int8_t* const* llr, const long long* batch,
                                 const KOut* o, int device, cudaStream_t st) {
  switch (kernel) {
    case 1: return launch_i8_multi<1, 19, 2, 6, true, true>(sh, n, llr, batch, o, device, st);
    case 2: return launch_i8_multi<1, 19, 2, 0, true, true>(sh, n, llr, batch, o, device, st);
    case 3: return launch_i8_multi<2, 10, 2, 0, true, true>(sh, n, llr, batch, o, device, st);
    default: return cudaErrorInvalidValue;
  }
}

#ifdef NRLDPC_PHASES
extern "C" int nrldpc_debug_phases(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, nr::nr_phase_stamps, sizeof(unsigned long long) * (size_t)n);
}
#endif
