// Float-engine launchers (Precision.F16 / F32): their own translation unit so
// the kernel instantiations compile in parallel with the int8 ones.
#include "nrldpc_host.h"

template <int PREC, int BG, bool FTM = false>
static cudaError_t launch_float_bg(Shape& sh, int device, const void* llr, long long batch, const KOut& o,
                                cudaStream_t st) {
  static bool attr_done[64] = {};
  auto kern = k_decode_flt<PREC, BG, FTM>;
  if (!attr_done[device & 63]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    attr_done[device & 63] = true;
  }
  if (!sh.occ) {
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, sh.threads, sh.smem);
    if (e != cudaSuccess) return e;
    sh.occ = occ > 0 ? occ : 1;
  }
  if (!llr) return cudaSuccess;
  KParams kp = sh.kp;
  kp.batch = batch;
  kp.trace = o.trace_w != nullptr;
  const long long per_cta = (long long)sh.groups * sh.lanes;
  const long long grid = (batch + per_cta - 1) / per_cta;
  // messages: stream-ordered workspace, [group][edge][z] x 4 bytes (FTM:
  // only the rows kept in global memory)
  uint32_t* ws = nullptr;
  // compile-time schedules: e_reg padded slots per group ([quad][z][4]);
  // generic: n_edges ([edge][z])
  const size_t ws_bytes = std::max<size_t>(16, (size_t)grid * sh.groups * (BG != 0 ? kp.e_reg : kp.n_edges) * kp.z * 4);
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&ws), ws_bytes, device, st);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)grid, sh.threads, sh.smem, st>>>(kp, llr, ws, o);
  ++g_launches;
  e = cudaGetLastError();
  const cudaError_t f = cudaFreeAsync(ws, st);
  return e != cudaSuccess ? e : f;
}

// compile-time row bodies for the BG1/BG2 schedules, generic loop otherwise
template <int PREC>
static cudaError_t launch_float(int schedule, Shape& sh, int device, const void* llr, long long batch,
                                const KOut& o, cudaStream_t st) {
  if (schedule == 1) return sh.tm ? launch_float_bg<PREC, 1, true>(sh, device, llr, batch, o, st)
                                  : launch_float_bg<PREC, 1>(sh, device, llr, batch, o, st);
  if (schedule == 2) return sh.tm ? launch_float_bg<PREC, 2, true>(sh, device, llr, batch, o, st)
                                  : launch_float_bg<PREC, 2>(sh, device, llr, batch, o, st);
  return launch_float_bg<PREC, 0>(sh, device, llr, batch, o, st);
}

cudaError_t launch_float_any(int precision, int schedule, Shape& sh, int device, const void* llr, long long batch,
                             const KOut& o, cudaStream_t st) {
  return precision == NRLDPC_F32 ? launch_float<NRLDPC_F32>(schedule, sh, device, llr, batch, o, st)
                                 : launch_float<NRLDPC_F16>(schedule, sh, device, llr, batch, o, st);
}
