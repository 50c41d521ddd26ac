// int8 launch templates (one instantiation per kernel variant), included by
// the int8 translation units.
#pragma once

#include <cstring>

#include "nrldpc_host.h"

// Launch (or, with llr == nullptr, only prepare: set the smem attribute and
// query occupancy) one decode kernel instance for `sh`.
template <int BG, int MAXW, int LANES, int NREG = 0, bool ABS = false, bool TM = false>
static cudaError_t launch_i8(Shape& sh, int device, const int8_t* llr, long long batch, const KOut& o,
                      cudaStream_t st) {
  static bool attr_done[64] = {};
  auto kern = k_decode_i8<BG, MAXW, LANES, NREG, ABS, TM>;
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
  kp.vec_load = ((long long)kp.n_blocks * kp.z) % 16 == 0 && ((uintptr_t)llr & 15) == 0;
  const long long per_cta = (long long)sh.groups * LANES;
  const long long grid = (batch + per_cta - 1) / per_cta;
  kern<<<(unsigned)grid, sh.threads, sh.smem, st>>>(kp, llr, o);
  ++g_launches;
  return cudaGetLastError();
}

// Persistent lane-refill launch (early-stop modes, single-group pair shapes):
// one CTA per resident slot, each refilling its lanes from a per-launch
// codeword counter.
template <int BG, int MAXW, int NREG, bool TM = false>
static cudaError_t launch_refill(Shape& sh, int device, const int8_t* llr, long long batch, const KOut& o,
                                 cudaStream_t st) {
  static bool attr_done[64] = {};
  static int sms[64] = {};
  auto kern = k_decode_i8_refill<BG, MAXW, NREG, TM>;
  const int d = device & 63;
  if (!attr_done[d]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms[d], cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    attr_done[d] = true;
  }
  // occupancy depends on this shape's threads and shared memory (one
  // instantiation serves several Z / rows_used): cached in the Shape, set at
  // plan creation (the llr == nullptr call)
  if (!sh.refill_occ) {
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, sh.threads, sh.smem);
    if (e != cudaSuccess) return e;
    sh.refill_occ = occ > 0 ? occ : 1;
  }
  if (!llr) return cudaSuccess;
  KParams kp = sh.kp;
  kp.batch = batch;
  kp.trace = 0;
  kp.vec_load = ((long long)kp.n_blocks * kp.z) % 16 == 0 && ((uintptr_t)llr & 15) == 0;
  const long long pairs = (batch + 1) / 2;
  const long long grid = std::min<long long>(pairs, (long long)sh.refill_occ * sms[d]);
  int32_t* work = nullptr;
  cudaError_t e = scratch_alloc(reinterpret_cast<void**>(&work), sizeof(int32_t), device, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(work, 0, sizeof(int32_t), st);
  if (e == cudaSuccess) {
    KOut oo = o;
    oo.work = work;
    kern<<<(unsigned)grid, sh.threads, sh.smem, st>>>(kp, llr, oo);
    ++g_launches;
    e = cudaGetLastError();
  }
  const cudaError_t f = cudaFreeAsync(work, st);
  return e != cudaSuccess ? e : f;
}


// Several shapes of one kernel variant in one launch (k_decode_i8_multi).
// All shapes share the CTA size; the launch takes the largest shared-memory
// request among them. Fixed iterations or early stop (pair kernel), no trace.
template <int BG, int MAXW, int LANES, int NREG = 0, bool ABS = false, bool TM = false>
static cudaError_t launch_i8_multi(Shape* const* sh, int n, const int8_t* const* llr, const long long* batch,
                                   const KOut* o, int device, cudaStream_t st) {
  static bool attr_done[64] = {};
  auto kern = k_decode_i8_multi<BG, MAXW, LANES, NREG, ABS, TM>;
  if (!attr_done[device & 63]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    attr_done[device & 63] = true;
  }
  if (n < 1 || n > kMultiShapes) return cudaErrorInvalidValue;
  static thread_local KMulti P;  // 30 KB: kept off the stack
  std::memset(&P, 0, sizeof(P));
  size_t smem = 0;
  long long ctas = 0;
  for (int i = 0; i < n; ++i) {
    if (sh[i]->threads != sh[0]->threads) return cudaErrorInvalidValue;
    KParams& kp = P.s[i];
    kp = sh[i]->kp;
    kp.batch = batch[i];
    kp.trace = 0;
    kp.vec_load = ((long long)kp.n_blocks * kp.z) % 16 == 0 && ((uintptr_t)llr[i] & 15) == 0;
    const long long per_cta = (long long)sh[i]->groups * LANES;
    ctas += (batch[i] + per_cta - 1) / per_cta;
    P.cta_end[i] = (int)ctas;
    P.llr[i] = llr[i];
    P.o[i] = o[i];
    smem = std::max(smem, sh[i]->smem);
  }
  P.n = n;
  if (ctas == 0) return cudaSuccess;
  kern<<<(unsigned)ctas, sh[0]->threads, smem, st>>>(P);
  ++g_launches;
  return cudaGetLastError();
}
