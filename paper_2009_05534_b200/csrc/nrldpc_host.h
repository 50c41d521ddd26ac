// Host-side declarations shared by nrldpc's translation units: error
// helpers, the plan and launch-shape structs, and the per-TU launchers
// (int8 TM / BG1 byte-pair / BG2+generic byte-pair, float engines).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "nrldpc_device.cuh"

namespace nrh {

extern thread_local std::string g_last_error;
extern thread_local int g_launches;

int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

}  // namespace nrh

#define NR_CUDA(call)                                          \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return nrh::cuda_fail(_e, #call);   \
  } while (0)

using namespace nr;
using nrh::g_launches;

// ---------------------------------------------------------------------------
// Host side

// Stream-ordered scratch (lane-refill work counters, float-engine message
// workspaces) comes from a library-private pool per device. Reuse of a freed
// block is limited to orderings the caller's own streams/events establish:
// with the default pool's internal-dependency reuse, a launch on stream B
// could be made to wait for an earlier launch on stream A whose block it
// recycles, which serialises independent batches on separate streams. The
// release threshold keeps freed blocks cached across synchronisations.
cudaError_t scratch_alloc(void** ptr, size_t bytes, int device, cudaStream_t st);

// One launch configuration of the decode kernel.
struct Shape {
  int lanes = 1;    // codewords per half2 lane pair
  int nreg = 0;     // leading rows whose messages live in registers (BG1 pairs)
  int groups = 1;   // codeword groups (of Z threads) per CTA
  int threads = 0;  // 0: no feasible shape
  size_t smem = 0;
  int occ = 0;      // resident CTAs per SM (0: not queried yet)
  int refill_occ = 0;  // the same for this shape's lane-refill kernel
  bool abs = false; // kp.cb holds absolute shared-window addresses
  bool tm = false;  // TM layout (half2 L, shared/tensor-memory messages)
  KParams kp{};
};

struct nrldpc_plan {
  int device = 0;
  bool coscheduled = false;  // launches share SMs with other plans' launches
  int precision = NRLDPC_INT8;
  int early_stop = NRLDPC_STOP_SYNDROME;
  int crc_kind = NRLDPC_CRC24B;
  uint32_t* d_crc_tab = nullptr;  // device: rem(x^(K-1-i+L), g) for i < K (crc mode)
  EncSched enc{};                 // systematic-encoder schedule (enc_ok)
  FloodTables flood{};            // column-major edge lists (flooding schedule)
  bool enc_ok = false;
  double beta = 0.75;
  int max_iter = 20;
  int k_b = 0, z = 0, rows = 0, n_blocks = 0, n_edges = 0, maxw = 0;
  int schedule = 0;  // 0 generic, 1/2: compile-time BG1/BG2 row schedule
  KParams base{};    // graph tables + config, before the shape-dependent scaling
  Shape main;        // the launch shape
  // host-path staging (nrldpc_decode_host[_async])
  std::mutex host_mu;
  // host pipeline: streams[0] copies inputs in (in chunk order), streams[1]
  // copies results out, the rest decode chunks as their input lands (one
  // event per chunk). Two slots of device buffers let one call's copies and
  // decode overlap the next call's (nrldpc_decode_host_async).
  static constexpr int kHostStreams = 18;
  static constexpr int kSlots = 2;
  cudaStream_t streams[kHostStreams] = {};
  std::vector<cudaEvent_t> chunk_ev;
  std::vector<cudaEvent_t> word_ev;  // nrldpc_decode_host_bytes: a chunk's packed words are on the host
  uint32_t* h_words = nullptr;       // pinned landing area of those words
  size_t h_words_cap = 0;
  struct Slot {
    void* d_buf = nullptr;
    size_t d_cap = 0;
    int32_t* h_status = nullptr;  // pinned: the slot's status word lands here
    cudaEvent_t done = nullptr;   // recorded after the slot's result copies
    int64_t ticket = -1;          // call in flight in this slot (-1: none)
    // pageable callers: inputs are staged through h_in (parallel host copy
    // into pinned memory, chunk by chunk, overlapped with the chunks' DMA);
    // results land in h_out and are copied to the caller's buffers when the
    // call retires
    uint8_t* h_in = nullptr;
    size_t h_in_cap = 0;
    uint8_t* h_out = nullptr;
    size_t h_out_cap = 0;
    struct Dst {
      void* p;
      size_t off, n;
    } dst[5] = {};
    int n_dst = 0;
  } slot[kSlots];
  int64_t next_ticket = 0;
  // Calls retired on behalf of a later call (slot reuse, or a synchronous
  // call draining the pipeline) whose input was rejected: their status is
  // kept here until their own nrldpc_host_wait, so an error is reported
  // against the call that caused it and never fails the call reusing the
  // slot. Bounded: the oldest entries go first.
  std::vector<int64_t> failed;
  static constexpr size_t kMaxFailed = 4096;
};


struct nrldpc_plan;

// int8 launchers (llr == nullptr: only set kernel attributes and cache the
// shape's occupancy). refill: the caller chose the lane-refill kernel.
cudaError_t launch_int8_tm(const nrldpc_plan* plan, Shape& sh, const int8_t* in, int64_t batch, const KOut& o,
                           cudaStream_t st, bool refill);
cudaError_t launch_int8_bg1(const nrldpc_plan* plan, Shape& sh, const int8_t* in, int64_t batch, const KOut& o,
                            cudaStream_t st, bool refill);
cudaError_t launch_int8_bg2(const nrldpc_plan* plan, Shape& sh, const int8_t* in, int64_t batch, const KOut& o,
                            cudaStream_t st, bool refill);
// Several shapes of one int8 kernel variant in one launch (mixed batches):
// `kernel` is the variant id (kernel_variant() in nrldpc.cu).
cudaError_t launch_int8_multi_tm(int kernel, Shape* const* sh, int n, const int8_t* const* llr,
                                 const long long* batch, const KOut* o, int device, cudaStream_t st);
cudaError_t launch_int8_multi_bg1(int kernel, Shape* const* sh, int n, const int8_t* const* llr,
                                  const long long* batch, const KOut* o, int device, cudaStream_t st);
cudaError_t launch_int8_multi_bg2(int kernel, Shape* const* sh, int n, const int8_t* const* llr,
                                  const long long* batch, const KOut* o, int device, cudaStream_t st);
// float engines (Precision.F16 / F32)
cudaError_t launch_float_any(int precision, int schedule, Shape& sh, int device, const void* llr, long long batch,
                             const KOut& o, cudaStream_t st);
