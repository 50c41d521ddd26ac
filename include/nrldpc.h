/*
 * nrldpc — B200 (sm_100a) layered min-sum decoder for 5G-NR-style QC-LDPC
 * codes (BG1/BG2, all 51 lifting sizes). C ABI: plain pointers and sizes,
 * no C++ or torch types. Every entry point returns 0 on success and a
 * negative status otherwise; the message is in nrldpc_last_error()
 * (thread-local). Nothing throws across the ABI.
 *
 * The reference exposes no FFI: its boundary is the Python function
 *   ldpclab.decoder.decode(llrs, bg, cfg, trace=None) -> DecodeResult
 *   (/root/reference/pkg/src/ldpclab/decoder.py:543-566)
 * and the quantizer that feeds it
 *   ldpclab.channel.quantize(llrs, cfg, params)
 *   (/root/reference/pkg/src/ldpclab/channel.py:64-83).
 * The entry points below are what that boundary binds to (see
 * INTEGRATION.md for the ctypes stub the Python mirror uses).
 */
#ifndef NRLDPC_H
#define NRLDPC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define NRLDPC_OK 0
#define NRLDPC_EINVAL (-1)   /* validation: maps to Python ValueError */
#define NRLDPC_ECUDA (-2)    /* CUDA runtime failure: RuntimeError */
#define NRLDPC_ENOMEM (-3)

/* precision (decoder.py:37-40) */
#define NRLDPC_INT8 0
#define NRLDPC_F16 1
#define NRLDPC_F32 2

/* early stop (decoder.py:43-46) */
#define NRLDPC_STOP_SYNDROME 0
#define NRLDPC_STOP_CRC 1
#define NRLDPC_STOP_NONE 2

/* CRC kinds (codec.py:16-20) */
#define NRLDPC_CRC24A 0
#define NRLDPC_CRC24B 1
#define NRLDPC_CRC16 2

/* quantize input dtypes */
#define NRLDPC_IN_F64 0
#define NRLDPC_IN_F32 1

typedef struct nrldpc_plan nrldpc_plan;

/*
 * Immutable decode plan for one (graph, Z, rows_used, config).
 * Replaces the per-call setup of init_workspace / _build_row_gather
 * (decoder.py:243-292) and the DecodeConfig knobs (decoder.py:49-85).
 *   row_start: rows_used+1 edge offsets; cols/shifts: per-edge base column and
 *   circulant shift (already mod z), rows in ascending order, columns ascending
 *   within a row (basegraph.py:79-82).
 *   beta in (0,1]; max_iter >= 1; the int8 beta rule is floor(beta*m) in
 *   float64 (decoder.py:208-212), tabulated here on the host.
 */
int nrldpc_plan_create(int device, int k_b, int z, int rows_used,
                       const int32_t* row_start, const int16_t* cols,
                       const int16_t* shifts, int precision, double beta,
                       int max_iter, int early_stop, int crc_kind,
                       nrldpc_plan** out);

int nrldpc_plan_destroy(nrldpc_plan* plan);

/*
 * Scheduling hint (no reference counterpart; results are unchanged): the
 * plan's launches will run concurrently with other plans' launches on the
 * same SMs, as in a mixed-shape batch. Selects the
 * int8 kernel variant measured fastest under co-scheduling. Call before the
 * plan's first decode; not safe concurrently with decodes on the same plan.
 */
int nrldpc_plan_set_coscheduled(nrldpc_plan* plan, int on);

/* K = k_b*z info bits, n_c = z*(k_b+rows_used), words = ceil(K/32). */
int nrldpc_plan_info(const nrldpc_plan* plan, int64_t* k, int64_t* n_c,
                     int64_t* n_tx, int64_t* words_per_cw, int* lanes,
                     int* groups_per_cta, int* threads_per_cta,
                     int64_t* smem_bytes);

/*
 * Depuncture + quantize (channel.py:64-83): llr_in is (batch, n_tx) float64
 * (bit-exact with the reference) or float32 (throughput mode); out is
 * (batch, n_c) with the 2Z punctured positions zeroed.
 *   out_mode NRLDPC_INT8: clip(rint(L*scale), -127, 127) -> int8
 *   out_mode NRLDPC_F16 : clip(clip(L, -clip, clip), +-65504) -> half (RNE)
 *   out_mode NRLDPC_F32 : clip(L, -clip, clip) -> float
 * Device pointers; asynchronous on `stream` (a cudaStream_t or NULL).
 */
int nrldpc_quantize(const nrldpc_plan* plan, const void* llr_in, int in_dtype,
                    int64_t batch, double scale, double clip, void* out,
                    int out_mode, void* stream);

/*
 * Soft demapper fused into the quantizer (channel.py:57-61 then 64-83):
 * symbols are received BPSK samples y (batch, n_tx); L = (2.0*y)/(sigma*sigma)
 * in float64, then exactly nrldpc_quantize's mapping.
 */
int nrldpc_demap_quantize(const nrldpc_plan* plan, const void* symbols, int in_dtype,
                          int64_t batch, double sigma, double scale, double clip, void* out,
                          int out_mode, void* stream);

/*
 * Layered min-sum decode (decoder.py:486-566). All pointers are device
 * pointers; asynchronous on `stream`. The plan caches per-device launch
 * data (occupancy) on first use; decode calls on one plan from several host
 * threads are safe once it has been used once.
 *   llr      : (batch, n_c) int8 | half | float per the plan's precision
 *   bits     : (batch, words) uint32, hard decisions of the first K
 *              positions, LSB-first (bit i of word w is position 32w+i)
 *   iters    : (batch,) int32   iterations run until exit
 *   synd     : (batch,) int32   unsatisfied checks at exit (0 if stopped early)
 *   success  : (batch,) uint8
 *   crc_ok   : (batch,) uint8 or NULL (crc mode only)
 *   trace_w/trace_m : NULL, or (batch, max_iter) int32 / float — syndrome
 *              weight and min|L_v| after every iteration; a non-NULL trace
 *              runs every codeword for max_iter iterations (results are
 *              unchanged; the host truncates like decoder.py:497-523).
 *   status   : (1,) int32 device word, set nonzero if an int8 input had
 *              magnitude > 127 (decoder.py:287-288); may be NULL.
 */
int nrldpc_decode(nrldpc_plan* plan, const void* llr, int64_t batch,
                  uint32_t* bits, int32_t* iters, int32_t* synd,
                  uint8_t* success, uint8_t* crc_ok, int32_t* trace_w,
                  float* trace_m, int32_t* status, void* stream);

/*
 * Mixed-size batches (BASELINE config 4; transport-block segmentation): one
 * launch decodes up to NRLDPC_MULTI_MAX groups, each with its own plan
 * (graph, Z, rows_used), when the plans share a kernel variant and CTA size
 * (nrldpc_plan_kernel). Same semantics per group as nrldpc_decode without a
 * trace; device pointers; one shared status word (may be NULL); crc_ok may
 * be NULL unless the plans are in crc mode. Many small per-shape launches
 * are limited by how many kernels run concurrently, not by their work; this
 * packs up to five shapes into one grid.
 */
#define NRLDPC_MULTI_MAX 5
int nrldpc_plan_kernel(const nrldpc_plan* plan, int* kernel, int* threads, int64_t* smem_bytes);
int nrldpc_decode_multi(nrldpc_plan* const* plans, int n, const void* const* llr, const int64_t* batch,
                        uint32_t* const* bits, int32_t* const* iters, int32_t* const* synd,
                        uint8_t* const* success, uint8_t* const* crc_ok, int32_t* status, void* stream);

/*
 * Flooding-schedule decode (decoder.py:337-365, 569-581): every row reads the
 * previous iteration's posteriors, then L = sat(L_b + sum of messages).
 * Same buffers, status word and early-stop semantics as nrldpc_decode
 * (device pointers).
 */
int nrldpc_decode_flooding(nrldpc_plan* plan, const void* llr, int64_t batch, uint32_t* bits,
                           int32_t* iters, int32_t* synd, uint8_t* success, uint8_t* crc_ok,
                           int32_t* trace_w, float* trace_m, int32_t* status, void* stream);

/*
 * Host-buffer entry point (the end-to-end path): llr_host (batch, n_c) and
 * outputs are HOST pointers. It pipelines H2D copy / decode / D2H copy over
 * `chunks` sub-batches on the plan's own streams, then synchronizes. Pinned
 * buffers are used in place; pageable ones are staged through the plan's
 * pinned buffers (inputs copied in by the library's host threads, chunk by
 * chunk, overlapped with the DMA; results copied out when the call
 * retires). Returns NRLDPC_EINVAL if an int8 input exceeded |127|.
 */
int nrldpc_decode_host(nrldpc_plan* plan, const void* llr_host, int64_t batch,
                       uint32_t* bits, int32_t* iters, int32_t* synd,
                       uint8_t* success, uint8_t* crc_ok, int chunks);

/*
 * nrldpc_decode_host with the hard decisions returned the way the reference's
 * DecodeResult holds them: bits is a HOST (batch, K) byte array of 0/1
 * (decoder.py:332-334, K = k_b * Z) instead of packed words. Each chunk's
 * packed words are copied back as soon as its decode ends and unpacked by
 * the library's host threads while later chunks still decode, so the
 * unpacking overlaps the pipeline instead of following it. Replaces the
 * decode + unpack pair behind ldpclab.decoder.decode (decoder.py:543-566).
 */
int nrldpc_decode_host_bytes(nrldpc_plan* plan, const void* llr_host, int64_t batch,
                             uint8_t* bits, int32_t* iters, int32_t* synd,
                             uint8_t* success, uint8_t* crc_ok, int chunks);

/*
 * The same call split in two for pipelined serving: _async enqueues the
 * copies and the decode and returns a ticket at once; nrldpc_host_wait
 * blocks until that call's results are in the host buffers (and reports its
 * status). The plan keeps two calls in flight, so a caller that waits for
 * call i after issuing call i+1 overlaps i+1's input copies with i's decode.
 * Issuing a third call first retires the oldest one. Host buffers must stay
 * valid until the wait returns; use pinned memory for overlap.
 */
int nrldpc_decode_host_async(nrldpc_plan* plan, const void* llr_host, int64_t batch,
                             uint32_t* bits, int32_t* iters, int32_t* synd,
                             uint8_t* success, uint8_t* crc_ok, int chunks,
                             int64_t* ticket);
int nrldpc_host_wait(nrldpc_plan* plan, int64_t ticket);

/*
 * Synthetic traffic on the GPU. nrldpc_encode: systematic
 * encoding (codec.py:66-139), msgs (batch, K) bytes 0/1 -> codewords
 * (batch, n_c) bytes 0/1, bit-exact. nrldpc_channel_awgn: BPSK + AWGN
 * (Philox4x32-10, Box-Muller) + L = 2y/sigma^2 + int8 quantize with the 2Z
 * punctured positions zeroed (channel.py:47-83); statistically equivalent to
 * the reference's numpy draws, not draw-for-draw. Device pointers, async.
 */
int nrldpc_encode(const nrldpc_plan* plan, const uint8_t* msgs, int64_t batch, uint8_t* out,
                  void* stream);
int nrldpc_channel_awgn(const nrldpc_plan* plan, const uint8_t* bits, int64_t batch, double sigma,
                        double scale, uint64_t seed, int8_t* out, void* stream);

/*
 * Roofline denominator: measured half2 instruction throughput of this GPU
 * (lane-ops/s, a lane-op = one 32-bit lane of one SASS instruction = two
 * codeword-values for the half2 kernels). alu: HMNMX2 only (ALU pipe);
 * mixed: HMNMX2+HFMA2 1:1 (dual-pipe issue ceiling). Synchronous.
 */
int nrldpc_alu_peak(int device, double* alu_lane_ops_per_s, double* mixed_lane_ops_per_s);

/*
 * The int8 beta rule floor(beta*m) (decoder.py:208-212) as exact half
 * arithmetic: mode=1 when RN_half(beta_h*(m - delta) + c) - c equals it for
 * every m in [0,127] (the kernel then skips its lookup table). Host only.
 */
int nrldpc_beta_rule(double beta, int* mode, float* beta_h, float* delta, float* c);

/*
 * Host helper for the reference's result layout (decoder.py:332-334):
 * packed hard decisions (batch, words_per_cw) uint32, LSB-first, -> (batch,
 * k) bytes 0/1. Multi-threaded on the library's host pool. Host pointers.
 */
int nrldpc_unpack_bits(const uint32_t* words, int64_t batch, int64_t words_per_cw, int64_t k,
                       uint8_t* out);

/* Number of kernel launches the last nrldpc_decode/_quantize issued. */
int nrldpc_launch_count(void);

const char* nrldpc_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* NRLDPC_H */
