/*
 * pbp.h -- C ABI of the B200 batched polar-code BP decoder (libpbp.so).
 *
 * This is the drop-in boundary: plain pointers and sizes, no torch or C++
 * types. Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj). The C++ mirror of the
 * reference headers (include/polarbp/*.hpp, namespace polarbp) is
 * implemented on top of these calls; see INTEGRATION.md for the bindings.
 *
 * Conventions
 *   - Rows are 0-based natural order, as in include/polarbp/bp_core.hpp:6-9.
 *   - Positive LLR favours bit 0 (include/polarbp/channel.hpp:2-3).
 *   - Bit vectors are packed little-endian into uint32 words: bit (r % 32)
 *     of word (r / 32) holds row r; ceil(n/32) words per frame.
 *   - Decoders compute in fp32 in the reference's fp32 operation order
 *     (SURVEY.md 8c "ref32"): hard decisions, iteration counts, PE counts,
 *     stop reasons and freeze-event counts equal the reference compiled in
 *     fp32 on the same fp32 LLRs. The *_f64 entry points decode double LLRs
 *     in the reference's own (shipped) double arithmetic instead ("ref64").
 *   - Every call returns PBP_OK (0) or a status; pbp_last_error() gives the
 *     message (thread-local). The reference throws std::invalid_argument /
 *     std::runtime_error with the same texts; the C++ wrapper rethrows them.
 *   - There is no CPU fallback: without a usable CUDA device every decode
 *     call fails with PBP_ENODEV.
 */
#ifndef PBP_H
#define PBP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBP_VERSION 1

typedef enum {
    PBP_OK = 0,
    PBP_EINVAL = 1,  /* std::invalid_argument in the reference */
    PBP_ERUNTIME = 2,/* std::runtime_error in the reference     */
    PBP_ECUDA = 3,   /* CUDA runtime failure                     */
    PBP_ENODEV = 4,  /* no CUDA device                           */
    PBP_ENOMEM = 5
} pbp_status;

/* DecoderKind (include/polarbp/sim_harness.hpp:19) */
typedef enum { PBP_BASELINE = 0, PBP_GMATRIX = 1, PBP_CSFG = 2 } pbp_decoder;
/* StopReason (include/polarbp/bp_core.hpp:48) */
typedef enum { PBP_STOP_MAX_ITER = 0, PBP_STOP_GMATRIX = 1, PBP_STOP_CSFG = 2 } pbp_stop_reason;

/* PolarCode (include/polarbp/polar_code.hpp:27-32): n = 2^m, k info rows,
 * frozen[r] != 0 marks a frozen row. Host memory, caller-owned. */
typedef struct {
    int32_t n;
    int32_t m;
    int32_t k;
    const uint8_t* frozen;
} pbp_code;

/* One device context: device buffers, stream, cached code tables. Not
 * thread-safe; use one context per host thread (reference decoders are
 * pure functions, SPEC: concurrent calls on distinct frames are safe).
 * From one thread, asynchronous device-pointer calls may be queued on
 * different streams of the same context: each call takes one of the
 * context's launch-resource slots in turn, and a slot's next use waits for
 * its previous one. */
typedef struct pbp_ctx pbp_ctx;

/* Per-frame outputs of a batch (DecodeOutcome, include/polarbp/bp_core.hpp:51-57
 * plus the FreezeEvent count of csfg_freeze.hpp:28-35). Any field may be NULL. */
typedef struct {
    uint32_t* u_hat_bits; /* frames x ceil(n/32) words */
    int32_t* iterations;  /* iterations_used           */
    int64_t* pe;          /* pe_activations            */
    uint8_t* stop;        /* pbp_stop_reason           */
    int32_t* n_events;    /* freeze events (csfg)      */
} pbp_frame_out;

/* Accumulator (src/sim_harness.cpp:56-63) plus event and stop histograms.
 * Integer sums: identical for any sharding of trials across GPUs. */
typedef struct {
    int64_t frames;
    int64_t bit_errors;
    int64_t frame_errors;
    int64_t sum_iters;
    int64_t sum_iters_sq;
    int64_t sum_pe;
    int64_t sum_events;
    int64_t stop_hist[3];
} pbp_counters;

const char* pbp_last_error(void);
int pbp_version(void);
/* Number of visible CUDA devices (0 on a CPU-only host). */
int pbp_device_count(void);

int pbp_ctx_create(int device, pbp_ctx** out);
int pbp_ctx_destroy(pbp_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) for callers that order their own work. */
void* pbp_ctx_stream(pbp_ctx* ctx);
int pbp_ctx_synchronize(pbp_ctx* ctx);

/* ---- host-side code helpers (PolarCode::construct, polar_code.cpp:53-66;
 *      polar_transform_inplace, polar_code.cpp:13-20; encode, :82-91) ---- */
int pbp_construct(int32_t n, int32_t k, double design_z, uint8_t* frozen_out);
int pbp_polar_transform(uint8_t* bits, int32_t n);
int pbp_encode(const pbp_code* code, const uint8_t* info, uint8_t* u_out, uint8_t* x_out);
/* noise_variance (src/channel.cpp:9-15) */
int pbp_noise_variance(double ebn0_db, double rate, double* out);

/* ---- decode ------------------------------------------------------------
 * Replaces decode_baseline / decode_gmatrix (include/polarbp/bp_core.hpp:84-87)
 * and decode_csfg (include/polarbp/csfg_freeze.hpp:109-111), batched over
 * `frames` independent frames. llrs: frames x n fp32, row-major.
 *
 * pbp_decode_batch: HOST buffers in and out (copies inside the call).
 * pbp_decode_batch_device: DEVICE pointers, asynchronous on `stream`
 * (NULL = the context stream); outputs valid after the stream syncs. */
int pbp_decode_batch(pbp_ctx* ctx, const pbp_code* code, int decoder, const float* llrs,
                     int64_t frames, float alpha, int32_t max_iter, pbp_frame_out* out);
int pbp_decode_batch_device(pbp_ctx* ctx, const pbp_code* code, int decoder,
                            const float* llrs_dev, int64_t frames, float alpha,
                            int32_t max_iter, pbp_frame_out* out_dev, void* stream);

/* Single-frame decode with the freeze-event trace of decode_csfg's
 * optional `events` out-param (csfg_freeze.hpp:109-111). events receives
 * 5 int32 per event (iteration 1-based, stage, block, start, size), at most
 * events_cap events; *n_events is the full count. Host buffers. */
int pbp_decode_trace(pbp_ctx* ctx, const pbp_code* code, int decoder, const float* llrs,
                     float alpha, int32_t max_iter, uint8_t* u_hat, int32_t* iterations,
                     int64_t* pe, int32_t* stop, int32_t* n_events, int32_t* events,
                     int32_t events_cap);
/* As pbp_decode_trace, plus FreezeEvent::x_hat (csfg_freeze.hpp:34): events_xhat
 * receives events_cap x ceil(n/32) words; event e's block decisions (the hard
 * decision of R(stage+1) at commit time) are bits start..start+size-1 of its
 * row-order word vector, every other bit 0. */
int pbp_decode_trace_x(pbp_ctx* ctx, const pbp_code* code, int decoder, const float* llrs,
                       float alpha, int32_t max_iter, uint8_t* u_hat, int32_t* iterations,
                       int64_t* pe, int32_t* stop, int32_t* n_events, int32_t* events,
                       int32_t events_cap, uint32_t* events_xhat);

/* ---- fp64: the reference as shipped --------------------------------------
 * Same calls with double LLRs and alpha, decoded in double in the reference's
 * operation order (src/bp_core.cpp:13-137 with `double`): results equal the
 * shipped fp64 reference frame by frame, converged or not. Served by the
 * generic kernel (about an order of magnitude below the fp32 fast path). */
int pbp_decode_batch_f64(pbp_ctx* ctx, const pbp_code* code, int decoder, const double* llrs,
                         int64_t frames, double alpha, int32_t max_iter, pbp_frame_out* out);
int pbp_decode_batch_f64_device(pbp_ctx* ctx, const pbp_code* code, int decoder,
                                const double* llrs_dev, int64_t frames, double alpha,
                                int32_t max_iter, pbp_frame_out* out_dev, void* stream);
int pbp_decode_trace_f64(pbp_ctx* ctx, const pbp_code* code, int decoder, const double* llrs,
                         double alpha, int32_t max_iter, uint8_t* u_hat, int32_t* iterations,
                         int64_t* pe, int32_t* stop, int32_t* n_events, int32_t* events,
                         int32_t events_cap);
int pbp_decode_trace_f64_x(pbp_ctx* ctx, const pbp_code* code, int decoder, const double* llrs,
                           double alpha, int32_t max_iter, uint8_t* u_hat, int32_t* iterations,
                           int64_t* pe, int32_t* stop, int32_t* n_events, int32_t* events,
                           int32_t events_cap, uint32_t* events_xhat);
/* run_point's counters with the reference's double LLRs (src/sim_harness.cpp:67-73). */
int pbp_simulate_point_f64(pbp_ctx* ctx, const pbp_code* code, int decoder, uint64_t seed,
                           int64_t first_trial, int64_t frames, double ebn0_db, int noiseless,
                           double alpha, int32_t max_iter, pbp_counters* out);

/* ---- channel -----------------------------------------------------------
 * decode_trial's frame generation (src/sim_harness.cpp:67-73): per trial
 * TrialRng(seed, trial) (src/channel.cpp:31-41), K info bits, encode,
 * BPSK, AWGN at Eb/N0 with rate k/n, LLR = 2y/sigma^2 in fp64, stored as
 * fp32 (and fp64 when llr64_dev != NULL). u_dev (optional) receives the
 * transmitted source word u bit-packed (frames x ceil(n/32)). Device
 * pointers, asynchronous on `stream`. */
int pbp_generate_device(pbp_ctx* ctx, const pbp_code* code, uint64_t seed, int64_t first_trial,
                        int64_t count, double ebn0_db, int noiseless, float* llr_dev,
                        double* llr64_dev, uint32_t* u_dev, void* stream);
/* Host-buffer convenience wrapper of pbp_generate_device. */
int pbp_generate(pbp_ctx* ctx, const pbp_code* code, uint64_t seed, int64_t first_trial,
                 int64_t count, double ebn0_db, int noiseless, float* llr, double* llr64,
                 uint32_t* u_bits);

/* ---- Monte-Carlo point (run_point, src/sim_harness.cpp:129-186, with
 *      min_frame_errors = infinity): trials [first_trial, first_trial+frames)
 *      generated on the device, decoded, counters accumulated on the device.
 *      Shard trial ranges across GPUs and sum the counters (one int64
 *      allreduce) for the multi-GPU run. */
int pbp_simulate_point(pbp_ctx* ctx, const pbp_code* code, int decoder, uint64_t seed,
                       int64_t first_trial, int64_t frames, double ebn0_db, int noiseless,
                       float alpha, int32_t max_iter, pbp_counters* out);
/* Device-side variant: counters (10 int64) accumulate into counters_dev
 * (not cleared); asynchronous on `stream`. */
int pbp_simulate_point_device(pbp_ctx* ctx, const pbp_code* code, int decoder, uint64_t seed,
                              int64_t first_trial, int64_t frames, double ebn0_db,
                              int noiseless, float alpha, int32_t max_iter,
                              int64_t* counters_dev, void* stream);

/* Counter accumulation for already-generated frames (device pointers):
 * decodes llrs_dev and compares against u_dev (from pbp_generate_device). */
int pbp_decode_count_device(pbp_ctx* ctx, const pbp_code* code, int decoder,
                            const float* llrs_dev, const uint32_t* u_dev, int64_t frames,
                            float alpha, int32_t max_iter, int64_t* counters_dev, void* stream);

/* As pbp_decode_count_device with one counter set per `batch` consecutive frames
 * (counters_dev: ceil(frames / batch) x 10 int64, accumulated): e.g. a whole Eb/N0
 * sweep stored point after point, decoded in ONE launch with per-point counters. */
int pbp_decode_count_batches_device(pbp_ctx* ctx, const pbp_code* code, int decoder,
                                    const float* llrs_dev, const uint32_t* u_dev, int64_t frames,
                                    int64_t batch, float alpha, int32_t max_iter,
                                    int64_t* counters_dev, void* stream);

/* run_point's batches (src/sim_harness.cpp:136-178, kBatchSize = 256 at :21): trials
 * [first_trial, first_trial + frames) generated and decoded as pbp_simulate_point does
 * (fp64 != 0: the reference's double LLRs decoded in double), with ONE counter set per
 * `batch` consecutive trials, so the caller can apply the reference's stop rule on batch
 * boundaries. counters_out (host) receives ceil(frames / batch) x 10 int64 in the
 * pbp_counters field order. */
int pbp_simulate_batches(pbp_ctx* ctx, const pbp_code* code, int decoder, uint64_t seed,
                         int64_t first_trial, int64_t frames, int32_t batch, double ebn0_db,
                         int noiseless, double alpha, int32_t max_iter, int fp64,
                         int64_t* counters_out);

/* Fixed-count Monte-Carlo sweep over several GPUs of one process (run_sweep with
 * min_frame_errors = infinity, src/sim_harness.cpp:129-196, whose workers split the
 * trials at :144-161): every point's trials [0, frames_per_point) are split into ndev
 * contiguous ranges, one host thread per device generates and decodes its range, and
 * the per-device counters (npoints x 10 int64) are summed in place with ONE
 * ncclAllReduce(int64, sum) over NVLink/NVSwitch (libnccl.so.2, loaded at first use).
 * Integer sums: the result equals the single-GPU and CPU aggregates. out: npoints sets. */
int pbp_simulate_sweep_multi(const int* devices, int ndev, const pbp_code* code, int decoder,
                             uint64_t seed, int64_t frames_per_point, const double* ebn0_db,
                             int npoints, int noiseless, float alpha, int32_t max_iter,
                             pbp_counters* out);

/* Which kernel serves a code length: 1 = warp-resident fast path
 * (n = 128..1024), 2 = CTA-per-frame register-pass path (n = 2048..16384),
 * 0 = the generic kernel only. For tests and bench introspection. */
int pbp_kernel_path(int32_t n);
/* CTAs per frame of the fast kernel for (n, decoder): 2 = the frame split
 * over a 2-CTA thread-block cluster (n = 16384, every decoder: each CTA holds
 * half of the frame on its SM, the frame's stage 0 exchanged through
 * distributed shared memory; environment PBP_PAIR=0 selects one CTA per
 * frame), 1 = one CTA (or warp) per frame, 0 = no fast kernel for n.
 * Freeze-event traces always decode one frame per CTA. */
int pbp_kernel_cluster(int32_t n, int decoder);
/* Route every decode of this context through the generic kernel (on != 0).
 * Test hook: lets the suite check both kernels against the oracle. */
int pbp_ctx_force_generic(pbp_ctx* ctx, int on);
/* Fast-kernel resources for code length n: shared bytes per warp (warp-resident
 * kernel, n <= 1024) or per CTA (CTA-per-frame kernel, n = 2048..16384), and resident
 * warps per SM (0 when n uses the generic kernel only or there is no device). */
int pbp_kernel_info(int32_t n, int decoder, int32_t* smem_bytes, int32_t* warps_per_sm);
/* Launch statistics of the last decode on this context (kernel launches,
 * frames re-routed to the generic kernel because |LLR| exceeded the
 * clamp-free bound or was not finite). */
int pbp_last_launch_info(pbp_ctx* ctx, int32_t* launches, int64_t* rerouted_frames);

#ifdef __cplusplus
}
#endif
#endif
