/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the polar BP decode hot path.
 *
 * Plain-C restatement of the reference algorithm (/root/reference/proj),
 * each function citing the reference file:line it follows. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker. The product (paper_1505_04979_b200) never links it.
 *
 * Parity pin: tests/test_oracle.py checks this restatement against
 *   (a) the reference core compiled in place (oracle/_ref/libpbp_ref.so,
 *       ref64 = shipped fp64, ref32 = same sources in fp32), and
 *   (b) the golden fixtures in tests/golden/ produced by that build
 *       (tests/golden/make_golden.py), plus the reference's own
 *       known-answer tests re-expressed in tests/test_oracle.py.
 *
 * Decoder math is instantiated twice: *_f32 (reference order in float, the
 * target of the CUDA kernels) and *_f64 (the shipped double reference).
 */
#ifndef PBP_ORACLE_H
#define PBP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_BASELINE = 0, ORC_GMATRIX = 1, ORC_CSFG = 2 };
enum { ORC_STOP_MAX_ITER = 0, ORC_STOP_GMATRIX = 1, ORC_STOP_CSFG = 2 };

/* polar_code.cpp:13-20 */
int orc_polar_transform(uint8_t* v, int n);
/* polar_code.cpp:27-66 ; returns 0 on success, -1 on bad arguments */
int orc_construct(int n, int k, double design_z, uint8_t* frozen_out);
/* polar_code.cpp:82-91 ; u_out/x_out length n */
int orc_encode(int n, const uint8_t* frozen, const uint8_t* info, uint8_t* u_out, uint8_t* x_out);

/* channel.cpp:9-60 (+ libstdc++ std::mt19937_64, GCC 13.3 random.h/.tcc) */
typedef struct {
    uint64_t mt[312];
    int idx;
} orc_mt64;
void orc_trial_rng(orc_mt64* g, uint64_t master_seed, uint64_t trial);
uint64_t orc_mt64_next(orc_mt64* g);
double orc_gaussian(orc_mt64* g);
double orc_noise_variance(double ebn0_db, double rate);
/* sim_harness.cpp:67-73: info bits (k) + fp64 LLRs (n) of one trial */
int orc_trial_frame(uint64_t seed, uint64_t trial, int n, const uint8_t* frozen, double ebn0_db,
                    int noiseless, uint8_t* info_out, double* llr_out);

/* bp_core.cpp:18-32 */
void orc_pe_update_f32(const float* in4, float alpha, float* out4);
void orc_pe_update_f64(const double* in4, double alpha, double* out4);

/* decode_baseline / decode_gmatrix (bp_core.cpp:119-137), decode_csfg
 * (csfg_freeze.cpp:99-152). ev (optional, 5 ints per event: iteration,
 * stage, block, start, size), ev_cap entries. Returns 0 or -1. */
int orc_decode_f32(int kind, int n, const uint8_t* frozen, const float* llr, float alpha,
                   int max_iter, uint8_t* u_hat, int* iterations, long long* pe, int* stop,
                   int* n_events, int* ev, int ev_cap);
int orc_decode_f64(int kind, int n, const uint8_t* frozen, const double* llr, double alpha,
                   int max_iter, uint8_t* u_hat, int* iterations, long long* pe, int* stop,
                   int* n_events, int* ev, int ev_cap);

/* Multi-threaded batch decode (frames x n, row-major) for the CPU baseline:
 * `threads` workers take frame indices from an atomic counter
 * (sim_harness.cpp:144-161). Per-frame outputs optional. */
int orc_decode_batch_f32(int kind, int n, const uint8_t* frozen, const float* llr,
                         long long frames, float alpha, int max_iter, int threads,
                         uint8_t* u_hat, int* iterations, long long* pe, int* stop,
                         int* n_events);
int orc_decode_batch_f64(int kind, int n, const uint8_t* frozen, const double* llr,
                         long long frames, double alpha, int max_iter, int threads,
                         uint8_t* u_hat, int* iterations, long long* pe, int* stop,
                         int* n_events);

#ifdef __cplusplus
}
#endif
#endif
