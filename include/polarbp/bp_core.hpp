#pragma once
// Drop-in for the reference's include/polarbp/bp_core.hpp decoder entry points.
// decode_baseline / decode_gmatrix run on the GPU through include/pbp.h in
// double, the reference's own arithmetic (pbp_decode_trace_f64: results equal
// the shipped reference frame by frame); decode_batch is the fp32 fast path
// (the reference's operation order in fp32) with a double overload. pe_update
// is kept as a host utility for the reference's known-answer tests. There is
// no CPU decoder behind these calls.
#include <cstdint>
#include <span>
#include <vector>

#include "polarbp/polar_code.hpp"

namespace polarbp {

inline constexpr double LLR_CAP = 1e30;

struct PeInputs {
    double l_top, l_bot, r_top, r_bot;
};
struct PeOutputs {
    double l_top, l_bot, r_top, r_bot;
};
// Eq. (1) scaled min-sum update, clamped to +-LLR_CAP, sgn(0) = +1 (host utility).
PeOutputs pe_update(const PeInputs& in, double alpha);

enum class StopReason { max_iter, gmatrix_converged, csfg_complete };
const char* to_string(StopReason reason);

struct DecodeOutcome {
    Bits u_hat;
    Bits info_bits;
    int iterations_used = 0;
    long long pe_activations = 0;
    StopReason stop_reason = StopReason::max_iter;
};

DecodeOutcome decode_baseline(const PolarCode& code, std::span<const double> llrs, double alpha,
                              int max_iter);
DecodeOutcome decode_gmatrix(const PolarCode& code, std::span<const double> llrs, double alpha,
                             int max_iter);

// Batched GPU decode (B200 addition): llrs is frames x n, row-major. fp32:
// the warp-resident fast path; double: the reference's double arithmetic.
enum class BatchDecoder { baseline = 0, gmatrix = 1, csfg = 2 };
std::vector<DecodeOutcome> decode_batch(const PolarCode& code, BatchDecoder decoder,
                                        std::span<const float> llrs, double alpha, int max_iter);
std::vector<DecodeOutcome> decode_batch(const PolarCode& code, BatchDecoder decoder,
                                        std::span<const double> llrs, double alpha, int max_iter);

}  // namespace polarbp
