#pragma once
// Drop-in for the reference's include/polarbp/bp_core.hpp decoder entry points.
// decode_baseline / decode_gmatrix run on the GPU through include/pbp.h in
// double, the reference's own arithmetic (pbp_decode_trace_f64: results equal
// the shipped reference frame by frame); decode_batch is the fp32 fast path
// (the reference's operation order in fp32) with a double overload. pe_update
// and the MessageState utilities are kept as host utilities for the
// reference's known-answer tests. There is no CPU decoder behind the decode calls.
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

// ---- state-level host utilities (the reference's fine-grained public API,
// include/polarbp/bp_core.hpp:38-80, kept for its known-answer tests). The
// decoders below never use them: they run on the GPU.
struct MessageState {
    int n = 0, m = 0;
    std::vector<double> l_msg, r_msg;  // (m+1) x n each, stage-major

    double& l(int stage, int row) { return l_msg[static_cast<size_t>(stage) * n + row]; }
    const double& l(int stage, int row) const { return l_msg[static_cast<size_t>(stage) * n + row]; }
    double& r(int stage, int row) { return r_msg[static_cast<size_t>(stage) * n + row]; }
    const double& r(int stage, int row) const { return r_msg[static_cast<size_t>(stage) * n + row]; }
};

struct FreezeState;  // polarbp/csfg_freeze.hpp

// R(0) = channel LLRs (clamped), L(m) = +LLR_CAP at frozen rows, all else 0.
// Throws std::invalid_argument("init_state: LLR length != n").
MessageState init_state(const PolarCode& code, std::span<const double> channel_llrs);
// The active PEs of one stage (freeze == nullptr: all); returns how many ran.
long long stage_pass(MessageState& state, double alpha, int stage, const FreezeState* freeze);
// Stages 0..m-1 in order; returns the PEs executed.
long long sweep(MessageState& state, double alpha, const FreezeState* freeze = nullptr);
// u_hat[r] = 0 at frozen rows, else (R(m, r) < 0).
Bits hard_output(const MessageState& state, const PolarCode& code);
// x_hat = sign(R(0) + L(0)) equals polar_transform(hard_output).
bool gmatrix_converged(const MessageState& state, const PolarCode& code);

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
