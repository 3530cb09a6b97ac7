// The reference's state-level public API as host utilities: MessageState,
// init_state, stage_pass, sweep, hard_output, gmatrix_converged
// (include/polarbp/bp_core.hpp:38-80, src/bp_core.cpp:43-102) and FreezeState,
// candidate_block, check_csfg, mld_oracle, apply_freeze, is_pe_active
// (include/polarbp/csfg_freeze.hpp:39-92, src/csfg_freeze.cpp:8-97).
//
// They exist so that code written against the reference's headers - its
// known-answer tests step a single PE, a stage, a sweep or a commit - keeps
// compiling and giving the same answers. None of the decoders calls them:
// decode_baseline / decode_gmatrix / decode_csfg / decode_batch and the
// harness run on the GPU through include/pbp.h (polarbp_host.cpp).
#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "polarbp/bp_core.hpp"
#include "polarbp/csfg_freeze.hpp"

namespace polarbp {

namespace {
double clamp_cap(double v) { return v < -LLR_CAP ? -LLR_CAP : (LLR_CAP < v ? LLR_CAP : v); }
}  // namespace

MessageState init_state(const PolarCode& code, std::span<const double> channel_llrs) {
    if (static_cast<int>(channel_llrs.size()) != code.n) throw std::invalid_argument("init_state: LLR length != n");
    MessageState st;
    st.n = code.n;
    st.m = code.m;
    const size_t cells = static_cast<size_t>(code.m + 1) * code.n;
    st.l_msg.assign(cells, 0.0);
    st.r_msg.assign(cells, 0.0);
    for (int row = 0; row < code.n; ++row) {
        st.r(0, row) = clamp_cap(channel_llrs[row]);
        st.l(code.m, row) = code.frozen[row] ? LLR_CAP : 0.0;
    }
    return st;
}

long long stage_pass(MessageState& state, double alpha, int stage, const FreezeState* freeze) {
    const int d = state.n >> (stage + 1);
    long long ran = 0;
    for (int top = 0; top < state.n; ++top) {
        if (top & d) continue;  // rows (top, top + d) with bit d clear
        if (freeze && !is_pe_active(*freeze, stage, top)) continue;
        const PeOutputs o = pe_update(
            {state.l(stage + 1, top), state.l(stage + 1, top + d), state.r(stage, top), state.r(stage, top + d)},
            alpha);
        state.l(stage, top) = o.l_top;
        state.l(stage, top + d) = o.l_bot;
        state.r(stage + 1, top) = o.r_top;
        state.r(stage + 1, top + d) = o.r_bot;
        ++ran;
    }
    return ran;
}

long long sweep(MessageState& state, double alpha, const FreezeState* freeze) {
    long long ran = 0;
    for (int s = 0; s < state.m; ++s) ran += stage_pass(state, alpha, s, freeze);
    return ran;
}

Bits hard_output(const MessageState& state, const PolarCode& code) {
    Bits u(code.n, 0);
    for (int row = 0; row < code.n; ++row) u[row] = (!code.frozen[row] && state.r(code.m, row) < 0.0) ? 1 : 0;
    return u;
}

bool gmatrix_converged(const MessageState& state, const PolarCode& code) {
    const Bits x = polar_transform(hard_output(state, code));
    for (int row = 0; row < code.n; ++row)
        if ((state.r(0, row) + state.l(0, row) < 0.0) != (x[row] != 0)) return false;
    return true;
}

BlockRef candidate_block(const FreezeState& freeze, int stage) { return candidate_block(freeze.n, freeze.frontier, stage); }

std::optional<CsfgDecision> check_csfg(const MessageState& state, const PolarCode& code, const BlockRef& block) {
    std::vector<double> rb(block.size);
    for (int i = 0; i < block.size; ++i) rb[i] = state.r(block.stage + 1, block.start + i);
    return freeze_decision(rb, std::span<const std::uint8_t>(code.frozen).subspan(block.start, block.size));
}

Bits mld_oracle(std::span<const double> r_block, std::span<const std::uint8_t> frozen_block,
                long long max_candidates) {
    if (r_block.size() != frozen_block.size()) throw std::invalid_argument("mld_oracle: span length mismatch");
    if (!is_power_of_two(static_cast<int>(r_block.size())))
        throw std::invalid_argument("mld_oracle: length must be a power of two");
    std::vector<int> free_rows;
    for (size_t i = 0; i < frozen_block.size(); ++i)
        if (!frozen_block[i]) free_rows.push_back(static_cast<int>(i));
    if (free_rows.size() >= 62 || (1ll << free_rows.size()) > max_candidates)
        throw std::invalid_argument("mld_oracle: candidate budget exceeded");
    const long long count = 1ll << free_rows.size();
    Bits best;
    double best_score = 0.0;
    Bits u(r_block.size(), 0);
    for (long long c = 0; c < count; ++c) {
        std::fill(u.begin(), u.end(), 0);
        // counter bits MSB-first onto the free rows in index order: candidates in
        // lexicographic u order, strict improvements keep the smallest maximizer
        const size_t nf = free_rows.size();
        for (size_t b = 0; b < nf; ++b) u[free_rows[b]] = (c >> (nf - 1 - b)) & 1;
        const Bits x = polar_transform(u);
        double score = 0.0;
        for (size_t i = 0; i < x.size(); ++i) score += x[i] ? -r_block[i] : r_block[i];
        if (best.empty() || score > best_score || (score == best_score && u < best)) {
            best = u;
            best_score = score;
        }
    }
    return best;
}

Bits mld_oracle(std::span<const double> r_block, const PolarCode& code, const BlockRef& block,
                long long max_candidates) {
    return mld_oracle(r_block, std::span<const std::uint8_t>(code.frozen).subspan(block.start, block.size),
                      max_candidates);
}

void apply_freeze(MessageState& state, FreezeState& freeze, const BlockRef& block, const CsfgDecision& decision,
                  int iteration) {
    for (int i = 0; i < block.size; ++i) {
        const int row = block.start + i;
        state.l(block.stage + 1, row) = decision.x_hat[i] ? -LLR_CAP : LLR_CAP;
        freeze.freeze_stage[row] = std::min(freeze.freeze_stage[row], block.stage);
        freeze.decided_u[row] = decision.u_hat[i];
    }
    freeze.frontier = block.start + block.size;
    freeze.events.push_back({iteration, block.stage, block.index, block.start, block.size, decision.x_hat});
}

bool is_pe_active(const FreezeState& freeze, int stage, int top_row) { return stage <= freeze.freeze_stage[top_row]; }

}  // namespace polarbp
