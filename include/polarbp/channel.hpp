#pragma once
// Drop-in for the reference's include/polarbp/channel.hpp: BPSK over AWGN with
// one deterministic std::mt19937_64 stream per (seed, trial); positive LLR = bit 0.
// Host implementation (bit-identical stream); the batched generator on the GPU is
// pbp_generate_device (include/pbp.h) / polarbp::generate_frames below.
#include <cstdint>
#include <random>
#include <span>
#include <vector>

#include "polarbp/polar_code.hpp"

namespace polarbp {

struct ChannelConfig {
    double ebn0_db = 0.0;
    double rate = 0.5;
    bool noiseless = false;
};

double noise_variance(double ebn0_db, double rate);

class TrialRng {
public:
    TrialRng(std::uint64_t master_seed, std::uint64_t trial);
    double gaussian();      // Box-Muller, cosine branch, two draws
    std::uint8_t bit();     // top bit of one draw
    std::uint64_t raw() { return engine_(); }

private:
    std::mt19937_64 engine_;
};

std::vector<double> modulate_bpsk(const Bits& x);
std::vector<double> transmit_awgn(std::span<const double> symbols, const ChannelConfig& config,
                                  TrialRng& rng);

// GPU batch of decode_trial frames: fp32 LLRs (count x n) and source words u (count x n).
void generate_frames(const PolarCode& code, std::uint64_t seed, std::int64_t first_trial,
                     std::int64_t count, const ChannelConfig& config, std::vector<float>& llrs,
                     std::vector<Bits>* u_words = nullptr);
// The same frames with the fp64 LLRs (the CUDA log/cos may differ from glibc's
// in the last bits near y = 0; the fp32 LLRs above match the host exactly).
void generate_frames(const PolarCode& code, std::uint64_t seed, std::int64_t first_trial,
                     std::int64_t count, const ChannelConfig& config, std::vector<double>& llrs,
                     std::vector<Bits>* u_words = nullptr);

}  // namespace polarbp
