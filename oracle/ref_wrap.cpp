// Test-infrastructure ONLY (oracle). Builds the *unmodified* reference core
// (/root/reference/proj/src/{polar_code,channel,bp_core,csfg_freeze}.cpp)
// in place -- nothing is copied -- and exposes it through a flat C ABI so
// the pytest suite and bench.py's CPU-baseline leg can call it via ctypes.
//
// Compiled twice (see oracle/Makefile):
//   REF_PREC=64 : the shipped double-precision reference   -> symbols ref64_*
//   REF_PREC=32 : the same sources with `#define double float` after every
//                 system header (SURVEY.md 0.3 / 8c "ref32") -> symbols ref32_*
// ref32 is the reference's own operation order evaluated in fp32, i.e. the
// bit-exact target of the fp32 CUDA kernels.
//
// The harness loop of decode_trial / run_point
// (/root/reference/proj/src/sim_harness.cpp:65-99,144-161) is restated below
// because sim_harness.cpp itself needs the absent vendor/json.hpp.
//
// Never linked into the product path.

// --- every system header the reference sources pull in, BEFORE the macro ---
#include <algorithm>
#include <atomic>
#include <cassert>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <numbers>
#include <numeric>
#include <optional>
#include <random>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#if REF_PREC == 32
#define double float
#define polarbp polarbp_ref32
#define REFSYM(name) ref32_##name
#elif REF_PREC == 64
#define polarbp polarbp_ref64
#define REFSYM(name) ref64_##name
#else
#error "REF_PREC must be 32 or 64"
#endif

// resolved through -I$(REF_DIR) (see Makefile); the files are read in place
#include "src/polar_code.cpp"
#include "src/channel.cpp"
#include "src/bp_core.cpp"
#include "src/csfg_freeze.cpp"

namespace {

thread_local std::string g_err;

polarbp::PolarCode make_code(int n, const std::uint8_t* frozen) {
    polarbp::Bits mask(frozen, frozen + n);
    return polarbp::PolarCode::from_frozen_mask(n, std::move(mask));
}

// One decode, reference semantics. kind: 0 baseline, 1 gmatrix, 2 csfg.
polarbp::DecodeOutcome run_one(int kind, const polarbp::PolarCode& code,
                               std::span<const double> llr, double alpha, int max_iter,
                               std::vector<polarbp::FreezeEvent>* events) {
    switch (kind) {
        case 0: return polarbp::decode_baseline(code, llr, alpha, max_iter);
        case 1: return polarbp::decode_gmatrix(code, llr, alpha, max_iter);
        case 2: return polarbp::decode_csfg(code, llr, alpha, max_iter, events);
    }
    throw std::invalid_argument("unknown decoder kind");
}

}  // namespace

extern "C" {

const char* REFSYM(last_error)() { return g_err.c_str(); }

void REFSYM(pe_update)(const double* in, double alpha, double* out) {
    const polarbp::PeOutputs o = polarbp::pe_update({in[0], in[1], in[2], in[3]}, alpha);
    out[0] = o.l_top;
    out[1] = o.l_bot;
    out[2] = o.r_top;
    out[3] = o.r_bot;
}

int REFSYM(polar_transform)(std::uint8_t* v, int n) {
    try {
        polarbp::polar_transform_inplace(std::span<std::uint8_t>(v, static_cast<size_t>(n)));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Decode one frame. ev (optional) receives 5 ints per event:
// iteration, stage, block, start, size. Returns 0 or -1 (see last_error).
int REFSYM(decode)(int kind, int n, const std::uint8_t* frozen, const double* llr,
                   double alpha, int max_iter, std::uint8_t* u_hat, int* iterations,
                   long long* pe, int* stop, int* n_events, int* ev, int ev_cap) {
    try {
        const polarbp::PolarCode code = make_code(n, frozen);
        std::vector<polarbp::FreezeEvent> events;
        const polarbp::DecodeOutcome o =
            run_one(kind, code, std::span<const double>(llr, static_cast<size_t>(n)), alpha,
                    max_iter, kind == 2 ? &events : nullptr);
        if (u_hat) std::memcpy(u_hat, o.u_hat.data(), static_cast<size_t>(n));
        *iterations = o.iterations_used;
        *pe = o.pe_activations;
        *stop = static_cast<int>(o.stop_reason);
        *n_events = static_cast<int>(events.size());
        if (ev) {
            for (int i = 0; i < static_cast<int>(events.size()) && i < ev_cap; ++i) {
                ev[5 * i + 0] = events[i].iteration;
                ev[5 * i + 1] = events[i].stage;
                ev[5 * i + 2] = events[i].block;
                ev[5 * i + 3] = events[i].start;
                ev[5 * i + 4] = events[i].size;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Batched decode over `frames` frames (row-major frames x n) on `threads`
// worker threads pulling frame indices from an atomic counter, the pattern
// of sim_harness.cpp:144-161. Per-frame outputs are optional (nullptr).
int REFSYM(decode_batch)(int kind, int n, const std::uint8_t* frozen, const double* llr,
                         long long frames, double alpha, int max_iter, int threads,
                         std::uint8_t* u_hat, int* iterations, long long* pe, int* stop,
                         int* n_events) {
    try {
        const polarbp::PolarCode code = make_code(n, frozen);
        std::atomic<long long> next{0};
        std::atomic<bool> failed{false};
        std::string err;
        auto work = [&]() {
            long long f;
            std::vector<polarbp::FreezeEvent> events;
            while ((f = next.fetch_add(1)) < frames) {
                try {
                    const std::span<const double> in(llr + f * n, static_cast<size_t>(n));
                    events.clear();
                    const polarbp::DecodeOutcome o =
                        run_one(kind, code, in, alpha, max_iter, n_events ? &events : nullptr);
                    if (u_hat) std::memcpy(u_hat + f * n, o.u_hat.data(), static_cast<size_t>(n));
                    if (iterations) iterations[f] = o.iterations_used;
                    if (pe) pe[f] = o.pe_activations;
                    if (stop) stop[f] = static_cast<int>(o.stop_reason);
                    if (n_events) n_events[f] = static_cast<int>(events.size());
                } catch (const std::exception& e) {
                    failed = true;
                }
            }
        };
        const int spawn = std::max(1, threads);
        std::vector<std::thread> pool;
        for (int w = 0; w < spawn; ++w) pool.emplace_back(work);
        for (auto& t : pool) t.join();
        if (failed) throw std::runtime_error("decode_batch: a frame failed");
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

#if REF_PREC == 64
int ref64_construct(int n, int k, double design_z, std::uint8_t* frozen) {
    try {
        const polarbp::PolarCode code = polarbp::PolarCode::construct(n, k, design_z);
        std::memcpy(frozen, code.frozen.data(), static_cast<size_t>(n));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

void ref64_rng_raw(std::uint64_t seed, std::uint64_t trial, int count, std::uint64_t* out) {
    polarbp::TrialRng rng(seed, trial);
    for (int i = 0; i < count; ++i) out[i] = rng.raw();
}

void ref64_rng_gaussian(std::uint64_t seed, std::uint64_t trial, int count, double* out) {
    polarbp::TrialRng rng(seed, trial);
    for (int i = 0; i < count; ++i) out[i] = rng.gaussian();
}

double ref64_noise_variance(double ebn0_db, double rate) {
    return polarbp::noise_variance(ebn0_db, rate);
}

// The channel part of decode_trial (sim_harness.cpp:67-73) for trials
// [first, first+count): info bits (count x k) and fp64 LLRs (count x n).
// Threads split the trial range; each trial owns its stream, so the output
// does not depend on `threads`.
int ref64_trials(std::uint64_t seed, long long first, long long count, int n,
                 const std::uint8_t* frozen, double ebn0_db, int noiseless, int threads,
                 std::uint8_t* info_out, double* llr_out) {
    try {
        const polarbp::PolarCode code = make_code(n, frozen);
        const polarbp::ChannelConfig ch{ebn0_db, static_cast<double>(code.k) / code.n,
                                        noiseless != 0};
        std::atomic<long long> next{0};
        auto work = [&]() {
            long long i;
            while ((i = next.fetch_add(1)) < count) {
                polarbp::TrialRng rng(seed, static_cast<std::uint64_t>(first + i));
                polarbp::Bits info(code.k);
                for (int b = 0; b < code.k; ++b) info[b] = rng.bit();
                const polarbp::Codeword cw = polarbp::encode(code, info);
                const std::vector<double> sym = polarbp::modulate_bpsk(cw.x);
                const std::vector<double> llr = polarbp::transmit_awgn(sym, ch, rng);
                if (info_out) std::memcpy(info_out + i * code.k, info.data(), static_cast<size_t>(code.k));
                std::memcpy(llr_out + i * n, llr.data(), sizeof(double) * static_cast<size_t>(n));
            }
        };
        const int spawn = std::max(1, threads);
        std::vector<std::thread> pool;
        for (int w = 0; w < spawn; ++w) pool.emplace_back(work);
        for (auto& t : pool) t.join();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}
#endif

}  // extern "C"
