// C++ drop-in check: the reference's unit tests (proj/tests/*.cpp, cited per
// case) re-expressed against include/polarbp/*.hpp linked to libpbp.so.
// Usage: test_dropin [--cpu-only]   (exit code = number of failed checks)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "polarbp/bp_core.hpp"
#include "polarbp/channel.hpp"
#include "polarbp/csfg_freeze.hpp"
#include "polarbp/polar_code.hpp"
#include "polarbp/sim_harness.hpp"

using namespace polarbp;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (cond) {                                                              \
            ++g_pass;                                                            \
        } else {                                                                 \
            ++g_fail;                                                            \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);          \
        }                                                                        \
    } while (0)
template <class F>
static bool throws(F f) {
    try {
        f();
    } catch (const std::exception&) {
        return true;
    }
    return false;
}

static void host_cases() {
    // test_polar_code.cpp:27-38, 130-135, 148-183
    CHECK(PolarCode::construct(2, 1, 0.5).frozen == (Bits{1, 0}));
    CHECK(PolarCode::construct(8, 4, 0.5).frozen_positions() == (std::vector<int>{0, 1, 2, 4}));
    CHECK(throws([] { PolarCode::construct(6, 3, 0.5); }));
    CHECK(throws([] { PolarCode::construct(8, 4, 1.0); }));
    CHECK(polar_transform(Bits{1, 1, 1, 1}) == (Bits{0, 0, 0, 1}));
    CHECK(throws([] { polar_transform(Bits{1, 0, 1}); }));
    const PolarCode c84 = PolarCode::construct(8, 4, 0.5);
    const Codeword cw = encode(c84, Bits{1, 0, 1, 1});
    CHECK(cw.u == (Bits{0, 0, 0, 1, 0, 0, 1, 1}));
    CHECK(extract_info_bits(c84, cw.u) == (Bits{1, 0, 1, 1}));
    CHECK(format_frozen_set(c84) == "n=8\nk=4\nfrozen=1,2,3,5\n");
    CHECK(parse_frozen_set("# c\nn=8\n# k\nk=4\nfrozen=1,2,3,5").k == 4);
    CHECK(throws([] { parse_frozen_set("n=8\nk=4\nfrozen=1,2,3,9"); }));
    CHECK(throws([] { parse_frozen_set("n=8\nk=4\nfrozen=3,2,1,5"); }));
    CHECK(throws([] { parse_frozen_set("n=8\nfrozen=1,2,3,5\nk=4"); }));
    // test_channel.cpp:9-15, 38-49; SURVEY.md 7.1 (first draw)
    CHECK(std::fabs(noise_variance(3.0, 0.5) - 1.0 / std::pow(10.0, 0.3)) < 1e-15);
    CHECK(TrialRng(1, 0).raw() == 0x884fa46695b1825bULL);
    {
        TrialRng a(42, 7), b(42, 7);
        bool same = true;
        for (int i = 0; i < 64; ++i) same = same && a.raw() == b.raw();
        CHECK(same);
    }
    // test_bp_core.cpp:23-37, 93-100
    const PeOutputs p = pe_update({2.0, -3.0, 1.0, 0.5}, 0.9375);
    CHECK(p.l_top == -1.875 && p.r_bot == 1.4375);
    CHECK(pe_update({LLR_CAP, LLR_CAP, LLR_CAP, LLR_CAP}, 1.0).l_bot == LLR_CAP);
    // test_csfg_freeze.cpp:51-97
    CHECK(candidate_block(8, 4, 1).start == 4 && candidate_block(8, 4, 1).size == 2);
    const std::vector<std::uint8_t> fr(c84.frozen.begin(), c84.frozen.begin() + 4);
    const auto d = freeze_decision(std::vector<double>{-3.0, -1.0, -2.0, -4.0}, fr);
    CHECK(d.has_value() && d->u_hat == (Bits{0, 0, 0, 1}));
    CHECK(!freeze_decision(std::vector<double>{-3.0, 1.0, 2.0, 4.0}, fr).has_value());
    // results CSV round trip + savings (test_sim_harness.cpp:93-182)
    std::vector<PointStats> rows(3);
    for (int i = 0; i < 3; ++i) {
        rows[i].decoder = static_cast<DecoderKind>(i);
        rows[i].snr_db = 3.0;
        rows[i].frames = 100;
        rows[i].avg_iters = 40.0 - 10 * i;
        rows[i].avg_pe_activations = 1000.0 - 100 * i;
    }
    const auto back = parse_results_csv(results_csv(rows));
    CHECK(back.size() == 3 && back[2].avg_iters == 20.0);
    const auto sv = compute_savings(rows);
    CHECK(sv.size() == 1 && std::fabs(sv[0].iters_vs_baseline - 0.5) < 1e-12);
}

static void gpu_cases() {
    // test_bp_core.cpp:185-204
    const PolarCode c84 = PolarCode::construct(8, 4, 0.5);
    const std::vector<double> twos(8, 2.0), fives(8, 5.0);
    DecodeOutcome o = decode_baseline(c84, twos, 0.9375, 40);
    CHECK(o.iterations_used == 40 && o.pe_activations == 480 && o.stop_reason == StopReason::max_iter);
    o = decode_gmatrix(c84, twos, 0.9375, 40);
    CHECK(o.iterations_used == 1 && o.pe_activations == 12 && o.stop_reason == StopReason::gmatrix_converged);
    CHECK(throws([&] { decode_baseline(c84, std::vector<double>(7, 0.0), 0.9375, 40); }));
    // test_csfg_freeze.cpp:222-246
    std::vector<FreezeEvent> ev;
    o = decode_csfg(c84, fives, 0.9375, 40, &ev);
    CHECK(o.iterations_used == 1 && o.pe_activations == 7);
    CHECK(ev.size() == 3 && ev[0].stage == 0 && ev[0].size == 4 && ev[1].start == 4 && ev[2].start == 6);
    // test_bp_core.cpp:206-227: 6 dB, (64,32), seed 99: <= 2 wrong of 50
    const PolarCode c64 = PolarCode::construct(64, 32, 0.5);
    int wrong = 0;
    for (int t = 0; t < 50; ++t) {
        TrialRng rng(99, t);
        Bits info(32);
        for (auto& b : info) b = rng.bit();
        const auto llr = transmit_awgn(modulate_bpsk(encode(c64, info).x), {6.0, 0.5, false}, rng);
        if (decode_baseline(c64, llr, 0.9375, 40).info_bits != info) ++wrong;
    }
    CHECK(wrong <= 2);
    // test_sim_harness.cpp:23-47: noiseless (16,8)
    SimConfig cfg;
    cfg.code = PolarCode::construct(16, 8, 0.5);
    cfg.snr_db = {1.0};
    cfg.max_iter = 10;
    cfg.noiseless = true;
    cfg.max_frames = 50;
    const auto r = run_sweep(cfg);
    CHECK(r.size() == 3 && r[0].frames == 50 && r[0].fer == 0.0 && r[0].low_confidence);
    CHECK(r[0].avg_iters == 10.0 && r[0].norm_computations == 1.0);
    CHECK(r[1].avg_iters == 1.0 && r[2].avg_iters == 1.0);
    CHECK(r[2].avg_pe_activations < r[1].avg_pe_activations);
    // 256-frame stop rule: stops on a batch boundary once every decoder has >= 3 frame errors
    SimConfig s2;
    s2.code = PolarCode::construct(64, 32, 0.5);
    s2.snr_db = {0.0};
    s2.min_frame_errors = 3;
    s2.max_frames = 5000;
    const auto r2 = run_sweep(s2);
    CHECK(r2[0].frames == 256 && r2[0].frame_errors >= 3);
}

int main(int argc, char** argv) {
    const bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu-only") == 0;
    host_cases();
    if (!cpu_only) gpu_cases();
    std::printf("%d passed, %d failed\n", g_pass, g_fail);
    return g_fail;
}
