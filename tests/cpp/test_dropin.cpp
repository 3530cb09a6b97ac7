// C++ drop-in check: the reference's unit tests (proj/tests/*.cpp, cited per
// case) re-expressed against include/polarbp/*.hpp linked to libpbp.so.
// Usage: test_dropin [--cpu-only]   (exit code = number of failed checks)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
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
    // test_bp_core.cpp:39-91: zero counts as positive; flipping the wire signs along a
    // codeword of the PE's check negates exactly the messages on the flipped wires;
    // scaling shrinks the two pure-product outputs
    {
        const PeOutputs z = pe_update({0.0, 2.0, 3.0, 1.0}, 1.0);
        CHECK(z.l_top == 0.0 && z.r_bot == 1.0 && z.r_top == 3.0);
        std::mt19937_64 gen(8101);
        std::uniform_real_distribution<double> uni(-20.0, 20.0);
        const int pat[3][3] = {{1, 1, 0}, {1, 0, 1}, {0, 1, 1}};  // flips of wires a, c, b
        int bad = 0;
        for (int rep = 0; rep < 10000; ++rep) {
            const PeInputs in{uni(gen), uni(gen), uni(gen), uni(gen)};
            if (in.l_top == 0.0 || in.l_bot == 0.0 || in.r_top == 0.0 || in.r_bot == 0.0) continue;
            const PeOutputs base = pe_update(in, 0.9375);
            for (const auto& f : pat) {
                const double fa = f[0] ? -1.0 : 1.0, fc = f[1] ? -1.0 : 1.0, fb = f[2] ? -1.0 : 1.0;
                const PeOutputs o = pe_update({fc * in.l_top, fb * in.l_bot, fa * in.r_top, fb * in.r_bot}, 0.9375);
                bad += !(o.l_top == fa * base.l_top && o.l_bot == fb * base.l_bot && o.r_top == fc * base.r_top &&
                         o.r_bot == fb * base.r_bot);
            }
        }
        CHECK(bad == 0);
        std::mt19937_64 g2(8102);
        bad = 0;
        for (int rep = 0; rep < 2000; ++rep) {
            const PeInputs in{uni(g2), uni(g2), uni(g2), uni(g2)};
            const PeOutputs h = pe_update(in, 0.5), f = pe_update(in, 1.0);
            bad += !(std::fabs(h.l_top) <= std::fabs(f.l_top) + 1e-12 && std::fabs(h.r_top) <= std::fabs(f.r_top) + 1e-12);
        }
        CHECK(bad == 0);
    }
    // test_csfg_freeze.cpp:51-97
    CHECK(candidate_block(8, 4, 1).start == 4 && candidate_block(8, 4, 1).size == 2);
    const std::vector<std::uint8_t> fr(c84.frozen.begin(), c84.frozen.begin() + 4);
    const auto d = freeze_decision(std::vector<double>{-3.0, -1.0, -2.0, -4.0}, fr);
    CHECK(d.has_value() && d->u_hat == (Bits{0, 0, 0, 1}));
    CHECK(!freeze_decision(std::vector<double>{-3.0, 1.0, 2.0, 4.0}, fr).has_value());
    // state-level host utilities (test_bp_core.cpp:102-183)
    {
        const std::vector<double> llrs{1, -2, 3, -4, 5, -6, 7, -8};
        const MessageState st = init_state(c84, llrs);
        bool ok = true;
        for (int r = 0; r < 8; ++r) {
            ok = ok && st.r(0, r) == llrs[r] && st.l(3, r) == (c84.frozen[r] ? LLR_CAP : 0.0);
            for (int s2 = 1; s2 <= 3; ++s2) ok = ok && st.r(s2, r) == 0.0;
            for (int s2 = 0; s2 < 3; ++s2) ok = ok && st.l(s2, r) == 0.0;
        }
        CHECK(ok);
        CHECK(throws([&] { init_state(c84, std::vector<double>(7, 0.0)); }));
        MessageState s1 = init_state(c84, std::vector<double>(8, 1.0));
        CHECK(sweep(s1, 0.9375) == 12);
        std::mt19937_64 gen(8103);
        std::uniform_real_distribution<double> uni(-5.0, 5.0);
        std::vector<double> rnd(8);
        for (double& v : rnd) v = uni(gen);
        MessageState s2 = init_state(c84, rnd);
        FreezeState all(8);
        all.freeze_stage.assign(8, -1);  // below every stage: no PE active
        const MessageState before = s2;
        CHECK(sweep(s2, 0.9375, &all) == 0 && s2.l_msg == before.l_msg && s2.r_msg == before.r_msg);
        const PolarCode c32 = PolarCode::construct(32, 16, 0.5);
        std::vector<double> r32(32);
        for (double& v : r32) v = uni(gen);
        MessageState s3 = init_state(c32, r32);
        const std::vector<double> lb = s3.l_msg;
        for (int t = 0; t < 5; ++t) sweep(s3, 0.9375);
        ok = true;
        for (int r = 0; r < 32; ++r) ok = ok && s3.r(0, r) == r32[r] && s3.l(c32.m, r) == lb[5 * 32 + r];
        CHECK(ok);
        MessageState s4 = init_state(c84, std::vector<double>(8, 2.0));
        sweep(s4, 0.9375);
        ok = true;
        for (int r = 0; r < 8; ++r) ok = ok && s4.r(3, r) > 0.0;
        CHECK(ok && hard_output(s4, c84) == Bits(8, 0));
        MessageState s5 = init_state(c84, std::vector<double>(8, 1.0));
        for (int r = 0; r < 8; ++r) s5.r(3, r) = 1.0;
        s5.r(3, 3) = -0.1;
        CHECK(hard_output(s5, c84) == (Bits{0, 0, 0, 1, 0, 0, 0, 0}));
        s5.r(3, 3) = 0.0;  // a tie decides 0
        CHECK(hard_output(s5, c84) == Bits(8, 0));
        s5.r(3, 0) = -9.0;  // frozen rows stay 0
        CHECK(hard_output(s5, c84) == Bits(8, 0));
        const PolarCode c22 = PolarCode::construct(2, 2, 0.5);
        CHECK(gmatrix_converged(init_state(c22, std::vector<double>{1.0, 1.0}), c22));
        CHECK(!gmatrix_converged(init_state(c22, std::vector<double>{-1.0, 1.0}), c22));
    }
    // FreezeState, apply_freeze, is_pe_active, mld_oracle (test_csfg_freeze.cpp:100-220)
    {
        MessageState st = init_state(c84, std::vector<double>(8, 1.0));
        FreezeState fz(8);
        apply_freeze(st, fz, BlockRef{1, 0, 0, 2}, {{1, 0}, {1, 1}}, 1);
        CHECK(fz.frontier == 2 && st.l(2, 0) == -LLR_CAP && st.l(2, 1) == LLR_CAP && fz.freeze_stage[0] == 1 &&
              fz.decided_u[0] == 1 && fz.decided_u[1] == 1);
        apply_freeze(st, fz, BlockRef{0, 0, 0, 4}, {{0, 0, 0, 0}, {0, 0, 0, 0}}, 2);  // the enclosing block supersedes
        bool ok = fz.frontier == 4;
        for (int r = 0; r < 4; ++r) ok = ok && st.l(1, r) == LLR_CAP && fz.freeze_stage[r] == 0 && fz.decided_u[r] == 0;
        CHECK(ok && fz.events.size() == 2 && fz.events[1].iteration == 2);
        CHECK(candidate_block(fz, 1).start == 4 && candidate_block(fz, 1).size == 2 && candidate_block(fz, 1).index == 2);
        auto count_active = [&](const FreezeState& f) {
            int a = 0;
            for (int s2 = 0; s2 < c84.m; ++s2)
                for (int r = 0; r < 8; ++r)
                    if (!(r & (8 >> (s2 + 1))) && is_pe_active(f, s2, r)) ++a;
            return a;
        };
        FreezeState f0(8);
        CHECK(count_active(f0) == 12);
        FreezeState f1(8);
        for (int r = 0; r < 4; ++r) f1.freeze_stage[r] = 0;
        CHECK(count_active(f1) == 8 && is_pe_active(f1, 0, 0) && !is_pe_active(f1, 1, 0) && !is_pe_active(f1, 2, 2));
        FreezeState f2(8);
        f2.freeze_stage[0] = f2.freeze_stage[1] = 1;
        CHECK(count_active(f2) == 11 && !is_pe_active(f2, 2, 0) && is_pe_active(f2, 1, 0));
        CHECK(mld_oracle(std::vector<double>{3.0, 1.0, 2.0, 4.0}, Bits{1, 1, 1, 0}) == Bits(4, 0));
        CHECK(throws([] { mld_oracle(std::vector<double>(16, 1.0), Bits(16, 0), 8); }));
        // csfg_freeze.cpp:44-53: texts, power-of-two length, MSB-first enumeration (ties keep
        // the lexicographically smallest u: all-zero LLRs tie every candidate)
        auto what = [](auto f) {
            try {
                f();
            } catch (const std::invalid_argument& e) {
                return std::string(e.what());
            }
            return std::string();
        };
        CHECK(what([] { mld_oracle(std::vector<double>(16, 1.0), Bits(16, 0), 8); }) ==
              "mld_oracle: candidate budget exceeded");
        CHECK(what([] { mld_oracle(std::vector<double>(3, 1.0), Bits(3, 1)); }) ==
              "mld_oracle: length must be a power of two");
        CHECK(what([] { mld_oracle(std::vector<double>(4, 1.0), Bits(2, 1)); }) == "mld_oracle: span length mismatch");
        CHECK(mld_oracle(std::vector<double>(4, 0.0), Bits{1, 0, 0, 1}) == Bits(4, 0));
        // freeze_decision accepts exactly when it equals the block ML decision
        std::mt19937_64 gen(9002);
        std::uniform_real_distribution<double> uni(-5.0, 5.0);
        int accepted = 0, agree = 0;
        for (int rep = 0; rep < 1000; ++rep) {
            const int len = 2 << (gen() % 4);
            std::vector<double> r(len);
            for (double& v : r)
                do v = uni(gen);
                while (v == 0.0);
            Bits fr(len);
            for (auto& f : fr) f = gen() & 1;
            const Bits ml = mld_oracle(r, fr);
            const auto dec = freeze_decision(r, fr);
            double abs_sum = 0.0, ml_score = 0.0;
            const Bits xm = polar_transform(ml);
            for (int i = 0; i < len; ++i) {
                abs_sum += std::fabs(r[i]);
                ml_score += xm[i] ? -r[i] : r[i];
            }
            if (dec) {
                ++accepted;
                agree += dec->u_hat == ml;
            } else {
                agree += ml_score < abs_sum;
            }
        }
        CHECK(agree == 1000 && accepted > 50);
    }
    // acceptance.cpp:302-309: the polar transform is an involution
    {
        std::mt19937_64 gen(9006);
        int bad = 0;
        for (int rep = 0; rep < 10000; ++rep) {
            Bits u(1u << (gen() % 11));
            for (auto& b : u) b = static_cast<std::uint8_t>(gen() >> 63);
            bad += polar_transform(polar_transform(u)) != u;
        }
        CHECK(bad == 0);
    }
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

// results_json in nlohmann::json::dump(2) form (sim_harness.cpp:250-289): sorted keys,
// one element per line, shortest round-trip doubles laid out like nlohmann's dtoa
static void json_case() {
    SimConfig cfg;
    cfg.code = PolarCode::construct(4, 2, 0.5);
    cfg.code_source = "construct \"z\"";
    cfg.decoders = {DecoderKind::csfg};
    cfg.snr_db = {1.5, 0.0001, 1e16, 1e15};  // 1e15: 16 integer digits > 15 -> e-notation
    cfg.seed = 18446744073709551615ull;
    PointStats r;
    r.decoder = DecoderKind::csfg;
    r.snr_db = 1.5;
    r.frames = 256;
    r.bit_errors = 3;
    r.frame_errors = 1;
    r.ber = 3.0 / 512.0;
    r.fer = 1.0 / 256.0;
    r.fer_ci95 = 1e-05;
    r.avg_iters = 40.0;
    r.iters_ci95 = 0.0;
    r.avg_pe_activations = 1234567.0;
    r.norm_computations = 0.1;
    r.low_confidence = true;
    const std::vector<PointStats> rows{r};
    const std::string want =
        "{\n  \"config\": {\n    \"alpha\": 0.9375,\n    \"code_source\": \"construct \\\"z\\\"\",\n"
        "    \"decoders\": [\n      \"csfg\"\n    ],\n    \"frozen\": [\n      1,\n      2\n    ],\n"
        "    \"k\": 2,\n    \"max_frames\": 100000,\n    \"max_iter\": 40,\n    \"min_frame_errors\": 100,\n"
        "    \"n\": 4,\n    \"noiseless\": false,\n    \"seed\": 18446744073709551615,\n"
        "    \"snr_db\": [\n      1.5,\n      0.0001,\n      1e+16,\n      1e+15\n    ],\n"
        "    \"workers\": 1\n  },\n  \"results\": [\n    {\n      \"avg_iters\": 40.0,\n"
        "      \"avg_pe_activations\": 1234567.0,\n      \"ber\": 0.005859375,\n      \"bit_errors\": 3,\n"
        "      \"decoder\": \"csfg\",\n      \"fer\": 0.00390625,\n      \"fer_ci95\": 1e-05,\n"
        "      \"frame_errors\": 1,\n      \"frames\": 256,\n      \"iters_ci95\": 0.0,\n"
        "      \"low_confidence\": true,\n      \"norm_computations\": 0.1,\n      \"snr_db\": 1.5\n    }\n  ]\n}\n";
    const std::string got = results_json(cfg, rows);
    CHECK(got == want);
    if (got != want) std::printf("%s", got.c_str());
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
    // test_csfg_freeze.cpp:248-293: 300 trials of (64,32) at 2 dB, seed 4242: the
    // frontier grows as a prefix, stamps increase, and replaying the GPU's freeze
    // events through FreezeState/is_pe_active reproduces its PE count
    {
        const PolarCode c64 = PolarCode::construct(64, 32, 0.5);
        int bad = 0;
        for (int t = 0; t < 300; ++t) {
            TrialRng rng(4242, t);
            Bits info(32);
            for (auto& b : info) b = rng.bit();
            const auto llr = transmit_awgn(modulate_bpsk(encode(c64, info).x), {2.0, 0.5, false}, rng);
            std::vector<FreezeEvent> evs;
            const DecodeOutcome out = decode_csfg(c64, llr, 0.9375, 40, &evs);
            for (int i : c64.frozen_positions()) bad += out.u_hat[i] != 0;
            int frontier = 0;
            for (size_t e = 0; e < evs.size(); ++e) {
                const FreezeEvent& ev = evs[e];
                bad += !(ev.start <= frontier && ev.start + ev.size > frontier && ev.start % ev.size == 0 &&
                         ev.size == 64 >> (ev.stage + 1));
                if (e) bad += !(ev.iteration > evs[e - 1].iteration ||
                                (ev.iteration == evs[e - 1].iteration && ev.stage > evs[e - 1].stage));
                frontier = ev.start + ev.size;
            }
            bad += (out.stop_reason == StopReason::csfg_complete) != (frontier == 64);
            FreezeState fz(64);
            long long pe = 0;
            size_t e = 0;
            for (int it = 1; it <= out.iterations_used; ++it)
                for (int s2 = 0; s2 < c64.m && fz.frontier < 64; ++s2) {
                    for (int r = 0; r < 64; ++r)
                        if (!(r & (64 >> (s2 + 1))) && is_pe_active(fz, s2, r)) ++pe;
                    if (e < evs.size() && evs[e].iteration == it && evs[e].stage == s2) {
                        for (int r = evs[e].start; r < evs[e].start + evs[e].size; ++r)
                            fz.freeze_stage[r] = std::min(fz.freeze_stage[r], s2);
                        fz.frontier = evs[e].start + evs[e].size;
                        ++e;
                    }
                }
            bad += pe != out.pe_activations;
        }
        CHECK(bad == 0);
    }
    // test_csfg_freeze.cpp:295-314: past the frontier, decode_csfg falls back to the hard
    // decisions (0 dB, two iterations: some frame stops at max_iter with frozen rows 0)
    {
        const PolarCode c64 = PolarCode::construct(64, 32, 0.5);
        bool saw = false;
        int bad = 0;
        for (int t = 0; t < 50 && !saw; ++t) {
            TrialRng rng(777, t);
            Bits info(32);
            for (auto& b : info) b = rng.bit();
            const auto llr = transmit_awgn(modulate_bpsk(encode(c64, info).x), {0.0, 0.5, false}, rng);
            const DecodeOutcome out = decode_csfg(c64, llr, 0.9375, 2);
            if (out.stop_reason == StopReason::max_iter) {
                saw = true;
                bad += out.iterations_used != 2;
                for (int i : c64.frozen_positions()) bad += out.u_hat[i] != 0;
            }
        }
        CHECK(saw && bad == 0);
    }
    // acceptance.cpp:209-272, 275-300 (criterion 6): 10^4 random small codes, lengths,
    // rates, design points, iteration caps and Eb/N0 - frozen-bit safety of csfg and
    // G-stop, prefix-only frontier growth with increasing (iteration, stage) stamps,
    // per-iteration activation counts that never increase, the replayed total equal to
    // the reported PE count, and the decided prefix of u_hat equal to the events'
    // polar_transform(x_hat) applied in order (each committed block frozen-consistent)
    {
        std::mt19937_64 gen(9006);
        std::uniform_real_distribution<double> unif(0.0, 1.0);
        long long frozen_bad = 0, frontier_bad = 0, mono_bad = 0;
        for (int rep = 0; rep < 10000; ++rep) {
            const int m = 2 + static_cast<int>(gen() % 5);
            const int n = 1 << m;
            const int k = 1 + static_cast<int>(gen() % n);
            const PolarCode code = PolarCode::construct(n, k, 0.25 + 0.5 * unif(gen));
            const int max_iter = 4 + static_cast<int>(gen() % 12);
            const double snr = 4.0 * unif(gen);
            TrialRng rng(9006, static_cast<std::uint64_t>(rep));
            Bits info(code.k);
            for (auto& b : info) b = rng.bit();
            const auto llr = transmit_awgn(modulate_bpsk(encode(code, info).x),
                                           {snr, static_cast<double>(code.k) / n, false}, rng);
            std::vector<FreezeEvent> evs;
            const DecodeOutcome oc = decode_csfg(code, llr, 0.9375, max_iter, &evs);
            const DecodeOutcome og = decode_gmatrix(code, llr, 0.9375, max_iter);
            for (int r = 0; r < n; ++r)
                if (code.frozen[r] && (oc.u_hat[r] || og.u_hat[r])) {
                    ++frozen_bad;
                    break;
                }
            long long f = 0;
            int pi = 0, ps = 0;
            bool ok = true;
            Bits decided(n, 0);
            for (const FreezeEvent& ev : evs) {
                ok = ok && static_cast<int>(ev.x_hat.size()) == ev.size;
                if (static_cast<int>(ev.x_hat.size()) == ev.size) {
                    const Bits ub = polar_transform(ev.x_hat);
                    for (int i = 0; i < ev.size; ++i) {
                        ok = ok && !(code.frozen[ev.start + i] && ub[i]);
                        decided[ev.start + i] = ub[i];
                    }
                }
                const int size = n >> (ev.stage + 1);
                ok = ok && ev.size == size && size > 0 && ev.start % size == 0 && ev.block == ev.start / size &&
                     ev.start <= f && ev.start + ev.size > f &&
                     (ev.iteration > pi || (ev.iteration == pi && ev.stage > ps));
                pi = ev.iteration;
                ps = ev.stage;
                f = ev.start + ev.size;
            }
            ok = ok && (oc.stop_reason == StopReason::csfg_complete) == (f == n);
            for (int r = 0; r < f; ++r) ok = ok && oc.u_hat[r] == decided[r];
            frontier_bad += !ok;
            FreezeState fz(n);
            long long total = 0, prev = -1;
            size_t e = 0;
            bool mono = true;
            for (int t = 1; t <= oc.iterations_used && fz.frontier < n; ++t) {
                long long cnt = 0;
                for (int s2 = 0; s2 < m && fz.frontier < n; ++s2) {
                    for (int r = 0; r < n; ++r)
                        if (!(r & (n >> (s2 + 1))) && is_pe_active(fz, s2, r)) ++cnt;
                    while (e < evs.size() && evs[e].iteration == t && evs[e].stage == s2) {
                        for (int r = evs[e].start; r < evs[e].start + evs[e].size; ++r)
                            fz.freeze_stage[r] = std::min(fz.freeze_stage[r], s2);
                        fz.frontier = evs[e].start + evs[e].size;
                        ++e;
                    }
                }
                total += cnt;
                mono = mono && (prev < 0 || cnt <= prev);
                prev = cnt;
            }
            mono_bad += !(mono && total == oc.pe_activations && e == evs.size());
        }
        CHECK(frozen_bad == 0 && frontier_bad == 0 && mono_bad == 0);
    }
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
    // proj/test_output.txt:16-18 (acceptance.cpp:129-150): 3.0 dB, seed 61803, device batch
    // counters merged with the stop rule -> 7168 frames, FER 0.01465 / 0.01409 / 0.01423
    SimConfig a3;
    a3.code = PolarCode::construct(1024, 512, 0.5);
    a3.snr_db = {3.0};
    a3.seed = 61803;
    const auto r3 = run_sweep(a3);
    char buf[3][96];
    for (int d = 0; d < 3; ++d)
        std::snprintf(buf[d], sizeof(buf[d]), "%lld %.4g %.2f %.0f", r3[d].frames, r3[d].fer, r3[d].avg_iters,
                      r3[d].avg_pe_activations);
    CHECK(std::string(buf[0]) == "7168 0.01465 40.00 204800");
    CHECK(std::string(buf[1]) == "7168 0.01409 24.70 126442");
    CHECK(std::string(buf[2]) == "7168 0.01423 24.69 123124");
}

int main(int argc, char** argv) {
    const bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu-only") == 0;
    host_cases();
    json_case();
    if (!cpu_only) gpu_cases();
    std::printf("%d passed, %d failed\n", g_pass, g_fail);
    return g_fail;
}
