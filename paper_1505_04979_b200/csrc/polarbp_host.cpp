// Host side of the C++ drop-in (include/polarbp/*.hpp): the reference's
// namespace polarbp re-implemented over the C ABI of include/pbp.h. Decoding,
// batch frame generation and the Monte-Carlo counters run on the GPU; code
// construction, file formats, the per-trial host RNG and report formatting are
// host utilities, as in the reference.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <numbers>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "pbp.h"
#include "polarbp/bp_core.hpp"
#include "polarbp/channel.hpp"
#include "polarbp/csfg_freeze.hpp"
#include "polarbp/polar_code.hpp"
#include "polarbp/sim_harness.hpp"

namespace polarbp {

namespace {

void raise(int rc) {
    if (rc == PBP_OK) return;
    const std::string msg = pbp_last_error();
    if (rc == PBP_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// one device context per host thread (pbp_ctx is not thread-safe)
struct CtxHolder {
    pbp_ctx* ctx = nullptr;
    ~CtxHolder() {
        if (ctx) pbp_ctx_destroy(ctx);
    }
};

pbp_ctx* ctx() {
    thread_local CtxHolder h;
    if (!h.ctx) {
        const char* dev = std::getenv("PBP_DEVICE");
        raise(pbp_ctx_create(dev ? std::atoi(dev) : 0, &h.ctx));
    }
    return h.ctx;
}

pbp_code view(const PolarCode& code) { return pbp_code{code.n, code.m, code.k, code.frozen.data()}; }

std::string g10(double v) {
    char b[64];
    std::snprintf(b, sizeof(b), "%.10g", v);
    return b;
}

}  // namespace

// ---------------------------------------------------------------- polar_code

bool is_power_of_two(int v) { return v > 0 && (v & (v - 1)) == 0; }

void polar_transform_inplace(std::span<std::uint8_t> v) {
    raise(pbp_polar_transform(v.data(), static_cast<int32_t>(v.size())));
}

Bits polar_transform(Bits v) {
    polar_transform_inplace(v);
    return v;
}

std::vector<double> bhattacharyya_profile(int n, double design_z) {
    if (!is_power_of_two(n)) throw std::invalid_argument("bhattacharyya_profile: n must be a power of two");
    if (!(design_z > 0.0 && design_z < 1.0))
        throw std::invalid_argument("bhattacharyya_profile: design_z must be in (0,1)");
    std::vector<double> z(n, design_z);
    for (int half = n / 2; half >= 1; half /= 2)
        for (int i = 0; i < n; ++i)
            if (!(i & half)) {
                const double a = z[i];
                z[i] = 2.0 * a - a * a;
                z[i + half] = a * a;
            }
    return z;
}

std::vector<int> PolarCode::frozen_positions() const {
    std::vector<int> out;
    for (int i = 0; i < n; ++i)
        if (frozen[i]) out.push_back(i);
    return out;
}

PolarCode PolarCode::construct(int n, int k, double design_z) {
    Bits mask(std::max(n, 1));
    raise(pbp_construct(n, k, design_z, mask.data()));
    return from_frozen_mask(n, std::move(mask));
}

PolarCode PolarCode::from_frozen_mask(int n, Bits mask) {
    if (!is_power_of_two(n)) throw std::invalid_argument("from_frozen_mask: n must be a power of two");
    if (static_cast<int>(mask.size()) != n) throw std::invalid_argument("from_frozen_mask: mask length != n");
    PolarCode c;
    c.n = n;
    while ((1 << c.m) < n) ++c.m;
    for (auto& b : mask) b = b ? 1 : 0;
    c.k = n - static_cast<int>(std::count(mask.begin(), mask.end(), 1));
    if (c.k < 1) throw std::invalid_argument("from_frozen_mask: no information positions");
    c.frozen = std::move(mask);
    return c;
}

Codeword encode(const PolarCode& code, const Bits& info_bits) {
    if (static_cast<int>(info_bits.size()) != code.k) throw std::invalid_argument("encode: info length != k");
    Codeword cw{Bits(code.n), Bits(code.n)};
    const pbp_code v = view(code);
    raise(pbp_encode(&v, info_bits.data(), cw.u.data(), cw.x.data()));
    return cw;
}

Bits extract_info_bits(const PolarCode& code, const Bits& u) {
    if (static_cast<int>(u.size()) != code.n) throw std::invalid_argument("extract_info_bits: length != n");
    Bits out;
    out.reserve(code.k);
    for (int i = 0; i < code.n; ++i)
        if (!code.frozen[i]) out.push_back(u[i]);
    return out;
}

std::string format_frozen_set(const PolarCode& code) {
    std::string s = "n=" + std::to_string(code.n) + "\nk=" + std::to_string(code.k) + "\nfrozen=";
    bool first = true;
    for (int i = 0; i < code.n; ++i)
        if (code.frozen[i]) {
            s += (first ? "" : ",") + std::to_string(i + 1);
            first = false;
        }
    return s + "\n";
}

namespace {

std::string strip(const std::string& s) {
    const auto a = s.find_first_not_of(" \t\r");
    if (a == std::string::npos) return "";
    return s.substr(a, s.find_last_not_of(" \t\r") - a + 1);
}

long long to_int(const std::string& s, const char* what) {
    size_t used = 0;
    long long v = 0;
    bool ok = true;
    try {
        v = std::stoll(s, &used);
    } catch (const std::exception&) {
        ok = false;
    }
    if (!ok || used != s.size())
        throw std::runtime_error(std::string("frozen-set file: bad ") + what + " value '" + s + "'");
    return v;
}

std::string field(std::istream& in, const std::string& key) {
    std::string line;
    while (std::getline(in, line)) {
        line = strip(line);
        if (line.empty() || line[0] == '#') continue;
        const auto eq = line.find('=');
        if (eq == std::string::npos || strip(line.substr(0, eq)) != key)
            throw std::runtime_error("frozen-set file: expected '" + key + "=...', got '" + line + "'");
        return strip(line.substr(eq + 1));
    }
    throw std::runtime_error("frozen-set file: missing '" + key + "=' line");
}

}  // namespace

PolarCode parse_frozen_set(const std::string& text) {
    std::istringstream in(text);
    const long long n = to_int(field(in, "n"), "n");
    const long long k = to_int(field(in, "k"), "k");
    const std::string list = field(in, "frozen");
    if (n < 1 || n > (1ll << 24) || !is_power_of_two(static_cast<int>(n)))
        throw std::runtime_error("frozen-set file: n must be a power of two");
    if (k < 1 || k > n) throw std::runtime_error("frozen-set file: k out of range");
    Bits mask(n, 0);
    long long count = 0, prev = 0;
    std::istringstream items(list);
    std::string item;
    while (std::getline(items, item, ',')) {
        item = strip(item);
        if (item.empty()) throw std::runtime_error("frozen-set file: empty frozen index");
        const long long idx = to_int(item, "frozen index");
        if (idx < 1 || idx > n)
            throw std::runtime_error("frozen-set file: frozen index " + std::to_string(idx) + " outside 1.." +
                                     std::to_string(n));
        if (idx <= prev) throw std::runtime_error("frozen-set file: frozen indices must be strictly ascending");
        prev = idx;
        mask[idx - 1] = 1;
        ++count;
    }
    if (count != n - k)
        throw std::runtime_error("frozen-set file: " + std::to_string(count) + " frozen indices but n-k=" +
                                 std::to_string(n - k));
    return PolarCode::from_frozen_mask(static_cast<int>(n), std::move(mask));
}

void save_frozen_set_file(const PolarCode& code, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open for write: " + path);
    out << format_frozen_set(code);
    if (!out) throw std::runtime_error("write failed: " + path);
}

PolarCode load_frozen_set_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open: " + path);
    std::ostringstream buf;
    buf << in.rdbuf();
    return parse_frozen_set(buf.str());
}

// ---------------------------------------------------------------- channel

double noise_variance(double ebn0_db, double rate) {
    double v = 0.0;
    raise(pbp_noise_variance(ebn0_db, rate, &v));
    return v;
}

namespace {
std::uint64_t splitmix_final(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
}  // namespace

TrialRng::TrialRng(std::uint64_t master_seed, std::uint64_t trial)
    : engine_(splitmix_final(master_seed + 0x9E3779B97F4A7C15ULL * (trial + 1))) {}

double TrialRng::gaussian() {
    const double u1 = static_cast<double>((engine_() >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(engine_() >> 11) * 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2);
}

std::uint8_t TrialRng::bit() { return static_cast<std::uint8_t>(engine_() >> 63); }

std::vector<double> modulate_bpsk(const Bits& x) {
    std::vector<double> s(x.size());
    for (size_t i = 0; i < x.size(); ++i) s[i] = x[i] ? -1.0 : 1.0;
    return s;
}

std::vector<double> transmit_awgn(std::span<const double> symbols, const ChannelConfig& config, TrialRng& rng) {
    const double s2 = noise_variance(config.ebn0_db, config.rate);
    const double sigma = std::sqrt(s2), scale = 2.0 / s2;
    std::vector<double> llr(symbols.size());
    for (size_t i = 0; i < symbols.size(); ++i)
        llr[i] = scale * (config.noiseless ? symbols[i] : symbols[i] + sigma * rng.gaussian());
    return llr;
}

namespace {
void unpack_u(const PolarCode& code, std::int64_t count, const std::vector<uint32_t>& ub, std::vector<Bits>* u_words) {
    const int nw = (code.n + 31) / 32;
    if (u_words) {
        u_words->assign(count, Bits(code.n));
        for (std::int64_t f = 0; f < count; ++f)
            for (int r = 0; r < code.n; ++r) (*u_words)[f][r] = (ub[f * nw + (r >> 5)] >> (r & 31)) & 1u;
    }
}
}  // namespace

void generate_frames(const PolarCode& code, std::uint64_t seed, std::int64_t first_trial, std::int64_t count,
                     const ChannelConfig& config, std::vector<double>& llrs, std::vector<Bits>* u_words) {
    const pbp_code v = view(code);
    const int nw = (code.n + 31) / 32;
    llrs.assign(static_cast<size_t>(count) * code.n, 0.0);
    std::vector<float> l32(static_cast<size_t>(count) * code.n);
    std::vector<uint32_t> ub(static_cast<size_t>(count) * nw);
    raise(pbp_generate(ctx(), &v, seed, first_trial, count, config.ebn0_db, config.noiseless ? 1 : 0, l32.data(),
                       llrs.data(), ub.data()));
    unpack_u(code, count, ub, u_words);
}

void generate_frames(const PolarCode& code, std::uint64_t seed, std::int64_t first_trial, std::int64_t count,
                     const ChannelConfig& config, std::vector<float>& llrs, std::vector<Bits>* u_words) {
    const pbp_code v = view(code);
    const int nw = (code.n + 31) / 32;
    llrs.assign(static_cast<size_t>(count) * code.n, 0.0f);
    std::vector<uint32_t> ub(static_cast<size_t>(count) * nw);
    raise(pbp_generate(ctx(), &v, seed, first_trial, count, config.ebn0_db, config.noiseless ? 1 : 0, llrs.data(),
                       nullptr, ub.data()));
    if (u_words) {
        u_words->assign(count, Bits(code.n));
        for (std::int64_t f = 0; f < count; ++f)
            for (int r = 0; r < code.n; ++r) (*u_words)[f][r] = (ub[f * nw + (r >> 5)] >> (r & 31)) & 1u;
    }
}

// ---------------------------------------------------------------- decoders

PeOutputs pe_update(const PeInputs& in, double alpha) {
    // host utility with the reference's sgn(0)=+1, std::min and clamp rules
    auto sg = [](double v) { return v < 0.0 ? -1.0 : 1.0; };
    auto mn = [](double a, double b) { return b < a ? b : a; };
    auto cl = [](double v) { return v < -LLR_CAP ? -LLR_CAP : (LLR_CAP < v ? LLR_CAP : v); };
    const double cross = alpha * sg(in.l_top) * sg(in.r_top) * mn(std::fabs(in.l_top), std::fabs(in.r_top));
    const double sb = in.l_bot + in.r_bot;
    return {cl(alpha * sg(in.l_top) * sg(sb) * mn(std::fabs(in.l_top), std::fabs(sb))), cl(in.l_bot + cross),
            cl(alpha * sg(in.r_top) * sg(sb) * mn(std::fabs(in.r_top), std::fabs(sb))), cl(in.r_bot + cross)};
}

const char* to_string(StopReason reason) {
    switch (reason) {
        case StopReason::max_iter: return "max_iter";
        case StopReason::gmatrix_converged: return "gmatrix_converged";
        case StopReason::csfg_complete: return "csfg_complete";
    }
    return "?";
}

namespace {

// one frame with its freeze-event trace: T = double (as shipped) or float (the fp32 path)
template <typename T>
DecodeOutcome one_frame(const PolarCode& code, int kind, std::span<const T> llrs, double alpha, int max_iter,
                        std::vector<FreezeEvent>* events) {
    if (static_cast<int>(llrs.size()) != code.n) throw std::invalid_argument("init_state: LLR length != n");
    const pbp_code v = view(code);
    DecodeOutcome out;
    out.u_hat.assign(code.n, 0);
    int32_t it = 0, stop = 0, nev = 0;
    int64_t pe = 0;
    // at most one commit per stage per iteration (csfg_freeze.cpp:111-118): never truncated
    const int cap = std::max(1, max_iter * code.m), nw = (code.n + 31) / 32;
    std::vector<int32_t> ev(events ? static_cast<size_t>(cap) * 5 : 5);
    std::vector<uint32_t> xw(events ? static_cast<size_t>(cap) * nw : 0);  // each event's x_hat
    uint32_t* xp = events ? xw.data() : nullptr;
    if constexpr (sizeof(T) == 8)
        raise(pbp_decode_trace_f64_x(ctx(), &v, kind, llrs.data(), alpha, max_iter, out.u_hat.data(), &it, &pe,
                                     &stop, &nev, ev.data(), events ? cap : 1, xp));
    else
        raise(pbp_decode_trace_x(ctx(), &v, kind, llrs.data(), static_cast<float>(alpha), max_iter,
                                 out.u_hat.data(), &it, &pe, &stop, &nev, ev.data(), events ? cap : 1, xp));
    out.info_bits = extract_info_bits(code, out.u_hat);
    out.iterations_used = it;
    out.pe_activations = pe;
    out.stop_reason = static_cast<StopReason>(stop);
    if (events) {
        events->clear();
        for (int i = 0; i < std::min(nev, cap); ++i) {
            FreezeEvent fe{ev[5 * i], ev[5 * i + 1], ev[5 * i + 2], ev[5 * i + 3], ev[5 * i + 4], {}};
            const uint32_t* w = xw.data() + static_cast<size_t>(i) * nw;
            fe.x_hat.resize(fe.size);
            for (int r = 0; r < fe.size; ++r) fe.x_hat[r] = (w[(fe.start + r) >> 5] >> ((fe.start + r) & 31)) & 1u;
            events->push_back(std::move(fe));
        }
    }
    return out;
}

}  // namespace

DecodeOutcome decode_baseline(const PolarCode& code, std::span<const double> llrs, double alpha, int max_iter) {
    return one_frame<double>(code, PBP_BASELINE, llrs, alpha, max_iter, nullptr);
}

DecodeOutcome decode_gmatrix(const PolarCode& code, std::span<const double> llrs, double alpha, int max_iter) {
    return one_frame<double>(code, PBP_GMATRIX, llrs, alpha, max_iter, nullptr);
}

DecodeOutcome decode_csfg(const PolarCode& code, std::span<const double> llrs, double alpha, int max_iter,
                          std::vector<FreezeEvent>* events) {
    return one_frame<double>(code, PBP_CSFG, llrs, alpha, max_iter, events);
}

namespace {
template <typename T>
std::vector<DecodeOutcome> batch_impl(const PolarCode& code, BatchDecoder decoder, std::span<const T> llrs,
                                      double alpha, int max_iter) {
    if (llrs.size() % code.n) throw std::invalid_argument("init_state: LLR length != n");
    const int64_t frames = static_cast<int64_t>(llrs.size() / code.n);
    const int nw = (code.n + 31) / 32;
    std::vector<uint32_t> ub(static_cast<size_t>(frames) * nw);
    std::vector<int32_t> it(frames), nev(frames);
    std::vector<int64_t> pe(frames);
    std::vector<uint8_t> stop(frames);
    pbp_frame_out fo{ub.data(), it.data(), pe.data(), stop.data(), nev.data()};
    const pbp_code v = view(code);
    if constexpr (sizeof(T) == 8)
        raise(pbp_decode_batch_f64(ctx(), &v, static_cast<int>(decoder), llrs.data(), frames, alpha, max_iter, &fo));
    else
        raise(pbp_decode_batch(ctx(), &v, static_cast<int>(decoder), llrs.data(), frames, static_cast<float>(alpha),
                               max_iter, &fo));
    std::vector<DecodeOutcome> out(frames);
    for (int64_t f = 0; f < frames; ++f) {
        out[f].u_hat.resize(code.n);
        for (int r = 0; r < code.n; ++r) out[f].u_hat[r] = (ub[f * nw + (r >> 5)] >> (r & 31)) & 1u;
        out[f].info_bits = extract_info_bits(code, out[f].u_hat);
        out[f].iterations_used = it[f];
        out[f].pe_activations = pe[f];
        out[f].stop_reason = static_cast<StopReason>(stop[f]);
    }
    return out;
}
}  // namespace

std::vector<DecodeOutcome> decode_batch(const PolarCode& code, BatchDecoder decoder, std::span<const float> llrs,
                                        double alpha, int max_iter) {
    return batch_impl<float>(code, decoder, llrs, alpha, max_iter);
}

std::vector<DecodeOutcome> decode_batch(const PolarCode& code, BatchDecoder decoder, std::span<const double> llrs,
                                        double alpha, int max_iter) {
    return batch_impl<double>(code, decoder, llrs, alpha, max_iter);
}

BlockRef candidate_block(int n, int frontier, int stage) {
    BlockRef b;
    b.stage = stage;
    b.size = n >> (stage + 1);
    b.index = frontier / b.size;
    b.start = b.index * b.size;
    return b;
}

std::optional<CsfgDecision> freeze_decision(std::span<const double> r_block, std::span<const std::uint8_t> frozen_block) {
    if (r_block.size() != frozen_block.size()) throw std::invalid_argument("freeze_decision: span length mismatch");
    CsfgDecision d;
    d.x_hat.resize(r_block.size());
    for (size_t i = 0; i < r_block.size(); ++i) d.x_hat[i] = r_block[i] < 0.0 ? 1 : 0;
    d.u_hat = polar_transform(d.x_hat);
    for (size_t i = 0; i < r_block.size(); ++i)
        if (frozen_block[i] && d.u_hat[i]) return std::nullopt;
    return d;
}

bool is_pe_active(std::span<const int> freeze_stage, int stage, int top_row) {
    return stage <= freeze_stage[top_row];
}

// ---------------------------------------------------------------- harness

const char* to_string(DecoderKind kind) {
    switch (kind) {
        case DecoderKind::baseline: return "baseline";
        case DecoderKind::gmatrix: return "gmatrix";
        case DecoderKind::csfg: return "csfg";
    }
    return "?";
}

DecoderKind parse_decoder(const std::string& name) {
    if (name == "baseline") return DecoderKind::baseline;
    if (name == "gmatrix") return DecoderKind::gmatrix;
    if (name == "csfg") return DecoderKind::csfg;
    throw std::invalid_argument("unknown decoder '" + name + "'");
}

namespace {

struct Acc {
    long long frames = 0, bit_errors = 0, frame_errors = 0, sum_iters = 0, sum_iters_sq = 0, sum_pe = 0;
};

PointStats stats_of(const SimConfig& cfg, DecoderKind kind, double snr, const Acc& a) {
    PointStats r;
    r.decoder = kind;
    r.snr_db = snr;
    r.frames = a.frames;
    r.bit_errors = a.bit_errors;
    r.frame_errors = a.frame_errors;
    const double f = static_cast<double>(a.frames);
    r.ber = static_cast<double>(a.bit_errors) / (f * cfg.code.k);
    r.fer = static_cast<double>(a.frame_errors) / f;
    r.fer_ci95 = 1.96 * std::sqrt(r.fer * (1.0 - r.fer) / f);
    r.avg_iters = static_cast<double>(a.sum_iters) / f;
    if (a.frames > 1) {
        const double var = (static_cast<double>(a.sum_iters_sq) - f * r.avg_iters * r.avg_iters) / (f - 1.0);
        r.iters_ci95 = 1.96 * std::sqrt(std::max(var, 0.0) / f);
    }
    r.avg_pe_activations = static_cast<double>(a.sum_pe) / f;
    const double full = static_cast<double>(cfg.max_iter) * cfg.code.m * (cfg.code.n / 2);
    r.norm_computations = full > 0.0 ? r.avg_pe_activations / full : 0.0;
    r.low_confidence = a.frame_errors < cfg.min_frame_errors;
    return r;
}

}  // namespace

namespace {

// one context per visible device for one run_point call (pbp_ctx is not
// thread-safe: each worker thread drives its own device's context)
struct DevicePool {
    std::vector<pbp_ctx*> ctx;
    explicit DevicePool(int want) {
        const int n = std::max(1, std::min(want, pbp_device_count()));
        for (int d = 0; d < n; ++d) {
            pbp_ctx* c = nullptr;
            const int rc = pbp_ctx_create(d, &c);
            if (rc) {
                this->~DevicePool();
                raise(rc);
            }
            ctx.push_back(c);
        }
    }
    ~DevicePool() {
        for (pbp_ctx* c : ctx)
            if (c) pbp_ctx_destroy(c);
        ctx.clear();
    }
};

void add_batch(Acc& a, const std::int64_t* c) {
    a.frames += c[0];
    a.bit_errors += c[1];
    a.frame_errors += c[2];
    a.sum_iters += c[3];
    a.sum_iters_sq += c[4];
    a.sum_pe += c[5];
}

}  // namespace

// run_point (sim_harness.cpp:129-186). Without a trace sink the trials are
// generated and decoded on the GPUs, which return one int64 counter set per
// 256-trial batch (pbp_simulate_batches); chunks of whole batches are split
// into contiguous per-device ranges (one host thread per visible GPU), and
// the batches are merged in trial order with the stop rule checked at every
// batch boundary, as in the reference -- so the rows are identical for any
// device count. With a trace sink (single device, as the reference forces one
// worker) each 256-trial batch is decoded frame by frame with its freeze
// events, and events are emitted only for the batches that are merged.
std::vector<PointStats> run_point(const SimConfig& cfg, double snr_db, const TraceSink* trace) {
    if (cfg.decoders.empty()) throw std::invalid_argument("run_point: no decoders");
    if (cfg.max_frames < 1) throw std::invalid_argument("run_point: max_frames < 1");
    constexpr long long kBatch = 256;  // stop rule granularity (sim_harness.cpp:21)
    const PolarCode& code = cfg.code;
    const size_t nd = cfg.decoders.size();
    std::vector<Acc> acc(nd);
    auto finish = [&]() {
        std::vector<PointStats> rows;
        for (size_t d = 0; d < nd; ++d) rows.push_back(stats_of(cfg, cfg.decoders[d], snr_db, acc[d]));
        return rows;
    };
    auto enough = [&]() {
        for (const Acc& a : acc)
            if (a.frame_errors < cfg.min_frame_errors) return false;
        return true;
    };
    long long frames = 0;
    if (trace) {
        const ChannelConfig ch{snr_db, static_cast<double>(code.k) / code.n, cfg.noiseless};
        while (frames < cfg.max_frames) {
            const long long c = std::min(kBatch, cfg.max_frames - frames);
            std::vector<float> llr;
            std::vector<double> llr64;
            std::vector<Bits> u;
            if (cfg.fp64)
                generate_frames(code, cfg.seed, frames, c, ch, llr64, &u);
            else
                generate_frames(code, cfg.seed, frames, c, ch, llr, &u);
            for (long long f = 0; f < c; ++f)
                for (size_t d = 0; d < nd; ++d) {
                    const int kind = static_cast<int>(cfg.decoders[d]);
                    std::vector<FreezeEvent> ev;
                    std::vector<FreezeEvent>* evp = cfg.decoders[d] == DecoderKind::csfg ? &ev : nullptr;
                    const DecodeOutcome o =
                        cfg.fp64 ? one_frame<double>(code, kind, std::span<const double>(llr64.data() + f * code.n, code.n),
                                                     cfg.alpha, cfg.max_iter, evp)
                                 : one_frame<float>(code, kind, std::span<const float>(llr.data() + f * code.n, code.n),
                                                    cfg.alpha, cfg.max_iter, evp);
                    for (const auto& e : ev) (*trace)(frames + f, e);
                    long long be = 0;
                    for (int r = 0; r < code.n; ++r)
                        if (!code.frozen[r] && o.u_hat[r] != u[f][r]) ++be;
                    const std::int64_t cell[6] = {1, be, be > 0, o.iterations_used,
                                                  static_cast<long long>(o.iterations_used) * o.iterations_used,
                                                  o.pe_activations};
                    add_batch(acc[d], cell);
                }
            frames += c;
            if (enough()) break;
        }
        return finish();
    }
    DevicePool pool(pbp_device_count());
    const int ng = static_cast<int>(pool.ctx.size());
    const pbp_code cv = view(code);
    long long chunk = kBatch * 16;
    std::vector<std::int64_t> cnt;
    while (frames < cfg.max_frames) {
        const long long c = std::min(chunk, cfg.max_frames - frames);
        const long long nb = (c + kBatch - 1) / kBatch;
        cnt.assign(static_cast<size_t>(nd * nb * 10), 0);
        // device g takes batches [nb*g/ng, nb*(g+1)/ng) of every decoder
        std::vector<int> rcs(ng, PBP_OK);
        std::vector<std::string> errs(ng);
        auto work = [&](int g) {
            const long long b0 = nb * g / ng, b1 = nb * (g + 1) / ng;
            if (b1 <= b0) return;
            const long long first = frames + b0 * kBatch;
            const long long count = std::min(c, b1 * kBatch) - b0 * kBatch;
            for (size_t d = 0; d < nd && !rcs[g]; ++d) {
                rcs[g] = pbp_simulate_batches(pool.ctx[g], &cv, static_cast<int>(cfg.decoders[d]), cfg.seed, first,
                                              count, static_cast<int32_t>(kBatch), snr_db, cfg.noiseless ? 1 : 0,
                                              cfg.alpha, cfg.max_iter, cfg.fp64 ? 1 : 0,
                                              cnt.data() + (d * nb + b0) * 10);
                if (rcs[g]) errs[g] = pbp_last_error();
            }
        };
        if (ng == 1) {
            work(0);
        } else {
            std::vector<std::thread> th;
            for (int g = 0; g < ng; ++g) th.emplace_back(work, g);
            for (auto& t : th) t.join();
        }
        for (int g = 0; g < ng; ++g)
            if (rcs[g]) {
                if (rcs[g] == PBP_EINVAL) throw std::invalid_argument(errs[g]);
                throw std::runtime_error(errs[g]);
            }
        // merge in trial order, stop rule on 256-frame batch boundaries
        for (long long b = 0; b < nb; ++b) {
            for (size_t d = 0; d < nd; ++d) add_batch(acc[d], cnt.data() + (d * nb + b) * 10);
            if (enough()) return finish();
        }
        frames += c;
        chunk = std::min(chunk * 2, kBatch * 1024);
    }
    return finish();
}

std::vector<PointStats> run_sweep(const SimConfig& cfg, const TraceSink* trace) {
    if (cfg.snr_db.empty()) throw std::invalid_argument("run_sweep: no SNR points");
    std::vector<PointStats> rows;
    for (double s : cfg.snr_db) {
        auto p = run_point(cfg, s, trace);
        rows.insert(rows.end(), p.begin(), p.end());
    }
    return rows;
}

namespace {
const char* kCsvHeader =
    "decoder,snr_db,frames,bit_errors,frame_errors,ber,fer,fer_ci95,avg_iters,iters_ci95,avg_pe_activations,"
    "norm_computations";
}

std::string results_csv(std::span<const PointStats> rows) {
    std::string s = std::string(kCsvHeader) + "\n";
    for (const auto& r : rows)
        s += std::string(to_string(r.decoder)) + "," + g10(r.snr_db) + "," + std::to_string(r.frames) + "," +
             std::to_string(r.bit_errors) + "," + std::to_string(r.frame_errors) + "," + g10(r.ber) + "," + g10(r.fer) +
             "," + g10(r.fer_ci95) + "," + g10(r.avg_iters) + "," + g10(r.iters_ci95) + "," +
             g10(r.avg_pe_activations) + "," + g10(r.norm_computations) + "\n";
    return s;
}

std::vector<PointStats> parse_results_csv(const std::string& text) {
    std::istringstream in(text);
    std::string line;
    if (!std::getline(in, line)) throw std::runtime_error("results CSV: empty input");
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line != kCsvHeader) throw std::runtime_error("results CSV: unexpected header");
    std::vector<PointStats> rows;
    while (std::getline(in, line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty()) continue;
        std::vector<std::string> f;
        std::istringstream ls(line);
        std::string x;
        while (std::getline(ls, x, ',')) f.push_back(x);
        if (f.size() != 12) throw std::runtime_error("results CSV: expected 12 fields, got line '" + line + "'");
        PointStats r;
        r.decoder = parse_decoder(f[0]);
        r.snr_db = std::stod(f[1]);
        r.frames = std::stoll(f[2]);
        r.bit_errors = std::stoll(f[3]);
        r.frame_errors = std::stoll(f[4]);
        r.ber = std::stod(f[5]);
        r.fer = std::stod(f[6]);
        r.fer_ci95 = std::stod(f[7]);
        r.avg_iters = std::stod(f[8]);
        r.iters_ci95 = std::stod(f[9]);
        r.avg_pe_activations = std::stod(f[10]);
        r.norm_computations = std::stod(f[11]);
        rows.push_back(r);
    }
    return rows;
}

namespace {

// A JSON value in the form nlohmann::json::dump(2) prints it (the reference's
// writer, sim_harness.cpp:250-289): objects are std::map-ordered (sorted
// keys), every array element and object member on its own line indented by 2
// per level, "key": value, empty containers as [] / {}, integers as-is,
// booleans true/false, doubles as the shortest round-trip digits laid out
// like nlohmann's format_buffer (fixed for decimal exponents -4 < n <= 15,
// with ".0" appended to integral values; else d[.igits]e+XX).
struct Json {
    enum Kind { kObj, kArr, kStr, kRaw } kind = kRaw;
    std::string text;                                // kStr / kRaw
    std::vector<std::pair<std::string, Json>> items; // kObj (key order fixed below) / kArr (key unused)
};

std::string json_double(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[64];
    const auto res = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
    // digits d.ddddde[+-]x -> digit string and decimal exponent of the last digit
    std::string sci(buf, res.ptr);
    std::string sign;
    if (sci[0] == '-') {
        sign = "-";
        sci.erase(0, 1);
    }
    const size_t epos = sci.find('e');
    const int e10 = std::atoi(sci.c_str() + epos + 1);
    std::string digits;
    for (size_t i = 0; i < epos; ++i)
        if (sci[i] != '.') digits += sci[i];
    while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
    const int k = static_cast<int>(digits.size());
    const int n = e10 + 1;  // decimal point position
    std::string out;
    if (k <= n && n <= 15) {
        out = digits + std::string(n - k, '0') + ".0";
    } else if (0 < n && n <= 15) {
        out = digits.substr(0, n) + "." + digits.substr(n);
    } else if (-4 < n && n <= 0) {
        out = "0." + std::string(-n, '0') + digits;
    } else {
        out = digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int x = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof(eb), "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
        out += eb;
    }
    return sign + out;
}

std::string json_escape(const std::string& s) {
    std::string o = "\"";
    for (unsigned char c : s) {
        switch (c) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\b': o += "\\b"; break;
            case '\f': o += "\\f"; break;
            case '\n': o += "\\n"; break;
            case '\r': o += "\\r"; break;
            case '\t': o += "\\t"; break;
            default:
                if (c < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof(b), "\\u%04x", c);
                    o += b;
                } else {
                    o += static_cast<char>(c);
                }
        }
    }
    return o + "\"";
}

Json jraw(std::string t) { return Json{Json::kRaw, std::move(t), {}}; }
Json jstr(const std::string& t) { return Json{Json::kStr, json_escape(t), {}}; }
Json jnum(double v) { return jraw(json_double(v)); }
template <class I>
Json jint(I v) { return jraw(std::to_string(v)); }
Json jbool(bool v) { return jraw(v ? "true" : "false"); }
Json jobj(std::vector<std::pair<std::string, Json>> m) {
    std::sort(m.begin(), m.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    return Json{Json::kObj, "", std::move(m)};
}
Json jarr(std::vector<Json> v) {
    Json j{Json::kArr, "", {}};
    for (auto& x : v) j.items.emplace_back("", std::move(x));
    return j;
}

void dump2(const Json& j, int depth, std::string& o) {
    if (j.kind == Json::kRaw || j.kind == Json::kStr) {
        o += j.text;
        return;
    }
    const char open = j.kind == Json::kObj ? '{' : '[', close = j.kind == Json::kObj ? '}' : ']';
    if (j.items.empty()) {
        o += open;
        o += close;
        return;
    }
    o += open;
    o += '\n';
    const std::string ind(2 * (depth + 1), ' ');
    for (size_t i = 0; i < j.items.size(); ++i) {
        o += ind;
        if (j.kind == Json::kObj) o += json_escape(j.items[i].first) + ": ";
        dump2(j.items[i].second, depth + 1, o);
        if (i + 1 < j.items.size()) o += ',';
        o += '\n';
    }
    o += std::string(2 * depth, ' ');
    o += close;
}

}  // namespace

std::string results_json(const SimConfig& cfg, std::span<const PointStats> rows) {
    std::vector<Json> frozen, decoders, snrs, results;
    for (int pos : cfg.code.frozen_positions()) frozen.push_back(jint(pos + 1));
    for (DecoderKind d : cfg.decoders) decoders.push_back(jstr(to_string(d)));
    for (double v : cfg.snr_db) snrs.push_back(jnum(v));
    for (const PointStats& r : rows)
        results.push_back(jobj({{"decoder", jstr(to_string(r.decoder))},
                                {"snr_db", jnum(r.snr_db)},
                                {"frames", jint(r.frames)},
                                {"bit_errors", jint(r.bit_errors)},
                                {"frame_errors", jint(r.frame_errors)},
                                {"ber", jnum(r.ber)},
                                {"fer", jnum(r.fer)},
                                {"fer_ci95", jnum(r.fer_ci95)},
                                {"avg_iters", jnum(r.avg_iters)},
                                {"iters_ci95", jnum(r.iters_ci95)},
                                {"avg_pe_activations", jnum(r.avg_pe_activations)},
                                {"norm_computations", jnum(r.norm_computations)},
                                {"low_confidence", jbool(r.low_confidence)}}));
    const Json j = jobj({{"config", jobj({{"n", jint(cfg.code.n)},
                                          {"k", jint(cfg.code.k)},
                                          {"frozen", jarr(frozen)},
                                          {"code_source", jstr(cfg.code_source)},
                                          {"decoders", jarr(decoders)},
                                          {"snr_db", jarr(snrs)},
                                          {"alpha", jnum(cfg.alpha)},
                                          {"max_iter", jint(cfg.max_iter)},
                                          {"min_frame_errors", jint(cfg.min_frame_errors)},
                                          {"max_frames", jint(cfg.max_frames)},
                                          {"seed", jint(cfg.seed)},
                                          {"workers", jint(cfg.workers)},
                                          {"noiseless", jbool(cfg.noiseless)}})},
                         {"results", jarr(results)}});
    std::string o;
    dump2(j, 0, o);
    return o + "\n";
}

std::vector<SavingsRow> compute_savings(std::span<const PointStats> rows) {
    std::map<double, std::map<DecoderKind, const PointStats*>> by;
    for (const auto& r : rows) by[r.snr_db][r.decoder] = &r;
    std::vector<SavingsRow> out;
    for (const auto& [snr, m] : by) {
        const auto c = m.find(DecoderKind::csfg);
        if (c == m.end()) continue;
        const auto b = m.find(DecoderKind::baseline), g = m.find(DecoderKind::gmatrix);
        if (b == m.end() || g == m.end())
            throw std::runtime_error("savings: missing baseline or gmatrix row at snr_db=" + g10(snr));
        out.push_back({snr, 1.0 - c->second->avg_iters / b->second->avg_iters,
                       1.0 - c->second->avg_iters / g->second->avg_iters,
                       1.0 - c->second->avg_pe_activations / b->second->avg_pe_activations,
                       1.0 - c->second->avg_pe_activations / g->second->avg_pe_activations});
    }
    if (out.empty()) throw std::runtime_error("savings: no csfg rows to report");
    return out;
}

std::string savings_table(std::span<const SavingsRow> rows) {
    char b[200];
    std::snprintf(b, sizeof(b), "%8s  %18s  %17s  %17s  %16s\n", "snr_db", "iters_vs_baseline", "iters_vs_gmatrix",
                  "comp_vs_baseline", "comp_vs_gmatrix");
    std::string s = b;
    for (const auto& r : rows) {
        std::snprintf(b, sizeof(b), "%8s  %17.1f%%  %16.1f%%  %16.1f%%  %15.1f%%\n", g10(r.snr_db).c_str(),
                      100.0 * r.iters_vs_baseline, 100.0 * r.iters_vs_gmatrix, 100.0 * r.comp_vs_baseline,
                      100.0 * r.comp_vs_gmatrix);
        s += b;
    }
    return s;
}

}  // namespace polarbp
