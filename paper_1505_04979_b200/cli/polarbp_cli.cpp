// polarbp: command-line front end of the B200 decoder (drop-in for the
// reference's proj/tools/polarbp_main.cpp:147-308). Same subcommands, options,
// defaults and output lines:
//   construct --n N --k K [--design-z Z] [--out FILE]
//   encode    (--n N --k K [--design-z Z] | --frozen-file F) --info BITS
//   decode    (code) --llr-file F [--decoder baseline|gmatrix|csfg] [--alpha A]
//             [--max-iter I] [--trace]
//   simulate  (code) --snr LIST [--decoders LIST] [--alpha A] [--max-iter I]
//             [--seed S | env POLARBP_SEED] [--workers W] [--min-frame-errors E]
//             [--max-frames F] [--out CSV] [--json FILE] [--trace] [--noiseless] [--fp64]
//   report    --in CSV
// Results go to stdout (or --out/--json), diagnostics and freeze-event traces to
// stderr. Exit status: 0 ok, 1 runtime error ("error: ..." on stderr, as the
// reference), 2 command-line usage error. Decoding runs on the GPU through
// libpbp.so (decode: double arithmetic as shipped; simulate: the fp32 fast
// path, --fp64 for double); there is no CPU decoder.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "polarbp/bp_core.hpp"
#include "polarbp/channel.hpp"
#include "polarbp/csfg_freeze.hpp"
#include "polarbp/polar_code.hpp"
#include "polarbp/sim_harness.hpp"

namespace {

using namespace polarbp;

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---- option table and parsing -------------------------------------------------
struct Spec {
    bool takes_value;
    bool required;
    std::string help;
};
using Table = std::map<std::string, Spec>;

struct Parsed {
    std::map<std::string, std::string> values;
    std::set<std::string> flags;
    bool has(const std::string& k) const { return values.count(k) || flags.count(k); }
    std::string get(const std::string& k, const std::string& dflt) const {
        auto it = values.find(k);
        return it == values.end() ? dflt : it->second;
    }
};

Parsed parse_options(const std::string& cmd, const Table& table, int argc, char** argv, int first) {
    Parsed p;
    for (int i = first; i < argc; ++i) {
        std::string tok = argv[i];
        if (tok.rfind("--", 0) != 0) throw UsageError(cmd + ": unexpected argument '" + tok + "'");
        std::string name = tok.substr(2), value;
        bool inline_value = false;
        if (const auto eq = name.find('='); eq != std::string::npos) {
            value = name.substr(eq + 1);
            name = name.substr(0, eq);
            inline_value = true;
        }
        const auto it = table.find(name);
        if (it == table.end()) throw UsageError(cmd + ": unknown option --" + name);
        if (!it->second.takes_value) {
            if (inline_value) throw UsageError(cmd + ": --" + name + " takes no value");
            p.flags.insert(name);
            continue;
        }
        if (!inline_value) {
            if (i + 1 >= argc) throw UsageError(cmd + ": --" + name + " needs a value");
            value = argv[++i];
        }
        if (p.values.count(name)) throw UsageError(cmd + ": --" + name + " given twice");
        p.values[name] = value;
    }
    for (const auto& [name, spec] : table)
        if (spec.required && !p.has(name)) throw UsageError(cmd + ": --" + name + " is required");
    return p;
}

long long to_int(const std::string& opt, const std::string& s) {
    std::size_t used = 0;
    long long v = 0;
    try {
        v = std::stoll(s, &used);
    } catch (const std::exception&) {
        used = 0;
    }
    if (used == 0 || used != s.size()) throw UsageError("--" + opt + ": not an integer: '" + s + "'");
    return v;
}

double to_real(const std::string& opt, const std::string& s) {
    std::size_t used = 0;
    double v = 0.0;
    try {
        v = std::stod(s, &used);
    } catch (const std::exception&) {
        used = 0;
    }
    if (used == 0 || used != s.size()) throw UsageError("--" + opt + ": not a number: '" + s + "'");
    return v;
}

// ---- shared pieces ----------------------------------------------------------------
void add_code_options(Table& t) {
    t["n"] = {true, false, "block length (power of two)"};
    t["k"] = {true, false, "information bits"};
    t["design-z"] = {true, false, "design-channel parameter for the frozen-set construction (0.5)"};
    t["frozen-file"] = {true, false, "frozen-set file to load"};
}

// --frozen-file, or --n with --k (+ --design-z); source text as in results_json
PolarCode code_from(const Parsed& p, std::string* source = nullptr) {
    const bool file = p.has("frozen-file"), n = p.has("n"), k = p.has("k");
    if (file && (n || k)) throw UsageError("--frozen-file excludes --n/--k");
    if (n != k) throw UsageError(n ? "--n needs --k" : "--k needs --n");
    if (file) {
        const std::string path = p.get("frozen-file", "");
        if (source) *source = "file:" + path;
        return load_frozen_set_file(path);
    }
    if (!n) throw std::runtime_error("specify either --frozen-file or --n/--k");
    const double z = to_real("design-z", p.get("design-z", "0.5"));
    if (source) {
        std::ostringstream s;
        s << "bhattacharyya design_z=" << z;
        *source = s.str();
    }
    return PolarCode::construct(static_cast<int>(to_int("n", p.get("n", ""))),
                                static_cast<int>(to_int("k", p.get("k", ""))), z);
}

std::string bit_text(const Bits& b) {
    std::string s;
    s.reserve(b.size());
    for (auto v : b) s.push_back(v ? '1' : '0');
    return s;
}

Bits bits_from_text(const std::string& text, int want, const char* what) {
    if (static_cast<int>(text.size()) != want)
        throw std::runtime_error(std::string(what) + ": expected " + std::to_string(want) + " bits, got " +
                                 std::to_string(text.size()));
    Bits b;
    b.reserve(text.size());
    for (char c : text) {
        if (c != '0' && c != '1') throw std::runtime_error(std::string(what) + ": bits must be 0 or 1");
        b.push_back(static_cast<std::uint8_t>(c == '1'));
    }
    return b;
}

std::vector<double> llrs_from_file(const std::string& path, int want) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open: " + path);
    std::vector<double> v;
    for (double x; in >> x;) v.push_back(x);
    if (!in.eof()) throw std::runtime_error("llr file: non-numeric content in " + path);
    if (static_cast<int>(v.size()) != want)
        throw std::runtime_error("llr file: expected " + std::to_string(want) + " values, got " +
                                 std::to_string(v.size()));
    return v;
}

// "a,b,c" or "start:stop:step" (inclusive, half-step slack)
std::vector<double> snr_points(const std::string& text) {
    std::vector<double> pts;
    if (text.find(':') != std::string::npos) {
        std::istringstream in(text);
        double lo = 0, hi = 0, step = 0;
        char c1 = 0, c2 = 0;
        if (!(in >> lo >> c1 >> hi >> c2 >> step) || c1 != ':' || c2 != ':' || !(in >> std::ws).eof())
            throw std::runtime_error("bad --snr range '" + text + "' (want start:stop:step)");
        if (step <= 0.0) throw std::runtime_error("--snr step must be positive");
        if (hi < lo) throw std::runtime_error("--snr stop below start");
        for (double v = lo; v <= hi + step / 2.0; v += step) pts.push_back(v);
    } else {
        std::size_t pos = 0;
        while (pos <= text.size()) {
            const std::size_t comma = text.find(',', pos);
            const std::string item = text.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
            if (item.empty()) throw std::runtime_error("empty --snr entry");
            std::size_t used = 0;
            const double v = std::stod(item, &used);
            if (used != item.size()) throw std::runtime_error("bad --snr value '" + item + "'");
            pts.push_back(v);
            if (comma == std::string::npos) break;
            pos = comma + 1;
        }
    }
    if (pts.empty()) throw std::runtime_error("--snr produced no points");
    return pts;
}

std::vector<DecoderKind> decoder_list(const std::string& text) {
    std::vector<DecoderKind> out;
    std::istringstream in(text);
    for (std::string item; std::getline(in, item, ',');) {
        const DecoderKind d = parse_decoder(item);
        bool dup = false;
        for (DecoderKind e : out) dup = dup || e == d;
        if (!dup) out.push_back(d);
    }
    if (out.empty()) throw std::runtime_error("--decoders produced no decoders");
    return out;
}

void trace_line(const FreezeEvent& ev) {  // 1-based stage / block / rows
    std::fprintf(stderr, "iter=%d stage=%d block=%d range=%d-%d\n", ev.iteration, ev.stage + 1, ev.block + 1,
                 ev.start + 1, ev.start + ev.size);
}

void write_file(const std::string& path, const std::string& text) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open for write: " + path);
    out << text;
    if (!out) throw std::runtime_error("write failed: " + path);
}

// ---- subcommands --------------------------------------------------------------------
int cmd_construct(int argc, char** argv, int first) {
    Table t;
    t["n"] = {true, true, "block length (power of two)"};
    t["k"] = {true, true, "information bits"};
    t["design-z"] = {true, false, "design-channel parameter (0.5)"};
    t["out"] = {true, false, "write the frozen-set file here"};
    const Parsed p = parse_options("construct", t, argc, argv, first);
    const PolarCode code = PolarCode::construct(static_cast<int>(to_int("n", p.get("n", ""))),
                                                static_cast<int>(to_int("k", p.get("k", ""))),
                                                to_real("design-z", p.get("design-z", "0.5")));
    const std::string text = format_frozen_set(code);
    if (!p.has("out")) {
        std::cout << text;
    } else {
        const std::string path = p.get("out", "");
        write_file(path, text);
        std::cerr << "wrote " << path << " (n=" << code.n << ", k=" << code.k << ", " << (code.n - code.k)
                  << " frozen)\n";
    }
    return 0;
}

int cmd_encode(int argc, char** argv, int first) {
    Table t;
    add_code_options(t);
    t["info"] = {true, true, "information bits, e.g. 1011"};
    const Parsed p = parse_options("encode", t, argc, argv, first);
    const PolarCode code = code_from(p);
    const Codeword cw = encode(code, bits_from_text(p.get("info", ""), code.k, "--info"));
    std::cout << "u=" << bit_text(cw.u) << "\n" << "x=" << bit_text(cw.x) << "\n";
    return 0;
}

int cmd_decode(int argc, char** argv, int first) {
    Table t;
    add_code_options(t);
    t["llr-file"] = {true, true, "one channel LLR per line"};
    t["decoder"] = {true, false, "baseline|gmatrix|csfg (csfg)"};
    t["alpha"] = {true, false, "min-sum scaling factor (0.9375)"};
    t["max-iter"] = {true, false, "iteration cap (40)"};
    t["trace"] = {false, false, "freeze events to stderr"};
    const Parsed p = parse_options("decode", t, argc, argv, first);
    const PolarCode code = code_from(p);
    const std::vector<double> llrs = llrs_from_file(p.get("llr-file", ""), code.n);
    const DecoderKind kind = parse_decoder(p.get("decoder", "csfg"));
    const double alpha = to_real("alpha", p.get("alpha", "0.9375"));
    const int max_iter = static_cast<int>(to_int("max-iter", p.get("max-iter", "40")));
    DecodeOutcome out;
    if (kind == DecoderKind::baseline) {
        out = decode_baseline(code, llrs, alpha, max_iter);
    } else if (kind == DecoderKind::gmatrix) {
        out = decode_gmatrix(code, llrs, alpha, max_iter);
    } else {
        const bool tr = p.has("trace");
        std::vector<FreezeEvent> events;
        out = decode_csfg(code, llrs, alpha, max_iter, tr ? &events : nullptr);
        for (const FreezeEvent& ev : events) trace_line(ev);
    }
    std::cout << "u_hat=" << bit_text(out.u_hat) << "\n"
              << "info_bits=" << bit_text(out.info_bits) << "\n"
              << "iterations_used=" << out.iterations_used << "\n"
              << "pe_activations=" << out.pe_activations << "\n"
              << "stop_reason=" << to_string(out.stop_reason) << "\n";
    return 0;
}

int cmd_simulate(int argc, char** argv, int first) {
    Table t;
    add_code_options(t);
    t["snr"] = {true, true, "Eb/N0 points: a,b,c or start:stop:step"};
    t["decoders"] = {true, false, "comma list of decoders (baseline,gmatrix,csfg)"};
    t["alpha"] = {true, false, "min-sum scaling factor (0.9375)"};
    t["max-iter"] = {true, false, "iteration cap (40)"};
    t["seed"] = {true, false, "master seed (env POLARBP_SEED, else 1)"};
    t["workers"] = {true, false, "worker threads 1..256 (accepted; the GPU sets the parallelism)"};
    t["min-frame-errors"] = {true, false, "stop a point after this many frame errors per decoder (100)"};
    t["max-frames"] = {true, false, "frame cap per point (100000)"};
    t["out"] = {true, false, "write the results CSV here (default stdout)"};
    t["json"] = {true, false, "also write a JSON report here"};
    t["trace"] = {false, false, "freeze events to stderr"};
    t["noiseless"] = {false, false, "disable channel noise (test hook)"};
    t["fp64"] = {false, false, "decode in double (the reference's arithmetic) instead of fp32"};
    const Parsed p = parse_options("simulate", t, argc, argv, first);
    SimConfig sim;
    sim.code = code_from(p, &sim.code_source);
    sim.snr_db = snr_points(p.get("snr", ""));
    sim.decoders = decoder_list(p.get("decoders", "baseline,gmatrix,csfg"));
    sim.alpha = to_real("alpha", p.get("alpha", "0.9375"));
    sim.max_iter = static_cast<int>(to_int("max-iter", p.get("max-iter", "40")));
    std::string seed = "1";
    if (const char* env = std::getenv("POLARBP_SEED"); env && *env) seed = env;
    sim.seed = static_cast<std::uint64_t>(to_int("seed", p.get("seed", seed)));
    sim.workers = static_cast<int>(to_int("workers", p.get("workers", "1")));
    if (sim.workers < 1 || sim.workers > 256) throw UsageError("--workers: not in [1, 256]");
    sim.min_frame_errors = static_cast<int>(to_int("min-frame-errors", p.get("min-frame-errors", "100")));
    sim.max_frames = to_int("max-frames", p.get("max-frames", "100000"));
    sim.noiseless = p.has("noiseless");
    sim.fp64 = p.has("fp64");
    const TraceSink sink = [](long long, const FreezeEvent& ev) { trace_line(ev); };
    const std::vector<PointStats> rows = run_sweep(sim, p.has("trace") ? &sink : nullptr);
    for (const PointStats& r : rows)
        if (r.low_confidence)
            std::fprintf(stderr, "note: decoder=%s snr_db=%g under-sampled (%lld frame errors in %lld frames)\n",
                         to_string(r.decoder), r.snr_db, static_cast<long long>(r.frame_errors),
                         static_cast<long long>(r.frames));
    const std::string csv = results_csv(rows);
    if (p.has("out"))
        write_file(p.get("out", ""), csv);
    else
        std::cout << csv;
    if (p.has("json")) write_file(p.get("json", ""), results_json(sim, rows));
    return 0;
}

int cmd_report(int argc, char** argv, int first) {
    Table t;
    t["in"] = {true, true, "results CSV produced by simulate"};
    const Parsed p = parse_options("report", t, argc, argv, first);
    const std::string path = p.get("in", "");
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open: " + path);
    std::ostringstream text;
    text << in.rdbuf();
    std::cout << savings_table(compute_savings(parse_results_csv(text.str())));
    return 0;
}

const char* kUsage =
    "usage: polarbp <construct|encode|decode|simulate|report> [options]\n"
    "polar-code BP decoding with sub-graph freezing (GPU); see the file header for options\n";

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2) throw UsageError("a subcommand is required");
        const std::string cmd = argv[1];
        if (cmd == "-h" || cmd == "--help") {
            std::cout << kUsage;
            return 0;
        }
        if (cmd == "construct") return cmd_construct(argc, argv, 2);
        if (cmd == "encode") return cmd_encode(argc, argv, 2);
        if (cmd == "decode") return cmd_decode(argc, argv, 2);
        if (cmd == "simulate") return cmd_simulate(argc, argv, 2);
        if (cmd == "report") return cmd_report(argc, argv, 2);
        throw UsageError("unknown subcommand '" + cmd + "'");
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << "\n" << kUsage;
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
