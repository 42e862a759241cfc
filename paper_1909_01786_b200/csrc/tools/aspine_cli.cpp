// `aspine` command-line drop-in over yasmin-b200 (C++ façade -> C-ABI -> GPU).
// Mirrors /root/reference/proj/tools/aspine.cpp:29-186: same subcommands,
// options, output format and exit codes (10 SAT, 20 UNSAT, 1 error, 2 usage /
// parse error). The `oracle` subcommand is the brute-force reference
// semantics (at most 22 atoms) and runs on the host.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "../../../include/yasmin/aspine.hpp"

namespace {

constexpr int kExitSat = 10, kExitUnsat = 20, kExitError = 1, kExitUsage = 2;

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

aspine::GroundProgram read_program(const std::string& path) {
    if (path == "-") return aspine::parse_program(std::cin);
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    return aspine::parse_program(in);
}

void print_models(const std::vector<aspine::Model>& models) {
    std::size_t n = 0;
    for (const aspine::Model& m : models) {
        std::cout << "Answer: " << ++n << '\n';
        for (std::size_t i = 0; i < m.atoms.size(); ++i) std::cout << (i ? " " : "") << m.atoms[i];
        std::cout << '\n';
    }
}

template <class T>
T number(const std::string& opt, const std::string& v) {
    try {
        std::size_t used = 0;
        const unsigned long long x = std::stoull(v, &used);
        if (used != v.size()) throw std::invalid_argument(v);
        return static_cast<T>(x);
    } catch (const std::exception&) {
        throw Usage(opt + ": not a number: " + v);
    }
}

int run_solve(int argc, char** argv) {
    aspine::SolverConfig cfg;
    std::string file, stats;
    bool trace = false;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw Usage(a + " needs a value");
            return argv[++i];
        };
        if (a == "--mode") {
            const std::string m = val();
            if (m != "fwd" && m != "res") throw Usage("--mode: fwd or res");
            cfg.mode = m == "res" ? aspine::LearnMode::res : aspine::LearnMode::fwd;
        } else if (a == "--heur") {
            const std::string h = val();
            if (h != "occ" && h != "jw" && h != "act") throw Usage("--heur: occ, jw or act");
            cfg.heuristic.kind = h == "jw" ? aspine::HeuristicKind::jeroslow_wang
                                 : h == "act" ? aspine::HeuristicKind::activity
                                              : aspine::HeuristicKind::occurrence_count;
        } else if (a == "--workers") {
            cfg.workers = number<unsigned>(a, val());
            if (cfg.workers < 1 || cfg.workers > 256) throw Usage("--workers: 1..256");
        } else if (a == "--restarts") {
            const std::string r = val();
            if (r != "off") {
                std::istringstream in(r);
                std::string kind, base, factor;
                std::getline(in, kind, ':');
                std::getline(in, base, ':');
                std::getline(in, factor, ':');
                if (kind != "geometric") throw Usage("--restarts: expected off or geometric:BASE:FACTOR");
                cfg.restarts.enabled = true;
                if (!base.empty()) cfg.restarts.base = number<std::uint64_t>(a, base);
                if (!factor.empty()) cfg.restarts.factor = std::stod(factor);
                if (cfg.restarts.base < 1 || cfg.restarts.factor <= 1.0) throw Usage("--restarts: need BASE >= 1 and FACTOR > 1");
            }
        } else if (a == "-n") {
            cfg.max_models = number<std::uint64_t>(a, val());
        } else if (a == "--deps-words") {
            cfg.deps_words = number<std::uint32_t>(a, val());
            if (cfg.deps_words < 1 || cfg.deps_words > 1024) throw Usage("--deps-words: 1..1024");
        } else if (a == "--fanout") {
            cfg.conflict_fanout = number<std::uint32_t>(a, val());
            if (cfg.conflict_fanout < 1 || cfg.conflict_fanout > 64) throw Usage("--fanout: 1..64");
        } else if (a == "--seed") {
            cfg.seed = number<std::uint64_t>(a, val());
        } else if (a == "--verify") {
            cfg.verify = true;
        } else if (a == "--stats") {
            stats = val();
            if (stats != "csv" && stats != "human") throw Usage("--stats: csv or human");
        } else if (a == "--trace") {
            trace = true;
        } else if (a == "--cubes") {  // device extension: ladder width for enumeration
            cfg.cube_atoms = number<std::uint32_t>(a, val());
        } else if (a == "--reference-order") {  // device extension: -n 0 as one search, the reference's model order
            cfg.reference_order = true;
        } else if (a == "--portfolio") {  // device extension: first-model portfolio of N searches
            cfg.portfolio = number<std::uint32_t>(a, val());
        } else if (a == "--devices") {  // device extension: GPUs of this process, e.g. 0,1,2,3
            std::istringstream in(val());
            cfg.devices.clear();
            for (std::string d; std::getline(in, d, ',');) cfg.devices.push_back(number<int>(a, d));
            if (cfg.devices.empty()) throw Usage("--devices: a comma-separated list of CUDA ordinals");
            cfg.device = cfg.devices.front();
        } else if (a.size() > 1 && a[0] == '-' && a != "-") {
            throw Usage("unknown option " + a);
        } else if (file.empty()) {
            file = a;
        } else {
            throw Usage("unexpected argument " + a);
        }
    }
    if (file.empty()) throw Usage("solve: file is required");
    if (trace)
        cfg.trace = [](const aspine::ConflictTrace& t) {
            std::cerr << "trace: mode=" << aspine::to_string(t.mode_used) << " conflict=" << t.conflict_id
                      << " learned_len=" << t.learned_length << " backjump=" << t.backjump_level << '\n';
        };
    aspine::GroundProgram prog = read_program(file);
    aspine::SolveResult res = aspine::solve(prog, cfg);
    print_models(res.models);
    std::cout << (res.status == aspine::SolveStatus::sat ? "SATISFIABLE" : "UNSATISFIABLE") << '\n';
    if (!stats.empty()) {
        aspine::StatsContext ctx{file, aspine::to_string(cfg.mode), aspine::to_string(cfg.heuristic.kind), cfg.workers,
                                 res.status, res.stats.models};
        if (stats == "csv")
            std::cout << aspine::stats_csv_header() << '\n'
                      << aspine::emit_stats(res.stats, ctx, aspine::StatsFormat::csv) << '\n';
        else
            std::cout << aspine::emit_stats(res.stats, ctx, aspine::StatsFormat::human) << '\n';
    }
    return res.status == aspine::SolveStatus::sat ? kExitSat : kExitUnsat;
}

// Brute-force answer sets (oracle.cpp:91-143 semantics), at most 22 atoms.
int run_oracle(int argc, char** argv) {
    if (argc != 3) throw Usage("oracle: exactly one file");
    aspine::GroundProgram prog = read_program(argv[2]);
    const std::uint32_t n = prog.atom_count();
    if (n > 22) throw std::invalid_argument("enumerate_answer_sets: more than 22 atoms");
    std::vector<std::uint32_t> ids;
    std::vector<std::pair<std::vector<std::uint32_t>, std::vector<std::string>>> order;
    for (std::uint64_t cand = 0; cand < (1ull << n); ++cand) {
        ids.clear();
        for (std::uint32_t a = 1; a <= n; ++a)
            if (cand & (1ull << (a - 1))) ids.push_back(a);
        if (!yas_verify_model(prog.handle(), ids.data(), ids.size())) continue;
        std::vector<std::string> names;
        for (std::uint32_t a : ids) names.push_back(prog.name(a));
        std::sort(names.begin(), names.end());
        order.emplace_back(ids, std::move(names));
    }
    std::size_t k = 0;
    // the reference prints the family sorted by atom-id vectors (oracle.cpp:141)
    std::sort(order.begin(), order.end());
    for (const auto& [v, names] : order) {
        std::cout << "Answer: " << ++k << '\n';
        for (std::size_t i = 0; i < names.size(); ++i) std::cout << (i ? " " : "") << names[i];
        std::cout << '\n';
    }
    std::cout << (order.empty() ? "UNSATISFIABLE" : "SATISFIABLE") << '\n';
    return order.empty() ? kExitUnsat : kExitSat;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2) throw Usage("usage: aspine solve|oracle <file> [options]");
        const std::string cmd = argv[1];
        if (cmd == "solve") return run_solve(argc, argv);
        if (cmd == "oracle") return run_oracle(argc, argv);
        if (cmd == "-h" || cmd == "--help") {
            std::cout << "aspine (yasmin-b200) - conflict-driven answer set solver on the GPU\n"
                         "  aspine solve <file|-> [--mode fwd|res] [--heur occ|jw|act] [--workers N]\n"
                         "        [--restarts off|geometric:B:F] [-n N] [--deps-words W] [--fanout K]\n"
                         "        [--seed S] [--verify] [--stats csv|human] [--trace] [--cubes K] [--portfolio N]\n"
                         "        [--devices D0,D1,...] [--reference-order]\n"
                         "  aspine oracle <file|->\n";
            return 0;
        }
        throw Usage("unknown subcommand " + cmd);
    } catch (const Usage& e) {
        std::cerr << e.what() << '\n';
        return kExitUsage;
    } catch (const aspine::ParseError& e) {
        std::cerr << "parse error: " << e.what() << '\n';
        return kExitUsage;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitError;
    }
}
