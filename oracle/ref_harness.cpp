// ORACLE HARNESS — test infrastructure only, never part of the product.
//
// Drives the UNMODIFIED reference solver (/root/reference/proj, compiled by
// oracle/Makefile into oracle/_ref/) through its own public API and prints JSON.
// Used to (a) generate the committed golden fixtures under tests/golden/ and
// (b) time the reference CPU path for bench.py --impl reference / cpu_baseline.
//
//   aspine_ref solve FILE|- [--mode fwd|res] [--heur occ|jw|act] [--decay D] [-n N]
//                           [--restarts B:F] [--fanout K] [--deps-words W] [--cap C]
//                           [--verify] [--trace] [--reps R] [--no-models]
//        -> parse_program + solve (P/src/solver.cpp:307), JSON models + SolveStats
//   aspine_ref dump FILE|-  -> compile_completion + NogoodStore::build goldens
//   aspine_ref corpus       -> the acceptance corpus (P/tests/acceptance/acceptance_main.cpp:51-65)
//                              as program text + brute-force oracle families
//   aspine_ref propstores SEED COUNT ATOMS MAXLEN
//        -> random stores (P/tests/support/gen.hpp:73-87) + reference Propagator fixpoint
//   aspine_ref cubes FILE CUBES PART NPARTS
//        -> enumerate all answer sets of FILE + cube c (for c % NPARTS == PART), one
//           reference solve per cube; CUBES has one cube per line, each a list of atom
//           names n standing for the integrity constraint ":- n." (the cube split of
//           SURVEY.md 8(e), run on CPU processes for the config-5 baseline)
//   aspine_ref planted ATOMS NOGOODS PCT SEED [REPS]
//        -> the planted 1M-nogood store of SURVEY.md App. C, reference propagate_and_check
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "aspine/completion.hpp"
#include "aspine/nogood_store.hpp"
#include "aspine/oracle.hpp"
#include "aspine/program.hpp"
#include "aspine/propagate.hpp"
#include "aspine/solver.hpp"
#include "support/corpus.hpp"
#include "support/gen.hpp"

using namespace aspine;

namespace {

std::string jstr(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') { o += '\\'; o += c; }
        else if (c == '\n') o += "\\n";
        else if (static_cast<unsigned char>(c) < 0x20) { char b[8]; std::snprintf(b, 8, "\\u%04x", c); o += b; }
        else o += c;
    }
    return o + "\"";
}

template <class T>
std::string jarr(const std::vector<T>& v) {
    std::ostringstream o;
    o << '[';
    for (std::size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << v[i];
    o << ']';
    return o.str();
}

GroundProgram read_program(const std::string& path) {
    if (path == "-") return parse_program(std::cin);
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    return parse_program(in);
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch()).count();
}

std::string stats_json(const SolveStats& s) {
    std::ostringstream o;
    o << "{\"decisions\":" << s.decisions << ",\"propagations\":" << s.propagations
      << ",\"conflicts\":" << s.conflicts << ",\"learned_count\":" << s.learned_count
      << ",\"learned_length_sum\":" << s.learned_length_sum << ",\"restarts\":" << s.restarts
      << ",\"models\":" << s.models << ",\"passes\":" << s.passes
      << ",\"watch_replacements\":" << s.watch_replacements
      << ",\"duplicate_learned\":" << s.duplicate_learned
      << ",\"blocking_nogoods\":" << s.blocking_nogoods << ",\"res_learned\":" << s.res_learned
      << ",\"fwd_learned\":" << s.fwd_learned << ",\"fwd_fallbacks\":" << s.fwd_fallbacks
      << ",\"uip_check_failures\":" << s.uip_check_failures
      << ",\"fwd_decision_only_failures\":" << s.fwd_decision_only_failures
      << ",\"asserting_failures\":" << s.asserting_failures << ",\"wall_ms\":" << s.wall_ms << "}";
    return o.str();
}

struct Opts {
    SolverConfig cfg;
    bool trace = false;
    bool models = true;
    int reps = 1;
};

Opts parse_opts(int argc, char** argv, int i) {
    Opts o;
    for (; i < argc; ++i) {
        std::string a = argv[i];
        auto next = [&]() -> std::string {
            if (i + 1 >= argc) throw std::runtime_error("missing value for " + a);
            return argv[++i];
        };
        if (a == "--mode") o.cfg.mode = next() == "res" ? LearnMode::res : LearnMode::fwd;
        else if (a == "--heur") {
            std::string h = next();
            o.cfg.heuristic.kind = h == "jw"    ? HeuristicKind::jeroslow_wang
                                   : h == "act" ? HeuristicKind::activity
                                                : HeuristicKind::occurrence_count;
        } else if (a == "--decay") o.cfg.heuristic.activity_decay = std::stod(next());
        else if (a == "-n") o.cfg.max_models = std::stoull(next());
        else if (a == "--restarts") {
            std::string s = next();
            auto c = s.find(':');
            o.cfg.restarts.enabled = true;
            o.cfg.restarts.base = std::stoull(s.substr(0, c));
            o.cfg.restarts.factor = std::stod(s.substr(c + 1));
        } else if (a == "--fanout") o.cfg.conflict_fanout = static_cast<std::uint32_t>(std::stoul(next()));
        else if (a == "--deps-words") o.cfg.deps_words = static_cast<std::uint32_t>(std::stoul(next()));
        else if (a == "--cap") o.cfg.learned_capacity = std::stoull(next());
        else if (a == "--workers") o.cfg.workers = static_cast<unsigned>(std::stoul(next()));
        else if (a == "--verify") o.cfg.verify = true;
        else if (a == "--trace") o.trace = true;
        else if (a == "--no-models") o.models = false;
        else if (a == "--reps") o.reps = std::stoi(next());
        else throw std::runtime_error("unknown option " + a);
    }
    return o;
}

int cmd_solve(const std::string& file, Opts o) {
    const double t0 = now_ms();
    GroundProgram prog = read_program(file);
    const double t1 = now_ms();
    std::vector<std::string> traces;
    if (o.trace)
        o.cfg.trace = [&](const ConflictTrace& t) {
            std::ostringstream s;
            s << '[' << (t.mode_used == LearnMode::fwd ? 0 : 1) << ',' << t.conflict_id << ','
              << t.learned_length << ',' << t.backjump_level << ']';
            traces.push_back(s.str());
        };
    SolveResult res;
    std::string error;
    std::vector<double> total_ms, run_ms;
    for (int r = 0; r < o.reps; ++r) {
        traces.clear();
        const double s0 = now_ms();
        try {
            res = solve(prog, o.cfg);
        } catch (const StoreCapacityError& e) {
            error = std::string("StoreCapacityError: ") + e.what();
        } catch (const VerificationError& e) {
            error = std::string("VerificationError: ") + e.what();
        } catch (const std::exception& e) {
            error = std::string("error: ") + e.what();
        }
        total_ms.push_back(now_ms() - s0);
        run_ms.push_back(res.stats.wall_ms);
    }
    std::ostringstream out;
    out << "{\"status\":" << jstr(res.status == SolveStatus::sat ? "SAT" : "UNSAT")
        << ",\"error\":" << jstr(error) << ",\"atoms\":" << prog.atom_count()
        << ",\"parse_ms\":" << (t1 - t0) << ",\"solve_ms\":" << jarr(total_ms)
        << ",\"run_ms\":" << jarr(run_ms) << ",\"stats\":" << stats_json(res.stats);
    if (o.models) {
        out << ",\"models\":[";
        for (std::size_t m = 0; m < res.models.size(); ++m) {
            out << (m ? "," : "") << jarr(res.models[m].atom_ids);
        }
        out << "],\"first_model_names\":[";
        if (!res.models.empty())
            for (std::size_t k = 0; k < res.models[0].atoms.size(); ++k)
                out << (k ? "," : "") << jstr(res.models[0].atoms[k]);
        out << "]";
    }
    if (o.trace) {
        out << ",\"trace\":[";
        for (std::size_t k = 0; k < traces.size(); ++k) out << (k ? "," : "") << traces[k];
        out << "]";
    }
    out << "}\n";
    std::cout << out.str();
    return 0;
}

int cmd_dump(const std::string& file) {
    GroundProgram prog = read_program(file);
    Completion comp = compile_completion(prog);
    const std::string dump = dump_nogoods(comp, prog);
    std::vector<std::string> aux;
    for (std::size_t r = 0; r < comp.aux.rule_count(); ++r) {
        const auto& ra = comp.aux.of_rule(static_cast<std::uint32_t>(r));
        std::ostringstream s;
        s << '[' << ra.b << ',' << ra.t << ',' << ra.n << ',' << (ra.vacuous ? 1 : 0) << ']';
        aux.push_back(s.str());
    }
    NogoodCensus census = nogood_census(prog);
    const AtomId total = comp.aux.total_atoms();
    std::vector<std::uint32_t> guards;
    for (const Nogood& n : comp.nogoods) guards.push_back(n.truth_guard());
    StoreBuild sb = NogoodStore::build(std::move(comp.nogoods), total);
    std::vector<std::int32_t> units;
    for (Lit l : sb.units) units.push_back(l.code());
    std::vector<std::int32_t> unit_ids(sb.store.unit_ids().begin(), sb.store.unit_ids().end());
    std::vector<std::uint32_t> store_guards;
    for (std::size_t id = 0; id < sb.store.size(); ++id)
        store_guards.push_back(sb.store.truth_guard(static_cast<NogoodId>(id)));
    auto b = sb.store.static_class_bounds();
    std::cout << "{\"atoms\":" << prog.atom_count() << ",\"total_atoms\":" << total
              << ",\"first_aux\":" << comp.aux.first_aux() << ",\"rules\":" << prog.rules().size()
              << ",\"constraints\":" << prog.constraints().size() << ",\"aux\":" << jarr(aux)
              << ",\"census\":[" << census.rule_nogoods << ',' << census.atom_nogoods << ','
              << census.constraint_nogoods << "],\"counts\":[" << comp.counts.rule_nogoods << ','
              << comp.counts.atom_nogoods << ',' << comp.counts.constraint_nogoods
              << "],\"dump\":" << jstr(dump) << ",\"guards\":" << jarr(guards)
              << ",\"csv\":" << jstr(sb.store.dump_csv()) << ",\"units\":" << jarr(units)
              << ",\"unit_ids\":" << jarr(unit_ids) << ",\"store_guards\":" << jarr(store_guards)
              << ",\"bounds\":[" << b[0] << ',' << b[1] << ',' << b[2] << ',' << b[3]
              << "],\"printed\":" << jstr(print_program(prog)) << "}\n";
    return 0;
}

int cmd_corpus() {
    std::cout << "[";
    bool first = true;
    auto emit = [&](const std::string& name, const GroundProgram& generated) {
        // ids of the emitted text (the re-parse relabels atoms in first-occurrence order)
        const GroundProgram prog = parse_program(print_program(generated));
        auto fam = enumerate_answer_sets(prog);
        std::ostringstream f;
        f << '[';
        for (std::size_t i = 0; i < fam.size(); ++i) f << (i ? "," : "") << jarr(fam[i]);
        f << ']';
        std::cout << (first ? "\n" : ",\n") << "{\"name\":" << jstr(name)
                  << ",\"text\":" << jstr(print_program(prog)) << ",\"atoms\":" << prog.atom_count()
                  << ",\"family\":" << f.str() << "}";
        first = false;
    };
    // Acceptance corpus: P/tests/acceptance/acceptance_main.cpp:51-65.
    for (auto& [name, text] : testing::handcrafted_programs()) emit(name, parse_program(text));
    testing::SplitMix64 rng(0xac0e97ed);
    for (int i = 0; i < 500; ++i) {
        testing::ProgramShape shape;
        emit("random_" + std::to_string(i), testing::random_program(rng, shape));
    }
    std::cout << "\n]\n";
    return 0;
}

std::string cells_json(const Assignment& a) {
    std::vector<std::int32_t> c;
    for (AtomId x = 0; x <= a.atom_count(); ++x) c.push_back(a.cell(x));
    return jarr(c);
}

std::string trail_json(const Assignment& a) {
    std::vector<std::int32_t> t;
    for (const auto& e : a.trail()) t.push_back(e.lit.code());
    return jarr(t);
}

std::string reasons_json(const Assignment& a) {
    std::vector<std::int32_t> r;
    for (AtomId x = 0; x <= a.atom_count(); ++x) {
        const Reason rs = a.reason(x);
        r.push_back(rs.kind == Reason::propagated ? rs.antecedent : -static_cast<int>(rs.kind) - 1);
    }
    return jarr(r);
}

std::string deps_json(const Assignment& a) {
    std::vector<std::uint64_t> d;
    for (AtomId x = 0; x <= a.atom_count(); ++x) {
        auto w = a.deps().of(x);
        d.push_back(w[0] | (a.deps().overflow(x) ? (1ull << 63) : 0));
    }
    return jarr(d);
}

// Random stores as in P/tests/test_propagate.cpp:190-235 and acceptance criterion 5
// (P/tests/acceptance/acceptance_main.cpp:225-258): initial propagation, a pass at
// level 1, then one decision on the lowest unassigned atom and propagation at level 2.
int cmd_propstores(std::uint64_t seed, int count, unsigned atoms, unsigned max_len) {
    testing::SplitMix64 rng(seed);
    std::cout << "[";
    for (int it = 0; it < count; ++it) {
        auto nogoods = testing::random_nogoods(rng, 1 + static_cast<unsigned>(rng.below(20)), atoms, max_len);
        std::vector<std::string> lits;
        for (const Nogood& n : nogoods) {
            std::vector<std::int32_t> c;
            for (Lit l : n) c.push_back(l.code());
            lits.push_back(jarr(c));
        }
        StoreBuild b = NogoodStore::build(nogoods, atoms);
        WorkerPool pool(1);
        Propagator prop(b.store, pool);
        Assignment a(atoms, 1);
        Frontier f;
        PropagationOutcome init = prop.initial_propagation(a, f);
        std::ostringstream o;
        o << "{\"nogoods\":" << jarr(lits) << ",\"init_violated\":" << init.violated
          << ",\"init_conflicts\":" << jarr(init.conflicts)
          << ",\"init_props\":" << init.propagations;
        std::int32_t decision = 0;
        if (!init.violated) {
            PropagationOutcome l1 = prop.propagate_and_check(a, f, 1);
            o << ",\"l1_violated\":" << l1.violated << ",\"l1_conflicts\":" << jarr(l1.conflicts)
              << ",\"l1_props\":" << l1.propagations << ",\"l1_passes\":" << l1.passes;
            if (!l1.violated) {
                o << ",\"l1_cells\":" << cells_json(a) << ",\"l1_trail\":" << trail_json(a);
                for (AtomId x = 1; x <= atoms; ++x)
                    if (a.unassigned(x)) {
                        a.push_decision(Lit::pos(x));
                        decision = static_cast<std::int32_t>(x);
                        f.clear();
                        f.seed(Lit::pos(x));
                        PropagationOutcome l2 = prop.propagate_and_check(a, f, 2);
                        o << ",\"l2_violated\":" << l2.violated
                          << ",\"l2_conflicts\":" << jarr(l2.conflicts)
                          << ",\"l2_props\":" << l2.propagations << ",\"l2_passes\":" << l2.passes;
                        break;
                    }
            }
        }
        o << ",\"decision\":" << decision << ",\"cells\":" << cells_json(a)
          << ",\"trail\":" << trail_json(a) << ",\"reasons\":" << reasons_json(a)
          << ",\"deps\":" << deps_json(a) << "}";
        std::cout << (it ? ",\n" : "\n") << o.str();
    }
    std::cout << "\n]\n";
    return 0;
}

// Planted store, SURVEY.md Appendix C (config 4b).
int cmd_planted(unsigned atoms, std::size_t count, unsigned pct, std::uint64_t seed, int reps) {
    testing::SplitMix64 rng(seed);
    std::vector<std::uint8_t> h(atoms + 1, 0);
    for (AtomId a = 1; a <= atoms; ++a) h[a] = rng.chance(50) ? 1 : 0;
    auto hlit = [&](AtomId a) { return h[a] ? Lit::pos(a) : Lit::neg(a); };
    std::vector<Nogood> nogoods;
    nogoods.reserve(count);
    while (nogoods.size() < count) {
        const unsigned len = 2 + static_cast<unsigned>(rng.below(5));
        std::vector<Lit> lits;
        for (unsigned k = 0; k < len; ++k) {
            const AtomId a = static_cast<AtomId>(1 + rng.below(atoms));
            lits.push_back(rng.chance(50) ? Lit::pos(a) : Lit::neg(a));
        }
        lits[0] = ~hlit(lits[0].atom());
        if (auto n = Nogood::make(std::move(lits), NogoodOrigin::constraint)) nogoods.push_back(std::move(*n));
    }
    std::vector<Lit> seeded;
    for (AtomId a = 2; a <= atoms; ++a)
        if (rng.below(100) < pct) seeded.push_back(hlit(a));
    const double b0 = now_ms();
    StoreBuild b = NogoodStore::build(nogoods, atoms);
    const double b1 = now_ms();
    std::vector<double> times;
    PropagationOutcome out;
    std::uint64_t digest = 0, rdigest = 0, ddigest = 0;
    std::size_t trail = 0;
    for (int r = 0; r < reps; ++r) {
        WorkerPool pool(1);
        Propagator prop(b.store, pool);
        Assignment a(atoms, 16);
        Frontier f;
        a.push_decision(hlit(1));
        f.seed(hlit(1));
        const std::vector<std::uint64_t> zero(16, 0);
        for (Lit l : seeded) {
            a.assign_propagated(l, 2, zero, false, 0);
            f.last.push_back(l);
        }
        const double t0 = now_ms();
        out = prop.propagate_and_check(a, f, 2);
        times.push_back(now_ms() - t0);
        digest = 0xcbf29ce484222325ull;
        rdigest = ddigest = 0xcbf29ce484222325ull;
        for (const auto& e : a.trail()) {
            digest = (digest ^ static_cast<std::uint32_t>(e.lit.code())) * 0x100000001b3ull;
            // antecedents (-1 for decision / seeded-without-reason) and Deps word 0 + overflow, trail order
            const AtomId x = e.lit.atom();
            const Reason rs = a.reason(x);
            const std::int32_t rv = rs.kind == Reason::propagated ? rs.antecedent : -1;
            rdigest = (rdigest ^ static_cast<std::uint32_t>(rv)) * 0x100000001b3ull;
            const std::uint64_t d0 = a.deps().of(x)[0];
            ddigest = (ddigest ^ static_cast<std::uint32_t>(d0)) * 0x100000001b3ull;
            ddigest = (ddigest ^ static_cast<std::uint32_t>(d0 >> 32)) * 0x100000001b3ull;
            ddigest = (ddigest ^ (a.deps().overflow(x) ? 1u : 0u)) * 0x100000001b3ull;
        }
        trail = a.trail().size();
    }
    std::cout << "{\"atoms\":" << atoms << ",\"nogoods\":" << nogoods.size() << ",\"pct\":" << pct
              << ",\"seeded\":" << seeded.size() << ",\"build_ms\":" << (b1 - b0)
              << ",\"violated\":" << out.violated << ",\"conflicts\":" << out.conflicts.size()
              << ",\"propagations\":" << out.propagations << ",\"passes\":" << out.passes
              << ",\"trail\":" << trail << ",\"trail_digest\":" << digest
              << ",\"reason_digest\":" << rdigest << ",\"deps_digest\":" << ddigest
              << ",\"prop_ms\":" << jarr(times) << "}\n";
    return 0;
}

// Config 5 on CPU processes: the same cube set the device enumerates, one
// reference solve (-n 0) of program + cube constraints per cube.
int cmd_cubes(const std::string& file, const std::string& cube_file, unsigned part, unsigned nparts) {
    std::ifstream in(file);
    if (!in) throw std::runtime_error("cannot open " + file);
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    std::ifstream cf(cube_file);
    if (!cf) throw std::runtime_error("cannot open " + cube_file);
    SolverConfig cfg;
    cfg.max_models = 0;
    const double t0 = now_ms();
    std::string line;
    std::size_t index = 0, solved = 0;
    std::ostringstream models;
    std::size_t count = 0;
    while (std::getline(cf, line)) {
        if (index++ % nparts != part) continue;
        std::string cube_text = text;
        std::istringstream names(line);
        for (std::string n; names >> n;) cube_text += "\n:- " + n + ".";
        const GroundProgram prog = parse_program(std::string_view(cube_text));
        const SolveResult r = solve(prog, cfg);
        for (const Model& m : r.models) models << (count++ ? "," : "") << jarr(m.atom_ids);
        ++solved;
    }
    std::cout << "{\"cubes\":" << solved << ",\"ms\":" << (now_ms() - t0) << ",\"models\":[" << models.str()
              << "]}\n";
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2) throw std::runtime_error("usage: aspine_ref solve|dump|corpus|propstores|planted ...");
        std::string cmd = argv[1];
        if (cmd == "solve" && argc >= 3) return cmd_solve(argv[2], parse_opts(argc, argv, 3));
        if (cmd == "dump" && argc >= 3) return cmd_dump(argv[2]);
        if (cmd == "corpus") return cmd_corpus();
        if (cmd == "propstores" && argc >= 6)
            return cmd_propstores(std::stoull(argv[2], nullptr, 0), std::stoi(argv[3]),
                                  static_cast<unsigned>(std::stoul(argv[4])),
                                  static_cast<unsigned>(std::stoul(argv[5])));
        if (cmd == "cubes" && argc >= 6)
            return cmd_cubes(argv[2], argv[3], static_cast<unsigned>(std::stoul(argv[4])),
                             static_cast<unsigned>(std::stoul(argv[5])));
        if (cmd == "planted" && argc >= 6)
            return cmd_planted(static_cast<unsigned>(std::stoul(argv[2])), std::stoull(argv[3]),
                               static_cast<unsigned>(std::stoul(argv[4])),
                               std::stoull(argv[5], nullptr, 0), argc >= 7 ? std::stoi(argv[6]) : 1);
        throw std::runtime_error("bad command line");
    } catch (const ParseError& e) {
        std::cout << "{\"parse_error\":" << jstr(e.what()) << ",\"line\":" << e.line << "}\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
