// C++ drop-in façade for callers of the reference solver's public API
// (/root/reference/proj/include/aspine/*.hpp), implemented over the
// yasmin-b200 C-ABI (include/yasmin_b200.h). Same names, argument meaning
// and error behaviour as the reference:
//   GroundProgram / Rule / Atom / intern / add_rule / rules / rules_of   program.hpp:33-77
//   parse_program(std::istream&) / (std::string_view)                   program.hpp:87-88
//   print_program / tp_step / validate                                  program.hpp:91-100
//   solve(const GroundProgram&, const SolverConfig&)                    solver.hpp:113
//   verify_model / emit_stats / stats_csv_header / to_string            solver.hpp:116-137
//   is_answer_set / enumerate_answer_sets                               oracle.hpp:49-55
//   ParseError{line}, StoreCapacityError, VerificationError, std::logic_error
// plus the low-level store / assignment / propagator API (yasmin/lowlevel.hpp).
// The reference's own include paths (aspine/program.hpp, aspine/solver.hpp, ...)
// forward here (include/aspine/). Header-only; link with -lyasmin_b200.
#pragma once

#include <functional>
#include <istream>
#include <iterator>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "../yasmin_b200.h"
#include "lowlevel.hpp"

namespace aspine {

struct ParseError : std::runtime_error {
    ParseError(int l, const std::string& what) : std::runtime_error(what), line(l) {}
    int line;
};
struct VerificationError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace detail {
[[noreturn]] inline void raise(int rc, const char* msg, int line = 0) {
    switch (rc) {
        case YAS_ERR_PARSE: throw ParseError(line, msg);
        case YAS_ERR_CAPACITY: throw StoreCapacityError(msg);
        case YAS_ERR_VERIFY: throw VerificationError(msg);
        case YAS_ERR_LOGIC: throw std::logic_error(msg);
        case YAS_ERR_ARG: throw std::invalid_argument(msg);
        default: throw std::runtime_error(msg);
    }
}
}  // namespace detail

// ---- the program model ---------------------------------------------------------

struct Atom {
    AtomId id = 0;
    std::string name;
};

/// head :- pos_body, not neg_body (head 0: a constraint); bodies sorted, no repeats.
struct Rule {
    AtomId head = 0;
    std::vector<AtomId> pos_body;
    std::vector<AtomId> neg_body;
    bool is_constraint() const { return head == 0; }
    bool is_fact() const { return head != 0 && pos_body.empty() && neg_body.empty(); }
    bool body_overlaps() const {
        for (AtomId a : pos_body)
            if (std::binary_search(neg_body.begin(), neg_body.end(), a)) return true;
        return false;
    }
};

/// The library owns the program (that is what solve() compiles); this class
/// mirrors its atoms and rules for reading. Copies share the library's
/// program until one of them is edited, so copies behave as values.
class GroundProgram {
public:
    GroundProgram() : p_(yas_program_create(), &yas_program_free) {
        if (!p_) throw std::bad_alloc();
        atoms_.push_back({0, ""});
        rules_of_.emplace_back();
    }
    explicit GroundProgram(yas_program* p) : p_(p, &yas_program_free) { mirror(); }

    AtomId intern(std::string_view name) {
        own();
        const AtomId id = yas_program_intern(p_.get(), std::string(name).c_str());
        if (id == 0) throw std::invalid_argument("intern failed");
        if (id > atom_count()) {
            atoms_.push_back({id, std::string(name)});
            rules_of_.emplace_back();
        }
        return id;
    }
    AtomId find(std::string_view name) const { return yas_program_find(p_.get(), std::string(name).c_str()); }
    void add_rule(Rule r) {
        own();
        for (auto* body : {&r.pos_body, &r.neg_body}) {
            std::sort(body->begin(), body->end());
            body->erase(std::unique(body->begin(), body->end()), body->end());
        }
        const int rc = yas_program_add_rule(p_.get(), r.head, r.pos_body.data(), r.pos_body.size(), r.neg_body.data(),
                                            r.neg_body.size());
        if (rc != YAS_OK) throw std::out_of_range("add_rule: atom id not interned");
        if (r.is_constraint()) {
            constraints_.push_back(std::move(r));
        } else {
            rules_of_.at(r.head).push_back(static_cast<std::uint32_t>(rules_.size()));
            rules_.push_back(std::move(r));
        }
    }

    AtomId atom_count() const { return static_cast<AtomId>(atoms_.size() - 1); }
    const Atom& atom(AtomId id) const { return atoms_.at(id); }
    const std::string& name(AtomId id) const { return atoms_.at(id).name; }
    const std::vector<Rule>& rules() const { return rules_; }
    const std::vector<Rule>& constraints() const { return constraints_; }
    const std::vector<std::uint32_t>& rules_of(AtomId p) const { return rules_of_.at(p); }
    const yas_program* handle() const { return p_.get(); }

private:
    void mirror() {
        const AtomId n = yas_program_atom_count(p_.get());
        atoms_.assign(1, Atom{0, ""});
        for (AtomId a = 1; a <= n; ++a) atoms_.push_back({a, yas_program_atom_name(p_.get(), a)});
        rules_of_.assign(static_cast<std::size_t>(n) + 1, {});
        rules_.clear();
        constraints_.clear();
        const std::uint32_t nr = yas_program_rule_count(p_.get()), nc = yas_program_constraint_count(p_.get());
        for (std::uint32_t r = 0; r < nr + nc; ++r) {
            Rule x;
            const std::uint32_t *pos = nullptr, *neg = nullptr;
            std::uint32_t np = 0, nn = 0;
            yas_program_rule(p_.get(), r, &x.head, &pos, &np, &neg, &nn);
            x.pos_body.assign(pos, pos + np);
            x.neg_body.assign(neg, neg + nn);
            if (r < nr) {
                rules_of_[x.head].push_back(r);
                rules_.push_back(std::move(x));
            } else {
                constraints_.push_back(std::move(x));
            }
        }
    }
    // copy on write: an edit never shows through another copy
    void own() {
        if (p_.use_count() == 1) return;
        std::shared_ptr<yas_program> q(yas_program_create(), &yas_program_free);
        for (AtomId a = 1; a <= atom_count(); ++a) yas_program_intern(q.get(), atoms_[a].name.c_str());
        for (const auto* list : {&rules_, &constraints_})
            for (const Rule& r : *list)
                yas_program_add_rule(q.get(), r.head, r.pos_body.data(), r.pos_body.size(), r.neg_body.data(),
                                     r.neg_body.size());
        p_ = std::move(q);
    }

    std::shared_ptr<yas_program> p_;
    std::vector<Atom> atoms_;
    std::vector<Rule> rules_;
    std::vector<Rule> constraints_;
    std::vector<std::vector<std::uint32_t>> rules_of_;
};

inline GroundProgram parse_program(std::string_view text) {
    yas_program* p = nullptr;
    int line = 0;
    char err[512];
    const int rc = yas_program_parse(text.data(), text.size(), &p, &line, err, sizeof err);
    if (rc != YAS_OK) detail::raise(rc, err, line);
    return GroundProgram(p);
}

inline GroundProgram parse_program(std::istream& in) {
    std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    return parse_program(std::string_view(text));
}

namespace detail {
template <class F>
std::string text_of(F&& call) {
    std::string s(call(nullptr, 0), '\0');
    call(s.data(), s.size() + 1);
    return s;
}
}  // namespace detail

inline std::string print_program(const GroundProgram& prog) {
    return detail::text_of([&](char* b, std::size_t c) { return yas_program_print(prog.handle(), b, c); });
}

/// Heads of the rules whose positive body lies in `interp` (sorted ids) and
/// whose negative body misses it; an id above atom_count() throws like vector::at.
inline std::vector<AtomId> tp_step(const GroundProgram& prog, std::span<const AtomId> interp) {
    std::vector<AtomId> out(prog.rules().size());
    const std::size_t n = yas_program_tp_step(prog.handle(), interp.data(), interp.size(), out.data(), out.size());
    if (n == SIZE_MAX) throw std::out_of_range("tp_step: atom id out of range");
    out.resize(n);
    return out;
}

inline std::vector<std::string> validate(const GroundProgram& prog) {
    const std::string all =
        detail::text_of([&](char* b, std::size_t c) { return yas_program_diagnostics(prog.handle(), b, c); });
    std::vector<std::string> out;
    std::size_t at = 0;
    while (at < all.size()) {
        const std::size_t nl = all.find('\n', at);
        out.push_back(all.substr(at, nl - at));
        at = nl == std::string::npos ? all.size() : nl + 1;
    }
    return out;
}

// ---- the brute-force oracle (oracle.hpp): definitional checks ------------------

/// Gelfond-Lifschitz reduct relative to m (sorted): rules and constraints whose
/// negative body meets m are dropped, the others lose their negative body.
struct ReductProgram {
    std::vector<Rule> rules;
    std::vector<Rule> constraints;
};

inline ReductProgram reduct(const GroundProgram& prog, std::span<const AtomId> m) {
    auto blocked = [&](const Rule& r) {
        return std::any_of(r.neg_body.begin(), r.neg_body.end(),
                           [&](AtomId a) { return std::binary_search(m.begin(), m.end(), a); });
    };
    ReductProgram out;
    for (const auto* src : {&prog.rules(), &prog.constraints()})
        for (const Rule& r : *src) {
            if (blocked(r)) continue;
            Rule k{r.head, r.pos_body, {}};
            (src == &prog.rules() ? out.rules : out.constraints).push_back(std::move(k));
        }
    return out;
}

/// Least model of a negation-free program by iterating its consequences from
/// the empty set; nullopt when a constraint body ends up true.
inline std::optional<std::vector<AtomId>> least_model(const ReductProgram& red) {
    std::vector<AtomId> in;  // sorted
    auto all_in = [&](const std::vector<AtomId>& body) {
        return std::all_of(body.begin(), body.end(), [&](AtomId a) { return std::binary_search(in.begin(), in.end(), a); });
    };
    for (bool grew = true; grew;) {
        grew = false;
        for (const Rule& r : red.rules)
            if (!std::binary_search(in.begin(), in.end(), r.head) && all_in(r.pos_body)) {
                in.insert(std::upper_bound(in.begin(), in.end(), r.head), r.head);
                grew = true;
            }
    }
    for (const Rule& c : red.constraints)
        if (all_in(c.pos_body)) return std::nullopt;
    return in;
}

inline bool is_answer_set(const GroundProgram& prog, std::span<const AtomId> m) {
    const int r = yas_verify_model(prog.handle(), m.data(), m.size());
    if (r < 0) throw std::out_of_range("is_answer_set: atom id out of range");
    return r == 1;
}

/// Every answer set of a program of at most 22 atoms, by testing all subsets;
/// each sorted, the family in lexicographic order.
inline std::vector<std::vector<AtomId>> enumerate_answer_sets(const GroundProgram& prog) {
    const AtomId n = prog.atom_count();
    if (n > 22) throw std::invalid_argument("enumerate_answer_sets: more than 22 atoms");
    std::vector<std::vector<AtomId>> fam;
    std::vector<AtomId> m;
    for (std::uint64_t mask = 0; mask < (1ull << n); ++mask) {
        m.clear();
        for (AtomId a = 1; a <= n; ++a)
            if ((mask >> (a - 1)) & 1ull) m.push_back(a);
        if (is_answer_set(prog, m)) fam.push_back(m);
    }
    std::sort(fam.begin(), fam.end());
    return fam;
}

enum class LearnMode : std::uint8_t { fwd, res };
enum class HeuristicKind : std::uint8_t { occurrence_count, jeroslow_wang, activity };
enum class SolveStatus : std::uint8_t { sat, unsat };

struct HeuristicConfig {
    HeuristicKind kind = HeuristicKind::occurrence_count;
    double activity_decay = 0.95;
};
struct RestartPolicy {
    bool enabled = false;
    std::uint64_t base = 100;
    double factor = 1.5;
};
struct ConflictTrace {
    LearnMode mode_used;
    std::int32_t conflict_id;
    std::size_t learned_length;
    std::uint32_t backjump_level;
};

struct SolverConfig {
    LearnMode mode = LearnMode::fwd;
    HeuristicConfig heuristic{};
    unsigned workers = 1;
    RestartPolicy restarts{};
    std::uint64_t max_models = 1;
    std::uint32_t deps_words = 16;
    std::uint32_t conflict_fanout = 1;
    std::uint64_t seed = 0;
    bool verify = false;
    bool debug_validate = false;
    std::size_t learned_capacity = 1u << 22;
    std::function<void(const ConflictTrace&)> trace;
    // device extensions (not in the reference)
    int device = 0;
    std::uint32_t cube_atoms = 0, cube_depth = 0;
    int rank = 0, world = 1;
    std::uint32_t portfolio = 0;  // first-model portfolio: concurrent searches with diverse (mode, heuristic)
    bool count_lits = false;      // exact literals of checked nogoods in stats.checked_lits
    std::vector<int> devices;     // cube enumeration / portfolio over these GPUs of this process
    bool reference_order = false; // enumerate as one search in the reference's model order
    yas_fleet* fleet = nullptr;   // processes sharing one enumeration / portfolio (yas_fleet_create*)
};

struct SolveStats : yas_stats {
    SolveStats() : yas_stats{} {}
    double avg_learned_len() const {
        return learned_count == 0 ? 0.0 : static_cast<double>(learned_length_sum) / static_cast<double>(learned_count);
    }
    double wall_seconds() const { return wall_ms / 1000.0; }
    double per_second(std::uint64_t c) const { return wall_ms <= 0.0 ? 0.0 : static_cast<double>(c) / wall_seconds(); }
    double propagations_per_sec() const { return per_second(propagations); }
    double decisions_per_sec() const { return per_second(decisions); }
    double learned_per_sec() const { return per_second(learned_count); }
};

struct Model {
    std::vector<AtomId> atom_ids;
    std::vector<std::string> atoms;
};

struct SolveResult {
    std::vector<Model> models;
    SolveStats stats;
    SolveStatus status = SolveStatus::unsat;
};

inline SolveResult solve(const GroundProgram& prog, const SolverConfig& cfg) {
    yas_config c;
    yas_config_default(&c);
    c.mode = cfg.mode == LearnMode::res ? 1 : 0;
    c.heuristic = static_cast<int>(cfg.heuristic.kind);
    c.activity_decay = cfg.heuristic.activity_decay;
    c.workers = cfg.workers;
    c.restarts_enabled = cfg.restarts.enabled;
    c.restart_base = cfg.restarts.base;
    c.restart_factor = cfg.restarts.factor;
    c.max_models = cfg.max_models;
    c.deps_words = cfg.deps_words;
    c.conflict_fanout = cfg.conflict_fanout;
    c.seed = cfg.seed;
    c.verify = cfg.verify;
    c.debug_validate = cfg.debug_validate;
    c.learned_capacity = cfg.learned_capacity;
    c.device = cfg.device;
    c.cube_atoms = cfg.cube_atoms;
    c.cube_depth = cfg.cube_depth;
    c.rank = cfg.rank;
    c.world = cfg.world;
    c.portfolio = cfg.portfolio;
    c.count_lits = cfg.count_lits ? 1u : 0u;
    if (cfg.devices.size() > 1) {
        c.n_devices = static_cast<std::uint32_t>(cfg.devices.size());
        c.devices = cfg.devices.data();
    }
    c.fleet = cfg.fleet;
    c.reference_order = cfg.reference_order ? 1 : 0;
    if (cfg.trace) {
        c.trace = [](const yas_trace* t, void* user) {
            (*static_cast<const std::function<void(const ConflictTrace&)>*>(user))(
                {t->mode ? LearnMode::res : LearnMode::fwd, t->conflict_id, static_cast<std::size_t>(t->learned_length),
                 t->backjump_level});
        };
        c.trace_user = const_cast<std::function<void(const ConflictTrace&)>*>(&cfg.trace);
    }
    yas_result* r = nullptr;
    char err[1024];
    const int rc = yas_solve(prog.handle(), &c, &r, err, sizeof err);
    if (rc != YAS_OK) detail::raise(rc, err);
    std::unique_ptr<yas_result, void (*)(yas_result*)> guard(r, &yas_result_free);
    SolveResult out;
    yas_result_stats(r, &out.stats);
    const std::uint64_t n = yas_result_model_count(r);
    out.models.reserve(n);
    for (std::uint64_t m = 0; m < n; ++m) {
        std::uint32_t len = 0;
        const std::uint32_t* ids = yas_result_model(r, m, &len);
        Model mo;
        mo.atom_ids.assign(ids, ids + len);
        for (AtomId a : mo.atom_ids) mo.atoms.push_back(prog.name(a));
        std::sort(mo.atoms.begin(), mo.atoms.end());
        out.models.push_back(std::move(mo));
    }
    out.status = yas_result_status(r) == 0 ? SolveStatus::sat : SolveStatus::unsat;
    return out;
}

inline bool verify_model(const GroundProgram& prog, const Model& m) {
    return yas_verify_model(prog.handle(), m.atom_ids.data(), m.atom_ids.size()) == 1;
}

inline const char* to_string(LearnMode m) { return m == LearnMode::fwd ? "fwd" : "res"; }
inline const char* to_string(HeuristicKind k) {
    return k == HeuristicKind::jeroslow_wang ? "jw" : k == HeuristicKind::activity ? "act" : "occ";
}
inline const char* to_string(SolveStatus s) { return s == SolveStatus::sat ? "SAT" : "UNSAT"; }

enum class StatsFormat : std::uint8_t { human, csv };
struct StatsContext {
    std::string instance, mode, heuristic;
    unsigned workers = 1;
    SolveStatus status = SolveStatus::unsat;
    std::uint64_t models = 0;
};

inline std::string stats_csv_header() {
    std::string s(yas_stats_csv_header(nullptr, 0), '\0');
    yas_stats_csv_header(s.data(), s.size() + 1);
    return s;
}

inline std::string emit_stats(const SolveStats& st, const StatsContext& ctx, StatsFormat f) {
    auto call = [&](char* buf, std::size_t cap) {
        return yas_emit_stats(&st, ctx.instance.c_str(), ctx.mode.c_str(), ctx.heuristic.c_str(), ctx.workers,
                              ctx.status == SolveStatus::sat ? 0 : 1, ctx.models, f == StatsFormat::csv, buf, cap);
    };
    std::string s(call(nullptr, 0), '\0');
    call(s.data(), s.size() + 1);
    return s;
}

}  // namespace aspine
