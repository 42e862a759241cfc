// C++ drop-in façade for callers of the reference solver's public API
// (/root/reference/proj/include/aspine/{program,solver}.hpp), implemented over
// the yasmin-b200 C-ABI (include/yasmin_b200.h). Same names, argument meaning
// and error behaviour as the reference:
//   aspine::parse_program(std::istream&) / (std::string_view)   program.hpp:87-88
//   aspine::solve(const GroundProgram&, const SolverConfig&)     solver.hpp:113
//   aspine::verify_model / emit_stats / stats_csv_header          solver.hpp:116-133
//   ParseError{line}, StoreCapacityError, VerificationError, std::logic_error
// Header-only; link with -lyasmin_b200.
#pragma once

#include <functional>
#include <istream>
#include <iterator>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "../yasmin_b200.h"

namespace aspine {

using AtomId = std::uint32_t;

struct ParseError : std::runtime_error {
    ParseError(int l, const std::string& what) : std::runtime_error(what), line(l) {}
    int line;
};
struct StoreCapacityError : std::runtime_error {
    using std::runtime_error::runtime_error;
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

class GroundProgram {
public:
    GroundProgram() = default;
    explicit GroundProgram(yas_program* p) : p_(p, &yas_program_free) {}
    AtomId atom_count() const { return yas_program_atom_count(p_.get()); }
    std::string name(AtomId id) const {
        const char* s = yas_program_atom_name(p_.get(), id);
        return s ? s : "";
    }
    AtomId find(std::string_view n) const { return yas_program_find(p_.get(), std::string(n).c_str()); }
    const yas_program* handle() const { return p_.get(); }

private:
    std::shared_ptr<yas_program> p_;
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
};

struct SolveStats : yas_stats {
    SolveStats() : yas_stats{} {}
    double avg_learned_len() const {
        return learned_count == 0 ? 0.0 : static_cast<double>(learned_length_sum) / static_cast<double>(learned_count);
    }
    double per_second(std::uint64_t c) const { return wall_ms <= 0.0 ? 0.0 : static_cast<double>(c) / (wall_ms / 1000.0); }
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
