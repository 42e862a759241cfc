// C-ABI of yasmin-b200 (include/yasmin_b200.h). Host orchestration only:
// parse -> completion -> static store -> device engine. There is no CPU
// solving path: when no CUDA device is usable the solve entry points fail
// with YAS_ERR_DEVICE.
#include "../../include/yasmin_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <memory>
#include <new>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "device/engine_api.hpp"
#include "fleet.hpp"
#include "host/compile.hpp"
#include "host/program.hpp"

using namespace yas;

struct yas_program {
    Program prog;
    // lazily compiled views
    std::unique_ptr<Completion> comp;
    std::unique_ptr<StaticStore> store;

    const Completion& completion() {
        if (!comp) comp = std::make_unique<Completion>(compile_completion(prog));
        return *comp;
    }
    const StaticStore& static_store() {
        if (!store) store = std::make_unique<StaticStore>(build_store(completion().nogoods, completion().total_atoms));
        return *store;
    }
};

struct yas_result {
    // models flat: model m is ids[off[m], off[m + 1]) (sorted atom ids)
    std::vector<std::uint32_t> ids;
    std::vector<std::uint64_t> off{0};
    std::size_t count() const { return off.size() - 1; }
    std::vector<std::uint32_t> cubes;
    yas_stats stats{};
    int status = 1;
};

struct yas_store {
    StaticStore st;
};

struct yas_propagator {
    std::unique_ptr<Session> s;
    std::uint32_t atoms = 0;
    char err[512] = {0};  // message of the last failed call (yas_propagator_last_error)
};

namespace {

void put_err(char* err, std::size_t cap, const std::string& msg) {
    if (!err || cap == 0) return;
    const std::size_t n = std::min(cap - 1, msg.size());
    std::memcpy(err, msg.data(), n);
    err[n] = '\0';
}

std::size_t put_text(const std::string& s, char* buf, std::size_t cap) {
    if (buf && cap) {
        const std::size_t n = std::min(cap - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = '\0';
    }
    return s.size();
}

struct DeviceMissing : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CapacityError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct VerifyError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

void require_device(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        throw DeviceMissing("no CUDA device available: yasmin-b200 has no CPU solving path");
    if (device < 0 || device >= n) throw DeviceMissing("CUDA device ordinal out of range");
}

template <class F>
int guarded(char* err, std::size_t cap, F&& f) {
    if (err && cap) err[0] = '\0';  // a message always describes the call that returned it
    try {
        return f();
    } catch (const ParseFailure& e) {
        put_err(err, cap, e.what());
        return YAS_ERR_PARSE;
    } catch (const CapacityError& e) {
        put_err(err, cap, e.what());
        return YAS_ERR_CAPACITY;
    } catch (const VerifyError& e) {
        put_err(err, cap, e.what());
        return YAS_ERR_VERIFY;
    } catch (const std::invalid_argument& e) {
        put_err(err, cap, e.what());
        return YAS_ERR_ARG;
    } catch (const std::length_error& e) {  // store beyond the device layout's limits
        put_err(err, cap, e.what());
        return YAS_ERR_CAPACITY;
    } catch (const std::out_of_range& e) {
        put_err(err, cap, e.what());
        return YAS_ERR_ARG;
    } catch (const std::logic_error& e) {
        put_err(err, cap, e.what());
        return YAS_ERR_LOGIC;
    } catch (const DeviceMissing& e) {
        put_err(err, cap, e.what());
        return YAS_ERR_DEVICE;
    } catch (const std::runtime_error& e) {
        put_err(err, cap, e.what());
        return static_cast<int>(std::string(e.what()).rfind("CUDA", 0) == 0 ? YAS_ERR_DEVICE : YAS_ERR_ARG);
    } catch (const std::exception& e) {
        put_err(err, cap, e.what());
        return YAS_ERR_ARG;
    }
}

// Choice atoms: a whose only rule is "a :- not b." where b has the rule
// "b :- not a." (the even-loop choice encoding). For such an atom
//   T a  <=>  F b   and the constraint ":- not a." is equivalent to ":- b.",
// so both cube polarities can be stated as *forcing* unit nogoods: F a as
// {T a}, T a as {T b}. Partners are skipped (b is determined by a).
//
// Any other atom a that heads a rule can split too: ":- a." is the unit nogood
// {T a} (asserts F a), ":- not a." the unit nogood {F a}; the latter may not
// assert T a (truth guard kNoTruth, nogood.hpp:62-73) and stays a passive
// check that fails when a becomes false. Such atoms (b = 0) follow the choice
// pairs, in atom order, so programs without even loops shard as well.
struct Choice {
    AtomId a, b;
};

std::vector<Choice> choice_atoms(const Program& prog) {
    std::vector<Choice> out;
    std::vector<char> taken(prog.atom_count() + 1, 0);
    for (AtomId a = 1; a <= prog.atom_count(); ++a) {
        if (taken[a] || prog.rules_of(a).size() != 1) continue;
        const Rule& r = prog.rules()[prog.rules_of(a)[0]];
        if (!r.pos_body.empty() || r.neg_body.size() != 1 || r.neg_body[0] == a) continue;
        const AtomId b = r.neg_body[0];
        bool pair = false;
        for (std::uint32_t ri : prog.rules_of(b)) {
            const Rule& q = prog.rules()[ri];
            pair |= q.pos_body.empty() && q.neg_body.size() == 1 && q.neg_body[0] == a;
        }
        if (!pair) continue;
        out.push_back({a, b});
        taken[a] = taken[b] = 1;
    }
    for (AtomId a = 1; a <= prog.atom_count(); ++a)
        if (!taken[a] && !prog.rules_of(a).empty()) out.push_back({a, 0});
    return out;
}

// Automatic split of a plain enumeration (max_models == 0, no cube_atoms):
// programs with at least this many even-loop choice pairs.
constexpr std::size_t kAutoCubePairs = 16;
constexpr std::uint32_t kAutoCubeWidth = 8;  // ladder width without an at-least-one group

// "At least one of these choices" groups: an integrity constraint whose body
// only says "none of a_1..a_k is true" (each literal "not a_i", or the pair
// partner b_i) — a queens row, the colours of a node. A ladder over one group
// asks which member is its first true one; its last cube (none) fails at once,
// so the cubes follow the problem's own structure. Groups come first in the
// choice order (constraint order, atoms ascending, no atom twice); the ladder
// width is the first group's size (0: no group).
std::uint32_t group_choices(const Program& prog, std::vector<Choice>& ch) {
    std::vector<std::int64_t> of_a(prog.atom_count() + 1, -1), of_b(prog.atom_count() + 1, -1);
    for (std::size_t i = 0; i < ch.size(); ++i)
        if (ch[i].b) {
            of_a[ch[i].a] = static_cast<std::int64_t>(i);
            of_b[ch[i].b] = static_cast<std::int64_t>(i);
        }
    std::vector<char> used(ch.size(), 0);
    std::vector<Choice> order;
    std::uint32_t width = 0;
    for (const Rule& c : prog.constraints()) {
        std::vector<std::size_t> g;
        bool ok = c.pos_body.size() + c.neg_body.size() >= 2;
        for (AtomId x : c.pos_body) {  // b_i true <=> a_i false
            if (!ok) break;
            ok = of_b[x] >= 0;
            if (ok) g.push_back(static_cast<std::size_t>(of_b[x]));
        }
        for (AtomId x : c.neg_body) {  // not a_i
            if (!ok) break;
            ok = of_a[x] >= 0;
            if (ok) g.push_back(static_cast<std::size_t>(of_a[x]));
        }
        if (!ok) continue;
        std::sort(g.begin(), g.end());
        if (std::adjacent_find(g.begin(), g.end()) != g.end()) continue;
        if (std::any_of(g.begin(), g.end(), [&](std::size_t i) { return used[i]; })) continue;
        if (!width) width = static_cast<std::uint32_t>(g.size());
        for (std::size_t i : g) {
            used[i] = 1;
            order.push_back(ch[i]);
        }
    }
    if (!width) return 0;
    for (std::size_t i = 0; i < ch.size(); ++i)
        if (!used[i]) order.push_back(ch[i]);
    ch.swap(order);
    return width;
}

bool first_choices_are_pairs(const Program& prog) {
    const std::vector<Choice> ch = choice_atoms(prog);
    return ch.size() >= kAutoCubePairs && ch[kAutoCubePairs - 1].b != 0;
}

// Nested "ladder" cubes over windows of L choice atoms: at each of d levels the
// cube picks i in [0, L]: i < L means (F a_0, ..., F a_{i-1}, T a_i) and i = L
// means all F. The (L+1)^d cubes partition the answer sets exactly. Cube c
// belongs to rank c % world. Returns this rank's cube count.
std::uint32_t make_cubes(const Program& prog, std::uint32_t L, std::uint32_t depth, std::uint32_t want, int rank,
                         int world, std::vector<std::int32_t>& cubes, std::uint32_t& width, bool grouped = false) {
    std::vector<Choice> ch = choice_atoms(prog);
    if (grouped) {  // automatic split: ladders over the at-least-one groups
        const std::uint32_t g = group_choices(prog, ch);
        L = g ? g : kAutoCubeWidth;
    }
    cubes.clear();
    width = 0;
    if (world < 1) world = 1;
    if (L == 0 || ch.empty()) return rank == 0 ? 1u : 0u;
    L = std::min<std::uint32_t>(L, static_cast<std::uint32_t>(ch.size()));
    std::uint32_t maxd = static_cast<std::uint32_t>(ch.size()) / L;
    if (depth == 0) {  // smallest depth giving `want` cubes, at most 2^17 cubes
        depth = 1;
        std::uint64_t n = L + 1;
        while (n < want && depth < maxd && n * (L + 1) <= (1u << 17)) {
            n *= L + 1;
            ++depth;
        }
    }
    depth = std::max<std::uint32_t>(1, std::min(depth, maxd));
    width = depth * L;
    std::uint64_t total = 1;
    for (std::uint32_t j = 0; j < depth; ++j) total *= L + 1;
    // the L literals of level j for pick p, precomputed: pat[(j * (L + 1) + p) * L + i]
    std::vector<std::int32_t> pat(static_cast<std::size_t>(depth) * (L + 1) * L, 0);
    for (std::uint32_t j = 0; j < depth; ++j)
        for (std::uint32_t p = 0; p <= L; ++p)
            for (std::uint32_t i = 0; i < L && i <= p; ++i) {
                const Choice& c = ch[j * L + i];
                // F a: nogood {T a}; T a: nogood {T b} (choice pair) or {F a}
                const std::int32_t t = c.b ? static_cast<std::int32_t>(c.b) : -static_cast<std::int32_t>(c.a);
                pat[(static_cast<std::size_t>(j) * (L + 1) + p) * L + i] = i < p ? static_cast<std::int32_t>(c.a) : t;
            }
    const std::uint64_t mine = total / static_cast<std::uint64_t>(world) +
                               (static_cast<std::uint64_t>(rank) < total % static_cast<std::uint64_t>(world) ? 1 : 0);
    cubes.resize(mine * width);
    std::int32_t* out = cubes.data();
    std::uint32_t n = 0;
    for (std::uint64_t cube = static_cast<std::uint64_t>(rank); cube < total; cube += static_cast<std::uint64_t>(world)) {
        std::uint64_t digits = cube;
        for (std::uint32_t j = 0; j < depth; ++j) {
            const std::uint32_t pick = static_cast<std::uint32_t>(digits % (L + 1));
            digits /= L + 1;
            std::memcpy(out, pat.data() + (static_cast<std::size_t>(j) * (L + 1) + pick) * L, L * sizeof(std::int32_t));
            out += L;
        }
        ++n;
    }
    cubes.resize(static_cast<std::size_t>(n) * width);
    return n;
}

void fill_stats(yas_stats& o, const dev::Stats& s) {
    o.decisions = s.decisions;
    o.propagations = s.propagations;
    o.conflicts = s.conflicts;
    o.learned_count = s.learned_count;
    o.learned_length_sum = s.learned_length_sum;
    o.restarts = s.restarts;
    o.models = s.models;
    o.passes = s.passes;
    o.watch_replacements = 0;  // no watched literals on the device
    o.duplicate_learned = s.duplicate_learned;
    o.blocking_nogoods = s.blocking_nogoods;
    o.res_learned = s.res_learned;
    o.fwd_learned = s.fwd_learned;
    o.fwd_fallbacks = s.fwd_fallbacks;
    o.uip_check_failures = s.uip_check_failures;
    o.fwd_decision_only_failures = s.fwd_decision_only_failures;
    o.asserting_failures = s.asserting_failures;
    o.checks = s.checks;
    o.searches = s.searches;
    o.checked_lits = s.checked_lits;
}

}  // namespace

extern "C" {

const char* yas_version(void) { return "yasmin-b200 0.1 (sm_100a)"; }

int yas_device_count(void) {
    int n = 0;
    return cudaGetDeviceCount(&n) == cudaSuccess ? n : 0;
}

int yas_device_name(int device, char* buf, size_t cap) {
    if (device < 0 || device >= yas_device_count()) return YAS_ERR_DEVICE;
    put_text(device_name(device), buf, cap);
    return YAS_OK;
}

int yas_program_parse(const char* text, size_t len, yas_program** out, int* err_line, char* err, size_t err_cap) {
    if (!out) return YAS_ERR_ARG;
    *out = nullptr;
    if (err_line) *err_line = 0;
    return guarded(err, err_cap, [&] {
        try {
            auto p = std::make_unique<yas_program>();
            p->prog = parse_text(std::string_view(text ? text : "", text ? len : 0));
            *out = p.release();
            return static_cast<int>(YAS_OK);
        } catch (const ParseFailure& e) {
            if (err_line) *err_line = e.line;
            throw;
        }
    });
}

int yas_program_parse_file(const char* path, yas_program** out, int* err_line, char* err, size_t err_cap) {
    if (!path || !out) return YAS_ERR_ARG;
    std::ifstream in(path, std::ios::binary);
    if (!in) {
        put_err(err, err_cap, std::string("cannot open ") + path);
        return YAS_ERR_IO;
    }
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    return yas_program_parse(text.data(), text.size(), out, err_line, err, err_cap);
}

yas_program* yas_program_create(void) { return new (std::nothrow) yas_program(); }

uint32_t yas_program_intern(yas_program* p, const char* name) {
    if (!p || !name) return 0;
    std::uint32_t id = 0;
    guarded(nullptr, 0, [&] {
        id = p->prog.intern(name);
        p->comp.reset();  // compiled views follow the program
        p->store.reset();
        return 0;
    });
    return id;
}

int yas_program_add_rule(yas_program* p, uint32_t head, const uint32_t* pos, size_t n_pos, const uint32_t* neg,
                         size_t n_neg) {
    if (!p || (n_pos && !pos) || (n_neg && !neg)) return YAS_ERR_ARG;
    const std::uint32_t n = p->prog.atom_count();
    if (head > n) return YAS_ERR_ARG;
    for (size_t i = 0; i < n_pos; ++i)
        if (pos[i] == 0 || pos[i] > n) return YAS_ERR_ARG;
    for (size_t i = 0; i < n_neg; ++i)
        if (neg[i] == 0 || neg[i] > n) return YAS_ERR_ARG;
    return guarded(nullptr, 0, [&] {
        Rule r;
        r.head = head;
        r.pos_body.assign(pos, pos + n_pos);
        r.neg_body.assign(neg, neg + n_neg);
        p->prog.add_rule(std::move(r));
        p->comp.reset();
        p->store.reset();
        return static_cast<int>(YAS_OK);
    });
}

void yas_program_free(yas_program* p) { delete p; }
uint32_t yas_program_atom_count(const yas_program* p) { return p ? p->prog.atom_count() : 0; }
uint32_t yas_program_rule_count(const yas_program* p) { return p ? static_cast<uint32_t>(p->prog.rules().size()) : 0; }
uint32_t yas_program_constraint_count(const yas_program* p) {
    return p ? static_cast<uint32_t>(p->prog.constraints().size()) : 0;
}
const char* yas_program_atom_name(const yas_program* p, uint32_t id) {
    if (!p || id > p->prog.atom_count()) return nullptr;
    return p->prog.name(id).c_str();
}
uint32_t yas_program_find(const yas_program* p, const char* name) { return p && name ? p->prog.find(name) : 0; }

int yas_program_rule(const yas_program* p, uint32_t r, uint32_t* head, const uint32_t** pos, uint32_t* n_pos,
                     const uint32_t** neg, uint32_t* n_neg) {
    if (!p) return YAS_ERR_ARG;
    const std::size_t nr = p->prog.rules().size();
    if (r >= nr + p->prog.constraints().size()) return YAS_ERR_ARG;
    const Rule& rule = r < nr ? p->prog.rules()[r] : p->prog.constraints()[r - nr];
    if (head) *head = rule.head;
    if (pos) *pos = rule.pos_body.data();
    if (n_pos) *n_pos = static_cast<uint32_t>(rule.pos_body.size());
    if (neg) *neg = rule.neg_body.data();
    if (n_neg) *n_neg = static_cast<uint32_t>(rule.neg_body.size());
    return YAS_OK;
}

size_t yas_program_print(const yas_program* p, char* buf, size_t cap) { return p ? put_text(print_text(p->prog), buf, cap) : 0; }
size_t yas_program_dump_nogoods(const yas_program* p, char* buf, size_t cap) {
    if (!p) return 0;
    auto* q = const_cast<yas_program*>(p);
    std::size_t n = 0;
    guarded(nullptr, 0, [&] { n = put_text(dump_nogoods(q->completion(), q->prog), buf, cap); return 0; });
    return n;
}
size_t yas_program_store_csv(const yas_program* p, char* buf, size_t cap) {
    if (!p) return 0;
    std::size_t n = 0;
    guarded(nullptr, 0, [&] { n = put_text(const_cast<yas_program*>(p)->static_store().dump_csv(), buf, cap); return 0; });
    return n;
}
size_t yas_program_diagnostics(const yas_program* p, char* buf, size_t cap) {
    if (!p) return 0;
    std::size_t n = 0;
    guarded(nullptr, 0, [&] {
        std::string s;
        for (const std::string& d : diagnostics(p->prog)) s += d + "\n";
        n = put_text(s, buf, cap);
        return 0;
    });
    return n;
}
int yas_program_rule_aux(const yas_program* p, uint32_t rule, uint32_t out[4]) {
    if (!p || !out || rule >= p->prog.rules().size()) return YAS_ERR_ARG;
    return guarded(nullptr, 0, [&] {
        const RuleAux& a = const_cast<yas_program*>(p)->completion().aux[rule];
        out[0] = a.b;
        out[1] = a.t;
        out[2] = a.n;
        out[3] = a.vacuous ? 1 : 0;
        return static_cast<int>(YAS_OK);
    });
}
uint32_t yas_program_total_atoms(const yas_program* p) {
    if (!p) return 0;
    std::uint32_t n = 0;
    guarded(nullptr, 0, [&] { n = const_cast<yas_program*>(p)->completion().total_atoms; return 0; });
    return n;
}
int yas_program_census(const yas_program* p, uint64_t census_out[3], uint64_t counts[3]) {
    if (!p || !census_out || !counts) return YAS_ERR_ARG;
    return guarded(nullptr, 0, [&] {
    const Census c = census(p->prog);
    const Census& k = const_cast<yas_program*>(p)->completion().counts;
    census_out[0] = c.rule_nogoods;
    census_out[1] = c.atom_nogoods;
    census_out[2] = c.constraint_nogoods;
    counts[0] = k.rule_nogoods;
    counts[1] = k.atom_nogoods;
    counts[2] = k.constraint_nogoods;
    return static_cast<int>(YAS_OK);
    });
}
size_t yas_program_tp_step(const yas_program* p, const uint32_t* interp, size_t n, uint32_t* out, size_t cap) {
    if (!p || (n && !interp)) return SIZE_MAX;
    for (size_t i = 0; i < n; ++i)
        if (interp[i] == 0 || interp[i] > p->prog.atom_count()) return SIZE_MAX;  // tp_step indexes with at()
    std::size_t total = SIZE_MAX;
    guarded(nullptr, 0, [&] {
        std::vector<AtomId> in(interp, interp + n);
        const std::vector<AtomId> r = tp_step(p->prog, in);
        for (std::size_t i = 0; i < r.size() && i < cap; ++i) out[i] = r[i];
        total = r.size();
        return 0;
    });
    return total;
}
size_t yas_program_cubes(const yas_program* p, uint32_t k, uint32_t depth, uint32_t want, int rank, int world,
                         int32_t* out, size_t cap, uint32_t* width) {
    if (!p) return 0;
    std::size_t n = 0;
    guarded(nullptr, 0, [&] {
        std::vector<std::int32_t> cubes;
        std::uint32_t w = 0;
        n = make_cubes(p->prog, k, depth, want ? want : 2368, rank, world, cubes, w, k == 0);
        if (width) *width = w;
        for (std::size_t i = 0; i < cubes.size() && out && i < cap; ++i) out[i] = cubes[i];
        return 0;
    });
    return n;
}

int yas_verify_model(const yas_program* p, const uint32_t* ids, size_t n) {
    if (!p || (n && !ids)) return -YAS_ERR_ARG;
    for (size_t i = 0; i < n; ++i)
        if (ids[i] == 0 || ids[i] > p->prog.atom_count()) return -YAS_ERR_ARG;
    int ok = -YAS_ERR_ARG;
    guarded(nullptr, 0, [&] {
        ok = is_answer_set(p->prog, std::vector<AtomId>(ids, ids + n)) ? 1 : 0;
        return 0;
    });
    return ok;
}

void yas_config_default(yas_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->mode = 0;
    c->heuristic = 0;
    c->activity_decay = 0.95;
    c->workers = 1;
    c->restart_base = 100;
    c->restart_factor = 1.5;
    c->max_models = 1;
    c->deps_words = 16;
    c->conflict_fanout = 1;
    c->learned_capacity = 1ull << 22;
    c->world = 1;
}

namespace {

// One engine run per GPU of this process, in parallel host threads; the
// models each GPU delivers are kept per GPU (merged by the caller).
struct DevRun {
    int device = 0;
    dev::Config dc{};
    EngineOptions eo;
    std::vector<std::int32_t> cubes;
    std::uint32_t n_cubes = 0;
    EngineResult er;
    std::vector<std::uint32_t> ids;
    std::vector<std::uint64_t> offs{0};
    std::vector<std::uint32_t> mcubes;
    std::vector<yas_trace> traces;
    std::exception_ptr error;
};

void run_device(DevRun& d, const EngineProgram& ep, const Program& prog, const yas_config& cfg, std::uint32_t width,
                std::atomic<std::uint64_t>* found = nullptr) {
    try {
        d.ids.clear();
        d.offs.assign(1, 0);
        d.mcubes.clear();
        d.traces.clear();
        EngineCallbacks cb;
        const std::uint32_t np = prog.atom_count();
        // every slot's models of one drain, in slot order
        cb.on_models = [&](const EngineDrain& dr) {
            std::uint64_t total = 0;
            for (std::uint32_t s = 0; s < dr.n_slots; ++s) total += dr.counts[s];
            if (total == 0) return true;
            d.offs.reserve(d.offs.size() + total);
            d.mcubes.reserve(d.mcubes.size() + total);
            for (std::uint32_t s = 0; s < dr.n_slots; ++s)
                for (std::uint32_t m = 0; m < dr.counts[s]; ++m) {
                    const std::size_t k = static_cast<std::size_t>(s) * dr.stride + m;
                    const std::uint32_t* bits = dr.bits + k * dr.nwords;
                    const std::size_t at = d.ids.size();
                    for (std::size_t w = 0; w < dr.nwords; ++w)
                        for (std::uint32_t b = bits[w]; b; b &= b - 1) {
                            const std::uint32_t a =
                                static_cast<std::uint32_t>(32 * w) + static_cast<std::uint32_t>(__builtin_ctz(b)) + 1;
                            if (a <= np) d.ids.push_back(a);
                        }
                    if (cfg.verify) {
                        // record_model's checks (solver.cpp:221-229)
                        const std::vector<std::uint32_t> ids(d.ids.begin() + static_cast<std::ptrdiff_t>(at), d.ids.end());
                        if (!is_answer_set(prog, ids)) throw VerifyError("computed model is not an answer set");
                        if (tp_step(prog, ids) != ids)
                            throw VerifyError("computed model is not a fixpoint of the consequence operator");
                    }
                    d.offs.push_back(d.ids.size());
                    d.mcubes.push_back(dr.cubes[k]);
                }
            // cube-parallel first models: stop this GPU's loop once enough arrived anywhere
            return !found || found->fetch_add(total) + total < cfg.max_models;
        };
        if (cfg.trace)
            cb.on_trace = [&](std::uint32_t mode, std::int32_t conflict, std::uint32_t len, std::uint32_t bj) {
                d.traces.push_back({static_cast<int>(mode), conflict, len, bj});
            };
        d.er = EngineResult{};
        if (d.n_cubes > 0) d.er = engine_solve(ep, d.dc, d.eo, d.cubes, d.n_cubes, width, cb);
    } catch (...) {
        d.error = std::current_exception();
    }
}

// Shared queue / claim block for the GPUs of this process (no fleet): in the
// first GPU's memory, mapped into the others over NVLink. Returns null when a
// GPU cannot reach it (then the cubes are dealt statically).
struct LocalFleet {
    dev::Fleet* ctl = nullptr;
    int home = 0;
    ~LocalFleet() {
        if (ctl) {
            cudaSetDevice(home);
            cudaFree(ctl);
        }
    }
};

bool local_fleet(LocalFleet& lf, const std::vector<int>& devs) {
    lf.home = devs[0];
    for (int d : devs) {
        if (d == lf.home) continue;
        int ok = 0;
        if (cudaDeviceCanAccessPeer(&ok, d, lf.home) != cudaSuccess || !ok) return false;
        ck_cuda(cudaSetDevice(d), "cudaSetDevice");
        const cudaError_t e = cudaDeviceEnablePeerAccess(lf.home, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else ck_cuda(e, "cudaDeviceEnablePeerAccess");
    }
    ck_cuda(cudaSetDevice(lf.home), "cudaSetDevice");
    ck_cuda(cudaMalloc(&lf.ctl, sizeof(dev::Fleet)), "cudaMalloc fleet");
    return true;
}

void reset_fleet_ctl(dev::Fleet* ctl, int device) {
    ck_cuda(cudaSetDevice(device), "cudaSetDevice");
    const dev::Fleet init{0u, 0u, 0xffffffffu, 0u};  // queue, stop, winner, found
    ck_cuda(cudaMemcpy(ctl, &init, sizeof init, cudaMemcpyHostToDevice), "fleet reset");
}

}  // namespace

int yas_solve(const yas_program* p, const yas_config* cfg_in, yas_result** out, char* err, size_t err_cap) {
    if (!p || !out) return YAS_ERR_ARG;
    *out = nullptr;
    yas_config cfg;
    if (cfg_in) cfg = *cfg_in;
    else yas_config_default(&cfg);
    return guarded(err, err_cap, [&] {
        if (cfg.deps_words < 1 || cfg.deps_words > 1024) throw std::invalid_argument("deps_words must be in [1, 1024]");
        yas_fleet* fl = cfg.fleet;
        if (fl) {
            if (cfg.n_devices > 1) throw std::invalid_argument("a fleet runs one GPU per process (n_devices must be <= 1)");
            cfg.rank = fl->rank;
            cfg.world = fl->world;
            cfg.device = fl->device;
        }
        if (cfg.world < 1) cfg.world = 1;
        const auto tp0 = std::chrono::steady_clock::now();
        const bool prof = std::getenv("YAS_PROFILE") != nullptr;
        auto lap = [&](const char* what) {
            if (prof)
                std::fprintf(stderr, "[yas host] %s at %.2f ms\n", what,
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count());
        };
        std::vector<int> devs;
        if (cfg.n_devices > 1)
            for (std::uint32_t i = 0; i < cfg.n_devices; ++i) devs.push_back(cfg.devices ? cfg.devices[i] : cfg.device + static_cast<int>(i));
        else
            devs.push_back(cfg.device);
        for (int d : devs) require_device(d);
        lap("device");
        auto* q = const_cast<yas_program*>(p);
        const Program& prog = q->prog;
        const Completion& comp = q->completion();
        const StaticStore& st = q->static_store();

        EngineProgram ep;
        ep.store = &st;
        ep.n_prog = prog.atom_count();
        ep.rules.reserve(prog.rules().size());
        for (std::size_t r = 0; r < prog.rules().size(); ++r) {
            const RuleAux& a = comp.aux[r];
            ep.rules.push_back({prog.rules()[r].head, a.b, a.t, a.n | (a.vacuous ? 0x80000000u : 0u)});
        }

        dev::Config dc{};
        dc.mode = cfg.mode == 1 ? 1u : 0u;
        dc.heur = cfg.heuristic == 1 ? 1u : cfg.heuristic == 2 ? 2u : 0u;
        dc.decay = cfg.activity_decay;
        dc.restarts = cfg.restarts_enabled ? 1u : 0u;
        dc.W = cfg.deps_words;
        dc.restart_base = cfg.restart_base;
        dc.restart_factor = cfg.restart_factor;
        dc.max_models = cfg.max_models;
        dc.fanout = std::max<std::uint32_t>(1, std::min<std::uint32_t>(cfg.conflict_fanout, 64));
        dc.debug_validate = cfg.debug_validate ? 1u : 0u;
        dc.learned_capacity = cfg.learned_capacity;
        dc.trace = cfg.trace ? 1u : 0u;
        dc.count_lits = cfg.count_lits ? 1u : 0u;

        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg.device);
        std::uint32_t per_sm = 8;  // concurrent searches per SM for cube enumeration
        if (const char* e = std::getenv("YAS_SEARCHES_PER_SM")) per_sm = static_cast<std::uint32_t>(std::strtoul(e, nullptr, 10));
        const std::uint32_t slots_per_gpu = cfg.slots ? cfg.slots : static_cast<std::uint32_t>(sms) * per_sm;
        // Enumerating every answer set of a program with many choice pairs is
        // split into cubes unless the caller asked for the reference's model
        // order (or traces the reference's conflict sequence): the answer-set
        // set and count are the reference's, the order becomes cube order.
        // Not on an explicitly requested whole-GPU engine: it runs one search
        // at a time, so cubes would only run one after another.
        bool auto_cubes = false;
        if (cfg.cube_atoms == 0 && cfg.max_models == 0 && !cfg.reference_order && !cfg.trace && cfg.engine != 2 &&
            first_choices_are_pairs(prog)) {
            cfg.cube_atoms = kAutoCubeWidth;  // the width itself comes from the program's groups
            auto_cubes = true;
        }
        // cube_atoms with max_models >= 1: cube-parallel search for the first
        // max_models answer sets (any of them; an extra mode like the portfolio)
        const bool enumerate = cfg.cube_atoms > 0;
        const bool portfolio = cfg.portfolio > 1 && cfg.max_models == 1 && cfg.cube_atoms == 0;
        if (!enumerate && !portfolio) devs.resize(1);  // one search: the first GPU
        const std::uint32_t ndev = static_cast<std::uint32_t>(devs.size());
        const std::uint32_t gpus = ndev * static_cast<std::uint32_t>(cfg.world);  // every GPU of the fleet

        // the shared queue: this process's GPUs (peer mappings) or the fleet (IPC)
        LocalFleet lf;
        dev::Fleet* shared = nullptr;
        int shared_dev = cfg.device;
        if (fl) {
            shared = fl->ctl;
            shared_dev = fl->device;
        } else if (ndev > 1 && local_fleet(lf, devs)) {
            shared = lf.ctl;
            shared_dev = lf.home;
        }
        const bool dynamic = fl ? fl->dynamic : shared != nullptr;

        std::vector<DevRun> runs(ndev);
        std::uint32_t width = 0;
        if (enumerate) {
            std::vector<std::int32_t> cubes;
            // one shared queue: every GPU gets the whole cube list; otherwise cube c
            // runs on GPU (rank * ndev + i) == c % gpus
            const int qrank = dynamic ? 0 : cfg.rank * static_cast<int>(ndev);
            const std::uint32_t total =
                make_cubes(prog, cfg.cube_atoms, cfg.cube_depth, 4 * slots_per_gpu * gpus, 0, 1, cubes, width, auto_cubes);
            for (std::uint32_t i = 0; i < ndev; ++i) {
                DevRun& d = runs[i];
                if (dynamic) {
                    d.cubes = cubes;
                    d.n_cubes = total;
                } else {
                    const std::uint32_t g = static_cast<std::uint32_t>(qrank) + i;
                    for (std::uint32_t c = g; c < total; c += gpus) {
                        d.cubes.insert(d.cubes.end(), cubes.begin() + static_cast<std::ptrdiff_t>(c) * width,
                                       cubes.begin() + static_cast<std::ptrdiff_t>(c + 1) * width);
                        ++d.n_cubes;
                    }
                }
            }
            if (total == 1 && width == 0) {  // no choice atoms: one search, on the first GPU of rank 0
                for (std::uint32_t i = 0; i < ndev; ++i) runs[i].n_cubes = (i == 0 && cfg.rank == 0) ? 1u : 0u;
            }
        } else if (portfolio) {  // one search per variant on every GPU
            for (std::uint32_t i = 0; i < ndev; ++i) runs[i].n_cubes = std::min<std::uint32_t>(cfg.portfolio, static_cast<std::uint32_t>(sms));
        } else {
            runs[0].n_cubes = cfg.rank == 0 ? 1u : 0u;  // a single search runs on rank 0 only
        }
        lap("compiled + cubes");

        const bool many = width > 0;
        const std::uint64_t cap = cfg.learned_capacity;
        const std::uint64_t cap1 = cap == UINT64_MAX ? cap : cap + 1;  // saturating: UINT64_MAX = unbounded
        for (std::uint32_t i = 0; i < ndev; ++i) {
            DevRun& d = runs[i];
            const std::uint32_t gi = static_cast<std::uint32_t>(cfg.rank) * ndev + i;  // GPU index in the fleet
            d.device = devs[i];
            d.dc = dc;
            if (portfolio) {
                d.dc.portfolio = 1;
                d.dc.pf_base = (dc.mode | dc.heur << 1) + gi * cfg.portfolio;
            }
            EngineOptions& eo = d.eo;
            eo.device = devs[i];
            eo.grid = !portfolio && (cfg.engine == 2 || (cfg.engine == 0 && st.size() >= (1u << 18) && width == 0));
            eo.slots = portfolio ? d.n_cubes : slots_per_gpu;
            eo.lcap = static_cast<std::uint32_t>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(cap1, many ? (1u << 13) : (1u << 18))));
            eo.lpool = many ? (1u << 16) : (1u << 22);
            eo.slice_ms = 500.0;
            // the shared block is mapped on this GPU: the home GPU, a peer of it, or this rank's IPC view
            eo.fleet = (shared && (dynamic || portfolio)) ? shared : nullptr;
            eo.fleet_tag = gi << 16;
        }

        auto res = std::make_unique<yas_result>();
        std::uint64_t fleet_vals[4] = {0, 0, 0, 0};
        for (int attempt = 0;; ++attempt) {
            if (shared) {
                if (!fl || fl->owner) reset_fleet_ctl(shared, shared_dev);
                if (fl && fl->comm) {  // nobody starts before rank 0 has reset the queue
                    std::uint64_t b = 0;
                    fl->comm->allreduce(&b, 1, FleetComm::kMax);
                }
            }
            std::atomic<std::uint64_t> found{0};
            std::atomic<std::uint64_t>* first_models = enumerate && cfg.max_models != 0 ? &found : nullptr;
            if (ndev == 1) {
                run_device(runs[0], ep, prog, cfg, width, first_models);
            } else {
                std::vector<std::thread> th;
                for (DevRun& d : runs)
                    th.emplace_back([&, dp = &d] { run_device(*dp, ep, prog, cfg, width, first_models); });
                for (std::thread& t : th) t.join();
            }
            lap("engine");
            std::uint32_t status = dev::kDone;
            std::exception_ptr first_error;
            for (DevRun& d : runs) {
                if (d.error && !first_error) first_error = d.error;
                if (d.er.status != dev::kDone && status == dev::kDone) status = d.er.status;
            }
            bool retry = status == dev::kErrArena && attempt < 8;
            if (fl && fl->comm) {  // every rank retries, or none (the shared queue restarts from 0)
                std::uint64_t v = retry ? 1 : 0;
                fl->comm->allreduce(&v, 1, FleetComm::kMax);
                retry = v != 0 && attempt < 8;
            }
            if (retry) {
                for (DevRun& d : runs) {
                    d.eo.lcap = static_cast<std::uint32_t>(std::min<std::uint64_t>({cap1, 2ull * d.eo.lcap, 0x7FFFFFFFull}));
                    d.eo.lpool *= 2;
                    if (many && d.eo.slots > 64) d.eo.slots /= 2;
                    d.error = nullptr;
                }
                continue;
            }
            // merge: GPUs in order; a portfolio reports the GPU whose search won the claim
            std::vector<std::uint32_t> order;
            int won = -1;
            for (std::uint32_t i = 0; i < ndev; ++i)
                if (runs[i].er.won) won = static_cast<int>(i);
            if (portfolio) {
                if (won >= 0) order.push_back(static_cast<std::uint32_t>(won));
            } else {
                for (std::uint32_t i = 0; i < ndev; ++i) order.push_back(i);
            }
            std::vector<yas_trace> traces;
            for (std::uint32_t i : order) {
                const DevRun& d = runs[i];
                const std::uint64_t base = res->ids.size();
                res->ids.insert(res->ids.end(), d.ids.begin(), d.ids.end());
                for (std::size_t m = 1; m < d.offs.size(); ++m) res->off.push_back(base + d.offs[m]);
                res->cubes.insert(res->cubes.end(), d.mcubes.begin(), d.mcubes.end());
                traces.insert(traces.end(), d.traces.begin(), d.traces.end());
            }
            lap("merged");
            if (enumerate && res->count() > 1) {  // cube order: the same for any scheduling of the cubes
                // stable counting sort by cube
                const std::size_t n = res->count();
                std::uint32_t maxc = 0;
                for (std::uint32_t cu : res->cubes) maxc = std::max(maxc, cu);
                std::vector<std::uint64_t> start(static_cast<std::size_t>(maxc) + 2, 0);
                for (std::uint32_t cu : res->cubes) ++start[static_cast<std::size_t>(cu) + 1];
                for (std::size_t k = 1; k < start.size(); ++k) start[k] += start[k - 1];
                std::vector<std::uint32_t> ord(n);
                for (std::uint32_t m = 0; m < n; ++m) ord[start[res->cubes[m]]++] = m;
                std::vector<std::uint64_t> off(n + 1, 0);
                std::vector<std::uint32_t> cubes(n);
                for (std::size_t i = 0; i < n; ++i) {
                    off[i + 1] = off[i] + (res->off[ord[i] + 1] - res->off[ord[i]]);
                    cubes[i] = res->cubes[ord[i]];
                }
                std::vector<std::uint32_t> ids(off[n]);
                for (std::size_t i = 0; i < n; ++i)
                    std::copy(res->ids.begin() + static_cast<std::ptrdiff_t>(res->off[ord[i]]),
                              res->ids.begin() + static_cast<std::ptrdiff_t>(res->off[ord[i] + 1]),
                              ids.begin() + static_cast<std::ptrdiff_t>(off[i]));
                res->ids.swap(ids);
                res->off.swap(off);
                res->cubes.swap(cubes);
            }
            lap("cube order");
            if (enumerate && cfg.max_models != 0 && res->count() > cfg.max_models) {  // first models: exactly max_models
                res->off.resize(cfg.max_models + 1);
                res->ids.resize(res->off.back());
                res->cubes.resize(cfg.max_models);
            }
            if (fl && fl->comm) {  // the final all-reduce: models, fleet-wide errors, the portfolio winner
                std::uint64_t sum[1] = {res->count()};
                fl->comm->allreduce(sum, 1, FleetComm::kSum);
                std::uint64_t mx[3] = {status != dev::kDone || first_error ? 1u : 0u,
                                       won >= 0 ? static_cast<std::uint64_t>(cfg.rank) + 1 : 0,
                                       won >= 0 && res->count() > 0 ? 1u : 0u};
                fl->comm->allreduce(mx, 3, FleetComm::kMax);
                fleet_vals[0] = sum[0];
                fleet_vals[1] = mx[0];
                fleet_vals[2] = mx[1];
                fleet_vals[3] = mx[2];
            }
            if (first_error) std::rethrow_exception(first_error);
            if (status == dev::kErrArena) throw std::runtime_error("device learned-nogood arena exhausted");
            if (status == dev::kErrCapacity)
                throw CapacityError("learned nogood store capacity exceeded (" + std::to_string(cap) + " nogoods)");
            if (status == dev::kErrLogic) throw std::logic_error("res_learning: literal at conflict level has no antecedent");
            if (status == dev::kErrValidate) throw std::logic_error("fixpoint invariant broken");
            if (cfg.trace)
                for (const yas_trace& t : traces) cfg.trace(&t, cfg.trace_user);
            dev::Stats tot{};
            double dev_ms = 0.0, wall_ms = 0.0;
            std::uint64_t launches = 0, searches = 0;
            for (std::uint32_t i = 0; i < ndev; ++i) {
                const EngineResult& er = runs[i].er;
                const unsigned long long* pb = &er.stats.decisions;
                unsigned long long* pa = &tot.decisions;
                if (!portfolio)
                    for (std::size_t k = 0; k < sizeof(dev::Stats) / 8; ++k) pa[k] += pb[k];
                searches += er.stats.searches;
                dev_ms = std::max(dev_ms, er.device_ms);
                wall_ms = std::max(wall_ms, er.wall_ms);
                launches += er.launches;
            }
            if (portfolio && won >= 0) tot = runs[static_cast<std::size_t>(won)].er.stats;  // the winner's trajectory
            fill_stats(res->stats, tot);
            res->stats.searches = searches;
            res->stats.models = res->count();
            res->stats.wall_ms = wall_ms;
            res->stats.device_ms = dev_ms;
            res->stats.launches = launches;
            res->stats.cubes = portfolio ? 0 : searches;  // cubes this process searched
            res->stats.portfolio_variant = won >= 0 ? runs[static_cast<std::size_t>(won)].er.variant : -1;
            res->stats.devices = ndev;
            res->stats.fleet_ranks = static_cast<std::uint32_t>(cfg.world);
            if (fl && fl->comm) {
                res->stats.fleet_models = fleet_vals[0];
                res->stats.fleet_winner = portfolio ? static_cast<std::int32_t>(fleet_vals[2]) - 1 : -1;
                res->status = portfolio ? (fleet_vals[3] ? 0 : 1) : (fleet_vals[0] ? 0 : 1);
            } else {
                res->stats.fleet_models = res->count();
                res->stats.fleet_winner = portfolio && won >= 0 ? 0 : -1;
                res->status = res->count() == 0 ? 1 : 0;
            }
            lap("result");
            break;
        }
        *out = res.release();
        return static_cast<int>(YAS_OK);
    });
}

namespace {

// Collectives through caller-supplied functions (e.g. torch.distributed or MPI).
class CallbackComm final : public FleetComm {
public:
    CallbackComm(yas_allreduce_fn ar, yas_broadcast_fn bc, void* user) : ar_(ar), bc_(bc), user_(user) {}
    void allreduce(std::uint64_t* vals, std::size_t n, Op op) override {
        if (ar_(vals, n, static_cast<int>(op), user_) != 0) throw std::runtime_error("fleet all-reduce callback failed");
    }
    void broadcast(void* buf, std::size_t bytes, int root) override {
        if (bc_(buf, bytes, root, user_) != 0) throw std::runtime_error("fleet broadcast callback failed");
    }

private:
    yas_allreduce_fn ar_;
    yas_broadcast_fn bc_;
    void* user_;
};

// Rank 0 allocates the shared block; its CUDA IPC handle goes to every rank,
// which maps it (NVLink peer access across processes). If any rank cannot,
// every rank keeps a private block and the cubes are dealt statically.
void fleet_attach(yas_fleet& f) {
    ck_cuda(cudaSetDevice(f.device), "cudaSetDevice");
    cudaIpcMemHandle_t h{};
    if (f.rank == 0) {
        ck_cuda(cudaMalloc(&f.ctl, sizeof(dev::Fleet)), "cudaMalloc fleet");
        f.owner = true;
        if (f.world > 1) ck_cuda(cudaIpcGetMemHandle(&h, f.ctl), "cudaIpcGetMemHandle");
    }
    if (f.world == 1) {
        f.dynamic = true;
        return;
    }
    f.comm->broadcast(&h, sizeof h, 0);
    std::uint64_t ok = 1;
    if (f.rank != 0) {
        void* ptr = nullptr;
        if (cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) {
            f.ctl = static_cast<dev::Fleet*>(ptr);
            f.ipc = true;
        } else {
            cudaGetLastError();
            ok = 0;
        }
    }
    f.comm->allreduce(&ok, 1, FleetComm::kMin);
    f.dynamic = ok == 1;
    if (!f.dynamic && f.rank != 0) {  // private block: portfolio stop within this rank only
        if (f.ipc) cudaIpcCloseMemHandle(f.ctl);
        f.ipc = false;
        ck_cuda(cudaMalloc(&f.ctl, sizeof(dev::Fleet)), "cudaMalloc fleet");
        f.owner = true;
    }
}

int fleet_make(int rank, int world, int device, std::unique_ptr<FleetComm> (*make)(void*), void* arg, yas_fleet** out,
               char* err, size_t cap) {
    if (!out) return YAS_ERR_ARG;
    *out = nullptr;
    return guarded(err, cap, [&] {
        if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("fleet: rank must be in [0, world)");
        require_device(device);
        auto f = std::make_unique<yas_fleet>();
        f->rank = rank;
        f->world = world;
        f->device = device;
        f->comm = make(arg);
        fleet_attach(*f);
        *out = f.release();
        return static_cast<int>(YAS_OK);
    });
}

}  // namespace

int yas_fleet_unique_id(uint8_t out[128], char* err, size_t err_cap) {
    if (!out) return YAS_ERR_ARG;
    return guarded(err, err_cap, [&] {
        require_device(0);
        nccl_unique_id(out);
        return static_cast<int>(YAS_OK);
    });
}

int yas_fleet_create_nccl(const uint8_t unique_id[128], int rank, int world, int device, yas_fleet** out, char* err,
                          size_t err_cap) {
    if (!unique_id) return YAS_ERR_ARG;
    struct A {
        const uint8_t* id;
        int rank, world, device;
    } a{unique_id, rank, world, device};
    return fleet_make(rank, world, device,
                      [](void* p) {
                          const A& x = *static_cast<const A*>(p);
                          return nccl_comm(x.id, x.rank, x.world, x.device);
                      },
                      &a, out, err, err_cap);
}

int yas_fleet_create(int rank, int world, int device, yas_allreduce_fn allreduce, yas_broadcast_fn broadcast, void* user,
                     yas_fleet** out, char* err, size_t err_cap) {
    if (!allreduce || !broadcast) return YAS_ERR_ARG;
    struct A {
        yas_allreduce_fn ar;
        yas_broadcast_fn bc;
        void* user;
    } a{allreduce, broadcast, user};
    return fleet_make(rank, world, device,
                      [](void* p) -> std::unique_ptr<FleetComm> {
                          const A& x = *static_cast<const A*>(p);
                          return std::make_unique<CallbackComm>(x.ar, x.bc, x.user);
                      },
                      &a, out, err, err_cap);
}

void yas_fleet_free(yas_fleet* f) {
    if (!f) return;
    cudaSetDevice(f->device);
    if (f->ipc) cudaIpcCloseMemHandle(f->ctl);
    else if (f->owner && f->ctl) cudaFree(f->ctl);
    delete f;
}

int yas_fleet_info(const yas_fleet* f, int* rank, int* world, int* device, int* dynamic) {
    if (!f) return YAS_ERR_ARG;
    if (rank) *rank = f->rank;
    if (world) *world = f->world;
    if (device) *device = f->device;
    if (dynamic) *dynamic = f->dynamic ? 1 : 0;
    return YAS_OK;
}

int yas_fleet_allreduce(yas_fleet* f, uint64_t* vals, size_t n, int op, char* err, size_t err_cap) {
    if (!f || (n && !vals) || op < 0 || op > 2) return YAS_ERR_ARG;
    return guarded(err, err_cap, [&] {
        f->comm->allreduce(vals, n, static_cast<FleetComm::Op>(op));
        return static_cast<int>(YAS_OK);
    });
}

int yas_result_status(const yas_result* r) { return r ? r->status : 1; }
uint64_t yas_result_model_count(const yas_result* r) { return r ? r->count() : 0; }
const uint32_t* yas_result_model(const yas_result* r, uint64_t m, uint32_t* n) {
    if (!r || m >= r->count()) {
        if (n) *n = 0;
        return nullptr;
    }
    if (n) *n = static_cast<uint32_t>(r->off[m + 1] - r->off[m]);
    return r->ids.data() + r->off[m];
}
size_t yas_result_models_flat(const yas_result* r, uint32_t* ids, size_t cap, uint64_t* offsets, uint32_t* cubes) {
    if (!r) return 0;
    const std::size_t total = r->ids.size(), n = r->count();
    if (ids) std::memcpy(ids, r->ids.data(), std::min(cap, total) * sizeof(uint32_t));
    if (offsets) std::memcpy(offsets, r->off.data(), (n + 1) * sizeof(uint64_t));
    if (cubes)
        for (std::size_t m = 0; m < n; ++m) cubes[m] = m < r->cubes.size() ? r->cubes[m] : 0;
    return total;
}
uint32_t yas_result_model_cube(const yas_result* r, uint64_t m) {
    return r && m < r->cubes.size() ? r->cubes[m] : 0;
}
void yas_result_stats(const yas_result* r, yas_stats* s) {
    if (r && s) *s = r->stats;
}
void yas_result_free(yas_result* r) { delete r; }

size_t yas_stats_csv_header(char* buf, size_t cap) {
    return put_text(
        "instance,mode,heuristic,workers,status,models,decisions,propagations,conflicts,learned,avg_learned_len,"
        "restarts,wall_ms,props_per_sec,decisions_per_sec,learned_per_sec",
        buf, cap);
}

size_t yas_emit_stats(const yas_stats* s, const char* instance, const char* mode, const char* heur, unsigned workers,
                      int status, uint64_t models, int csv, char* buf, size_t cap) {
    // SolveStats rates and emit_stats formatting (solver.hpp:80-92, solver.cpp:336-360)
    const double avg = s->learned_count ? static_cast<double>(s->learned_length_sum) / static_cast<double>(s->learned_count) : 0.0;
    auto rate = [&](uint64_t c) { return s->wall_ms <= 0.0 ? 0.0 : static_cast<double>(c) / (s->wall_ms / 1000.0); };
    const char* st = status == 0 ? "SAT" : "UNSAT";
    std::ostringstream o;
    if (csv) {
        o << (instance ? instance : "") << ',' << (mode ? mode : "") << ',' << (heur ? heur : "") << ',' << workers << ','
          << st << ',' << models << ',' << s->decisions << ',' << s->propagations << ',' << s->conflicts << ','
          << s->learned_count << ',' << avg << ',' << s->restarts << ',' << s->wall_ms << ',' << rate(s->propagations)
          << ',' << rate(s->decisions) << ',' << rate(s->learned_count);
    } else {
        o << "instance       : " << (instance ? instance : "") << '\n'
          << "mode/heuristic : " << (mode ? mode : "") << '/' << (heur ? heur : "") << " (workers " << workers << ")\n"
          << "status         : " << st << '\n'
          << "models         : " << models << '\n'
          << "decisions      : " << s->decisions << " (" << rate(s->decisions) << "/s)\n"
          << "propagations   : " << s->propagations << " (" << rate(s->propagations) << "/s)\n"
          << "conflicts      : " << s->conflicts << '\n'
          << "learned        : " << s->learned_count << " (" << rate(s->learned_count) << "/s, avg len " << avg << ")\n"
          << "restarts       : " << s->restarts << '\n'
          << "wall time      : " << s->wall_ms << " ms";
    }
    return put_text(o.str(), buf, cap);
}

int yas_store_build(const int32_t* lits, const uint32_t* offsets, size_t n, const uint32_t* guards,
                    const uint8_t* origins, uint32_t total_atoms, yas_store** out, char* err, size_t err_cap) {
    if (!out) return YAS_ERR_ARG;
    *out = nullptr;
    return guarded(err, err_cap, [&] {
        NogoodSet ngs;
        for (size_t k = 0; k < n; ++k) {
            std::vector<std::int32_t> l(lits + offsets[k], lits + offsets[k + 1]);
            for (std::int32_t x : l)
                if (x == 0 || lit_atom(x) > total_atoms) throw std::invalid_argument("literal out of range");
            auto ng = Nogood::make(std::move(l), origins ? origins[k] : static_cast<std::uint8_t>(kConstraint), guards ? guards[k] : kAnyTruth);
            if (!ng || ng->lits.empty()) throw std::invalid_argument("vacuous or empty nogood " + std::to_string(k));
            ngs.push(*ng);
        }
        auto s = std::make_unique<yas_store>();
        s->st = build_store(ngs, total_atoms);
        *out = s.release();
        return static_cast<int>(YAS_OK);
    });
}

void yas_store_free(yas_store* s) { delete s; }
uint32_t yas_store_size(const yas_store* s) { return s ? s->st.size() : 0; }
uint32_t yas_store_total_atoms(const yas_store* s) { return s ? s->st.total_atoms : 0; }
size_t yas_store_dump_csv(const yas_store* s, char* buf, size_t cap) { return s ? put_text(s->st.dump_csv(), buf, cap) : 0; }
size_t yas_store_nogood(const yas_store* s, uint32_t id, int32_t* lits, size_t cap, uint32_t* guard, uint8_t* origin) {
    if (!s || id >= s->st.size()) return 0;
    const std::uint32_t lo = s->st.off[id], len = s->st.off[id + 1] - lo;
    for (std::uint32_t k = 0; k < len && lits && k < cap; ++k) lits[k] = s->st.pool[lo + k];
    if (guard) *guard = s->st.guard[id];
    if (origin) *origin = id < s->st.origin.size() ? s->st.origin[id] : 1;
    return len;
}

size_t yas_store_units(const yas_store* s, int32_t* out, size_t cap) {
    if (!s) return 0;
    for (size_t i = 0; i < s->st.units.size() && i < cap; ++i) out[i] = s->st.units[i];
    return s->st.units.size();
}
size_t yas_store_unit_ids(const yas_store* s, int32_t* out, size_t cap) {
    if (!s) return 0;
    for (size_t i = 0; i < s->st.unit_ids.size() && i < cap; ++i) out[i] = s->st.unit_ids[i];
    return s->st.unit_ids.size();
}
void yas_store_bounds(const yas_store* s, uint32_t out[4]) {
    for (int i = 0; i < 4; ++i) out[i] = s ? s->st.bounds[i] : 0;
}
size_t yas_store_occurrences(const yas_store* s, int32_t lit, uint32_t cls, int32_t* out, size_t cap) {
    if (!s || cls > 3 || lit == 0 || lit_atom(lit) > s->st.total_atoms) return 0;
    const std::uint32_t key = lit_index(lit) * 4 + cls;
    const std::uint32_t lo = s->st.occ_off[key], hi = s->st.occ_off[key + 1];
    for (std::uint32_t i = lo; i < hi && i - lo < cap; ++i) out[i - lo] = s->st.occ_ids[i];
    return hi - lo;
}

int yas_store_planted(uint32_t atoms, uint64_t count, uint32_t pct, uint64_t seed, yas_store** out, int32_t** seeded,
                      size_t* n_seeded, int32_t* decision) {
    if (!out || atoms < 2) return YAS_ERR_ARG;
    // SplitMix64 stream as in /root/reference/proj/tests/support/gen.hpp:16-29.
    std::uint64_t state = seed;
    auto next = [&]() {
        std::uint64_t z = (state += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    };
    auto below = [&](std::uint64_t n) { return n == 0 ? 0 : next() % n; };
    std::vector<std::uint8_t> h(atoms + 1, 0);
    for (uint32_t a = 1; a <= atoms; ++a) h[a] = below(100) < 50 ? 1 : 0;
    auto hlit = [&](uint32_t a) { return h[a] ? static_cast<std::int32_t>(a) : -static_cast<std::int32_t>(a); };
    NogoodSet ngs;
    while (ngs.size() < count) {
        const uint32_t len = 2 + static_cast<uint32_t>(below(5));
        std::vector<std::int32_t> l;
        for (uint32_t k = 0; k < len; ++k) {
            const std::int32_t a = static_cast<std::int32_t>(1 + below(atoms));
            l.push_back(below(100) < 50 ? a : -a);
        }
        l[0] = -hlit(lit_atom(l[0]));
        if (auto ng = Nogood::make(std::move(l), kConstraint)) ngs.push(*ng);
    }
    std::vector<std::int32_t> sd;
    for (uint32_t a = 2; a <= atoms; ++a)
        if (below(100) < pct) sd.push_back(hlit(a));
    auto s = std::make_unique<yas_store>();
    s->st = build_store(ngs, atoms);
    *out = s.release();
    if (decision) *decision = hlit(1);
    if (seeded && n_seeded) {
        *n_seeded = sd.size();
        *seeded = static_cast<int32_t*>(std::malloc(std::max<size_t>(1, sd.size()) * sizeof(int32_t)));
        std::copy(sd.begin(), sd.end(), *seeded);
    }
    return YAS_OK;
}

void yas_free_ints(int32_t* p) { std::free(p); }

int yas_propagator_create(const yas_store* s, uint32_t deps_words, int engine, int device, yas_propagator** out,
                          char* err, size_t err_cap) {
    if (!s || !out) return YAS_ERR_ARG;
    *out = nullptr;
    return guarded(err, err_cap, [&] {
        require_device(device);
        if (deps_words < 1 || deps_words > 1024) throw std::invalid_argument("deps_words must be in [1, 1024]");
        auto p = std::make_unique<yas_propagator>();
        const bool grid = engine == 2 || (engine == 0 && s->st.size() >= (1u << 18));
        p->s = std::make_unique<Session>(s->st, deps_words, grid, device);
        p->atoms = s->st.total_atoms;
        *out = p.release();
        return static_cast<int>(YAS_OK);
    });
}

void yas_propagator_free(yas_propagator* p) { delete p; }

// Counter deltas of the last propagation op (the device snapshots the
// counters when the op starts, so no read-back is needed before the launch and
// the recorded state-changing calls run in the same kernel).
static void outcome_from(yas_propagator* p, bool violated, yas_outcome* o) {
    if (!o) return;
    const dev::Ctl& c = p->s->ctl();
    o->violated = violated ? 1 : 0;
    o->propagations = c.st.propagations - c.opsnap[0];
    o->passes = c.st.passes - c.opsnap[1];
    o->checks = c.st.checks - c.opsnap[2];
    o->checked_lits = c.st.checked_lits - c.opsnap[3];
    o->n_conflicts = c.n_confl;
    o->device_ms = p->s->last_ms();
}

int yas_propagator_flush(yas_propagator* p) {
    if (!p) return YAS_ERR_ARG;
    return guarded(p->err, sizeof p->err, [&] { p->s->flush(); return static_cast<int>(YAS_OK); });
}
int yas_propagator_reset(yas_propagator* p) {
    if (!p) return YAS_ERR_ARG;
    return guarded(p->err, sizeof p->err, [&] { p->s->reset(); return static_cast<int>(YAS_OK); });
}
int yas_propagator_initial(yas_propagator* p, yas_outcome* o) {
    if (!p) return YAS_ERR_ARG;
    return guarded(p->err, sizeof p->err, [&] {
        const bool v = p->s->initial_propagation();
        outcome_from(p, v, o);
        return static_cast<int>(YAS_OK);
    });
}
int yas_propagator_propagate(yas_propagator* p, uint32_t level, yas_outcome* o) {
    if (!p) return YAS_ERR_ARG;
    return guarded(p->err, sizeof p->err, [&] {
        const bool v = p->s->propagate(level);
        outcome_from(p, v, o);
        return static_cast<int>(YAS_OK);
    });
}
int yas_propagator_push_decision(yas_propagator* p, int32_t lit) {
    if (!p) return YAS_ERR_ARG;
    return guarded(p->err, sizeof p->err, [&] { p->s->push_decision(lit); return static_cast<int>(YAS_OK); });
}
int yas_propagator_assign(yas_propagator* p, const int32_t* lits, size_t n, uint32_t level, const uint64_t* deps,
                          uint32_t n_deps, int overflow, int32_t antecedent) {
    if (!p || (n && !lits)) return YAS_ERR_ARG;
    return guarded(p->err, sizeof p->err, [&] {
        p->s->assign(lits, n, level, antecedent, reinterpret_cast<const unsigned long long*>(deps), deps ? n_deps : 0,
                     overflow != 0);
        return static_cast<int>(YAS_OK);
    });
}
int yas_propagator_seed(yas_propagator* p, const int32_t* lits, size_t n) {
    if (!p) return YAS_ERR_ARG;
    return guarded(p->err, sizeof p->err, [&] { p->s->seed(lits, n); return static_cast<int>(YAS_OK); });
}
int yas_propagator_transfers(const yas_propagator* p, uint64_t* h2d, uint64_t* d2h) {
    if (!p) return YAS_ERR_ARG;
    unsigned long long a = 0, b = 0;
    p->s->transfers(a, b);
    if (h2d) *h2d = a;
    if (d2h) *d2h = b;
    return YAS_OK;
}
int yas_propagator_clear_frontier(yas_propagator* p) {
    if (!p) return YAS_ERR_ARG;
    return guarded(p->err, sizeof p->err, [&] { p->s->clear_frontier(); return static_cast<int>(YAS_OK); });
}
int32_t yas_propagator_add_learned(yas_propagator* p, const int32_t* lits, size_t n) {
    if (!p || (n && !lits)) return -1;
    int32_t id = -1;
    guarded(p->err, sizeof p->err, [&] { id = p->s->add_learned(std::vector<std::int32_t>(lits, lits + n)); return 0; });
    return id;
}
size_t yas_propagator_last_error(const yas_propagator* p, char* buf, size_t cap) {
    return p ? put_text(p->err, buf, cap) : 0;
}
int yas_propagator_count_literals(yas_propagator* p, int on) {
    if (!p) return YAS_ERR_ARG;
    p->s->set_count_lits(on != 0);
    return YAS_OK;
}
uint32_t yas_propagator_atoms(const yas_propagator* p) { return p ? p->atoms : 0; }
int yas_propagator_pass_trace(yas_propagator* p, int on, uint64_t* out, size_t cap, uint32_t* blocks) {
    if (!p) return YAS_ERR_ARG;
    return guarded(p->err, sizeof p->err, [&] {
        if (on >= 0) p->s->set_pass_trace(on != 0);
        if (out) {
            std::uint32_t b = 0;
            const auto v = p->s->pass_trace(b);
            for (size_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
            if (blocks) *blocks = b;
        }
        return static_cast<int>(YAS_OK);
    });
}
int yas_propagator_profile(const yas_propagator* p, uint64_t out[16]) {
    if (!p || !out) return YAS_ERR_ARG;
    return guarded(const_cast<yas_propagator*>(p)->err, sizeof p->err, [&] {
        const dev::Ctl& c = p->s->ctl();
        for (int k = 0; k < 16; ++k) out[k] = c.prof[k];
        return static_cast<int>(YAS_OK);
    });
}
// Read-backs: a CUDA failure leaves the message in yas_propagator_last_error;
// the size_t variants then return 0.
}  // extern "C"
namespace {
yas_propagator* mut(const yas_propagator* p) { return const_cast<yas_propagator*>(p); }
template <class F>
size_t guarded_size(const yas_propagator* p, F&& f) {
    size_t n = 0;
    if (guarded(mut(p)->err, sizeof p->err, [&] { n = f(); return static_cast<int>(YAS_OK); }) != YAS_OK) return 0;
    return n;
}
}  // namespace
extern "C" {
uint32_t yas_propagator_level(const yas_propagator* p) {
    return p ? static_cast<uint32_t>(guarded_size(p, [&] { return static_cast<size_t>(p->s->ctl().cdl); })) : 0;
}
int yas_propagator_cells(const yas_propagator* p, int32_t* out) {
    if (!p || !out) return YAS_ERR_ARG;
    return guarded(mut(p)->err, sizeof p->err, [&] {
        const auto v = p->s->cells();
        std::copy(v.begin(), v.end(), out);
        return static_cast<int>(YAS_OK);
    });
}
int yas_propagator_reasons(const yas_propagator* p, int32_t* out) {
    if (!p || !out) return YAS_ERR_ARG;
    return guarded(mut(p)->err, sizeof p->err, [&] {
        const auto v = p->s->reasons();
        std::copy(v.begin(), v.end(), out);
        return static_cast<int>(YAS_OK);
    });
}
int yas_propagator_deps(const yas_propagator* p, uint32_t word, uint64_t* out, uint8_t* overflow) {
    if (!p || !out || word >= p->s->deps_words()) return YAS_ERR_ARG;
    return guarded(mut(p)->err, sizeof p->err, [&] {
        const auto v = p->s->deps_word(word);
        std::copy(v.begin(), v.end(), out);
        if (overflow) {
            const auto o = p->s->deps_overflow();
            std::copy(o.begin(), o.end(), overflow);
        }
        return static_cast<int>(YAS_OK);
    });
}
size_t yas_propagator_trail(const yas_propagator* p, int32_t* out, size_t cap) {
    return p ? guarded_size(p, [&] { return p->s->trail_into(out, cap); }) : 0;
}
size_t yas_propagator_conflicts(const yas_propagator* p, int32_t* out, size_t cap) {
    return p ? guarded_size(p, [&] {
        const auto v = p->s->conflicts();
        for (size_t i = 0; i < v.size() && out && i < cap; ++i) out[i] = v[i];
        return v.size();
    }) : 0;
}
size_t yas_propagator_frontier(const yas_propagator* p, int32_t* out, size_t cap) {
    return p ? guarded_size(p, [&] {
        const auto v = p->s->frontier();
        for (size_t i = 0; i < v.size() && out && i < cap; ++i) out[i] = v[i];
        return v.size();
    }) : 0;
}

}  // extern "C"
