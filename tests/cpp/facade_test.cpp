// Reference-API conformance of the C++ facade, written against the reference's
// own names and include paths (aspine/*.hpp) and built with only
//   g++ -std=c++20 -I include tests/cpp/facade_test.cpp -L<lib dir> -lyasmin_b200
// Cases follow the reference's unit tests case by case:
//   /root/reference/proj/tests/test_propagate.cpp:28-154,291-309 (propagation),
//   test_store.cpp:40-75 (CSR layout), test_solver.cpp:42-110 (solve),
//   test_program.cpp (program model), plus a randomized fixpoint-vs-closure
//   check in the manner of test_propagate.cpp:190-235.
// Needs a CUDA device (propagation and solving run on the GPU). Exit code 0 =
// every check passed; failures are printed with their line.
#include <cstdio>
#include <random>
#include <set>
#include <sstream>

#include "aspine/oracle.hpp"
#include "aspine/propagate.hpp"
#include "aspine/solver.hpp"

using namespace aspine;

namespace {

int g_checks = 0, g_failed = 0;
#define EXPECT(cond)                                                             \
    do {                                                                         \
        ++g_checks;                                                              \
        if (!(cond)) {                                                           \
            ++g_failed;                                                          \
            std::fprintf(stderr, "%s:%d: check failed: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                        \
    } while (0)

Nogood ng(std::vector<Lit> lits) { return *Nogood::make(std::move(lits), NogoodOrigin::constraint); }

std::vector<Lit> assigned(const Assignment& a) {
    std::vector<Lit> out;
    for (AtomId x = 1; x <= a.atom_count(); ++x)
        if (a.cell(x) != 0) out.push_back(a.cell(x) > 0 ? Lit::pos(x) : Lit::neg(x));
    return out;
}

std::set<std::vector<AtomId>> family(const SolveResult& r) {
    std::set<std::vector<AtomId>> f;
    for (const Model& m : r.models) f.insert(m.atom_ids);
    return f;
}

void propagation_cases() {
    {  // units force their complements at level 1
        StoreBuild b = NogoodStore::build({ng({Lit::pos(1)}), ng({Lit::pos(2)})}, 2);
        WorkerPool pool(1);
        Propagator prop(b.store, pool);
        Assignment a(2, 1);
        Frontier f;
        PropagationOutcome out = prop.initial_propagation(a, f);
        EXPECT(!out.violated && a.cell(1) == -1 && a.cell(2) == -1 && out.propagations == 2 && f.last.size() == 2);
    }
    {  // inconsistent units: a pseudo-id conflict
        StoreBuild b = NogoodStore::build({ng({Lit::pos(1)}), ng({Lit::neg(1)})}, 1);
        WorkerPool pool(1);
        Propagator prop(b.store, pool);
        Assignment a(1, 1);
        Frontier f;
        PropagationOutcome out = prop.initial_propagation(a, f);
        EXPECT(out.violated && out.conflicts.size() == 1 && is_unit_pseudo_id(out.conflicts[0]));
    }
    {  // learned units are replayed, idempotently
        StoreBuild b = NogoodStore::build({ng({Lit::pos(1), Lit::pos(2)})}, 3);
        const NogoodId learned = b.store.add_learned(*Nogood::make({Lit::pos(3)}, NogoodOrigin::learned, kNoTruth));
        EXPECT(b.store.learned_unit_ids() == std::vector<NogoodId>{learned});
        WorkerPool pool(1);
        Propagator prop(b.store, pool);
        Assignment a(3, 1);
        Frontier f;
        PropagationOutcome out = prop.initial_propagation(a, f);
        EXPECT(!out.violated && a.has(Lit::neg(3)) && a.level_of(3) == 1);
        Frontier f2;
        PropagationOutcome again = prop.initial_propagation(a, f2);
        EXPECT(!again.violated && f2.last.empty());
    }
    {  // no units, no work
        StoreBuild b = NogoodStore::build({ng({Lit::pos(1), Lit::pos(2)})}, 2);
        WorkerPool pool(1);
        Propagator prop(b.store, pool);
        Assignment a(2, 1);
        Frontier f;
        EXPECT(!prop.initial_propagation(a, f).violated && a.trail().empty());
    }
    {  // unit propagation: level, reason, Deps copied from the trigger
        StoreBuild b = NogoodStore::build({ng({Lit::pos(1), Lit::pos(2)})}, 2);
        WorkerPool pool(1);
        Propagator prop(b.store, pool);
        Assignment a(2, 2);
        Frontier f;
        a.push_decision(Lit::pos(1));
        f.seed(Lit::pos(1));
        PropagationOutcome out = prop.propagate_and_check(a, f, a.decision_level());
        EXPECT(!out.violated && a.has(Lit::neg(2)) && a.level_of(2) == 2);
        EXPECT(a.reason(2).kind == Reason::propagated && a.reason(2).antecedent == 0);
        std::vector<std::uint64_t> d1(a.deps().of(1).begin(), a.deps().of(1).end());
        std::vector<std::uint64_t> d2(a.deps().of(2).begin(), a.deps().of(2).end());
        EXPECT(d1 == d2 && out.propagations == 1);
    }
    {  // a satisfied nogood does nothing
        StoreBuild b = NogoodStore::build({ng({Lit::pos(1), Lit::neg(2)})}, 2);
        WorkerPool pool(1);
        Propagator prop(b.store, pool);
        Assignment a(2, 1);
        Frontier f;
        a.push_decision(Lit::pos(1));
        a.assign_propagated(Lit::pos(2), 2, std::vector<std::uint64_t>{0}, false, 0);
        f.seed(Lit::pos(1));
        PropagationOutcome out = prop.propagate_and_check(a, f, 2);
        EXPECT(!out.violated && out.propagations == 0);
    }
    {  // a fully assigned nogood is a conflict
        StoreBuild b = NogoodStore::build({ng({Lit::pos(1), Lit::pos(2), Lit::pos(3)})}, 3);
        WorkerPool pool(1);
        Propagator prop(b.store, pool);
        Assignment a(3, 1);
        Frontier f;
        a.push_decision(Lit::pos(1));
        a.push_decision(Lit::pos(2));
        a.assign_propagated(Lit::pos(3), 3, std::vector<std::uint64_t>{0b100}, false, 0);
        f.seed(Lit::pos(3));
        PropagationOutcome out = prop.propagate_and_check(a, f, 3);
        EXPECT(out.violated && out.conflicts.size() == 1 && out.conflicts[0] == 0);
    }
    for (unsigned workers : {1u, 2u}) {  // race: the first proposal in item order wins
        StoreBuild b = NogoodStore::build({ng({Lit::pos(1), Lit::pos(2)}), ng({Lit::pos(1), Lit::neg(2)})}, 2);
        WorkerPool pool(workers);
        Propagator prop(b.store, pool);
        Assignment a(2, 1);
        Frontier f;
        a.push_decision(Lit::pos(1));
        f.seed(Lit::pos(1));
        PropagationOutcome out = prop.propagate_and_check(a, f, 2);
        EXPECT(out.violated && a.has(Lit::neg(2)) && out.conflicts.size() == 1 && out.conflicts[0] == 1);
    }
    {  // chain T1 -> F2 -> T3 -> F4: a pass per link
        StoreBuild b = NogoodStore::build(
            {ng({Lit::pos(1), Lit::pos(2)}), ng({Lit::neg(2), Lit::neg(3)}), ng({Lit::pos(3), Lit::pos(4)})}, 4);
        WorkerPool pool(1);
        Propagator prop(b.store, pool);
        Assignment a(4, 1);
        Frontier f;
        a.push_decision(Lit::pos(1));
        f.seed(Lit::pos(1));
        PropagationOutcome out = prop.propagate_and_check(a, f, 2);
        EXPECT(!out.violated && out.propagations == 3 && out.passes >= 3);
        EXPECT(a.has(Lit::neg(2)) && a.has(Lit::pos(3)) && a.has(Lit::neg(4)));
    }
    {  // mk_dl_bitmap ORs the other literals' rows, skipping level-1 atoms
        Assignment b(4, 1);
        b.push_decision(Lit::pos(4));
        b.push_decision(Lit::pos(3));
        b.assign_propagated(Lit::pos(1), 3, std::vector<std::uint64_t>{0b0101}, false, 0);
        b.assign_propagated(Lit::neg(2), 3, std::vector<std::uint64_t>{0b0011}, false, 0);
        std::vector<Lit> delta{Lit::pos(1), Lit::neg(2), Lit::pos(4)};
        auto [bits, ovf] = Propagator::mk_dl_bitmap(delta, Lit::pos(4), b);
        EXPECT(!ovf && bits.size() == 1 && bits[0] == 0b0111);
        Assignment u(3, 1);
        u.assign_unit(Lit::pos(1));
        u.assign_unit(Lit::neg(2));
        std::vector<Lit> d2{Lit::pos(1), Lit::neg(2), Lit::pos(3)};
        auto [bits2, ovf2] = Propagator::mk_dl_bitmap(d2, Lit::neg(3), u);
        EXPECT(!ovf2 && !bitmap_any(bits2));
    }
}

// Fixpoint of the device equals a rescan-until-stable closure (our own), over
// random stores, with one decision on top; Deps of every propagated atom equal
// mk_dl_bitmap of its antecedent (the replay audit), across many decisions.
void random_stores() {
    std::mt19937_64 rng(0xc105e001);
    auto below = [&](std::uint64_t n) { return static_cast<std::uint32_t>(rng() % n); };
    int conflicts = 0;
    for (int iter = 0; iter < 120; ++iter) {
        std::vector<Nogood> in;
        const unsigned count = 1 + below(20);
        while (in.size() < count) {
            std::vector<Lit> lits;
            for (unsigned k = 0, len = 1 + below(4); k < len; ++k) {
                const AtomId x = 1 + below(10);
                lits.push_back(below(2) ? Lit::pos(x) : Lit::neg(x));
            }
            if (auto n = Nogood::make(lits, NogoodOrigin::constraint)) in.push_back(*n);
        }
        StoreBuild b = NogoodStore::build(in, 10);
        WorkerPool pool(1);
        Propagator prop(b.store, pool);
        Assignment a(10, 1);
        Frontier f;
        bool violated = prop.initial_propagation(a, f).violated;
        if (!violated) violated = prop.propagate_and_check(a, f, 1).violated;
        std::vector<Lit> seed;
        for (AtomId x = 1; x <= 10 && !violated; ++x)
            if (a.unassigned(x)) {
                a.push_decision(Lit::pos(x));
                seed.push_back(Lit::pos(x));
                f.clear();
                f.seed(Lit::pos(x));
                violated = prop.propagate_and_check(a, f, 2).violated;
                break;
            }
        // closure: units' complements + seed, rescanning every nogood until stable
        std::vector<int> val(11, 0);
        bool clash = false;
        auto put = [&](Lit l) {
            const int v = l.positive() ? 1 : -1;
            if (val[l.atom()] == -v) clash = true;
            const bool fresh = val[l.atom()] == 0;
            if (fresh) val[l.atom()] = v;
            return fresh;
        };
        for (Lit l : seed) put(l);
        for (Lit u : b.store.static_units()) put(~u);
        for (bool grew = true; grew && !clash;) {
            grew = false;
            for (NogoodId id = 0; id < static_cast<NogoodId>(b.store.size()) && !clash; ++id) {
                int hold = 0, open = 0;
                bool dead = false;
                Lit last;
                for (Lit l : b.store.literals(id)) {
                    const int v = val[l.atom()];
                    if (v == 0) { ++open; last = l; }
                    else if ((v > 0) == l.positive()) ++hold;
                    else dead = true;
                }
                if (dead) continue;
                if (open == 0) clash = true;
                else if (open == 1) grew |= put(~last);
            }
        }
        EXPECT(clash == violated);
        if (violated) {
            ++conflicts;
            continue;
        }
        std::vector<Lit> want;
        for (AtomId x = 1; x <= 10; ++x)
            if (val[x]) want.push_back(val[x] > 0 ? Lit::pos(x) : Lit::neg(x));
        EXPECT(want == assigned(a));
        std::string why;
        EXPECT(validate_fixpoint(b.store, a, &why));
    }
    EXPECT(conflicts > 5);
    for (int iter = 0; iter < 40; ++iter) {  // replay audit over a chain of decisions
        std::vector<Nogood> in;
        while (in.size() < 2 + below(16)) {
            std::vector<Lit> lits;
            for (unsigned k = 0, len = 1 + below(4); k < len; ++k) {
                const AtomId x = 1 + below(8);
                lits.push_back(below(2) ? Lit::pos(x) : Lit::neg(x));
            }
            if (auto n = Nogood::make(lits, NogoodOrigin::constraint)) in.push_back(*n);
        }
        StoreBuild b = NogoodStore::build(in, 8);
        WorkerPool pool(1);
        Propagator prop(b.store, pool);
        Assignment a(8, 1);
        Frontier f;
        if (prop.initial_propagation(a, f).violated || prop.propagate_and_check(a, f, 1).violated) continue;
        for (;;) {
            AtomId pick = 0;
            for (AtomId x = 1; x <= 8 && !pick; ++x)
                if (a.unassigned(x)) pick = x;
            if (!pick) break;
            const Lit d = below(2) ? Lit::pos(pick) : Lit::neg(pick);
            a.push_decision(d);
            f.clear();
            f.seed(d);
            if (prop.propagate_and_check(a, f, a.decision_level()).violated) break;
        }
        for (const auto& e : a.trail()) {
            const Reason r = a.reason(e.lit.atom());
            if (r.kind != Reason::propagated) continue;
            auto [bits, ovf] = Propagator::mk_dl_bitmap(b.store.literals(r.antecedent), e.lit, a);
            EXPECT(std::equal(bits.begin(), bits.end(), a.deps().of(e.lit.atom()).begin()));
            EXPECT(ovf == a.deps().overflow(e.lit.atom()));
        }
        // a backjump and further decisions: the facade replays the trail on the device
        if (a.decision_level() > 2) {
            a.backjump(2);
            f.clear();
            AtomId pick = 0;
            for (AtomId x = 1; x <= 8 && !pick; ++x)
                if (a.unassigned(x)) pick = x;
            if (pick) {
                a.push_decision(Lit::neg(pick));
                f.seed(Lit::neg(pick));
                if (!prop.propagate_and_check(a, f, a.decision_level()).violated) EXPECT(validate_fixpoint(b.store, a));
            }
        }
    }
}

void store_cases() {
    std::vector<Nogood> in;
    in.push_back(ng({Lit::pos(1), Lit::pos(2), Lit::pos(3)}));
    in.push_back(ng({Lit::neg(4)}));
    in.push_back(ng({Lit::pos(1), Lit::neg(2)}));
    in.push_back(ng({Lit::neg(3), Lit::pos(5)}));
    StoreBuild b = NogoodStore::build(std::move(in), 5);
    EXPECT(b.units.size() == 1 && b.units[0] == Lit::neg(4));
    EXPECT(b.store.size() == 3 && b.store.length(0) == 2 && b.store.length(1) == 2 && b.store.length(2) == 3);
    EXPECT(b.store.literals(0)[0] == Lit::pos(1) && b.store.literals(1)[0] == Lit::neg(3));
    EXPECT(b.store.dump_csv() == "offsets,0,2,4,7\npool,1,-2,-3,5,1,2,3\n");
    const auto bounds = b.store.static_class_bounds();
    EXPECT(bounds[0] == 0 && bounds[1] == 2 && bounds[2] == 3 && bounds[3] == 3);
    EXPECT(b.store.occurrences(Lit::pos(1), LengthClass::binary) == std::vector<NogoodId>{0});
    EXPECT(b.store.nogoods_of(Lit::pos(1)) == (std::vector<NogoodId>{0, 2}));
    EXPECT(NogoodStore::build({}, 3).store.dump_csv() == "offsets,0\npool\n");
    EXPECT(!Nogood::make({Lit::pos(1), Lit::neg(1)}, NogoodOrigin::constraint));  // vacuous
    StoreBuild c = NogoodStore::build({ng({Lit::pos(1), Lit::pos(2)})}, 2, 1);
    c.store.add_learned(*Nogood::make({Lit::neg(1)}, NogoodOrigin::learned, kNoTruth));
    bool threw = false;
    try {
        c.store.add_learned(*Nogood::make({Lit::neg(2)}, NogoodOrigin::learned, kNoTruth));
    } catch (const StoreCapacityError&) {
        threw = true;
    }
    EXPECT(threw);
}

void solver_cases() {
    SolverConfig base;
    base.max_models = 0;
    base.verify = true;
    base.debug_validate = true;
    {
        GroundProgram p = parse_program("a :- not b.\nb :- not a.");
        SolveResult r = solve(p, base);
        EXPECT(r.status == SolveStatus::sat && r.models.size() == 2);
        std::set<std::vector<AtomId>> oracle;
        for (const auto& m : enumerate_answer_sets(p)) oracle.insert(m);
        EXPECT(family(r) == oracle);
        EXPECT(r.stats.uip_check_failures == 0 && r.stats.asserting_failures == 0);
    }
    {
        SolveResult r = solve(parse_program("p :- q.\nq :- p."), base);
        EXPECT(r.status == SolveStatus::sat && r.models.size() == 1 && r.models[0].atom_ids.empty());
    }
    {
        SolveResult r = solve(parse_program("a.\n:- a."), base);
        EXPECT(r.status == SolveStatus::unsat && r.models.empty());
    }
    for (const char* text : {"p :- p.\np :- not p.\n", "p :- p.\np :- not p.\n:- not p.\n",
                             "c.\np :- p.\nx :- not y.\ny :- not x.\n:- c, not p.\n"}) {
        GroundProgram p = parse_program(text);
        EXPECT(enumerate_answer_sets(p).empty());
        for (LearnMode mode : {LearnMode::fwd, LearnMode::res}) {
            SolverConfig cfg = base;
            cfg.mode = mode;
            SolveResult r = solve(p, cfg);
            EXPECT(r.status == SolveStatus::unsat && r.models.empty());
        }
    }
    {
        GroundProgram p = parse_program("p :- q.\nq :- p.\np :- z.\nz :- not w.\nw :- not z.\n:- not p.\n");
        for (LearnMode mode : {LearnMode::fwd, LearnMode::res}) {
            SolverConfig cfg = base;
            cfg.mode = mode;
            SolveResult r = solve(p, cfg);
            EXPECT(r.models.size() == 1 && r.models[0].atoms == (std::vector<std::string>{"p", "q", "z"}));
        }
    }
    {
        SolveResult r = solve(parse_program("a."), base);
        EXPECT(r.status == SolveStatus::sat && r.models.size() == 1 && r.stats.decisions == 0);
        EXPECT(r.stats.wall_seconds() >= 0.0);
    }
    {
        SolverConfig cfg = base;
        cfg.learned_capacity = 0;
        bool threw = false;
        try {
            solve(parse_program("a :- not b.\nb :- not a.\nc :- not d.\nd :- not c.\n:- a, c.\n:- b, d.\n"), cfg);
        } catch (const StoreCapacityError&) {
            threw = true;
        }
        EXPECT(threw);
    }
}

void program_cases() {
    GroundProgram p = parse_program("a :- b, not c.\n% comment\n:- a, not d.\nd.\n");
    EXPECT(p.atom_count() == 4 && p.name(1) == "a" && p.atom(3).name == "c" && p.find("d") == 4 && p.find("zz") == 0);
    EXPECT(p.rules().size() == 2 && p.constraints().size() == 1);
    EXPECT(p.rules()[0].head == 1 && p.rules()[0].pos_body == std::vector<AtomId>{2} &&
           p.rules()[0].neg_body == std::vector<AtomId>{3});
    EXPECT(p.rules_of(4) == std::vector<std::uint32_t>{1} && p.rules()[1].is_fact());
    EXPECT(p.constraints()[0].is_constraint());
    EXPECT(print_program(p) == "a :- b, not c.\nd.\n:- a, not d.\n");
    std::vector<AtomId> m{2, 4};
    EXPECT(tp_step(p, m) == (std::vector<AtomId>{1, 4}));
    bool threw = false;
    try {
        std::vector<AtomId> bad{9};
        tp_step(p, bad);
    } catch (const std::out_of_range&) {
        threw = true;
    }
    EXPECT(threw);
    EXPECT(!validate(p).empty());  // b and c have no rules
    try {
        parse_program("a :- b\n");
        EXPECT(false);
    } catch (const ParseError& e) {
        EXPECT(e.line == 1);
    }
    // programmatic construction, as the reference's generators do (tests/support/gen.hpp)
    GroundProgram q;
    for (const char* n : {"x", "y", "z"}) q.intern(n);
    Rule r1;
    r1.head = 1;
    r1.neg_body = {2, 2};
    q.add_rule(r1);
    Rule r2;
    r2.head = 2;
    r2.neg_body = {1};
    q.add_rule(r2);
    Rule c;
    c.pos_body = {3};
    q.add_rule(c);
    EXPECT(q.atom_count() == 3 && q.rules().size() == 2 && q.rules()[0].neg_body == std::vector<AtomId>{2});
    GroundProgram copy = q;  // value semantics: editing the copy leaves q alone
    Rule r3;
    r3.head = 3;
    copy.add_rule(r3);
    EXPECT(q.rules().size() == 2 && copy.rules().size() == 3);
    SolverConfig all;
    all.max_models = 0;
    EXPECT(solve(q, all).models.size() == 2);  // {x}, {y}; z is never supported
    EXPECT(solve(copy, all).models.empty());   // z is a fact and violates ":- z."
}

}  // namespace

int main() {
    try {
        program_cases();
        store_cases();
        propagation_cases();
        random_stores();
        solver_cases();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "exception: %s\n", e.what());
        return 2;
    }
    std::printf("facade_test: %d checks, %d failed\n", g_checks, g_failed);
    return g_failed ? 1 : 0;
}
