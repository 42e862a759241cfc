// C++ drop-in for the reference's low-level propagation API, over the C-ABI:
//   Lit / Nogood / kAnyTruth / kNoTruth         /root/reference/proj/include/aspine/nogood.hpp:32-116
//   NogoodStore / StoreBuild / LengthClass       nogood_store.hpp:33-157
//   Assignment / DepsMap / Reason / Frontier     assignment.hpp:31-171
//   Propagator / PropagationOutcome              propagate.hpp:31-97
//   WorkerPool (accepted, no threads: the GPU is the parallelism)  worker_pool.hpp:27-55
//
// Where the state lives: Lit, Nogood, Assignment and Frontier are host values,
// as in the reference, so callers read and edit them directly. A NogoodStore
// is uploaded to the GPU once per Propagator; propagation runs there
// (libyasmin_b200: the device pass engine) and its result — cells, trail,
// reasons, Deps rows, next frontier — is written back into the caller's
// Assignment and Frontier. The host edits made since the Propagator last saw
// an Assignment (decisions, assignments) are replayed on the device first;
// anything else (a backjump, a direct Deps edit, another Assignment) makes it
// start from a fresh device assignment and replay the whole trail.
// Header-only; link with -lyasmin_b200.
#pragma once

#include <algorithm>
#include <array>
#include <bit>
#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <utility>
#include <vector>

#include "../yasmin_b200.h"

namespace aspine {

using AtomId = std::uint32_t;
using NogoodId = std::int32_t;

// ---- literals and nogoods --------------------------------------------------

/// T p / F p as the signed code +p / -p (the device's literal encoding too).
class Lit {
public:
    constexpr Lit() = default;
    static constexpr Lit pos(AtomId a) { return Lit(static_cast<std::int32_t>(a)); }
    static constexpr Lit neg(AtomId a) { return Lit(-static_cast<std::int32_t>(a)); }
    static constexpr Lit from_code(std::int32_t code) { return Lit(code); }
    constexpr std::int32_t code() const { return v_; }
    constexpr AtomId atom() const { return static_cast<AtomId>(v_ >= 0 ? v_ : -v_); }
    constexpr bool positive() const { return v_ > 0; }
    constexpr bool valid() const { return v_ != 0; }
    constexpr Lit operator~() const { return Lit(-v_); }
    /// 2 * atom + sign bit: the row of per-literal tables.
    constexpr std::size_t index() const { return (static_cast<std::size_t>(atom()) << 1) | (v_ < 0 ? 1u : 0u); }
    friend constexpr bool operator==(Lit x, Lit y) { return x.v_ == y.v_; }
    friend constexpr bool operator!=(Lit x, Lit y) { return x.v_ != y.v_; }

private:
    constexpr explicit Lit(std::int32_t v) : v_(v) {}
    std::int32_t v_ = 0;
};

/// The order of literals inside a nogood: atom id, then sign.
constexpr bool atom_less(Lit x, Lit y) { return x.atom() != y.atom() ? x.atom() < y.atom() : x.code() < y.code(); }

enum class NogoodOrigin : std::uint8_t { completion, constraint, learned };

/// Truth guard: the atom this nogood may derive T for (kNoTruth: none,
/// kAnyTruth: any); falsities may always be derived.
inline constexpr AtomId kAnyTruth = 0xFFFFFFFFu;
inline constexpr AtomId kNoTruth = 0u;

class Nogood {
public:
    /// Sorted by atom, repeats dropped; nullopt when both signs of an atom occur.
    static std::optional<Nogood> make(std::vector<Lit> lits, NogoodOrigin origin, AtomId truth_guard = kAnyTruth) {
        std::sort(lits.begin(), lits.end(), atom_less);
        lits.erase(std::unique(lits.begin(), lits.end()), lits.end());
        const auto clash = std::adjacent_find(lits.begin(), lits.end(), [](Lit x, Lit y) { return x.atom() == y.atom(); });
        if (clash != lits.end()) return std::nullopt;
        Nogood n;
        n.lits_ = std::move(lits);
        n.origin_ = origin;
        n.guard_ = truth_guard;
        return n;
    }
    const std::vector<Lit>& literals() const { return lits_; }
    std::size_t size() const { return lits_.size(); }
    bool empty() const { return lits_.empty(); }
    Lit operator[](std::size_t i) const { return lits_[i]; }
    std::vector<Lit>::const_iterator begin() const { return lits_.begin(); }
    std::vector<Lit>::const_iterator end() const { return lits_.end(); }
    NogoodOrigin origin() const { return origin_; }
    AtomId truth_guard() const { return guard_; }
    bool may_assert(Lit l) const { return !l.positive() || guard_ == kAnyTruth || guard_ == l.atom(); }
    bool contains(Lit l) const { return std::binary_search(lits_.begin(), lits_.end(), l, atom_less); }
    friend bool operator==(const Nogood& x, const Nogood& y) { return x.lits_ == y.lits_; }

private:
    Nogood() = default;
    std::vector<Lit> lits_;
    NogoodOrigin origin_ = NogoodOrigin::constraint;
    AtomId guard_ = kAnyTruth;
};

// ---- the store ---------------------------------------------------------------

inline constexpr NogoodId unit_pseudo_id(std::size_t k) { return -static_cast<NogoodId>(k) - 1; }
inline constexpr bool is_unit_pseudo_id(NogoodId id) { return id < 0; }

enum class LengthClass : std::uint8_t { unit = 0, binary = 1, ternary = 2, long_ = 3 };
inline LengthClass length_class(std::size_t len) {
    return len >= 4 ? LengthClass::long_ : static_cast<LengthClass>(len == 0 ? 0 : len - 1);
}

struct StoreCapacityError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

class Propagator;
struct StoreBuild;

/// The static partition is built by the library (same ids as the reference:
/// units split out, the rest stable-sorted by length) and mirrored here for
/// reading; learned nogoods are appended behind it with kNoTruth guards.
class NogoodStore {
public:
    static StoreBuild build(std::vector<Nogood> nogoods, AtomId total_atoms, std::size_t learned_capacity = 1u << 22);

    NogoodId add_learned(const Nogood& ng) {
        if (learned_count() >= learned_cap_) throw StoreCapacityError("learned nogood capacity exhausted");
        std::vector<std::int32_t> key;
        for (Lit l : ng) key.push_back(l.code());
        if (!seen_.insert(key).second) ++dups_;  // counted, still stored
        const NogoodId id = static_cast<NogoodId>(size());
        append(ng.literals(), NogoodOrigin::learned, kNoTruth);
        if (ng.size() == 1) unit_ids_.push_back(id);
        return id;
    }

    std::size_t size() const { return off_.size() - 1; }
    std::size_t static_count() const { return static_count_; }
    std::size_t learned_count() const { return size() - static_count_; }
    std::size_t duplicate_learned() const { return dups_; }
    std::span<const Lit> literals(NogoodId id) const { return {pool_.data() + off_[id], pool_.data() + off_[id + 1]}; }
    std::size_t length(NogoodId id) const { return off_[id + 1] - off_[id]; }
    LengthClass cls(NogoodId id) const { return length_class(length(id)); }
    NogoodOrigin origin(NogoodId id) const { return origin_[id]; }
    std::array<std::uint32_t, 4> static_class_bounds() const { return bounds_; }
    const std::vector<Lit>& static_units() const { return units_; }
    const std::vector<NogoodId>& unit_ids() const { return unit_ids_; }
    std::vector<NogoodId> learned_unit_ids() const {
        std::vector<NogoodId> out;
        std::copy_if(unit_ids_.begin(), unit_ids_.end(), std::back_inserter(out),
                     [&](NogoodId id) { return id >= static_cast<NogoodId>(static_count_); });
        return out;
    }
    const std::vector<NogoodId>& occurrences(Lit l, LengthClass c) const {
        return occ_[l.index()][static_cast<std::size_t>(c)];
    }
    std::vector<NogoodId> nogoods_of(Lit l) const {
        std::vector<NogoodId> out;
        for (const auto& list : occ_[l.index()]) out.insert(out.end(), list.begin(), list.end());
        return out;
    }
    AtomId truth_guard(NogoodId id) const { return guard_[id]; }
    bool may_assert(NogoodId id, Lit l) const {
        return !l.positive() || guard_[id] == kAnyTruth || guard_[id] == l.atom();
    }
    AtomId total_atoms() const { return total_; }
    std::string dump_csv() const {
        std::ostringstream o;
        o << "offsets";
        for (std::uint32_t x : off_) o << ',' << x;
        o << "\npool";
        for (Lit l : pool_) o << ',' << l.code();
        o << '\n';
        return o.str();
    }
    /// The library's copy of the static partition (uploaded by each Propagator).
    const yas_store* handle() const { return h_.get(); }

private:
    friend class Propagator;
    void append(const std::vector<Lit>& lits, NogoodOrigin o, AtomId guard) {
        const NogoodId id = static_cast<NogoodId>(size());
        pool_.insert(pool_.end(), lits.begin(), lits.end());
        off_.push_back(static_cast<std::uint32_t>(pool_.size()));
        origin_.push_back(o);
        guard_.push_back(guard);
        for (Lit l : lits) occ_[l.index()][static_cast<std::size_t>(length_class(lits.size()))].push_back(id);
    }

    std::shared_ptr<yas_store> h_;
    std::vector<Lit> pool_;
    std::vector<std::uint32_t> off_{0};
    std::vector<NogoodOrigin> origin_;
    std::vector<AtomId> guard_;
    std::vector<Lit> units_;
    std::vector<NogoodId> unit_ids_;
    std::vector<std::array<std::vector<NogoodId>, 4>> occ_;
    std::array<std::uint32_t, 4> bounds_{0, 0, 0, 0};
    std::size_t static_count_ = 0, learned_cap_ = 0, dups_ = 0;
    AtomId total_ = 0;
    struct KeyHash {
        std::size_t operator()(const std::vector<std::int32_t>& v) const {
            std::size_t h = 1469598103934665603ull;
            for (std::int32_t c : v) h = (h ^ static_cast<std::uint32_t>(c)) * 1099511628211ull;
            return h;
        }
    };
    std::unordered_set<std::vector<std::int32_t>, KeyHash> seen_;
};

struct StoreBuild {
    NogoodStore store;
    std::vector<Lit> units;
};

inline StoreBuild NogoodStore::build(std::vector<Nogood> nogoods, AtomId total_atoms, std::size_t learned_capacity) {
    std::vector<std::int32_t> lits;
    std::vector<std::uint32_t> offs{0}, guards;
    std::vector<std::uint8_t> origins;
    for (const Nogood& n : nogoods) {
        for (Lit l : n) lits.push_back(l.code());
        offs.push_back(static_cast<std::uint32_t>(lits.size()));
        guards.push_back(n.truth_guard());
        origins.push_back(static_cast<std::uint8_t>(n.origin()));
    }
    yas_store* h = nullptr;
    char err[512];
    const int rc = yas_store_build(lits.data(), offs.data(), nogoods.size(), guards.data(), origins.data(), total_atoms,
                                   &h, err, sizeof err);
    if (rc == YAS_ERR_CAPACITY) throw StoreCapacityError(err);
    if (rc != YAS_OK) throw std::invalid_argument(err);
    StoreBuild b;
    NogoodStore& s = b.store;
    s.h_.reset(h, &yas_store_free);
    s.total_ = total_atoms;
    s.learned_cap_ = learned_capacity;
    s.occ_.resize(2 * static_cast<std::size_t>(total_atoms) + 2);
    const std::uint32_t n = yas_store_size(h);
    std::vector<std::int32_t> buf;
    for (std::uint32_t id = 0; id < n; ++id) {
        std::uint32_t guard = 0;
        std::uint8_t origin = 1;
        buf.resize(yas_store_nogood(h, id, nullptr, 0, nullptr, nullptr));
        yas_store_nogood(h, id, buf.data(), buf.size(), &guard, &origin);
        std::vector<Lit> ls;
        for (std::int32_t c : buf) ls.push_back(Lit::from_code(c));
        s.append(ls, static_cast<NogoodOrigin>(origin), guard);
    }
    s.static_count_ = n;
    std::vector<std::int32_t> tmp(yas_store_units(h, nullptr, 0));
    yas_store_units(h, tmp.data(), tmp.size());
    for (std::int32_t c : tmp) s.units_.push_back(Lit::from_code(c));
    tmp.assign(yas_store_unit_ids(h, nullptr, 0), 0);
    yas_store_unit_ids(h, tmp.data(), tmp.size());
    s.unit_ids_.assign(tmp.begin(), tmp.end());
    yas_store_bounds(h, s.bounds_.data());
    b.units = s.units_;
    return b;
}

// ---- the assignment -----------------------------------------------------------

enum class AssignResult : std::uint8_t { newly_set, agreed, conflict };

struct Reason {
    enum Kind : std::int8_t { none = 0, decision, unit_input, propagated, completion };
    Kind kind = none;
    NogoodId antecedent = -1;
    static Reason make_decision() { return {decision, -1}; }
    static Reason make_unit() { return {unit_input, -1}; }
    static Reason make_propagated(NogoodId id) { return {propagated, id}; }
    static Reason make_completion() { return {completion, -1}; }
};

/// Level j is bit j-1 of an atom's row; rows are `words` 64-bit words.
class DepsMap {
public:
    DepsMap(AtomId total_atoms, std::uint32_t words)
        : w_(words), rows_((static_cast<std::size_t>(total_atoms) + 1) * words, 0ull), ovf_(total_atoms + 1, 0) {}
    std::uint32_t words() const { return w_; }
    std::uint32_t capacity_levels() const { return 64u * w_; }
    std::span<const std::uint64_t> of(AtomId a) const { return {rows_.data() + static_cast<std::size_t>(a) * w_, w_}; }
    bool overflow(AtomId a) const { return ovf_[a] != 0; }
    // direct edits (the Assignment's own bookkeeping uses the quiet forms below,
    // which a Propagator can replay; these make it start from a fresh copy)
    void clear_atom(AtomId a) {
        clear_q(a);
        ++version_;
    }
    void set(AtomId a, std::span<const std::uint64_t> bits, bool overflow) {
        set_q(a, bits, overflow);
        ++version_;
    }
    void set_decision(AtomId a, std::uint32_t level) {
        decision_q(a, level);
        ++version_;
    }
    void set_all_decision_levels(AtomId a, std::uint32_t cdl) {
        all_q(a, cdl);
        ++version_;
    }
    std::uint64_t version() const { return version_; }

private:
    friend class Assignment;
    void clear_q(AtomId a) {
        std::fill_n(row(a), w_, 0ull);
        ovf_[a] = 0;
    }
    void set_q(AtomId a, std::span<const std::uint64_t> bits, bool overflow) {
        std::uint64_t* r = row(a);
        for (std::uint32_t w = 0; w < w_; ++w) r[w] = w < bits.size() ? bits[w] : 0ull;
        ovf_[a] = overflow ? 1 : 0;
    }
    void decision_q(AtomId a, std::uint32_t level) {
        clear_q(a);
        mark(a, level);
    }
    void all_q(AtomId a, std::uint32_t cdl) {
        clear_q(a);
        for (std::uint32_t l = 2; l <= cdl && !ovf_[a]; ++l) mark(a, l);
    }
    std::uint64_t* row(AtomId a) { return rows_.data() + static_cast<std::size_t>(a) * w_; }
    void mark(AtomId a, std::uint32_t level) {
        const std::uint32_t bit = level - 1;
        if (bit >= capacity_levels()) ovf_[a] = 1;
        else row(a)[bit >> 6] |= 1ull << (bit & 63);
    }
    friend class Propagator;
    std::uint32_t w_;
    std::vector<std::uint64_t> rows_;
    std::vector<std::uint8_t> ovf_;
    std::uint64_t version_ = 0;
};

inline void bitmap_or(std::span<std::uint64_t> dst, std::span<const std::uint64_t> src) {
    for (std::size_t i = 0; i < dst.size() && i < src.size(); ++i) dst[i] |= src[i];
}
inline bool bitmap_any(std::span<const std::uint64_t> bits) {
    return std::any_of(bits.begin(), bits.end(), [](std::uint64_t w) { return w != 0; });
}
inline bool bitmap_test_level(std::span<const std::uint64_t> bits, std::uint32_t level) {
    const std::uint32_t bit = level - 1;
    return bit / 64 < bits.size() && ((bits[bit / 64] >> (bit % 64)) & 1ull);
}
inline std::uint32_t bitmap_highest_level_below(std::span<const std::uint64_t> bits, std::uint32_t below) {
    for (std::uint32_t l = below; l > 1;)
        if (bitmap_test_level(bits, --l)) return l;
    return 0;
}
inline std::vector<std::uint32_t> bitmap_levels(std::span<const std::uint64_t> bits) {
    std::vector<std::uint32_t> out;
    for (std::size_t w = 0; w < bits.size(); ++w)
        for (std::uint64_t x = bits[w]; x; x &= x - 1) out.push_back(static_cast<std::uint32_t>(64 * w + std::countr_zero(x)) + 1);
    return out;
}

class Assignment {
public:
    struct TrailEntry {
        Lit lit;
        std::uint32_t level;
    };

    Assignment(AtomId total_atoms, std::uint32_t deps_words)
        : n_(total_atoms), atoms_(total_atoms + 1), dec_(2), deps_(total_atoms, deps_words) {
        trail_.reserve(total_atoms);
    }

    AtomId atom_count() const { return n_; }
    std::uint32_t decision_level() const { return cdl_; }
    std::int32_t cell(AtomId a) const { return atoms_[a].cell; }
    bool unassigned(AtomId a) const { return atoms_[a].cell == 0; }
    bool has(Lit l) const {
        const std::int32_t c = atoms_[l.atom()].cell;
        return c != 0 && (c > 0) == l.positive();
    }
    std::uint32_t level_of(AtomId a) const {
        const std::int32_t c = atoms_[a].cell;
        return static_cast<std::uint32_t>(c >= 0 ? c : -c);
    }
    std::size_t trail_index(AtomId a) const { return atoms_[a].pos; }
    Reason reason(AtomId a) const { return atoms_[a].why; }

    AssignResult assign_unit(Lit l) {
        const AssignResult r = put(l, 1, Reason::make_unit());
        if (r == AssignResult::newly_set) deps_.clear_q(l.atom());
        return r;
    }
    AssignResult assign_propagated(Lit l, std::uint32_t level, std::span<const std::uint64_t> deps, bool deps_overflow,
                                   NogoodId antecedent) {
        const AssignResult r = put(l, level, Reason::make_propagated(antecedent));
        if (r == AssignResult::newly_set) deps_.set_q(l.atom(), deps, deps_overflow);
        return r;
    }
    AssignResult assign_completion(Lit l) {
        const AssignResult r = put(l, cdl_, Reason::make_completion());
        if (r == AssignResult::newly_set) deps_.all_q(l.atom(), cdl_);
        return r;
    }
    void push_decision(Lit l) {
        dec_.push_back(l);
        put(l, ++cdl_, Reason::make_decision());
        deps_.decision_q(l.atom(), cdl_);
    }
    void backjump(std::uint32_t target_level) {
        while (!trail_.empty() && trail_.back().level > target_level) {
            const AtomId a = trail_.back().lit.atom();
            atoms_[a] = Slot{};
            deps_.clear_q(a);
            trail_.pop_back();
        }
        dec_.resize(target_level + 1);
        cdl_ = target_level;
        ++edits_;  // the device copy cannot follow a backjump by replay: start over
    }
    bool is_total() const { return trail_.size() == n_; }
    std::span<const TrailEntry> trail() const { return trail_; }
    Lit level_decision(std::uint32_t level) const { return dec_[level]; }
    std::vector<Lit> decisions() const { return {dec_.begin() + 2, dec_.end()}; }
    DepsMap& deps() { return deps_; }
    const DepsMap& deps() const { return deps_; }

    std::string debug_trail(const std::function<std::string(AtomId)>& namer) const {
        std::ostringstream o;
        for (const TrailEntry& e : trail_) {
            const Reason r = atoms_[e.lit.atom()].why;
            o << (e.lit.positive() ? "T " : "F ") << namer(e.lit.atom()) << '@' << e.level;
            if (r.kind == Reason::propagated) o << " <- " << r.antecedent;
            else
                o << (r.kind == Reason::decision     ? " (decision)"
                      : r.kind == Reason::unit_input ? " (unit)"
                      : r.kind == Reason::completion ? " (completion)"
                                                     : " (?)");
            o << '\n';
        }
        return o.str();
    }

private:
    friend class Propagator;
    struct Slot {
        std::int32_t cell = 0;
        std::size_t pos = 0;
        Reason why{};
    };
    AssignResult put(Lit l, std::uint32_t level, Reason why) {
        Slot& s = atoms_[l.atom()];
        if (s.cell != 0) return (s.cell > 0) == l.positive() ? AssignResult::agreed : AssignResult::conflict;
        s.cell = l.positive() ? static_cast<std::int32_t>(level) : -static_cast<std::int32_t>(level);
        s.pos = trail_.size();
        s.why = why;
        trail_.push_back({l, level});
        return AssignResult::newly_set;
    }

    AtomId n_;
    std::vector<Slot> atoms_;
    std::vector<TrailEntry> trail_;
    std::vector<Lit> dec_;  // [level]; levels 0 and 1 hold no decision
    std::uint32_t cdl_ = 1;
    DepsMap deps_;
    std::uint64_t edits_ = 0;  // non-replayable edits (backjumps)
};

struct Frontier {
    std::vector<Lit> last, next;
    void seed(Lit l) { last.push_back(l); }
    void advance() {
        std::swap(last, next);
        next.clear();
    }
    void clear() {
        last.clear();
        next.clear();
    }
    bool idle() const { return last.empty() && next.empty(); }
};

// ---- propagation -------------------------------------------------------------

/// The reference spreads a pass over a CPU pool; here the pass runs on the GPU
/// and the worker count is accepted for source compatibility only.
class WorkerPool {
public:
    explicit WorkerPool(unsigned workers) : n_(workers ? workers : 1) {}
    WorkerPool(const WorkerPool&) = delete;
    WorkerPool& operator=(const WorkerPool&) = delete;
    unsigned size() const { return n_; }

private:
    unsigned n_;
};

struct PropagationOutcome {
    bool violated = false;
    std::vector<NogoodId> conflicts;
    std::uint64_t propagations = 0;
    std::uint64_t passes = 0;
    std::uint64_t watch_replacements = 0;  // no watched literals on the device: always 0
};

class Propagator {
public:
    Propagator(NogoodStore& store, WorkerPool& pool, int device = 0) : store_(&store), pool_(&pool), device_(device) {
        (void)pool_;
    }
    Propagator(const Propagator&) = delete;
    Propagator& operator=(const Propagator&) = delete;

    PropagationOutcome initial_propagation(Assignment& a, Frontier& f) { return run(a, f, 0, true); }
    PropagationOutcome propagate_and_check(Assignment& a, Frontier& f, std::uint32_t level) {
        return run(a, f, level, false);
    }

    /// OR of the Deps rows of delta's atoms other than w's, skipping level <= 1
    /// (propagate.cpp:49-69); the same rows the device writes for a proposal.
    static std::pair<std::vector<std::uint64_t>, bool> mk_dl_bitmap(std::span<const Lit> delta, Lit w,
                                                                    const Assignment& a) {
        std::vector<std::uint64_t> acc(a.deps().words(), 0ull);
        bool ovf = false;
        for (Lit x : delta) {
            if (x.atom() == w.atom() || a.level_of(x.atom()) <= 1) continue;
            bitmap_or(acc, a.deps().of(x.atom()));
            ovf = ovf || a.deps().overflow(x.atom());
        }
        return {std::move(acc), ovf};
    }

private:
    struct Session {
        yas_propagator* p = nullptr;
        ~Session() { yas_propagator_free(p); }
    };

    [[noreturn]] void fail(const char* what) const {
        char msg[512] = {0};
        if (s_ && s_->p) yas_propagator_last_error(s_->p, msg, sizeof msg);
        throw std::runtime_error(std::string(what) + (msg[0] ? ": " : "") + msg);
    }
    void ck(int rc, const char* what) const {
        if (rc != YAS_OK) fail(what);
    }

    void open(std::uint32_t words) {
        if (s_ && words_ == words) return;
        s_ = std::make_unique<Session>();
        char err[512];
        if (yas_propagator_create(store_->handle(), words, 0, device_, &s_->p, err, sizeof err) != YAS_OK)
            throw std::runtime_error(err);
        words_ = words;
        bound_ = nullptr;
    }

    // One device op for the trail entry k of `a` (a decision, or an assignment
    // with its level, Deps row, overflow flag and reason).
    void replay_entry(const Assignment& a, std::size_t k) {
        const Assignment::TrailEntry& e = a.trail_[k];
        const Reason r = a.atoms_[e.lit.atom()].why;
        if (r.kind == Reason::decision) {
            ck(yas_propagator_push_decision(s_->p, e.lit.code()), "push_decision");
            return;
        }
        const std::int32_t code = e.lit.code();
        const std::int32_t ante = r.kind == Reason::propagated ? r.antecedent
                                  : r.kind == Reason::unit_input ? -3
                                  : r.kind == Reason::completion ? -4
                                                                 : -1;
        const std::span<const std::uint64_t> d = a.deps_.of(e.lit.atom());
        ck(yas_propagator_assign(s_->p, &code, 1, e.level, d.data(), static_cast<std::uint32_t>(d.size()),
                                 a.deps_.overflow(e.lit.atom()) ? 1 : 0, ante),
           "assign");
    }

    // Bring the device assignment to `a`: replay only what was appended since
    // this propagator last wrote `a`, otherwise start from a fresh one.
    void sync(const Assignment& a) {
        const bool same = bound_ == &a && bound_edits_ == a.edits_ && bound_deps_ == a.deps_.version() &&
                          bound_trail_ <= a.trail_.size() && bound_learned_ <= store_->learned_count();
        std::size_t from = 0;
        if (same) {
            from = bound_trail_;
        } else {
            ck(yas_propagator_reset(s_->p), "reset");
            bound_learned_ = 0;
        }
        for (std::size_t k = bound_learned_; k < store_->learned_count(); ++k) {  // learned nogoods, in id order
            const NogoodId id = static_cast<NogoodId>(store_->static_count() + k);
            std::vector<std::int32_t> codes;
            for (Lit l : store_->literals(id)) codes.push_back(l.code());
            if (yas_propagator_add_learned(s_->p, codes.data(), codes.size()) != id) fail("add_learned");
        }
        bound_learned_ = store_->learned_count();
        for (std::size_t k = from; k < a.trail_.size(); ++k) replay_entry(a, k);
    }

    PropagationOutcome run(Assignment& a, Frontier& f, std::uint32_t level, bool initial) {
        if (a.atom_count() != store_->total_atoms()) throw std::invalid_argument("assignment and store differ in atoms");
        open(a.deps().words());
        sync(a);
        if (!initial) {  // the device frontier becomes f.last
            std::vector<std::int32_t> seed;
            for (Lit l : f.last) seed.push_back(l.code());
            ck(yas_propagator_clear_frontier(s_->p), "frontier");
            if (!seed.empty()) ck(yas_propagator_seed(s_->p, seed.data(), seed.size()), "seed");
        }
        yas_outcome o{};
        ck(initial ? yas_propagator_initial(s_->p, &o) : yas_propagator_propagate(s_->p, level, &o),
           initial ? "initial_propagation" : "propagate_and_check");
        PropagationOutcome out;
        out.violated = o.violated != 0;
        out.propagations = o.propagations;
        out.passes = o.passes;
        out.conflicts.resize(o.n_conflicts);
        if (o.n_conflicts) yas_propagator_conflicts(s_->p, out.conflicts.data(), out.conflicts.size());
        read_back(a);
        std::vector<std::int32_t> fr(static_cast<std::size_t>(a.atom_count()) + 1);
        fr.resize(yas_propagator_frontier(s_->p, fr.data(), fr.size()));
        if (!initial) f.last.clear();
        for (std::int32_t c : fr) f.last.push_back(Lit::from_code(c));
        f.next.clear();
        return out;
    }

    // The device's assignment becomes the caller's (cells, trail, reasons, Deps).
    void read_back(Assignment& a) {
        const std::size_t n = static_cast<std::size_t>(a.atom_count()) + 1;
        std::vector<std::int32_t> cells(n), reasons(n), trail(n);
        ck(yas_propagator_cells(s_->p, cells.data()), "cells");
        ck(yas_propagator_reasons(s_->p, reasons.data()), "reasons");
        trail.resize(yas_propagator_trail(s_->p, trail.data(), trail.size()));
        std::vector<std::uint64_t> word(n);
        std::vector<std::uint8_t> ovf(n);
        for (std::uint32_t w = 0; w < words_; ++w) {
            ck(yas_propagator_deps(s_->p, w, word.data(), ovf.data()), "deps");
            for (std::size_t x = 0; x < n; ++x) a.deps_.rows_[x * words_ + w] = word[x];
        }
        for (std::size_t x = 0; x < n; ++x) a.deps_.ovf_[x] = ovf[x];
        a.trail_.clear();
        for (std::size_t x = 0; x < n; ++x) a.atoms_[x] = Assignment::Slot{};
        for (std::int32_t code : trail) {
            const Lit l = Lit::from_code(code);
            Assignment::Slot& s = a.atoms_[l.atom()];
            s.cell = cells[l.atom()];
            s.pos = a.trail_.size();
            const std::int32_t r = reasons[l.atom()];
            s.why = r >= 0 ? Reason::make_propagated(r)
                    : r == -2 ? Reason::make_decision()
                    : r == -3 ? Reason::make_unit()
                    : r == -4 ? Reason::make_completion()
                              : Reason{};
            a.trail_.push_back({l, a.level_of(l.atom())});
        }
        bound_ = &a;
        bound_edits_ = a.edits_;
        bound_deps_ = a.deps_.version();
        bound_trail_ = a.trail_.size();
    }

    NogoodStore* store_;
    WorkerPool* pool_;
    int device_;
    std::unique_ptr<Session> s_;
    std::uint32_t words_ = 0;
    const Assignment* bound_ = nullptr;
    std::uint64_t bound_edits_ = 0, bound_deps_ = 0;
    std::size_t bound_trail_ = 0, bound_learned_ = 0;
};

/// No unit-resolvable and no violated CSR nogood under `a` (a passive unit —
/// one open literal the truth guard bars — is a legal resting state), and
/// every static unit's complement holds (propagate.cpp:246-300 semantics).
inline bool validate_fixpoint(const NogoodStore& store, const Assignment& a, std::string* why = nullptr) {
    auto bad = [&](const std::string& msg) {
        if (why) *why = msg;
        return false;
    };
    for (std::size_t k = 0; k < store.static_units().size(); ++k)
        if (!a.has(~store.static_units()[k])) return bad("static unit " + std::to_string(k) + " not asserted");
    for (NogoodId id = 0; id < static_cast<NogoodId>(store.size()); ++id) {
        std::size_t hold = 0, open = 0;
        bool dead = false;
        Lit last_open;
        for (Lit l : store.literals(id)) {
            if (a.unassigned(l.atom())) {
                ++open;
                last_open = l;
            } else if (a.has(l)) {
                ++hold;
            } else {
                dead = true;
            }
        }
        if (dead) continue;
        if (open == 0) return bad("nogood " + std::to_string(id) + " violated");
        if (open == 1 && store.may_assert(id, ~last_open)) return bad("nogood " + std::to_string(id) + " is unit");
    }
    return true;
}

/// The device keeps no watched literals; the property the reference's watch
/// discipline guards at a no-conflict fixpoint — every CSR nogood of length >= 2
/// is satisfied, has two open literals, or is a passive unit — is checked
/// directly on the assignment.
inline bool validate_watch_invariant(const NogoodStore& store, const Assignment& a, std::string* why = nullptr) {
    return validate_fixpoint(store, a, why);
}

}  // namespace aspine
