// Program -> completion nogoods -> length-sorted CSR store (host, runs once per
// solve). Both steps define the nogood ids and auxiliary atom ids that the
// device engine and every trajectory counter depend on, so they follow the
// reference's emission order exactly:
//   compile_completion  /root/reference/proj/src/completion.cpp:60-146
//   nogood_census       /root/reference/proj/src/completion.cpp:153-173
//   NogoodStore::build  /root/reference/proj/src/nogood_store.cpp:25-74
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <new>
#include <utility>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "program.hpp"

namespace yas {

// Signed literal code: +atom for T atom, -atom for F atom.
inline AtomId lit_atom(std::int32_t c) { return static_cast<AtomId>(c < 0 ? -c : c); }
inline std::uint32_t lit_index(std::int32_t c) { return 2u * lit_atom(c) + (c < 0 ? 1u : 0u); }

inline constexpr std::uint32_t kAnyTruth = 0xFFFFFFFFu;
inline constexpr std::uint32_t kNoTruth = 0u;

enum Origin : std::uint8_t { kCompletion = 0, kConstraint = 1, kLearned = 2 };

struct Nogood {
    std::vector<std::int32_t> lits;  // sorted by atom, duplicate free
    std::uint8_t origin = kCompletion;
    std::uint32_t guard = kAnyTruth;

    /// Canonicalises (sort by atom, drop repeats); nullopt when the set holds
    /// both signs of one atom. Contract of Nogood::make, nogood.hpp:80-87.
    static std::optional<Nogood> make(std::vector<std::int32_t> lits, std::uint8_t origin,
                                      std::uint32_t guard = kAnyTruth);
    bool may_assert(std::int32_t l) const { return l < 0 || guard == kAnyTruth || guard == lit_atom(l); }
};

/// Allocator whose value-initialisation is a no-op: large host arrays that are
/// written in full (in parallel) right after sizing skip the zero fill.
template <class T>
struct NoInit : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = NoInit<U>;
    };
    NoInit() = default;
    template <class U>
    NoInit(const NoInit<U>&) noexcept {}
    template <class U>
    void construct(U* p) noexcept {
        ::new (static_cast<void*>(p)) U;
    }
    template <class U, class... A>
    void construct(U* p, A&&... a) {
        ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
};
template <class T>
using BigVec = std::vector<T, NoInit<T>>;

/// Flat list of canonical nogoods (literals of nogood k are
/// lits[off[k], off[k + 1]), sorted by atom): the completion's output and the
/// store builder's input, one allocation per array instead of per nogood.
struct NogoodSet {
    std::vector<std::int32_t> lits;
    std::vector<std::uint64_t> off{0};
    std::vector<std::uint32_t> guard;
    std::vector<std::uint8_t> origin;

    std::size_t size() const { return guard.size(); }
    std::size_t length(std::size_t k) const { return static_cast<std::size_t>(off[k + 1] - off[k]); }
    const std::int32_t* begin(std::size_t k) const { return lits.data() + off[k]; }
    bool may_assert(std::size_t k, std::int32_t l) const {
        return l < 0 || guard[k] == kAnyTruth || guard[k] == lit_atom(l);
    }
    void push(const Nogood& n) {
        lits.insert(lits.end(), n.lits.begin(), n.lits.end());
        off.push_back(lits.size());
        guard.push_back(n.guard);
        origin.push_back(n.origin);
    }
};

struct RuleAux {
    AtomId b = 0, t = 0, n = 0;
    bool vacuous = false;
};

struct Census {
    std::size_t rule_nogoods = 0, atom_nogoods = 0, constraint_nogoods = 0;
    std::size_t total() const { return rule_nogoods + atom_nogoods + constraint_nogoods; }
};

struct Completion {
    NogoodSet nogoods;
    std::vector<RuleAux> aux;      // per rule
    std::vector<std::uint32_t> aux_rule;  // aux atom - first_aux -> rule index
    std::vector<std::uint8_t> aux_kind;   // 0 body, 1 pos test, 2 neg test
    AtomId first_aux = 0;
    AtomId total_atoms = 0;
    Census counts;
    std::string atom_name(AtomId a, const Program& prog) const;
};

Completion compile_completion(const Program& prog);
Census census(const Program& prog);
std::string dump_nogoods(const Completion& comp, const Program& prog);

/// Static store, laid out for upload. Length-1 nogoods whose complement may be
/// asserted become `units` (kept in order); everything else is stable-sorted by
/// length into CSR ids 0..N-1. Occurrence lists are CSR over the key
/// (2*atom + neg) * 4 + length_class, ids ascending.
struct StaticStore {
    AtomId total_atoms = 0;
    std::vector<std::uint32_t> off{0};
    BigVec<std::int32_t> pool;
    std::vector<std::uint32_t> guard;
    std::vector<std::uint8_t> origin;
    std::vector<std::int32_t> units;     // literals of the static unit nogoods
    std::vector<std::int32_t> unit_ids;  // CSR ids of length-1 entries
    std::vector<std::uint32_t> occ_off;  // (2A+2)*4 + 1
    BigVec<std::int32_t> occ_ids;
    // Device copy of the occurrence lists: per (literal, nogood) one 16-byte
    // entry {id | length_class << 30, guard, x, y} with x, y two *other*
    // literals of the nogood (0 when absent), so binary/ternary nogoods are
    // decided from the entry; a long nogood's entry carries a third other
    // literal instead of the guard (three blockers: most long nogoods are
    // decided without reading their literals). Nogood ids stay below 2^30.
    BigVec<std::int32_t> occ_fat;  // 4 ints per occurrence, same order as occ_ids
    std::array<std::uint32_t, 4> bounds{0, 0, 0, 0};

    std::uint32_t size() const { return static_cast<std::uint32_t>(off.size() - 1); }
    std::uint32_t length(std::uint32_t id) const { return off[id + 1] - off[id]; }
    std::string dump_csv() const;
};

inline std::uint32_t length_class(std::uint32_t len) { return len >= 4 ? 3u : len - 1u; }

StaticStore build_store(const NogoodSet& nogoods, AtomId total_atoms);

}  // namespace yas
