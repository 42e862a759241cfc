#include "compile.hpp"

#include <algorithm>
#include <stdexcept>

namespace yas {

std::optional<Nogood> Nogood::make(std::vector<std::int32_t> lits, std::uint8_t origin,
                                   std::uint32_t guard) {
    std::sort(lits.begin(), lits.end(), [](std::int32_t a, std::int32_t b) {
        const AtomId x = lit_atom(a), y = lit_atom(b);
        return x < y || (x == y && a < b);
    });
    lits.erase(std::unique(lits.begin(), lits.end()), lits.end());
    for (std::size_t i = 1; i < lits.size(); ++i)
        if (lit_atom(lits[i]) == lit_atom(lits[i - 1])) return std::nullopt;
    Nogood n;
    n.lits = std::move(lits);
    n.origin = origin;
    n.guard = guard;
    return n;
}

std::string Completion::atom_name(AtomId a, const Program& prog) const {
    if (a < first_aux || a > total_atoms) return prog.name(a);
    static const char* tags[3] = {"b_r", "t_r", "n_r"};
    return std::string(tags[aux_kind[a - first_aux]]) + "(" + std::to_string(aux_rule[a - first_aux] + 1) + ")";
}

namespace {

// Emission helper: one nogood per call, counted into its category.
struct Emitter {
    Completion& c;
    AtomId next;

    AtomId fresh(std::uint32_t rule, std::uint8_t kind) {
        c.aux_rule.push_back(rule);
        c.aux_kind.push_back(kind);
        return next++;
    }
    void put(std::vector<std::int32_t> lits, std::uint8_t origin, std::size_t& counter, std::uint32_t guard) {
        auto n = Nogood::make(std::move(lits), origin, guard);
        c.nogoods.push_back(std::move(*n));  // completion sets are never vacuous
        ++counter;
    }
};

inline std::int32_t T(AtomId a) { return static_cast<std::int32_t>(a); }
inline std::int32_t F(AtomId a) { return -static_cast<std::int32_t>(a); }

}  // namespace

Completion compile_completion(const Program& prog) {
    Completion c;
    c.first_aux = prog.atom_count() + 1;
    Emitter em{c, c.first_aux};

    // Rule side: b_r <-> t_r & n_r, t_r <-> body+, n_r <-> not body-
    // (completion.cpp:60-114). Guards name the atom a nogood may derive true.
    for (std::uint32_t ri = 0; ri < prog.rules().size(); ++ri) {
        const Rule& r = prog.rules()[ri];
        RuleAux ax;
        ax.b = em.fresh(ri, 0);
        std::size_t& k = c.counts.rule_nogoods;
        if (r.body_overlaps()) {
            ax.vacuous = true;
            em.put({T(ax.b)}, kCompletion, k, kNoTruth);
            c.aux.push_back(ax);
            continue;
        }
        const bool pos = !r.pos_body.empty(), neg = !r.neg_body.empty();
        if (pos) ax.t = em.fresh(ri, 1);
        if (neg) ax.n = em.fresh(ri, 2);
        if (pos && neg) {
            em.put({F(ax.b), T(ax.t), T(ax.n)}, kCompletion, k, ax.b);
            em.put({T(ax.b), F(ax.t)}, kCompletion, k, ax.t);
            em.put({T(ax.b), F(ax.n)}, kCompletion, k, ax.n);
        } else if (pos || neg) {
            const AtomId test = pos ? ax.t : ax.n;
            em.put({F(ax.b), T(test)}, kCompletion, k, ax.b);
            em.put({T(ax.b), F(test)}, kCompletion, k, test);
        } else {
            em.put({F(ax.b)}, kCompletion, k, ax.b);
        }
        if (pos) {
            std::vector<std::int32_t> all{F(ax.t)};
            for (AtomId p : r.pos_body) {
                em.put({T(ax.t), F(p)}, kCompletion, k, kNoTruth);
                all.push_back(T(p));
            }
            em.put(std::move(all), kCompletion, k, ax.t);
        }
        if (neg) {
            std::vector<std::int32_t> all{F(ax.n)};
            for (AtomId q : r.neg_body) {
                em.put({T(ax.n), T(q)}, kCompletion, k, kNoTruth);
                all.push_back(F(q));
            }
            em.put(std::move(all), kCompletion, k, ax.n);
        }
        c.aux.push_back(ax);
    }
    // Atom side: p <-> OR b_r (completion.cpp:116-130).
    for (AtomId p = 1; p <= prog.atom_count(); ++p) {
        const auto& defs = prog.rules_of(p);
        std::size_t& k = c.counts.atom_nogoods;
        if (defs.empty()) {
            em.put({T(p)}, kCompletion, k, kNoTruth);
            continue;
        }
        std::vector<std::int32_t> support{T(p)};
        for (std::uint32_t ri : defs) {
            em.put({F(p), T(c.aux[ri].b)}, kCompletion, k, p);
            support.push_back(F(c.aux[ri].b));
        }
        em.put(std::move(support), kCompletion, k, kNoTruth);
    }
    // Integrity constraints (completion.cpp:132-138).
    for (const Rule& r : prog.constraints()) {
        if (r.body_overlaps()) continue;
        std::vector<std::int32_t> lits;
        for (AtomId p : r.pos_body) lits.push_back(T(p));
        for (AtomId q : r.neg_body) lits.push_back(F(q));
        em.put(std::move(lits), kConstraint, c.counts.constraint_nogoods, kNoTruth);
    }
    c.total_atoms = em.next - 1;
    return c;
}

Census census(const Program& prog) {
    Census s;
    for (const Rule& r : prog.rules()) {
        if (r.body_overlaps()) {
            s.rule_nogoods += 1;
            continue;
        }
        const std::size_t np = r.pos_body.size(), nn = r.neg_body.size();
        s.rule_nogoods += (np && nn) ? 3 : (np || nn) ? 2 : 1;
        if (np) s.rule_nogoods += np + 1;
        if (nn) s.rule_nogoods += nn + 1;
    }
    for (AtomId p = 1; p <= prog.atom_count(); ++p) s.atom_nogoods += prog.rules_of(p).size() + 1;
    for (const Rule& r : prog.constraints())
        if (!r.body_overlaps()) s.constraint_nogoods += 1;
    return s;
}

std::string dump_nogoods(const Completion& comp, const Program& prog) {
    static const char* origins[3] = {"completion", "constraint", "learned"};
    std::string out;
    for (const Nogood& n : comp.nogoods) {
        out += '{';
        for (std::size_t i = 0; i < n.lits.size(); ++i) {
            if (i) out += ", ";
            out += n.lits[i] > 0 ? "T " : "F ";
            out += comp.atom_name(lit_atom(n.lits[i]), prog);
        }
        out += "} ";
        out += origins[n.origin];
        out += '\n';
    }
    return out;
}

StaticStore build_store(const std::vector<Nogood>& nogoods, AtomId total_atoms) {
    StaticStore st;
    st.total_atoms = total_atoms;
    std::vector<const Nogood*> rest;
    rest.reserve(nogoods.size());
    for (const Nogood& n : nogoods) {
        if (n.lits.size() == 1 && n.may_assert(-n.lits[0])) st.units.push_back(n.lits[0]);
        else rest.push_back(&n);
    }
    // ids carry their length class in the top two bits of the device's
    // occurrence entries, and offsets are 32-bit (compile.hpp)
    std::size_t lits = 0;
    for (const Nogood* n : rest) lits += n->lits.size();
    if (rest.size() >= (std::size_t{1} << 30) || lits > 0xFFFFFFFFull)
        throw std::length_error("store too large: at most 2^30 - 1 nogoods and 2^32 - 1 literals");
    std::stable_sort(rest.begin(), rest.end(),
                     [](const Nogood* a, const Nogood* b) { return a->lits.size() < b->lits.size(); });
    st.off.reserve(rest.size() + 1);
    st.guard.reserve(rest.size());
    const std::size_t keys = (2 * static_cast<std::size_t>(total_atoms) + 2) * 4;
    std::vector<std::uint32_t> count(keys + 1, 0);
    for (const Nogood* n : rest) {
        const std::uint32_t id = st.size();
        st.pool.insert(st.pool.end(), n->lits.begin(), n->lits.end());
        st.off.push_back(static_cast<std::uint32_t>(st.pool.size()));
        st.guard.push_back(n->guard);
        st.origin.push_back(n->origin);
        if (n->lits.size() == 1) st.unit_ids.push_back(static_cast<std::int32_t>(id));
        const std::uint32_t cls = length_class(static_cast<std::uint32_t>(n->lits.size()));
        for (std::int32_t l : n->lits) ++count[lit_index(l) * 4 + cls + 1];
    }
    // Counting sort of (literal, class) occurrences; ids are visited in
    // ascending order so every list comes out ascending.
    for (std::size_t k = 0; k < keys; ++k) count[k + 1] += count[k];
    st.occ_off = count;
    st.occ_ids.resize(st.pool.size());
    st.occ_fat.resize(4 * st.pool.size());
    std::vector<std::uint32_t> fill(count.begin(), count.end() - 1);
    for (std::uint32_t id = 0; id < st.size(); ++id) {
        const std::uint32_t cls = length_class(st.length(id));
        for (std::uint32_t k = st.off[id]; k < st.off[id + 1]; ++k) {
            const std::uint32_t at = fill[lit_index(st.pool[k]) * 4 + cls]++;
            st.occ_ids[at] = static_cast<std::int32_t>(id);
            std::int32_t other[2] = {0, 0};
            for (std::uint32_t q = st.off[id], n = 0; q < st.off[id + 1] && n < 2; ++q)
                if (q != k) other[n++] = st.pool[q];
            st.occ_fat[4 * at + 0] = static_cast<std::int32_t>(id | cls << 30);  // class in the top bits
            st.occ_fat[4 * at + 1] = static_cast<std::int32_t>(st.guard[id]);
            st.occ_fat[4 * at + 2] = other[0];
            st.occ_fat[4 * at + 3] = other[1];
        }
    }
    auto first_of_len = [&](std::uint32_t len) {
        std::uint32_t i = 0;
        while (i < st.size() && st.length(i) < len) ++i;
        return i;
    };
    st.bounds = {first_of_len(2), first_of_len(3), first_of_len(4), st.size()};
    return st;
}

std::string StaticStore::dump_csv() const {
    std::string out = "offsets";
    for (std::uint32_t o : off) out += "," + std::to_string(o);
    out += "\npool";
    for (std::int32_t l : pool) out += "," + std::to_string(l);
    out += '\n';
    return out;
}

}  // namespace yas
