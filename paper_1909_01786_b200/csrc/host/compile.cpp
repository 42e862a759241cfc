#include "compile.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <iterator>
#include <stdexcept>

#include "parallel.hpp"

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

inline std::int32_t T(AtomId a) { return static_cast<std::int32_t>(a); }
inline std::int32_t F(AtomId a) { return -static_cast<std::int32_t>(a); }

// Writes nogoods into preallocated slots: nogood k at literal position `at`.
struct Writer {
    NogoodSet& ns;
    std::size_t k, at;

    template <class It>
    void put(It first, It last, std::uint8_t origin, std::uint32_t guard) {
        std::int32_t* out = ns.lits.data() + at;
        const std::size_t len = static_cast<std::size_t>(std::distance(first, last));
        std::copy(first, last, out);
        std::sort(out, out + len, [](std::int32_t a, std::int32_t b) { return lit_atom(a) < lit_atom(b); });
        at += len;
        ns.off[k + 1] = at;
        ns.guard[k] = guard;
        ns.origin[k] = origin;
        ++k;
    }
    void put(std::initializer_list<std::int32_t> l, std::uint8_t origin, std::uint32_t guard) {
        put(l.begin(), l.end(), origin, guard);
    }
};

}  // namespace

// Emission order, ids and guards of completion.cpp:60-146.
// Every rule, atom and constraint knows up front how many aux atoms, nogoods
// and literals it emits, so prefix sums place each one's output and the
// three sections are filled by all host threads at once.
Completion compile_completion(const Program& prog) {
    Completion c;
    const std::vector<Rule>& rules = prog.rules();
    const std::vector<Rule>& cons = prog.constraints();
    const std::size_t R = rules.size(), C = cons.size();
    const AtomId n = prog.atom_count();
    c.first_aux = n + 1;
    // counts: [0, R) rules, [R, R + n) atoms, [R + n, R + n + C) constraints
    const std::size_t items = R + n + C;
    std::vector<std::uint64_t> ng(items + 1, 0), li(items + 1, 0), ax(R + 1, 0);
    std::vector<std::uint8_t> vac(R, 0);
    parallel_chunks(items, 1 << 14, [&](unsigned, std::size_t b, std::size_t e) {
        for (std::size_t i = b; i < e; ++i) {
            if (i < R) {
                const Rule& r = rules[i];
                if (r.body_overlaps()) {
                    vac[i] = 1;
                    ax[i] = 1, ng[i] = 1, li[i] = 1;
                    continue;
                }
                const std::size_t np = r.pos_body.size(), nn = r.neg_body.size();
                ax[i] = 1 + (np ? 1 : 0) + (nn ? 1 : 0);
                ng[i] = (np && nn) ? 3 : (np || nn) ? 2 : 1;
                li[i] = (np && nn) ? 7 : (np || nn) ? 4 : 1;
                if (np) ng[i] += np + 1, li[i] += 3 * np + 1;
                if (nn) ng[i] += nn + 1, li[i] += 3 * nn + 1;
            } else if (i < R + n) {
                const std::size_t d = prog.rules_of(static_cast<AtomId>(i - R + 1)).size();
                ng[i] = d ? d + 1 : 1;
                li[i] = d ? 3 * d + 1 : 1;
            } else {
                const Rule& r = cons[i - R - n];
                if (r.body_overlaps()) continue;
                ng[i] = 1;
                li[i] = r.pos_body.size() + r.neg_body.size();
            }
        }
    });
    const std::uint64_t total_ng = exclusive_scan_inplace(ng), total_li = exclusive_scan_inplace(li);
    const std::uint64_t total_aux = exclusive_scan_inplace(ax);
    NogoodSet& ns = c.nogoods;
    ns.lits.resize(total_li);
    ns.off.assign(total_ng + 1, 0);
    ns.guard.resize(total_ng);
    ns.origin.resize(total_ng);
    c.aux.resize(R);
    c.aux_rule.resize(total_aux);
    c.aux_kind.resize(total_aux);
    for (std::size_t i = 0; i < R; ++i) c.counts.rule_nogoods += ng[i + 1] - ng[i];
    for (std::size_t i = R; i < R + n; ++i) c.counts.atom_nogoods += ng[i + 1] - ng[i];
    for (std::size_t i = R + n; i < items; ++i) c.counts.constraint_nogoods += ng[i + 1] - ng[i];
    c.total_atoms = static_cast<AtomId>(n + total_aux);

    // aux ids first: the atom side refers to b_r of every rule
    parallel_chunks(R, 1 << 14, [&](unsigned, std::size_t b, std::size_t e) {
        for (std::size_t r = b; r < e; ++r) {
            AtomId next = c.first_aux + static_cast<AtomId>(ax[r]);
            auto fresh = [&](std::uint8_t kind) {
                c.aux_rule[next - c.first_aux] = static_cast<std::uint32_t>(r);
                c.aux_kind[next - c.first_aux] = kind;
                return next++;
            };
            RuleAux& a = c.aux[r];
            a.b = fresh(0);
            if (vac[r]) {
                a.vacuous = true;
                continue;
            }
            if (!rules[r].pos_body.empty()) a.t = fresh(1);
            if (!rules[r].neg_body.empty()) a.n = fresh(2);
        }
    });
    parallel_chunks(items, 1 << 13, [&](unsigned, std::size_t b, std::size_t e) {
        std::vector<std::int32_t> all;
        for (std::size_t i = b; i < e; ++i) {
            Writer w{ns, ng[i], li[i]};
            if (i < R) {  // rule side: b_r <-> t_r & n_r, t_r <-> body+, n_r <-> not body-
                const Rule& r = rules[i];
                const RuleAux& a = c.aux[i];
                if (a.vacuous) {
                    w.put({T(a.b)}, kCompletion, kNoTruth);
                    continue;
                }
                const bool pos = a.t != 0, neg = a.n != 0;
                if (pos && neg) {
                    w.put({F(a.b), T(a.t), T(a.n)}, kCompletion, a.b);
                    w.put({T(a.b), F(a.t)}, kCompletion, a.t);
                    w.put({T(a.b), F(a.n)}, kCompletion, a.n);
                } else if (pos || neg) {
                    const AtomId test = pos ? a.t : a.n;
                    w.put({F(a.b), T(test)}, kCompletion, a.b);
                    w.put({T(a.b), F(test)}, kCompletion, test);
                } else {
                    w.put({F(a.b)}, kCompletion, a.b);
                }
                if (pos) {
                    all.assign(1, F(a.t));
                    for (AtomId p : r.pos_body) {
                        w.put({T(a.t), F(p)}, kCompletion, kNoTruth);
                        all.push_back(T(p));
                    }
                    w.put(all.begin(), all.end(), kCompletion, a.t);
                }
                if (neg) {
                    all.assign(1, F(a.n));
                    for (AtomId q : r.neg_body) {
                        w.put({T(a.n), T(q)}, kCompletion, kNoTruth);
                        all.push_back(F(q));
                    }
                    w.put(all.begin(), all.end(), kCompletion, a.n);
                }
            } else if (i < R + n) {  // atom side: p <-> OR b_r (completion.cpp:116-130)
                const AtomId p = static_cast<AtomId>(i - R + 1);
                const auto& defs = prog.rules_of(p);
                if (defs.empty()) {
                    w.put({T(p)}, kCompletion, kNoTruth);
                    continue;
                }
                all.assign(1, T(p));
                for (std::uint32_t ri : defs) {
                    w.put({F(p), T(c.aux[ri].b)}, kCompletion, p);
                    all.push_back(F(c.aux[ri].b));
                }
                w.put(all.begin(), all.end(), kCompletion, kNoTruth);
            } else {  // integrity constraints (completion.cpp:132-138)
                const Rule& r = cons[i - R - n];
                if (r.body_overlaps()) continue;
                all.clear();
                for (AtomId p : r.pos_body) all.push_back(T(p));
                for (AtomId q : r.neg_body) all.push_back(F(q));
                w.put(all.begin(), all.end(), kConstraint, kNoTruth);
            }
        }
    });
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
    const NogoodSet& ns = comp.nogoods;
    std::string out;
    for (std::size_t k = 0; k < ns.size(); ++k) {
        out += '{';
        for (std::size_t i = 0; i < ns.length(k); ++i) {
            const std::int32_t l = ns.begin(k)[i];
            if (i) out += ", ";
            out += l > 0 ? "T " : "F ";
            out += comp.atom_name(lit_atom(l), prog);
        }
        out += "} ";
        out += origins[ns.origin[k]];
        out += '\n';
    }
    return out;
}

namespace {

// Stable LSD radix sort of positions 0..n-1 by key[] (11-bit digits, chunked
// histograms): the order of equal keys is the position order.
BigVec<std::uint32_t> radix_order(const BigVec<std::uint32_t>& key, std::uint32_t max_key) {
    const std::size_t n = key.size();
    BigVec<std::uint32_t> idx(n), tmp(n);
    parallel_chunks(n, 1 << 16, [&](unsigned, std::size_t b, std::size_t e) {
        for (std::size_t i = b; i < e; ++i) idx[i] = static_cast<std::uint32_t>(i);
    });
    constexpr unsigned kBits = 11, kBins = 1u << kBits;
    const unsigned parts = chunk_count(n, 1 << 16);
    std::vector<std::uint32_t> hist(static_cast<std::size_t>(parts) * kBins);
    for (unsigned shift = 0; shift == 0 || (max_key >> shift) != 0; shift += kBits) {
        std::fill(hist.begin(), hist.end(), 0u);
        parallel_chunks(n, 1 << 16, [&](unsigned c, std::size_t b, std::size_t e) {
            std::uint32_t* h = hist.data() + static_cast<std::size_t>(c) * kBins;
            for (std::size_t i = b; i < e; ++i) ++h[(key[idx[i]] >> shift) & (kBins - 1)];
        }, parts);
        std::uint32_t run = 0;  // digit-major, chunk-minor: stable
        for (unsigned d = 0; d < kBins; ++d)
            for (unsigned c = 0; c < parts; ++c) {
                std::uint32_t& h = hist[static_cast<std::size_t>(c) * kBins + d];
                const std::uint32_t x = h;
                h = run;
                run += x;
            }
        parallel_chunks(n, 1 << 16, [&](unsigned c, std::size_t b, std::size_t e) {
            std::uint32_t* h = hist.data() + static_cast<std::size_t>(c) * kBins;
            for (std::size_t i = b; i < e; ++i) tmp[h[(key[idx[i]] >> shift) & (kBins - 1)]++] = idx[i];
        }, parts);
        idx.swap(tmp);
        if (shift + kBits >= 32) break;
    }
    return idx;
}

}  // namespace

// NogoodStore::build (nogood_store.cpp:25-74): assertable units split out in
// order, the rest stable-sorted by length into CSR ids, occurrence lists per
// (literal, class) with ids ascending. Large stores use every host thread:
// the length sort is a chunked counting sort, the occurrence index a stable
// radix sort of the pool positions by key.
StaticStore build_store(const NogoodSet& ns, AtomId total_atoms) {
    const bool lapon = std::getenv("YAS_LAPS") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* w) {
        if (!lapon) return;
        auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "  store %s %.1f ms\n", w, std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    };
    StaticStore st;
    st.total_atoms = total_atoms;
    const std::size_t N0 = ns.size();
    std::vector<std::uint32_t> rest;
    rest.reserve(N0);
    std::size_t maxlen = 0;
    for (std::size_t k = 0; k < N0; ++k) {
        const std::size_t len = ns.length(k);
        if (len == 1 && ns.may_assert(k, -ns.begin(k)[0])) {
            st.units.push_back(ns.begin(k)[0]);
        } else {
            rest.push_back(static_cast<std::uint32_t>(k));
            maxlen = std::max(maxlen, len);
        }
    }
    // ids carry their length class in the top two bits of the device's
    // occurrence entries, and offsets are 32-bit (compile.hpp)
    std::uint64_t lits = 0;
    for (std::uint32_t k : rest) lits += ns.length(k);
    if (rest.size() >= (std::size_t{1} << 30) || lits > 0xFFFFFFFFull)
        throw std::length_error("store too large: at most 2^30 - 1 nogoods and 2^32 - 1 literals");
    const std::size_t N = rest.size();
    lap("units");
    // stable sort by length
    std::vector<std::uint32_t> order(N);
    if (maxlen <= 4096) {
        const unsigned parts = chunk_count(N, 1 << 15);
        const std::size_t bins = maxlen + 1;
        std::vector<std::uint64_t> hist(static_cast<std::size_t>(parts) * bins, 0);
        parallel_chunks(N, 1 << 15, [&](unsigned c, std::size_t b, std::size_t e) {
            for (std::size_t i = b; i < e; ++i) ++hist[c * bins + ns.length(rest[i])];
        }, parts);
        std::uint64_t run = 0;
        for (std::size_t l = 0; l < bins; ++l)
            for (unsigned c = 0; c < parts; ++c) {
                std::uint64_t& h = hist[c * bins + l];
                const std::uint64_t x = h;
                h = run;
                run += x;
            }
        parallel_chunks(N, 1 << 15, [&](unsigned c, std::size_t b, std::size_t e) {
            for (std::size_t i = b; i < e; ++i) order[hist[c * bins + ns.length(rest[i])]++] = rest[i];
        }, parts);
    } else {
        order = rest;
        std::stable_sort(order.begin(), order.end(),
                         [&](std::uint32_t a, std::uint32_t b) { return ns.length(a) < ns.length(b); });
    }
    lap("sort");
    st.off.assign(N + 1, 0);
    for (std::size_t i = 0; i < N; ++i) st.off[i + 1] = st.off[i] + static_cast<std::uint32_t>(ns.length(order[i]));
    st.pool.resize(st.off[N]);
    st.guard.resize(N);
    st.origin.resize(N);
    BigVec<std::uint32_t> owner(st.pool.size());  // CSR id of every pool position
    parallel_chunks(N, 1 << 14, [&](unsigned, std::size_t b, std::size_t e) {
        for (std::size_t i = b; i < e; ++i) {
            const std::uint32_t k = order[i];
            std::copy(ns.begin(k), ns.begin(k) + ns.length(k), st.pool.begin() + st.off[i]);
            std::fill(owner.begin() + st.off[i], owner.begin() + st.off[i + 1], static_cast<std::uint32_t>(i));
            st.guard[i] = ns.guard[k];
            st.origin[i] = ns.origin[k];
        }
    });
    lap("fill");
    for (std::uint32_t id = 0; id < N && st.length(id) == 1; ++id) st.unit_ids.push_back(static_cast<std::int32_t>(id));
    // occurrence index
    const std::size_t P = st.pool.size();
    const std::size_t keys = (2 * static_cast<std::size_t>(total_atoms) + 2) * 4;
    std::vector<std::uint32_t, NoInit<std::uint32_t>> key(P);
    parallel_chunks(P, 1 << 16, [&](unsigned, std::size_t b, std::size_t e) {
        for (std::size_t i = b; i < e; ++i) key[i] = lit_index(st.pool[i]) * 4 + length_class(st.length(owner[i]));
    });
    lap("keys");
    BigVec<std::uint32_t> pos;  // pool positions, grouped by key, ids ascending within a key
    if (P < (1u << 16)) {
        std::vector<std::uint32_t> cnt(keys + 1, 0);
        for (std::size_t i = 0; i < P; ++i) ++cnt[key[i] + 1];
        for (std::size_t k = 0; k < keys; ++k) cnt[k + 1] += cnt[k];
        pos.resize(P);
        for (std::size_t i = 0; i < P; ++i) pos[cnt[key[i]]++] = static_cast<std::uint32_t>(i);
    } else {
        pos = radix_order(key, static_cast<std::uint32_t>(keys - 1));
    }
    lap("radix");
    st.occ_off.assign(keys + 1, 0);
    parallel_chunks(P, 1 << 16, [&](unsigned, std::size_t b, std::size_t e) {
        for (std::size_t j = b; j < e; ++j) {  // occ_off[k] = first j with key >= k
            const std::uint32_t kj = key[pos[j]];
            const std::uint32_t kp = j == 0 ? 0u : key[pos[j - 1]] + 1;
            for (std::uint32_t k = kp; k <= kj; ++k) st.occ_off[k] = static_cast<std::uint32_t>(j);
        }
    });
    {
        const std::uint32_t last = P ? key[pos[P - 1]] + 1 : 0u;
        for (std::size_t k = last; k <= keys; ++k) st.occ_off[k] = static_cast<std::uint32_t>(P);
    }
    lap("occ_off");
    st.occ_ids.resize(P);
    st.occ_fat.resize(4 * P);
    BigVec<std::uint32_t> slot(P);  // pool position -> its occurrence entry
    parallel_chunks(P, 1 << 16, [&](unsigned, std::size_t b, std::size_t e) {
        for (std::size_t j = b; j < e; ++j) slot[pos[j]] = static_cast<std::uint32_t>(j);
    });
    // nogood by nogood (sequential reads), scattering its entries
    parallel_chunks(N, 1 << 14, [&](unsigned, std::size_t b, std::size_t e) {
        for (std::size_t id = b; id < e; ++id) {
            const std::uint32_t lo = st.off[id], hi = st.off[id + 1];
            const std::uint32_t cls = length_class(hi - lo);
            for (std::uint32_t at = lo; at < hi; ++at) {
                std::int32_t other[3] = {0, 0, 0};
                for (std::uint32_t q = lo, m = 0; q < hi && m < 3; ++q)
                    if (q != at) other[m++] = st.pool[q];
                const std::uint32_t j = slot[at];
                st.occ_ids[j] = static_cast<std::int32_t>(id);
                std::int32_t* f = st.occ_fat.data() + 4ull * j;
                f[0] = static_cast<std::int32_t>(static_cast<std::uint32_t>(id) | cls << 30);  // class in the top bits
                // binary / ternary: the truth guard; long: a third blocker (the guard is read when proposing)
                f[1] = cls == 3 ? other[2] : static_cast<std::int32_t>(st.guard[id]);
                f[2] = other[0];
                f[3] = other[1];
            }
        }
    });
    auto first_of_len = [&](std::uint32_t len) {
        std::uint32_t lo = 0, hi = st.size();  // lengths ascend with the id
        while (lo < hi) {
            const std::uint32_t mid = (lo + hi) / 2;
            if (st.length(mid) < len) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    st.bounds = {first_of_len(2), first_of_len(3), first_of_len(4), st.size()};
    lap("fat");
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
