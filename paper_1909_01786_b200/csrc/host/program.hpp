// Ground program model, canonical-format parser and printer (host side of the
// drop-in boundary). Re-designed from the reference's contract, not copied:
//   GroundProgram / Rule           /root/reference/proj/include/aspine/program.hpp:41-77
//   parse_program (line format)    /root/reference/proj/src/program.cpp:141-179
//   print_program / tp_step        /root/reference/proj/src/program.cpp:181-229
// Atom ids are interned in first-occurrence order (head, then body left to
// right); bodies are kept sorted and duplicate-free. These ids are the ids the
// device store uses, so they must be identical to the reference's.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

namespace yas {

using AtomId = std::uint32_t;

struct Rule {
    AtomId head = 0;  // 0 marks an integrity constraint
    std::vector<AtomId> pos_body;
    std::vector<AtomId> neg_body;
    bool is_constraint() const { return head == 0; }
    bool is_fact() const { return head != 0 && pos_body.empty() && neg_body.empty(); }
    bool body_overlaps() const;
};

class Program {
public:
    Program() { names_.emplace_back(); }

    AtomId intern(std::string_view name) { return intern_hashed(name, name_hash(name)); }
    AtomId intern_hashed(std::string_view name, std::uint64_t hash);
    AtomId find(std::string_view name) const;
    static std::uint64_t name_hash(std::string_view name);
    void add_rule(Rule r);
    /// Bulk construction (parse_text): distinct names in id order with their
    /// hashes, then the statements in file order (bodies sorted, no repeats).
    void adopt(std::vector<std::string> names, std::vector<std::uint64_t> hashes, std::vector<Rule> stmts);

    AtomId atom_count() const { return static_cast<AtomId>(names_.size() - 1); }
    const std::string& name(AtomId id) const { return names_.at(id); }
    const std::vector<Rule>& rules() const { return rules_; }
    const std::vector<Rule>& constraints() const { return constraints_; }
    const std::vector<std::uint32_t>& rules_of(AtomId p) const { return rules_of_.at(p); }

private:
    std::vector<std::string> names_;  // [0] reserved
    std::vector<Rule> rules_;
    std::vector<Rule> constraints_;
    std::vector<std::vector<std::uint32_t>> rules_of_{1};
    // open-addressing name table keyed by name_hash: slot = hash high bits | id
    // (0 empty), so a probe touches the name only on a likely match
    std::vector<std::uint64_t> table_;
    std::vector<std::uint64_t> hashes_{0};  // per id
    void grow();

public:
    /// Hint: the slot `hash` probes first will be read soon (parse_text prefetches ahead).
    void prefetch(std::uint64_t hash) const {
        if (!table_.empty()) __builtin_prefetch(table_.data() + (hash & (table_.size() - 1)));
    }
};

struct ParseFailure : std::runtime_error {
    ParseFailure(int line_no, const std::string& what)
        : std::runtime_error("line " + std::to_string(line_no) + ": " + what), line(line_no) {}
    int line;
};

Program parse_text(std::string_view text);
std::string print_text(const Program& prog);
std::vector<AtomId> tp_step(const Program& prog, const std::vector<AtomId>& sorted_interp);
std::vector<std::string> diagnostics(const Program& prog);

/// Definitional answer-set check (reduct + least model), used for cfg.verify.
/// Semantics of /root/reference/proj/src/oracle.cpp:43-89.
bool is_answer_set(const Program& prog, const std::vector<AtomId>& sorted_model);

}  // namespace yas
