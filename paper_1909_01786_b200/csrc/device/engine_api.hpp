// Host interface of the device engine (used by the C-ABI layer).
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../host/compile.hpp"
#include "engine.cuh"

namespace yas {

struct RuleRec {
    std::uint32_t head, b, t, n;  // n carries the vacuous flag in bit 31
};

struct EngineProgram {
    const StaticStore* store = nullptr;
    std::vector<RuleRec> rules;
    std::uint32_t n_prog = 0;
};

struct EngineOptions {
    int device = 0;
    bool grid = false;           // one search over the whole GPU
    std::uint32_t slots = 1;     // concurrent searches (block mode)
    std::uint32_t lcap = 1u << 16;   // learned nogoods per slot (device arena)
    std::uint32_t lpool = 1u << 20;  // learned literals per slot
    std::uint32_t mcap = 4096;       // models buffered per slot between drains
    std::uint32_t tcap = 8192;       // trace records per slot between drains
    double slice_ms = 200.0;         // kernel time slice before a yield
    dev::Fleet* fleet = nullptr;     // shared cube queue / portfolio claim (device pointer valid on `device`)
    std::uint32_t fleet_tag = 0;     // portfolio claim tag base of this GPU
};

// The answer sets every slot buffered since the last drain (valid during the
// callback only): model m of slot s is the bitset bits + (s * stride + m) * nwords
// (bit a-1 set <=> program atom a true), found in cube cubes[s * stride + m].
struct EngineDrain {
    const std::uint32_t* bits = nullptr;
    const std::uint32_t* cubes = nullptr;
    const std::uint32_t* counts = nullptr;  // models per slot (0 for a slot that does not report)
    std::uint32_t n_slots = 0, stride = 0;
    std::size_t nwords = 0;
};

struct EngineResult {
    std::uint32_t status = dev::kDone;
    dev::Stats stats{};
    std::uint32_t launches = 0;
    double device_ms = 0.0;  // sum of kernel time (CUDA events)
    double wall_ms = 0.0;    // host wall time of the launch loop
    std::int32_t variant = -1;  // portfolio: (mode | heuristic << 1) of the search that finished first
    bool won = false;           // portfolio: a search of this run claimed the first finish
};

struct EngineCallbacks {
    std::function<bool(const EngineDrain&)> on_models;  // return false to stop early
    std::function<void(std::uint32_t mode, std::int32_t conflict, std::uint32_t len, std::uint32_t bj)> on_trace;
};

class DeviceStore;  // uploaded static store (shared by runs)

/// Full solve: one or many searches (cubes) to completion.
EngineResult engine_solve(const EngineProgram& prog, const dev::Config& cfg, const EngineOptions& opt,
                          const std::vector<std::int32_t>& cubes, std::uint32_t n_cubes,
                          std::uint32_t cube_width, const EngineCallbacks& cb);

/// Propagator-style session over one slot (tests + propagation benchmark).
class Session {
public:
    Session(const StaticStore& store, std::uint32_t deps_words, bool grid, int device,
            std::uint32_t lcap = 1024, std::uint32_t lpool = 1u << 16);
    ~Session();
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;

    void reset();
    void flush();  // launch the recorded ops now
    bool initial_propagation();
    bool propagate(std::uint32_t level);
    void push_decision(std::int32_t lit);
    void assign(const std::int32_t* lits, std::size_t n, std::uint32_t level, std::int32_t antecedent,
                const unsigned long long* deps, std::size_t n_deps, bool ovf);
    void seed(const std::int32_t* lits, std::size_t n);
    void clear_frontier();
    std::int32_t add_learned(const std::vector<std::int32_t>& lits);
    void set_count_lits(bool on);
    // diagnostics: per-pass x per-block phase timestamps of grid propagations
    void set_pass_trace(bool on);
    std::vector<unsigned long long> pass_trace(std::uint32_t& blocks) const;

    // read back
    const dev::Ctl& ctl() const;  // synchronises with the session's stream
    std::vector<std::int32_t> cells() const;
    std::vector<std::int32_t> trail() const;
    std::size_t trail_into(std::int32_t* out, std::size_t cap) const;  // returns the trail size
    std::vector<std::int32_t> reasons() const;
    std::vector<unsigned long long> deps_word(std::uint32_t w) const;
    std::vector<std::uint8_t> deps_overflow() const;
    std::vector<std::int32_t> conflicts() const;
    std::vector<std::int32_t> frontier() const;
    float last_ms() const { return last_ms_; }
    // cumulative host->device / device->host bytes of this session (counted at every copy)
    void transfers(unsigned long long& h2d, unsigned long long& d2h) const;
    std::uint32_t deps_words() const { return W_; }

    struct Impl;

private:
    void check_op_error() const;  // raises (and clears) an op the device rejected
    std::unique_ptr<Impl> impl_;
    std::uint32_t W_;
    float last_ms_ = 0.f;
};

std::string device_name(int device);

}  // namespace yas
