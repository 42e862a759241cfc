// Device-resident solver state shared between the host launcher and the
// sm_100a kernels. One "slot" = the complete mutable state of one search
// (assignment, trail, Deps bitmaps, learned arena, pass scratch). The static
// store is shared read-only by all slots.
//
// Everything a search needs lives in device memory, so a kernel can stop at a
// loop boundary (model buffer full, time slice over) and a relaunch resumes
// exactly where it stopped; this is how models/traces stream to the host.
#pragma once

#include <cstdint>

namespace yas::dev {

constexpr std::uint32_t kAny = 0xFFFFFFFFu;  // kAnyTruth (nogood.hpp:72)
constexpr std::uint32_t kNone = 0u;          // kNoTruth  (nogood.hpp:73)

// reason[] encoding: >= 0 is the antecedent nogood id (Reason::propagated).
constexpr std::int32_t kReasonNone = -1;
constexpr std::int32_t kReasonDecision = -2;
constexpr std::int32_t kReasonUnit = -3;
constexpr std::int32_t kReasonCompletion = -4;

enum Status : std::uint32_t {
    kRunning = 0,
    kDone = 1,
    kYield = 2,
    kErrCapacity = 3,  // StoreCapacityError (nogood_store.cpp:83-85)
    kErrArena = 4,     // device arena too small: host re-runs with more memory
    kErrLogic = 5,     // res_learning without antecedent (learn.cpp:97-100)
    kErrValidate = 6,  // debug_validate fixpoint check failed (solver.cpp:77-82)
};

enum Phase : std::uint32_t { kIdle = 0, kInit = 1, kLoop = 2, kAfterModel = 3, kFinished = 4 };

// Coordination shared by every GPU (and process) of one enumeration or
// portfolio: the cube queue, the portfolio stop flag and the first finisher's
// claim. It lives in the home GPU's memory; the other GPUs reach it through
// NVLink peer mappings (CUDA IPC across processes) with system-scope atomics.
struct Fleet {
    std::uint32_t cube_next;  // next cube of the shared queue
    std::uint32_t stop;       // portfolio: a search finished, every other search ends
    std::uint32_t winner;     // portfolio: tag of the first finisher (~0 = none yet)
    std::uint32_t found;      // cube-parallel first models: models found so far by every search
};

struct Config {
    std::uint32_t mode;  // 0 fwd, 1 res
    std::uint32_t heur;  // 0 occ, 1 jw, 2 act
    double decay;
    std::uint32_t restarts;
    std::uint32_t W;  // deps words
    std::uint64_t restart_base;
    double restart_factor;
    std::uint64_t max_models;  // 0 = all
    std::uint32_t fanout;
    std::uint32_t debug_validate;
    std::uint64_t learned_capacity;
    std::uint32_t trace;
    std::uint32_t n_cubes;
    std::uint32_t cube_width;   // literals per cube
    std::uint64_t slice_ns;     // time slice per launch before yielding
    std::uint32_t count_lits;   // accumulate literals of checked nogoods (roofline accounting)
    unsigned long long* ptrace; // diagnostics: per-pass, per-block phase timestamps (null = off)
    std::uint32_t phase_prof;   // diagnostics: per-phase cycle buckets of single-CTA searches (YAS_PROFILE)
    // first-model portfolio: search k runs variant (pf_base + k) % 6 of
    // (mode, heuristic) = (v & 1, v >> 1); the first to finish stops the others
    std::uint32_t portfolio, pf_base;
    std::uint32_t warp_pass_t;  // single-CTA searches: passes with at most this many entries run in one warp
    Fleet* fleet;               // cube queue / portfolio claim shared across GPUs (null: this GPU's Shared)
    std::uint32_t fleet_tag;    // this GPU's portfolio claim tag base (slot index added)
};

// Read-only static store + program rules (host-built, uploaded once).
struct Static {
    std::uint32_t A;       // total atoms (program + aux)
    std::uint32_t n_prog;  // program atoms 1..n_prog
    std::uint32_t N;       // static CSR nogoods
    std::uint32_t n_units, n_uids, R;
    const std::uint32_t* off;   // N+1
    const std::int32_t* pool;   // literal codes
    const std::uint32_t* guard; // N
    const std::uint32_t* occ_off;  // (2A+2)*4+1, key = lit_index*4 + class
    const int4* occ;               // {id, guard, x, y} per occurrence (see StaticStore::occ_fat)
    const std::int32_t* units;     // static unit literals (nogood literal sigma)
    const std::int32_t* uids;      // static length-1 CSR ids
    const uint4* rules;            // (head, b, t, n | vacuous<<31)
    // decision scan: rule r packed in 8 bytes (head | t << 21 | n << 42 | vacuous << 63;
    // null when an atom id needs more than 21 bits) and the static occurrence
    // count of both literals of every atom
    const unsigned long long* rules8;
    const std::uint32_t* socc;
    const std::int32_t* cubes;     // n_cubes * cube_width nogood literals (0 = pad)
    // L2 cache policies (createpolicy, made once on the device): evict-first
    // for streamed occurrence entries, evict-last for claim words
    unsigned long long pol_first, pol_last;
};

struct Stats {
    unsigned long long decisions, propagations, conflicts, learned_count, learned_length_sum,
        restarts, models, passes, duplicate_learned, blocking_nogoods, res_learned, fwd_learned,
        fwd_fallbacks, uip_check_failures, fwd_decision_only_failures, asserting_failures,
        checks, searches, checked_lits;
};

// Per-slot control block. Mirrored into shared memory by single-CTA searches.
struct Ctl {
    std::uint32_t phase, status;
    std::uint32_t cdl, ts, F, cur, T, gen;
    std::uint32_t n_props, n_confl, n_pending, n_mbuf, n_trace;
    std::uint32_t learned_n, lpool_used, locc_used, lunits_n;
    std::uint32_t cube, epoch, stamp, pad0;
    // Propagator API: an op rejected on the device (seed past the frontier
    // capacity); the host raises it at the next result-returning call
    std::uint32_t op_err;
    std::uint32_t won;  // portfolio: this search claimed the first finish
    // Deps rows may hold words beyond their atom's level (Propagator API only:
    // Deps given to assign, propagation below the decision level); the next
    // reset then clears whole rows
    std::uint32_t rows_wide, variant;  // variant: portfolio (mode | heuristic << 1) of this search
    unsigned long long restart_threshold, conflicts_at_restart;
    double act_inc;
    std::uint32_t b[16];  // leader -> group broadcast scratch
    Stats st;
    unsigned long long prof[16];  // clock64 cycles per phase (leader view, after barriers)
    unsigned long long opsnap[4]; // counters at the start of the last propagation op: propagations, passes, checks, literals
    unsigned long long prof_t;
    unsigned long long done_ns;  // portfolio: global time at which this search finished
};

struct Caps {
    std::uint32_t items;   // claim/props/confl entries (>= N + learned)
    std::uint32_t tbits;   // expansion bitmap bits / lit_at entries
    std::uint32_t lcap;    // learned nogoods (arena)
    std::uint32_t lpool;   // learned literals
    std::uint32_t larena;  // learned occurrence arena (ids)
    std::uint32_t dupcap;  // power of two
    std::uint32_t mcap;    // models per slot buffer
    std::uint32_t tcap;    // trace records per slot
    std::uint32_t mwords;  // words per model bitset
};

// All mutable state of one search lives in one contiguous chunk of device
// memory; slot k starts at base + k * bytes. Arrays are addressed as
// chunk + constant offset, so kernels never load per-slot pointers.
struct SlotLayout {
    char* base;
    unsigned long long bytes;
    unsigned long long o_ctl, o_cells, o_tpos, o_reason, o_deps, o_dovf, o_trail, o_ldec, o_fr0, o_fr1, o_froff,
        o_claim, o_win, o_props, o_confl, o_pending, o_bitmap, o_litat, o_loff, o_lpool, o_lhdr, o_larena,
        o_lunits, o_ltot, o_act, o_dup, o_scratch, o_mark, o_merged, o_mbuf, o_mcube, o_tbuf, o_occat, o_gmirror, o_obat, o_frb;
};

#if defined(__CUDACC__)
#define YAS_HD __host__ __device__ __forceinline__
#else
#define YAS_HD inline
#endif

struct Slot {
    char* b;
    const SlotLayout* L;
    template <class T>
    YAS_HD T* at(unsigned long long off) const { return reinterpret_cast<T*>(b + off); }
    YAS_HD Ctl* ctl() const { return at<Ctl>(L->o_ctl); }
    YAS_HD std::int32_t* cells() const { return at<std::int32_t>(L->o_cells); }
    YAS_HD std::uint32_t* tpos() const { return at<std::uint32_t>(L->o_tpos); }
    YAS_HD std::int32_t* reason() const { return at<std::int32_t>(L->o_reason); }
    YAS_HD unsigned long long* deps() const { return at<unsigned long long>(L->o_deps); }  // word-major
    YAS_HD std::uint8_t* dovf() const { return at<std::uint8_t>(L->o_dovf); }
    YAS_HD std::int32_t* trail() const { return at<std::int32_t>(L->o_trail); }
    YAS_HD std::int32_t* ldec() const { return at<std::int32_t>(L->o_ldec); }
    YAS_HD std::int32_t* fr(std::uint32_t k) const { return at<std::int32_t>(k ? L->o_fr1 : L->o_fr0); }
    YAS_HD std::uint32_t* froff() const { return at<std::uint32_t>(L->o_froff); }
    YAS_HD unsigned long long* claim() const { return at<unsigned long long>(L->o_claim); }  // (~gen<<32)|min e
    YAS_HD unsigned long long* win() const { return at<unsigned long long>(L->o_win); }  // (~gen<<32)|(e<<1)|neg
    YAS_HD int4* props() const { return at<int4>(L->o_props); }  // (id, lit, e, -)
    YAS_HD std::int32_t* confl() const { return at<std::int32_t>(L->o_confl); }
    YAS_HD std::int32_t* pending() const { return at<std::int32_t>(L->o_pending); }
    YAS_HD std::uint32_t* bitmap() const { return at<std::uint32_t>(L->o_bitmap); }
    YAS_HD std::int32_t* litat() const { return at<std::int32_t>(L->o_litat); }
    YAS_HD std::uint32_t* occat() const { return at<std::uint32_t>(L->o_occat); }  // grid slots only
    // grid slots only: 2 bits per atom (bit 0 assigned, bit 1 true), 16 atoms per word
    YAS_HD std::uint32_t* gmirror() const { return at<std::uint32_t>(L->o_gmirror); }
    // grid slots only: static occurrence-list base of the winner at e, and of
    // frontier literal p (saves the offset lookup on the expansion path)
    YAS_HD std::uint32_t* obat() const { return at<std::uint32_t>(L->o_obat); }
    YAS_HD std::uint32_t* frb() const { return at<std::uint32_t>(L->o_frb); }
    YAS_HD std::uint32_t* loff() const { return at<std::uint32_t>(L->o_loff); }
    YAS_HD std::int32_t* lpool() const { return at<std::int32_t>(L->o_lpool); }
    YAS_HD std::uint32_t* lhdr() const { return at<std::uint32_t>(L->o_lhdr); }  // (2A+2)*4 * {ptr,size,cap}
    YAS_HD int4* larena() const { return at<int4>(L->o_larena); }  // learned occurrence entries
    YAS_HD std::int32_t* lunits() const { return at<std::int32_t>(L->o_lunits); }
    YAS_HD std::uint32_t* ltot() const { return at<std::uint32_t>(L->o_ltot); }
    YAS_HD double* act() const { return at<double>(L->o_act); }
    YAS_HD unsigned long long* dup() const { return at<unsigned long long>(L->o_dup); }
    YAS_HD std::int32_t* scratch() const { return at<std::int32_t>(L->o_scratch); }
    YAS_HD std::uint32_t* mark() const { return at<std::uint32_t>(L->o_mark); }
    YAS_HD unsigned long long* merged() const { return at<unsigned long long>(L->o_merged); }
    YAS_HD std::uint32_t* mbuf() const { return at<std::uint32_t>(L->o_mbuf); }
    YAS_HD std::uint32_t* mcube() const { return at<std::uint32_t>(L->o_mcube); }
    YAS_HD uint4* tbuf() const { return at<uint4>(L->o_tbuf); }
};

struct Shared {  // global (all-slot) coordination
    std::uint32_t cube_next;
    std::uint32_t stop;
    std::uint32_t bar_count, bar_gen;
    unsigned long long t_start;
    std::uint32_t winner;  // portfolio on one GPU without a fleet: first finisher's tag (~0 = none)
    std::uint32_t found;   // cube-parallel first models on one GPU without a fleet
    std::uint32_t partial_pad[25];
    // grid barrier: block b publishes the epoch of the barrier it reached
    std::uint32_t arrive[1024];
};

}  // namespace yas::dev
