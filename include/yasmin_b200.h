/*
 * yasmin-b200 — C-ABI of the B200-native yasmin core.
 *
 * This is the drop-in boundary for the reference solver ("aspine") program
 * loading / solve / enumerate path. Every entry point names the reference
 * interface it replaces (paths under /root/reference/proj). Plain C types
 * only; no torch or CUDA types cross this boundary. All functions are
 * synchronous and re-entrant (no globals), like aspine::solve.
 *
 * Errors: functions return a yas_status; on failure a message is written to
 * the caller's (err, err_cap) buffer when given. The reference's exception
 * classes map to status codes:
 *   ParseError (program.hpp:79-83)          -> YAS_ERR_PARSE (+ line number)
 *   StoreCapacityError (nogood_store.hpp:47)-> YAS_ERR_CAPACITY
 *   VerificationError (solver.hpp:109-111)  -> YAS_ERR_VERIFY
 *   std::logic_error (learn.cpp:97-100, solver.cpp:77-82) -> YAS_ERR_LOGIC
 */
#ifndef YASMIN_B200_H
#define YASMIN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum yas_status {
    YAS_OK = 0,
    YAS_ERR_PARSE = 1,
    YAS_ERR_CAPACITY = 2,
    YAS_ERR_VERIFY = 3,
    YAS_ERR_LOGIC = 4,
    YAS_ERR_DEVICE = 5, /* CUDA error / no device: the product has no CPU fallback */
    YAS_ERR_ARG = 6,
    YAS_ERR_IO = 7
} yas_status;

typedef struct yas_program yas_program;       /* aspine::GroundProgram */
typedef struct yas_result yas_result;         /* aspine::SolveResult */
typedef struct yas_store yas_store;           /* aspine::NogoodStore (static partition) */
typedef struct yas_propagator yas_propagator; /* aspine::Propagator + Assignment + Frontier */

/* ---- library ------------------------------------------------------------ */
const char* yas_version(void);
/* Number of CUDA devices visible (0 when none). */
int yas_device_count(void);
/* Device name into buf; returns YAS_ERR_DEVICE when unavailable. */
int yas_device_name(int device, char* buf, size_t cap);

/* ---- program loading: parse_program (program.hpp:87-88, program.cpp:141-179) */
int yas_program_parse(const char* text, size_t len, yas_program** out, int* err_line, char* err, size_t err_cap);
int yas_program_parse_file(const char* path, yas_program** out, int* err_line, char* err, size_t err_cap);
void yas_program_free(yas_program* p);
/* Programmatic construction (GroundProgram(), intern, add_rule; program.hpp:51-62):
 * an empty program, then atoms and rules in the caller's order. add_rule sorts and
 * dedups the bodies; head 0 is a constraint; ids must be interned already. */
yas_program* yas_program_create(void);
uint32_t yas_program_intern(yas_program* p, const char* name); /* 0 on failure */
int yas_program_add_rule(yas_program* p, uint32_t head, const uint32_t* pos, size_t n_pos, const uint32_t* neg,
                         size_t n_neg);
uint32_t yas_program_atom_count(const yas_program* p);       /* GroundProgram::atom_count */
uint32_t yas_program_rule_count(const yas_program* p);       /* rules().size() */
uint32_t yas_program_constraint_count(const yas_program* p); /* constraints().size() */
/* Atom name (GroundProgram::name), NUL-terminated, valid while p lives. */
const char* yas_program_atom_name(const yas_program* p, uint32_t id);
uint32_t yas_program_find(const yas_program* p, const char* name); /* GroundProgram::find */
/* Rule r: head, |pos|, |neg| and the bodies (program.hpp:41-49). */
int yas_program_rule(const yas_program* p, uint32_t r, uint32_t* head, const uint32_t** pos, uint32_t* n_pos,
                     const uint32_t** neg, uint32_t* n_neg);
/* Text outputs: return the full length; copy at most cap-1 bytes + NUL. */
size_t yas_program_print(const yas_program* p, char* buf, size_t cap);         /* print_program */
size_t yas_program_dump_nogoods(const yas_program* p, char* buf, size_t cap);  /* dump_nogoods */
size_t yas_program_store_csv(const yas_program* p, char* buf, size_t cap);     /* NogoodStore::dump_csv */
size_t yas_program_diagnostics(const yas_program* p, char* buf, size_t cap);   /* validate, '\n'-joined */
/* Completion ids (completion.hpp:48-80): out = {b, t, n, vacuous}. */
int yas_program_rule_aux(const yas_program* p, uint32_t rule, uint32_t out[4]);
uint32_t yas_program_total_atoms(const yas_program* p); /* AuxMap::total_atoms */
/* nogood_census vs compiled counts: census[3], counts[3] = rule, atom, constraint. */
int yas_program_census(const yas_program* p, uint64_t census[3], uint64_t counts[3]);
/* tp_step (program.hpp:96): interp sorted; out gets up to cap ids; returns count,
 * or SIZE_MAX when an id is 0 or above atom_count (the reference throws
 * std::out_of_range from vector::at there). */
size_t yas_program_tp_step(const yas_program* p, const uint32_t* interp, size_t n, uint32_t* out, size_t cap);
/* Cube split used by yas_solve when cfg.cube_atoms > 0. Choice atoms are
 * atoms a whose only rule is "a :- not b." with "b :- not a." present,
 * followed by every other atom that heads a rule (T a is then the passive unit
 * nogood {F a}, -a below). The
 * first depth*k of them form `depth` nested ladders of width k: per level a
 * cube fixes (F a_0..F a_{i-1}, T a_i) or all F, so the (k+1)^depth cubes
 * partition the answer sets. depth 0 = smallest depth with >= want cubes.
 * Cube c runs on rank c % world. Each cube is width = depth*k unit-nogood
 * literals (0 = none): +a (":- a."), +b (":- b.", i.e. T a) or -a (":- not a."). k = 0: the
 * automatic split of a plain enumeration (ladders over at-least-one groups). Returns this
 * rank's cube count; host-only. */
size_t yas_program_cubes(const yas_program* p, uint32_t k, uint32_t depth, uint32_t want, int rank, int world,
                         int32_t* out, size_t cap, uint32_t* width);
/* verify_model (solver.hpp:116): 1 when the sorted atom set is an answer set, 0
 * when not, -YAS_ERR_ARG when an id is 0 or above atom_count. */
int yas_verify_model(const yas_program* p, const uint32_t* atom_ids, size_t n);

/* ---- solve / enumerate: solve(GroundProgram, SolverConfig) (solver.hpp:113) */
typedef struct yas_trace {
    int mode; /* 0 fwd, 1 res */
    int32_t conflict_id;
    uint64_t learned_length;
    uint32_t backjump_level;
} yas_trace; /* ConflictTrace, solver.hpp:37-42 */
typedef void (*yas_trace_fn)(const yas_trace* t, void* user);

/* ---- fleets: one enumeration / portfolio over the GPUs of several processes --
 * (no reference counterpart: the reference is single-process).
 * Rank 0's GPU holds the shared cube queue and the portfolio claim; every other
 * rank maps it through CUDA IPC (NVLink peer access) and takes cubes from it
 * with system-scope atomics, so work is balanced across GPUs while it runs.
 * The only collective of a solve is the final all-reduce of model counts,
 * error and termination flags: NCCL (yas_fleet_create_nccl), or the caller's
 * own transport (yas_fleet_create with two callbacks, e.g. torch.distributed).
 * If a rank cannot map rank 0's block, cubes are dealt statically (c % world). */
typedef struct yas_fleet yas_fleet;
/* In place over all ranks; op 0 sum, 1 max, 2 min. Return 0 on success. */
typedef int (*yas_allreduce_fn)(uint64_t* vals, size_t n, int op, void* user);
/* In place: root's bytes to every rank. Return 0 on success. */
typedef int (*yas_broadcast_fn)(void* buf, size_t bytes, int root, void* user);
/* ncclGetUniqueId; rank 0 creates it and the caller hands the 128 bytes to every rank. */
int yas_fleet_unique_id(uint8_t out[128], char* err, size_t err_cap);
int yas_fleet_create_nccl(const uint8_t unique_id[128], int rank, int world, int device, yas_fleet** out, char* err,
                          size_t err_cap);
int yas_fleet_create(int rank, int world, int device, yas_allreduce_fn allreduce, yas_broadcast_fn broadcast,
                     void* user, yas_fleet** out, char* err, size_t err_cap);
void yas_fleet_free(yas_fleet* f);
/* dynamic = 1 when every rank takes cubes from rank 0's shared queue. */
int yas_fleet_info(const yas_fleet* f, int* rank, int* world, int* device, int* dynamic);
int yas_fleet_allreduce(yas_fleet* f, uint64_t* vals, size_t n, int op, char* err, size_t err_cap);

typedef struct yas_config {
    /* SolverConfig (solver.hpp:44-57) */
    int mode;              /* 0 fwd (default), 1 res */
    int heuristic;         /* 0 occ (default), 1 jw, 2 act */
    double activity_decay; /* 0.95 */
    unsigned workers;      /* accepted for API parity; the device decides parallelism */
    int restarts_enabled;
    uint64_t restart_base;  /* 100 */
    double restart_factor;  /* 1.5 */
    uint64_t max_models;    /* 1; 0 = enumerate all */
    uint32_t deps_words;    /* 16 */
    uint32_t conflict_fanout; /* 1 */
    uint64_t seed;          /* accepted, unused (as in the reference) */
    int verify;
    int debug_validate;
    uint64_t learned_capacity; /* 1 << 22 */
    yas_trace_fn trace;
    void* trace_user;
    /* device extensions */
    int device;          /* CUDA ordinal */
    int engine;          /* 0 auto, 1 one CTA per search, 2 whole-grid search */
    uint32_t cube_atoms; /* enumeration split: ladder width k over choice atoms (0 = single search); with
                            max_models >= 1, the first max_models answer sets found by any cube search */
    uint32_t cube_depth; /* ladder levels (0 = auto: enough cubes for every search slot) */
    uint32_t slots;      /* concurrent searches per GPU for cubes (0 = auto) */
    int rank, world;     /* cube partition across processes/GPUs: cube i runs on rank i % world */
    uint32_t portfolio;  /* first-model portfolio (max_models == 1 without cubes): this many
                            concurrent searches with diverse (mode, heuristic), variant (v0 + rank * portfolio
                            + k) % 6 with v0 = mode | heuristic << 1 first; the first search to finish reports
                            its model or UNSAT (0 or 1 = off) */
    uint32_t count_lits; /* 1: exact literal counts of the checked nogoods in yas_stats.checked_lits
                            (roofline accounting; one extra load per decided long nogood, off by default) */
    uint32_t n_devices;  /* cube enumeration / portfolio over this many GPUs of this process (0 or 1: `device`
                            only); cubes come from one queue in the first GPU's memory (NVLink peer access) */
    const int* devices;  /* n_devices CUDA ordinals (NULL: device, device + 1, ...); an ordinal may repeat */
    int reference_order; /* 1: an enumeration (max_models == 0) is one search with the reference's model
                            order and trajectory. 0 (default): a program with >= 16 even-loop choice pairs
                            is enumerated as cubes over the GPU(s) — ladders over its "at least one of"
                            constraint groups (a queens row, a node's colours), else 8 pairs wide; same
                            answer sets and count, models in cube order (deterministic). Tracing, or
                            engine 2 (one whole-GPU search at a time), keeps the reference order. */
    yas_fleet* fleet;    /* several processes share the enumeration / portfolio; overrides rank, world and
                            device (one GPU per process). Every rank calls yas_solve with the same program
                            and options; each returns the models its GPU found. */
} yas_config;

void yas_config_default(yas_config* cfg);

typedef struct yas_stats {
    /* SolveStats (solver.hpp:59-93) */
    uint64_t decisions, propagations, conflicts, learned_count, learned_length_sum, restarts, models;
    double wall_ms;
    uint64_t passes, watch_replacements, duplicate_learned, blocking_nogoods, res_learned, fwd_learned,
        fwd_fallbacks, uip_check_failures, fwd_decision_only_failures, asserting_failures;
    /* device extensions */
    uint64_t checks;   /* nogood checks (deduplicated propagation items) */
    uint64_t searches; /* searches run (cubes) */
    uint64_t launches; /* kernel launches */
    double device_ms;  /* kernel time, CUDA events */
    uint64_t cubes;    /* cubes assigned to this rank */
    uint64_t checked_lits; /* literals of the checked nogoods (algorithmic traffic) */
    int64_t portfolio_variant; /* winning (mode | heuristic << 1) of a portfolio run, -1 otherwise */
    uint64_t fleet_models;     /* models found by every GPU / rank of the solve (all-reduced) */
    uint32_t devices;          /* GPUs of this process that ran */
    uint32_t fleet_ranks;      /* processes of the fleet (1 without) */
    int32_t fleet_winner;      /* portfolio: rank whose search finished first (-1: none / not a portfolio) */
    uint32_t pad;
} yas_stats;

int yas_solve(const yas_program* p, const yas_config* cfg, yas_result** out, char* err, size_t err_cap);
int yas_result_status(const yas_result* r); /* SolveStatus: 0 sat, 1 unsat */
uint64_t yas_result_model_count(const yas_result* r);
/* Model m: sorted program atom ids (Model::atom_ids); n receives the size. */
const uint32_t* yas_result_model(const yas_result* r, uint64_t m, uint32_t* n);
uint32_t yas_result_model_cube(const yas_result* r, uint64_t m);
/* All models at once: ids of model m are ids[offsets[m] .. offsets[m+1]) (offsets
 * has model_count + 1 entries), cubes[m] its cube; any output may be NULL.
 * Returns the total number of ids (copies at most cap). */
size_t yas_result_models_flat(const yas_result* r, uint32_t* ids, size_t cap, uint64_t* offsets, uint32_t* cubes);
void yas_result_stats(const yas_result* r, yas_stats* s);
void yas_result_free(yas_result* r);
/* emit_stats / stats_csv_header (solver.hpp:131-133); ctx strings may be NULL. */
size_t yas_stats_csv_header(char* buf, size_t cap);
size_t yas_emit_stats(const yas_stats* s, const char* instance, const char* mode, const char* heur,
                      unsigned workers, int status, uint64_t models, int csv, char* buf, size_t cap);

/* ---- low level: NogoodStore::build (nogood_store.hpp:64-65) ------------- */
/* Nogood k = lits[offsets[k] .. offsets[k+1]), canonicalised like Nogood::make
 * (nogood.hpp:80-87); a vacuous set is YAS_ERR_ARG. guards may be NULL
 * (kAnyTruth = 0xFFFFFFFF); origins may be NULL (constraint). */
int yas_store_build(const int32_t* lits, const uint32_t* offsets, size_t n_nogoods, const uint32_t* guards,
                    const uint8_t* origins, uint32_t total_atoms, yas_store** out, char* err, size_t err_cap);
void yas_store_free(yas_store* s);
uint32_t yas_store_size(const yas_store* s);
uint32_t yas_store_total_atoms(const yas_store* s);
size_t yas_store_dump_csv(const yas_store* s, char* buf, size_t cap);
/* CSR nogood `id` (NogoodStore::literals / truth_guard / origin): copies at most cap
 * literal codes, returns the length (0 for an id out of range); origin 0
 * completion, 1 constraint, 2 learned. */
size_t yas_store_nogood(const yas_store* s, uint32_t id, int32_t* lits, size_t cap, uint32_t* guard, uint8_t* origin);
/* static_units (literals), unit_ids, static_class_bounds */
size_t yas_store_units(const yas_store* s, int32_t* out, size_t cap);
size_t yas_store_unit_ids(const yas_store* s, int32_t* out, size_t cap);
void yas_store_bounds(const yas_store* s, uint32_t out[4]);
/* occurrences(l, class) (nogood_store.hpp:98-100) */
size_t yas_store_occurrences(const yas_store* s, int32_t lit, uint32_t cls, int32_t* out, size_t cap);
/* Planted benchmark store: builds the store and
 * the seeded frontier; decision = H-literal of atom 1. */
int yas_store_planted(uint32_t atoms, uint64_t nogoods, uint32_t pct, uint64_t seed, yas_store** out,
                      int32_t** seeded, size_t* n_seeded, int32_t* decision);
void yas_free_ints(int32_t* p);

/* ---- low level: Propagator (propagate.hpp:54-97) over one device search -- */
typedef struct yas_outcome {
    int violated;
    uint64_t propagations, passes, checks, checked_lits;
    uint32_t n_conflicts;
    float device_ms;
} yas_outcome; /* PropagationOutcome (+ device extras) */

int yas_propagator_create(const yas_store* s, uint32_t deps_words, int engine, int device, yas_propagator** out,
                          char* err, size_t err_cap);
void yas_propagator_free(yas_propagator* p);
int yas_propagator_reset(yas_propagator* p); /* fresh Assignment + Frontier */
/* Calls that only change device state (reset, push_decision, assign, seed) are
 * recorded and launched together with the next call that returns a result
 * (one kernel, one upload). flush launches the recorded calls now (no
 * reference counterpart; used to time a propagation alone). */
int yas_propagator_flush(yas_propagator* p);
int yas_propagator_initial(yas_propagator* p, yas_outcome* o);                 /* initial_propagation */
int yas_propagator_propagate(yas_propagator* p, uint32_t level, yas_outcome* o); /* propagate_and_check */
int yas_propagator_push_decision(yas_propagator* p, int32_t lit);              /* Assignment::push_decision */
/* Assignment::assign_propagated for each literal (same level/deps/antecedent). */
int yas_propagator_assign(yas_propagator* p, const int32_t* lits, size_t n, uint32_t level,
                          const uint64_t* deps, uint32_t n_deps, int overflow, int32_t antecedent);
int yas_propagator_seed(yas_propagator* p, const int32_t* lits, size_t n); /* Frontier::seed / last.push_back */
int yas_propagator_clear_frontier(yas_propagator* p);                     /* Frontier::clear */
/* Bytes this propagator has moved host->device (staged inputs, kernel arguments) and
 * device->host (control blocks, read-backs) since it was created, counted at each copy. */
int yas_propagator_transfers(const yas_propagator* p, uint64_t* h2d, uint64_t* d2h);
/* NogoodStore::add_learned (nogood_store.cpp:81-107): the literals are
 * canonicalised like Nogood::make; returns the new id, or -1 for an empty or
 * vacuous set, a literal 0 or an atom above the store's total_atoms (message
 * in yas_propagator_last_error). */
int32_t yas_propagator_add_learned(yas_propagator* p, const int32_t* lits, size_t n);
/* Message of the last failed propagator call (CUDA error, invalid argument, a
 * seed beyond A + 1 frontier literals — the latter is detected on the device
 * and reported by the next result-returning call). Returns the full length. */
size_t yas_propagator_last_error(const yas_propagator* p, char* buf, size_t cap);
/* Exact literal counts of checked nogoods in yas_outcome.checked_lits (roofline
 * accounting; costs an extra load per decided long nogood, off by default). */
int yas_propagator_count_literals(yas_propagator* p, int on);
/* Read back. cells: A+1 entries (cell[p] = +-level). reasons: >= 0 antecedent,
 * -1 none, -2 decision, -3 unit, -4 completion. deps: word w of every atom. */
uint32_t yas_propagator_atoms(const yas_propagator* p);
int yas_propagator_cells(const yas_propagator* p, int32_t* out);
int yas_propagator_reasons(const yas_propagator* p, int32_t* out);
int yas_propagator_deps(const yas_propagator* p, uint32_t word, uint64_t* out, uint8_t* overflow);
size_t yas_propagator_trail(const yas_propagator* p, int32_t* out, size_t cap);
size_t yas_propagator_conflicts(const yas_propagator* p, int32_t* out, size_t cap);
size_t yas_propagator_frontier(const yas_propagator* p, int32_t* out, size_t cap);
uint32_t yas_propagator_level(const yas_propagator* p);
/* Diagnostics (no reference counterpart): SM clock cycles spent per phase of the
 * propagation loop since the propagator was created, measured by the leader
 * thread between barriers: [1] frontier offsets, [2] expand+evaluate,
 * [3] resolve, [4] apply, [5] compact. */
int yas_propagator_profile(const yas_propagator* p, uint64_t out[16]);
/* Diagnostics: on = 1/0 enables/disables per-pass, per-block phase timestamps
 * (global timer, ns) for whole-grid propagations, -1 leaves it; out (when
 * given) receives 64 passes x blocks x 10 stamps: [0] pass start, [1] expand
 * done, [2] after barrier, [3] resolve done, [4] after barrier, [5] select
 * done, [6] after barrier, [7] place done, [8] after barrier; stamp [9] of
 * block 0 = T << 32 | F of the pass. */
int yas_propagator_pass_trace(yas_propagator* p, int on, uint64_t* out, size_t cap, uint32_t* blocks);

#ifdef __cplusplus
}
#endif

#endif /* YASMIN_B200_H */
