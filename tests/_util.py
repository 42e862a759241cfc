"""Shared test helpers: golden fixtures and config mapping."""
import functools
import json
import os

import paper_1909_01786_b200 as Y

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# trajectory fingerprint: every SolveStats counter the reference reports except
# wall time and watch_replacements (watches are not used on the device).
STAT_KEYS = ["decisions", "propagations", "conflicts", "learned_count", "learned_length_sum", "restarts", "models",
             "passes", "duplicate_learned", "blocking_nogoods", "res_learned", "fwd_learned", "fwd_fallbacks",
             "uip_check_failures", "fwd_decision_only_failures", "asserting_failures"]
HEUR = {"occ": Y.HeuristicKind.occurrence_count, "jw": Y.HeuristicKind.jeroslow_wang,
        "act": Y.HeuristicKind.activity}


@functools.lru_cache(maxsize=None)
def golden(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)


def config_from_opts(opts, **kw):
    """SolverConfig from the reference harness options (oracle/ref_harness.cpp)."""
    cfg = Y.SolverConfig(max_models=0, **kw)
    it = iter(opts)
    for o in it:
        v = next(it)
        if o == "--mode":
            cfg.mode = Y.LearnMode[v]
        elif o == "--heur":
            cfg.heuristic.kind = HEUR[v]
        elif o == "--decay":
            cfg.heuristic.activity_decay = float(v)
        elif o == "--restarts":
            b, f = v.split(":")
            cfg.restarts = Y.RestartPolicy(True, int(b), float(f))
        elif o == "--fanout":
            cfg.conflict_fanout = int(v)
        elif o == "--deps-words":
            cfg.deps_words = int(v)
        elif o == "--cap":
            cfg.learned_capacity = int(v)
        elif o == "-n":
            cfg.max_models = int(v)
    return cfg


def stats_diff(stats, expected):
    return {k: (getattr(stats, k), expected[k]) for k in STAT_KEYS if getattr(stats, k) != expected[k]}


def fnv(seq, h=0xcbf29ce484222325):
    """FNV-1a over 32-bit words (oracle/ref_harness.cpp cmd_planted digests)."""
    for c in seq:
        h = ((h ^ (int(c) & 0xFFFFFFFF)) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def trail_digests(p):
    """(trail, reason, Deps) digests of a Propagator's assignment in trail order,
    as the reference harness prints them: the literal sequence; the antecedent of
    each trail atom (-1 unless propagated); Deps word 0 (low, high) + overflow."""
    tr = p.trail()
    reasons = p.reasons()
    d0, ovf = p.deps(0)
    rs, ds = [], []
    for lit in tr:
        x = abs(lit)
        rs.append(reasons[x] if reasons[x] >= 0 else -1)
        ds += [d0[x] & 0xFFFFFFFF, d0[x] >> 32, 1 if ovf[x] else 0]
    return len(tr), fnv(tr), fnv(rs), fnv(ds)


def model_set_digest(models):
    """Order-independent digest of a set of answer sets (tests/golden/make_golden.py)."""
    words = []
    for m in sorted(tuple(sorted(x)) for x in models):
        words += list(m) + [0]
    return fnv(words)
