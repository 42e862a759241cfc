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
