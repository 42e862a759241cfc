"""C-ABI surface: the library loads and exports every symbol include/yasmin_b200.h declares."""
import ctypes
import os
import re

import pytest

import paper_1909_01786_b200 as Y
from paper_1909_01786_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "yasmin_b200.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(yas_[a-z0-9_]+)\s*\(", text)) - {"yas_trace_fn"})


def test_header_symbols_exported():
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 50
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_native.EXPORTS) == syms


def test_version_and_config_defaults():
    L = _native.lib()
    assert b"sm_100a" in L.yas_version()
    c = _native.yas_config()
    L.yas_config_default(ctypes.byref(c))
    # SolverConfig defaults (solver.hpp:44-57)
    assert (c.mode, c.heuristic, c.max_models, c.deps_words, c.conflict_fanout) == (0, 0, 1, 16, 1)
    assert c.activity_decay == 0.95 and c.restart_base == 100 and c.restart_factor == 1.5
    assert c.learned_capacity == 1 << 22 and c.world == 1


@pytest.mark.skipif(Y.device_count() > 0, reason="a GPU is present")
def test_no_cpu_fallback_without_device():
    p = Y.parse_program("a :- not b.\nb :- not a.\n")
    with pytest.raises(Y.DeviceError):
        Y.solve(p)
    s = Y.NogoodStore.build([[1, 2]], 2)
    with pytest.raises(Y.DeviceError):
        Y.Propagator(s)


def test_parse_errors_map_to_status():
    with pytest.raises(Y.ParseError) as e:
        Y.parse_program("a.\nb :- ,c.\n")
    assert e.value.line == 2
    with pytest.raises(OSError):
        Y.parse_file("/nonexistent/file.lp")
