"""ctypes wrapper of the oracle restatement (oracle/yasmin_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py, never by the product package.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libyasmin_oracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.check_call(["make", "-C", HERE, "port"], stdout=subprocess.DEVNULL)
        L = C.CDLL(LIB)
        L.ora_solve.restype = C.c_void_p
        L.ora_solve.argtypes = [C.c_char_p, C.c_size_t, C.c_uint64, C.c_int, C.c_int, C.c_uint32, C.c_int,
                                C.c_uint64, C.c_double, C.c_uint32, C.c_uint64, C.c_double]
        L.ora_propstore.restype = C.c_void_p
        L.ora_propstore.argtypes = [C.POINTER(C.c_int32), C.POINTER(C.c_uint32), C.c_size_t, C.c_uint32, C.c_uint32]
        L.ora_planted.restype = C.c_void_p
        L.ora_planted.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64]
        L.ora_free.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _take(ptr):
    s = C.cast(ptr, C.c_char_p).value.decode()
    lib().ora_free(ptr)
    return json.loads(s)


def solve(text: str, max_models: int = 1, mode: str = "fwd", heur: str = "occ", fanout: int = 1,
          restarts=None, deps_words: int = 16, capacity: int = 1 << 22, decay: float = 0.95) -> dict:
    b = text.encode()
    rb, rf = restarts if restarts else (100, 1.5)
    return _take(lib().ora_solve(b, len(b), max_models, 1 if mode == "res" else 0,
                                 {"occ": 0, "jw": 1, "act": 2}[heur], fanout, 1 if restarts else 0, rb, rf,
                                 deps_words, capacity, decay))


def propstore(nogoods, atoms: int, deps_words: int = 1) -> dict:
    lits, offs = [], [0]
    for ng in nogoods:
        lits.extend(ng)
        offs.append(len(lits))
    L = (C.c_int32 * max(1, len(lits)))(*lits)
    O = (C.c_uint32 * len(offs))(*offs)
    return _take(lib().ora_propstore(L, O, len(nogoods), atoms, deps_words))


def planted(atoms: int, nogoods: int, pct: int, seed: int = 0x1B00B5) -> dict:
    """Planted-store propagation (config 4b): checks/passes/propagations + trail digest."""
    return _take(lib().ora_planted(atoms, nogoods, pct, seed))
