"""Synthetic ground programs of the BASELINE.json configurations.

All generators are deterministic and emit the reference's canonical text
format; CPU reference and GPU engine consume the same text. Seeds are pinned.
"""
from __future__ import annotations

import random


def queens(n: int) -> str:
    """n-queens: choice pair per cell, one queen per row, no two attacking."""
    q = lambda i, j: f"q({i},{j})"  # noqa: E731
    nq = lambda i, j: f"nq({i},{j})"  # noqa: E731
    out = []
    for i in range(1, n + 1):
        for j in range(1, n + 1):
            out.append(f"{q(i, j)} :- not {nq(i, j)}.")
            out.append(f"{nq(i, j)} :- not {q(i, j)}.")
    for i in range(1, n + 1):
        out.append(":- " + ", ".join(nq(i, j) for j in range(1, n + 1)) + ".")
    for i in range(1, n + 1):
        for j in range(1, n + 1):
            for k in range(j + 1, n + 1):
                out.append(f":- {q(i, j)}, {q(i, k)}.")
    for j in range(1, n + 1):
        for i in range(1, n + 1):
            for k in range(i + 1, n + 1):
                out.append(f":- {q(i, j)}, {q(k, j)}.")
    for i in range(1, n + 1):
        for j in range(1, n + 1):
            for d in range(1, n):
                if i + d <= n and j + d <= n:
                    out.append(f":- {q(i, j)}, {q(i + d, j + d)}.")
                if i + d <= n and j - d >= 1:
                    out.append(f":- {q(i, j)}, {q(i + d, j - d)}.")
    return "\n".join(out) + "\n"


def colouring(n: int, degree: float = 4.0, k: int = 3, seed: int = 1) -> str:
    """k-colouring of a random graph with n*degree/2 distinct undirected edges."""
    rng = random.Random(seed)
    m = int(n * degree / 2)
    edges, seen = [], set()
    while len(edges) < m:
        u, v = rng.randrange(1, n + 1), rng.randrange(1, n + 1)
        if u == v:
            continue
        key = (min(u, v), max(u, v))
        if key in seen:
            continue
        seen.add(key)
        edges.append(key)
    col = lambda v, c: f"col({v},{c})"  # noqa: E731
    ncol = lambda v, c: f"ncol({v},{c})"  # noqa: E731
    out = []
    for v in range(1, n + 1):
        for c in range(1, k + 1):
            out.append(f"{col(v, c)} :- not {ncol(v, c)}.")
            out.append(f"{ncol(v, c)} :- not {col(v, c)}.")
        out.append(":- " + ", ".join(ncol(v, c) for c in range(1, k + 1)) + ".")
        for c in range(1, k + 1):
            for d in range(c + 1, k + 1):
                out.append(f":- {col(v, c)}, {col(v, d)}.")
    for (u, v) in edges:
        for c in range(1, k + 1):
            out.append(f":- {col(u, c)}, {col(v, c)}.")
    return "\n".join(out) + "\n"


def hamiltonian(n: int, extra: float = 1.0, seed: int = 1) -> str:
    """Hamiltonian cycle on a random digraph with a planted cycle (avg out-degree 1+extra)."""
    rng = random.Random(seed)
    order = list(range(2, n + 1))
    rng.shuffle(order)
    cycle = [1] + order
    arcs, seen = [], set()
    for i in range(n):
        a = (cycle[i], cycle[(i + 1) % n])
        arcs.append(a)
        seen.add(a)
    target = int(n * (1 + extra))
    while len(arcs) < target:
        u, v = rng.randrange(1, n + 1), rng.randrange(1, n + 1)
        if u == v or (u, v) in seen:
            continue
        seen.add((u, v))
        arcs.append((u, v))
    arcs.sort()
    inn = lambda u, v: f"in({u},{v})"  # noqa: E731
    out_ = lambda u, v: f"out({u},{v})"  # noqa: E731
    lines = []
    for (u, v) in arcs:
        lines.append(f"{inn(u, v)} :- not {out_(u, v)}.")
        lines.append(f"{out_(u, v)} :- not {inn(u, v)}.")
    by_src, by_dst = {}, {}
    for (u, v) in arcs:
        by_src.setdefault(u, []).append(v)
        by_dst.setdefault(v, []).append(u)
    for u in sorted(by_src):
        vs = by_src[u]
        for i in range(len(vs)):
            for j in range(i + 1, len(vs)):
                lines.append(f":- {inn(u, vs[i])}, {inn(u, vs[j])}.")
    for v in sorted(by_dst):
        us = by_dst[v]
        for i in range(len(us)):
            for j in range(i + 1, len(us)):
                lines.append(f":- {inn(us[i], v)}, {inn(us[j], v)}.")
    for (u, v) in arcs:
        if u == 1:
            lines.append(f"r({v}) :- {inn(1, v)}.")
        else:
            lines.append(f"r({v}) :- r({u}), {inn(u, v)}.")
    for v in range(1, n + 1):
        lines.append(f":- not r({v}).")
    return "\n".join(lines) + "\n"


def random_program(atoms: int = 100_000, rules: int = 111_000, max_body: int = 3, seed: int = 2) -> str:
    """random_program-shaped program, no constraints (config 4a)."""
    rng = random.Random(seed)
    out = []
    for _ in range(rules):
        pos = [rng.randrange(1, atoms + 1) for _ in range(rng.randrange(0, max_body + 1))]
        neg = [rng.randrange(1, atoms + 1) for _ in range(rng.randrange(0, max_body + 1))]
        head = rng.randrange(1, atoms + 1)
        body = [f"p{a}" for a in pos] + [f"not p{a}" for a in neg]
        out.append(f"p{head} :- {', '.join(body)}." if body else f"p{head}.")
    return "\n".join(out) + "\n"


def pigeonhole(pigeons: int, holes: int) -> str:
    """Same schema as /root/reference/proj/tests/support/corpus.hpp:47-70."""
    out = []
    for p in range(1, pigeons + 1):
        for h in range(1, holes + 1):
            out.append(f"in({p},{h}) :- not out({p},{h}).")
            out.append(f"out({p},{h}) :- not in({p},{h}).")
    for p in range(1, pigeons + 1):
        out.append(":- " + ", ".join(f"out({p},{h})" for h in range(1, holes + 1)) + ".")
    for h in range(1, holes + 1):
        for p in range(1, pigeons + 1):
            for q in range(p + 1, pigeons + 1):
                out.append(f":- in({p},{h}), in({q},{h}).")
    return "\n".join(out) + "\n"


CONFIGS = {
    "queens8": lambda: queens(8),
    "colour2000": lambda: colouring(2000, 4.0, 3, 1),
    "ham200": lambda: hamiltonian(200, 1.0, 1),
    "rand100k": lambda: random_program(),
    "queens12": lambda: queens(12),
}
