"""Host-side mirror of the reference solver's public API over the C-ABI.

Names, argument meaning and error behaviour follow the reference ("aspine"):

  parse_program            /root/reference/proj/include/aspine/program.hpp:87-88
  GroundProgram            program.hpp:51-77           ParseError  program.hpp:79-83
  SolverConfig             solver.hpp:44-57            solve       solver.hpp:113
  SolveResult/Model/Stats  solver.hpp:59-107           verify_model solver.hpp:116
  emit_stats/csv header    solver.hpp:131-133
  NogoodStore.build        nogood_store.hpp:64-65      Propagator  propagate.hpp:54-97
  StoreCapacityError       nogood_store.hpp:47         VerificationError solver.hpp:109

Everything computes on the GPU through ``libyasmin_b200.so``; this module only
marshals arguments.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from collections.abc import Sequence
from typing import Callable, Iterable, List, Optional

import numpy as np

from . import _native as N

kAnyTruth = 0xFFFFFFFF
kNoTruth = 0


class ParseError(RuntimeError):
    def __init__(self, line: int, what: str):
        super().__init__(what)
        self.line = line


class StoreCapacityError(RuntimeError):
    pass


class VerificationError(RuntimeError):
    pass


class LogicError(RuntimeError):
    """std::logic_error in the reference (res_learning, debug_validate)."""


class DeviceError(RuntimeError):
    """No usable CUDA device / CUDA failure. There is no CPU fallback."""


def _raise(code: int, msg: bytes, line: int = 0):
    text = msg.decode(errors="replace") if msg else f"error {code}"
    if code == 1:
        raise ParseError(line, text)
    exc = {2: StoreCapacityError, 3: VerificationError, 4: LogicError, 5: DeviceError, 7: OSError}.get(code, ValueError)
    raise exc(text)


def _text(fn, *args) -> str:
    n = fn(*args, None, 0)
    buf = C.create_string_buffer(n + 1)
    fn(*args, buf, n + 1)
    return buf.value.decode()


class LearnMode(enum.IntEnum):
    fwd = 0
    res = 1


class HeuristicKind(enum.IntEnum):
    occurrence_count = 0
    jeroslow_wang = 1
    activity = 2


class SolveStatus(enum.IntEnum):
    sat = 0
    unsat = 1


def to_string(x) -> str:
    if isinstance(x, LearnMode):
        return "fwd" if x == LearnMode.fwd else "res"
    if isinstance(x, HeuristicKind):
        return {0: "occ", 1: "jw", 2: "act"}[int(x)]
    if isinstance(x, SolveStatus):
        return "SAT" if x == SolveStatus.sat else "UNSAT"
    raise TypeError(x)


@dataclass
class HeuristicConfig:
    kind: HeuristicKind = HeuristicKind.occurrence_count
    activity_decay: float = 0.95


@dataclass
class RestartPolicy:
    enabled: bool = False
    base: int = 100
    factor: float = 1.5


@dataclass
class ConflictTrace:
    mode_used: LearnMode
    conflict_id: int
    learned_length: int
    backjump_level: int


@dataclass
class SolverConfig:
    mode: LearnMode = LearnMode.fwd
    heuristic: HeuristicConfig = field(default_factory=HeuristicConfig)
    workers: int = 1
    restarts: RestartPolicy = field(default_factory=RestartPolicy)
    max_models: int = 1
    deps_words: int = 16
    conflict_fanout: int = 1
    seed: int = 0
    verify: bool = False
    debug_validate: bool = False
    learned_capacity: int = 1 << 22
    trace: Optional[Callable[[ConflictTrace], None]] = None
    # device extensions
    device: int = 0
    engine: str = "auto"  # "auto" | "block" | "grid"
    cube_atoms: int = 0
    cube_depth: int = 0
    slots: int = 0
    rank: int = 0
    world: int = 1
    portfolio: int = 0  # first-model portfolio: concurrent searches with diverse (mode, heuristic)
    count_lits: bool = False  # exact literals of checked nogoods in stats.checked_lits (roofline accounting)
    devices: Optional[Sequence[int]] = None  # cube enumeration / portfolio over these GPUs of this process
    reference_order: bool = False  # enumerate as one search in the reference's model order (no automatic cubes)
    fleet: Optional["Fleet"] = None  # several processes share the enumeration / portfolio (one GPU each)


_STAT_FIELDS = ["decisions", "propagations", "conflicts", "learned_count", "learned_length_sum", "restarts",
                "models", "wall_ms", "passes", "watch_replacements", "duplicate_learned", "blocking_nogoods",
                "res_learned", "fwd_learned", "fwd_fallbacks", "uip_check_failures",
                "fwd_decision_only_failures", "asserting_failures", "checks", "searches", "launches",
                "device_ms", "cubes", "checked_lits", "portfolio_variant", "fleet_models", "devices",
                "fleet_ranks", "fleet_winner"]


@dataclass
class SolveStats:
    decisions: int = 0
    propagations: int = 0
    conflicts: int = 0
    learned_count: int = 0
    learned_length_sum: int = 0
    restarts: int = 0
    models: int = 0
    wall_ms: float = 0.0
    passes: int = 0
    watch_replacements: int = 0
    duplicate_learned: int = 0
    blocking_nogoods: int = 0
    res_learned: int = 0
    fwd_learned: int = 0
    fwd_fallbacks: int = 0
    uip_check_failures: int = 0
    fwd_decision_only_failures: int = 0
    asserting_failures: int = 0
    checks: int = 0
    searches: int = 0
    launches: int = 0
    device_ms: float = 0.0
    cubes: int = 0
    checked_lits: int = 0
    portfolio_variant: int = -1
    fleet_models: int = 0  # models of every GPU / rank of the solve (all-reduced)
    devices: int = 1       # GPUs of this process that ran
    fleet_ranks: int = 1   # processes of the fleet
    fleet_winner: int = -1  # portfolio: rank whose search finished first

    def avg_learned_len(self) -> float:
        return 0.0 if self.learned_count == 0 else self.learned_length_sum / self.learned_count

    def wall_seconds(self) -> float:
        return self.wall_ms / 1000.0

    def per_second(self, counter: int) -> float:
        return 0.0 if self.wall_ms <= 0.0 else counter / self.wall_seconds()

    def propagations_per_sec(self) -> float:
        return self.per_second(self.propagations)

    def decisions_per_sec(self) -> float:
        return self.per_second(self.decisions)

    def learned_per_sec(self) -> float:
        return self.per_second(self.learned_count)

    def _c(self) -> N.yas_stats:
        s = N.yas_stats()
        for f in _STAT_FIELDS:
            setattr(s, f, getattr(self, f))
        return s


class Model:
    """Model (solver.hpp:96-99): sorted atom ids; names sorted lexicographically
    (resolved on first access, so enumerating many models stays cheap)."""

    __slots__ = ("atom_ids", "_atoms", "_prog")

    def __init__(self, atom_ids: List[int], atoms: Optional[List[str]] = None, prog: "Optional[GroundProgram]" = None):
        self.atom_ids = atom_ids
        self._atoms = atoms
        self._prog = prog

    @property
    def atoms(self) -> List[str]:
        if self._atoms is None:
            self._atoms = sorted(self._prog.name(a) for a in self.atom_ids) if self._prog is not None else []
        return self._atoms

    def __eq__(self, other):
        return isinstance(other, Model) and self.atom_ids == other.atom_ids and self.atoms == other.atoms

    def __repr__(self):
        return f"Model(atom_ids={self.atom_ids!r}, atoms={self.atoms!r})"


class ModelList(Sequence):
    """The models of a SolveResult as a read-only sequence over the flat id
    buffer; Model objects are built on access (an enumeration may return tens
    of thousands of models that the caller only counts)."""

    def __init__(self, ids: np.ndarray, offs: np.ndarray, count: int, prog: "GroundProgram"):
        self._ids, self._offs, self._n, self._prog = ids, offs, count, prog

    def __len__(self) -> int:
        return self._n

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(self._n))]
        if i < 0:
            i += self._n
        if not 0 <= i < self._n:
            raise IndexError(i)
        return Model(self._ids[int(self._offs[i]):int(self._offs[i + 1])].tolist(), None, self._prog)

    def __eq__(self, other):
        return list(self) == list(other)

    def __repr__(self):
        return f"ModelList({len(self)} models)"


@dataclass
class SolveResult:
    models: List[Model]
    stats: SolveStats
    status: SolveStatus
    cubes: List[int] = field(default_factory=list)


class GroundProgram:
    """Handle to a parsed program (immutable, shareable read-only)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        self._names: Optional[List[str]] = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            N.lib().yas_program_free(h)
            self._h = C.c_void_p(0)

    def atom_count(self) -> int:
        return N.lib().yas_program_atom_count(self._h)

    def name(self, atom_id: int) -> str:
        if self._names is None:
            L = N.lib()
            self._names = [""] + [L.yas_program_atom_name(self._h, i).decode() for i in range(1, self.atom_count() + 1)]
        return self._names[atom_id]

    def find(self, name: str) -> int:
        return N.lib().yas_program_find(self._h, name.encode())

    def rule_count(self) -> int:
        return N.lib().yas_program_rule_count(self._h)

    def constraint_count(self) -> int:
        return N.lib().yas_program_constraint_count(self._h)

    def total_atoms(self) -> int:
        return N.lib().yas_program_total_atoms(self._h)

    def _rule(self, r: int):
        head = C.c_uint32()
        pos, neg = C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint32)()
        np_, nn = C.c_uint32(), C.c_uint32()
        if N.lib().yas_program_rule(self._h, r, C.byref(head), C.byref(pos), C.byref(np_), C.byref(neg),
                                    C.byref(nn)) != 0:
            raise IndexError(r)
        return head.value, list(pos[: np_.value]), list(neg[: nn.value])

    def rules(self):
        """[(head, pos_body, neg_body)] in rule order (GroundProgram::rules)."""
        return [self._rule(r) for r in range(self.rule_count())]

    def constraints(self):
        nr = self.rule_count()
        return [self._rule(nr + c) for c in range(self.constraint_count())]

    def rules_of(self, atom: int):
        return [i for i, (h, _, _) in enumerate(self.rules()) if h == atom]

    def rule_aux(self, rule: int):
        out = (C.c_uint32 * 4)()
        if N.lib().yas_program_rule_aux(self._h, rule, out) != 0:
            raise IndexError(rule)
        return {"b": out[0], "t": out[1], "n": out[2], "vacuous": bool(out[3])}

    def census(self):
        a, b = (C.c_uint64 * 3)(), (C.c_uint64 * 3)()
        N.lib().yas_program_census(self._h, a, b)
        return tuple(a), tuple(b)


def parse_program(text) -> GroundProgram:
    """parse_program(std::string_view) — raises ParseError(line) on bad input."""
    if isinstance(text, str):
        text = text.encode()
    h = C.c_void_p()
    line = C.c_int(0)
    err = C.create_string_buffer(512)
    rc = N.lib().yas_program_parse(text, len(text), C.byref(h), C.byref(line), err, 512)
    if rc != 0:
        _raise(rc, err.value, line.value)
    return GroundProgram(h.value)


def parse_file(path: str) -> GroundProgram:
    h = C.c_void_p()
    line = C.c_int(0)
    err = C.create_string_buffer(512)
    rc = N.lib().yas_program_parse_file(path.encode(), C.byref(h), C.byref(line), err, 512)
    if rc != 0:
        _raise(rc, err.value, line.value)
    return GroundProgram(h.value)


def print_program(prog: GroundProgram) -> str:
    return _text(N.lib().yas_program_print, prog._h)


def dump_nogoods(prog: GroundProgram) -> str:
    return _text(N.lib().yas_program_dump_nogoods, prog._h)


def store_csv(prog: GroundProgram) -> str:
    return _text(N.lib().yas_program_store_csv, prog._h)


def validate(prog: GroundProgram) -> List[str]:
    t = _text(N.lib().yas_program_diagnostics, prog._h)
    return [x for x in t.split("\n") if x]


def tp_step(prog: GroundProgram, interp: Sequence[int]) -> List[int]:
    arr = (C.c_uint32 * max(1, len(interp)))(*interp)
    cap = prog.atom_count() + 1
    out = (C.c_uint32 * cap)()
    n = N.lib().yas_program_tp_step(prog._h, arr, len(interp), out, cap)
    if n == C.c_size_t(-1).value:
        raise ValueError("tp_step: atom id 0 or above atom_count")
    return list(out[:n])


def cubes(prog: GroundProgram, k: int, depth: int = 1, rank: int = 0, world: int = 1, want: int = 0):
    """Cube split used by solve(cube_atoms=k, cube_depth=depth): this rank's cubes (unit nogood literals)."""
    width = C.c_uint32(0)
    n = N.lib().yas_program_cubes(prog._h, k, depth, want, rank, world, None, 0, C.byref(width))
    out = (C.c_int32 * max(1, n * max(1, width.value)))()
    N.lib().yas_program_cubes(prog._h, k, depth, want, rank, world, out, n * width.value, C.byref(width))
    w = width.value
    return [list(out[i * w:(i + 1) * w]) for i in range(n)]


def verify_model(prog: GroundProgram, model: Model) -> bool:
    ids = (C.c_uint32 * max(1, len(model.atom_ids)))(*model.atom_ids)
    r = N.lib().yas_verify_model(prog._h, ids, len(model.atom_ids))
    if r < 0:
        raise ValueError("verify_model: atom id 0 or above atom_count")
    return r == 1


def _config(cfg: SolverConfig) -> N.yas_config:
    c = N.yas_config()
    N.lib().yas_config_default(C.byref(c))
    c.mode = int(cfg.mode)
    c.heuristic = int(cfg.heuristic.kind)
    c.activity_decay = cfg.heuristic.activity_decay
    c.workers = cfg.workers
    c.restarts_enabled = 1 if cfg.restarts.enabled else 0
    c.restart_base = cfg.restarts.base
    c.restart_factor = cfg.restarts.factor
    c.max_models = cfg.max_models
    c.deps_words = cfg.deps_words
    c.conflict_fanout = cfg.conflict_fanout
    c.seed = cfg.seed
    c.verify = 1 if cfg.verify else 0
    c.debug_validate = 1 if cfg.debug_validate else 0
    c.learned_capacity = cfg.learned_capacity
    c.device = cfg.device
    c.engine = {"auto": 0, "block": 1, "grid": 2}[cfg.engine]
    c.cube_atoms = cfg.cube_atoms
    c.cube_depth = cfg.cube_depth
    c.slots = cfg.slots
    c.rank = cfg.rank
    c.world = cfg.world
    c.portfolio = cfg.portfolio
    c.count_lits = 1 if cfg.count_lits else 0
    if cfg.devices:
        c.n_devices = len(cfg.devices)
        c._devs = (C.c_int * len(cfg.devices))(*cfg.devices)  # kept alive with the struct
        c.devices = C.cast(c._devs, C.POINTER(C.c_int))
    c.reference_order = 1 if cfg.reference_order else 0
    if cfg.fleet is not None:
        c.fleet = cfg.fleet._h
    return c


def solve(prog: GroundProgram, cfg: Optional[SolverConfig] = None) -> SolveResult:
    """solve(GroundProgram, SolverConfig) — max_models = 0 enumerates all."""
    cfg = cfg or SolverConfig()
    c = _config(cfg)
    keep = None
    if cfg.trace is not None:
        user = cfg.trace

        def _cb(tp, _user):
            t = tp.contents
            user(ConflictTrace(LearnMode(t.mode), t.conflict_id, t.learned_length, t.backjump_level))

        keep = N.TRACE_FN(_cb)
        c.trace = keep
    L = N.lib()
    h = C.c_void_p()
    err = C.create_string_buffer(1024)
    rc = L.yas_solve(prog._h, C.byref(c), C.byref(h), err, 1024)
    del keep
    if rc != 0:
        _raise(rc, err.value)
    try:
        st = N.yas_stats()
        L.yas_result_stats(h, C.byref(st))
        stats = SolveStats(**{f: getattr(st, f) for f in _STAT_FIELDS})
        count = L.yas_result_model_count(h)
        total = L.yas_result_models_flat(h, None, 0, None, None)
        ids = np.empty(max(1, total), dtype=np.uint32)
        offs = np.empty(count + 1, dtype=np.uint64)
        cub = np.empty(max(1, count), dtype=np.uint32)
        L.yas_result_models_flat(h, ids.ctypes.data_as(C.POINTER(C.c_uint32)), ids.size,
                                 offs.ctypes.data_as(C.POINTER(C.c_uint64)), cub.ctypes.data_as(C.POINTER(C.c_uint32)))
        models = ModelList(ids, offs, count, prog)
        cubes = cub[:count].tolist()
        status = SolveStatus(L.yas_result_status(h))
    finally:
        L.yas_result_free(h)
    return SolveResult(models, stats, status, cubes)


class Fleet:
    """Processes (one GPU each) sharing one cube enumeration or first-model portfolio.

    Rank 0's GPU holds the shared cube queue; the other ranks map it through CUDA
    IPC and take cubes with system-scope atomics, and the final model counts and
    flags are all-reduced. Transport: NCCL (``Fleet.nccl``) or any process group
    given as two collectives (``Fleet.from_process_group`` for torch.distributed).
    """

    def __init__(self, handle, keep=()):
        self._h = handle
        self._keep = keep  # ctypes callbacks must outlive the fleet

    @staticmethod
    def _share_nccl():
        # libnccl.so.2 is opened once per process: load torch's copy first when torch
        # is installed, so both use the same (newer) NCCL
        try:
            import torch  # noqa: F401
        except ImportError:
            pass

    @staticmethod
    def unique_id() -> bytes:
        Fleet._share_nccl()
        buf = (C.c_uint8 * 128)()
        err = C.create_string_buffer(512)
        rc = N.lib().yas_fleet_unique_id(buf, err, 512)
        if rc != 0:
            _raise(rc, err.value)
        return bytes(buf)

    @classmethod
    def nccl(cls, unique_id: bytes, rank: int, world: int, device: int) -> "Fleet":
        cls._share_nccl()
        uid = (C.c_uint8 * 128)(*unique_id)
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = N.lib().yas_fleet_create_nccl(uid, rank, world, device, C.byref(h), err, 512)
        if rc != 0:
            _raise(rc, err.value)
        return cls(h.value)

    @classmethod
    def from_collectives(cls, rank: int, world: int, device: int, allreduce, broadcast) -> "Fleet":
        """allreduce(list[int], op) -> list[int] with op 'sum'|'max'|'min'; broadcast(bytes, root) -> bytes."""
        ops = {0: "sum", 1: "max", 2: "min"}

        def _ar(vals, n, op, _user):
            try:
                out = allreduce([vals[i] for i in range(n)], ops[op])
                for i in range(n):
                    vals[i] = int(out[i])
                return 0
            except Exception:  # reported as a failed collective by the C side
                return 1

        def _bc(buf, nbytes, root, _user):
            try:
                data = broadcast(C.string_at(buf, nbytes), root)
                C.memmove(buf, data, nbytes)
                return 0
            except Exception:
                return 1

        ar, bc = N.ALLREDUCE_FN(_ar), N.BROADCAST_FN(_bc)
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = N.lib().yas_fleet_create(rank, world, device, ar, bc, None, C.byref(h), err, 512)
        if rc != 0:
            _raise(rc, err.value)
        return cls(h.value, (ar, bc))

    @classmethod
    def from_process_group(cls, device: int, group=None) -> "Fleet":
        """A fleet over an initialised torch.distributed process group (gloo or nccl)."""
        import torch
        import torch.distributed as dist
        dev = "cpu" if dist.get_backend(group) == "gloo" else f"cuda:{device}"
        red = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN}

        def allreduce(vals, op):
            t = torch.tensor(vals, dtype=torch.int64, device=dev)  # counts and flags stay below 2^63
            dist.all_reduce(t, op=red[op], group=group)
            return [int(x) & 0xFFFFFFFFFFFFFFFF for x in t.tolist()]

        def broadcast(data, root):
            t = torch.tensor(list(data), dtype=torch.uint8, device=dev)
            dist.broadcast(t, src=root, group=group)
            return bytes(t.cpu().tolist())

        return cls.from_collectives(dist.get_rank(group), dist.get_world_size(group), device, allreduce, broadcast)

    def info(self):
        r, w, d, dyn = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        N.lib().yas_fleet_info(self._h, C.byref(r), C.byref(w), C.byref(d), C.byref(dyn))
        return {"rank": r.value, "world": w.value, "device": d.value, "dynamic": bool(dyn.value)}

    def allreduce(self, vals, op: str = "sum"):
        arr = (C.c_uint64 * len(vals))(*vals)
        err = C.create_string_buffer(512)
        rc = N.lib().yas_fleet_allreduce(self._h, arr, len(vals), {"sum": 0, "max": 1, "min": 2}[op], err, 512)
        if rc != 0:
            _raise(rc, err.value)
        return list(arr)

    def close(self):
        if self._h:
            N.lib().yas_fleet_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def stats_csv_header() -> str:
    return _text(N.lib().yas_stats_csv_header)


@dataclass
class StatsContext:
    instance: str = ""
    mode: str = ""
    heuristic: str = ""
    workers: int = 1
    status: SolveStatus = SolveStatus.unsat
    models: int = 0


def emit_stats(stats: SolveStats, ctx: StatsContext, csv: bool) -> str:
    s = stats._c()
    L = N.lib()
    args = (C.byref(s), ctx.instance.encode(), ctx.mode.encode(), ctx.heuristic.encode(), ctx.workers,
            int(ctx.status), ctx.models, 1 if csv else 0)
    n = L.yas_emit_stats(*args, None, 0)
    buf = C.create_string_buffer(n + 1)
    L.yas_emit_stats(*args, buf, n + 1)
    return buf.value.decode()


# ---------------------------------------------------------------------------
# low level: store + propagator
# ---------------------------------------------------------------------------
def _ints(xs: Sequence[int]):
    """int32 buffer for the C-ABI: numpy int32 arrays are passed without a copy."""
    if isinstance(xs, np.ndarray):
        a = np.ascontiguousarray(xs, dtype=np.int32)
        return a.ctypes.data_as(C.POINTER(C.c_int32)) if a.size else (C.c_int32 * 1)()
    return (C.c_int32 * max(1, len(xs)))(*xs)


class NogoodStore:
    """Static partition of the nogood store (NogoodStore::build)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and N is not None and N.lib is not None:
            N.lib().yas_store_free(h)
            self._h = C.c_void_p(0)

    @staticmethod
    def build(nogoods: Iterable[Sequence[int]], total_atoms: int, guards: Optional[Sequence[int]] = None,
              origins: Optional[Sequence[int]] = None) -> "NogoodStore":
        lits, offs = [], [0]
        for ng in nogoods:
            lits.extend(ng)
            offs.append(len(lits))
        n = len(offs) - 1
        h = C.c_void_p()
        err = C.create_string_buffer(256)
        g = (C.c_uint32 * max(1, n))(*guards) if guards is not None else None
        o = (C.c_uint8 * max(1, n))(*origins) if origins is not None else None
        rc = N.lib().yas_store_build(_ints(lits), (C.c_uint32 * len(offs))(*offs), n, g, o, total_atoms,
                                     C.byref(h), err, 256)
        if rc != 0:
            _raise(rc, err.value)
        return NogoodStore(h.value)

    @staticmethod
    def planted(atoms: int, nogoods: int, pct: int, seed: int = 0x1B00B5):
        """Config 4b store + seeded frontier."""
        h = C.c_void_p()
        p = C.POINTER(C.c_int32)()
        n = C.c_size_t(0)
        d = C.c_int32(0)
        rc = N.lib().yas_store_planted(atoms, nogoods, pct, seed, C.byref(h), C.byref(p), C.byref(n), C.byref(d))
        if rc != 0:
            _raise(rc, b"planted store")
        seeded = list(p[: n.value])
        N.lib().yas_free_ints(p)
        return NogoodStore(h.value), seeded, d.value

    def size(self) -> int:
        return N.lib().yas_store_size(self._h)

    def total_atoms(self) -> int:
        return N.lib().yas_store_total_atoms(self._h)

    def dump_csv(self) -> str:
        return _text(N.lib().yas_store_dump_csv, self._h)

    def static_units(self) -> List[int]:
        n = N.lib().yas_store_units(self._h, None, 0)
        out = (C.c_int32 * max(1, n))()
        N.lib().yas_store_units(self._h, out, n)
        return list(out[:n])

    def unit_ids(self) -> List[int]:
        n = N.lib().yas_store_unit_ids(self._h, None, 0)
        out = (C.c_int32 * max(1, n))()
        N.lib().yas_store_unit_ids(self._h, out, n)
        return list(out[:n])

    def static_class_bounds(self) -> List[int]:
        out = (C.c_uint32 * 4)()
        N.lib().yas_store_bounds(self._h, out)
        return list(out)

    def occurrences(self, lit: int, cls: int) -> List[int]:
        n = N.lib().yas_store_occurrences(self._h, lit, cls, None, 0)
        out = (C.c_int32 * max(1, n))()
        N.lib().yas_store_occurrences(self._h, lit, cls, out, n)
        return list(out[:n])


@dataclass
class PropagationOutcome:
    violated: bool
    conflicts: List[int]
    propagations: int
    passes: int
    checks: int
    device_ms: float
    checked_lits: int = 0


REASON_NONE, REASON_DECISION, REASON_UNIT, REASON_COMPLETION = -1, -2, -3, -4


class Propagator:
    """Propagator + Assignment + Frontier of one device search."""

    def __init__(self, store: NogoodStore, deps_words: int = 16, engine: str = "auto", device: int = 0):
        self.store = store
        self.deps_words = deps_words
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = N.lib().yas_propagator_create(store._h, deps_words, {"auto": 0, "block": 1, "grid": 2}[engine], device,
                                           C.byref(h), err, 512)
        if rc != 0:
            _raise(rc, err.value)
        self._h = h
        self.atoms = N.lib().yas_propagator_atoms(h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and N is not None and N.lib is not None:
            N.lib().yas_propagator_free(h)
            self._h = C.c_void_p(0)

    def _check(self, rc: int):
        """Every yas_propagator_* status is checked: a CUDA or argument failure raises."""
        if rc != 0:
            _raise(rc, _text(N.lib().yas_propagator_last_error, self._h).encode())

    def _outcome(self, o: N.yas_outcome) -> PropagationOutcome:
        confl = self.conflicts() if o.n_conflicts else []
        return PropagationOutcome(bool(o.violated), confl, o.propagations, o.passes, o.checks, o.device_ms,
                                  o.checked_lits)

    def reset(self):
        self._check(N.lib().yas_propagator_reset(self._h))

    def flush(self):
        """Launch the recorded state-changing calls now (they otherwise run with the next result-returning call)."""
        self._check(N.lib().yas_propagator_flush(self._h))

    def initial_propagation(self) -> PropagationOutcome:
        o = N.yas_outcome()
        self._check(N.lib().yas_propagator_initial(self._h, C.byref(o)))
        return self._outcome(o)

    def propagate_and_check(self, level: int) -> PropagationOutcome:
        o = N.yas_outcome()
        self._check(N.lib().yas_propagator_propagate(self._h, level, C.byref(o)))
        return self._outcome(o)

    def push_decision(self, lit: int):
        self._check(N.lib().yas_propagator_push_decision(self._h, lit))

    def assign_propagated(self, lits: Sequence[int], level: int, deps: Sequence[int] = (), overflow: bool = False,
                          antecedent: int = 0):
        d = (C.c_uint64 * max(1, len(deps)))(*deps)
        self._check(N.lib().yas_propagator_assign(self._h, _ints(lits), len(lits), level, d, len(deps),
                                                  1 if overflow else 0, antecedent))

    def seed(self, lits: Sequence[int]):
        self._check(N.lib().yas_propagator_seed(self._h, _ints(lits), len(lits)))

    def add_learned(self, lits: Sequence[int]) -> int:
        i = N.lib().yas_propagator_add_learned(self._h, _ints(lits), len(lits))
        if i < 0:
            raise ValueError(_text(N.lib().yas_propagator_last_error, self._h))
        return i

    def count_literals(self, on: bool = True):
        """Exact checked-literal accounting (roofline bytes); off by default."""
        self._check(N.lib().yas_propagator_count_literals(self._h, 1 if on else 0))

    def level(self) -> int:
        return N.lib().yas_propagator_level(self._h)

    def transfers(self):
        """(host->device, device->host) bytes moved by this propagator so far (counted)."""
        a, b = C.c_uint64(0), C.c_uint64(0)
        self._check(N.lib().yas_propagator_transfers(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def pass_trace(self, on: Optional[bool] = None):
        """Diagnostics: enable/disable (on) and read the per-pass, per-block
        phase timestamps of whole-grid propagations: array [64, blocks, 10]."""
        N.lib().yas_propagator_pass_trace(self._h, -1 if on is None else int(bool(on)), None, 0, None)
        blocks = C.c_uint32(0)
        out = np.zeros(64 * 148 * 10 * 4 + 64 * 16, dtype=np.uint64)
        N.lib().yas_propagator_pass_trace(self._h, -1, out.ctypes.data_as(C.POINTER(C.c_uint64)), out.size,
                                          C.byref(blocks))
        b = max(1, blocks.value)
        self.pass_debug = out[64 * b * 10: 64 * b * 10 + 64 * 16].reshape(64, 16)
        return out[: 64 * b * 10].reshape(64, b, 10)

    def profile(self) -> List[int]:
        """Diagnostics: SM cycles per propagation phase (see yas_propagator_profile)."""
        out = (C.c_uint64 * 16)()
        self._check(N.lib().yas_propagator_profile(self._h, out))
        return list(out)

    def cells(self) -> List[int]:
        out = (C.c_int32 * (self.atoms + 1))()
        self._check(N.lib().yas_propagator_cells(self._h, out))
        return list(out)

    def reasons(self) -> List[int]:
        out = (C.c_int32 * (self.atoms + 1))()
        self._check(N.lib().yas_propagator_reasons(self._h, out))
        return list(out)

    def deps(self, word: int = 0):
        out = (C.c_uint64 * (self.atoms + 1))()
        ovf = (C.c_uint8 * (self.atoms + 1))()
        self._check(N.lib().yas_propagator_deps(self._h, word, out, ovf))
        return list(out), list(ovf)

    def _array(self, fn, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.atoms + 1, dtype=np.int32)  # trail, frontier, conflicts: one pass, <= A entries
        n = fn(self._h, out.ctypes.data_as(C.POINTER(C.c_int32)), out.size)
        if n == 0:
            msg = _text(N.lib().yas_propagator_last_error, self._h)
            if msg:
                raise DeviceError(msg)
        if n > out.size:  # (cannot happen for trail/frontier; conflicts may exceed A)
            out = np.empty(n, dtype=np.int32)
            n = fn(self._h, out.ctypes.data_as(C.POINTER(C.c_int32)), out.size)
        return out[:n]

    def _list(self, fn) -> List[int]:
        return self._array(fn).tolist()

    def trail(self) -> List[int]:
        return self._list(N.lib().yas_propagator_trail)

    def trail_array(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        """The trail as an int32 numpy array (one D2H copy, no Python list);
        `out` (int32, >= atoms + 1 entries, e.g. pinned) is filled and sliced."""
        return self._array(N.lib().yas_propagator_trail, out)

    def conflicts(self) -> List[int]:
        return self._list(N.lib().yas_propagator_conflicts)

    def frontier(self) -> List[int]:
        return self._list(N.lib().yas_propagator_frontier)


def device_count() -> int:
    return N.lib().yas_device_count()
