"""The reference's `tilemul` interface for the execution path, backed by the
B200-native library (C ABI in include/tilemul_b200.h).

Names, argument meaning and error behaviour follow
/root/reference/proj/include/tilemul/*.hpp so a caller of the reference (and
the restated reference tests in tests/) reads the same:

    d = parse_name("C2A1C0")
    bs = derive_blocksizes(d, hier, Shape(2048, 2048, 2048))
    nest = build_plan(d, bs, hier, shape)
    execute(nest, A, B, C)            # C += A·B on the GPU

Operands are column-major FP64: CUDA torch tensors (device path, async on
the current stream) or numpy arrays (host path: copy in, run, copy back).
Errors: ParseError (with .rule), ValidationFailure (with .violations),
InfeasibleError, ValueError (the reference's std::invalid_argument),
CudaError (device runtime failures).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

from . import _native as N

DIMS = ("m", "n", "k")
OPERANDS = ("A", "B", "C")


# ------------------------------------------------------------------ errors
@dataclass(frozen=True)
class Violation:  # types.hpp:132-138
    rule: str
    level: int = -1
    lhs: int = 0
    rhs: int = 0


class ParseError(ValueError):  # types.hpp:148-154
    def __init__(self, rule: str, msg: str):
        super().__init__(msg)
        self.rule = rule


class ValidationFailure(RuntimeError):  # types.hpp:157-170
    def __init__(self, violations: List[Violation], msg: str):
        super().__init__(msg)
        self.violations = violations


class InfeasibleError(RuntimeError):  # types.hpp:173-176
    pass


class CudaError(RuntimeError):
    pass


def _rules() -> List[Violation]:
    out = []
    for ln in N.lib().tm_last_rules().decode().splitlines():
        if not ln:
            continue
        r, lvl, lhs, rhs = ln.rsplit(":", 3)
        out.append(Violation(r, int(lvl), int(lhs), int(rhs)))
    return out


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = N.lib().tm_last_error().decode()
    if rc == 1:
        rules = _rules()
        if msg.startswith("validation failed"):
            raise ValidationFailure(rules, msg)
        if rules and rules[0].rule == "infeasible":
            raise InfeasibleError(msg)
        raise ParseError(rules[0].rule if rules else "", msg)
    if rc == 3:
        raise CudaError(msg)
    raise ValueError(msg)


# -------------------------------------------------------------- vocabulary
@dataclass(frozen=True)
class Shape:  # types.hpp:103-129
    m: int = 1
    n: int = 1
    k: int = 1

    def __post_init__(self):
        if self.m < 1 or self.n < 1 or self.k < 1:
            raise ValueError("shape extents must be >= 1")

    def extent(self, d: str) -> int:
        return {"m": self.m, "n": self.n, "k": self.k}[d]

    def flops(self) -> int:
        return 2 * self.m * self.n * self.k

    def rows(self, op: str) -> int:
        return {"A": self.m, "B": self.k, "C": self.m}[op]

    def cols(self, op: str) -> int:
        return {"A": self.k, "B": self.n, "C": self.n}[op]


@dataclass(frozen=True)
class CacheLevel:  # cache.hpp:12-19
    index: int
    capacity_elements: int
    granularity: int = 1
    inclusive: bool = False
    write_allocate: bool = True
    write_back: bool = True


class CacheHierarchy:  # cache.hpp:23-49
    def __init__(self, levels: Sequence[CacheLevel]):
        levels = list(levels)
        if not levels:
            raise ValueError("hierarchy needs at least one level")
        for i, lv in enumerate(levels):
            if lv.index != i:
                raise ValueError("hierarchy level indices must be contiguous from 0")
            if lv.capacity_elements < 1:
                raise ValueError("cache capacity must be >= 1")
            if lv.granularity < 1:
                raise ValueError("cache granularity must be >= 1")
            if i > 0 and lv.capacity_elements <= levels[i - 1].capacity_elements:
                raise ValueError("cache capacities must strictly increase with level")
        self._levels = levels

    @classmethod
    def from_capacities(cls, caps: Sequence[int], inclusive: Sequence[bool] = ()):
        inc = list(inclusive) + [False] * (len(caps) - len(inclusive))
        return cls([CacheLevel(i, int(c), 1, bool(inc[i])) for i, c in enumerate(caps)])

    def size(self) -> int:
        return len(self._levels)

    def level(self, h: int) -> CacheLevel:
        return self._levels[h]

    def levels(self) -> List[CacheLevel]:
        return list(self._levels)

    def top_level(self) -> int:
        return len(self._levels) - 1

    def capacity(self, h: int) -> int:
        return self._levels[h].capacity_elements

    def _c(self):
        arr = (N.tm_level * len(self._levels))()
        for i, lv in enumerate(self._levels):
            arr[i] = N.tm_level(lv.capacity_elements, lv.granularity, int(lv.inclusive), int(lv.write_allocate),
                                int(lv.write_back))
        return arr, len(self._levels)


def gpu_hierarchy(tile: int = 128) -> CacheHierarchy:
    """The current B200's hierarchy in FP64 elements: 0 = CTA C tile,
    1 = shared memory per block, 2 = L2 (queried from the device)."""
    arr = (N.tm_level * 8)()
    cnt = C.c_int(0)
    _check(N.lib().tm_gpu_hierarchy(tile, arr, 8, C.byref(cnt)))
    return CacheHierarchy([CacheLevel(i, arr[i].capacity_elements) for i in range(cnt.value)])


# ------------------------------------------------------------- descriptors
@dataclass(frozen=True)
class LevelPlan:  # descriptor.hpp:18-25
    level: int
    resident: str
    outer_dim: str
    inner_dim: str


@dataclass
class AlgorithmDescriptor:  # descriptor.hpp:30-43
    plans: List[LevelPlan] = field(default_factory=list)
    allow_non_c_registers: bool = False

    def plan_at(self, level: int) -> Optional[LevelPlan]:
        for p in self.plans:
            if p.level == level:
                return p
        return None

    def top_level(self) -> int:
        return self.plans[0].level if self.plans else -1

    def __eq__(self, other):
        return isinstance(other, AlgorithmDescriptor) and self.plans == other.plans

    @property
    def name(self) -> str:
        return format_name(self)


def guest_operand(below: LevelPlan) -> str:  # descriptor.hpp:47
    return {"n": "A", "m": "B", "k": "C"}[below.inner_dim]


def _tiers_to_desc(arr, n, allow) -> AlgorithmDescriptor:
    return AlgorithmDescriptor([LevelPlan(arr[i].level, arr[i].resident.decode(), arr[i].outer_dim.decode(),
                                          arr[i].inner_dim.decode()) for i in range(n)], allow)


def parse_name(text: str, allow_non_c_registers: bool = False) -> AlgorithmDescriptor:
    arr = (N.tm_tier * 16)()
    cnt = C.c_int(0)
    _check(N.lib().tm_parse_name(text.encode(), int(allow_non_c_registers), arr, 16, C.byref(cnt)))
    return _tiers_to_desc(arr, cnt.value, allow_non_c_registers)


def make_descriptor(residents: Sequence[Tuple[int, str]], allow_non_c_registers: bool = False) -> AlgorithmDescriptor:
    lv = (C.c_int32 * max(1, len(residents)))(*[r[0] for r in residents])
    ops = "".join(r[1] for r in residents).encode()
    arr = (N.tm_tier * 16)()
    cnt = C.c_int(0)
    name = C.create_string_buffer(64)
    _check(N.lib().tm_compose(lv, ops, len(residents), int(allow_non_c_registers), name, 64, arr, 16, C.byref(cnt)))
    return _tiers_to_desc(arr, cnt.value, allow_non_c_registers)


def format_name(d: AlgorithmDescriptor) -> str:  # descriptor.hpp:128-136
    s = ""
    for p in d.plans:
        if p.level > 9:
            raise ValueError("names only cover cache levels 0..9")
        s += f"{p.resident}{p.level}"
    return s


def validate_structure(d: AlgorithmDescriptor) -> List[Violation]:
    arr = (N.tm_tier * max(1, len(d.plans)))()
    for i, p in enumerate(d.plans):
        arr[i] = N.tm_tier(p.level, p.resident.encode(), p.outer_dim.encode(), p.inner_dim.encode())
    rc = N.lib().tm_validate_structure(arr, len(d.plans), int(d.allow_non_c_registers))
    if rc < 0:
        _check(-rc)
    return _rules() if rc > 0 else []


def skip_level(d: AlgorithmDescriptor, h: int) -> AlgorithmDescriptor:
    out = C.create_string_buffer(64)
    _check(N.lib().tm_skip_level(format_name(d).encode(), h, out, 64))
    return parse_name(out.value.decode(), d.allow_non_c_registers)


def select_algorithm(s: Shape, outer_capacity: int) -> str:
    r = C.create_string_buffer(2)
    _check(N.lib().tm_select_outer(s.m, s.n, s.k, outer_capacity, r))
    return r.value.decode()


# -------------------------------------------------------------- blocksizes
class BlocksizeSet:  # blocksizes.hpp:22-56
    def __init__(self, entries: Optional[Dict[Tuple[int, str], int]] = None):
        self._v: Dict[Tuple[int, str], int] = {}
        for (lv, d), v in (entries or {}).items():
            self.set(lv, d, v)

    def set(self, level: int, dim: str, value: int) -> None:
        if value < 1:
            raise ValueError("blocksize must be >= 1")
        self._v[(int(level), dim)] = int(value)

    def has(self, level: int, dim: str) -> bool:
        return (level, dim) in self._v

    def get(self, level: int, dim: str) -> int:
        if (level, dim) not in self._v:
            raise KeyError(f"no blocksize for level {level} dim {dim}")
        return self._v[(level, dim)]

    def entries(self) -> List[Tuple[Tuple[int, str], int]]:
        return sorted(self._v.items(), key=lambda kv: (kv[0][0], DIMS.index(kv[0][1])))

    def as_dict(self) -> Dict[Tuple[int, str], int]:
        return dict(self._v)

    def __eq__(self, other):
        return isinstance(other, BlocksizeSet) and self._v == other._v

    def __repr__(self):
        return "BlocksizeSet(" + ", ".join(f"{lv}:{d}={v}" for (lv, d), v in self.entries()) + ")"

    def _c(self):
        ent = self.entries()
        arr = (N.tm_blocksize * max(1, len(ent)))()
        for i, ((lv, d), v) in enumerate(ent):
            arr[i] = N.tm_blocksize(lv, d.encode(), v)
        return arr, len(ent)


@dataclass
class AccessCosts:  # blocksizes.hpp:59-76
    beta_a: float = 1.0
    beta_b: float = 1.0
    beta_c: float = 1.0


@dataclass
class MicroTile:  # blocksizes.hpp:79-82
    m_r: int = 4
    n_r: int = 12


@dataclass
class DeriveOptions:  # blocksizes.hpp:84-87
    slack: float = 1.0 / 16.0
    micro: MicroTile = field(default_factory=MicroTile)


def derive_blocksizes(d: AlgorithmDescriptor, hier: CacheHierarchy, shape: Shape, costs: AccessCosts = None,
                      opts: DeriveOptions = None, pinned: BlocksizeSet = None) -> BlocksizeSet:
    costs = costs or AccessCosts()
    opts = opts or DeriveOptions()
    pinned = pinned or BlocksizeSet()
    h, nh = hier._c()
    p, npin = pinned._c()
    o = N.tm_derive_opts(opts.slack, opts.micro.m_r, opts.micro.n_r, costs.beta_a, costs.beta_b, costs.beta_c)
    out = (N.tm_blocksize * 64)()
    cnt = C.c_int(0)
    _check(N.lib().tm_derive(format_name(d).encode(), h, nh, shape.m, shape.n, shape.k, C.byref(o), p, npin, out, 64,
                             C.byref(cnt)))
    return BlocksizeSet({(out[i].level, out[i].dim.decode()): out[i].value for i in range(cnt.value)})


def validate_blocksizes(d: AlgorithmDescriptor, bs: BlocksizeSet, hier: CacheHierarchy, shape: Shape) -> List[Violation]:
    h, nh = hier._c()
    b, nb = bs._c()
    rc = N.lib().tm_validate(format_name(d).encode(), h, nh, shape.m, shape.n, shape.k, b, nb)
    if rc < 0:
        _check(-rc)
    return _rules() if rc > 0 else []


@dataclass(frozen=True)
class NestStep:  # blocksizes.hpp:428-434
    level: int
    dim: str
    blocksize: int
    cap: bool = False


# ------------------------------------------------------------------- model
@dataclass
class OperandTraffic:
    reads: int = 0
    writes: int = 0

    def total(self) -> int:
        return self.reads + self.writes


@dataclass
class LevelTraffic:
    level: int
    per_operand: Dict[str, OperandTraffic]

    def of(self, op: str) -> OperandTraffic:
        return self.per_operand[op]

    def reads(self) -> int:
        return sum(t.reads for t in self.per_operand.values())

    def writes(self) -> int:
        return sum(t.writes for t in self.per_operand.values())

    def total_elements(self) -> int:
        return self.reads() + self.writes()

    def total_bytes(self, elem_bytes: Dict[str, float] = None) -> float:
        eb = elem_bytes or {"A": 8, "B": 8, "C": 8}
        return sum(eb[o] * (t.reads + t.writes) for o, t in self.per_operand.items())


@dataclass
class CostReport:  # costmodel.hpp:44-62
    shape: Shape
    flops: int
    levels: List[LevelTraffic]
    boundary_level: int

    def at_level(self, h: int) -> LevelTraffic:
        for lt in self.levels:
            if lt.level == h:
                return lt
        raise KeyError(f"no traffic entry for level {h}")

    def intensity_flops_per_byte(self) -> float:
        b = self.at_level(self.boundary_level).total_bytes()
        return float("inf") if b == 0 else self.flops / b


def _report(shape: Shape, raw, nlev: int) -> CostReport:
    levels = []
    for h in range(nlev):
        levels.append(LevelTraffic(h, {op: OperandTraffic(raw[(h * 3 + i) * 2], raw[(h * 3 + i) * 2 + 1])
                                       for i, op in enumerate(OPERANDS)}))
    return CostReport(shape, shape.flops(), levels, nlev - 1)


def multilevel_cost(d: AlgorithmDescriptor, bs: BlocksizeSet, hier: CacheHierarchy, shape: Shape,
                    boundary_level: int = -1) -> CostReport:
    h, nh = hier._c()
    b, nb = bs._c()
    raw = (C.c_int64 * (nh * 6))()
    _check(N.lib().tm_model(format_name(d).encode(), int(d.allow_non_c_registers), h, nh, shape.m, shape.n, shape.k,
                            b, nb, raw, nh * 6))
    rep = _report(shape, raw, nh)
    if boundary_level >= 0:
        rep.boundary_level = boundary_level
    return rep


def io_lower_bound(s: Shape, M: int) -> OperandTraffic:
    r, w = C.c_int64(0), C.c_int64(0)
    _check(N.lib().tm_io_lower_bound(s.m, s.n, s.k, M, C.byref(r), C.byref(w)))
    return OperandTraffic(r.value, w.value)


def resident_cost(variant: str, s: Shape, b_first: int, b_second: int) -> LevelTraffic:
    raw = (C.c_int64 * 6)()
    _check(N.lib().tm_resident_cost(variant.encode(), s.m, s.n, s.k, b_first, b_second, raw))
    return LevelTraffic(0, {op: OperandTraffic(raw[i * 2], raw[i * 2 + 1]) for i, op in enumerate(OPERANDS)})


def _dbl(v: float) -> float:
    if v < 0:
        raise ValueError(N.lib().tm_last_error().decode())
    return v


def streaming_efficiency(variant: str, b_first: int, b_second: int) -> float:
    return _dbl(N.lib().tm_streaming_efficiency(variant.encode(), b_first, b_second))


def goto_efficiency(k_c: int, n_c: int) -> float:
    return _dbl(N.lib().tm_goto_efficiency(k_c, n_c))


def efficiency(report: CostReport, level: int = -1, write_weight: float = 1.0) -> Tuple[float, float]:
    lt = report.at_level(report.boundary_level if level < 0 else level)
    el = lt.reads() + write_weight * lt.writes()
    if el <= 0:
        return float("inf"), float("inf")
    fpe = report.flops / el
    return fpe, fpe / 8.0


def roofline_bound(intensity: float, peak: float, bandwidth: float) -> float:
    return _dbl(N.lib().tm_roofline_bound(intensity, peak, bandwidth))


@dataclass
class ParetoPoint:  # costmodel.hpp:286-293
    ratio: float
    inner_capacity: int
    outer_block_k: int
    outer_block_n: int
    inner_block_m: int
    inner_block_k: int
    eff_outer_flops_per_element: float
    eff_inner_flops_per_element: float


def pareto_sweep(outer_capacity: int, ratios: Sequence[float], shape: Shape,
                 opts: Optional["DeriveOptions"] = None) -> List[ParetoPoint]:  # costmodel.hpp:299-328
    """Sweeps the capacity ratio of a cache pair: B2A1C0 (B in the outer
    cache, A in the inner one, C in registers) with blocks derived under the
    fit rules at each ratio, and both levels' modelled efficiencies."""
    o = opts or DeriveOptions()
    reg = max(o.micro.m_r * o.micro.n_r, 1)
    d = parse_name("B2A1C0")
    points = []
    for r in sorted(ratios):
        if not r > 1.0:
            raise ValueError("ratios must be > 1")
        inner = int(float(outer_capacity) / r)
        if inner <= reg:
            raise InfeasibleError(f"infeasible ratio {r}: the inner cache cannot hold even one register tile")
        hier = CacheHierarchy([CacheLevel(0, reg), CacheLevel(1, inner), CacheLevel(2, outer_capacity)])
        bs = derive_blocksizes(d, hier, shape, None, o)
        rep = multilevel_cost(d, bs, hier, shape)
        points.append(ParetoPoint(r, inner, bs.get(2, "k"), bs.get(2, "n"), bs.get(1, "m"), bs.get(1, "k"),
                                  efficiency(rep, 2)[0], efficiency(rep, 1)[0]))
    return points


# --------------------------------------------------------------- the plan
NUMERICS = {"dmma": 0, "fma": 1, "exact": 2}
SCHEDULES = {"fused": 0, "faithful": 1}
STAGINGS = {"auto": 0, "cpasync": 1, "tma": 2}
B200_L2_BYTES = 132644864  # cudaDevAttrL2CacheSize on the B200s of this pool (126.5 MiB)
STAGING_NAMES = {0: None, 1: "cpasync", 2: "tma"}


@dataclass
class ExecOptions:  # exec.hpp:48-53, re-targeted
    numerics: str = "dmma"      # dmma | fma | exact
    schedule: str = "fused"     # fused | faithful
    split_k: int = 1            # fused: k slices with a fixed-order reduction (0 = auto)
    ctas: int = 0               # persistent grid (0 = SMs x occupancy)
    tile: int = 0               # CTA tile rows 64/128 (0 = from the register tile)
    tile_n: int = 0             # CTA tile columns (0 = tile); 128x64 runs two CTAs per SM
    parallel_loop: int = -1     # faithful: loop whose iterations run as independent workers (-1 = nest order)
    staging: str = "auto"       # DMMA kernels: auto | cpasync | tma (how A/B k-slabs reach shared memory)

    def _c(self):
        return N.tm_exec_opts(NUMERICS[self.numerics], SCHEDULES[self.schedule], self.split_k, self.ctas, self.tile,
                              self.tile_n, self.parallel_loop + 1, STAGINGS[self.staging])


class LoopNest:  # plan.hpp:25-85
    """An executable nest on the GPU. Owns the native plan."""

    def __init__(self, d: AlgorithmDescriptor, bs: BlocksizeSet, hier: CacheHierarchy, shape: Shape):
        h, nh = hier._c()
        b, nb = bs._c()
        ptr = C.c_void_p(None)
        _check(N.lib().tm_plan_create(format_name(d).encode(), h, nh, shape.m, shape.n, shape.k, b, nb,
                                      C.byref(ptr)))
        self._ptr = ptr
        self.shape = shape
        self.descriptor = d
        self.blocksizes = bs
        self.hierarchy = hier
        arr = (N.tm_loop * 64)()
        cnt = C.c_int(0)
        _check(N.lib().tm_plan_loops(self._ptr, arr, 64, C.byref(cnt)))
        self.loops = [NestStep(arr[i].level, arr[i].dim.decode(), arr[i].blocksize, bool(arr[i].cap))
                      for i in range(cnt.value)]
        self.m_r = bs.get(0, "m")
        self.n_r = bs.get(0, "n")

    @classmethod
    def from_loops(cls, loops: Sequence[NestStep], m_r: int, n_r: int, shape: Shape,
                   name: Optional[str] = None) -> "LoopNest":
        """An executable nest from its loop list alone (plan.hpp:25-31), the
        way the reference's execute(nest, A, B, C, opts) receives it: no
        hierarchy (so no model()); tm_plan_create_loops checks what execution
        relies on."""
        self = cls.__new__(cls)
        arr = (N.tm_loop * max(1, len(loops)))()
        for i, L in enumerate(loops):
            arr[i] = N.tm_loop(L.level, L.dim.encode(), L.blocksize, 1 if L.cap else 0)
        ptr = C.c_void_p(None)
        _check(N.lib().tm_plan_create_loops(name.encode() if name else None, arr, len(loops), m_r, n_r, shape.m,
                                            shape.n, shape.k, C.byref(ptr)))
        self._ptr = ptr
        self.shape = shape
        self.descriptor = parse_name(name) if name else None
        self.blocksizes = None
        self.hierarchy = None
        self.loops = list(loops)
        self.m_r, self.n_r = m_r, n_r
        return self

    def __del__(self):
        p = getattr(self, "_ptr", None)
        if p is not None and p.value and N is not None and N._lib is not None:
            N._lib.tm_plan_destroy(p)
            self._ptr = None

    def cell_count(self) -> int:
        return int(N.lib().tm_plan_cells(self._ptr))

    def model(self) -> CostReport:
        nh = N.lib().tm_plan_levels(self._ptr)
        raw = (C.c_int64 * (nh * 6))()
        _check(N.lib().tm_plan_model(self._ptr, raw, nh * 6))
        return _report(self.shape, raw, nh)

    def gpu_model(self, opts: "ExecOptions" = None, sms: int = 148, l2_bytes: Optional[int] = None,
                  elem_bytes: Sequence[float] = (8, 8, 8)) -> Dict[str, object]:
        """GPU-mode I/O model of the schedule execute() runs with `opts`
        (tm_plan_gpu_model; no GPU needed): elements into the SMEM level per
        operand (exact over the task list, FIFO staging) and bytes across
        the HBM boundary from a lockstep run of the task list through an LRU
        of the L2 (default: the B200's 126.5 MiB, cudaDevAttrL2CacheSize)."""
        o = (opts or ExecOptions())._c()
        eb = (C.c_double * 3)(*elem_bytes)
        out = (C.c_int64 * 18)()
        _check(N.lib().tm_plan_gpu_model(self._ptr, C.byref(o), sms, l2_bytes or B200_L2_BYTES, eb, out, 18))
        smem = {op: (out[2 * q], out[2 * q + 1]) for q, op in enumerate(OPERANDS)}
        hbm = {op: (out[6 + 2 * q], out[6 + 2 * q + 1]) for q, op in enumerate(OPERANDS)}
        smem_bytes = sum(elem_bytes[q] * (out[2 * q] + out[2 * q + 1]) for q in range(3))
        return {"smem_elements": smem, "smem_bytes": smem_bytes, "hbm_bytes": hbm,
                "hbm_total_bytes": sum(r + w for r, w in hbm.values()),
                "hbm_read_bytes": sum(r for r, _ in hbm.values()),
                "tasks": out[12], "grid": out[13], "lockstep_slabs": out[14], "kernel": out[15],
                "tile": (out[16], out[17])}

    def gpu_model_tc(self, dtype: str = "bf16", opts: "ExecOptions" = None, sms: int = 148,
                     l2_bytes: Optional[int] = None) -> Dict[str, object]:
        """The GPU-mode model of the tcgen05 path execute_tc runs (tm_plan_gpu_model_tc): the task list of
        the kernel `opts` selects (default: 256 x 512 SM-pair tiles, one per cluster, sms / 2 clusters in
        flight), bf16 (2-byte) or tf32 (4-byte) inputs, fp32 C."""
        o = (opts or ExecOptions())._c()
        out = (C.c_int64 * 18)()
        _check(N.lib().tm_plan_gpu_model_tc(self._ptr, DTYPES[dtype], C.byref(o), sms, l2_bytes or B200_L2_BYTES,
                                            out, 18))
        eb = (2, 2, 4) if dtype == "bf16" else (4, 4, 4)
        smem = {op: (out[2 * q], out[2 * q + 1]) for q, op in enumerate(OPERANDS)}
        hbm = {op: (out[6 + 2 * q], out[6 + 2 * q + 1]) for q, op in enumerate(OPERANDS)}
        return {"smem_elements": smem, "smem_bytes": sum(eb[q] * (out[2 * q] + out[2 * q + 1]) for q in range(3)),
                "hbm_bytes": hbm, "hbm_total_bytes": sum(r + w for r, w in hbm.values()),
                "hbm_read_bytes": sum(r for r, _ in hbm.values()),
                "tasks": out[12], "grid": out[13], "lockstep_slabs": out[14], "kernel": out[15],
                "tile": (out[16], out[17])}

    def tasks(self, opts: "ExecOptions" = None, sms: int = 148):
        """The lowered task list (host half of the lowering): list of dicts
        (i0, j0, p0, m, n, k, slice, from_c, fixup, seq), the grid, and per-CTA
        ranges for stream-K (None when CTA c runs tasks c, c + grid, ...)."""
        o = (opts or ExecOptions())._c()
        cnt, grid = C.c_int64(0), C.c_int32(0)
        _check(N.lib().tm_plan_tasks(self._ptr, C.byref(o), sms, None, 0, C.byref(cnt), C.byref(grid), None, 0))
        buf = (C.c_int32 * max(1, 10 * cnt.value))()
        first = (C.c_int32 * (grid.value + 1))()
        _check(N.lib().tm_plan_tasks(self._ptr, C.byref(o), sms, buf, cnt.value, C.byref(cnt), C.byref(grid), first,
                                     grid.value + 1))
        keys = ("i0", "j0", "p0", "m", "n", "k", "slice", "from_c", "fixup", "seq")
        ts = [dict(zip(keys, buf[10 * q:10 * q + 10])) for q in range(cnt.value)]
        ranges = None if first[0] == -1 else list(first)
        return ts, grid.value, ranges

    def host_pipe_steps(self) -> List[Dict]:
        """The upload order of the host-buffer pipeline (tm_execute_host) for this
        nest's extents: one dict per data flag, {"pieces": [(op, r0, rows, c0,
        cols), ...], "box": (i0, i1, j0, j1), "chunk": q} -- the pieces copied
        before the flag and the cells whose tasks wait for it (host logic only)."""
        cnt = C.c_int64(0)
        _check(N.lib().tm_host_pipe_steps(self._ptr, None, 0, C.byref(cnt)))
        buf = (C.c_int64 * (6 * max(1, cnt.value)))()
        _check(N.lib().tm_host_pipe_steps(self._ptr, buf, cnt.value, C.byref(cnt)))
        steps, pieces = [], []
        for r in range(cnt.value):
            kind, a, b, c, d, e = buf[6 * r:6 * r + 6]
            if kind == 0:
                steps.append({"pieces": pieces, "box": (a, b, c, d), "chunk": e})
                pieces = []
            else:
                pieces.append(("?ABC"[kind], a, b, c, d))
        return steps

    def last_launch(self) -> Dict[str, int]:
        t, l, c = C.c_int64(0), C.c_int32(0), C.c_int32(0)
        _check(N.lib().tm_plan_last_launch(self._ptr, C.byref(t), C.byref(l), C.byref(c)))
        st = C.c_int32(0)
        _check(N.lib().tm_plan_last_staging(self._ptr, C.byref(st)))
        return {"tasks": t.value, "launches": l.value, "ctas": c.value, "staging": STAGING_NAMES[st.value]}


def build_plan(d: AlgorithmDescriptor, bs: BlocksizeSet, hier: CacheHierarchy, shape: Shape) -> LoopNest:
    return LoopNest(d, bs, hier, shape)


# --------------------------------------------------------------- execute
def _colmajor_view(x, rows: int, cols: int, name: str):
    """(pointer, leading dim, is_device) of a column-major FP64 operand."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(x, torch.Tensor):
        if x.dtype != torch.float64:
            raise ValueError(f"{name} must be float64")
        if x.dim() == 1:
            if x.numel() != rows * cols or x.stride(0) != 1:
                raise ValueError(f"{name} extents do not match the plan's shape")
            ld = rows
        elif x.dim() == 2:
            if tuple(x.shape) != (rows, cols) or x.stride(0) != 1:
                raise ValueError(f"{name} must be a column-major {rows}x{cols} view (stride(0) == 1)")
            ld = max(x.stride(1), rows)
        else:
            raise ValueError(f"{name} must be 1-D or 2-D")
        return x.data_ptr(), ld, x.is_cuda
    import numpy as np

    if not isinstance(x, np.ndarray) or x.dtype != np.float64:
        raise ValueError(f"{name} must be a float64 numpy array or torch tensor")
    if x.size != rows * cols:
        raise ValueError(f"{name} extents do not match the plan's shape")
    if x.ndim == 2 and not (x.shape == (rows, cols) and x.flags.f_contiguous):
        raise ValueError(f"{name} must be a Fortran-ordered {rows}x{cols} array")
    if x.ndim == 1 and not x.flags.c_contiguous:
        raise ValueError(f"{name} must be contiguous")
    return x.ctypes.data, rows, False


def execute(nest: LoopNest, A, B, C_, opts: ExecOptions = None, stream=None) -> None:
    """C += A·B through the nest on the GPU (exec.hpp:94-138).

    Device tensors: asynchronous on `stream` (a torch.cuda.Stream, a raw
    cudaStream_t int, or None = torch's current stream). Host numpy arrays:
    synchronous copy-in / run / copy-out."""
    opts = opts or ExecOptions()
    s = nest.shape
    pa, lda, da = _colmajor_view(A, s.m, s.k, "A")
    pb, ldb, db = _colmajor_view(B, s.k, s.n, "B")
    pc, ldc, dc = _colmajor_view(C_, s.m, s.n, "C")
    o = opts._c()
    if da and db and dc:
        if stream is None:
            import torch

            stream = torch.cuda.current_stream().cuda_stream
        elif hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        _check(N.lib().tm_execute(nest._ptr, pa, lda, pb, ldb, pc, ldc, C.byref(o), C.c_void_p(stream)))
    elif not (da or db or dc):
        if lda != s.m or ldb != s.k or ldc != s.m:
            raise ValueError("host operands must be dense column-major")
        _check(N.lib().tm_execute_host(nest._ptr, pa, pb, pc, C.byref(o)))
    else:
        raise ValueError("operands must be all on the device or all on the host")


def fill_seeded(seed: int, shapes):
    """Host inputs exactly as the reference's `run` command fills them
    (mt19937_64 uniform(-1,1), operands in order). Returns flat
    column-major float64 numpy arrays."""
    import numpy as np

    arrs = [np.empty(r * c, dtype=np.float64) for r, c in shapes] + [None] * (3 - len(shapes))
    args = []
    for x in arrs[:3]:
        args += [x.ctypes.data if x is not None else None, x.size if x is not None else 0]
    _check(N.lib().tm_fill_seeded(seed, *args))
    return [x for x in arrs if x is not None]


# ---------------------------------------------------- prepacked layouts
@dataclass(frozen=True)
class BlockLayout:  # layout.hpp:17-98
    rows: int
    cols: int
    steps: Tuple[Tuple[bool, int], ...] = ()  # (on_rows, blocksize), outermost first

    def blocked(self) -> bool:
        return bool(self.steps)

    def element_address(self, i: int, j: int) -> int:
        n = len(self.steps)
        on = (C.c_int32 * max(1, n))(*[int(s[0]) for s in self.steps])
        sz = (C.c_int64 * max(1, n))(*[s[1] for s in self.steps])
        out = C.c_int64(0)
        _check(N.lib().tm_layout_address(self.rows, self.cols, on, sz, n, i, j, C.byref(out)))
        return out.value


def layout_for(nest: "LoopNest", op: str) -> BlockLayout:  # plan.hpp:113-119
    on = (C.c_int32 * 64)()
    sz = (C.c_int64 * 64)()
    n = C.c_int(0)
    _check(N.lib().tm_plan_layout(nest._ptr, op.encode(), on, sz, 64, C.byref(n)))
    s = nest.shape
    return BlockLayout(s.rows(op), s.cols(op), tuple((bool(on[i]), int(sz[i])) for i in range(n.value)))


def _stream_of(stream):
    import torch

    return torch.cuda.current_stream().cuda_stream if stream is None else getattr(stream, "cuda_stream", stream)


def pack(x, nest: "LoopNest", op: str, stream=None):
    """Column-major CUDA tensor -> the plan's hierarchical layout (layout.hpp:122-135)."""
    import torch

    y = torch.empty_like(x)
    _check(N.lib().tm_pack(nest._ptr, op.encode(), x.data_ptr(), y.data_ptr(), C.c_void_p(_stream_of(stream))))
    return y


def unpack(x, nest: "LoopNest", op: str, stream=None):
    """The plan's hierarchical layout -> column-major (layout.hpp:138-145)."""
    import torch

    y = torch.empty_like(x)
    _check(N.lib().tm_unpack(nest._ptr, op.encode(), x.data_ptr(), y.data_ptr(), C.c_void_p(_stream_of(stream))))
    return y


def execute_packed(nest: "LoopNest", Ap, Bp, Cp, opts: ExecOptions = None, stream=None) -> None:
    """execute() on CUDA buffers prepacked in layout_for(nest, op)."""
    o = (opts or ExecOptions())._c()
    _check(N.lib().tm_execute_packed(nest._ptr, Ap.data_ptr(), Bp.data_ptr(), Cp.data_ptr(), C.byref(o),
                                     C.c_void_p(_stream_of(stream))))


DTYPES = {"bf16": 1, "tf32": 2}


def execute_tc(nest: LoopNest, A, B, C_, dtype: str = "bf16", opts: ExecOptions = None, stream=None) -> None:
    """C (fp32) += A·B on the tcgen05 tensor cores. A, B: CUDA tensors,
    column-major flat (bf16 as torch.bfloat16/int16 storage, tf32 as float32
    holding TF32 values). Fused schedule."""
    import torch

    opts = opts or ExecOptions()
    s = nest.shape
    for x, n_, name in ((A, s.m * s.k, "A"), (B, s.k * s.n, "B"), (C_, s.m * s.n, "C")):
        if not (isinstance(x, torch.Tensor) and x.is_cuda and x.numel() == n_ and x.is_contiguous()):
            raise ValueError(f"{name} must be a contiguous CUDA tensor of {n_} elements")
    if C_.dtype != torch.float32:
        raise ValueError("C must be float32")
    st = torch.cuda.current_stream().cuda_stream if stream is None else getattr(stream, "cuda_stream", stream)
    o = opts._c()
    _check(N.lib().tm_execute_tc(nest._ptr, DTYPES[dtype], A.data_ptr(), s.m, B.data_ptr(), s.k, C_.data_ptr(), s.m,
                                 C.byref(o), C.c_void_p(st)))


def round_inputs(x, dtype: str, stream=None):
    """FP64 CUDA tensor -> bf16 (returned as torch.bfloat16) or TF32-valued float32, RNE."""
    import torch

    y = torch.empty(x.numel(), dtype=torch.bfloat16 if dtype == "bf16" else torch.float32, device=x.device)
    st = torch.cuda.current_stream().cuda_stream if stream is None else getattr(stream, "cuda_stream", stream)
    _check(N.lib().tm_round_inputs(DTYPES[dtype], x.data_ptr(), y.data_ptr(), x.numel(), C.c_void_p(st)))
    return y


def fill_uniform_device(x, seed: int, offset: int = 0, stream=None) -> None:
    """Counter-based uniform[-1,1) fill of a CUDA float64 tensor."""
    import torch

    st = torch.cuda.current_stream().cuda_stream if stream is None else getattr(stream, "cuda_stream", stream)
    _check(N.lib().tm_fill_uniform_device(x.data_ptr(), x.numel(), seed, offset, C.c_void_p(st)))


def fill_uniform_block(x, rows: int, cols: int, ld: int, seed: int, row0: int, col0: int, global_ld: int,
                       stream=None) -> None:
    """x(i, j) = counter-based value of global element (row0+i, col0+j) of a
    column-major matrix with leading dimension global_ld (CUDA float64)."""
    import torch

    st = torch.cuda.current_stream().cuda_stream if stream is None else getattr(stream, "cuda_stream", stream)
    _check(N.lib().tm_fill_uniform_block(x.data_ptr(), rows, cols, ld, seed, row0, col0, global_ld, C.c_void_p(st)))


# ------------------------------------------ multi-GPU exchange (copy engines)
def ipc_export(x) -> Tuple[bytes, int]:
    """(CUDA IPC handle of the allocation holding CUDA tensor x, x's byte
    offset in it) -- for a peer process to map with ipc_open."""
    h = (C.c_ubyte * 64)()
    off = C.c_int64(0)
    _check(N.lib().tm_ipc_export(C.c_void_p(x.data_ptr()), h, C.byref(off)))
    return bytes(h), off.value


def ipc_open(handle: bytes, offset: int) -> int:
    """Map a peer's exported allocation on the current device; returns the
    device address of the exported tensor's first byte."""
    h = (C.c_ubyte * 64).from_buffer_copy(handle)
    p = C.c_void_p(None)
    _check(N.lib().tm_ipc_open(h, offset, C.byref(p)))
    return p.value


def ipc_close(ptr: int, offset: int) -> None:
    _check(N.lib().tm_ipc_close(C.c_void_p(ptr), offset))


def copy_async(dst: int, src: int, nbytes: int, stream) -> None:
    """Device-to-device copy by the copy engines on `stream` (a
    torch.cuda.Stream or raw handle); src may be a mapped peer address."""
    st = getattr(stream, "cuda_stream", stream)
    _check(N.lib().tm_copy_async(C.c_void_p(dst), C.c_void_p(src), nbytes, C.c_void_p(st)))


def measure_tc_peak(dtype: str = "bf16", launches: int = 10, sustained: bool = False) -> float:
    """Peak tcgen05 MMA TFLOP/s of the current device for bf16 or tf32 inputs
    (roofline denominator): ~5 ms bursts at full clocks, or ~200 ms launches
    under the power cap (sustained=True)."""
    v = C.c_double(0)
    _check(N.lib().tm_measure_tc_peak(DTYPES.get(dtype, 0), launches, int(sustained), C.byref(v)))
    return v.value


def measure_fp64_peak(launches: int = 20) -> float:
    """Sustained FP64 DMMA TFLOP/s of the current device (roofline denominator)."""
    v = C.c_double(0)
    _check(N.lib().tm_measure_fp64_peak(launches, C.byref(v)))
    return v.value


# ------------------------------------------- trace-driven model check
# trace.hpp / cachesim.hpp: the element-access stream of a nest, replayed
# through a multilevel fully associative LRU hierarchy (native, C ABI
# tm_trace / tm_sim_*), and the model-vs-simulation comparison.
READ, WRITE = "R", "W"  # AccessKind::read / write


@dataclass(frozen=True)
class TraceEvent:  # trace.hpp:17-21
    op: str
    index: int
    kind: str  # "R" | "W"


@dataclass(frozen=True)
class TraceLayouts:  # trace.hpp:27-46
    """Operand addressing of a trace: column-major, or the nest's packed layouts."""
    a: BlockLayout
    b: BlockLayout
    c: BlockLayout
    packed_layouts: bool = False

    @staticmethod
    def column_major(s: Shape) -> "TraceLayouts":
        return TraceLayouts(BlockLayout(s.m, s.k), BlockLayout(s.k, s.n), BlockLayout(s.m, s.n), False)

    @staticmethod
    def packed(nest: "LoopNest") -> "TraceLayouts":
        return TraceLayouts(layout_for(nest, "A"), layout_for(nest, "B"), layout_for(nest, "C"), True)

    def of(self, op: str) -> BlockLayout:
        return {"A": self.a, "B": self.b, "C": self.c}[op]


def trace_event_count(nest: "LoopNest") -> int:  # trace.hpp:73-79
    r = int(N.lib().tm_trace_event_count(nest._ptr))
    if r < 0:
        _check(-r)
    return r


def generate_trace(nest: "LoopNest", lay: TraceLayouts, sink=None, limit: Optional[int] = None):
    """The nest's element accesses in program order (trace.hpp:51-71). Calls
    sink(event) per event when given, else returns the list. `limit` caps the
    number of events materialised (the full stream is trace_event_count)."""
    total = trace_event_count(nest)
    cap = total if limit is None else min(limit, total)
    ops = (C.c_char * max(1, cap))()
    idx = (C.c_int64 * max(1, cap))()
    wr = (C.c_uint8 * max(1, cap))()
    cnt = C.c_int64(0)
    _check(N.lib().tm_trace(nest._ptr, int(lay.packed_layouts), cap, ops, idx, wr, C.byref(cnt)))
    raw = bytes(ops)[:cap].decode()
    events = [TraceEvent(raw[e], idx[e], WRITE if wr[e] else READ) for e in range(cap)]
    if sink is None:
        return events
    for e in events:
        sink(e)
    return None


def write_trace_event(out, e: TraceEvent) -> None:  # trace.hpp:82-84: "OPERAND index R|W"
    out.write(f"{e.op} {e.index} {e.kind}\n")


@dataclass
class SimLevelStats:  # cachesim.hpp:18-38
    level: int
    capacity_lines: int
    granularity: int
    hits: int
    read_misses: int
    write_misses: int
    fetched_lines: int
    passthrough_writes: int
    writebacks: int
    per_operand_misses: Dict[str, int]
    per_operand_writebacks: Dict[str, int]

    def misses(self) -> int:
        return self.read_misses + self.write_misses

    def transferred_elements(self) -> int:
        """Elements crossing the boundary above this level, both directions."""
        return self.granularity * (self.fetched_lines + self.writebacks) + self.passthrough_writes


@dataclass
class SimResult:  # cachesim.hpp:40-50
    levels: List[SimLevelStats]
    events: int

    def at_level(self, h: int) -> SimLevelStats:
        for s in self.levels:
            if s.level == h:
                return s
        raise KeyError("level not simulated")

    def outermost(self) -> SimLevelStats:
        return self.levels[-1]


@dataclass
class SimOptions:  # cachesim.hpp:52-55
    include_registers: bool = False
    flush_dirty_at_end: bool = True


class LruSimulator:  # cachesim.hpp:61-354
    """Fully associative LRU per level, inward-out lookups, inclusive
    back-invalidation, write-allocate / write-back per level (native)."""

    def __init__(self, hier: CacheHierarchy, shape: Shape, opts: Optional[SimOptions] = None):
        o = opts or SimOptions()
        h, nh = hier._c()
        ptr = C.c_void_p(None)
        _check(N.lib().tm_sim_create(h, nh, shape.m, shape.n, shape.k, int(o.include_registers),
                                     int(o.flush_dirty_at_end), C.byref(ptr)))
        self._ptr = ptr
        self._nlev = hier.size() - (0 if o.include_registers else 1)

    def __del__(self):
        p = getattr(self, "_ptr", None)
        if p is not None and p.value and N is not None and N._lib is not None:
            N._lib.tm_sim_destroy(p)
            self._ptr = None

    def access(self, e) -> None:
        """One event: a TraceEvent or an (op, index, kind) tuple."""
        op, index, kind = (e.op, e.index, e.kind) if isinstance(e, TraceEvent) else e
        self.access_many([op], [index], [kind == WRITE])

    def access_many(self, ops: Sequence[str], indices: Sequence[int], writes: Optional[Sequence[bool]] = None) -> None:
        n = len(indices)
        o = "".join(ops).encode()
        if len(o) != n:
            raise ValueError("ops and indices differ in length")
        ix = (C.c_int64 * max(1, n))(*indices)
        wr = (C.c_uint8 * max(1, n))(*([int(bool(w)) for w in writes] if writes is not None else [0] * n))
        _check(N.lib().tm_sim_access(self._ptr, o, ix, wr, n))

    def replay(self, nest: "LoopNest", lay: TraceLayouts) -> None:
        _check(N.lib().tm_sim_replay(self._ptr, nest._ptr, int(lay.packed_layouts)))

    def simulated_levels(self) -> int:
        return self._nlev

    def finish(self) -> SimResult:
        arr = (N.tm_sim_level * 16)()
        cnt, ev = C.c_int(0), C.c_int64(0)
        _check(N.lib().tm_sim_finish(self._ptr, arr, 16, C.byref(cnt), C.byref(ev)))
        lv = []
        for i in range(cnt.value):
            a = arr[i]
            lv.append(SimLevelStats(a.level, a.capacity_lines, a.granularity, a.hits, a.read_misses, a.write_misses,
                                    a.fetched_lines, a.passthrough_writes, a.writebacks,
                                    dict(zip(OPERANDS, list(a.per_operand_misses))),
                                    dict(zip(OPERANDS, list(a.per_operand_writebacks)))))
        return SimResult(lv, ev.value)

    def resident_lines(self, position: int) -> List[int]:
        cnt = C.c_int(0)
        _check(N.lib().tm_sim_resident_lines(self._ptr, position, None, 0, C.byref(cnt)))
        buf = (C.c_int64 * max(1, cnt.value))()
        _check(N.lib().tm_sim_resident_lines(self._ptr, position, buf, cnt.value, C.byref(cnt)))
        return list(buf[:cnt.value])


def simulate(nest: "LoopNest", lay: TraceLayouts, hier: CacheHierarchy,
             opts: Optional[SimOptions] = None) -> SimResult:  # cachesim.hpp:356-362
    sim = LruSimulator(hier, nest.shape, opts)
    sim.replay(nest, lay)
    return sim.finish()


@dataclass
class LevelComparison:  # cachesim.hpp:367-372
    level: int
    model_elements: int
    sim_elements: int
    rel_error: float


@dataclass
class ComparisonReport:
    levels: List[LevelComparison]
    max_rel_error: float


def compare_model(sim: SimResult, model: CostReport) -> ComparisonReport:  # cachesim.hpp:379-392
    """Per simulated level: the model's reads+writes into that level against
    the simulated boundary transfers. ValueError on mismatched hierarchies."""
    out, worst = [], 0.0
    for s in sim.levels:
        try:
            lt = model.at_level(s.level)
        except KeyError:
            raise ValueError(f"simulated level {s.level} missing from the model report: mismatched hierarchies")
        me, se = lt.total_elements(), s.transferred_elements()
        err = (0.0 if se == 0 else float("inf")) if me == 0 else abs(se - me) / me
        worst = max(worst, err)
        out.append(LevelComparison(s.level, me, se, err))
    return ComparisonReport(out, worst)
