"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracle.

Two libraries, both checkers, never the thing measured or shipped:

* ``oracle/liboracle.so`` — plain-C restatement of the reference's execution
  path (``oracle/oracle.c``; exec.hpp:15-46, plan.hpp:61-84) and of the
  seeded generator of ``tilemul run`` (tools/tilemul_main.cpp:236-242).
* ``oracle/_ref/libtilemul_ref.so`` — the reference headers themselves,
  compiled unmodified by ``oracle/Makefile`` (``ref_shim.cpp`` only adds a
  C ABI). Present wherever it was built (this container, and the GPU box via
  the gpurun snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline
leg and the ``--impl reference`` arm) may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtilemul_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")

_lib = None
_ref = None

DIM_INDEX = {"m": 0, "n": 1, "k": 2}


def build() -> None:
    """Compile the oracle (and the reference, when its tree is present)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.or_fill_uniform.argtypes = [C.c_uint64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]
        L.or_fill_uniform.restype = None
        L.or_reference_gemm.argtypes = [C.c_int64] * 3 + [_dp, _dp, _dp]
        L.or_reference_gemm.restype = None
        L.or_execute.argtypes = [C.c_int64] * 3 + [_i32p, _i64p, C.c_int, C.c_int64, C.c_int64, _dp, _dp, _dp, C.c_int]
        L.or_execute.restype = C.c_int64
        L.or_entries.argtypes = [C.c_int64] * 3 + [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                                  _i64p, _i64p, C.c_int64, C.c_int, _dp, C.c_void_p]
        L.or_entries.restype = None
        L.or_abs_product.argtypes = [C.c_int64] * 3 + [_dp, _dp, _dp]
        L.or_abs_product.restype = None
        _lib = L
    return _lib


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference itself (oracle/_ref). Raises if it was never built."""
    global _ref
    if _ref is None:
        if not have_ref():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        L = C.CDLL(REF_SO)
        cp = C.c_char_p
        L.ref_fill_uniform.argtypes = [C.c_uint64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]
        L.ref_fill_uniform.restype = None
        L.ref_mt19937_64.argtypes = [C.c_uint64, C.c_int64]
        L.ref_mt19937_64.restype = C.c_uint64
        L.ref_parse.argtypes = [cp, _i32p, C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_int), C.c_char_p, C.c_int]
        hier = [_i64p, _i32p, C.c_int, C.c_int64, C.c_int64, C.c_int64]
        bs = [_i32p, C.c_char_p, _i64p, C.c_int]
        L.ref_derive.argtypes = hier + [C.c_double, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_double] + bs + [
            _i32p, C.c_char_p, _i64p, C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.ref_derive.argtypes = [cp] + L.ref_derive.argtypes
        L.ref_validate.argtypes = [cp] + hier + bs + [C.c_char_p, C.c_int]
        L.ref_cost.argtypes = [cp] + hier + bs + [_i64p, C.c_char_p, C.c_int]
        L.ref_nest.argtypes = [cp] + hier + bs + [_i32p, C.c_char_p, _i64p, _i32p, C.POINTER(C.c_int),
                                                  C.POINTER(C.c_int64), C.c_char_p, C.c_int]
        L.ref_execute.argtypes = [cp] + hier + bs + [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                                     C.POINTER(C.c_double), C.c_char_p, C.c_int]
        L.ref_reference_gemm.argtypes = [C.c_int64] * 3 + [_dp, _dp, _dp]
        L.ref_reference_gemm.restype = None
        L.ref_micro_kernel.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                       C.c_int64, C.c_int64, C.c_int64]
        L.ref_micro_kernel.restype = None
        L.ref_io_lower_bound.argtypes = [C.c_int64] * 4 + [C.POINTER(C.c_int64)] * 2
        L.ref_io_lower_bound.restype = None
        L.ref_resident_cost.argtypes = [C.c_char] + [C.c_int64] * 5 + [_i64p]
        L.ref_resident_cost.restype = None
        L.ref_streaming_efficiency.argtypes = [C.c_char, C.c_int64, C.c_int64]
        L.ref_streaming_efficiency.restype = C.c_double
        L.ref_goto_efficiency.argtypes = [C.c_int64, C.c_int64]
        L.ref_goto_efficiency.restype = C.c_double
        L.ref_pack.argtypes = [cp] + hier + bs + [C.c_char, C.c_void_p, C.c_void_p, C.c_char_p, C.c_int]
        L.ref_select.argtypes = [C.c_int64] * 4
        L.ref_select.restype = C.c_char
        shier = [_i64p, _i64p, _i32p, C.c_int]
        L.ref_sim_events.argtypes = shier + [C.c_int64] * 3 + [C.c_int, C.c_int, C.c_char_p, _i64p,
                                                               np.ctypeslib.ndpointer(dtype=np.uint8), C.c_int64,
                                                               _i64p, C.POINTER(C.c_int), C.POINTER(C.c_int64),
                                                               C.c_char_p, C.c_int]
        L.ref_simulate.argtypes = [cp] + hier + bs + shier + [C.c_int, C.c_int, C.c_int, _i64p, C.POINTER(C.c_int),
                                                              C.POINTER(C.c_int64), C.c_char_p, C.c_int]
        L.ref_pareto.argtypes = [C.c_int64, _dp, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_int64,
                                 C.c_int64, _dp, C.c_char_p, C.c_int]
        L.ref_trace.argtypes = [cp] + hier + bs + [C.c_int, C.c_int64, C.c_char_p, _i64p,
                                                   np.ctypeslib.ndpointer(dtype=np.uint8), C.POINTER(C.c_int64),
                                                   C.c_char_p, C.c_int]
        _ref = L
    return _ref


# --------------------------------------------------------------------------
# Restatement (liboracle.so)
# --------------------------------------------------------------------------

def fill_uniform(seed: int, shapes, lib_=None):
    """Seeded matrices exactly as ``tilemul run`` fills them: one mt19937_64
    stream, uniform(-1,1), operands in the given order (A, B[, C]).
    ``shapes`` = list of (rows, cols); returns column-major float64 arrays
    (flat, Fortran order)."""
    arrs = [np.empty(r * c, dtype=np.float64) for r, c in shapes]
    while len(arrs) < 3:
        arrs.append(None)
    L = lib_ or lib()
    fn = L.or_fill_uniform if hasattr(L, "or_fill_uniform") else L.ref_fill_uniform
    args = [C.c_uint64(seed)]
    for a in arrs[:3]:
        args += [a.ctypes.data if a is not None else None, C.c_int64(a.size if a is not None else 0)]
    fn(*args)
    return [a for a in arrs if a is not None]


def reference_gemm(m, n, k, a, b, c):
    """In place: c += a·b, naive i-j-p (exec.hpp:15-30)."""
    lib().or_reference_gemm(m, n, k, a, b, c)


def execute_nest(m, n, k, loops, mr, nr, a, b, c, fused=False) -> int:
    """In place: the restated execute() over a nest given as [(dim, bs)]."""
    dims = np.array([DIM_INDEX[d] for d, _ in loops], dtype=np.int32)
    bsz = np.array([b for _, b in loops], dtype=np.int64)
    return lib().or_execute(m, n, k, dims, bsz, len(loops), mr, nr, a, b, c, 1 if fused else 0)


def entries(k, a, lda, b, ldb, c0, ldc, ii, jj, fused=False):
    """Sequential-k values of sampled C entries plus (|A||B|)_ij for each."""
    ii = np.ascontiguousarray(ii, dtype=np.int64)
    jj = np.ascontiguousarray(jj, dtype=np.int64)
    out = np.empty(ii.size, dtype=np.float64)
    ab = np.empty(ii.size, dtype=np.float64)
    lib().or_entries(0, 0, k, a.ctypes.data, lda, b.ctypes.data, ldb,
                     c0.ctypes.data if c0 is not None else None, ldc, ii, jj, ii.size, 1 if fused else 0,
                     out, ab.ctypes.data)
    return out, ab


def abs_product(m, n, k, a, b):
    out = np.empty(m * n, dtype=np.float64)
    lib().or_abs_product(m, n, k, np.abs(a), np.abs(b), out)
    return out


# --------------------------------------------------------------------------
# The reference (oracle/_ref)
# --------------------------------------------------------------------------

def _hier_args(caps, inclusive=None):
    caps = np.ascontiguousarray(caps, dtype=np.int64)
    inc = np.ascontiguousarray(inclusive if inclusive is not None else [0] * caps.size, dtype=np.int32)
    return caps, inc, caps.size


def _bs_args(bs):
    """bs: dict {(level, dim): value} or list of (level, dim, value)."""
    items = sorted(bs.items()) if isinstance(bs, dict) else list(bs)
    if isinstance(bs, dict):
        items = [(lv, d, v) for (lv, d), v in items]
    lvl = np.array([i[0] for i in items], dtype=np.int32)
    dim = "".join(i[1] for i in items).encode()
    val = np.array([i[2] for i in items], dtype=np.int64)
    return lvl, dim, val, len(items)


def ref_derive(name, caps, shape, slack=1.0 / 16.0, mr=4, nr=12, betas=(1.0, 1.0, 1.0), pinned=None,
               inclusive=None):
    L = ref()
    lvl, dim, val, npin = _bs_args(pinned or {})
    ol = np.zeros(64, dtype=np.int32)
    od = C.create_string_buffer(64)
    ov = np.zeros(64, dtype=np.int64)
    no = C.c_int(0)
    err = C.create_string_buffer(4096)
    rc = L.ref_derive(name.encode(), *_hier_args(caps, inclusive), *shape, slack, mr, nr, *betas,
                      lvl, dim, val, npin, ol, od, ov, C.byref(no), err, 4096)
    if rc != 0:
        return rc, err.value.decode()
    return 0, {(int(ol[i]), od.raw[i:i + 1].decode()): int(ov[i]) for i in range(no.value)}


def ref_validate(name, caps, shape, bs, inclusive=None):
    L = ref()
    err = C.create_string_buffer(1 << 16)
    n = L.ref_validate(name.encode(), *_hier_args(caps, inclusive), *shape, *_bs_args(bs), err, 1 << 16)
    rules = [ln.split(":") for ln in err.value.decode().splitlines() if ln]
    return n, [(r[0], int(r[1]), int(r[2]), int(r[3])) for r in rules] if n > 0 else []


def ref_cost(name, caps, shape, bs, inclusive=None):
    L = ref()
    caps_a = np.ascontiguousarray(caps, dtype=np.int64)
    out = np.zeros(caps_a.size * 6, dtype=np.int64)
    err = C.create_string_buffer(4096)
    rc = L.ref_cost(name.encode(), *_hier_args(caps, inclusive), *shape, *_bs_args(bs), out, err, 4096)
    if rc != 0:
        raise ValueError(err.value.decode())
    return out.reshape(caps_a.size, 3, 2)


def ref_nest(name, caps, shape, bs, inclusive=None):
    L = ref()
    ol = np.zeros(64, dtype=np.int32)
    od = C.create_string_buffer(64)
    ob = np.zeros(64, dtype=np.int64)
    oc = np.zeros(64, dtype=np.int32)
    nl = C.c_int(0)
    cells = C.c_int64(0)
    err = C.create_string_buffer(4096)
    rc = L.ref_nest(name.encode(), *_hier_args(caps, inclusive), *shape, *_bs_args(bs), ol, od, ob, oc,
                    C.byref(nl), C.byref(cells), err, 4096)
    if rc != 0:
        raise ValueError(err.value.decode())
    loops = [(int(ol[i]), od.raw[i:i + 1].decode(), int(ob[i]), bool(oc[i])) for i in range(nl.value)]
    return loops, cells.value


def ref_execute(name, caps, shape, bs, a, b, c, workers=1, parallel_loop=-1, packed=False, inclusive=None):
    """In place on c (float64 column-major). Returns execute() seconds."""
    L = ref()
    secs = C.c_double(0)
    err = C.create_string_buffer(4096)
    rc = L.ref_execute(name.encode(), *_hier_args(caps, inclusive), *shape, *_bs_args(bs), a.ctypes.data,
                       b.ctypes.data, c.ctypes.data, workers, parallel_loop, 1 if packed else 0, C.byref(secs),
                       err, 4096)
    if rc != 0:
        raise ValueError(f"rc={rc}: {err.value.decode()}")
    return secs.value


def counter_uniform(seed: int, index):
    """The device generator (tm_fill_uniform_*), restated in numpy:
    v = 2u - 1, u = top 53 bits of splitmix64(seed + (index + 1) * golden)."""
    idx = np.asarray(index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (idx + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return 2.0 * u - 1.0


def round_rne(x, bits: int):
    """x (float64) rounded to `bits` significant bits, round-to-nearest-even,
    in one step (no double rounding through fp32): bf16 = 8 bits, TF32 = 11.
    The restatement of the device's k_round_bf16 / k_round_tf32 for values in
    the normal range of fp32 (every uniform[-1,1) input)."""
    x = np.asarray(x, dtype=np.float64)
    mant, ex = np.frexp(x)                      # x = mant * 2^ex, 0.5 <= |mant| < 1
    return np.ldexp(np.rint(np.ldexp(mant, bits)), ex - bits)  # np.rint: half to even


def counter_entries(k, ii, jj, seeds=(1, 2, 3), lda=None, ldb=None, ldc=None, row0=0, col0=0, steps=1,
                    a_round=None, c0=True):
    """Sampled entries of C = C0 + steps·A·B where A (lda-strided, column-major),
    B and C0 are the device's counter-based fills (tm_fill_uniform_*, restated
    by counter_uniform) over GLOBAL indices: A(i, p) = u(seeds[0], i + p·lda),
    B(p, j) = u(seeds[1], p + j·ldb), C0(i, j) = u(seeds[2], i + j·ldc);
    (ii, jj) are local indices offset by (row0, col0). Nothing is read back
    from the GPU: the inputs are regenerated here.

    a_round (bits): round A and B as the tensor-core path does (round_rne).
    Returns (want, absprod, c0) for the bound 4(steps·k+1)u(steps·|A||B| + |C0|):
    want = c0 + steps·Σ_p a·b, summed sequentially in ascending p (or_entries)."""
    ii = np.asarray(ii, dtype=np.int64)
    jj = np.asarray(jj, dtype=np.int64)
    S = ii.size
    gi = (ii + row0).astype(np.uint64)
    gj = (jj + col0).astype(np.uint64)
    p = np.arange(k, dtype=np.uint64)
    rows = counter_uniform(seeds[0], gi[:, None] + p[None, :] * np.uint64(lda))     # (S, k)
    cols = counter_uniform(seeds[1], p[None, :] + gj[:, None] * np.uint64(ldb))     # (S, k)
    if a_round:
        rows, cols = round_rne(rows, a_round), round_rne(cols, a_round)
    a_s = np.asfortranarray(rows).ravel(order="F")   # S x k column-major: a_s[t + p*S]
    b_s = np.ascontiguousarray(cols).ravel()          # k x S column-major: b_s[p + t*k]
    t = np.arange(S, dtype=np.int64)
    dot, ab = entries(k, a_s, S, b_s, k, None, S, t, t)
    cz = counter_uniform(seeds[2], gi + gj * np.uint64(ldc)) if c0 else np.zeros(S)
    return cz + steps * dot, ab, cz


def ref_pack(name, caps, shape, bs, op, src, inclusive=None):
    """The reference's pack(src, nest) of operand `op` (column-major -> layout_for)."""
    L = ref()
    dst = np.empty_like(src)
    err = C.create_string_buffer(4096)
    rc = L.ref_pack(name.encode(), *_hier_args(caps, inclusive), *shape, *_bs_args(bs), op.encode(), src.ctypes.data,
                    dst.ctypes.data, err, 4096)
    if rc != 0:
        raise ValueError(err.value.decode())
    return dst


# --- trace generator / LRU simulator of the reference ----------------------
SIM_FIELDS = ("level", "capacity_lines", "granularity", "hits", "read_misses", "write_misses", "fetched_lines",
              "passthrough_writes", "writebacks", "misses_A", "misses_B", "misses_C", "writebacks_A",
              "writebacks_B", "writebacks_C")


def _sim_hier(levels):
    """levels: [(capacity, granularity, inclusive, write_allocate, write_back)]."""
    caps = np.array([lv[0] for lv in levels], dtype=np.int64)
    gran = np.array([lv[1] for lv in levels], dtype=np.int64)
    flags = np.array([int(bool(x)) for lv in levels for x in lv[2:5]], dtype=np.int32)
    return caps, gran, flags, len(levels)


def _sim_out(rc, out, nout, events, err):
    if rc != 0:
        raise ValueError(err.value.decode())
    return [dict(zip(SIM_FIELDS, map(int, out[15 * i:15 * i + 15]))) for i in range(nout.value)], events.value


def ref_sim_events(levels, shape, ops, idx, writes, include_registers=False, flush=True):
    """The reference LruSimulator over an explicit event list -> ([level stats], events)."""
    L = ref()
    out = np.zeros(15 * 16, dtype=np.int64)
    nout, ev = C.c_int(0), C.c_int64(0)
    err = C.create_string_buffer(4096)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    wr = np.ascontiguousarray(writes, dtype=np.uint8)
    rc = L.ref_sim_events(*_sim_hier(levels), *shape, int(include_registers), int(flush), "".join(ops).encode(),
                          idx, wr, idx.size, out, C.byref(nout), C.byref(ev), err, 4096)
    return _sim_out(rc, out, nout, ev, err)


def ref_simulate(name, caps, shape, bs, sim_levels, packed=False, include_registers=False, flush=True):
    """The reference simulate() of build_plan(name, caps, shape, bs) through sim_levels."""
    L = ref()
    out = np.zeros(15 * 16, dtype=np.int64)
    nout, ev = C.c_int(0), C.c_int64(0)
    err = C.create_string_buffer(4096)
    rc = L.ref_simulate(name.encode(), *_hier_args(caps), *shape, *_bs_args(bs), *_sim_hier(sim_levels),
                        int(packed), int(include_registers), int(flush), out, C.byref(nout), C.byref(ev), err, 4096)
    return _sim_out(rc, out, nout, ev, err)


def ref_trace(name, caps, shape, bs, packed=False, cap=1 << 20):
    """The reference generate_trace (first `cap` events) -> (ops str, idx, writes, total count)."""
    L = ref()
    ops = C.create_string_buffer(max(1, cap))
    idx = np.zeros(max(1, cap), dtype=np.int64)
    wr = np.zeros(max(1, cap), dtype=np.uint8)
    cnt = C.c_int64(0)
    err = C.create_string_buffer(4096)
    rc = L.ref_trace(name.encode(), *_hier_args(caps), *shape, *_bs_args(bs), int(packed), cap, ops, idx, wr,
                     C.byref(cnt), err, 4096)
    if rc != 0:
        raise ValueError(err.value.decode())
    n = min(cap, cnt.value)
    return ops.raw[:n].decode(), idx[:n], wr[:n], cnt.value


def ref_pareto(outer, ratios, shape, slack=1.0 / 16.0, mr=4, nr=12):
    """The reference pareto_sweep -> list of 8-tuples (ParetoPoint fields), or ValueError."""
    L = ref()
    r = np.ascontiguousarray(ratios, dtype=np.float64)
    out = np.zeros(8 * max(1, r.size), dtype=np.float64)
    err = C.create_string_buffer(4096)
    rc = L.ref_pareto(outer, r, r.size, *shape, slack, mr, nr, out, err, 4096)
    if rc != 0:
        raise ValueError(err.value.decode())
    return [tuple(out[8 * i:8 * i + 8]) for i in range(r.size)]
