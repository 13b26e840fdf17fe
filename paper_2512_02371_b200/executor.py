"""GPU backend for ``interp.run_program`` on convolution-family programs.

Drop-in for the reference executor (interp.py:570-619) on the programs the
conv rules produce (rules.py:766-836, 887-902) and on their source forms
(tools/make_corpus.py:142-208):

* lowered:  ``wmma_zero`` / ``ConvolutionShuffle`` | ``PolyphaseShuffle`` |
  ``Shuffle(load K ...)`` / ``wmma_mma(wmma_load_a, wmma_load_b, acc)`` /
  ``wmma_store``, optionally inside ``For`` loops with affine bases;
* source:   ``Store(acc, ramp, VectorReduceAdd(Load I · Load K) + Load acc)``
  and plain buffer copies.

Each conv statement group runs as ONE launch of ``ts_run_conv_group`` over
every program instance (``run_program_batch``: e.g. all seeds of a
difftest), reproducing interp's arithmetic exactly (operand re-rounding,
f32 products, left-to-right sums, ``acc + s``) — results are bit-identical,
so the reference's own difftest (cli.py:161-183) passes bitwise.

Programs are duck-typed: real ``tensorsel.ir`` objects or the mirrors in
:mod:`irlite`.  Anything outside this family raises ``UnsupportedProgram``;
there is no CPU fallback.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib, layout
from .errors import (DivideByZero, EvalError, I32Overflow, OutOfBounds, ShapeUnregistered,
                     UnknownIntrinsic)

HARDWARE_SHAPES = (("wmma", 32, 16, 8), ("wmma", 16, 16, 16), ("amx", 16, 32, 16))
_KIND = {"f32": 0, "f16": 1, "bf16": 2}


class UnsupportedProgram(EvalError):
    """A statement outside the conv family the GPU executor implements."""


try:  # the drop-in case: return the reference's own Buffer / BufferStore types
    from tensorsel.interp import Buffer, BufferStore  # noqa: F401
except Exception:  # reference not installed (e.g. on the GPU box): same-shaped mirrors
    class Buffer:
        """interp.Buffer (interp.py:132-136)."""

        def __init__(self, kind, location, data):
            self.kind, self.location, self.data = kind, location, data

        def __repr__(self):
            return f"Buffer({self.kind!r}, {self.location!r}, <{len(self.data)}>)"

    class BufferStore(dict):
        """interp.BufferStore (interp.py:139-140): name -> Buffer."""


def _cls(x):
    return type(x).__name__


# ------------------------------------------------------------------ expressions
def _check_i32(v):
    """interp._check_i32 (interp.py:156-159)."""
    if v >= 2 ** 31 or v < -(2 ** 31):
        raise I32Overflow(f"i32 range exceeded (max {v}, min {v})")
    return v


def _check_i32_vec(a):
    if a.size and (a.max() >= 2 ** 31 or a.min() < -(2 ** 31)):
        raise I32Overflow(f"i32 range exceeded (max {a.max()}, min {a.min()})")
    return a


def _int_bop(op, a, b):
    """interp._bop on i32 (interp.py:251-266): Euclidean / and %, overflow-checked."""
    if op == "+":
        return a + b
    if op == "-":
        return a - b
    if op == "*":
        return a * b
    if op in ("/", "%"):
        if np.any(np.asarray(b) == 0):
            raise DivideByZero(f"integer {op} by zero")
        r = np.mod(a, np.abs(b))
        return r if op == "%" else (a - r) // b
    raise EvalError(f"unknown op {op}")


def _eval_int(e, env):
    c = _cls(e)
    if c == "Imm":
        return _check_i32(int(e.value))
    if c == "Var":
        if e.name not in env:
            raise EvalError(f"unbound variable {e.name!r}")
        return env[e.name]
    if c == "Bop":
        a, b = _eval_int(e.lhs, env), _eval_int(e.rhs, env)
        return _check_i32(int(_int_bop(e.op, a, b)))
    raise UnsupportedProgram(f"non-scalar integer expression {c}")


def _eval_index(e, env):
    """Index vector of a Ramp/Broadcast tree (interp.py:191-202)."""
    c = _cls(e)
    if c in ("Imm", "Var", "Bop"):
        if c == "Bop" and (_cls(e.lhs) in ("Ramp", "Broadcast")
                           or _cls(e.rhs) in ("Ramp", "Broadcast")):
            a, b = _eval_index(e.lhs, env), _eval_index(e.rhs, env)
            return _check_i32_vec(_int_bop(e.op, a, b))
        return np.array([_eval_int(e, env)], np.int64)
    if c == "Ramp":
        base = _eval_index(e.base, env)
        stride = _eval_index(e.stride, env)
        steps = np.arange(e.steps).reshape(-1, 1)
        return _check_i32_vec((base + steps * stride).reshape(-1))
    if c == "Broadcast":
        return np.tile(_eval_index(e.operand, env), e.copies)
    raise UnsupportedProgram(f"index expression {c}")


def _unit_ramp(index):
    return (_cls(index) == "Ramp" and _cls(index.stride) == "Imm"
            and int(index.stride.value) == 1)


def _is_flat(index, length=None):
    return (_cls(index) == "Ramp" and _cls(index.base) == "Imm" and int(index.base.value) == 0
            and _cls(index.stride) == "Imm" and int(index.stride.value) == 1
            and (length is None or index.steps == length))


# ------------------------------------------------------------------ plan
class _Group:
    """One conv statement group (one ts_run_conv_group launch)."""

    def __init__(self, acc, src, kern, m, k, n):
        self.acc, self.src, self.kern = acc, src, kern
        self.m, self.k, self.n = m, k, n
        self.a_stride = 0
        self.a_base, self.k_base = [], []
        self.b_off = None
        self.a_idx, self.b_idx = [], []   # explicit mode (source form)
        self.tmp = None                    # lowered: the temporary holding B
        self.paths = []                    # statement path of every iteration


class _Plan:
    def __init__(self):
        self.ops = []


def _shape_registry(p, extra_shapes, strict):
    decls = set(HARDWARE_SHAPES)
    if not strict:
        for s in tuple(getattr(p, "shapes", ())) + tuple(extra_shapes):
            decls.add((s.target, s.m, s.k, s.n))
    return decls


def _matrix_offsets(call, env):
    """(kernel buffer, window base, k*n offsets or -1) for a B builder:
    ConvolutionShuffle / PolyphaseShuffle (interp.py:488-534) or a desugared
    Shuffle over a kernel load (interp.py:220-225)."""
    c = _cls(call)
    if c == "Call" and call.name in ("ConvolutionShuffle", "PolyphaseShuffle"):
        kbuf = call.args[0].name
        base = _eval_int(call.args[1], env)
        if call.name == "ConvolutionShuffle":
            rows, cols = int(call.args[2].value), int(call.args[3].value)
            spec = layout.ToeplitzSpec(l=rows - cols, k=cols)
        else:
            l, k, pp, s = (int(a.value) for a in call.args[2:6])
            spec = layout.ToeplitzSpec(l=l, k=k, s=s, p=pp)
        idx = np.asarray(layout.shuffle_indices_for(spec, 0, 1 << 30), np.int64)
        off = np.where(idx < 0, -1, idx - 1)  # lane 0 is the zero lane
        return kbuf, base, off.astype(np.int32), spec.k
    if c == "Shuffle":
        src = call.source
        if _cls(src) != "Load" or _cls(src.index) != "Ramp" or _cls(src.index.stride) != "Imm" \
                or int(src.index.stride.value) != 1:
            raise UnsupportedProgram("shuffle source must be a unit-stride kernel load")
        base = _eval_int(src.index.base, env)
        return src.buffer, base, np.asarray(call.indices, np.int32), None
    raise UnsupportedProgram(f"not a weight builder: {c} {getattr(call, 'name', '')}")


def _annotate(err, sp):
    """interp._exec_stmts's error annotation (interp.py:615-619): the first
    (innermost) statement path is prefixed to the message."""
    if not getattr(err, "stmt_path", None):
        err.stmt_path = sp
        err.args = (f"{sp}: {err.args[0]}",) if err.args else (sp,)
    return err


def _first_oob(idx, length):
    bad = idx[(idx < 0) | (idx >= length)]
    return int(bad.reshape(-1)[0]) if bad.size else None


def _compile(p, extra_shapes, strict):
    """Walk the program like interp._exec_stmts (interp.py:591-619) and
    record its statements as plan ops.  Every index a conv-family program
    touches is affine in the loop variables, so bounds are checked here, on
    the host, in the reference's evaluation order; errors carry the
    reference's statement path (``body[i][j]``)."""
    shapes = _shape_registry(p, extra_shapes, strict)
    kinds = {prm.name: prm.kind for prm in p.params}
    lengths = {prm.name: prm.length for prm in p.params}
    plan = _Plan()
    tmp_defs = {}  # temporary name -> (kernel buf, base, offsets) of the current iteration

    def need(name):
        if name not in lengths:
            raise EvalError(f"unknown buffer {name!r}")
        return lengths[name]

    def check_range(name, lo, hi):
        """A gather/scatter of indices [lo, hi] into `name` (interp._gather / _scatter)."""
        n = need(name)
        if lo < 0:
            raise OutOfBounds(name, int(lo))
        if hi >= n:
            raise OutOfBounds(name, int(hi) if lo >= n else n)

    def emit_stmt(s, env, sp):
        try:
            emit_one(s, env, sp)
        except EvalError as err:
            raise _annotate(err, sp)

    def emit_one(s, env, sp):
        c = _cls(s)
        if c == "Allocate":
            kinds[s.name] = s.kind
            lengths[s.name] = s.length
            plan.ops.append(("alloc", s.name, s.kind, s.length, s.location))
            return
        if c == "Evaluate":
            v = s.value
            if _cls(v) == "Call" and v.name == "wmma_store":
                out = v.args[0].name
                base = _eval_int(v.args[1], env)
                stride = _eval_int(v.args[2], env)
                cols = int(v.args[3].value)
                tile = v.args[4]
                if _cls(tile) != "Load" or not _is_flat(tile.index):
                    raise UnsupportedProgram("wmma_store of a non-buffer tile")
                lanes = tile.index.steps
                check_range(tile.buffer, 0, lanes - 1)
                rows = lanes // cols
                idx = base + stride * np.arange(rows)[:, None] + np.arange(cols)[None, :]
                bad = _first_oob(idx, need(out))
                if bad is not None:
                    raise OutOfBounds(out, bad)
                plan.ops.append(("store", out, tile.buffer, idx.reshape(-1), lanes, sp))
                return
            raise UnsupportedProgram(f"evaluate of {getattr(v, 'name', _cls(v))}")
        if c == "For":
            for it in range(s.min, s.min + s.extent):
                env2 = dict(env)
                env2[s.var] = it
                for j, b in enumerate(s.body):
                    emit_stmt(b, env2, f"{sp}[{j}]")
            return
        if c != "Store":
            raise UnsupportedProgram(f"statement {c}")
        v = s.value
        vc = _cls(v)
        # acc = wmma_zero(m, n)
        if vc == "Call" and v.name == "wmma_zero":
            lanes = int(v.args[0].value) * int(v.args[1].value)
            if not _is_flat(s.index, lanes):
                raise UnsupportedProgram("wmma_zero must fill its accumulator from 0")
            check_range(s.buffer, 0, lanes - 1)
            plan.ops.append(("zero", s.buffer, lanes))
            return
        # tmp = weight builder
        if (vc == "Call" and v.name in ("ConvolutionShuffle", "PolyphaseShuffle")) or vc == "Shuffle":
            # recorded, not executed: the group that consumes it gathers B
            # on the fly, and materialises the last iteration's temporary
            kbuf, base, off, _ = _matrix_offsets(v, env)
            used = off[off >= 0]
            if used.size:  # the kernel window read (interp.py:488-534, 220-225)
                check_range(kbuf, base + int(used.min()), base + int(used.max()))
            if not _is_flat(s.index, len(off)):
                raise UnsupportedProgram("weight temporary must be stored from 0")
            check_range(s.buffer, 0, len(off) - 1)
            tmp_defs[s.buffer] = (kbuf, base, off)
            return
        # acc = wmma_mma(load_a, load_b, acc)
        if vc == "Call" and v.name == "wmma_mma":
            la, lb, lc = v.args
            if _cls(la) != "Call" or la.name != "wmma_load_a" or _cls(lb) != "Call" \
                    or lb.name != "wmma_load_b":
                raise UnsupportedProgram("wmma_mma operands must be wmma_load_a / wmma_load_b")
            src = la.args[0].name
            a_base, a_stride = _eval_int(la.args[1], env), _eval_int(la.args[2], env)
            m, k = int(la.args[3].value), int(la.args[4].value)
            tmp = lb.args[0].name
            b_base, b_stride = _eval_int(lb.args[1], env), _eval_int(lb.args[2], env)
            bk, bn = int(lb.args[3].value), int(lb.args[4].value)
            # operand A: src[a_base + i*a_stride + kk] (interp._tile_gather, interp.py:408-410)
            rows_off = a_stride * np.arange(m)
            check_range(src, a_base + int(rows_off.min()), a_base + int(rows_off.max()) + k - 1)
            if bk != k:
                raise UnsupportedProgram("wmma_load_b rows must equal wmma_load_a columns")
            if tmp in tmp_defs:  # B = a Toeplitz temporary (conv-toeplitz / upsample-polyphase)
                if b_base != 0 or b_stride != bn:
                    raise UnsupportedProgram("wmma_load_b must read the whole temporary row-major")
                check_range(tmp, 0, k * bn - 1)
                kbuf, kb, off = tmp_defs[tmp]
                if len(off) != k * bn:
                    raise EvalError(f"temporary {tmp!r} has {len(off)} lanes, B needs {k * bn}")
            else:
                # B = a plain buffer tile (the wmma-mma rule's matmul form,
                # rules.py:904-1008): B[b_base + b_stride*r + c], r < k, c < n
                off = (b_stride * np.arange(k)[:, None] + np.arange(bn)[None, :]).reshape(-1)
                check_range(tmp, b_base + int(off.min()), b_base + int(off.max()))
                kbuf, kb, off = tmp, b_base, off.astype(np.int32)
                tmp = None  # nothing to materialise
            if _cls(lc) == "Load" and lc.buffer == s.buffer and _is_flat(lc.index, m * bn):
                check_range(s.buffer, 0, m * bn - 1)
            elif _cls(lc) == "Call" and lc.name == "wmma_zero":
                plan.ops.append(("zero", s.buffer, m * bn))
            else:
                raise UnsupportedProgram("wmma_mma accumulator must be the stored buffer")
            if ("wmma", m, k, bn) not in shapes:
                raise ShapeUnregistered(f"wmma_mma: shape wmma {m}x{k}x{bn} not registered")
            if not _is_flat(s.index):
                raise UnsupportedProgram("wmma_mma result must be stored from 0")
            if s.index.steps != m * bn:
                raise EvalError(f"store index {s.index.steps} lanes, value {m * bn}")
            check_range(s.buffer, 0, m * bn - 1)
            key = ("lowered", s.buffer, src, kbuf, m, k, bn, a_stride, off.tobytes())
            _append_iteration(plan, key, s.buffer, src, kbuf, m, k, bn, a_stride, a_base, kb, off,
                              tmp, sp)
            return
        # acc = VectorReduceAdd(Load I * Load K) + Load acc  (source form)
        if vc == "Bop" and v.op == "+":
            red, acc = v.lhs, v.rhs
            if _cls(red) != "VectorReduceAdd":
                red, acc = acc, red
            if _cls(red) == "VectorReduceAdd" and _cls(acc) == "Load" and acc.buffer == s.buffer:
                _source_conv(plan, s, red, acc, env, check_range, sp)
                return
        # dst = Load src (flat copy)
        if vc == "Load" and _is_flat(s.index) and _is_flat(v.index, s.index.steps):
            n = s.index.steps
            check_range(v.buffer, 0, n - 1)
            check_range(s.buffer, 0, n - 1)
            plan.ops.append(("copy", s.buffer, v.buffer, n, 0, 0))
            return
        # dst[ramp(bd, 1, n)] = Load src[ramp(bs, 1, n)]: a window copy at affine
        # offsets (e.g. each For iteration's accumulator into its output slot)
        if vc == "Load" and _unit_ramp(s.index) and _unit_ramp(v.index) \
                and v.index.steps == s.index.steps:
            n = s.index.steps
            bd, bs = _eval_int(s.index.base, env), _eval_int(v.index.base, env)
            check_range(v.buffer, bs, bs + n - 1)
            check_range(s.buffer, bd, bd + n - 1)
            plan.ops.append(("copy", s.buffer, v.buffer, n, bd, bs))
            return
        if vc == "Broadcast" and _cls(v.operand) == "Imm" and _is_flat(s.index):
            check_range(s.buffer, 0, s.index.steps - 1)
            plan.ops.append(("fill", s.buffer, float(v.operand.value), s.index.steps))
            return
        raise UnsupportedProgram(f"store into {s.buffer!r} of {vc} {getattr(v, 'name', '')}")

    for i, st in enumerate(p.body):
        emit_stmt(st, {}, f"body[{i}]")
    plan.ops = _fuse_independent_iterations(plan.ops)
    return plan


_PLANS: "dict" = {}
_PLANS_MAX = 64


def _compiled(p, extra_shapes, strict):
    """_compile, cached per (program, extra_shapes, strict): programs are
    immutable (frozen dataclasses, here and in tensorsel.ir), and a plan
    only depends on the program, so repeated runs (difftest trials, batches
    of frames) skip the host-side unrolling."""
    try:
        key = (p, tuple(extra_shapes), bool(strict))
        hash(key)
    except TypeError:
        return _compile(p, extra_shapes, strict)
    plan = _PLANS.get(key)
    if plan is None:
        plan = _compile(p, extra_shapes, strict)
        if len(_PLANS) >= _PLANS_MAX:
            _PLANS.pop(next(iter(_PLANS)))
        _PLANS[key] = plan
    return plan


def _fuse_independent_iterations(ops):
    """Peephole over the unrolled plan: a run of For iterations whose body is
    ``acc = 0; acc = conv(...) + acc; out[base_v ..] = acc`` (copy or
    wmma_store) becomes ONE ("scatter", ...) op — every iteration computed
    from zero in parallel and stored to its own slot, then acc set to the
    last iteration's value (the reference's final buffer state).  Each
    iteration's arithmetic is unchanged (0 + s, interp.py:485 / 270-284)."""
    out, i = [], 0
    while i < len(ops):
        run = []
        j = i
        while j + 2 < len(ops):
            f, g, c = ops[j], ops[j + 1], ops[j + 2]
            if f[0] not in ("fill", "zero") or (f[0] == "fill" and f[2] != 0.0):
                break
            if g[0] != "group" or len(g[2].a_base) != 1:
                break
            grp = g[2]
            acc, n = f[1], f[-1]
            if grp.acc != acc or grp.m * grp.n != n or acc in (grp.src, grp.kern):
                break
            if c[1] in (grp.src, grp.kern):  # an iteration would read an earlier one's output
                break
            if c[0] == "copy" and c[2] == acc and c[3] == n and c[5] == 0 and c[1] != acc:
                dst, base, off = c[1], c[4], None
            elif c[0] == "store" and c[2] == acc and c[4] == n and c[1] != acc \
                    and len(np.unique(c[3])) == n:
                dst, base, off = c[1], int(c[3][0]), np.asarray(c[3], np.int64) - int(c[3][0])
            else:
                break
            if run:
                k0, g0, d0, o0 = run[0][1], run[0][2], run[0][3], run[0][5]
                if g[1] != k0 or dst != d0 or acc != g0.acc or \
                        (off is None) != (o0 is None) or (off is not None and
                                                          not np.array_equal(off, o0)):
                    break
            run.append((f, g[1], grp, dst, base, off))
            j += 3
        if len(run) >= 2:
            g0 = run[0][2]
            G = _Group(g0.acc, g0.src, g0.kern, g0.m, g0.k, g0.n)
            G.a_stride, G.b_off, G.tmp = g0.a_stride, g0.b_off, g0.tmp
            for _, _, grp, _, _, _ in run:
                G.a_base += grp.a_base
                G.k_base += grp.k_base
                G.a_idx += grp.a_idx
                G.b_idx += grp.b_idx
                G.paths += grp.paths
            out.append(("scatter", run[0][1], G, run[0][3], [r[4] for r in run], run[0][5],
                        g0.m * g0.n))
            i = j
        else:
            out.append(ops[i])
            i += 1
    return out


def _append_iteration(plan, key, acc, src, kbuf, m, k, n, a_stride, a_base, k_base, off, tmp, sp):
    last = plan.ops[-1] if plan.ops else None
    if last is not None and last[0] == "group" and last[1] == key:
        g = last[2]
    else:
        g = _Group(acc, src, kbuf, m, k, n)
        g.a_stride, g.b_off, g.tmp = a_stride, off, tmp
        plan.ops.append(("group", key, g))
    g.a_base.append(a_base)
    g.k_base.append(k_base)
    g.paths.append(sp)


def _strip_cast(e):
    """Drop Cast-to-f32 nodes: on values already rounded to their buffer kind
    they are the identity (interp._cast, interp.py:241-248).  A cast to any
    other kind rounds or truncates, which the conv kernel does not model."""
    while _cls(e) == "Cast":
        if e.vtype.kind != "f32":
            raise UnsupportedProgram(f"cast to {e.vtype.kind} inside a conv statement")
        e = e.operand
    return e


def _source_conv(plan, s, red, acc, env, check_range, sp):
    """VectorReduceAdd(n_out, Cast(Load I) * [Broadcast](Cast(Load K))) + acc."""
    prod = _strip_cast(red.operand)
    if _cls(prod) != "Bop" or prod.op != "*":
        raise UnsupportedProgram("reduction operand must be a product")
    loads = []
    for side in (prod.lhs, prod.rhs):
        e = _strip_cast(side)
        if _cls(e) == "Broadcast":
            e2 = _strip_cast(e.operand)
            if _cls(e2) != "Load":
                raise UnsupportedProgram("broadcast of a non-load")
            ix = _eval_index(e2.index, env)
            loads.append((e2.buffer, ix, np.tile(ix, e.copies)))
        elif _cls(e) == "Load":
            ix = _eval_index(e.index, env)
            loads.append((e.buffer, ix, ix))
        else:
            raise UnsupportedProgram("product of non-loads")
    for buf, ix, _ in loads:  # gathers in evaluation order (interp.py:183-185)
        if ix.size:
            check_range(buf, int(ix.min()), int(ix.max()))
    (ib, _, ia), (kb, _, ka) = loads
    n_out = red.result_lanes
    if len(ia) != len(ka) or len(ia) % n_out:
        raise EvalError(f"cannot reduce {len(ia)} lanes to {n_out}")
    taps = len(ia) // n_out
    if not _is_flat(acc.index, n_out):
        raise UnsupportedProgram("source-form accumulator must be a flat load of its outputs")
    check_range(acc.buffer, 0, n_out - 1)
    if not _is_flat(s.index, n_out):
        raise UnsupportedProgram("source-form store must be a flat ramp")
    check_range(s.buffer, 0, n_out - 1)
    key = ("source", s.buffer, ib, kb, n_out, taps)
    last = plan.ops[-1] if plan.ops else None
    if last is not None and last[0] == "group" and last[1] == key:
        g = last[2]
    else:
        g = _Group(s.buffer, ib, kb, n_out, taps, 1)
        plan.ops.append(("group", key, g))
    g.a_idx.append(ia.reshape(n_out, taps).astype(np.int32))
    g.b_idx.append(ka.reshape(n_out, taps).astype(np.int32))
    g.a_base.append(0)
    g.k_base.append(0)
    g.paths.append(sp)


# ------------------------------------------------------------------ execution
def _as_data(x):
    return x.data if hasattr(x, "data") and not isinstance(x, np.ndarray) else x


def run_program_batch(p, inputs_list, extra_shapes=(), strict=False, lint_sink=None, device=None):
    """Run program `p` once per element of `inputs_list` (name -> Buffer or
    array) on the GPU; returns one BufferStore per instance (parameters,
    allocations and temporaries, like interp.run_program)."""
    import torch

    if not torch.cuda.is_available():
        from .errors import NoDevice
        raise NoDevice("run_program_batch needs a CUDA device")
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    lib = _lib.load()
    T = len(inputs_list)
    plan = _compiled(p, extra_shapes, strict)
    bufs, meta = {}, {}
    for prm in p.params:
        if prm.kind == "i32":
            raise UnsupportedProgram("i32 parameters are outside the conv family")
        rows = []
        for ins in inputs_list:
            if prm.name not in ins:
                raise EvalError(f"missing input buffer {prm.name!r}")
            d = np.asarray(_as_data(ins[prm.name]), dtype=np.float32)
            if len(d) != prm.length:
                raise EvalError(f"input {prm.name!r} has length {len(d)}, declared {prm.length}")
            rows.append(d)
        bufs[prm.name] = torch.from_numpy(np.stack(rows) if rows else
                                          np.zeros((0, prm.length), np.float32)).to(dev)
        meta[prm.name] = (prm.kind, getattr(prm, "location", "mem"))
    stream = torch.cuda.current_stream(dev).cuda_stream
    err = torch.zeros(3, dtype=torch.int32, device=dev)
    for op in plan.ops:
        kind = op[0]
        if kind == "alloc":
            _, name, k, length, loc = op
            if k == "i32":
                raise UnsupportedProgram("i32 allocations are outside the conv family")
            bufs[name] = torch.zeros((T, length), dtype=torch.float32, device=dev)
            meta[name] = (k, loc)
        elif kind == "zero":
            bufs[op[1]][:, :op[2]] = 0
        elif kind == "fill":
            _, name, val, n = op
            bufs[name][:, :n] = val
        elif kind == "copy":
            _, dst, src, n, bd, bs = op
            for name, b in ((dst, bd), (src, bs)):
                if b < 0 or b + n > bufs[name].shape[1]:
                    raise OutOfBounds(name, b if b < 0 else b + n - 1)
            bufs[dst][:, bd:bd + n] = bufs[src][:, bs:bs + n]
        elif kind == "tmp":
            _, name, kbuf, base, off = op
            K = bufs[kbuf]
            o = torch.from_numpy(off.astype(np.int64)).to(dev)
            if int(off.max(initial=-1)) + base >= K.shape[1] or (off >= 0).any() and base < 0:
                raise OutOfBounds(kbuf, int(base + off.max()))
            vals = K[:, (base + o).clamp(min=0)]
            bufs[name][:, :len(off)] = torch.where(o >= 0, vals, torch.zeros_like(vals))
        elif kind == "store":
            _, out, tile, idx, lanes, _sp = op
            pos = np.arange(lanes)
            if len(np.unique(idx)) != len(idx):
                # interp._scatter (interp.py:549-553): colliding lanes, last wins + a lint
                if lint_sink is not None:
                    lint_sink.extend([f"store into {out!r} has colliding lanes (last wins)"] * T)
                last = {}
                for q, i in enumerate(idx.tolist()):
                    last[i] = q
                pos = np.fromiter(last.values(), np.int64)
                idx = np.fromiter(last.keys(), np.int64)
            src_pos = torch.from_numpy(pos).to(dev)
            bufs[out][:, torch.from_numpy(idx).to(dev)] = bufs[tile][:, src_pos]
        elif kind == "group":
            _run_group(lib, op[2], bufs, meta, T, dev, stream, err)
        elif kind == "scatter":
            _, _, g, dst, bases, off, n = op
            _run_group(lib, g, bufs, meta, T, dev, stream, err, scatter=(dst, bases, off))
            # the accumulator ends holding the last iteration's result
            last = bases[-1] + (torch.from_numpy(off).to(dev) if off is not None
                                else torch.arange(n, device=dev))
            bufs[g.acc][:, :n] = bufs[dst][:, last]
        else:
            raise UnknownIntrinsic(kind)
    torch.cuda.synchronize(dev)
    out = []
    host = {n: b.cpu().numpy() for n, b in bufs.items()}
    for t in range(T):
        st = BufferStore()
        for n, data in host.items():
            k, loc = meta[n]
            st[n] = Buffer(k, loc, data[t])  # a view: each instance owns its row
        out.append(st)
    return out


def _compact(a_idx, b_idx):
    """(table, b table, per-iteration shifts) when every iteration's gather
    is the first one shifted by a constant (e.g. a For loop sliding a conv
    window), else None."""
    A = np.stack(a_idx)
    shifts = A[:, :1, :1] - A[:1, :1, :1]
    if not np.array_equal(A - shifts, np.broadcast_to(A[:1], A.shape)):
        return None
    B = np.stack(b_idx)
    if not np.array_equal(B, np.broadcast_to(B[:1], B.shape)):
        return None
    return A[0], B[0], shifts.reshape(-1)


def _run_group(lib, g, bufs, meta, T, dev, stream, err, scatter=None):
    import torch
    src, kern, acc = bufs[g.src], bufs[g.kern], bufs[g.acc]
    V = len(g.a_base)
    # the group's index tables are fixed per compiled plan: upload once per
    # device and keep them on the group (plans are cached, _compiled)
    cache = g.__dict__.setdefault("_dev_tables", {})
    tables = cache.setdefault(str(dev), {})

    def dptr(arr, name):
        t = tables.get(name)
        if t is None:
            t = tables[name] = torch.from_numpy(
                np.ascontiguousarray(arr() if callable(arr) else arr, dtype=np.int32)).to(dev)
        return t.data_ptr()

    c = _lib.ConvGroup()
    c.instances = T
    c.src, c.src_stride, c.src_len = src.data_ptr(), src.shape[1], src.shape[1]
    # lowered loads re-round to the buffer kind (interp.py:441-442); source-form
    # loads and casts to f32 do not (interp.py:183-188, 241-248)
    c.src_kind = 0 if g.a_idx else _KIND.get(meta[g.src][0], 0)
    c.kern, c.kern_stride, c.kern_len = kern.data_ptr(), kern.shape[1], kern.shape[1]
    c.kern_kind = 0 if g.a_idx else _KIND.get(meta[g.kern][0], 0)
    c.acc, c.acc_stride, c.zero_init = acc.data_ptr(), acc.shape[1], 0
    c.m, c.k, c.n, c.a_stride = g.m, g.k, g.n, g.a_stride
    c.iterations = V
    if g.a_idx:
        if "compact" not in g.__dict__:
            g.compact = _compact(g.a_idx, g.b_idx) if V > 1 else None
        comp = g.compact
        if comp is not None:  # one gather table + a shift per iteration
            c.a_idx, c.b_idx = dptr(comp[0], "a_tab"), dptr(comp[1], "b_tab")
            c.a_shift = dptr(comp[2], "a_shift")
        else:
            c.a_idx = dptr(lambda: np.stack(g.a_idx), "a_idx")
            c.b_idx = dptr(lambda: np.stack(g.b_idx), "b_idx")
    else:
        c.a_base, c.k_base = dptr(g.a_base, "a_base"), dptr(g.k_base, "k_base")
        c.b_off = dptr(g.b_off, "b_off")
    if scatter is not None:
        dst, bases, off = scatter
        out = bufs[dst]
        c.out, c.out_stride = out.data_ptr(), out.shape[1]
        c.out_base = dptr(bases, "out_base")
        if off is not None:
            c.out_off = dptr(off, "out_off")
    err.zero_()
    c.error = err.data_ptr()
    _lib.check(lib.ts_run_conv_group(ctypes.byref(c), stream), "ts_run_conv_group")
    code, index, it = (int(v) for v in err.tolist())
    if code:  # backstop: _compile checks every index on the host first
        raise _annotate(OutOfBounds(g.src if code == 1 else g.kern, index),
                        g.paths[it] if 0 <= it < len(g.paths) else "body")
    if g.tmp is not None and g.tmp in bufs:  # materialise the last iteration's temporary
        o = torch.from_numpy(g.b_off.astype(np.int64)).to(dev)
        vals = kern[:, (g.k_base[-1] + o).clamp(min=0)]
        bufs[g.tmp][:, :len(g.b_off)] = torch.where(o >= 0, vals, torch.zeros_like(vals))


def run_program(p, inputs, extra_shapes=(), strict=False, lint_sink=None):
    """interp.run_program (interp.py:570-589) on the GPU, same signature."""
    return run_program_batch(p, [inputs], extra_shapes, strict, lint_sink)[0]


__all__ = ["run_program", "run_program_batch", "UnsupportedProgram", "Buffer", "BufferStore",
           "HARDWARE_SHAPES"]
