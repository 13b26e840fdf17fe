"""A minimal mirror of the reference IR (ir.py:54-209) and a reader for its
s-expression syntax (ir.py:714-802), restricted to the node types the GPU
executor consumes.

The executor is duck-typed: it accepts real ``tensorsel.ir`` objects (the
drop-in case) or these mirrors (same class names and fields), so it runs
where the reference package is not installed — e.g. on the GPU box.  This is
not a replacement for the reference parser/validator.
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field


@dataclass(frozen=True)
class VecType:
    kind: str
    lanes: int


@dataclass(frozen=True)
class Imm:
    kind: str
    value: float


@dataclass(frozen=True)
class Var:
    name: str


@dataclass(frozen=True)
class Load:
    buffer: str
    vtype: VecType
    index: object


@dataclass(frozen=True)
class Cast:
    vtype: VecType
    operand: object


@dataclass(frozen=True)
class Bop:
    op: str
    lhs: object
    rhs: object


@dataclass(frozen=True)
class Ramp:
    base: object
    stride: object
    steps: int


@dataclass(frozen=True)
class Broadcast:
    operand: object
    copies: int


@dataclass(frozen=True)
class VectorReduceAdd:
    result_lanes: int
    operand: object


@dataclass(frozen=True)
class Call:
    name: str
    args: tuple


@dataclass(frozen=True)
class Shuffle:
    source: object
    indices: tuple


@dataclass(frozen=True)
class Allocate:
    name: str
    kind: str
    length: int
    location: str


@dataclass(frozen=True)
class Store:
    buffer: str
    index: object
    value: object


@dataclass(frozen=True)
class Evaluate:
    value: object


@dataclass(frozen=True)
class For:
    var: str
    min: int
    extent: int
    body: tuple


@dataclass(frozen=True)
class Param:
    name: str
    kind: str
    length: int
    location: str = "mem"


@dataclass(frozen=True)
class ShapeDecl:
    target: str
    m: int
    k: int
    n: int


@dataclass(frozen=True)
class Program:
    params: tuple = ()
    body: tuple = ()
    shapes: tuple = field(default_factory=tuple)


_OPS = {"add": "+", "sub": "-", "mul": "*", "div": "/", "mod": "%"}
_TOKEN = re.compile(r"\(|\)|[^\s()]+")


def _tokens(text):
    return _TOKEN.findall(text)


def _read(tokens, pos):
    tok = tokens[pos]
    if tok == "(":
        out = []
        pos += 1
        while tokens[pos] != ")":
            item, pos = _read(tokens, pos)
            out.append(item)
        return out, pos + 1
    return tok, pos + 1


def _num(s):
    return float(s) if any(c in s for c in ".eE") and not s.lstrip("-").isdigit() else int(s)


def _vt(x):
    return VecType(x[0], int(x[1]))


def _expr(x):
    if not isinstance(x, list):
        raise ValueError(f"unexpected atom {x!r}")
    head = x[0]
    if head == "imm":
        v = _num(x[2])
        return Imm(x[1], float(v) if x[1] != "i32" else int(v))
    if head == "var":
        return Var(x[1])
    if head == "load":
        return Load(x[1], _vt(x[2]), _expr(x[3]))
    if head == "cast":
        return Cast(_vt(x[1]), _expr(x[2]))
    if head in _OPS:
        return Bop(_OPS[head], _expr(x[1]), _expr(x[2]))
    if head == "ramp":
        return Ramp(_expr(x[1]), _expr(x[2]), int(x[3]))
    if head == "broadcast":
        return Broadcast(_expr(x[1]), int(x[2]))
    if head == "vector-reduce-add":
        return VectorReduceAdd(int(x[1]), _expr(x[2]))
    if head == "call":
        return Call(x[1], tuple(_expr(a) for a in x[2:]))
    if head == "shuffle":
        return Shuffle(_expr(x[1]), tuple(int(i) for i in x[2]))
    raise ValueError(f"unsupported expression {head!r}")


def _stmt(x):
    head = x[0]
    if head == "allocate":
        return Allocate(x[1], x[2], int(x[3]), x[4])
    if head == "store":
        return Store(x[1], _expr(x[2]), _expr(x[3]))
    if head == "evaluate":
        return Evaluate(_expr(x[1]))
    if head == "for":
        return For(x[1], int(x[2]), int(x[3]), tuple(_stmt(s) for s in x[4:]))
    raise ValueError(f"unsupported statement {head!r}")


def parse_program(text: str) -> Program:
    """Read the reference's program syntax (ir.py:714-802, the subset used
    by the conv corpus and lowered conv programs)."""
    toks = _tokens(text)
    pos = 0
    params, body, shapes = [], [], []
    while pos < len(toks):
        form, pos = _read(toks, pos)
        head = form[0]
        if head == "param":
            params.append(Param(form[1], form[2], int(form[3]), form[4] if len(form) > 4 else "mem"))
        elif head == "wmma-shape":
            shapes.append(ShapeDecl("wmma", int(form[1]), int(form[2]), int(form[3])))
        elif head == "amx-shape":
            shapes.append(ShapeDecl("amx", int(form[1]), int(form[2]), int(form[3])))
        else:
            body.append(_stmt(form))
    return Program(tuple(params), tuple(body), tuple(shapes))
