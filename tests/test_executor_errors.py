"""The executor's error surface against the reference interpreter's
(interp.py:32-55, 156-159, 251-269, 537-555, 591-619).

CPU tests: every conv-family index is affine in the loop variables, so the
executor checks bounds while compiling, on the host, and raises the
reference's exception with the reference's statement path.  Where the
reference package is installed (baseline/_ref, git-ignored), the same bad
programs are run through interp.run_program and the messages compared.
GPU test: colliding store lanes are last-lane-wins and reported to
lint_sink, like interp._scatter."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from paper_2512_02371_b200 import errors, executor, irlite

REF = os.path.join(ROOT, "baseline", "_ref")
HAVE_REF = os.path.isdir(os.path.join(REF, "tensorsel"))

R = "(ramp (imm i32 0) (imm i32 1) {n})"


def lowered_conv(a_base="(imm i32 0)", in_len=264, acc_len=256, k_base="(imm i32 0)", k_len=8,
                 a_stride=8, loop=None):
    """A lowered 32x16x8 conv statement (the conv1d_k8 corpus shape) with
    adjustable bases/lengths; `loop` wraps the mma in a For."""
    mma = (f"(store conv {R.format(n=256)} (call wmma_mma "
           f"(call wmma_load_a (var I) {a_base} (imm i32 {a_stride}) (imm i32 32) (imm i32 16)) "
           f"(call wmma_load_b (var sw) (imm i32 0) (imm i32 8) (imm i32 16) (imm i32 8)) "
           f"(load conv (f32 256) {R.format(n=256)})))")
    body = [
        f"(param K f16 {k_len} mem)", f"(param I f16 {in_len} mem)", "(param out f32 256 mem)",
        "(allocate sw f16 128 mem)", f"(allocate conv f32 {acc_len} wmma)",
        f"(store conv {R.format(n=256)} (call wmma_zero (imm i32 32) (imm i32 8)))",
        f"(store sw {R.format(n=128)} (call ConvolutionShuffle (var K) {k_base} (imm i32 16) (imm i32 8)))",
        mma if loop is None else f"(for v 0 {loop} {mma})",
        f"(evaluate (call wmma_store (var out) (imm i32 0) (imm i32 8) (imm i32 8) "
        f"(load conv (f32 256) {R.format(n=256)})))",
    ]
    return "\n".join(body)


def _ours(text):
    try:
        executor._compile(irlite.parse_program(text), (), False)
    except errors.EvalError as e:
        return type(e).__name__, str(e), getattr(e, "stmt_path", None)
    return None


def _reference(text):
    code = r"""
import json, sys
import numpy as np
from tensorsel import interp, ir
p = ir.parse_program(sys.stdin.read())
ins = interp.random_inputs(p, 0)
try:
    interp.run_program(p, ins)
    print(json.dumps(None))
except interp.EvalError as e:
    print(json.dumps([type(e).__name__, str(e), getattr(e, "stmt_path", None)]))
"""
    env = {**os.environ, "PYTHONPATH": REF, "PYTHONDONTWRITEBYTECODE": "1"}
    r = subprocess.run([sys.executable, "-c", code], input=text, capture_output=True, text=True,
                       env=env, check=True)
    import json
    v = json.loads(r.stdout)
    return tuple(v) if v else None


BAD = {
    # wmma_load_a base of -1: ADVICE round 1 (an index of -1 used to encode as "no error")
    "a_base_minus_1": (lowered_conv(a_base="(imm i32 -1)"), "OutOfBounds", "body[4]"),
    "a_past_end": (lowered_conv(in_len=260), "OutOfBounds", "body[4]"),
    "kernel_window": (lowered_conv(k_base="(imm i32 1)"), "OutOfBounds", "body[3]"),
    "short_accumulator": (lowered_conv(acc_len=200), "OutOfBounds", "body[2]"),
    "loop_walks_off": (lowered_conv(a_base="(mul (var v) (imm i32 8))", loop=4),
                       "OutOfBounds", "body[4][0]"),
    "divide_by_zero": (lowered_conv(a_base="(div (imm i32 8) (imm i32 0))"), "DivideByZero",
                       "body[4]"),
    "i32_overflow": (lowered_conv(a_base="(mul (imm i32 65536) (imm i32 65536))"), "I32Overflow",
                     "body[4]"),
}


@pytest.mark.parametrize("name", sorted(BAD))
def test_errors_match_reference_classes_and_paths(name):
    text, cls, path = BAD[name]
    got = _ours(text)
    assert got is not None, name
    assert got[0] == cls and got[2] == path, got
    assert got[1].startswith(path + ": "), got
    if HAVE_REF:
        ref = _reference(text)
        assert ref is not None and ref[0] == cls and ref[2] == path, ref
        assert got[1] == ref[1], (got, ref)


def test_good_program_compiles():
    assert _ours(lowered_conv()) is None
    assert _ours(lowered_conv(a_base="(mul (var v) (imm i32 0))", loop=8)) is None


def test_euclidean_index_arithmetic():
    env = {"v": -7}
    e = irlite.parse_program(
        f"(param A f32 4 mem)\n(store A {R.format(n=4)} (broadcast (imm f32 0.0) 4))").body[0]
    assert e is not None
    for op, want in (("/", -4), ("%", 1)):
        b = irlite.Bop(op, irlite.Var("v"), irlite.Imm("i32", 2))
        assert executor._eval_int(b, env) == want  # interp.py:262-264: Euclidean


def test_non_f32_cast_in_source_form_is_rejected():
    text = ("(param K bf16 3 mem)\n(param I bf16 10 mem)\n(param out f32 8 mem)\n"
            "(allocate conv f32 8 wmma)\n"
            f"(store conv {R.format(n=8)} (add (vector-reduce-add 8 (mul "
            "(cast (bf16 24) (load I (bf16 24) (ramp (ramp (imm i32 0) (imm i32 1) 3) "
            "(broadcast (imm i32 1) 3) 8))) "
            "(broadcast (cast (f32 3) (load K (bf16 3) (ramp (imm i32 0) (imm i32 1) 3))) 8))) "
            f"(load conv (f32 8) {R.format(n=8)})))")
    with pytest.raises(executor.UnsupportedProgram):
        executor._compile(irlite.parse_program(text), (), False)


@pytest.mark.skipif(not HAVE_REF, reason="reference not installed in baseline/_ref")
def test_exception_classes_interoperate_with_the_reference():
    code = ("import tensorsel.interp as I, tensorsel.layout as L\n"
            "from paper_2512_02371_b200 import errors as E, executor as X\n"
            "assert issubclass(E.OutOfBounds, I.OutOfBounds) and issubclass(E.EvalError, I.EvalError)\n"
            "assert issubclass(E.DivideByZero, I.DivideByZero)\n"
            "assert issubclass(E.ShapeUnregistered, I.ShapeUnregistered)\n"
            "assert issubclass(E.PhaseMismatch, L.PhaseMismatch)\n"
            "assert X.Buffer is I.Buffer and X.BufferStore is I.BufferStore\n"
            "try:\n    raise E.OutOfBounds('I', 3)\nexcept I.OutOfBounds as e:\n"
            "    assert (e.buffer, e.index) == ('I', 3)\n"
            "print('ok')\n")
    env = {**os.environ, "PYTHONPATH": REF + os.pathsep + ROOT, "PYTHONDONTWRITEBYTECODE": "1"}
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr


COLLIDE = "\n".join([
    "(param K f16 8 mem)", "(param I f16 264 mem)", "(param out f32 16 mem)",
    "(allocate sw f16 128 mem)", "(allocate conv f32 256 wmma)",
    f"(store conv {R.format(n=256)} (call wmma_zero (imm i32 32) (imm i32 8)))",
    f"(store sw {R.format(n=128)} (call ConvolutionShuffle (var K) (imm i32 0) (imm i32 16) (imm i32 8)))",
    f"(store conv {R.format(n=256)} (call wmma_mma "
    "(call wmma_load_a (var I) (imm i32 0) (imm i32 8) (imm i32 32) (imm i32 16)) "
    "(call wmma_load_b (var sw) (imm i32 0) (imm i32 8) (imm i32 16) (imm i32 8)) "
    f"(load conv (f32 256) {R.format(n=256)})))",
    # stride 0: all 32 rows land on out[0..8): rows collide, the last row wins
    f"(evaluate (call wmma_store (var out) (imm i32 0) (imm i32 0) (imm i32 8) "
    f"(load conv (f32 256) {R.format(n=256)})))",
])


@pytest.mark.gpu
def test_colliding_store_lanes_last_wins_with_lint():
    from oracle import interp_ref
    p = irlite.parse_program(COLLIDE)
    ins = interp_ref.random_fill([("K", "f16", 8), ("I", "f16", 264), ("out", "f32", 16)], 5)
    lints = []
    st = executor.run_program(p, ins, lint_sink=lints)
    conv = st["conv"].data.reshape(32, 8)
    assert np.array_equal(st["out"].data[:8].view(np.uint32), conv[31].view(np.uint32))
    assert np.all(st["out"].data[8:] == ins["out"][8:])
    assert lints == ["store into 'out' has colliding lanes (last wins)"]
