"""GPU run_program backend for conv-family programs.

CPU: the program reader and the compiled statement groups.  GPU: every
corpus program (source form, lowered, lowered with shuffle intrinsics) and
the Lanczos-3 tile program run through executor.run_program_batch over the
reference's seeds and must reproduce the reference's outputs BIT-EXACTLY
(tests/golden/, produced by interp.run_program itself)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2512_02371_b200 import executor, irlite


@pytest.fixture(scope="module")
def programs():
    with open(os.path.join(GOLDEN, "reference_golden.json")) as f:
        return json.load(f)["programs"]


@pytest.fixture(scope="module")
def G():
    return np.load(os.path.join(GOLDEN, "reference_golden.npz"))


def _groups(plan):
    return [(len(o[2].a_base), o[2].m, o[2].k, o[2].n) for o in plan.ops if o[0] == "group"]


def test_reader_and_groups(programs):
    want = {"conv1d_k8": (1, 32, 16, 8), "conv1d_k16": (2, 32, 16, 8),
            "conv2d_outer_ry": (8, 32, 16, 8), "downsample2_1d": (1, 32, 24, 8),
            "upsample2_1d": (1, 32, 16, 8), "lanczos_tile": (1, 32, 28, 8)}
    for name, forms in programs.items():
        for form in ("lowered", "lowered_shuffle_intrinsics"):
            plan = executor._compile(irlite.parse_program(forms[form]), (), False)
            assert _groups(plan) == [want[name]], (name, form)
        plan = executor._compile(irlite.parse_program(forms["source"]), (), False)
        assert len(_groups(plan)) == 1


def test_strict_mode_rejects_declared_shapes(programs):
    p = irlite.parse_program(programs["downsample2_1d"]["lowered"])
    executor._compile(p, (), False)
    with pytest.raises(executor.ShapeUnregistered):
        executor._compile(p, (), True)


def test_unsupported_statements_fail_loudly():
    p = irlite.parse_program("(param A f32 4 mem)\n(store A (ramp (imm i32 0) (imm i32 1) 4) "
                             "(add (load A (f32 4) (ramp (imm i32 0) (imm i32 1) 4)) "
                             "(load A (f32 4) (ramp (imm i32 0) (imm i32 1) 4))))")
    with pytest.raises(executor.UnsupportedProgram):
        executor._compile(p, (), False)


def test_accepts_reference_ir_objects(programs):
    # duck typing: the real tensorsel.ir classes compile to the same plan
    tensorsel_ir = pytest.importorskip("tensorsel.ir") if _has_ref() else pytest.skip("no reference")
    for name, forms in programs.items():
        a = executor._compile(tensorsel_ir.parse_program(forms["lowered"]), (), False)
        b = executor._compile(irlite.parse_program(forms["lowered"]), (), False)
        assert _groups(a) == _groups(b)


def _has_ref():
    import sys
    for cand in ("/root/reference/pkg/src", os.path.join(os.path.dirname(GOLDEN), "..", "baseline", "_ref")):
        if os.path.isdir(os.path.join(cand, "tensorsel")):
            if cand not in sys.path:
                sys.path.append(cand)
            return True
    return False


def _inputs(G, name, seed):
    if name == "lanczos_tile":
        return {"K": G["lanczos_tile_K"], "I": G["lanczos_tile_I"],
                "output": np.zeros(256, np.float32)}
    return {"K": G[f"corpus_{name}_{seed}_K"], "I": G[f"corpus_{name}_{seed}_I"],
            "output": np.zeros(256, np.float32)}


def _want(G, name, seed):
    return G["lanczos_tile_out"] if name == "lanczos_tile" else G[f"corpus_{name}_{seed}_out"]


@pytest.mark.gpu
@pytest.mark.parametrize("form", ["source", "lowered", "lowered_shuffle_intrinsics"])
def test_gpu_run_program_bit_exact(programs, G, form):
    for name, forms in programs.items():
        p = irlite.parse_program(forms[form])
        seeds = [0] if name == "lanczos_tile" else [0, 1, 2]
        stores = executor.run_program_batch(p, [_inputs(G, name, s) for s in seeds])
        for s, st in zip(seeds, stores):
            got = st["output"].data
            assert got.dtype == np.float32
            assert got.tobytes() == _want(G, name, s).tobytes(), (name, form, s)


@pytest.mark.gpu
def test_gpu_run_program_single_and_errors(programs, G):
    p = irlite.parse_program(programs["conv1d_k16"]["lowered"])
    st = executor.run_program(p, _inputs(G, "conv1d_k16", 1))
    assert st["output"].data.tobytes() == _want(G, "conv1d_k16", 1).tobytes()
    assert set(st) >= {"K", "I", "output", "conv", "swizzle0"}
    bad = dict(_inputs(G, "conv1d_k16", 1))
    bad["I"] = bad["I"][:100]
    with pytest.raises(executor.EvalError):
        executor.run_program(p, bad)


@pytest.mark.gpu
def test_gpu_batched_difftest_many_seeds(programs):
    # the reference's difftest (cli.py:161-183) in one launch per group:
    # source vs lowered over 200 seeds, bitwise
    from oracle import interp_ref
    src = irlite.parse_program(programs["conv2d_outer_ry"]["source"])
    low = irlite.parse_program(programs["conv2d_outer_ry"]["lowered"])
    params = [(prm.name, prm.kind, prm.length) for prm in src.params]
    ins = [interp_ref.random_fill(params, seed) for seed in range(200)]
    a = executor.run_program_batch(src, ins)
    b = executor.run_program_batch(low, ins)
    for x, y in zip(a, b):
        assert x["output"].data.tobytes() == y["output"].data.tobytes()


def test_for_loop_of_independent_conv_windows_fuses_to_one_launch():
    """A For loop whose body is fill / conv / copy-out (the image-scale
    generated program of tests/test_cli.py) compiles to ONE scatter op with
    every iteration, instead of 3 ops per iteration; its gathers compact to
    one table plus a shift per iteration."""
    from test_cli import _lanczos_stream_program
    plan = executor._compile(irlite.parse_program(_lanczos_stream_program(64)), (), False)
    kinds = [o[0] for o in plan.ops]
    assert kinds.count("scatter") == 1 and "copy" not in kinds, kinds
    op = next(o for o in plan.ops if o[0] == "scatter")
    g = op[2]
    assert len(g.a_base) == 64 and op[4] == [256 * t for t in range(64)]
    table, btable, shifts = executor._compact(g.a_idx, g.b_idx)
    assert table.shape == (256, 12) and list(shifts[:3]) == [0, 512, 1024]


def mm_program_text(n_tiles, fixed_left):
    """The DCT fixture programs of oracle/make_golden.py (mm_program): C_t =
    A_t · B_t for n_tiles 16x16 tiles, wmma_load_a / wmma_load_b of plain
    buffers (the wmma-mma rule's matmul form, rules.py:904-1008)."""
    R = "(ramp (imm i32 0) (imm i32 1) 256)"
    base = "(mul (var t) (imm i32 256))"
    a_len, b_len = (256, 256 * n_tiles) if fixed_left else (256 * n_tiles, 256)
    a_base, b_base = ("(imm i32 0)", base) if fixed_left else (base, "(imm i32 0)")
    return (f"(param A f32 {a_len} mem)\n(param B f32 {b_len} mem)\n"
            f"(param O f32 {256 * n_tiles} mem)\n(wmma-shape 16 16 16)\n"
            f"(allocate acc f32 256 wmma)\n"
            f"(for t 0 {n_tiles}\n"
            f" (store acc {R} (call wmma_zero (imm i32 16) (imm i32 16)))\n"
            f" (store acc {R} (call wmma_mma (call wmma_load_a (var A) {a_base} (imm i32 16) "
            f"(imm i32 16) (imm i32 16)) (call wmma_load_b (var B) {b_base} (imm i32 16) "
            f"(imm i32 16) (imm i32 16)) (load acc (f32 256) {R})))\n"
            f" (evaluate (call wmma_store (var O) {base} (imm i32 16) (imm i32 16) "
            f"(load acc (f32 256) {R}))))\n")


def test_plain_buffer_matmul_compiles_to_one_scatter():
    plan = executor._compile(irlite.parse_program(mm_program_text(12, True)), (), True)
    kinds = [o[0] for o in plan.ops]
    assert kinds.count("scatter") == 1, kinds
    g = next(o for o in plan.ops if o[0] == "scatter")[2]
    assert len(g.a_base) == 12 and g.k_base[:3] == [0, 256, 512] and g.tmp is None


@pytest.mark.gpu
def test_dct_fixture_programs_run_bit_exactly_on_the_gpu(G):
    """The four 16x16x16 products per tile of the DCT fixture, run as the
    same wmma programs the reference ran (oracle/make_golden.py) through the
    GPU executor: the forward coefficients equal the reference's bit for
    bit."""
    Dw = G["dct_Dw"]
    want = G["dct_coeffs"]
    P, ty, tx = want.shape[:3]
    n = P * ty * tx
    import oracle.pipelines_ref as R
    T = R.dct_tiles(G["dct_img"]).reshape(n, 16, 16)
    left = irlite.parse_program(mm_program_text(n, True))
    right = irlite.parse_program(mm_program_text(n, False))
    P1 = executor.run_program(left, {"A": Dw.reshape(-1), "B": T.reshape(-1),
                                     "O": np.zeros(256 * n, np.float32)}, strict=True)["O"].data
    C = executor.run_program(right, {"A": P1, "B": np.ascontiguousarray(Dw.T).reshape(-1),
                                     "O": np.zeros(256 * n, np.float32)}, strict=True)["O"].data
    assert C.tobytes() == want.astype(np.float32).tobytes()
