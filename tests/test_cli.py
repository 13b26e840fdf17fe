"""`python -m paper_2512_02371_b200 run` — the reference CLI's `run`
(cli.py:80-111) on the GPU executor.  CPU: the seeded fills against the
reference's known answers and golden inputs, usage/parse exit codes.  GPU:
outputs bit-identical to the reference's interp.run_program."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2512_02371_b200 import cli, fills, irlite, wire

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "reference_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def G():
    return np.load(os.path.join(GOLDEN, "reference_golden.npz"))


def test_splitmix_known_answers(golden):
    rng = fills.SplitMix64(0)
    want = golden["splitmix0_u64"]
    assert [hex(rng.next_u64()) for _ in range(len(want))] == want
    rng = fills.SplitMix64(12345)
    got = [rng.uniform() for _ in range(len(golden["splitmix12345_uniform"]))]
    assert got == golden["splitmix12345_uniform"]


@pytest.mark.parametrize("name", ["conv1d_k8", "conv1d_k16", "conv2d_outer_ry",
                                  "downsample2_1d", "upsample2_1d"])
def test_seeded_fills_match_reference_inputs(golden, G, name):
    prog = irlite.parse_program(golden["programs"][name]["lowered"])
    for seed in (0, 1, 2):
        got = fills.random_inputs(prog, seed)
        assert got["K"].tobytes() == G[f"corpus_{name}_{seed}_K"].tobytes()
        assert got["I"].tobytes() == G[f"corpus_{name}_{seed}_I"].tobytes()


def test_usage_and_parse_errors(tmp_path):
    assert cli.main(["run", str(tmp_path / "missing.sexp")]) == 2
    bad = tmp_path / "bad.sexp"
    bad.write_text("(param I f16 8) (store out (")
    assert cli.main(["run", str(bad)]) == 2
    assert cli.main(["frobnicate"]) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["conv1d_k16", "downsample2_1d", "upsample2_1d"])
def test_cli_run_matches_reference_outputs(golden, G, name, tmp_path):
    src = tmp_path / f"{name}.sexp"
    src.write_text(golden["programs"][name]["lowered"])
    out = tmp_path / "out"
    r = subprocess.run([sys.executable, "-m", "paper_2512_02371_b200", "run", str(src),
                        "--seed", "1", "--output", str(out), "--json"],
                       cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    summary = json.loads(r.stdout)["buffers"]
    assert summary["output"] == {"kind": "f32", "length": 256}
    got = wire.load_buffers(out)["output"][2]
    assert got.tobytes() == G[f"corpus_{name}_1_out"].tobytes()
    # the written directory round-trips as --inputs
    out2 = tmp_path / "out2"
    assert cli.main(["run", str(src), "--inputs", str(out), "--output", str(out2)]) == 0
    assert (out2 / "manifest.json").exists()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["conv1d_k8", "conv1d_k16", "conv2d_outer_ry",
                                  "downsample2_1d", "upsample2_1d"])
@pytest.mark.parametrize("form", ["source", "lowered"])
def test_cli_difftest_gpu_vs_reference_interpreter(golden, name, form, tmp_path):
    """`difftest` (the reference's cli.py:131-183, with the GPU executor and
    the reference interpreter as the two sides): bitwise over seeded fills."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "tensorsel")):
        pytest.skip("reference interpreter not installed under baseline/_ref")
    src = tmp_path / f"{name}.sexp"
    src.write_text(golden["programs"][name][form])
    r = subprocess.run([sys.executable, "-m", "paper_2512_02371_b200", "difftest", str(src),
                        "--trials", "8", "--seed", "3", "--json"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    rep = json.loads(r.stdout)
    assert rep["divergence"] is None and rep["seeds"] == list(range(3, 11))


def _lanczos_stream_program(n):
    """An image-scale generated program: the Lanczos-3 2x conv statement
    (12 taps, stride 2; the golden `lanczos_tile` statement) inside a For loop
    over `n` consecutive 256-output windows of one long row."""
    body = ("(store conv (ramp (imm i32 0) (imm i32 1) 256) (broadcast (imm f32 0.0) 256)) "
            "(store conv (ramp (imm i32 0) (imm i32 1) 256) (add (vector-reduce-add 256 "
            "(mul (cast (f32 3072) (load I (f16 3072) (ramp (ramp (mul (imm i32 512) (var t)) "
            "(imm i32 1) 12) (broadcast (imm i32 2) 12) 256))) (broadcast (cast (f32 12) "
            "(load K (f16 12) (ramp (imm i32 0) (imm i32 1) 12))) 256))) (load conv (f32 256) "
            "(ramp (imm i32 0) (imm i32 1) 256)))) "
            "(store output (ramp (mul (imm i32 256) (var t)) (imm i32 1) 256) "
            "(load conv (f32 256) (ramp (imm i32 0) (imm i32 1) 256)))")
    return (f"(param K f16 12 mem)\n(param I f16 {512 * n + 12} mem)\n"
            f"(param output f32 {256 * n} mem)\n(wmma-shape 32 28 8)\n"
            f"(allocate conv f32 256 wmma)\n(for t 0 {n} {body})\n")


@pytest.mark.gpu
def test_cli_difftest_image_scale_generated_program(tmp_path):
    """SURVEY §8(f)1's gate at image scale: 512 Lanczos windows (131072
    outputs) per trial, GPU executor vs the reference interpreter, bitwise."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "tensorsel")):
        pytest.skip("reference interpreter not installed under baseline/_ref")
    src = tmp_path / "lanczos_stream.sexp"
    src.write_text(_lanczos_stream_program(512))
    r = subprocess.run([sys.executable, "-m", "paper_2512_02371_b200", "difftest", str(src),
                        "--trials", "2", "--json"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert json.loads(r.stdout)["divergence"] is None
