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
