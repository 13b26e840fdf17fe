"""Pin the CPU oracle to the reference (tests/golden/, made by oracle/make_golden.py).

Every comparison here is bit-exact: the reference sums left to right in f32
(interp.py:1-7) and the oracle restates exactly that.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import interp_ref, layout_ref, pipelines_ref


@pytest.fixture(scope="module")
def G():
    return np.load(os.path.join(GOLDEN, "reference_golden.npz"))


@pytest.fixture(scope="module")
def J():
    with open(os.path.join(GOLDEN, "reference_golden.json")) as f:
        return json.load(f)


def same_bits(a, b):
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def test_splitmix_known_answers(J):
    # test_interp.py:88-92 pins the first three; the fixture has eight
    r = interp_ref.SplitMix64(0)
    got = [hex(r.next_u64()) for _ in range(8)]
    assert got == J["splitmix0_u64"]
    assert got[:3] == ["0xe220a8397b1dcdaf", "0x6e789e6aa1b965f4", "0x6c45d188009454f"]
    r = interp_ref.SplitMix64(12345)
    assert [r.uniform() for _ in range(8)] == J["splitmix12345_uniform"]


def test_rounding_matches_reference(G):
    x = G["round_in"]
    for fn, key in ((interp_ref.round_bf16, "round_bf16"), (interp_ref.round_f16, "round_f16")):
        got, want = fn(x), G[key]
        nan = np.isnan(want)
        assert np.array_equal(np.isnan(got), nan)
        assert got[~nan].tobytes() == want[~nan].tobytes(), key


def test_random_fill_matches_random_inputs(G):
    got = interp_ref.random_fill([("K", "f16", 8), ("I", "f16", 264), ("output", "f32", 256)], 7)
    assert same_bits(got["K"], G["rand_conv1d_k8_K"])
    assert same_bits(got["I"], G["rand_conv1d_k8_I"])


def _corpus_eval(name, K, I):
    """The corpus programs' source semantics, restated (corpus/*.sexp)."""
    cs = interp_ref.conv_statement
    if name == "conv1d_k8":
        return cs(I, K, 0, 8, 1, 256, np.zeros(256, np.float32))
    if name == "conv1d_k16":
        acc = np.zeros(256, np.float32)
        for rx in range(2):
            acc = cs(I, K[8 * rx:8 * rx + 8], 8 * rx, 8, 1, 256, acc)
        return acc
    if name == "conv2d_outer_ry":
        acc = np.zeros(256, np.float32)
        for ry in range(8):
            acc = cs(I, K[8 * ry:8 * ry + 8], 264 * ry, 8, 1, 256, acc)
        return acc
    if name == "downsample2_1d":
        return cs(I, K, 0, 8, 2, 256, np.zeros(256, np.float32))
    if name == "upsample2_1d":
        # out[2x + d] = Σ_u I[x + u] · K[2u + d]   (polyphase, p=2, l=12)
        o = np.arange(256)
        x, d = o // 2, o % 2
        u = np.arange(12)
        prods = (np.asarray(I, np.float32)[x[:, None] + u[None, :]]
                 * np.asarray(K, np.float32)[2 * u[None, :] + d[:, None]]).astype(np.float32)
        return (interp_ref.foldl_rows(prods) + np.float32(0)).astype(np.float32)
    raise KeyError(name)


@pytest.mark.parametrize("name", ["conv1d_k8", "conv1d_k16", "conv2d_outer_ry",
                                  "downsample2_1d", "upsample2_1d"])
def test_corpus_programs_bit_exact(G, J, name):
    assert J["corpus"][name]["lowered"]
    for seed in range(3):
        K = G[f"corpus_{name}_{seed}_K"]
        I = G[f"corpus_{name}_{seed}_I"]
        assert same_bits(_corpus_eval(name, K, I), G[f"corpus_{name}_{seed}_out"]), seed


def test_lanczos_tile_statement_bit_exact(G, J):
    # the Lanczos-3 2x statement lowers with (wmma-shape 32 28 8) to
    # PolyphaseShuffle + wmma_mma and is bit-exact with its source form
    assert J["lanczos_tile"]["lowered"]
    assert "PolyphaseShuffle" in J["lanczos_tile"]["intrinsics"]
    got = interp_ref.conv_statement(G["lanczos_tile_I"], G["lanczos_tile_K"], 0, 12, 2, 256)
    assert same_bits(got, G["lanczos_tile_out"])


def test_lanczos_tile_as_wmma_tiles(G):
    # the same statement through the oracle's wmma_mma / tile-gather restatement:
    # A = 32 windows x 28 (stride 16), B = 28 x 8 strided Toeplitz
    K, I = G["lanczos_tile_K"], G["lanczos_tile_I"]
    a = interp_ref.tile_gather(I, 0, 16, 32, 28)
    b = layout_ref.dense(K, 12, 8, s=2)
    out = interp_ref.wmma_mma(a, b.reshape(-1), np.zeros(256, np.float32), 32, 28, 8)
    # the Toeplitz zeros add exact zeros: same bits as the source form
    assert same_bits(out, G["lanczos_tile_out"])


def test_separable_lanczos_image_bit_exact(G):
    rows = (G["lz_rows_first"], G["lz_rows_w"])
    cols = (G["lz_cols_first"], G["lz_cols_w"])
    got = pipelines_ref.separable(G["img"], rows, cols)
    assert same_bits(got, G["lz_out"])


@pytest.mark.parametrize("taps", [9, 31])
def test_separable_gaussian_image_bit_exact(G, taps):
    img = G["img"]
    k = G[f"gauss{taps}_k"]
    H, W = img.shape
    got = pipelines_ref.separable(img, pipelines_ref.centred_axis(H, k),
                                  pipelines_ref.centred_axis(W, k))
    assert same_bits(got, G[f"gauss{taps}_out"])


def test_column_walk_bit_exact(G, J):
    cw = J["colwalk"]
    img = G["img"]
    first = cw["stride"] * np.arange(cw["n_out"])
    w = np.tile(G["colwalk_K"], (cw["n_out"], 1))
    got = pipelines_ref.axis_pass(img[:, cw["col"]:cw["col"] + 1], first, w, axis=-2)[:, 0]
    assert same_bits(got, G["colwalk_out"])


def test_layout_oracle_matches_reference(J):
    L = J["layout"]
    assert layout_ref.dense(np.array([5.0, 7.0, 9.0], np.float32), 3, 2).tolist() == L["toeplitz_3tap_k2"]
    assert layout_ref.dense(np.array([1.0, 1.0], np.float32), 2, 2, s=2).tolist() == L["strided_2tap_k2_s2"]
    assert layout_ref.dense(np.array([2.0, 3.0], np.float32), 1, 4, p=2).tolist() == L["polyphase_1tap_k4_p2"]
    assert layout_ref.shuffle_indices(3, 2, 1, 1, 0, 3) == L["shuffle_l3_k2"]
    for case in L["random"]:
        kern = np.array(case["kernel"], np.float32)
        m = layout_ref.dense(kern, case["l"], case["k"], case["s"], case["p"])
        assert m.tolist() == case["matrix"]
        assert layout_ref.shuffle_indices(case["l"], case["k"], case["s"], case["p"], case["base"],
                                          case["base"] + len(kern) + 2) == case["shuffle"]


def test_lanczos_weights_properties():
    first, w = pipelines_ref.lanczos3_weights(3840, 1920)
    assert w.shape == (1920, 12)
    assert list(first[:3]) == [-5, -3, -1]
    np.testing.assert_allclose(w.sum(1), 1.0, atol=1e-6)
    np.testing.assert_allclose(w[0], w[0][::-1], atol=1e-7)  # symmetric
    # known interior values (SURVEY appendix A probe)
    np.testing.assert_allclose(w[100, :6], [0.0037, 0.0151, -0.0340, -0.0666, 0.1355, 0.4464],
                               atol=1e-4)


def test_dct_oracle_pinned_to_reference_wmma_programs(G, J):
    """DCT-16 denoise: the oracle's four 16x16x16 products per tile are
    bit-identical to wmma_mma programs run by the reference interpreter in
    strict mode (oracle/make_golden.py: mm_program), and so is the whole
    denoise (hard, soft, threshold 0) of a 2x40x56 bf16 image."""
    img = G["dct_img"]
    assert J["dct"]["strict"] and J["dct"]["wmma_shape"] == [16, 16, 16]
    assert same_bits(pipelines_ref.dct_window_matrix(), G["dct_Dw"])
    assert same_bits(pipelines_ref.dct_coefficients(img), G["dct_coeffs"])
    thr = J["dct"]["threshold"]
    assert same_bits(pipelines_ref.dct_denoise(img, thr, "hard"), G["dct_out_hard"])
    assert same_bits(pipelines_ref.dct_denoise(img, thr, "soft"), G["dct_out_soft"])
    assert same_bits(pipelines_ref.dct_denoise(img, 0.0, "soft"), G["dct_out_zero"])


def test_dct_flip_mask():
    rng = np.random.default_rng(3)
    yy, xx = np.mgrid[0:96, 0:128]
    img = np.clip(0.5 + 0.4 * np.sin(xx / 17.0) * np.cos(yy / 23.0)
                  + rng.normal(0, 0.05, (1, 96, 128)), 0, 1).astype(np.float32)
    C = pipelines_ref.dct_coefficients(img)
    m0 = pipelines_ref.dct_flip_mask(img, 0.15, 0.0)
    m1 = pipelines_ref.dct_flip_mask(img, 0.15, 3e-3)
    assert m0.shape == img.shape and m0.sum() <= m1.sum()
    assert m1.any() and not m1.all()
    # a coefficient exactly at the threshold flags its tile's 16x16 footprint
    c = abs(float(C[0, 2, 3, 4, 5]))
    m = pipelines_ref.dct_flip_mask(img, c, 0.0)
    assert m[0, 8:24, 16:32].all()
