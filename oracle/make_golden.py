"""Generate tests/golden/ fixtures by running the *reference* implementation.

TEST INFRASTRUCTURE ONLY.  Run in the development container, where the
reference package is importable (read-only) from /root/reference/pkg/src or
from baseline/_ref:

    python oracle/make_golden.py

Everything written here comes out of the reference's own code paths
(layout.*, interp.round_*, interp.SplitMix64 / random_inputs,
interp.run_program on corpus programs and on programs generated with the
corpus template tools/make_corpus.py:142-150, selector.select_program for
the lowered forms).  The oracle is then checked against these fixtures in
tests/test_oracle_golden.py; nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for cand in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
    if os.path.isdir(os.path.join(cand, "tensorsel")):
        sys.path.insert(0, cand)
        break

from tensorsel import interp, ir, layout, selector  # noqa: E402
from tensorsel.ir import (Bop, Broadcast, Cast, Imm, Load, Param, Program, Ramp,  # noqa: E402
                          ShapeDecl, Store, Allocate, VecType, VectorReduceAdd)

sys.path.insert(0, ROOT)
from oracle import pipelines_ref  # noqa: E402  (weights only)

OUT = os.path.join(ROOT, "tests", "golden")
CORPUS = "/root/reference/pkg/corpus"


def i32(v):
    return Imm("i32", v)


def f32x(n):
    return VecType("f32", n)


def flat(n):
    return Ramp(i32(0), i32(1), n)


def conv_program(kind, taps, n_out, in_len, stride=1, elem_stride=1, base=0, shapes=()):
    """The corpus conv template (make_corpus.conv_update / conv_program,
    tools/make_corpus.py:142-157) generalised to n_out outputs, input kind,
    output stride and element stride (elem_stride=W walks an image column)."""
    lanes = n_out * taps
    i_idx = Ramp(Ramp(i32(base), i32(elem_stride), taps),
                 Broadcast(i32(stride * elem_stride), taps), n_out)
    i_op = Cast(f32x(lanes), Load("I", VecType(kind, lanes), i_idx))
    k_load = Load("K", VecType(kind, taps), Ramp(i32(0), i32(1), taps))
    k_op = Broadcast(Cast(f32x(taps), k_load), n_out)
    acc = Load("conv", f32x(n_out), flat(n_out))
    update = Store("conv", flat(n_out), Bop("+", VectorReduceAdd(n_out, Bop("*", i_op, k_op)), acc))
    body = (Allocate("conv", "f32", n_out, "wmma"),
            Store("conv", flat(n_out), Broadcast(Imm("f32", 0.0), n_out)),
            update,
            Store("output", flat(n_out), Load("conv", f32x(n_out), flat(n_out))))
    params = (Param("K", kind, taps), Param("I", kind, in_len), Param("output", "f32", n_out))
    return Program(params, body, tuple(shapes))


def run(prog, K, I):
    st = interp.run_program(prog, {"K": np.asarray(K, np.float32), "I": np.asarray(I, np.float32),
                                   "output": np.zeros(prog.params[2].length, np.float32)})
    return st["output"].data.copy()


def layout_fixtures(rng):
    out = {
        "toeplitz_3tap_k2": layout.toeplitz_matrix(np.array([5.0, 7.0, 9.0], np.float32), 2).tolist(),
        "strided_2tap_k2_s2": layout.strided_toeplitz(np.array([1.0, 1.0], np.float32), 2, 2).tolist(),
        "polyphase_1tap_k4_p2": layout.polyphase_toeplitz(np.array([2.0, 3.0], np.float32), 4, 2).tolist(),
        "shuffle_l3_k2": layout.shuffle_indices_for(layout.ToeplitzSpec(l=3, k=2), 0, 3),
        "kway_2_4_2": layout.kway_interleave_indices(2, 4, 2),
        "random": [],
    }
    for _ in range(40):
        s = int(rng.choice([1, 2, 3]))
        p = int(rng.choice([1, 2, 4])) if s == 1 else 1
        l = int(rng.integers(1, 17))
        k = int(rng.integers(1, 33))
        if p > 1:
            k = max(p, (k // p) * p)
        spec = layout.ToeplitzSpec(l=l, k=k, s=s, p=p)
        kern = rng.uniform(-1, 1, spec.kernel_length).astype(np.float32)
        base = int(rng.integers(0, 3))
        out["random"].append({
            "l": l, "k": k, "s": s, "p": p, "kernel": kern.tolist(),
            "matrix": layout.matrix_for(kern, spec).tolist(),
            "base": base,
            "shuffle": layout.shuffle_indices_for(spec, base, base + spec.kernel_length + 2),
        })
    return out


def mm_program(n_tiles, fixed_left):
    """C_t = A_t · B_t for n_tiles 16x16 tiles as a For loop of
    wmma_load_a / wmma_load_b / wmma_mma / wmma_store (the lowered-conv
    intrinsics, interp.py:419-486).  fixed_left: A is one 16x16 matrix and B
    varies per tile, else A varies and B is fixed."""
    R = "(ramp (imm i32 0) (imm i32 1) 256)"
    base = "(mul (var t) (imm i32 256))"
    a_len, b_len = (256, 256 * n_tiles) if fixed_left else (256 * n_tiles, 256)
    a_base, b_base = ("(imm i32 0)", base) if fixed_left else (base, "(imm i32 0)")
    return ir.parse_program(f"""(param A f32 {a_len} mem)
(param B f32 {b_len} mem)
(param O f32 {256 * n_tiles} mem)
(wmma-shape 16 16 16)
(allocate acc f32 256 wmma)
(for t 0 {n_tiles}
 (store acc {R} (call wmma_zero (imm i32 16) (imm i32 16)))
 (store acc {R} (call wmma_mma (call wmma_load_a (var A) {a_base} (imm i32 16) (imm i32 16) (imm i32 16)) (call wmma_load_b (var B) {b_base} (imm i32 16) (imm i32 16) (imm i32 16)) (load acc (f32 256) {R})))
 (evaluate (call wmma_store (var O) {base} (imm i32 16) (imm i32 16) (load acc (f32 256) {R}))))
""")


def ref_mm(A, B, fixed_left):
    """Run mm_program through interp.run_program (strict hardware shapes)."""
    tiles = B if fixed_left else A
    n = tiles.shape[0]
    prog = mm_program(n, fixed_left)
    st = interp.run_program(prog, {"A": np.ascontiguousarray(A, np.float32).reshape(-1),
                                   "B": np.ascontiguousarray(B, np.float32).reshape(-1),
                                   "O": np.zeros(256 * n, np.float32)}, strict=True)
    return st["O"].data.reshape(n, 16, 16).copy()


def dct_fixtures(arrays, kats, rng):
    P, H, W = 2, 40, 56
    yy, xx = np.mgrid[0:H, 0:W]
    clean = 0.5 + 0.4 * np.sin(xx / 7.0) * np.cos(yy / 5.0)
    img = interp.round_bf16(np.clip(clean + rng.normal(0, 0.05, (P, H, W)), 0, 1).astype(np.float32))
    arrays["dct_img"] = img
    n, h = 16, 8
    k = np.arange(n)[:, None]
    m = np.arange(n)[None, :]
    D = np.cos(np.pi * (2 * m + 1) * k / (2 * n)) * np.sqrt(2.0 / n)
    D[0, :] = np.sqrt(1.0 / n)
    w = np.sin(np.pi * (np.arange(n) + 0.5) / n)
    Dw = (D * w[None, :]).astype(np.float32)
    arrays["dct_Dw"] = Dw
    xp = np.pad(img, ((0, 0), (h, h), (h, h)), mode="edge")
    ty, tx = H // h + 1, W // h + 1
    T = np.stack([xp[p, h * i:h * i + n, h * j:h * j + n]
                  for p in range(P) for i in range(ty) for j in range(tx)])
    C = ref_mm(ref_mm(Dw, T, True), np.ascontiguousarray(Dw.T), False)
    arrays["dct_coeffs"] = C.reshape(P, ty, tx, n, n)
    thr = 0.15
    for mode in ("hard", "soft", "zero"):
        Cc = C.copy()
        if mode == "hard":
            Cc = np.where(np.abs(C) < np.float32(thr), np.float32(0), C).astype(np.float32)
        elif mode == "soft":
            Cc = (np.sign(C) * np.maximum(np.abs(C) - np.float32(thr), np.float32(0))).astype(np.float32)
        Cc[:, 0, 0] = C[:, 0, 0]
        Rt = ref_mm(ref_mm(np.ascontiguousarray(Dw.T), Cc, True), Dw, False).reshape(P, ty, tx, n, n)
        out = np.zeros((P, H + 2 * h, W + 2 * h), np.float32)
        for py in range(2):  # each pixel: ((0 + t00) + t01) + t10) + t11, phase order
            for px in range(2):
                for i in range(py, ty, 2):
                    for j in range(px, tx, 2):
                        out[:, h * i:h * i + n, h * j:h * j + n] += Rt[:, i, j]
        arrays[f"dct_out_{mode}"] = out[:, h:h + H, h:h + W].copy()
    kats["dct"] = {"threshold": thr, "tiles_per_plane": [ty, tx], "planes": P,
                   "wmma_shape": [16, 16, 16], "strict": True}


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(0x251202371)
    arrays = {}

    # -- generator and rounding KATs (interp.py:62-115)
    sm = interp.SplitMix64(0)
    kats = {"splitmix0_u64": [hex(sm.next_u64()) for _ in range(8)]}
    sm = interp.SplitMix64(12345)
    kats["splitmix12345_uniform"] = [sm.uniform() for _ in range(8)]
    special = np.array([0.0, -0.0, 1.0, -1.0, 65504.0, 65520.0, 1e-8, 3.0e38, np.inf, -np.inf,
                        np.nan, 1.00390625, 1.01171875, -2.5e-5], np.float32)
    vals = np.concatenate([special, rng.standard_normal(500).astype(np.float32) * 10.0 ** rng.integers(-6, 6, 500)])
    arrays["round_in"] = vals.astype(np.float32)
    arrays["round_bf16"] = interp.round_bf16(vals)
    arrays["round_f16"] = interp.round_f16(vals)

    # -- random_inputs on a corpus program (interp.py:622-634)
    p = ir.parse_program(open(os.path.join(CORPUS, "conv1d_k8.sexp")).read())
    ri = interp.random_inputs(p, 7)
    arrays["rand_conv1d_k8_K"] = ri["K"].data
    arrays["rand_conv1d_k8_I"] = ri["I"].data

    # -- conv corpus: source form == lowered form, outputs recorded
    corpus = {}
    programs = {}
    for name in ("conv1d_k8", "conv1d_k16", "conv2d_outer_ry", "downsample2_1d", "upsample2_1d"):
        prog = ir.parse_program(open(os.path.join(CORPUS, f"{name}.sexp")).read())
        low, rep = selector.select_program(prog, selector.SelectionConfig(target="wmma"))
        low_nd, _ = selector.select_program(
            prog, selector.SelectionConfig(target="wmma", desugar=False))
        programs[name] = {"source": ir.print_program(prog), "lowered": ir.print_program(low),
                          "lowered_shuffle_intrinsics": ir.print_program(low_nd)}
        for seed in range(3):
            ins = interp.random_inputs(prog, seed)
            a = interp.run_program(prog, ins)
            b = interp.run_program(low, ins)
            assert a["output"].data.tobytes() == b["output"].data.tobytes(), (name, seed)
            arrays[f"corpus_{name}_{seed}_K"] = ins["K"].data
            arrays[f"corpus_{name}_{seed}_I"] = ins["I"].data
            arrays[f"corpus_{name}_{seed}_out"] = a["output"].data
        corpus[name] = {"lowered": bool(rep.ok), "intrinsics": sorted(
            {i for s in rep.statements for i in s.intrinsics})}
    kats["corpus"] = corpus

    # -- Lanczos-3 2x statement: f16, declared wmma shape 32x28x8, 256 outputs
    first, w = pipelines_ref.lanczos3_weights(512, 256)
    K = interp.round_f16(w[10])  # interior output: 12 taps
    # the lowered form reads 32 windows of matrix_rows = s*n + l = 28 (31*16 + 28 = 524)
    I = interp.round_f16(rng.uniform(0, 1, 524).astype(np.float32))
    prog = conv_program("f16", 12, 256, len(I), stride=2, shapes=(ShapeDecl("wmma", 32, 28, 8),))
    low, rep = selector.select_program(prog, selector.SelectionConfig(target="wmma"))
    out_src = run(prog, K, I)
    out_low = run(low, K, I)
    assert out_src.tobytes() == out_low.tobytes()
    kats["lanczos_tile"] = {"lowered": bool(rep.ok), "intrinsics": sorted(
        {i for s in rep.statements for i in s.intrinsics})}
    low_nd, _ = selector.select_program(prog, selector.SelectionConfig(target="wmma", desugar=False))
    programs["lanczos_tile"] = {"source": ir.print_program(prog), "lowered": ir.print_program(low),
                                "lowered_shuffle_intrinsics": ir.print_program(low_nd)}
    kats["programs"] = programs
    arrays["lanczos_tile_K"], arrays["lanczos_tile_I"], arrays["lanczos_tile_out"] = K, I, out_src

    # -- image-level goldens: a small bf16 image through reference programs,
    #    clamp-to-edge by pre-padding the windows (the oracle's policy)
    H, W = 48, 64
    img = interp.round_bf16(rng.uniform(0, 1, (H, W)).astype(np.float32))
    arrays["img"] = img

    def ref_pass_rows_fast(x, first, weights):
        """Same, one program per (row, run of identical interior weights):
        interior outputs of a Toeplitz axis share the kernel, so a single
        strided statement covers them (the corpus form)."""
        n_out, taps = weights.shape
        out = np.zeros((x.shape[0], n_out), np.float32)
        step = first[1] - first[0] if n_out > 1 else 1
        interior = [o for o in range(n_out)
                    if first[o] >= 0 and first[o] + taps <= x.shape[1]
                    and np.array_equal(weights[o], weights[n_out // 2])
                    and first[o] == first[0] + step * o]
        edge = [o for o in range(n_out) if o not in interior]
        if interior:
            o0, o1 = interior[0], interior[-1]
            n = o1 - o0 + 1
            prog = conv_program("bf16", taps, n, x.shape[1], stride=step, base=int(first[o0]))
            for r in range(x.shape[0]):
                out[r, o0:o1 + 1] = run(prog, weights[o0], x[r])
        for o in edge:
            idx = np.clip(first[o] + np.arange(taps), 0, x.shape[1] - 1)
            prog = conv_program("bf16", taps, 1, taps)
            for r in range(x.shape[0]):
                out[r, o] = run(prog, weights[o], x[r, idx])[0]
        return out

    def ref_separable(x, rows, cols):
        h = ref_pass_rows_fast(x, *cols)            # horizontal
        return ref_pass_rows_fast(h.T.copy(), *rows).T.copy()  # vertical on the transpose

    # weights rounded to bf16 so the K buffers are exactly representable
    rw = pipelines_ref.lanczos3_weights(H, H // 2)
    cw = pipelines_ref.lanczos3_weights(W, W // 2)
    rw = (rw[0], interp.round_bf16(rw[1]))
    cw = (cw[0], interp.round_bf16(cw[1]))
    arrays["lz_rows_first"], arrays["lz_rows_w"] = rw
    arrays["lz_cols_first"], arrays["lz_cols_w"] = cw
    arrays["lz_out"] = ref_separable(img, rw, cw)

    for taps in (9, 31):
        k = interp.round_bf16(pipelines_ref.gaussian_kernel(taps))
        ra = pipelines_ref.centred_axis(H, k)
        ca = pipelines_ref.centred_axis(W, k)
        arrays[f"gauss{taps}_k"] = k
        arrays[f"gauss{taps}_out"] = ref_separable(img, ra, ca)

    # column walk (vertical window, element stride W): the reference cannot
    # lower it (rules.py:793) but its source-form semantics are defined
    col = 5
    prog = conv_program("bf16", 12, 8, H * W, stride=2, elem_stride=W, base=col)
    arrays["colwalk_K"] = interp.round_bf16(w[10])
    arrays["colwalk_out"] = run(prog, arrays["colwalk_K"], img.reshape(-1))
    kats["colwalk"] = {"col": col, "W": W, "stride": 2, "n_out": 8}

    # -- DCT-16 denoise: the four 16x16x16 products per tile run by the
    #    reference as wmma_mma programs (strict: the hardware shape 16x16x16,
    #    interp.py:25-29); tiles, coring and overlap-add are numpy glue here
    dct_fixtures(arrays, kats, rng)

    # -- layout
    kats["layout"] = layout_fixtures(rng)

    # -- buffer-directory wire format written by the reference (interp.py:640-678)
    wire = os.path.join(OUT, "wire_conv1d_k8")
    st = interp.run_program(ir.parse_program(open(os.path.join(CORPUS, "conv1d_k8.sexp")).read()),
                            interp.random_inputs(ir.parse_program(open(os.path.join(CORPUS, "conv1d_k8.sexp")).read()), 3))
    st["bfvec"] = interp.Buffer("bf16", "mem", interp.round_bf16(rng.uniform(-2, 2, 37).astype(np.float32)))
    st["ivec"] = interp.Buffer("i32", "mem", np.arange(-5, 6, dtype=np.int64))
    interp.save_buffers(st, wire)

    np.savez_compressed(os.path.join(OUT, "reference_golden.npz"), **arrays)
    with open(os.path.join(OUT, "reference_golden.json"), "w") as f:
        json.dump(kats, f, indent=1)
    print("wrote", len(arrays), "arrays and", len(kats), "KAT groups to", OUT)


if __name__ == "__main__":
    main()
