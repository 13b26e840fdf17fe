"""Numpy model of DCT-16 denoise intermediates rounded to a 16-bit type
(fp16 / bf16) at every MMA operand boundary, against the f32 oracle: max
error (soft coring) and the fraction of hard-coring threshold flips."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import numpy as np
from oracle import pipelines_ref as pr


def r16(a, kind):
    a = np.asarray(a, np.float32)
    if kind == "f16":
        return a.astype(np.float16).astype(np.float32)
    if kind == "bf16":
        b = a.view(np.uint32).astype(np.uint64)
        b = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
        return b.astype(np.uint32).view(np.float32)
    return a


def sim(img, threshold, mode, kind, n=16):
    x = img.reshape((-1,) + img.shape[-2:])
    h = n // 2
    H, W = x.shape[-2:]
    D = pr.dct_matrix(n); w = pr.sine_window(n)
    Dw = r16((D * w[None, :]).astype(np.float32), kind)
    xp = np.pad(x, ((0, 0), (h, h), (h, h)), mode="edge")
    ty, tx = H // h + 1, W // h + 1
    s = xp.strides
    t = np.lib.stride_tricks.as_strided(xp, shape=(x.shape[0], ty, tx, n, n), strides=(s[0], s[1] * h, s[2] * h, s[1], s[2]))
    t = r16(t, kind)
    d1 = r16(np.einsum("km,ptxmn->ptxkn", Dw, t).astype(np.float32), kind)
    C = np.einsum("ptxkn,ln->ptxkl", d1, Dw).astype(np.float32)
    dc = C[..., 0, 0].copy()
    if mode == "hard":
        C = np.where(np.abs(C) < threshold, np.float32(0), C)
    else:
        C = np.sign(C) * np.maximum(np.abs(C) - threshold, 0)
    C[..., 0, 0] = dc
    C = r16(C, kind)
    d3 = r16(np.einsum("ptxkl,ln->ptxkn", C, Dw).astype(np.float32), kind)
    T = np.einsum("km,ptxkn->ptxmn", Dw, d3).astype(np.float32)
    out = np.zeros_like(xp)
    for py in range(2):
        for px in range(2):
            sub = T[:, py::2, px::2]
            ny, nx = sub.shape[1], sub.shape[2]
            blk = sub.transpose(0, 1, 3, 2, 4).reshape(x.shape[0], ny * n, nx * n)
            out[:, py * h:py * h + ny * n, px * h:px * h + nx * n] += blk
    return out[:, h:h + H, h:h + W]


if __name__ == "__main__":
    rng = np.random.default_rng(3)
    H, W = 544, 960
    yy, xx = np.mgrid[0:H, 0:W]
    clean = 0.5 + 0.4 * np.sin(xx / 17.0) * np.cos(yy / 23.0)
    x = np.clip(clean + rng.normal(0, 0.05, (1, H, W)), 0, 1).astype(np.float32)
    x = r16(x, "bf16")
    for kind in ("f16", "bf16"):
        for mode in ("soft", "hard"):
            ref = pr.dct_denoise(x, 0.15, mode)
            d = np.abs(sim(x, 0.15, mode, kind) - ref)
            print(kind, mode, "max", float(d.max()), "frac>1e-2", float((d > 1e-2).mean()))
        d = np.abs(sim(x, 0.0, "soft", kind) - x[0])
        print(kind, "identity max", float(d.max()))
