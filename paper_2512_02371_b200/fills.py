"""Seeded input fills of the reference CLI's `run --seed` / difftest:
SplitMix64 (interp.py:94-115) and random_inputs (interp.py:622-634), with the
bf16 / f16 rounding of interp.round_to_kind (interp.py:62-87).  Host-side
utility for `python -m paper_2512_02371_b200 run`; pinned against the
reference's known-answer values by tests/test_cli.py."""

from __future__ import annotations

import numpy as np

_M = (1 << 64) - 1


class SplitMix64:
    def __init__(self, seed: int):
        self.s = seed & _M

    def next_u64(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & _M
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M
        return z ^ (z >> 31)

    def uniform(self) -> float:  # [-1, 1)
        return (self.next_u64() >> 11) / float(1 << 53) * 2.0 - 1.0

    def small_int(self) -> int:  # [0, 16)
        return self.next_u64() >> 60


def round_bf16(x):
    """Round-to-nearest-even into the bf16 value set, carried in f32."""
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    nan = np.isnan(np.asarray(x, dtype=np.float32))
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32)
    return np.where(nan, np.float32(np.nan), out).astype(np.float32)


def round_to_kind(x, kind: str):
    if kind == "bf16":
        return round_bf16(x)
    if kind == "f16":
        with np.errstate(over="ignore"):
            return np.asarray(x, dtype=np.float32).astype(np.float16).astype(np.float32)
    return np.asarray(x, dtype=np.float32)


def random_inputs(program, seed: int):
    """One SplitMix64 stream over the program's params in declaration order:
    i32 -> [0, 16), floats -> uniform [-1, 1) rounded to the param kind."""
    rng = SplitMix64(seed)
    out = {}
    for prm in program.params:
        if prm.kind == "i32":
            out[prm.name] = np.array([rng.small_int() for _ in range(prm.length)], np.int64)
        else:
            raw = np.array([rng.uniform() for _ in range(prm.length)], np.float32)
            out[prm.name] = round_to_kind(raw, prm.kind)
    return out
