"""Diagnostics-library checks (tools only; not part of tests/ — run by hand
on a GPU box after `make -C paper_2512_02371_b200/csrc diag`):

    python -m pytest tools/diag/test_diag.py -q
"""

import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch


def test_probe_umma_layouts():
    torch = _torch()
    from paper_2512_02371_b200 import _lib
    g = torch.Generator(device="cpu").manual_seed(0)
    for k, n in ((16, 16), (48, 16), (64, 32), (128, 128), (256, 256)):
        a = torch.randn(128, k, generator=g).bfloat16().float().cuda()
        b = torch.randn(k, n, generator=g).bfloat16().float().cuda()
        d = torch.zeros(128, n, device="cuda")
        _lib.check(_lib.load_diag().ts_probe_umma(a.data_ptr(), b.data_ptr(), d.data_ptr(), k, n,
                                             torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        ref = a @ b
        err = (d - ref).abs().max().item()
        assert err < 1e-3 * max(1.0, ref.abs().max().item()), (k, n, err)


