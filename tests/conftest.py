import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and the built native library")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available() and torch.cuda.get_device_capability(0)[0] == 10
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no sm_100 GPU in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def _plane_worker(args):
    fn_name, plane, fargs = args
    from oracle import pipelines_ref
    return getattr(pipelines_ref, fn_name)(plane[None], *fargs)[0]


def oracle_planes(fn_name, img, *fargs):
    """oracle.pipelines_ref.<fn_name>(img, *fargs) with one worker process
    per plane (the full-frame parity tests: 3 planes of 4K/8K in parallel
    on the GPU box's host cores).  Planes are independent in every
    pipeline, so the result equals one call over all planes."""
    import multiprocessing as mp
    import numpy as np
    planes = np.asarray(img).reshape((-1,) + img.shape[-2:])
    with mp.get_context("fork").Pool(min(len(planes), os.cpu_count() or 1)) as pool:
        outs = pool.map(_plane_worker, [(fn_name, p, fargs) for p in planes])
    return np.stack(outs).reshape(img.shape[:-2] + outs[0].shape[-2:])
