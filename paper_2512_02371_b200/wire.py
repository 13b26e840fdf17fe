"""Buffer-directory wire format (interp.py:640-678), straight to and from the GPU.

A directory holds ``manifest.json`` ({"buffers": [{name, kind, length,
location}, ...]}) and one little-endian ``<name>.bin`` per buffer: f32 as
<f4, f16 as <f2, i32 as <i4, bf16 as the upper 16 bits of the f32 pattern
(<u2).  ``load_buffers(dir, device=...)`` reads each file into pinned host
memory and copies it to the device asynchronously (bf16 files land as
torch.bfloat16 tensors, no f32 round trip); ``save_buffers`` is the inverse.
Without ``device`` the functions return / accept numpy f32 carriers exactly
like the reference, so directories are interchangeable with
``tensorsel run --inputs`` (cli.py:85-95).
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

_NP_DTYPE = {"f32": "<f4", "f16": "<f2", "i32": "<i4", "bf16": "<u2"}


def read_manifest(dirpath):
    return json.loads((Path(dirpath) / "manifest.json").read_text())["buffers"]


def load_buffers(dirpath, device=None):
    """name -> (kind, location, data).  data: numpy carrier (f32, or int64 for
    i32) when device is None; otherwise a torch tensor on `device` in the
    file's native dtype (bf16 -> torch.bfloat16, f16 -> float16, ...)."""
    d = Path(dirpath)
    out = {}
    for e in read_manifest(d):
        name, kind = e["name"], e["kind"]
        raw = np.fromfile(d / f"{name}.bin", dtype=_NP_DTYPE[kind])
        if len(raw) != e["length"]:
            from .errors import EvalError
            raise EvalError(f"{name}.bin has {len(raw)} elements, manifest says {e['length']}")
        loc = e.get("location", "mem")
        if device is None:
            if kind == "bf16":
                data = (raw.astype(np.uint32) << 16).view(np.float32).copy()
            elif kind == "i32":
                data = raw.astype(np.int64)
            else:
                data = raw.astype(np.float32)
        else:
            import torch
            tdt = {"f32": torch.float32, "f16": torch.float16, "i32": torch.int32,
                   "bf16": torch.bfloat16}[kind]
            host = torch.from_numpy(raw.view(np.int16) if kind == "bf16" else raw)
            if kind == "bf16":
                host = host.view(torch.bfloat16)
            data = host.pin_memory().to(device, non_blocking=True).to(tdt)
        out[name] = (kind, loc, data)
    return out


def save_buffers(store, dirpath):
    """store: name -> (kind, location, data) or an object with .kind/.location
    /.data (interp.Buffer, executor.Buffer).  Torch tensors are read back from
    the device."""
    d = Path(dirpath)
    d.mkdir(parents=True, exist_ok=True)
    manifest = []
    for name in sorted(store):
        b = store[name]
        kind, loc, data = (b if isinstance(b, tuple) else (b.kind, b.location, b.data))
        if hasattr(data, "detach"):  # torch tensor
            import torch
            t = data.detach().cpu()
            if kind == "bf16":
                raw = t.to(torch.bfloat16).contiguous().view(torch.int16).numpy().view("<u2")
            else:
                raw = t.numpy().astype(_NP_DTYPE[kind])
        elif kind == "bf16":
            raw = (np.asarray(data, np.float32).view(np.uint32) >> 16).astype("<u2")
        else:
            raw = np.asarray(data).astype(_NP_DTYPE[kind])
        manifest.append({"name": name, "kind": kind, "length": int(raw.size), "location": loc})
        raw.tofile(d / f"{name}.bin")
    (d / "manifest.json").write_text(json.dumps({"buffers": manifest}, indent=2) + "\n")
