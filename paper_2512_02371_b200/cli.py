"""`python -m paper_2512_02371_b200 run FILE [--seed N | --inputs DIR]
[--output DIR] [--json]` — the reference CLI's `run` (cli.py:80-111) with the
GPU executor: the program (reference .sexp syntax) runs through
`executor.run_program`, inputs come from a buffer directory (interp.py:640-678)
or the seeded fills, results can be written back as a buffer directory.

Exit codes as the reference's (cli.py:3-6): 0 success, 1 evaluation failure
(EvalError: OutOfBounds, ShapeUnregistered, ... or UnsupportedProgram for
statements outside the convolution family), 2 usage or parse failure.  The
reference's program validator (ir.validate_program) is not re-implemented
here; programs are parsed and executed."""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path


def _load(path):
    from . import irlite
    try:
        text = Path(path).read_text()
    except OSError as e:
        print(f"error: cannot read {path}: {e}", file=sys.stderr)
        raise SystemExit(2)
    try:
        return irlite.parse_program(text)
    except (ValueError, IndexError) as e:
        print(f"error: {path}: {e}", file=sys.stderr)
        raise SystemExit(2)


def cmd_run(args) -> int:
    from . import executor, fills, wire
    from .errors import EvalError
    prog = _load(args.file)
    if args.inputs:
        try:
            raw = wire.load_buffers(args.inputs)
        except (OSError, ValueError, EvalError) as e:
            print(f"error: {e}", file=sys.stderr)
            return 1
        inputs = {}
        for prm in prog.params:
            if prm.name not in raw:
                print(f"error: inputs are missing {prm.name!r}", file=sys.stderr)
                return 1
            data = raw[prm.name][2]
            if len(data) != prm.length:
                print(f"error: input {prm.name!r} has length {len(data)}, manifest/program "
                      f"disagree", file=sys.stderr)
                return 1
            inputs[prm.name] = data
    else:
        inputs = fills.random_inputs(prog, args.seed)
    lints = []
    try:
        out = executor.run_program(prog, inputs, lint_sink=lints)
    except EvalError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    for lint in lints:
        print(f"warning: {lint}", file=sys.stderr)
    if args.output:
        wire.save_buffers(out, args.output)
    summary = {name: {"kind": buf.kind, "length": len(buf.data)}
               for name, buf in sorted(out.items())}
    if args.json:
        print(json.dumps({"buffers": summary}, indent=2))
    else:
        for name, meta in summary.items():
            print(f"{name}: {meta['kind']} x {meta['length']}")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2512_02371_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("run", help="execute a convolution-family program on the GPU")
    p.add_argument("file")
    g = p.add_mutually_exclusive_group()
    g.add_argument("--seed", type=int, default=0, help="seeded inputs (SplitMix64)")
    g.add_argument("--inputs", help="directory with manifest.json and .bin buffers")
    p.add_argument("--output", help="write the final buffers to this directory")
    p.add_argument("--json", action="store_true", help="JSON output")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    try:
        return cmd_run(args)
    except SystemExit as e:
        return int(e.code)
