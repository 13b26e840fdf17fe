"""`python -m paper_2512_02371_b200 run FILE [--seed N | --inputs DIR]
[--output DIR] [--json]` — the reference CLI's `run` (cli.py:80-111) with the
GPU executor: the program (reference .sexp syntax) runs through
`executor.run_program`, inputs come from a buffer directory (interp.py:640-678)
or the seeded fills, results can be written back as a buffer directory.

`python -m paper_2512_02371_b200 difftest FILE [--trials N] [--seed S] [--ulp U]
[--json]` is the reference's `difftest` (cli.py:131-183) with the two sides
being the GPU executor and the reference interpreter itself
(`tensorsel.interp.run_program`, imported from the environment or from the
offline install under baseline/_ref): every output parameter compared
bitwise (or within --ulp) over `trials` seeded fills; the report has the
reference's DiffTestResult fields.

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


def _reference_interp():
    """The reference package (tensorsel) — only the difftest uses it."""
    try:
        import tensorsel  # noqa: F401
    except ImportError:
        ref = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
        if ref.is_dir():
            sys.path.insert(0, str(ref))
    try:
        from tensorsel import interp as rinterp, ir as rir
    except ImportError:
        return None
    return rinterp, rir


def _ulp_equal(a, b, ulps) -> bool:
    """The reference's comparison (cli.py:121-128): bitwise, or within `ulps`
    units in the last place of the f32 carriers (ints exactly)."""
    import numpy as np
    if a.dtype == np.int64 or b.dtype == np.int64:
        return np.array_equal(a, b)
    ai = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    bi = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    ai = np.where(ai < 0, -(2**31) - ai, ai)
    bi = np.where(bi < 0, -(2**31) - bi, bi)
    return bool(np.all(np.abs(ai - bi) <= ulps))


def cmd_difftest(args) -> int:
    import numpy as np
    from . import executor, fills
    from .errors import EvalError
    prog = _load(args.file)
    ref = _reference_interp()
    if ref is None:
        print("error: the reference interpreter (tensorsel) is not importable; install it "
              "offline under baseline/_ref", file=sys.stderr)
        return 2
    rinterp, rir = ref
    try:
        rprog = rir.parse_program(Path(args.file).read_text())
    except Exception as e:  # the reference's own parse error
        print(f"error: {args.file}: {e}", file=sys.stderr)
        return 2
    result = {"program": Path(args.file).stem, "trials": args.trials, "seeds": [],
              "selection_ok": True, "divergence": None}
    try:
        for t in range(args.trials):
            seed = args.seed + t
            result["seeds"].append(seed)
            inputs = fills.random_inputs(prog, seed)
            out_gpu = executor.run_program(prog, inputs)
            out_ref = rinterp.run_program(rprog, {k: np.array(v) for k, v in inputs.items()})
            for prm in prog.params:
                a = np.asarray(out_ref[prm.name].data)
                b = np.asarray(out_gpu[prm.name].data)
                same = (_ulp_equal(a, b, args.ulp) if args.ulp
                        else a.astype(b.dtype).tobytes() == b.tobytes())
                if not same:
                    lane = int(np.nonzero(a != b)[0][0])
                    result["divergence"] = {"seed": seed, "buffer": prm.name, "lane": lane,
                                            "lhs": float(a[lane]), "rhs": float(b[lane])}
                    break
            if result["divergence"]:
                break
    except EvalError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    if args.json:
        print(json.dumps(result, indent=2))
    else:
        status = "diverged" if result["divergence"] else "ok"
        print(f"{result['program']}: {len(result['seeds'])} trials: {status}")
        if result["divergence"]:
            d = result["divergence"]
            print(f"  seed {d['seed']} buffer {d['buffer']} lane {d['lane']}: "
                  f"{d['lhs']} vs {d['rhs']}")
    return 1 if result["divergence"] else 0


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
    p.set_defaults(fn=cmd_run)
    p = sub.add_parser("difftest", help="GPU executor vs the reference interpreter, "
                                        "bitwise or within --ulp, over seeded fills")
    p.add_argument("file")
    p.add_argument("--trials", type=int, default=100)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--ulp", type=int, default=0, help="tolerate this many ULPs (default: bitwise)")
    p.add_argument("--json", action="store_true", help="JSON output")
    p.set_defaults(fn=cmd_difftest)
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    try:
        return args.fn(args)
    except SystemExit as e:
        return int(e.code)
