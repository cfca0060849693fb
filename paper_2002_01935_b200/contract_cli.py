"""`contract` command of the SPEC CLI (`/root/reference/SPEC.md:553`, `:661-667`)
on the B200 executor.

    python -m paper_2002_01935_b200.contract_cli NETWORK.json PATH.json \
        [--slices SLICES.json | --target-width W] [--slice-range S0 S1] [--precision 3xtf32]

Reads the network interchange JSON (network.py:283-374 format), a path document
(``{"format": "linear"|"ssa", "path": ...}``, tree.py:195-223) and optionally a
SliceSet document (``{"labels": [...], ...}``); writes the result
document ``{"value": [re, im] | {"shape", "re", "im"}, "exponent10", "op_count",
"peak_memory_elements", "W_s", "d_sliced", "slices_run"}`` to stdout.  Exit
codes follow SPEC.md:664: 2 usage, 4 data, 5 numeric.
"""

from __future__ import annotations

import argparse
import json
import sys

import numpy as np


def result_document(value, exponent10, op_count, plan_stats, slices_run):
    arr = np.asarray(value)
    if arr.ndim == 0:
        val = [float(arr.real), float(arr.imag)]
    else:
        val = {"shape": list(arr.shape), "re": arr.real.ravel().tolist(), "im": arr.imag.ravel().tolist()}
    return {"value": val, "exponent10": float(exponent10), "op_count": str(op_count),
            "peak_memory_elements": int(plan_stats["peak_elements"]), "W_s": plan_stats["W_s"],
            "d_sliced": str(plan_stats["d"]), "slices_run": str(slices_run)}


def main(argv=None):
    from .refpkg import DataError, load_network
    from .refpkg import tree_from_path_dict
    from .slicing import SliceSet, greedy_slice
    from .executor import SlicedPlan, _finish, _combine_exp

    ap = argparse.ArgumentParser(prog="contract")
    ap.add_argument("network")
    ap.add_argument("path")
    ap.add_argument("--slices")
    ap.add_argument("--target-width", type=float)
    ap.add_argument("--slice-range", type=int, nargs=2)
    ap.add_argument("--precision", default="3xtf32", choices=["3xtf32", "fp32", "tf32-bf16x"])
    ap.add_argument("--strip-exponent", action="store_true")
    ap.add_argument("--device", type=int, default=0)
    try:
        args = ap.parse_args(argv)
    except SystemExit:
        return 2
    try:
        tn = load_network(args.network)
        with open(args.path) as fh:
            tree = tree_from_path_dict(json.load(fh), tn)
        if args.slices:
            with open(args.slices) as fh:
                ss = SliceSet.from_dict(json.load(fh), tree, tn)
        elif args.target_width is not None:
            ss = greedy_slice(tree, tn, args.target_width)
        else:
            ss = SliceSet.from_labels(tree, tn, ())
    except DataError as exc:
        print(json.dumps({"error": str(exc)}), file=sys.stderr)
        return 4
    except (ValueError, OSError, json.JSONDecodeError) as exc:
        print(json.dumps({"error": str(exc)}), file=sys.stderr)
        return 2

    def err(code, exc):
        print(json.dumps({"error": str(exc)}), file=sys.stderr)
        return code

    try:
        # strip_exponent: every intermediate is renormalised on the
        # device, so networks whose value overflows complex64/128 still contract
        plan = SlicedPlan(tn, tree, ss, device=args.device, precision=args.precision,
                          strip_exponent=args.strip_exponent)
    except DataError as exc:
        return err(4, exc)
    except ValueError as exc:
        return err(2, exc)
    except MemoryError as exc:
        return err(5, exc)
    try:
        s0, s1 = args.slice_range if args.slice_range else (0, plan.d)
        if not 0 <= s0 <= s1 <= plan.d:
            return err(2, ValueError(f"--slice-range [{s0}, {s1}) out of [0, {plan.d})"))
        plan.bind()
        plan.run(s0, s1)
        if args.strip_exponent:
            val, e10 = _combine_exp([plan.result_exp()], tn)
        else:
            val, e10 = _finish(plan.result(), tn, False)
        doc = result_document(val, e10, plan.ops_per_slice * (s1 - s0), plan.stats(), s1 - s0)
    except FloatingPointError as exc:
        return err(5, exc)
    except DataError as exc:
        return err(4, exc)
    except ValueError as exc:
        return err(2, exc)
    except (MemoryError, RuntimeError) as exc:
        return err(5, exc)
    finally:
        plan.close()
    print(json.dumps(doc))
    return 0


if __name__ == "__main__":
    sys.exit(main())
