"""portten-bench on the B200: the reference's measurement harness.

  python -m paper_1606_04884_b200.bench_cli apply --sizes 1e3,1e4,1e5,1e6,1e7 --reps 5 --out bw.csv
  python -m paper_1606_04884_b200.bench_cli model --name vgg-a --scale 1 --batch 64 \\
      --impl implicitgemm-sm100a --backward --out layers.csv --summary summary.csv

CSV schemas: bandwidth (size,reps,mean_time_s,gb_per_s); layers
(index,type,geometry,mean_time_s,checksum); summary (type,layers,total_time_s,fraction).
Exit codes: 0 success, 2 ValidationError, 3 BackendError.
"""
from __future__ import annotations

import argparse
import sys

from ._lib import BackendError, ValidationError
from . import model as M


def _sizes(text):
    try:
        return [int(float(t)) for t in text.split(",") if t]
    except ValueError:
        raise ValidationError(f"bad --sizes '{text}'") from None


def _write(path, text):
    if path in (None, "-"):
        sys.stdout.write(text)
    else:
        with open(path, "w") as f:
            f.write(text)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="portten-bench")
    sub = ap.add_subparsers(dest="cmd", required=True)
    a = sub.add_parser("apply", help="per-element bandwidth sweep (Fig. 1-2)")
    a.add_argument("--sizes", default="1e3,1e4,1e5,1e6,1e7")
    a.add_argument("--reps", type=int, default=5)
    a.add_argument("--expr", default="x = x * s")
    a.add_argument("--backend", default="auto", choices=["auto", "device"])
    a.add_argument("--out", default="-")
    m = sub.add_parser("model", help="per-layer model timings with a per-type summary (Fig. 4-5)")
    m.add_argument("--name", required=True, help="alexnet | vgg-a | path to a spec file")
    m.add_argument("--scale", type=int, default=1)
    m.add_argument("--batch", type=int, default=1)
    m.add_argument("--impl", default="implicitgemm-sm100a", choices=list(M.IMPLS))
    m.add_argument("--backward", action="store_true")
    m.add_argument("--reps", type=int, default=5)
    m.add_argument("--backend", default="auto", choices=["auto", "device"])
    m.add_argument("--out", default="-")
    m.add_argument("--summary", default=None)
    args = ap.parse_args(argv)
    try:
        if args.cmd == "apply":
            rows = M.bench_apply(_sizes(args.sizes), args.reps, args.expr)
            _write(args.out, M.to_csv(rows, M.BANDWIDTH_COLUMNS))
        else:
            spec = M.model_spec_load(args.name)
            rows, summary = M.bench_model(spec, args.scale, args.batch, args.backward, args.impl,
                                          args.reps)
            _write(args.out, M.to_csv(rows, M.LAYER_COLUMNS))
            if args.summary:
                _write(args.summary, M.to_csv(summary, M.SUMMARY_COLUMNS))
        return 0
    except ValidationError as ex:
        print(f"portten-bench: {ex}", file=sys.stderr)
        return 2
    except BackendError as ex:
        print(f"portten-bench: {ex}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
