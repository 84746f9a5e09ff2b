"""``python -m paper_2502_02704_b200 run|compare --config FILE`` (ref/cli.py:31-60).

Exit code 2 on any SolverError, as the reference's ``parabgk`` entry point.
"""

from __future__ import annotations

import argparse
import sys
from dataclasses import replace

from .errors import SolverError
from .runner import MODES, parse_config, run_comparison, run_mode


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2502_02704_b200",
                                 description="B200 kinetic/fluid parareal solver (1D/3V BGK)")
    sub = ap.add_subparsers(dest="command", required=True)
    for name, helptext in (("run", "run one mode and write its artifacts"),
                           ("compare", "run all modes and report timings")):
        p = sub.add_parser(name, help=helptext)
        p.add_argument("--config", required=True)
        p.add_argument("--workers", type=int, default=None)
        p.add_argument("--out", default=None)
        if name == "run":
            p.add_argument("--mode", choices=MODES, default=None)
    args = ap.parse_args(argv)
    try:
        cfg = parse_config(args.config)
        if getattr(args, "mode", None):
            cfg = replace(cfg, mode=args.mode)
        if args.workers is not None:
            cfg = replace(cfg, workers=args.workers)
        if args.out is not None:
            cfg = replace(cfg, out_dir=args.out)
        if args.command == "run":
            out = run_mode(cfg)
            print("wrote %s artifacts to %s" % (cfg.mode, out))
        else:
            rep = run_comparison(cfg)
            print("speedup %.3f over the serial fine run; suggested iteration bound %s"
                  % (rep.speedup, rep.k_opt))
    except SolverError as exc:
        print("error: %s" % exc, file=sys.stderr)
        return 2
    return 0


if __name__ == "__main__":
    sys.exit(main())
