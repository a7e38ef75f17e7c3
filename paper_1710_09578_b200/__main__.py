"""``python -m paper_1710_09578_b200 verify [--max-size N] [--seed S]``: the
reference CLI's self-check subcommand (pkg/src/linopkit/cli.py:75-80,
125-133) on the device — one PASS/FAIL line per operator instance, a summary
line, exit code 0 (all pass), 1 (a failure) or 2 (usage error).  The
reference's ``bench`` / ``list-scenarios`` subcommands (dense-vs-structured
timing) are outside this package; ``bench.py`` at the repository root
measures the transforms."""

from __future__ import annotations

import argparse
import sys


def cli_main(argv=None) -> int:
    parser = argparse.ArgumentParser(prog="paper_1710_09578_b200",
                                     description="B200 structured operators: device self-checks.")
    sub = parser.add_subparsers(dest="command", required=True)
    v = sub.add_parser("verify", help="run the oracle/adjoint property suite on the device")
    v.add_argument("--max-size", type=int, default=64, help="largest operator dimension in the zoo")
    v.add_argument("--seed", type=int, default=0)
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return exc.code if isinstance(exc.code, int) else 2
    if args.max_size < 1:
        print("paper_1710_09578_b200 verify: error: --max-size must be >= 1", file=sys.stderr)
        return 2
    from .selfcheck import run_verification

    results = run_verification(max_size=args.max_size, seed=args.seed)
    failures = [r for r in results if not r.passed]
    print(f"{len(results) - len(failures)}/{len(results)} checks passed")
    return 1 if failures else 0


if __name__ == "__main__":
    sys.exit(cli_main())
