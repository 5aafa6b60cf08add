"""`python -m paper_2007_05239_b200.cli <command>` -- the reference's command
line (cli.py:1-102) on the B200 backend: same subcommands, flags and exit
codes (0 ok, 2 configuration, 3 numerical, 4 input/output).  --threads is
accepted and sets the host FFT workers of the plan-time transforms."""

import argparse
import logging
import os
import sys

from .config import load_config
from .errors import ConfigError, FormatError, NumericalError
from .runner import run_classify, run_eig, run_fastsum_bench, run_sbm_bench, run_segment_image

COMMANDS = {
    "classify": (run_classify, "semi-supervised classification from features or edge lists"),
    "segment-image": (run_segment_image, "pixel classification of RGB PNG images"),
    "sbm-bench": (run_sbm_bench, "stochastic block model benchmark (not in the B200 backend)"),
    "fastsum-bench": (run_fastsum_bench, "fast summation accuracy and scaling tables"),
    "eig": (run_eig, "write the k smallest power mean eigenvalues"),
}


def build_parser():
    ap = argparse.ArgumentParser(prog="multilap-b200", description=(
        "Multilayer graph clustering via power mean Laplacians on B200: NFFT fast-summation "
        "kernel graphs, power-mean eigensolves and Allen-Cahn label propagation."))
    sub = ap.add_subparsers(dest="command", required=True)
    for name, (_, text) in COMMANDS.items():
        p = sub.add_parser(name, help=text)
        p.add_argument("--config", metavar="PATH", default=None, help="JSON configuration file")
        p.add_argument("--seed", type=int, default=0, help="RNG seed (default 0)")
        p.add_argument("--out", metavar="DIR", default=".", help="output directory (default: current)")
        p.add_argument("--threads", type=int, default=1, help="host FFT worker threads (default 1)")
    return ap


def main(argv=None):
    level = getattr(logging, os.environ.get("MULTILAP_LOG_LEVEL", "WARNING").upper(), logging.WARNING)
    logging.basicConfig(level=level if isinstance(level, int) else logging.WARNING, stream=sys.stderr,
                        format="%(levelname)s %(name)s: %(message)s")
    args = build_parser().parse_args(argv)
    if args.seed < 0:
        print("error: --seed must be nonnegative", file=sys.stderr)
        return 2
    if args.threads < 1:
        print("error: --threads must be at least 1", file=sys.stderr)
        return 2
    try:
        from . import fastsum
        fastsum.set_fft_workers(args.threads)
        report = COMMANDS[args.command][0](load_config(args.config), args.seed, out_dir=args.out,
                                           threads=args.threads)
    except (ConfigError, NumericalError, FormatError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return exc.exit_code
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return FormatError.exit_code
    parts = [f"{args.command}: done"]
    if isinstance(report.get("accuracy"), float):
        parts.append(f"accuracy {report['accuracy']:.4f}")
    if "report" in report.get("outputs", {}):
        parts.append(f"report {report['outputs']['report']}")
    print("; ".join(parts))
    return 0


if __name__ == "__main__":
    sys.exit(main())
