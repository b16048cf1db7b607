"""Command-line front end for the hot path: ``gen`` and ``jump``.

Mirrors the reference CLI (/root/reference/pkg/src/slprng/cli.py): the same
arguments, output formats and exit codes (0 ok, 1 I/O, 2 usage).
``gen --format raw`` streams little-endian words produced on the GPU
(LanedStream -> kernels K1/K2, cli.py:88-97 in the reference); ``hex`` and
``json`` print the scalar sequence (cli.py:98-104); ``jump`` prints the flat
state after a jump (cli.py:163-180); ``hwd --algo`` runs the HWD test with
the GPU counting consumer (cli.py:122-160).  ``hwd --stdin`` and ``analyze``
are outside this package's scope.

    python -m paper_1805_01407_b200 gen --algo xoshiro256starstar --seed 42 --values 1e9 > out.bin
"""

from __future__ import annotations

import argparse
import json
import os
import sys

from . import generators
from .generators import Generator, GeneratorSpec

EXIT_OK = 0
EXIT_IO = 1
EXIT_USAGE = 2


class CliError(Exception):
    def __init__(self, message, code=EXIT_USAGE):
        super().__init__(message)
        self.code = code


def _parse_int(text: str) -> int:
    return int(text, 0)


def _parse_count(text: str) -> int:
    """Counts accept 4e9-style notation (cli.py:36-44)."""
    try:
        return int(text, 0)
    except ValueError:
        v = float(text)
        if v < 0 or v != int(v):
            raise argparse.ArgumentTypeError(f"not a whole count: {text!r}")
        return int(v)


def _get_spec(name: str) -> GeneratorSpec:
    try:
        return generators.get_spec(name)
    except KeyError:
        known = ", ".join(sorted(generators.registry_names(include_analysis=True)))
        raise CliError(f"unknown algorithm {name!r} (known: {known})")


def _make_generator(args) -> Generator:
    spec = _get_spec(args.algo)
    if getattr(args, "state", None):
        try:
            words = [int(t, 16) for t in args.state.replace(",", " ").split()]
            return Generator(spec, words)
        except ValueError as e:
            raise CliError(f"bad --state: {e}")
    return Generator.from_seed(spec, args.seed)


# superbatch geometry for raw output: any (lanes, lane_len) gives the same
# stream (LanedStream contract); 2^16 lanes x 1024 = 512 MiB of u64 per chunk
_RAW_LANE_LEN = 1024
_RAW_MAX_LANES = 1 << 16


def _grow_pipe(out) -> None:
    """A 64 KiB pipe caps the raw stream at ~3 GB/s; ask for the largest
    pipe the system allows (Linux F_SETPIPE_SZ, /proc/sys/fs/pipe-max-size)."""
    try:
        import fcntl
        import stat

        fd = out.fileno()
        if not stat.S_ISFIFO(os.fstat(fd).st_mode):
            return
        try:
            with open("/proc/sys/fs/pipe-max-size") as f:
                size = int(f.read())
        except OSError:
            size = 1 << 20
        fcntl.fcntl(fd, fcntl.F_SETPIPE_SZ, size)
    except (OSError, AttributeError, ValueError, ImportError):
        pass


def write_raw(spec: GeneratorSpec, gen: Generator, n: int, out) -> None:
    """Little-endian w-bit words of the stream of ``gen`` (n values) to ``out``."""
    import numpy as np

    if n <= 0:
        return
    lanes = max(1, min(_RAW_MAX_LANES, -(-n // _RAW_LANE_LEN)))
    stream = generators.LanedStream(spec, generator=gen, lanes=lanes, lane_len=_RAW_LANE_LEN)
    dtype = np.dtype("<u8") if spec.kind.w == 64 else np.dtype("<u4")
    _grow_pipe(out)
    # pipelined GPU -> pinned staging -> output, no intermediate copies
    for chunk in stream.chunks(n, native=True, _views=True):
        out.write(memoryview(chunk.astype(dtype, copy=False)).cast("B"))


def cmd_gen(args) -> int:
    spec = _get_spec(args.algo)
    gen = _make_generator(args)
    n = args.values
    if args.format == "raw":
        out = sys.stdout.buffer
        try:
            write_raw(spec, gen, n, out)
        except RuntimeError as e:
            raise CliError(str(e), EXIT_IO)
        out.flush()
        return EXIT_OK
    digits = spec.kind.w // 4
    if args.format == "hex":
        for _ in range(n):
            print(f"{gen.next():0{digits}x}")
        return EXIT_OK
    print(json.dumps({"algo": args.algo, "seed": args.seed, "values": [gen.next() for _ in range(n)]}))
    return EXIT_OK


def cmd_jump(args) -> int:
    spec = _get_spec(args.algo)
    gen = _make_generator(args)
    if args.steps is not None:
        jp = generators.compute_jump_poly(spec, args.steps)
    else:
        jump, long_jump = generators.default_jumps(spec)
        jp = long_jump if args.long_jump else jump
    if jp.step_count:
        gen.jump(jp)
    digits = spec.kind.w // 4
    state = [f"{x:0{digits}x}" for x in gen.flat_words()]
    if args.json:
        print(json.dumps({"algo": args.algo, "steps": str(jp.step_count), "state": state}))
    else:
        print(f"state after {jp.step_count} steps: {' '.join(state)}")
    return EXIT_OK


EXIT_STAT_FAIL = 3


def cmd_hwd(args) -> int:
    """HWD test of a named generator with the GPU counting consumer
    (reference cli.py:122-160; --stdin sources are not supported here)."""
    from . import hwd

    if args.stdin or not args.algo:
        raise CliError("this build tests generators on the GPU: use --algo NAME (no --stdin)")
    config = hwd.HwdConfig(w=args.w, k=args.k, ell=args.ell, C=args.C, batch_size=args.batch_size,
                           p_threshold=args.p_threshold, byte_limit=args.limit, mode=args.mode, split=args.split)
    try:
        report = hwd.run_generator(_get_spec(args.algo), config, seed=args.seed,
                                   checkpoint_start=args.checkpoint_start)
    except RuntimeError as e:
        raise CliError(str(e), EXIT_IO)
    if args.json:
        print(json.dumps(report.to_dict()))
    else:
        print(f"mode={report.mode} w={report.w} k={report.k} ell={report.ell}")
        for ck in report.history:
            print(f"  {ck.bytes:>16d} bytes  p = {ck.p_value:.6g}  "
                  f"signature {ck.faulty_signature} (category {ck.faulty_category})")
        verdict = {"failed": "FAILED (p-value threshold tripped)", "passed": "passed to the byte limit",
                   "inconclusive": "inconclusive (source exhausted)"}[report.status]
        print(f"{verdict}: {report.bytes_processed} bytes, p = {report.p_value:.6g}, "
              f"faulty signature {report.faulty_signature!r}")
    return EXIT_STAT_FAIL if report.status == "failed" else EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1805_01407_b200",
                                 description="Scrambled linear generators on B200: bulk output and jumps.")
    sub = ap.add_subparsers(dest="command", required=True)
    g = sub.add_parser("gen", help="emit generator output")
    g.add_argument("--algo", required=True)
    g.add_argument("--seed", type=_parse_int, default=0)
    g.add_argument("--state", help="full state as hex words (overrides --seed)")
    g.add_argument("--values", type=_parse_count, default=16)
    g.add_argument("--format", choices=("raw", "hex", "json"), default="raw")
    g.set_defaults(func=cmd_gen)
    h = sub.add_parser("hwd", help="run the Hamming-weight dependency test on a generator (GPU)")
    h.add_argument("--algo")
    h.add_argument("--stdin", action="store_true", help="not supported by this build")
    h.add_argument("--seed", type=_parse_int, default=1)
    h.add_argument("--w", type=int, default=64)
    h.add_argument("--k", type=int, default=8)
    h.add_argument("--ell", type=int, default=None)
    h.add_argument("--C", type=int, default=None)
    h.add_argument("--mode", choices=("standard", "transitional"), default="standard")
    h.add_argument("--limit", type=_parse_count, default=10**15, help="byte limit")
    h.add_argument("--p-threshold", type=float, default=1e-20, dest="p_threshold")
    h.add_argument("--batch-size", type=_parse_count, default=None, dest="batch_size")
    h.add_argument("--split", action="store_true", help="break 64-bit source words into two 32-bit test values")
    h.add_argument("--checkpoint-start", type=_parse_count, default=None, dest="checkpoint_start")
    h.add_argument("--json", action="store_true")
    h.set_defaults(func=cmd_hwd)
    j = sub.add_parser("jump", help="print the state after a jump")
    j.add_argument("--algo", required=True)
    j.add_argument("--seed", type=_parse_int, default=0)
    j.add_argument("--state")
    j.add_argument("--steps", type=_parse_count, default=None,
                   help="step count (default: the generator's jump, 2^(n/2))")
    j.add_argument("--long-jump", action="store_true", dest="long_jump",
                   help="use the long jump, 2^(3n/4) steps")
    j.add_argument("--json", action="store_true")
    j.set_defaults(func=cmd_jump)
    return ap


def main(argv=None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    try:
        return args.func(args)
    except CliError as e:
        print(f"error: {e}", file=sys.stderr)
        return e.code
    except BrokenPipeError:
        return EXIT_IO
    except OSError as e:
        print(f"I/O error: {e}", file=sys.stderr)
        return EXIT_IO
