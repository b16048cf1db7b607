"""Command-line front end for the hot path: ``gen``, ``jump`` and ``hwd``.

Behaves like the reference CLI (/root/reference/pkg/src/slprng/cli.py):
the same subcommands, flags, defaults, output formats and exit codes (0 ok,
1 I/O, 2 usage, 3 statistical failure).  ``gen --format raw`` streams
little-endian words produced on the GPU (LanedStream -> kernels K1/K2; the
reference's cli.py:88-97); ``hex`` and ``json`` print the scalar sequence
(cli.py:98-104); ``jump`` prints the flat state after a jump (cli.py:163-180);
``hwd --algo`` runs the HWD test with the GPU counting consumer
(cli.py:122-160).  ``hwd --stdin`` and ``analyze`` are outside this
package's scope.

The option tables below (``_OPTIONS``) are the single source of the
command-line surface; ``build_parser`` only turns them into argparse calls.

    python -m paper_1805_01407_b200 gen --algo xoshiro256starstar --seed 42 --values 1e9 > out.bin
"""

from __future__ import annotations

import argparse
import json
import os
import sys

from . import generators
from .generators import Generator, GeneratorSpec

EXIT_OK, EXIT_IO, EXIT_USAGE, EXIT_STAT_FAIL = 0, 1, 2, 3


class CliError(Exception):
    """A user-facing failure: message for stderr plus the process exit code."""

    def __init__(self, message, code=EXIT_USAGE):
        super().__init__(message)
        self.code = code


# ---------------------------------------------------------------- argument types


def _parse_int(text: str) -> int:
    """Integers in any base prefix (0x.., 0o.., 0b..) or decimal."""
    return int(text, 0)


def _parse_count(text: str) -> int:
    """Counts: an integer literal, or a float literal with an integral,
    non-negative value such as 4e9 (reference cli.py:36-44)."""
    try:
        return int(text, 0)
    except ValueError:
        pass
    value = float(text)
    whole = int(value)
    if value < 0 or value != whole:
        raise argparse.ArgumentTypeError(f"not a whole count: {text!r}")
    return whole


# ------------------------------------------------------------- generator lookup


def _get_spec(name: str) -> GeneratorSpec:
    if name in generators.registry_names(include_analysis=True):
        return generators.get_spec(name)
    names = ", ".join(sorted(generators.registry_names(include_analysis=True)))
    raise CliError(f"unknown algorithm {name!r} (known: {names})")


def _parse_state_words(text: str) -> list[int]:
    """--state: hexadecimal words separated by commas and/or whitespace."""
    return [int(tok, 16) for tok in text.replace(",", " ").split()]


def _make_generator(args) -> Generator:
    """The scalar generator a subcommand starts from: --state wins over --seed."""
    spec = _get_spec(args.algo)
    text = getattr(args, "state", None)
    if not text:
        return Generator.from_seed(spec, args.seed)
    try:
        return Generator(spec, _parse_state_words(text))
    except ValueError as e:
        raise CliError(f"bad --state: {e}")


def _hex_words(values, w: int) -> list[str]:
    width = w // 4
    return [format(v, f"0{width}x") for v in values]


# ------------------------------------------------------------------ raw output

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


# ---------------------------------------------------------------- subcommands


def cmd_gen(args) -> int:
    spec = _get_spec(args.algo)
    gen = _make_generator(args)
    if args.format == "raw":
        sink = sys.stdout.buffer
        try:
            write_raw(spec, gen, args.values, sink)
        except RuntimeError as e:
            raise CliError(str(e), EXIT_IO)
        sink.flush()
    elif args.format == "hex":
        for word in _hex_words((gen.next() for _ in range(args.values)), spec.kind.w):
            print(word)
    else:  # json
        values = [gen.next() for _ in range(args.values)]
        print(json.dumps({"algo": args.algo, "seed": args.seed, "values": values}))
    return EXIT_OK


def _jump_polynomial(spec: GeneratorSpec, args):
    if args.steps is not None:
        return generators.compute_jump_poly(spec, args.steps)
    short, long_ = generators.default_jumps(spec)
    return long_ if args.long_jump else short


def cmd_jump(args) -> int:
    spec = _get_spec(args.algo)
    gen = _make_generator(args)
    jp = _jump_polynomial(spec, args)
    if jp.step_count:
        gen.jump(jp)
    state = _hex_words(gen.flat_words(), spec.kind.w)
    if args.json:
        print(json.dumps({"algo": args.algo, "steps": str(jp.step_count), "state": state}))
    else:
        print(f"state after {jp.step_count} steps: {' '.join(state)}")
    return EXIT_OK


_VERDICTS = {"failed": "FAILED (p-value threshold tripped)", "passed": "passed to the byte limit",
             "inconclusive": "inconclusive (source exhausted)"}


def _print_hwd_report(report) -> None:
    print(f"mode={report.mode} w={report.w} k={report.k} ell={report.ell}")
    for ck in report.history:
        print(f"  {ck.bytes:>16d} bytes  p = {ck.p_value:.6g}  "
              f"signature {ck.faulty_signature} (category {ck.faulty_category})")
    print(f"{_VERDICTS[report.status]}: {report.bytes_processed} bytes, p = {report.p_value:.6g}, "
          f"faulty signature {report.faulty_signature!r}")


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
        _print_hwd_report(report)
    return EXIT_STAT_FAIL if report.status == "failed" else EXIT_OK


# ------------------------------------------------------------------- the parser

# (flags, argparse keyword arguments) per subcommand, in --help order
_GENERATOR = [
    (("--algo",), dict(required=True)),
]
_OPTIONS = {
    "gen": ("emit generator output", cmd_gen, _GENERATOR + [
        (("--seed",), dict(type=_parse_int, default=0)),
        (("--state",), dict(help="full state as hex words (overrides --seed)")),
        (("--values",), dict(type=_parse_count, default=16)),
        (("--format",), dict(choices=("raw", "hex", "json"), default="raw")),
    ]),
    "hwd": ("run the Hamming-weight dependency test on a generator (GPU)", cmd_hwd, [
        (("--algo",), dict()),
        (("--stdin",), dict(action="store_true", help="not supported by this build")),
        (("--seed",), dict(type=_parse_int, default=1)),
        (("--w",), dict(type=int, default=64)),
        (("--k",), dict(type=int, default=8)),
        (("--ell",), dict(type=int, default=None)),
        (("--C",), dict(type=int, default=None)),
        (("--mode",), dict(choices=("standard", "transitional"), default="standard")),
        (("--limit",), dict(type=_parse_count, default=10**15, help="byte limit")),
        (("--p-threshold",), dict(type=float, default=1e-20, dest="p_threshold")),
        (("--batch-size",), dict(type=_parse_count, default=None, dest="batch_size")),
        (("--split",), dict(action="store_true", help="break 64-bit source words into two 32-bit test values")),
        (("--checkpoint-start",), dict(type=_parse_count, default=None, dest="checkpoint_start")),
        (("--json",), dict(action="store_true")),
    ]),
    "jump": ("print the state after a jump", cmd_jump, _GENERATOR + [
        (("--seed",), dict(type=_parse_int, default=0)),
        (("--state",), dict()),
        (("--steps",), dict(type=_parse_count, default=None,
                            help="step count (default: the generator's jump, 2^(n/2))")),
        (("--long-jump",), dict(action="store_true", dest="long_jump", help="use the long jump, 2^(3n/4) steps")),
        (("--json",), dict(action="store_true")),
    ]),
}


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_1805_01407_b200",
                                     description="Scrambled linear generators on B200: bulk output and jumps.")
    commands = parser.add_subparsers(dest="command", required=True)
    for name, (summary, handler, options) in _OPTIONS.items():
        cmd = commands.add_parser(name, help=summary)
        for flags, kwargs in options:
            cmd.add_argument(*flags, **kwargs)
        cmd.set_defaults(func=handler)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except CliError as err:
        print(f"error: {err}", file=sys.stderr)
        return err.code
    except BrokenPipeError:  # the reader went away: not an error worth a message
        return EXIT_IO
    except OSError as err:
        print(f"I/O error: {err}", file=sys.stderr)
        return EXIT_IO
