"""Output functions (+, *, ++, **) on flat state words.

Same public surface as /root/reference/pkg/src/slprng/scramblers.py
(``ScramblerSpec`` :48-95 and ``scramble_*`` :26-45): field names, kinds,
validation rules and error messages.  Scramblers read the state BEFORE the
engine step; for ``++`` the first word is the one added back.  The device
kernels implement the same functions in registers (csrc/slp_gen.cuh,
``Gen::output``); this module is the host-side scalar form.
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["ScramblerSpec", "scramble_plus", "scramble_star", "scramble_plusplus",
           "scramble_starstar", "SCRAMBLER_KINDS", "SCRAMBLER_CODE"]

SCRAMBLER_KINDS = ("none", "plus", "star", "plusplus", "starstar")
SCRAMBLER_CODE = {k: i for i, k in enumerate(SCRAMBLER_KINDS)}  # the C ABI's SLP_SC_* order


def _wrap(x: int, w: int) -> int:
    """x modulo 2^w."""
    return x & ((1 << w) - 1)


def _rotl(x: int, r: int, w: int) -> int:
    return _wrap(x << r | x >> (w - r), w)


def scramble_plus(x: int, y: int, w: int) -> int:
    return _wrap(x + y, w)


def scramble_star(x: int, s: int, w: int) -> int:
    return _wrap(x * s, w)


def scramble_plusplus(x: int, y: int, r: int, w: int) -> int:
    """rotl(x + y, r) + x."""
    return _wrap(_rotl(_wrap(x + y, w), r, w) + x, w)


def scramble_starstar(x: int, s: int, r: int, t: int, w: int) -> int:
    """rotl(x * s, r) * t."""
    return _wrap(_rotl(_wrap(x * s, w), r, w) * t, w)


def _odd(v) -> bool:
    return v is not None and v % 2 == 1


# (kinds a rule applies to, predicate on (spec, k, w), message) -- the range
# checks of the reference's ScramblerSpec.validate (scramblers.py:68-82), in its order
_RULES = (
    (SCRAMBLER_KINDS, lambda s, k, w: 0 <= s.word_i < k, "word_i out of range"),
    (("plus", "plusplus"), lambda s, k, w: s.word_j is not None and 0 <= s.word_j < k, "word_j out of range"),
    (("star", "starstar"), lambda s, k, w: _odd(s.S), "multiplier S must be odd"),
    (("plusplus", "starstar"), lambda s, k, w: s.R is not None and 0 < s.R < w, "rotation R out of range"),
    (("starstar",), lambda s, k, w: _odd(s.T), "multiplier T must be odd"),
)

# kind -> f(spec, words, w)
_APPLY = {
    "none": lambda s, words, w: words[s.word_i],
    "plus": lambda s, words, w: scramble_plus(words[s.word_i], words[s.word_j], w),
    "star": lambda s, words, w: scramble_star(words[s.word_i], s.S, w),
    "plusplus": lambda s, words, w: scramble_plusplus(words[s.word_i], words[s.word_j], s.R, w),
    "starstar": lambda s, words, w: scramble_starstar(words[s.word_i], s.S, s.R, s.T, w),
}


@dataclass(frozen=True)
class ScramblerSpec:
    """Output function ``kind`` applied to flat state word ``word_i`` (and
    ``word_j`` for + and ++) with multipliers S, T and rotation R."""

    kind: str
    word_i: int = 0
    word_j: int | None = None
    S: int | None = None
    R: int | None = None
    T: int | None = None

    def __post_init__(self):
        if self.kind not in SCRAMBLER_KINDS:
            raise ValueError(f"unknown scrambler kind {self.kind!r}")

    def validate(self, k: int, w: int):
        """Raise ValueError unless the spec fits a k-word, w-bit engine."""
        for kinds, ok, message in _RULES:
            if self.kind in kinds and not ok(self, k, w):
                raise ValueError(message)

    def apply(self, words, w: int) -> int:
        """Scramble the flat state words (before the engine step)."""
        return _APPLY[self.kind](self, words, w)
