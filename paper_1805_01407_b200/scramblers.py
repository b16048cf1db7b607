"""Output functions (+, *, ++, **) on flat state words.

Mirrors /root/reference/pkg/src/slprng/scramblers.py (``ScramblerSpec``
:48-95 and ``scramble_*`` :26-45).  Scramblers read the state BEFORE the
engine step; for ``++`` the first word is the one added back.  The device
kernels implement the same functions in registers (csrc/slp_gen.cuh,
``Gen::output``).
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["ScramblerSpec", "scramble_plus", "scramble_star", "scramble_plusplus",
           "scramble_starstar", "SCRAMBLER_KINDS", "SCRAMBLER_CODE"]

SCRAMBLER_KINDS = ("none", "plus", "star", "plusplus", "starstar")
SCRAMBLER_CODE = {k: i for i, k in enumerate(SCRAMBLER_KINDS)}


def _mask(w):
    return (1 << w) - 1


def scramble_plus(x: int, y: int, w: int) -> int:
    return (x + y) & _mask(w)


def scramble_star(x: int, s: int, w: int) -> int:
    return (x * s) & _mask(w)


def _rl(x, r, w):
    return ((x << r) | (x >> (w - r))) & _mask(w)


def scramble_plusplus(x: int, y: int, r: int, w: int) -> int:
    return (_rl((x + y) & _mask(w), r, w) + x) & _mask(w)


def scramble_starstar(x: int, s: int, r: int, t: int, w: int) -> int:
    return (_rl((x * s) & _mask(w), r, w) * t) & _mask(w)


@dataclass(frozen=True)
class ScramblerSpec:
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
        """Range checks of scramblers.py:68-82."""
        if not 0 <= self.word_i < k:
            raise ValueError("word_i out of range")
        if self.kind in ("plus", "plusplus") and (self.word_j is None or not 0 <= self.word_j < k):
            raise ValueError("word_j out of range")
        if self.kind in ("star", "starstar") and (self.S is None or self.S % 2 == 0):
            raise ValueError("multiplier S must be odd")
        if self.kind in ("plusplus", "starstar") and (self.R is None or not 0 < self.R < w):
            raise ValueError("rotation R out of range")
        if self.kind == "starstar" and (self.T is None or self.T % 2 == 0):
            raise ValueError("multiplier T must be odd")

    def apply(self, words, w: int) -> int:
        x = words[self.word_i]
        kind = self.kind
        if kind == "none":
            return x
        if kind == "plus":
            return scramble_plus(x, words[self.word_j], w)
        if kind == "star":
            return scramble_star(x, self.S, w)
        if kind == "plusplus":
            return scramble_plusplus(x, words[self.word_j], self.R, w)
        return scramble_starstar(x, self.S, self.R, self.T, w)
