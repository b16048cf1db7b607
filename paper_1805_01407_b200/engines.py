"""Engine kinds, parameters and the scalar flat-view step.

Mirrors the public surface of the reference module
(/root/reference/pkg/src/slprng/engines.py): ``EngineKind`` / ``EngineParams``
(:43-77), ``rotl`` (:80-86), ``step`` (:100-140) and the bit-vector helpers
(:143-152).  This is host-side scalar code (setup, single generators, tests);
bulk stepping runs on the GPU (``device.py``).

Flat view (engines.py:14-18): word j occupies bits [j*w, (j+1)*w) of the
state vector; for the ring xoroshiro engines flat word 0 is the word the
next step reads first and flat word k-1 the one it reads second.
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["EngineKind", "EngineParams", "rotl", "step", "state_to_bits", "bits_to_words",
           "check_params", "FAMILIES", "VecStepper"]


def __getattr__(name):
    # engines.VecStepper (engines.py:276-361): the device-backed lane stepper
    # of device.py, imported lazily (device.py imports torch and this module)
    if name == "VecStepper":
        from .device import VecStepper

        return VecStepper
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")

FAMILIES = ("xoroshiro", "xoshiro", "xorshift")
FAMILY_CODE = {"xoroshiro": 0, "xoshiro": 1, "xorshift": 2}


@dataclass(frozen=True)
class EngineParams:
    a: int
    b: int
    c: int | None = None

    def __post_init__(self):
        for label in ("a", "b", "c"):
            v = getattr(self, label)
            if v is not None and not isinstance(v, int):
                raise TypeError(f"parameter {label} must be an int, got {type(v).__name__}")


@dataclass(frozen=True)
class EngineKind:
    family: str
    k: int
    w: int

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ValueError(f"unknown engine family {self.family!r}")
        if self.family == "xoshiro" and self.k not in (4, 8):
            raise ValueError("xoshiro is defined only for k in {4, 8}")
        if self.family == "xoroshiro" and self.k < 2:
            raise ValueError("xoroshiro requires k >= 2")
        if self.family == "xorshift" and self.k != 2:
            raise ValueError("only the two-word xorshift is supported")
        if self.w < 2:
            raise ValueError("word size must be >= 2")

    @property
    def n(self) -> int:
        """State size in bits."""
        return self.k * self.w


def rotl(x: int, r: int, w: int) -> int:
    if r < 0 or r >= w:
        raise ValueError(f"rotation {r} out of range for w={w}")
    m = (1 << w) - 1
    return ((x << r) | (x >> (w - r))) & m if r else x


def check_params(kind: EngineKind, params: EngineParams):
    """Parameter ranges of engines.py:89-97."""
    needs_c = kind.family != "xoshiro"
    if needs_c and params.c is None:
        raise ValueError(f"{kind.family} needs three parameters")
    names = ("a", "b", "c") if needs_c else ("a", "b")
    for label in names:
        v = getattr(params, label)
        if not 0 < v < kind.w:
            raise ValueError(f"parameter {label}={v} out of range for w={kind.w}")


def step(kind: EngineKind, params: EngineParams, words: tuple) -> tuple:
    """One engine step on a flat state (pure function; engines.py:100-140)."""
    w = kind.w
    m = (1 << w) - 1
    a, b, c = params.a, params.b, params.c

    def rl(x, r):
        return ((x << r) | (x >> (w - r))) & m

    fam = kind.family
    if fam == "xoroshiro":
        first = words[0]
        last = words[-1] ^ first
        hi = rl(first, a) ^ last ^ ((last << b) & m)
        lo = rl(last, c)
        return tuple(words[1:-1]) + (hi, lo)
    if fam == "xorshift":
        s0, s1 = words
        t = s0 ^ ((s0 << a) & m)
        return (s1, t ^ (t >> b) ^ s1 ^ (s1 >> c))
    s = list(words)
    t = (s[1] << a) & m
    if kind.k == 4:
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = rl(s[3], b)
    else:
        s[2] ^= s[0]
        s[5] ^= s[1]
        s[1] ^= s[2]
        s[7] ^= s[3]
        s[3] ^= s[4]
        s[4] ^= s[5]
        s[0] ^= s[6]
        s[6] ^= s[7]
        s[6] ^= t
        s[7] = rl(s[7], b)
    return tuple(s)


def state_to_bits(words, w: int) -> int:
    v = 0
    for j, x in enumerate(words):
        v |= int(x) << (j * w)
    return v


def bits_to_words(v: int, k: int, w: int) -> tuple:
    m = (1 << w) - 1
    return tuple((v >> (j * w)) & m for j in range(k))
