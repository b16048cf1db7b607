"""B200-native bulk generator for the scrambled linear pseudorandom
generators of Blackman & Vigna (arXiv 1805.01407).

Drop-in for the hot path of the reference package ``slprng``
(/root/reference/pkg/src/slprng/__init__.py:4-43): the same registry, seeding,
scalar Generator and jump API, with the bulk path (``LanedStream``,
``output_stream``) and the new device API (``Substreams``, ``fill``,
``fused_checksum``) running on hand-written sm_100a CUDA kernels behind the C
ABI of include/slp_b200.h.
"""

from .engines import EngineKind, EngineParams, bits_to_words, rotl, state_to_bits, step
from .generators import (
    ANALYSIS_REGISTRY,
    REGISTRY,
    Generator,
    GeneratorSpec,
    JumpPolynomial,
    LanedStream,
    compute_jump_poly,
    custom_spec,
    default_jumps,
    engine_char_poly,
    get_spec,
    output_stream,
    registry_names,
    seed_state,
    splitmix64,
)
from .gf2 import GF2Poly, Gf2Error, poly_mod_mul, poly_mod_pow, poly_weight
from .scramblers import ScramblerSpec, scramble_plus, scramble_plusplus, scramble_star, scramble_starstar

__version__ = "0.1.0"


def __getattr__(name):
    # the device API imports torch; load it lazily
    if name in ("Substreams", "Checksum", "fill", "fused_checksum", "device"):
        import importlib

        _d = importlib.import_module(__name__ + ".device")
        return _d if name == "device" else getattr(_d, name)
    # the reference re-exports these from hwd (__init__.py:36); HwdCounters and
    # batch_size size the reference's packed host counters, which the exact
    # GPU counters of kernel K6 do not need
    if name in ("hwd", "HwdConfig", "HwdReport", "choose_ell"):
        import importlib

        _h = importlib.import_module(__name__ + ".hwd")
        return _h if name == "hwd" else getattr(_h, name)
    raise AttributeError(name)
