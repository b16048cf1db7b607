"""Device-resident substreams and the bulk fill / fused-consumer API.

``Substreams`` holds the states of many independent substreams of one
generator on a GPU, in the SoA layout of include/slp_b200.h ((k, ld) words,
flat word order, uint64 for w = 64 and uint32 for w = 32).  Substream i of
block b starts at  base * M^(b * block_stride + i * stride)  — with the
defaults stride = 2^(n/2) (``jump()``) and block_stride = 2^(3n/4)
(``long_jump``), i.e. exactly the states the reference reaches with
``Generator.jump`` / ``compute_jump_poly`` (generators.py:315-334, :397-419)
and ``LanedStream`` lane set-up (:435-463).

Everything here runs through the C ABI (kernels K1, K2/K3, K4); torch only
supplies device memory and the current CUDA stream.  There is no CPU path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .generators import Generator, GeneratorSpec, JumpPolynomial, compute_jump_poly, native_id

__all__ = ["Substreams", "Checksum", "fill", "fused_checksum", "require_cuda"]

_KIND = {"native": _native.OUT_NATIVE, "u64": _native.OUT_U64, "f64": _native.OUT_F64, "f32": _native.OUT_F32}
_LAYOUT = {"stream": _native.STREAM_MAJOR, "position": _native.POSITION_MAJOR}


def require_cuda(device=None) -> torch.device:
    """The CUDA device to use; raises if there is none (no CPU fallback)."""
    _native.lib()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1805_01407_b200 bulk generation requires a CUDA device (sm_100a); none found")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def _stream_ptr(dev: torch.device):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _word_dtype(w: int):
    return torch.uint64 if w == 64 else torch.uint32


def _out_dtype(spec: GeneratorSpec, kind: str):
    w = spec.kind.w
    if kind == "native":
        return _word_dtype(w)
    if kind == "u64":
        return torch.uint64
    if kind == "f64":
        if w != 64:
            raise ValueError("f64 output requires a 64-bit generator (generators.py:309-310)")
        return torch.float64
    if kind == "f32":
        if w != 32:
            raise ValueError("f32 output (x >> 8) * 2^-24 is defined for 32-bit generators")
        return torch.float32
    raise ValueError(f"unknown output kind {kind!r}")


@dataclass(frozen=True)
class Checksum:
    """Exact reduction of a set of outputs (see slp_checksum in include/slp_b200.h)."""

    w: int
    sum: int                # wrapping sum mod 2^64
    sum_exact: int | None   # exact integer sum (exact mode)
    xor: int
    mant: int | None        # exact sum of (x >> 11) (w=64) / (x >> 8) (w=32) (exact mode)
    count: int
    fsum_f64: float | None  # float64 accumulation in the kernel (summation order differs)

    @property
    def fsum(self) -> float | None:
        """mant * 2^-53 (w=64) / 2^-24 (w=32), correctly rounded once."""
        from fractions import Fraction

        if self.mant is None:
            return None
        return float(Fraction(self.mant, 1 << (53 if self.w == 64 else 24)))

    @classmethod
    def from_raw(cls, raw: _native.Checksum, w: int, exact: bool, with_f64: bool):
        shift = 11 if w == 64 else 8
        if exact:
            tot = (int(raw.sum_hi) << 64) | int(raw.sum_lo)
            mant = (tot - int(raw.low_sum)) >> shift
        else:
            tot = mant = None
        return cls(w, int(raw.sum_lo), tot, int(raw.xor_all), mant, int(raw.count),
                   float(raw.fsum) if with_f64 else None)

    @classmethod
    def fold(cls, parts):
        """Combine checksums of disjoint output sets (order-independent, exact)."""
        parts = list(parts)
        w = parts[0].w
        x = 0
        for p in parts:
            x ^= p.xor
        exact = mant = None
        if all(p.sum_exact is not None for p in parts):
            exact = sum(p.sum_exact for p in parts)
            mant = sum(p.mant for p in parts)
        f64 = None
        if all(p.fsum_f64 is not None for p in parts):
            f64 = float(sum(p.fsum_f64 for p in parts))
        return cls(w, sum(p.sum for p in parts) & ((1 << 64) - 1), exact, x, mant,
                   sum(p.count for p in parts), f64)


def fill(spec: GeneratorSpec, states: torch.Tensor, T: int, *, out: torch.Tensor | None = None,
         kind: str = "native", layout: str = "stream", nstreams: int | None = None,
         states_out: torch.Tensor | None = None, advance: bool = True) -> torch.Tensor:
    """Kernel K2/K3: T outputs of each substream whose SoA states are ``states``
    ((k, ld) words).  Returns ``out`` of shape (nstreams, T) (stream-major) or
    (T, nstreams) (position-major).  States advance in place unless
    ``advance=False`` or ``states_out`` is given."""
    gid = native_id(spec)
    k = spec.kind.k
    if states.dim() != 2 or states.shape[0] != k or states.dtype != _word_dtype(spec.kind.w) or not states.is_cuda:
        raise ValueError(f"states must be a CUDA ({k}, ld) {_word_dtype(spec.kind.w)} tensor")
    if states.stride(1) != 1 or (k > 1 and states.stride(0) < states.shape[1]):
        raise ValueError("states must have unit column stride (a column slice of a (k, ld) tensor)")
    ld = states.stride(0) if k > 1 else states.shape[1]
    n = states.shape[1] if nstreams is None else int(nstreams)
    if T < 0 or n < 0 or n > states.shape[1]:
        raise ValueError("bad T / nstreams")
    dt = _out_dtype(spec, kind)
    if layout not in _LAYOUT:
        raise ValueError(f"unknown layout {layout!r}")
    shape = (n, T) if layout == "stream" else (T, n)
    if out is None:
        out = torch.empty(shape, dtype=dt, device=states.device)
    elif out.dtype != dt or out.device != states.device or out.dim() != 2 or out.stride(1) != 1 \
            or tuple(out.shape) != shape:
        raise ValueError(f"out must be a {shape} {dt} tensor on {states.device} with unit inner stride")
    ld_out = out.stride(0) if out.shape[0] > 1 else shape[1]
    if states_out is None:
        sout = states.data_ptr() if advance else None
    else:
        if states_out.shape != states.shape or states_out.dtype != states.dtype \
                or states_out.stride() != states.stride():
            raise ValueError("states_out must match states (shape, dtype, strides)")
        sout = states_out.data_ptr()
    L = _native.lib()
    with torch.cuda.device(states.device):
        rc = L.slp_fill(gid, ctypes.c_void_p(states.data_ptr()), ctypes.c_void_p(sout), ld, n, T,
                        _KIND[kind], _LAYOUT[layout], ctypes.c_void_p(out.data_ptr()), ld_out,
                        _stream_ptr(states.device))
    _native.check(rc, "fill")
    return out


def set_fill_pace(gbps: int | None) -> int:
    """Store pacing of the fill kernels (C ABI ``slp_set_fill_pace``): their
    tile stores are offered at no more than ``gbps`` GB/s in aggregate, which
    HBM absorbs faster than an unpaced stream.  0 turns pacing
    off, None only queries.  Returns the previous target.  Results never
    depend on it."""
    return int(_native.lib().slp_set_fill_pace(-1 if gbps is None else int(gbps)))


def _split_factor(spec: GeneratorSpec, n: int, T: int, layout: str, ld_out: int, es: int | None = None) -> int:
    """Segments per substream the C ABI uses internally for few, long
    substreams (slp_split_factor): contiguous and padded stream-major rows
    (padded: 16-byte row pitch and segment length) and position-major."""
    J = int(_native.lib().slp_split_factor(native_id(spec), n, T))
    if J > 1 and layout == "stream" and ld_out != T:
        es = es or spec.kind.w // 8
        if (ld_out * es) % 16 or ((T // J) * es) % 16:
            return 1
    return J


_ws_bytes: dict = {}


def _workspace(gid: int, dev: torch.device) -> torch.Tensor:
    """Per-call scratch for the per-CTA partials (tens of KB).  Allocated from
    torch's stream-ordered caching allocator on every call, so concurrent
    checksums on different streams never share partials."""
    key = (gid, dev.index)
    nbytes = _ws_bytes.get(key)
    if nbytes is None:
        with torch.cuda.device(dev):
            nbytes = max(int(_native.lib().slp_fused_workspace_bytes(gid, 0)), 64)
        _ws_bytes[key] = nbytes
    return torch.empty(nbytes, dtype=torch.uint8, device=dev)


def fused_checksum_async(spec: GeneratorSpec, states: torch.Tensor, T: int, *, exact: bool = True,
                         f64: bool = False, nstreams: int | None = None, advance: bool = True,
                         result: torch.Tensor | None = None) -> torch.Tensor:
    """Kernel K4: reduce T outputs of each substream in-kernel; returns the
    48-byte slp_checksum as a uint8 CUDA tensor (no host synchronisation)."""
    gid = native_id(spec)
    if states.dim() != 2 or states.dtype != _word_dtype(spec.kind.w) or not states.is_cuda \
            or states.shape[0] != spec.kind.k or states.stride(1) != 1:
        raise ValueError(f"states must be a CUDA ({spec.kind.k}, ld) {_word_dtype(spec.kind.w)} tensor "
                         "with unit column stride")
    ld = states.stride(0) if spec.kind.k > 1 else states.shape[1]
    n = states.shape[1] if nstreams is None else int(nstreams)
    if n < 0 or n > states.shape[1]:
        raise ValueError("bad nstreams")
    dev = states.device
    ws = _workspace(gid, dev)
    if result is None:
        result = torch.empty(_native.CHECKSUM_BYTES, dtype=torch.uint8, device=dev)
    flags = _native.FUSE_INT | (_native.FUSE_EXACT if exact else 0) | (_native.FUSE_F64 if f64 else 0)
    L = _native.lib()
    with torch.cuda.device(dev):
        rc = L.slp_fused(gid, ctypes.c_void_p(states.data_ptr()),
                         ctypes.c_void_p(states.data_ptr() if advance else None), ld, n, T, flags,
                         ctypes.c_void_p(result.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                         _stream_ptr(dev))
    _native.check(rc, "fused")
    return result


def fill_checksum(spec: GeneratorSpec, states: torch.Tensor, T: int, *, out: torch.Tensor | None = None,
                  kind: str = "native") -> tuple[torch.Tensor, Checksum]:
    """Store AND checksum in one pass (stream-major): returns (out, Checksum of
    the integer outputs, exact mode).  States advance in place.  When the
    output cannot take the TMA path, runs K4 on a copy of the states, then K2."""
    gid = native_id(spec)
    k = spec.kind.k
    if states.dim() != 2 or states.shape[0] != k or not states.is_cuda or states.dtype != _word_dtype(spec.kind.w) \
            or not states.is_contiguous():
        raise ValueError(f"states must be a contiguous CUDA ({k}, n) {_word_dtype(spec.kind.w)} tensor")
    n = states.shape[1]
    dt = _out_dtype(spec, kind)
    if out is None:
        out = torch.empty((n, T), dtype=dt, device=states.device)
    elif tuple(out.shape) != (n, T) or out.dtype != dt or out.stride(1) != 1 or out.device != states.device:
        raise ValueError(f"out must be a ({n}, {T}) {dt} tensor with unit inner stride")
    dev = states.device
    ws = _workspace(gid, dev)
    res = torch.empty(_native.CHECKSUM_BYTES, dtype=torch.uint8, device=dev)
    ld_out = out.stride(0) if n > 1 else T
    with torch.cuda.device(dev):
        rc = _native.lib().slp_fill_checksum(gid, ctypes.c_void_p(states.data_ptr()),
                                             ctypes.c_void_p(states.data_ptr()), n, n, T, _KIND[kind],
                                             ctypes.c_void_p(out.data_ptr()), ld_out,
                                             ctypes.c_void_p(res.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                             ws.numel(), _stream_ptr(dev))
    if rc == _native.SLP_ERR_UNSUPPORTED:
        c = fused_checksum(spec, states, T, exact=True, advance=False)
        fill(spec, states, T, out=out, kind=kind)
        return out, c
    _native.check(rc, "fill_checksum")
    return out, decode_checksum(res, spec.kind.w, True, False)


def decode_checksum(raw: torch.Tensor | bytes, w: int, exact: bool = True, f64: bool = False) -> Checksum:
    b = bytes(raw.cpu().numpy().tobytes()) if isinstance(raw, torch.Tensor) else bytes(raw)
    return Checksum.from_raw(_native.Checksum.from_buffer_copy(b), w, exact or f64, f64)


def fused_checksum(spec: GeneratorSpec, states: torch.Tensor, T: int, *, exact: bool = True, f64: bool = False,
                   nstreams: int | None = None, advance: bool = True) -> Checksum:
    raw = fused_checksum_async(spec, states, T, exact=exact, f64=f64, nstreams=nstreams, advance=advance)
    return decode_checksum(raw, spec.kind.w, exact, f64)


def fill_to_host(spec: GeneratorSpec, states: torch.Tensor, T: int, host_out: torch.Tensor, *,
                 kind: str = "native", slice_streams: int = 1 << 15, _bufs: list | None = None) -> torch.Tensor:
    """Stream-major fill delivered to HOST memory: the GPU generates slices of
    ``slice_streams`` substreams into two device buffers while a copy stream
    moves the previous slice to ``host_out`` (pinned (n, T) tensor), so the
    device-to-host copy overlaps generation.  States advance in place."""
    n = states.shape[1]
    dev = states.device
    if tuple(host_out.shape) != (n, T) or host_out.device.type != "cpu":
        raise ValueError(f"host_out must be a ({n}, {T}) CPU tensor")
    dt = _out_dtype(spec, kind)
    if host_out.dtype != dt:
        raise ValueError(f"host_out dtype must be {dt}")
    sl = max(1, min(slice_streams, n))
    bufs = _bufs if _bufs is not None else [torch.empty((sl, T), dtype=dt, device=dev) for _ in range(2)]
    nb = len(bufs)
    compute = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    done = [None] * nb
    for i, a in enumerate(range(0, n, sl)):
        b = min(n, a + sl)
        buf = bufs[i % nb][: b - a]
        if done[i % nb] is not None:
            compute.wait_event(done[i % nb])
        fill(spec, states[:, a:b], T, out=buf, kind=kind)
        ready = torch.cuda.Event()
        ready.record(compute)
        with torch.cuda.stream(copy):
            copy.wait_event(ready)
            host_out[a:b].copy_(buf, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
        done[i % nb] = ev
    compute.wait_stream(copy)
    return host_out


class Substreams:
    """States of ``blocks x n`` substreams of one generator, resident on a GPU."""

    def __init__(self, spec: GeneratorSpec, states: torch.Tensor, n: int, blocks: int = 1):
        self.spec = spec
        self.states = states
        self.n = n
        self.blocks = blocks
        self.gid = native_id(spec)

    @property
    def count(self) -> int:
        return self.n * self.blocks

    @property
    def device(self) -> torch.device:
        return self.states.device

    @classmethod
    def from_generator(cls, generator: Generator, n: int, *, stride: int | None = None, blocks: int = 1,
                       block_stride: int | None = None, first_block: int = 0, base_offset: int = 0,
                       device=None) -> "Substreams":
        """Substream i of block b = generator jumped by
        base_offset + (first_block + b) * block_stride + i * stride  (kernel K1)."""
        spec = generator.spec
        gid = native_id(spec)
        dev = require_cuda(device)
        nbits = spec.kind.n
        stride = (1 << (nbits // 2)) if stride is None else int(stride)
        block_stride = (1 << (3 * nbits // 4)) if block_stride is None else int(block_stride)
        if n < 1 or blocks < 1 or stride < 0 or block_stride < 0 or base_offset < 0 or first_block < 0:
            raise ValueError("bad substream geometry")
        k = spec.kind.k
        # block bases on the host: one jump to the first block, then one cached
        # block_stride jump per further block (native scalar jumps, microseconds)
        g = generator.clone()
        off0 = base_offset + first_block * block_stride
        if off0:
            g.jump(compute_jump_poly(spec, off0))
        step = compute_jump_poly(spec, block_stride) if blocks > 1 and block_stride else None
        bases = []
        for b in range(blocks):
            if b and step is not None:
                g.jump(step)
            bases.extend(g.flat_words())
        base = (ctypes.c_uint64 * len(bases))(*bases)
        sw, sn = _native.int_to_words(stride)
        states = torch.empty((k, n * blocks), dtype=_word_dtype(spec.kind.w), device=dev)
        with torch.cuda.device(dev):
            rc = _native.lib().slp_init_substreams(gid, base, blocks, sw, sn, ctypes.c_void_p(states.data_ptr()),
                                                   n * blocks, n, _stream_ptr(dev))
        _native.check(rc, "init_substreams")
        return cls(spec, states, n, blocks)

    @classmethod
    def from_seed(cls, spec: GeneratorSpec, seed: int, n: int, **kw) -> "Substreams":
        return cls.from_generator(Generator.from_seed(spec, seed), n, **kw)

    @classmethod
    def from_states(cls, spec: GeneratorSpec, flat: np.ndarray, device=None) -> "Substreams":
        """Upload explicit flat states, a (k, L) integer array."""
        dev = require_cuda(device)
        flat = np.asarray(flat)
        if flat.ndim != 2 or flat.shape[0] != spec.kind.k:
            raise ValueError("flat states must have shape (k, L)")
        npdt = np.uint64 if spec.kind.w == 64 else np.uint32
        t = torch.from_numpy(np.ascontiguousarray(flat.astype(npdt))).to(dev)
        return cls(spec, t, flat.shape[1], 1)

    def states_numpy(self) -> np.ndarray:
        return self.states.cpu().numpy()

    def fill(self, T: int, *, out=None, kind: str = "native", layout: str = "stream", advance: bool = True):
        return fill(self.spec, self.states, T, out=out, kind=kind, layout=layout, advance=advance)

    def checksum(self, T: int, *, exact: bool = True, f64: bool = False, advance: bool = True) -> Checksum:
        return fused_checksum(self.spec, self.states, T, exact=exact, f64=f64, advance=advance)

    def checksum_async(self, T: int, *, exact: bool = True, f64: bool = False, advance: bool = True,
                       result=None) -> torch.Tensor:
        return fused_checksum_async(self.spec, self.states, T, exact=exact, f64=f64, advance=advance,
                                    result=result)

    def jump(self, jp: JumpPolynomial) -> "Substreams":
        """Advance every substream by jp.step_count steps (kernel K1, in place)."""
        if jp.engine_key != self.spec.engine_key:
            raise ValueError("jump polynomial was built for a different engine")
        if jp.poly.bits == 0:
            raise ValueError("jump polynomial is zero")
        pw, pn = _native.int_to_words(jp.poly.bits)
        ptr = ctypes.c_void_p(self.states.data_ptr())
        ld = self.states.stride(0)
        with torch.cuda.device(self.device):
            if self.spec.kind.n > 256 and self.count >= (1 << 16):
                # out of place, so the table-driven kernel K1t can run (its
                # wide-engine slices cannot update in place), then copy back
                tmp = torch.empty((self.spec.kind.k, self.count), dtype=self.states.dtype, device=self.device)
                rc = _native.lib().slp_jump_states(self.gid, pw, pn, ptr, ld, ctypes.c_void_p(tmp.data_ptr()),
                                                   self.count, self.count, _stream_ptr(self.device))
                _native.check(rc, "jump_states")
                self.states[:, : self.count].copy_(tmp)
                return self
            rc = _native.lib().slp_jump_states(self.gid, pw, pn, ptr, ld, ptr, ld, self.count,
                                               _stream_ptr(self.device))
        _native.check(rc, "jump_states")
        return self


class VecStepper:
    """Device counterpart of the reference's numpy lane stepper
    (engines.py:276-361): advances many states of one engine in lockstep.

    ``S`` is a CUDA (k, L) tensor of native words (uint64 for w = 64, uint32
    for w = 32) in flat word order; unlike the reference, the ring engines are
    stored physically in flat order, so ``word(S, i)`` is ``S[i]`` and no
    rolling offset is kept.  ``step`` runs one engine step (kernel K2 with
    T = 1 into a scratch row); ``advance(S, steps)`` jumps by any number of
    steps (kernel K1)."""

    def __init__(self, kind, params):
        from .engines import check_params
        from .generators import _TABLE
        from .scramblers import ScramblerSpec

        if kind.w not in (32, 64):  # engines.py:291-292
            raise ValueError("vector stepping supports w in {32, 64} only")
        check_params(kind, params)
        match = [s for s in _TABLE if s.kind == kind and s.params == params]
        # any other engine (custom_spec) runs on the run-time parameter kernels
        self.spec = match[0] if match else GeneratorSpec(f"{kind.family}{kind.n}-vec", kind, params,
                                                           ScramblerSpec("none", 0))
        self.kind = kind
        self.params = params
        self.off = 0
        self._scratch = None

    def _check(self, S):
        if not isinstance(S, torch.Tensor) or not S.is_cuda:
            raise TypeError("device VecStepper states must be a CUDA tensor (k, L)")
        if S.dim() != 2 or S.shape[0] != self.kind.k or S.dtype != _word_dtype(self.kind.w):
            raise ValueError(f"states must be ({self.kind.k}, L) {_word_dtype(self.kind.w)}")

    def word(self, S, i: int):
        return S[i]  # flat order is physical: no rolling offset (engines.py:302-303)

    def flat(self, S):
        return S

    def set_flat(self, S, flat):
        if isinstance(S, np.ndarray):
            S[...] = np.asarray(flat, dtype=S.dtype)
        else:
            S.copy_(flat)
        self.off = 0

    def _host(self, S, op):
        """The reference's numpy (k, L) uint64 arrays (engines.py:276-283):
        run ``op`` on a device copy and write the result back in place."""
        dt = _word_dtype(self.kind.w)
        if S.ndim != 2 or S.shape[0] != self.kind.k:
            raise ValueError(f"states must be a ({self.kind.k}, L) array")
        D = torch.from_numpy(np.ascontiguousarray(S).astype(np.uint64 if dt == torch.uint64 else np.uint32))
        D = D.to(require_cuda())
        op(D)
        S[...] = D.cpu().numpy().astype(S.dtype, copy=False)

    def step(self, S):
        if isinstance(S, np.ndarray):
            return self._host(S, self.step)
        self._check(S)
        L = S.shape[1]
        if self._scratch is None or self._scratch.shape[1] < L or self._scratch.device != S.device:
            self._scratch = torch.empty((1, L), dtype=S.dtype, device=S.device)
        if S.is_contiguous():
            fill(self.spec, S, 1, out=self._scratch[:, :L], layout="position")
        else:  # K2 needs unit column stride: step a contiguous copy, then write it back
            C = S.contiguous()
            fill(self.spec, C, 1, out=self._scratch[:, :L], layout="position")
            S.copy_(C)

    def advance(self, S, steps: int):
        if isinstance(S, np.ndarray):
            return self._host(S, lambda D: self.advance(D, steps))
        self._check(S)
        if steps == 0:
            return
        jp = compute_jump_poly(self.spec, steps)
        pw, pn = _native.int_to_words(jp.poly.bits)
        if S.stride(1) != 1:
            C = S.contiguous()
            self.advance(C, steps)
            S.copy_(C)
            return
        ptr = ctypes.c_void_p(S.data_ptr())
        L = S.shape[1]
        ld = S.stride(0) if S.shape[0] > 1 else L
        with torch.cuda.device(S.device):
            rc = _native.lib().slp_jump_states(native_id(self.spec), pw, pn, ptr, ld, ptr, ld, L,
                                               _stream_ptr(S.device))
        _native.check(rc, "advance")
