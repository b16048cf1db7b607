"""The Hamming-weight dependency (HWD) test with a GPU counting consumer.

Drop-in for the generator-driven entry point of the reference test
(/root/reference/pkg/src/slprng/hwd.py): ``run_generator`` streams the
generator's single output stream straight into kernel K6 (generate ->
test value -> popcount -> trit -> signature -> per-signature count and
weight sum, csrc/slp_hwd.cuh) without ever storing the outputs, and
evaluates at every doubling of consumed values exactly like ``run``
(hwd.py:516-595).  The evaluation (Kronecker-power transform, erfc p-values,
category compensation) is host code restating hwd.py:101-132 and :260-326
operation for operation, so equal counts give bit-identical p-values.

Counters are exact 64-bit totals; the reference's packed small counters
(13-bit count / 19-bit sum, hwd.py:167-247) agree with them whenever they did
not overflow, which its batch sizing makes an event of probability <= 1e-100
(it then reports a forced failure).  This module therefore never reports an
overflow and needs no batch sizing.
"""

from __future__ import annotations

import ctypes
import math
import os
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .generators import Generator, compute_jump_poly, get_spec, native_id

__all__ = ["HwdConfig", "HwdCheckpoint", "HwdReport", "choose_ell", "central_probability", "trit_of",
           "signature_update", "format_signature", "transform", "evaluate_counts", "run_generator"]

FIXED_POINT_RECIP = 0x55555556  # ceil(2**32 / 3)
_R2, _R3, _R6 = math.sqrt(2.0), math.sqrt(3.0), math.sqrt(6.0)


def choose_ell(w: int) -> int:
    """Largest ell whose 2*ell+1 central weights hold probability <= 1/2 (hwd.py:51-68)."""
    if w < 2 or w % 2:
        raise ValueError("value width must be even and >= 2")
    half, total = w // 2, 1 << w
    mass = math.comb(w, half)
    ell = 0
    while ell + 1 <= half:
        grown = mass + math.comb(w, half - ell - 1) + math.comb(w, half + ell + 1)
        if 2 * grown > total:
            break
        mass = grown
        ell += 1
    if 2 * mass > total:
        raise ValueError(f"no valid ell for w={w}")
    return ell


def central_probability(w: int, ell: int) -> float:
    half = w // 2
    return sum(math.comb(w, i) for i in range(half - ell, half + ell + 1)) / float(1 << w)


def trit_of(x: int, w: int, ell: int) -> int:
    nu = int(x).bit_count()
    return 0 if nu < w // 2 - ell else (1 if nu <= w // 2 + ell else 2)


def signature_update(s: int, t: int, k: int) -> int:
    """floor(s / 3) + t * 3**(k-1) with the fixed-point division of hwd.py:84-91."""
    return ((FIXED_POINT_RECIP * s) >> 32) + t * 3 ** (k - 1)


def format_signature(index: int, k: int) -> str:
    out = []
    for _ in range(k):
        out.append(str(index % 3))
        index //= 3
    return "".join(out)


def transform(v: np.ndarray) -> np.ndarray:
    """In-place k-th Kronecker power of the orthogonal 3x3 base (hwd.py:101-126)."""
    n = v.shape[0]
    m = n
    while m > 1:
        if m % 3:
            raise ValueError("length must be a power of 3")
        m //= 3
    stride = n // 3
    while stride >= 1:
        blk = v.reshape(-1, 3, stride)
        a, b, c = blk[:, 0].copy(), blk[:, 1].copy(), blk[:, 2].copy()
        blk[:, 0] = (a + b + c) / _R3
        blk[:, 1] = (a - c) / _R2
        blk[:, 2] = (2 * b - a - c) / _R6
        stride //= 3
    return v


@dataclass
class HwdConfig:
    """Test parameters (hwd.py:133-166).  ``batch_size`` is accepted for
    compatibility; the GPU counters are exact and need no batching."""

    w: int = 64
    k: int = 8
    ell: int | None = None
    C: int | None = None
    batch_size: int | None = None
    p_threshold: float = 1e-20
    byte_limit: int = 10**15
    mode: str = "standard"
    split: bool = False

    def __post_init__(self):
        if not 1 <= self.k <= 16:
            raise ValueError("k must be in 1..16 (3**k counters must fit in memory)")
        if self.mode not in ("standard", "transitional"):
            raise ValueError("mode must be 'standard' or 'transitional'")
        if self.ell is None:
            self.ell = choose_ell(self.w)
        elif self.ell > self.w // 2:
            raise ValueError("ell must be at most w/2")
        if self.C is None:
            self.C = self.k // 2 + 1
        if not 1 <= self.C <= self.k:
            raise ValueError("C must be in 1..k")
        if self.batch_size is not None:
            if self.batch_size < 1:
                raise ValueError("batch_size must be positive")
            # the reference (hwd.py:167-247, 543-555) flushes 13/19-bit packed
            # counters every batch_size values and reports a forced failure
            # (p = 1e-100, overflow=True) when one overflowed; its default
            # sizing makes that a <= 1e-100 event.  The GPU counters are exact,
            # so a caller-chosen batch size that would overflow there does not
            # fail here.
            warnings.warn("HwdConfig.batch_size is ignored: the GPU counters are exact; the reference's "
                          "per-batch overflow failure (hwd.py:543-555) is not reproduced", RuntimeWarning,
                          stacklevel=3)


@dataclass
class HwdCheckpoint:
    values: int
    bytes: int
    p_value: float
    faulty_signature: str
    faulty_category: int

    def to_dict(self):
        return {"values": self.values, "bytes": self.bytes, "p_value": self.p_value,
                "signature": self.faulty_signature, "category": self.faulty_category}


@dataclass
class HwdReport:
    status: str  # "failed" | "passed" | "inconclusive"
    bytes_processed: int
    values: int
    p_value: float
    faulty_signature: str
    faulty_category: int
    w: int
    k: int
    ell: int
    mode: str
    overflow: bool = False
    history: list = field(default_factory=list)

    def to_dict(self):
        return {"status": self.status, "bytes": self.bytes_processed, "values": self.values,
                "p_value": self.p_value, "signature": self.faulty_signature, "category": self.faulty_category,
                "mode": self.mode, "w": self.w, "k": self.k, "ell": self.ell, "overflow": self.overflow,
                "history": [h.to_dict() for h in self.history]}


_cat_cache: dict = {}


def _categories(k: int, C: int):
    key = (k, C)
    if key not in _cat_cache:
        idx = np.arange(3 ** k)
        nonzero = np.zeros(3 ** k, dtype=np.int64)
        rest = idx.copy()
        for _ in range(k):
            nonzero += (rest % 3) != 0
            rest //= 3
        cats = np.minimum(nonzero, C)
        _cat_cache[key] = tuple(np.nonzero(cats == c)[0] for c in range(C + 1))
    return _cat_cache[key]


def _compensate(p: float, count: int) -> float:
    """1 - (1 - p)^count, in log space."""
    with np.errstate(divide="ignore"):
        return float(-np.expm1(count * np.log1p(-p)))


def evaluate_counts(counts: np.ndarray, sums: np.ndarray, cfg: HwdConfig, values_seen: int) -> HwdCheckpoint:
    """p-value of the per-signature counts / weight sums (hwd.py:297-326)."""
    from scipy.special import erfc

    k, C, w = cfg.k, cfg.C, cfg.w
    cnt = counts.astype(np.float64)
    ws = sums.astype(np.float64)
    v = np.zeros(3 ** k)
    nz = cnt > 0
    v[nz] = (ws[nz] - cnt[nz] * (w / 2.0)) / np.sqrt(cnt[nz] * (w / 4.0))
    transform(v)
    p_elem = erfc(np.abs(v) / _R2)
    cats = _categories(k, C)
    best_comp, best_cat, best_idx = 2.0, 0, 0
    for c in range(1, C + 1):
        idx = cats[c]
        pos = int(np.argmin(p_elem[idx]))
        comp = _compensate(float(p_elem[idx][pos]), idx.size)
        if comp < best_comp:
            best_comp, best_cat, best_idx = comp, c, int(idx[pos])
    return HwdCheckpoint(values=values_seen, bytes=values_seen * (w // 8), p_value=_compensate(best_comp, C),
                         faulty_signature=format_signature(best_idx, k), faulty_category=best_cat)


def _checkpoint_start() -> int:
    env = os.environ.get("SLPRNG_HWD_CHECKPOINT_START")
    return int(float(env)) if env else 10 ** 7


class _GpuCounter:
    """Counts test values at positions [c0, c1) of a generator's stream with kernel K6."""

    TARGET_THREADS = 148 * 2048

    def __init__(self, spec, seed: int, cfg: HwdConfig, device=None):
        import torch

        from .device import require_cuda

        self.torch = torch
        self.dev = require_cuda(device)
        self.spec, self.seed, self.cfg = spec, seed, cfg
        self.gid = native_id(spec)
        self.factor = 2 if cfg.split else 1  # test values per source word
        self.trans = cfg.mode == "transitional"
        n = 3 ** cfg.k
        self.counts = torch.zeros(n, dtype=torch.uint64, device=self.dev)
        self.sums = torch.zeros(n, dtype=torch.uint64, device=self.dev)
        self.overflow = torch.zeros(1, dtype=torch.uint64, device=self.dev)  # CTAs recounted exactly
        self.lo = cfg.w // 2 - cfg.ell
        self.hi = cfg.w // 2 + cfg.ell
        self.dtype = torch.uint64 if spec.kind.w == 64 else torch.uint32

    def _state_at(self, pos_values: int):
        g = Generator.from_seed(self.spec, self.seed)
        src = pos_values // self.factor
        if src:
            g.jump(compute_jump_poly(self.spec, src))
        return list(g.flat_words())

    def count(self, c0: int, c1: int):
        k = self.cfg.k
        W = k + (1 if self.trans else 0)
        if self.factor == 2:
            W += (c0 - W) & 1  # thread starts on source-word boundaries
        # packed 13-bit shared counters: keep the busiest signature (all
        # trits central, probability pc^k) at <= 4096 expected counts per
        # CTA of 256 segments; overflows are recounted exactly in the kernel
        pc = central_probability(self.cfg.w, self.cfg.ell)
        tmax = int(4096 / (256 * pc ** k)) - W
        tmax = max(64, min(tmax, (1 << 16) - 64))
        if self.factor == 2:
            tmax -= tmax & 1
        while c0 < c1:
            L = c1 - c0
            tseg = -(-L // self.TARGET_THREADS)
            tseg = max(64, min(tmax, tseg))
            if self.factor == 2:
                tseg += tseg & 1
            nthreads = min(-(-L // tseg), 1 << 21)
            sub_end = min(c1, c0 + nthreads * tseg)
            self._launch(c0, sub_end, tseg, nthreads, W)
            c0 = sub_end

    def _launch(self, c0, c1, tseg, nthreads, W):
        torch = self.torch
        k_words = self.spec.kind.k
        states = torch.empty((k_words, nthreads), dtype=self.dtype, device=self.dev)
        stream = ctypes.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)
        L = _native.lib()
        S0 = c0 - W
        stride = (tseg // self.factor)
        sw, sn = _native.int_to_words(stride)
        esize = self.spec.kind.w // 8
        if S0 >= 0:
            base = (ctypes.c_uint64 * k_words)(*self._state_at(S0))
            warm0 = W
            first, ptr_off = 0, 0
        else:
            # stream start: thread 0 begins at position 0 (carry 0), the others at S0 + i*tseg
            words = self._state_at(0)
            col0 = torch.tensor(np.array(words, dtype=np.uint64 if esize == 8 else np.uint32).reshape(k_words, 1),
                                device=self.dev)
            states[:, :1].copy_(col0)
            warm0 = c0
            base = (ctypes.c_uint64 * k_words)(*self._state_at(S0 + tseg))
            first, ptr_off = 1, esize
        n_init = nthreads - first
        with torch.cuda.device(self.dev):
            if n_init > 0:
                _native.check(L.slp_init_substreams(self.gid, base, 1, sw, sn,
                                                    ctypes.c_void_p(states.data_ptr() + ptr_off), nthreads,
                                                    n_init, stream), "hwd init")
            _native.check(L.slp_hwd_count(self.gid, ctypes.c_void_p(states.data_ptr()), nthreads, nthreads, tseg,
                                          c1 - c0, W, warm0, self.cfg.k, self.lo, self.hi, int(self.trans),
                                          int(self.factor == 2),
                                          ctypes.cast(self.counts.data_ptr(), _native.u64p),
                                          ctypes.cast(self.sums.data_ptr(), _native.u64p),
                                          ctypes.cast(self.overflow.data_ptr(), _native.u64p), stream), "hwd count")

    def totals(self):
        """(counts, sums) int64 views of the cumulative counters on the device."""
        return self.counts.view(self.torch.int64), self.sums.view(self.torch.int64)

    def snapshot(self):
        return self.counts.cpu().numpy(), self.sums.cpu().numpy()


def _global_totals(counter, group):
    """Counters summed over all ranks (one all-reduce of the 2 x 3^k totals;
    a plain copy on one rank), as numpy uint64 arrays."""
    return _totals_async(counter, group)()


def _totals_async(counter, group):
    """Enqueue a snapshot of the (all-reduced) counters and return a function
    that waits for it.  On the GPU the snapshot is a device copy, the
    all-reduce and an async copy to pinned memory, all ordered on the
    current stream, so counting of the next range can be enqueued before
    the host waits for this one."""
    import torch

    cnt, ws = counter.totals()
    both = torch.cat([cnt, ws])  # a copy: later ranges keep counting into cnt / ws
    if group is not None:
        import torch.distributed as dist

        # torch's NCCL group rejects uint64; the int64 view sums the same bits
        # (two's complement addition is the same modulo 2^64)
        dist.all_reduce(both.view(torch.int64), op=dist.ReduceOp.SUM, group=group)
    n = cnt.numel()
    if not both.is_cuda:
        host = both.numpy().view(np.uint64)
        return lambda: (host[:n], host[n:])
    host = torch.empty(both.shape, dtype=both.dtype, pin_memory=True)
    host.copy_(both, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()

    def wait():
        ev.synchronize()
        h = host.numpy().view(np.uint64)
        return h[:n], h[n:]

    return wait


def run_generator(spec_or_name, config: HwdConfig, seed: int = 1, checkpoint_start: int | None = None,
                  lanes: int = 4096, lane_len: int = 4096, device=None, group=None,
                  _counter_cls=None) -> HwdReport:
    """Run the HWD test on a named generator (hwd.py:598-621) with the GPU
    counting consumer.  ``lanes``/``lane_len`` only shape the reference's
    numpy pipeline and do not change the stream; they are accepted and ignored.

    Multi-GPU: with torch.distributed initialised (or ``group`` given), every
    checkpoint range of the stream is split into one contiguous slice per
    rank, each rank counts its slice, and the per-signature counters are
    summed with one all-reduce before each evaluation -- every rank then
    evaluates the same totals and returns the same report."""
    world, rank = 1, 0
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            world, rank = dist.get_world_size(group), dist.get_rank(group)
            if group is None:
                group = dist.group.WORLD
    except ImportError:
        pass
    if world == 1:
        group = None
    spec = get_spec(spec_or_name) if isinstance(spec_or_name, str) else spec_or_name
    src_w = spec.kind.w
    if config.split:
        if src_w != 64 or config.w != 32:
            raise ValueError("split mode expects a 64-bit source and w=32")
    elif src_w != config.w:
        raise ValueError(f"generator emits {src_w}-bit words but config.w={config.w}")
    factor = 2 if config.split else 1
    stream_end = (config.byte_limit // (src_w // 8)) * factor   # test values the source provides
    bpv = config.w // 8
    value_limit = config.byte_limit // bpv
    next_cp = checkpoint_start if checkpoint_start is not None else _checkpoint_start()
    counter = (_counter_cls or _GpuCounter)(spec, seed, config, device)
    history: list[HwdCheckpoint] = []
    seen = 0

    def count_range(a, b):
        part = -(-(b - a) // world)  # count() accepts any start position (also mid-word in split mode)
        ra, rb = a + rank * part, min(b, a + (rank + 1) * part)
        if rb > ra:
            counter.count(ra, rb)

    def report(status, ck):
        return HwdReport(status=status, bytes_processed=seen * bpv, values=seen,
                         p_value=ck.p_value if ck else 1.0, faulty_signature=ck.faulty_signature if ck else "",
                         faulty_category=ck.faulty_category if ck else 0, w=config.w, k=config.k,
                         ell=config.ell, mode=config.mode, overflow=False, history=history)

    # The checkpoint schedule is fixed in advance (doubling targets, the byte
    # limit, the end of the source); only a failing checkpoint stops early.
    # Counting of range i+1 is enqueued before checkpoint i is evaluated on
    # the host, so evaluations overlap the GPU (a stop discards the extra range).
    pending = []  # (seen, at_cp, at_limit, wait)

    def evaluate(item):
        at_seen, at_cp, at_limit, wait = item
        cnt, ws = wait()
        ck = evaluate_counts(cnt, ws, config, at_seen)
        history.append(ck)
        nonlocal seen
        if ck.p_value < config.p_threshold:
            seen = at_seen
            return report("failed", ck)
        if at_limit:
            seen = at_seen
            return report("passed", ck)
        return None

    while seen < stream_end:
        target = min(next_cp, value_limit, stream_end)
        lo_pos = max(seen, config.k)
        if target > lo_pos:
            count_range(lo_pos, target)
        seen = target
        at_cp, at_limit = seen >= next_cp, seen >= value_limit
        if at_cp:
            next_cp *= 2
        if at_cp or at_limit:
            pending.append((seen, at_cp, at_limit, _totals_async(counter, group)))
        while len(pending) > (0 if at_limit else 1):
            r = evaluate(pending.pop(0))
            if r is not None:
                return r
        if at_limit:
            break
    while pending:
        r = evaluate(pending.pop(0))
        if r is not None:
            return r
    ck = None
    if seen > config.k:
        cnt, ws = _global_totals(counter, group)
        ck = evaluate_counts(cnt, ws, config, seen)
        history.append(ck)
        if ck.p_value < config.p_threshold:
            return report("failed", ck)
    return report("inconclusive", ck)
