"""Orbit partitioning across GPUs (one process per GPU, torch.distributed).

The reference's only decomposition is "clone + jump to partition the orbit"
(generators.py:189-190; default long jump 2^(3n/4), :408-419).  Config 5
(BASELINE.json) splits 2^34 outputs into ``nblocks`` long-jump blocks x ``S``
substreams (jump 2^(n/2)) x ``T`` outputs; GPU g of G takes the blocks
b == g (mod G), so the set of outputs -- and therefore the checksum -- does
not depend on G.  The data path needs no collective; the per-GPU checksums
are combined with ONE all_gather of a 64-byte record per rank (NCCL has no
XOR reduction, nccl.h:260-264) and folded in rank order on every rank, which
makes the result exact and identical everywhere.
"""

from __future__ import annotations

import torch

from .generators import GeneratorSpec

__all__ = ["blocks_for_rank", "collective_device", "gather_checksums", "sharded_checksum", "CHECKSUM_WORDS"]

CHECKSUM_WORDS = 8  # words per rank in the all_gather, see _pack()


def blocks_for_rank(rank: int, world: int, nblocks: int) -> list[int]:
    """Long-jump blocks owned by ``rank``: b = rank, rank + world, ..."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return list(range(rank, nblocks, world))


def _pack(c) -> list[int]:
    """Checksum -> 8 uint64 words (sum, exact sum as 2 words, xor, mant as 2 words, count, has_exact)."""
    M = (1 << 64) - 1
    ex = c.sum_exact if c.sum_exact is not None else 0
    mant = c.mant if c.mant is not None else 0
    return [c.sum & M, ex & M, ex >> 64, c.xor, mant & M, mant >> 64, c.count, int(c.sum_exact is not None)]


def _unpack(words, w: int):
    from .device import Checksum

    words = [int(x) & ((1 << 64) - 1) for x in words]
    exact = words[7] == 1
    return Checksum(w, words[0], (words[1] | (words[2] << 64)) if exact else None, words[3],
                    (words[4] | (words[5] << 64)) if exact else None, words[6], None)


def collective_device(group=None, device=None):
    """Device for the all_gather tensors: ``device`` if given, else the current
    CUDA device under NCCL (which rejects CPU tensors), else the CPU (gloo)."""
    import torch.distributed as dist

    if device is not None:
        return torch.device(device)
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def gather_checksums(c, w: int, group=None, device=None):
    """all_gather every rank's Checksum (one collective) and fold in rank order.
    ``device=None`` picks the backend's device (``collective_device``)."""
    import torch.distributed as dist

    from .device import Checksum

    world = dist.get_world_size(group)
    device = collective_device(group, device)
    # reinterpret: values >= 2^63 wrap to negative int64, exact round trip
    mine = torch.tensor([x - (1 << 64) if x >= (1 << 63) else x for x in _pack(c)], dtype=torch.int64,
                        device=device)
    outs = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(outs, mine, group=group)
    parts = [_unpack(o.cpu().tolist(), w) for o in outs]
    return Checksum.fold(parts), parts


def sharded_checksum(spec: GeneratorSpec, seed: int, nblocks: int, S: int, T: int, *, rank: int = 0,
                     world: int = 1, exact: bool = True, group=None, compute=None, device=None):
    """Checksum of config-5 style work: blocks b == rank (mod world), S
    substreams each, T outputs per substream; folded over all ranks.

    ``compute(spec, seed, blocks, S, T) -> Checksum`` defaults to the GPU path
    (kernels K1 + K4); tests pass a CPU oracle instead to exercise the
    multi-rank host logic without a GPU."""
    blocks = blocks_for_rank(rank, world, nblocks)
    if compute is None:
        compute = _device_compute
    local = compute(spec, seed, blocks, S, T, exact=exact)
    if world == 1:
        return local, [local]
    return gather_checksums(local, spec.kind.w, group=group, device=device)


def _device_compute(spec, seed, blocks, S, T, exact=True):
    from .device import Checksum, Substreams
    from .generators import Generator

    if not blocks:
        return Checksum(spec.kind.w, 0, 0 if exact else None, 0, 0 if exact else None, 0, None)
    g = Generator.from_seed(spec, seed)
    lj = 1 << (3 * spec.kind.n // 4)
    stride = blocks[1] - blocks[0] if len(blocks) > 1 else 1
    if any(b1 - b0 != stride for b0, b1 in zip(blocks, blocks[1:])):
        raise ValueError("blocks must be an arithmetic progression")
    # all of this rank's blocks in one K1 init (block i = seed * M^((b0 + i*stride) * 2^(3n/4)))
    # and ONE fused K4 launch over blocks x S substreams
    sub = Substreams.from_generator(g, S, blocks=len(blocks), block_stride=stride * lj,
                                    first_block=0, base_offset=blocks[0] * lj)
    return sub.checksum(T, exact=exact)
