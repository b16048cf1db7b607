"""output_stream / LanedStream.chunks host chunks (generators.py:465-513):
chunks arrive by DMA in pooled page-locked buffers handed to the caller and
recycled only when the caller drops them.  Chunks the caller keeps must
never change; the concatenation must stay the reference's stream."""

import gc

import numpy as np
import pytest
import torch

import paper_1805_01407_b200 as P
from paper_1805_01407_b200.generators import _ChunkPool
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def want_stream(name, seed, total, lanes, lane_len):
    return O.laned_stream(name, seed, total, lanes, lane_len)


@pytest.mark.parametrize("name", ["xoshiro256starstar", "xoshiro128plusplus", "xoroshiro1024plus"])
def test_kept_chunks_are_never_overwritten(name):
    spec = P.get_spec(name)
    lanes, lane_len, total = 64, 512, 64 * 512 * 9 + 1000     # 10 chunks, the last one short
    chunks = list(P.output_stream(spec, 3, total, lanes=lanes, lane_len=lane_len))  # caller keeps all
    assert [c.size for c in chunks] == [lanes * lane_len] * 9 + [1000]
    assert all(c.dtype == np.uint64 for c in chunks)
    np.testing.assert_array_equal(np.concatenate(chunks), want_stream(name, 3, total, lanes, lane_len))


def test_streaming_consumer_recycles_pooled_buffers():
    spec = P.get_spec("xoshiro256starstar")
    lanes, lane_len = 128, 1024
    total = lanes * lane_len * 12
    want = want_stream("xoshiro256starstar", 5, total, lanes, lane_len)
    pool = _ChunkPool.get(torch.device("cuda", torch.cuda.current_device()), torch.uint64, lanes * lane_len)
    pos, pooled, firsts = 0, 0, []
    for c in P.output_stream(spec, 5, total, lanes=lanes, lane_len=lane_len):
        np.testing.assert_array_equal(c, want[pos:pos + c.size])
        pooled += isinstance(c.base, torch.Tensor)
        firsts.append(c[:4].copy())
        pos += c.size
    assert pos == total
    assert pooled == 12          # every chunk was a pooled DMA target (no fallback copy)
    assert pool.made <= pool.cap
    gc.collect()
    # a view that outlives its chunk keeps the buffer out of the pool
    it = P.output_stream(spec, 5, total, lanes=lanes, lane_len=lane_len)
    keep = next(it)[100:200]
    rest = [c[:8].copy() for c in it]
    np.testing.assert_array_equal(keep, want[100:200])
    assert len(rest) == 11


def test_early_close_returns_buffers():
    spec = P.get_spec("xoroshiro128plus")
    lanes, lane_len = 96, 1024
    pool = _ChunkPool.get(torch.device("cuda", torch.cuda.current_device()), torch.uint64, lanes * lane_len)
    for _ in range(5):
        it = P.output_stream(spec, 1, None, lanes=lanes, lane_len=lane_len)
        first = next(it)
        assert first.size == lanes * lane_len
        it.close()
        del first
        gc.collect()
    assert pool.made <= pool.cap and len(pool.free) == pool.made
