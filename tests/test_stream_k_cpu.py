"""Invariants of the stream-K segment schedule (CPU restatement of
for_each_seg in csrc/gemm_sm100.cu, alcop_pipelined_gemm_pair_kernel<..., kSK>):
every (tile, chunk) is computed exactly once; a tile is cut between at most
two clusters; a cluster's only partial writer segment is its first stream-K
segment and its only finisher segment its last; the writer of the tile a
cluster finishes is the next cluster (the kernel reads flag/slot cluster+1)."""
import itertools

import pytest


def segments(num_tiles, E, n, c):
    """Cluster c's segments (k, tile, cb, ce), as the kernel enumerates them."""
    out = []
    dp_waves = num_tiles // n - 1
    k = 0
    for k in range(dp_waves):
        out.append((k, c + k * n, 0, E))
    k = dp_waves
    t0 = dp_waves * n
    T = (num_tiles - t0) * E
    e0 = T * (c + 1) // n
    g = T * c // n
    while g < e0:
        t = g // E
        cb = g - t * E
        ce = min(E, cb + (e0 - g))
        out.append((k, t0 + t, cb, ce))
        g += ce - cb
        k += 1
    return out


CASES = [(192, 12, 74), (144, 12, 74), (148, 12, 74), (80, 256, 74), (96, 12, 74), (1024, 128, 74),
         (256, 64, 74), (75, 1, 74), (74, 3, 74), (157, 7, 74), (300, 2, 16), (9, 5, 8)]


@pytest.mark.parametrize("num_tiles,E,n", CASES)
def test_stream_k_partition(num_tiles, E, n):
    assert num_tiles >= n  # host precondition (launch_gemm enables stream-K only then)
    seen = {}
    writers, finishers = {}, {}
    for c in range(n):
        segs = segments(num_tiles, E, n, c)
        assert [s[0] for s in segs] == list(range(len(segs)))  # k counts segments (accumulator ring index)
        for idx, (k, t, cb, ce) in enumerate(segs):
            assert 0 <= cb < ce <= E and 0 <= t < num_tiles
            for ch in range(cb, ce):
                assert (t, ch) not in seen, "chunk computed twice"
                seen[(t, ch)] = c
            if cb > 0:  # writer: the tile's last chunks
                assert ce == E and idx == num_tiles // n - 1, "writer must be the first stream-K segment"
                assert c not in writers
                writers[c] = t
            if cb == 0 and ce < E:  # finisher: the tile's first chunks
                assert idx == len(segs) - 1, "finisher must be the cluster's last segment (drained ring)"
                finishers[c] = t
    assert len(seen) == num_tiles * E
    # every cut tile: finisher c, writer c + 1, nobody else touches it
    for c, t in finishers.items():
        assert writers.get(c + 1) == t
        owners = {seen[(t, ch)] for ch in range(E)}
        assert owners == {c, c + 1}
    assert len(writers) == len(finishers)


def test_stream_k_balance_ffn1():
    """FFN1 (192 pair tiles, E = 12, 74 clusters): 31-32 chunks per cluster instead of 24 or 36."""
    per = [sum(ce - cb for _, _, cb, ce in segments(192, 12, 74, c)) for c in range(74)]
    assert min(per) >= 31 and max(per) <= 32
    whole = [12 * len(range(c, 192, 74)) for c in range(74)]
    assert max(whole) == 36
