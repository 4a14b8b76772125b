"""Bit-exact stage bookkeeping of the product (libalcop.so's host enumerator,
which the GPU tests pin to the device trace) against the reference.

WRAP mode is the reference-faithful emission: for every single-level golden
program, one CTA walking all output tiles must issue exactly the reference's
copies (slot, chunk) in order, consume exactly its slots, and carry the
interpreter's group counters (TraceEvent, interp.hpp:20-26) at every event.
"""
import pytest

from oracle import coracle
from tests import golden_util as G

pytestmark = []


def _product_events(alcop, tiles, E, sA, sB, mode):
    prod = alcop.enumerate_pipeline(tiles, E, sA, sB, mode, 0)
    cons = alcop.enumerate_pipeline(tiles, E, sA, sB, mode, 1)
    return prod, cons


SINGLE = [c for c in G.gemm_cases() if c["tA"] == 0 and c["tB"] == 0]


@pytest.mark.parametrize("case", SINGLE, ids=lambda c: c["name"])
def test_wrap_mode_equals_reference(alcop, case):
    E = case["ko"]
    tiles = G.tiles_of(case)
    sA = max(case["sA"], 1)  # "no hint" = a one-slot ring on B200
    sB = max(case["sB"], 1)
    prod, cons = _product_events(alcop, tiles, E, sA, sB, alcop.MODE_WRAP)
    walk = G.walk(case["name"])
    tileK = case["K"] // case["ko"]
    ref_trace = G.trace(case["name"])
    for b, side in enumerate("AB"):
        s = case["s" + side]
        if s < 2:
            continue
        buf = side + "_shared"
        # producer: per tile the reference's copies (slot, chunk)
        ref_copies = G.producer_copies(walk, buf, tileK, case["batch"] > 1)
        mine = [(e["slot"], e["chunk"]) for e in prod if e["buf"] == b]
        assert mine == ref_copies * tiles
        # consumer: slot of each use (E per tile) then s-1 drains
        ref_cons = [c[2] for c in G.consumer_slots(walk, buf) if c[1] == 0]
        uses = [e for e in cons if e["buf"] == b and e["kind"] == 1]
        per_tile = len(uses) // tiles
        assert per_tile == E + s - 1
        for t in range(tiles):
            assert [e["slot"] for e in uses[t * per_tile:t * per_tile + E]] == ref_cons
        # counters: producer events carry (acquired, committed) after commit,
        # consumer events (waited, released) — the interpreter's values
        ref_commit = [(r["acquired"], r["committed"]) for r in ref_trace
                      if r["group"] == buf and r["kind"] == "producer_commit"]
        assert [(e["acquired"], e["committed"]) for e in prod if e["buf"] == b] == ref_commit
        ref_cons_ev = [(1 if r["kind"] == "consumer_wait" else 2, r["waited"], r["released"]) for r in ref_trace
                       if r["group"] == buf and r["kind"] in ("consumer_wait", "consumer_release")]
        assert [(e["kind"], e["waited"], e["released"]) for e in cons if e["buf"] == b] == ref_cons_ev


@pytest.mark.parametrize("tiles,E,sA,sB", [(1, 1, 1, 1), (3, 5, 2, 2), (4, 2, 4, 3), (2, 7, 1, 5), (5, 3, 8, 8)])
def test_fused_mode_invariants(alcop, tiles, E, sA, sB):
    """FUSED: one lookahead window over the flattened (tile, chunk) stream —
    each chunk loaded exactly once, slots cyclic, no drains, and the merged
    counter invariant released <= waited <= committed <= acquired with at
    most s groups in flight."""
    prod, cons = _product_events(alcop, tiles, E, sA, sB, alcop.MODE_FUSED)
    for b, s in ((0, sA), (1, sB)):
        p = [e for e in prod if e["buf"] == b]
        assert [(e["tile"], e["chunk"]) for e in p] == [(t, k) for t in range(tiles) for k in range(E)]
        assert [e["slot"] for e in p] == [i % s for i in range(tiles * E)]
        c = [e for e in cons if e["buf"] == b]
        assert len(c) == 2 * tiles * E
        assert [e["slot"] for e in c if e["kind"] == 1] == [i % s for i in range(tiles * E)]
        # phase parity seen by each side equals (use index / s) & 1
        assert [e["parity"] for e in p] == [((i // s) & 1) ^ 1 for i in range(tiles * E)]
        assert [e["parity"] for e in c if e["kind"] == 1] == [(i // s) & 1 for i in range(tiles * E)]
    # a legal interleaving exists: producer of load j may run once release j-s happened
    for b, s in ((0, sA), (1, sB)):
        p = [e for e in prod if e["buf"] == b]
        rel = [e for e in cons if e["buf"] == b and e["kind"] == 2]
        inflight_max = 0
        committed = released = 0
        ri = 0
        for e in p:
            while committed - released >= s:
                released = rel[ri]["released"]
                ri += 1
            committed = e["committed"]
            inflight_max = max(inflight_max, committed - released)
        assert inflight_max <= s


@pytest.mark.parametrize("tiles,E,s", [(1, 4, 2), (3, 4, 3), (2, 2, 4), (3, 1, 3)])
def test_wrap_mode_matches_oracle_restatement(alcop, tiles, E, s):
    """Beyond the golden corpus: the WRAP enumerator equals the oracle's
    restated root algebra and counters for arbitrary (tiles, E, s)."""
    prod, cons = _product_events(alcop, tiles, E, s, s, alcop.MODE_WRAP)
    ps, pc, cs = coracle.root_schedule(E, s)
    mine = [(e["slot"], e["chunk"]) for e in prod if e["buf"] == 0]
    assert mine == list(zip(ps.tolist(), pc.tolist())) * tiles
    tr = coracle.sync_trace(tiles, E, 1, s, s)
    ref = [(r["acquired"], r["committed"]) for r in tr if r["group"] == "A_shared" and r["kind"] == "producer_commit"]
    assert [(e["acquired"], e["committed"]) for e in prod if e["buf"] == 0] == ref
