"""The event-level simulator (§8(f) rank 4) through the C ABI:
alcop_simulate_pipeline / alcop_simulate_two_level equal the reference's
sim::simulate_pipeline / simulate_two_level (pipe_sim.hpp:55-167) on every
golden query (tests/golden/model.jsonl, produced by the reference itself via
oracle/ref_driver), and alcop_simulate_kernel (the B200 two-level analogue)
is checked for its structural properties here and against device timings
in the gpu test."""
import pytest

from tests import golden_util as G


def _close(a, b):
    return abs(a - b) <= 1e-9 * max(1.0, abs(a), abs(b))


def _queries(prefix):
    return [it for it in G.model_queries() if it["q"].split()[0] == prefix]


def test_simulate_pipeline_matches_reference(alcop):
    qs = _queries("sim")
    assert len(qs) > 150
    for it in qs:
        a = it["q"].split()[1:]
        cfg = alcop.sim_config(float(a[0]), float(a[1]), int(a[2]), int(a[3]), int(a[4]))
        if it["a"] == "error":
            with pytest.raises(alcop.AlcopError) as ei:
                alcop.simulate_pipeline(cfg)
            assert ei.value.code == alcop.ALCOP_ERR_CONFIG and ei.value.rule == "BadSimConfig"
            continue
        want = [float(x) for x in it["a"].split()]
        got = alcop.simulate_pipeline(cfg)
        for k, w in zip(("makespan", "firstComputeStart", "busy", "idleFraction", "comparable"), want):
            assert _close(got[k], w), (it, k, got[k], w)


def test_simulate_pipeline_trace_matches_reference(alcop):
    qs = _queries("simtrace")
    assert len(qs) > 40
    for it in qs:
        a = it["q"].split()[1:]
        cfg = alcop.sim_config(float(a[0]), float(a[1]), int(a[2]), int(a[3]), int(a[4]))
        got = alcop.simulate_pipeline(cfg, trace=True)["trace"]
        want = [e.split(":") for e in it["a"].split()]
        assert len(got) == len(want)
        for g, w in zip(got, want):
            assert _close(g[0], float(w[0])) and g[1] == int(w[1]) and g[2] == w[2] and g[3] == int(w[3]), (g, w)


def test_simulate_two_level_matches_reference(alcop):
    qs = _queries("sim2")
    assert len(qs) > 150
    for it in qs:
        a = it["q"].split()[1:]
        outer = alcop.sim_config(float(a[0]), float(a[1]), int(a[2]), int(a[3]))
        inner = alcop.sim_config(float(a[4]), float(a[5]), int(a[6]), int(a[7]))
        fused = int(a[8]) != 0
        if it["a"] == "error":
            with pytest.raises(alcop.AlcopError):
                alcop.simulate_two_level(outer, inner, fused)
            continue
        assert _close(alcop.simulate_two_level(outer, inner, fused), float(it["a"])), it


def test_two_level_fused_never_slower_than_restart(alcop):
    for tl in (0, 50, 400, 2000):
        for tu in (1, 10, 40):
            for s in (1, 2, 4):
                outer = alcop.sim_config(tl, 0, 12, s)
                inner = alcop.sim_config(5, tu, 4, 2)
                assert alcop.simulate_two_level(outer, inner, True) <= alcop.simulate_two_level(outer, inner, False)


def test_simulate_kernel_structure(alcop):
    """B200 kernel sim: a second TMEM accumulator never hurts and hides the
    epilogue behind the next tile's main loop; FUSED (run-ahead across tiles)
    never loses to WRAP (ring restart + s-1 drained loads); more smem stages
    never hurt; counts follow the schedule."""
    d = alcop.gemm_desc(8192, 8192, 512)
    for st in (1, 2, 4):
        s1 = alcop.make_schedule(tileN=256, tileK=64, n_stage=st, n_stage_inner=1)
        s2 = alcop.make_schedule(tileN=256, tileK=64, n_stage=st, n_stage_inner=2)
        k1, k2 = alcop.simulate_kernel(d, s1), alcop.simulate_kernel(d, s2)
        assert k2["tBody"] <= k1["tBody"] + 1e-6
        assert k1["tilesPerUnit"] == k2["tilesPerUnit"] == -(-(64 * 32) // 148)
        assert k1["loads"] == k1["tilesPerUnit"] * 8
        w = alcop.simulate_kernel(d, alcop.make_schedule(tileN=256, tileK=64, n_stage=st, n_stage_inner=2,
                                                         mode=alcop.MODE_WRAP))
        assert w["loads"] == w["tilesPerUnit"] * (8 + st - 1)
        assert k2["tBody"] <= w["tBody"] + 1e-6
    prev = None
    for st in range(1, 5):
        t = alcop.simulate_kernel(d, alcop.make_schedule(tileN=256, tileK=64, n_stage=st))["tBody"]
        if prev is not None:
            assert t <= prev + 1e-6
        prev = t


def _pairs(rows, key):
    import itertools
    agree = tot = 0
    for sh in {tuple(r["shape"]) for r in rows}:
        rs = [r for r in rows if tuple(r["shape"]) == sh]
        for a, b in itertools.combinations(rs, 2):
            if abs(a["ms"] / b["ms"] - 1) < 0.02:
                continue
            tot += 1
            agree += (a["ms"] < b["ms"]) == (a[key] < b[key])
    return agree, tot


def test_simulate_kernel_vs_committed_device_timings(alcop):
    """profiles/sim_vs_device_r01.json (tools/sim_vs_device.py on a B200):
    re-simulated with the current library, the two-level simulation orders
    every schedule pair whose measured times differ by > 2% (stages x t x
    FUSED/WRAP) and stays within 20% mean abs error."""
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "sim_vs_device_r01.json")
    rows = json.load(open(path))
    assert len(rows) >= 40
    for r in rows:
        d = alcop.gemm_desc(*r["shape"])
        s = alcop.make_schedule(tileN=r["tileN"], tileK=r["tileK"], n_stage=r["n_stage"],
                                n_stage_inner=r["n_stage_inner"], mode=r["mode"])
        r["sim_now"] = alcop.simulate_kernel(d, s)["seconds"] * 1e3
    agree, tot = _pairs(rows, "sim_now")
    assert tot > 100 and agree >= 0.97 * tot, (agree, tot)
    mape = sum(abs(r["sim_now"] / r["ms"] - 1) for r in rows) / len(rows)
    assert mape < 0.20, mape


@pytest.mark.gpu
def test_simulate_kernel_vs_live_device(alcop):
    """Live: the outer ring depth (n_stage 2 vs 4) and FUSED vs WRAP on a
    many-tiles-per-CTA GEMM — the simulation orders them as measured and its
    speed-up ratios are within 25% of the measured ones."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from sim_vs_device import measure
    kws = [dict(tileN=256, tileK=64, n_stage=2, n_stage_inner=2, mode=alcop.MODE_FUSED),
           dict(tileN=256, tileK=64, n_stage=4, n_stage_inner=2, mode=alcop.MODE_FUSED),
           dict(tileN=256, tileK=64, n_stage=4, n_stage_inner=2, mode=alcop.MODE_WRAP)]
    r1, r4, rw = measure(8192, 8192, 256, kws)
    for slow, fast in ((r1, r4), (rw, r4)):
        meas, sim = slow["ms"] / fast["ms"], slow["sim_ms"] / fast["sim_ms"]
        assert meas > 1.0 and sim > 1.0, (slow, fast)
        assert abs(sim / meas - 1) < 0.25, (meas, sim)
