"""The reference's schedule surface (apply_script, schedule.hpp:590-646, plus
the pass's rule checks) through the C ABI: every golden script yields the same
accept/reject decision and rule tag as the reference, and accepted scripts map
to the B200 schedule lower() implies (schedule.hpp:371-374)."""
import pytest

from tests import golden_util as G

CASES = G.scripts()
# The reference's ValidationError cases are its own lower() emitting a program
# its validator rejects (a batched pre-op program whose A index drops the batch
# dim; a register cache of a global tensor whose consumer already reads the
# shared cache): lowering-IR defects, not schedule-surface decisions, and the
# B200 path has no lowered IR.  They are excluded from the parity set.
FUZZ = [c for c in G.scripts_fuzz() if c["result"].get("class") != "ValidationError"]


@pytest.mark.parametrize("case", CASES + FUZZ, ids=lambda c: c["name"])
def test_script_matches_reference(alcop, case):
    desc = alcop.gemm_desc(case["M"], case["N"], case["K"], case["batch"], pre_op=case.get("preop", 0))
    res = case["result"]
    if res["ok"]:
        s, warns = alcop.apply_script(desc, case["script"])
        assert warns == []
        plan = {p["buffer"]: p for p in res["plan"]}
        for side, field in (("A", "n_stage_smem_A"), ("B", "n_stage_smem_B")):
            names = [side + "_shared"] + (["S2_shared"] if side == "A" else [])
            hit = [plan[n]["stages"] for n in names if n in plan]
            assert getattr(s, field) == (hit[0] if hit else 1)
        regs = [p["stages"] for b, p in plan.items() if b.endswith("_reg")]
        assert s.n_stage_inner == (min(max(regs), 2) if regs else 1)
        assert s.mode == alcop.MODE_WRAP
        return
    with pytest.raises(alcop.AlcopError) as ei:
        alcop.apply_script(desc, case["script"])
    err = ei.value
    if res["class"] == "AnalysisError":
        assert err.code == alcop.ALCOP_ERR_ANALYSIS
        assert err.rule == res["rule"], (err, res)
    else:  # ConfigError / std::exception -> cli kConfig (cli.hpp:110-115)
        assert err.code == alcop.ALCOP_ERR_CONFIG, (err, res)


def test_config1_script_maps_to_baseline_schedule(alcop):
    text = open(G.case_dir("config1") + "/script.txt").read()
    s, _ = alcop.apply_script(alcop.gemm_desc(512, 512, 512, 1, alcop.F16, alcop.F32), text)
    assert (s.tileM, s.tileN, s.tileK) == (128, 128, 32)
    assert (s.n_stage_smem_A, s.n_stage_smem_B, s.n_stage_inner) == (2, 2, 2)
    alcop.validate(alcop.gemm_desc(512, 512, 512, 1, alcop.F16, alcop.F32), s)
