"""Experiment report and memory-budget sweep (harness.py:213-394) against the
reference's own outputs frozen in tests/golden/sweep.json
(tests/golden/make_sweep_golden.py imports the unmodified reference)."""

import json
import os

import pytest

from paper_2508_04711_b200 import harness

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden():
    with open(os.path.join(GOLDEN, "sweep.json")) as f:
        return json.load(f)


def test_sweep_matches_reference_bit_exact():
    for sw in _golden()["sweeps"]:
        got = harness.sweep_max_tokens(sw["budget"], sw["cp_sizes"], sw["embed_dim"], sw["dtype"]).to_json_dict()
        assert got == sw["json"]


def test_modeled_rank_bytes_matches_reference():
    for m in _golden()["modeled"]:
        assert harness.modeled_rank_bytes(m["L"], m["cp"], m["embed_dim"], m["dtype_size"]) == m["bytes"]


def test_sweep_trend_and_errors():
    # test_harness.py:107-125: non-decreasing in cp, cp=8 >= 4x cp=1; budget / cp errors
    ls = [r["max_supported_length"] for r in harness.sweep_max_tokens(16_777_216, [1, 2, 4, 8]).rows]
    assert ls == sorted(ls) and ls[-1] >= 4 * ls[0]
    with pytest.raises(ValueError, match="budget"):
        harness.sweep_max_tokens(10, [1])
    with pytest.raises(ValueError):
        harness.sweep_max_tokens(16_777_216, [0])
    with pytest.raises(ValueError):
        harness.ExperimentConfig(dtype="f16")


def test_config_json_has_reference_fields():
    keys = _golden()["report_keys"]["config"]
    cfg = harness.ExperimentConfig(cp_size=2, batch_size=2, min_len=0, max_len=24, max_length=32, seed=23)
    assert set(keys) <= set(cfg.to_json_dict())


@pytest.mark.gpu
def test_run_experiment_report_on_gpu():
    # the reference's golden config (tests/golden/bench_cp2_seed23.json): same
    # report schema, same integer fields, bf16-level equivalence error
    g = _golden()["report_keys"]
    with open(os.path.join(GOLDEN, "plans.json")) as f:
        exp = json.load(f)["experiment"]
    cfg = harness.ExperimentConfig(cp_size=2, batch_size=2, min_len=0, max_len=24, max_length=32, embed_dim=128,
                                   seed=23)
    payload = harness.run_experiment(cfg).to_json_dict()
    assert set(payload) == set(g)
    for k, sub in g.items():
        if sub is not None and k not in ("config", "metadata"):
            assert sorted(payload[k]) == sub, k
    assert "accounting" in payload["metadata"] and payload["metadata"]["gpu"]["pipeline_ms"] > 0
    assert payload["resident_tokens_per_rank"] == exp["resident_tokens_per_rank"]
    assert payload["flops"]["per_rank"] == exp["flops"]["per_rank"]
    assert payload["max_rel_error"] <= 2e-2
    assert 0.0 <= payload["memory_reduction_ratio"] < 1.0
    json.dumps(payload)  # serialisable
