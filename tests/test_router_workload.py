"""Router and workload generator vs traces produced by the reference
(tests/golden/router_traces.json, tests/golden/workload.json)."""

import json
from pathlib import Path
from types import SimpleNamespace

import pytest

from paper_2602_12029_b200 import router as R
from paper_2602_12029_b200 import workload as wl

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_router_matches_reference_traces():
    traces = json.loads((GOLDEN / "router_traces.json").read_text())
    for tr in traces:
        r = R.Router(R.ServingMode(tr["mode"]), tr["models"])
        for st in tr["steps"]:
            req = SimpleNamespace(session_id=st["session"], model_id=st["model"])
            if "error" in st:
                with pytest.raises(R.ConfigurationError):
                    r.route_prefill(req, st["depths"])
                continue
            assert r.route_prefill(req, st["depths"]) == st["prefill"]
            assert r.decode_worker(req) == st["decode"]
            assert r.prefill_namespace(st["model"]) == st["ns"]


def test_routing_table_conflict():
    t = R.RoutingTable()
    t.pin(1, 2)
    t.pin(1, 2)
    with pytest.raises(RuntimeError):
        t.pin(1, 3)
    assert t.get(1) == 2 and t.get(9) is None


def test_placement_split_and_colocated():
    p = R.Placement.split(4, [0, 1], [2, 3, 4, 5, 6, 7])
    assert p.prefill_gpus == (0, 1, 0, 1) and p.decode_gpus == (2, 3, 4, 5)
    assert not p.handoff_is_local(0, 0)
    c = R.Placement.colocated(4)
    assert c.handoff_is_local(3, 2)
    assert p.replicas(1) == (3,) and p.decode_models_on(4) == [2]


def test_placement_decode_replicas_use_every_decode_gpu():
    """2 prefill + 6 decode GPUs, 4 models: every decode GPU holds a replica
    (models 0 and 1 get two), the logical decode worker ids are unchanged."""
    p = R.Placement.split(4, [0, 1], [2, 3, 4, 5, 6, 7], n_prefill=2, replicate=True)
    assert p.prefill_gpus == (0, 1) and p.decode_gpus == (2, 3, 4, 5)
    assert [p.replicas(m) for m in range(4)] == [(2, 6), (3, 7), (4,), (5,)]
    assert sorted(g for m in range(4) for g in p.replicas(m)) == [2, 3, 4, 5, 6, 7]
    assert p.decode_models_on(6) == [0] and p.decode_models_on(0) == []
    r = R.Router(R.ServingMode.PREFILLSHARE, ["a", "b", "c", "d"])

    class Req:
        model_id = "b"
    assert r.decode_worker(Req) == 5  # n_models + index, whatever the replicas
    # fewer decode GPUs than models: no replicas, GPUs host several models
    q = R.Placement.split(4, [0], [1, 2], replicate=True)
    assert q.decode_replicas is None and q.decode_gpus == (1, 2, 1, 2)


def test_workload_matches_reference():
    g = json.loads((GOLDEN / "workload.json").read_text())
    s = wl.splitmix64(0)
    assert [next(s) for _ in range(8)] == [int(x) for x in g["splitmix64_seed0"]]
    assert next(wl.splitmix64(0)) == 0xE220A8397B1DCDAF  # test_workload.py:12-17
    assert str(wl.mix_seed(1, 2)) == g["mix_seed"]["1,2"]
    assert str(wl.mix_seed(0)) == g["mix_seed"]["0"]
    assert str(wl.mix_seed(0, 0)) == g["mix_seed"]["0,0"]
    assert [str(t) for t in wl.synth_tokens(3, 5, 4)] == g["synth_tokens_3_5_4"]
    cfg = wl.WorkloadConfig(pattern="react", arrival_rate_per_s=4.0, duration_s=20.0, seed=3)
    assert json.loads(wl.export_sessions(wl.generate(cfg))) == g["generate_react_seed3_20s"]
    sessions = wl.generate(cfg)
    assert wl.import_sessions(wl.export_sessions(sessions)) == sessions


def test_synth_tokens_limits_and_disjoint():
    with pytest.raises(ValueError):
        wl.synth_tokens(0, 0, -1)
    with pytest.raises(ValueError):
        wl.synth_tokens(0, 1 << 16, 4)
    assert not set(wl.synth_tokens(1, 0, 64)) & set(wl.synth_tokens(2, 0, 64))
