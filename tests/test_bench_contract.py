"""bench.py's reference arm keeps the driver's JSON contract (CPU-only: the
oracle sample is stubbed so the test runs in seconds)."""

import json
import sys


def test_reference_arm_json_line(monkeypatch, capsys):
    import bench
    calls = []

    class FakeRef:
        def __init__(self, n_sessions=32):
            self.n = n_sessions

        def sample(self):
            calls.append(self.n)
            return {"value": 0.01, "unit": "req/s", "cores": 4, "kind": "port", "sample": "stub"}
    monkeypatch.setattr(bench, "CpuReference", FakeRef)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1"])
    monkeypatch.delenv("RANK", raising=False)
    bench.main()
    line = capsys.readouterr().out.strip().splitlines()[-1]
    d = json.loads(line)
    assert d["impl"] == "reference" and d["warmup"] == 3  # W >= 3 enforced
    assert len(calls) == d["warmup"] + d["steps"] and calls[0] == 32
    for k in ("metric", "value", "unit", "n_gpus", "steps", "higher_is_better", "scaling", "vs_baseline",
              "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["e2e"] == {"value": d["value"], "unit": "req/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("configs[1]")


def test_reference_arm_other_ranks_exit_quietly(monkeypatch, capsys):
    import bench
    monkeypatch.setattr(bench, "CpuReference", lambda n=1: (_ for _ in ()).throw(AssertionError))
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference"])
    monkeypatch.setenv("RANK", "1")
    bench.main()
    assert capsys.readouterr().out == ""
