"""bench.py host-side contract (CPU): the weak-scaling shard map and the reference arm's JSON
line (the oracle on a bounded C4 sample; rank 0 alone prints)."""
import json
import types

import bench


def test_weak_shards_disjoint_and_cover():
    B = 4096
    for world in (1, 2, 4, 8):
        spans = [bench._slice(B, r, world) for r in range(world)]
        assert all(n == B for _, n in spans)  # per-GPU work fixed as N grows
        starts = sorted(s for s, _ in spans)
        assert starts == [r * B for r in range(world)]  # disjoint, covering [0, world * B)
        cfg = bench._config(B, world)
        assert cfg["batch"] == B and cfg["global_batch"] == B * world


def _args(steps=1, warmup=0):
    return types.SimpleNamespace(steps=steps, warmup=warmup, batch=bench.C4_BATCH, gpus=1, impl="reference")


def test_reference_arm_line(monkeypatch, capsys):
    monkeypatch.setattr(bench, "CPU_SAMPLE_SECONDS", 0.5)
    bench.run_reference(_args(), 0, 1)
    out = capsys.readouterr().out.strip().splitlines()
    assert len(out) == 1
    line = json.loads(out[0])
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC
    assert line["unit"] == "roundings/s" and line["higher_is_better"] is True
    assert line["scaling"] == "weak" and line["n_gpus"] == 1
    assert line["value"] > 0 and line["cpu_baseline"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "roundings/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_silent(capsys):
    bench.run_reference(_args(), 1, 2)
    assert capsys.readouterr().out == ""
