"""CPU checks of bench.py's host logic: the JSON line contract and the reference arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_make_line_contract():
    import bench
    from paper_2512_06230_b200.scenes import CONFIGS
    line = bench.make_line(
        cfg_id=3, cfg=CONFIGS[3], world=1, steps=4, warmup=3, elapsed_ms=10.0, evals_total=4.0e10,
        pairs_per_launch=1.0e10, stage_ms={"predict": [0.06] * 4, "birth": [0.01] * 4,
                                           "compat": [2.4] * 4, "reweight": [0.08] * 4},
        sm_count=148, clocks={"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": []},
        T_surv=1024, B_local=16, T_local=1040, P=8192, M_mean=1198.0, traffic=None,
        e2e={"value": 1.0, "unit": "evals/s", "h2d_bytes_per_step": 1, "d2h_bytes_per_step": 1},
        cpu={"value": 1.0, "unit": "evals/s", "cores": 8, "kind": "oracle", "sample": "x", "seconds": 1})
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "gpu_launches", "clocks"):
        assert key in line
    assert line["value"] == pytest.approx(4.0e12)
    assert line["ms_per_step"] == pytest.approx(2.5)
    r = line["roofline"]
    assert r["bound"] == "alu" and 0 < r["frac"] < 1 and r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert r["peak"] == pytest.approx(148 * (124.0 + 8 * 15.94) / 13 * 1.965e9 / 1e9)   # 5 lanes + 1 exp per pair
    assert line["gpu_launches"] == 16
    assert line["cpu_baseline"]["cores"] == 8 and "seconds" not in line["cpu_baseline"]
    assert "workload" in line["config"]
    json.dumps(line)


@pytest.mark.slow
def test_reference_arm_runs_on_cpu():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--config", "0"],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    # the same config object as the GPU arm prints for this workload (bench.workload_config)
    import bench
    from paper_2512_06230_b200.scenes import CONFIGS
    assert set(line["config"]) == set(bench.workload_config(0, CONFIGS[0], 1, 6.0, 1.0))
    assert "every track" in line["sample"]


def test_reweight_bytes_counts_tracks_with_a_measurement():
    """bench.reweight_bytes: 16 B per particle for a local track with an assigned measurement,
    8 B (w copied) for one without; theta_i = global column + 1 (0 clutter)."""
    import types

    import numpy as np

    import bench
    th = np.array([0, 3, 3, 1, 0, 7], np.int32)          # columns 2 (twice), 0, 6
    scene = types.SimpleNamespace(theta=[th])
    st = types.SimpleNamespace(scene=scene, P=8, T_local=4, col_of_row=np.array([0, 1, 2, 6]))
    assert bench.reweight_bytes(st, 0) == 8 * (16 * 3 + 8 * 1)
    st2 = types.SimpleNamespace(scene=scene, P=8, T_local=2, col_of_row=np.array([3, 4]))   # another rank
    assert bench.reweight_bytes(st2, 5) == 8 * (8 * 2)
