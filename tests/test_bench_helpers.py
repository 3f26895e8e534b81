"""CPU checks of bench.py's measurement helpers (no GPU): the paper's timing statistic T^ww
(mean without the worst call), the result throughput's array sizes,
the per-cell algorithmic bytes / flops behind the rooflines, and the config dict shared by both
arms."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import fe_inputs as fi  # noqa: E402


def test_step_stats_tww():
    xs = [1.0, 2.0, 3.0, 10.0]
    st = bench.step_stats(xs)
    assert st["tww"] == pytest.approx(2.0)        # (1 + 2 + 3) / 3: the worst call dropped
    assert st["mean"] == pytest.approx(4.0)
    assert st["median"] == pytest.approx(2.5)
    assert st["min"] == 1.0 and st["n"] == 4
    assert bench.step_stats([5.0])["tww"] == 5.0


def test_result_bytes_and_alg_bytes():
    pr = fi.make_config("C2", N=4)
    nd = pr.nb
    assert bench.result_bytes(pr, "matrix", 8) == pr.n_elems * nd * nd * 8
    assert bench.result_bytes(pr, "residual", 4) == pr.n_elems * nd * 4
    # C2 matrix: one vertex + conn (56 B) + kappa per qp (27 x 8) + K (27 x 27 x 8) per cell
    assert bench.alg_bytes(fi.DIFFUSION, "matrix", 2, 27, 27, 1, fi.MAT_PER_QP) == 56 + 216 + 5832
    # C2 matrix 6,104 B per cell
    assert bench.alg_bytes(fi.DIFFUSION, "matrix", 2, 27, 27, 1, fi.MAT_PER_QP) == 6104


def test_split_cfg_and_subconfigs():
    assert bench.split_cfg("C4f32") == ("C4", "f32")
    assert bench.split_cfg("C3") == ("C3", None)
    for name in bench.SUB_CONFIGS:
        assert bench.split_cfg(name)[0] in bench.WORKLOADS


def test_config_dict_same_in_both_arms():
    """--impl reference prints the same `config` object as the measured arm."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "C1", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    pr = bench.build_problem("C1")
    assert line["config"] == bench.config_dict("C1", pr, bench.WORKLOADS["C1"]["modes"], 1,
                                               "nccl", "f64")
    assert line["impl"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle"
