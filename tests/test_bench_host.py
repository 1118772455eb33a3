"""Host-side pieces of bench.py that run without a GPU: the byte models behind `roofline.achieved`
 and the clock sampler's behaviour when neither NVML nor nvidia-smi is there."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def test_algorithmic_bytes_follow_the_survey_figures():
    # C3 refactor + solve = 91.5 + 190.6 + 131.3 MB, +220 MB for one FGMRES iteration
    n, nnz_a, nnz_f = 238000, 1332800, 9435168
    ab = bench.algorithmic_bytes(n, nnz_a, nnz_f, 1)
    assert abs(ab["eliminate"] - (20 * nnz_f + 8 * n)) < 1
    assert abs(ab["eliminate"] / 1e6 - 190.6) < 0.2
    assert abs(ab["total"] / 1e6 - 633) < 5
    # the batch model shares one copy of the indices between the scenarios
    bb = bench.batch_algorithmic_bytes(256, 55700, 311920, 2203476, 1)
    assert bb["eliminate"] == 256 * 16 * 2203476 + 4 * 2203476 + 8 * 55700


def test_clock_sampler_reports_instead_of_failing():
    s = bench.ClockSampler(0)
    s.window_start()
    time.sleep(0.02)
    s.window_stop()
    out = s.stop()
    assert "reasons" in out and "sm_mhz" in out
    if out["sm_mhz"] is None:  # no GPU in this container
        assert out["reasons"] == ["nvml and nvidia-smi unavailable"]
    else:
        assert out["samples"] >= 1
