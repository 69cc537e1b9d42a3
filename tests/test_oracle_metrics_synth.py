"""Pins for the evaluation utility (Table I) and the input generator."""
import numpy as np
import pytest

import synth
from oracle import metrics

from conftest import golden_value


def test_table1_arithmetic():
    # Table I row "3D snakuscules": P = 0.97, R = 0.84 -> F = 0.90;
    # G23: SPEC AC10's 0.8953 is wrong, F(0.97, 0.84) = 0.9003.
    assert metrics.f_measure(0.97, 0.84) == pytest.approx(golden_value("f_measure_spec_ac10"), abs=5e-5)
    assert round(metrics.f_measure(0.97, 0.84), 2) == 0.90
    # G22: the CellSegm row is internally inconsistent (0.7615, printed 0.82)
    assert metrics.f_measure(0.66, 0.90) == pytest.approx(golden_value("f_measure_cellsegm"), abs=5e-5)
    assert metrics.prf(0, 0, 0) == (0.0, 0.0, 0.0)


def test_match_detections():
    truth = np.array([[0, 0, 0], [10, 0, 0], [20, 0, 0]], float)
    m = metrics.match_detections(truth + 0.5, truth, 1.0)
    assert (m["tp"], m["fp"], m["fn"]) == (3, 0, 0) and m["prf"][2] == 1.0
    m = metrics.match_detections(np.array([[50, 0, 0]] * 3, float), truth[:2], 1.0)
    assert (m["tp"], m["fp"], m["fn"]) == (0, 3, 2)
    # one-to-one: two detections near one truth -> one TP, one FP
    m = metrics.match_detections(np.array([[0.1, 0, 0], [0.2, 0, 0]]), truth[:1], 1.0)
    assert (m["tp"], m["fp"]) == (1, 1) and m["matches"][0][0] == 0


def test_config_sizes():
    c = synth.CONFIGS
    assert synth.nuclei("C4").shape[0] == 198_927
    assert len(synth.nuclei("C3")) == 10_192 and c["C3"].iso_n == (512, 512, 256)
    assert len(synth.nuclei("C2")) == 2025
    assert [len(synth.nuclei(f"C5_{i}")) for i in range(4)] == [2312, 5324, 9477, 20825]
    assert c["C4"].window == 5 and c["C3"].window == 4 and c["C2"].window == 9


def test_slab_reproducibility():
    cfg = synth.CONFIGS["C3"]
    full = synth.generate(cfg, 40, 60)
    part = synth.generate(cfg, 47, 52)
    assert np.array_equal(full[7:12], part)
    a = synth.generate("C1")
    assert np.array_equal(a, synth.generate("C1"))
    assert a.dtype == np.uint16 and a.shape == (64, 64, 64)


def test_c1_layout():
    t = synth.nuclei("C1")
    assert len(t) == 8
    for cc in t["c"]:
        for v in cc:
            assert min(abs(v - 16), abs(v - 48)) <= 2.0
    assert np.all((t["rbar"] >= 6) & (t["rbar"] <= 9))
