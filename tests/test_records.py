"""Reference-compatible value types (schemes.py:58-101, theta_tables.py,
matcore.py:38-66): validation rules of pkg/tests/test_schemes.py /
test_driver.py / test_matcore.py restated."""
from fractions import Fraction

import numpy as np
import pytest

import paper_2010_00465_b200 as csm


@pytest.mark.parametrize("family,k", [
    (csm.SchemeFamily.COS_SIN_TAYLOR, 5), (csm.SchemeFamily.COS_SIN_TAYLOR, 0),
    (csm.SchemeFamily.WAVE_KERNEL, 6), (csm.SchemeFamily.PADE8, 4)])
def test_scheme_id_rejects_bad_k(family, k):
    with pytest.raises(ValueError):
        csm.SchemeId(family, k)


def test_theta_table_rejects_nonincreasing_thresholds():
    with pytest.raises(ValueError):
        csm.ThetaTable(csm.Precision.DOUBLE, (
            csm.ThetaEntry(csm.SchemeId(csm.SchemeFamily.COS_SIN_TAYLOR, 3),
                           1.0, 1.0, Fraction(3)),
            csm.ThetaEntry(csm.SchemeId(csm.SchemeFamily.COS_SIN_TAYLOR, 4),
                           0.5, 0.5, Fraction(4))))
    with pytest.raises(ValueError):
        csm.ThetaTable(csm.Precision.DOUBLE, ())


def test_cost_ledger():
    led = csm.CostLedger()
    led.charge_product()
    led.charge_product(2)
    led.charge_lu(solves=2)
    assert led.total_cost == Fraction(3) + Fraction(1, 3) + 2
    with pytest.raises(ValueError):
        led.charge_product(-1)


def test_matrix_from_rows_validation():
    assert csm.matrix_from_rows([[1, 2], [3, 4]]).dtype == np.float64
    for bad in ([[1, 2], [3]], [], [[float("inf")]]):
        with pytest.raises(csm.MatrixInputError):
            csm.matrix_from_rows(bad)


def test_public_namespace_covers_the_hot_path():
    for name in ("cos_sin", "wave_cos_sin", "select_scheme", "taylor_cos_sin",
                 "wave_kernels", "norm1", "ComputationReport", "CosSinResult",
                 "WaveResult", "CostLedger", "MatrixInputError", "Precision",
                 "SchemeFamily", "SchemeId", "ThetaEntry", "ThetaTable",
                 "TAYLOR_TABLE", "WAVE_TABLE"):
        assert hasattr(csm, name), name


def test_compute_without_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        csm.cos_sin(np.eye(3))
