"""Reference-compatible value types of the cos/sin hot path.

Same names, fields and validation rules as the reference package
(paths under /root/reference/pkg/src/cossinm):

* SchemeFamily / SchemeId ........ schemes.py:58-87
* CosSinResult / WaveResult ...... schemes.py:90-101
* Precision / UNIT_ROUNDOFF ...... theta_tables.py:27-35
* ThetaEntry / ThetaTable ........ theta_tables.py:38-69
* TAYLOR_TABLE / WAVE_TABLE ...... theta_tables.py:79-144 (values read from
  the C library, which holds the reference's float64 bits; one source for
  host and device)
* CostLedger ..................... matcore.py:38-66
* MatrixInputError ............... matcore.py:30-31
* SingularMatrixError ............ matcore.py:34-35
* PADE_TABLE ..................... theta_tables.py:108-119
* ComputationReport .............. driver.py:56-61
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Any, TypeAlias

import numpy as np

from . import _lib

DenseMatrix: TypeAlias = Any  # numpy.ndarray or torch.Tensor (CUDA)


class MatrixInputError(ValueError):
    """Malformed matrix input: not square or not finite."""


class SingularMatrixError(RuntimeError):
    """Pade denominator singular to working precision."""


class SchemeFamily(enum.Enum):
    COS_SIN_TAYLOR = "cos_sin_taylor"
    WAVE_KERNEL = "wave_kernel"
    PADE8 = "pade8"


_ALLOWED_K = {
    SchemeFamily.COS_SIN_TAYLOR: (3, 4, 6, 7),
    SchemeFamily.WAVE_KERNEL: (3, 4, 5),
    SchemeFamily.PADE8: (5,),
}


@dataclass(frozen=True)
class SchemeId:
    """A scheme: its family and the products one cos+sin pair costs."""

    family: SchemeFamily
    k_products: int

    def __post_init__(self) -> None:
        allowed = _ALLOWED_K[self.family]
        if self.k_products not in allowed:
            raise ValueError(
                f"k_products for {self.family.value} must be one of "
                f"{allowed}, got {self.k_products}")


@dataclass
class CostLedger:
    """Exact product count of one computation (LU terms kept for parity)."""

    products: Fraction = field(default_factory=lambda: Fraction(0))
    lu_factorizations: int = 0
    lu_solves: int = 0

    def charge_product(self, count: int = 1) -> None:
        if count < 0:
            raise ValueError("cost counters only increase")
        self.products += count

    def charge_lu(self, solves: int) -> None:
        if solves < 0:
            raise ValueError("cost counters only increase")
        self.lu_factorizations += 1
        self.lu_solves += solves

    @property
    def total_cost(self) -> Fraction:
        return (self.products + Fraction(self.lu_factorizations, 3)
                + self.lu_solves)


# the Pade baseline's scheme id (schemes.py:87)
PADE8 = SchemeId(SchemeFamily.PADE8, 5)


@dataclass
class CosSinResult:
    cos_part: DenseMatrix
    sin_part: DenseMatrix
    cost: CostLedger


@dataclass
class WaveResult:
    c_part: DenseMatrix
    s_part: DenseMatrix
    cost: CostLedger


class Precision(enum.Enum):
    DOUBLE = "double"
    SINGLE = "single"


UNIT_ROUNDOFF: dict[Precision, float] = {
    Precision.DOUBLE: 2.0 ** -53,
    Precision.SINGLE: 2.0 ** -24,
}


@dataclass(frozen=True)
class ThetaEntry:
    scheme: SchemeId
    theta_cos: float
    theta_sin: float
    cost: Fraction

    @property
    def theta_eff(self) -> float:
        return min(self.theta_cos, self.theta_sin)


@dataclass(frozen=True)
class ThetaTable:
    precision: Precision
    entries: tuple[ThetaEntry, ...]

    def __post_init__(self) -> None:
        if not self.entries:
            raise ValueError("theta table needs at least one entry")
        if any(not (e.theta_cos > 0.0 and e.theta_sin > 0.0)
               for e in self.entries):
            raise ValueError("theta thresholds must be positive")
        for lo, hi in zip(self.entries[:-1], self.entries[1:]):
            if not hi.cost > lo.cost:
                raise ValueError("entries must be sorted by ascending cost")
            if not (hi.theta_cos > lo.theta_cos
                    and hi.theta_sin > lo.theta_sin):
                raise ValueError("thresholds must increase with scheme order")


@dataclass
class ComputationReport:
    result: CosSinResult | WaveResult
    scheme_used: SchemeId
    scaling_exponent: int
    total_products: Fraction


_PREC_CODE = {Precision.DOUBLE: _lib.PREC_DOUBLE,
              Precision.SINGLE: _lib.PREC_SINGLE}


def _library_table(family: SchemeFamily, precision: Precision) -> ThetaTable:
    code = {SchemeFamily.COS_SIN_TAYLOR: _lib.FAMILY_TAYLOR,
            SchemeFamily.WAVE_KERNEL: _lib.FAMILY_WAVE,
            SchemeFamily.PADE8: _lib.FAMILY_PADE}[family]
    tc = np.zeros(8, dtype=np.float64)
    ts = np.zeros(8, dtype=np.float64)
    kk = np.zeros(8, dtype=np.int32)
    count = _lib.check(_lib.lib().csm_theta_table(
        code, _PREC_CODE[precision], tc.ctypes.data_as(ctypes.c_void_p),
        ts.ctypes.data_as(ctypes.c_void_p), kk.ctypes.data_as(ctypes.c_void_p),
        8), "csm_theta_table")
    return ThetaTable(precision, tuple(
        ThetaEntry(SchemeId(family, int(kk[i])), float(tc[i]), float(ts[i]),
                   PADE8_COST if family is SchemeFamily.PADE8
                   else Fraction(int(kk[i])))
        for i in range(count)))


# five products + one LU (1/3) + two solves (driver.py:159, matcore.py:136)
PADE8_COST = Fraction(22, 3)

TAYLOR_TABLE: dict[Precision, ThetaTable] = {
    p: _library_table(SchemeFamily.COS_SIN_TAYLOR, p) for p in Precision}
WAVE_TABLE: dict[Precision, ThetaTable] = {
    p: _library_table(SchemeFamily.WAVE_KERNEL, p) for p in Precision}
PADE_TABLE: dict[Precision, ThetaTable] = {
    p: _library_table(SchemeFamily.PADE8, p) for p in Precision}


def table_for(family: SchemeFamily, precision: Precision) -> ThetaTable:
    if family is SchemeFamily.COS_SIN_TAYLOR:
        return TAYLOR_TABLE[precision]
    if family is SchemeFamily.WAVE_KERNEL:
        return WAVE_TABLE[precision]
    return PADE_TABLE[precision]
