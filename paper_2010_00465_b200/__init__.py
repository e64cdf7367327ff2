"""B200-native matrix cosine/sine (arXiv 2010.00465), drop-in for `cossinm`.

The public names of the reference's hot path (pkg/src/cossinm/__init__.py)
with the same signatures, plus batched entry points.  Every computation
runs in libcossin_b200.so (sm_100a kernels: FP64 DMMA by default; the
Ozaki-II engine on the int8 tensor cores is opt-in, see set_engine)
through the C-ABI in include/cossin_b200.h; importing this package fails if
the library has not been built, and computing without a CUDA device raises.
"""
from .api import (
    BatchReport,
    cos_sin,
    cos_sin_batched,
    engine_scope,
    get_engine,
    set_engine,
    identity,
    matrix_from_rows,
    norm1,
    pade8_cos_sin,
    pade_cos_sin,
    pade_cos_sin_batched,
    pythagorean_residual,
    read_matrix,
    select_batch,
    select_scheme,
    taylor_cos_sin,
    taylor_sin9,
    wave_cos_sin,
    wave_cos_sin_batched,
    wave_kernels,
    wave_sin34,
    write_matrix,
)
from . import corpus, plan, verify
from .verify import reference_cos_sin, reference_cos_sin_batched
from .plan import BatchPlan
from .records import (
    PADE8,
    PADE_TABLE,
    TAYLOR_TABLE,
    UNIT_ROUNDOFF,
    WAVE_TABLE,
    ComputationReport,
    CosSinResult,
    CostLedger,
    DenseMatrix,
    MatrixInputError,
    Precision,
    SchemeFamily,
    SchemeId,
    SingularMatrixError,
    ThetaEntry,
    ThetaTable,
    WaveResult,
    table_for,
)

__version__ = "0.1.0"

__all__ = [
    "BatchPlan",
    "BatchReport",
    "ComputationReport",
    "CosSinResult",
    "CostLedger",
    "DenseMatrix",
    "MatrixInputError",
    "Precision",
    "SchemeFamily",
    "SchemeId",
    "SingularMatrixError",
    "PADE8",
    "PADE_TABLE",
    "TAYLOR_TABLE",
    "ThetaEntry",
    "ThetaTable",
    "UNIT_ROUNDOFF",
    "WAVE_TABLE",
    "WaveResult",
    "cos_sin",
    "cos_sin_batched",
    "engine_scope",
    "get_engine",
    "set_engine",
    "identity",
    "matrix_from_rows",
    "norm1",
    "pade8_cos_sin",
    "pade_cos_sin",
    "pade_cos_sin_batched",
    "pythagorean_residual",
    "read_matrix",
    "reference_cos_sin",
    "reference_cos_sin_batched",
    "select_batch",
    "select_scheme",
    "table_for",
    "taylor_cos_sin",
    "taylor_sin9",
    "wave_cos_sin",
    "wave_cos_sin_batched",
    "wave_kernels",
    "wave_sin34",
    "write_matrix",
]
