"""B200-native (sm_100a) SolveBak column sweep — drop-in for the solve path of
the reference package ``baksolve`` 0.1.0 (arXiv 2104.12570, Algorithm 1).

    from paper_2104_12570_b200 import SolveConfig, solve_bak
    rep = solve_bak(x, y, SolveConfig(max_iter=100, tol=0))

Names mirror ``baksolve`` (reference __init__.py:9-10): SolveConfig,
SolveReport, solve_bak, coordinate_update, residual_norm, DRIFT_TOL.
The blocked solver of the reference's bakp.py (Algorithm 2): solve_bakp,
block_deltas, BlockConfig, DivergenceError, DIVERGENCE_FACTOR.
Greedy column scoring / forward selection of select.py:
score_all_columns, select_features, FeatureSelectConfig,
FeatureSelectionReport, SelectionExhaustedError, REFITS.
BAKM / CSV matrix files of matio.py (§8f row 4): save_matrix, load_matrix,
load_vector, MatrixFormatError, plus load_matrix_pinned / load_matrix_device.
Extension: solve_bak_batched for many independent small systems.
"""

from .bak import (DRIFT_TOL, ORDERINGS, BatchSolveReport, DeviceBatch, DeviceMatrix, SolveConfig, SolveReport,
                  colnorms, coordinate_update, residual_norm, solve_bak, solve_bak_batched, to_device_batch,
                  to_device_matrix)
from .bakp import DIVERGENCE_FACTOR, BlockConfig, DivergenceError, block_deltas, solve_bakp
from .matio import (FORMATS, MAGIC, MatrixFormatError, load_matrix, load_matrix_device, load_matrix_pinned,
                    load_vector, save_matrix)
from .select import (REFITS, FeatureSelectConfig, FeatureSelectionReport, SelectionExhaustedError,
                     score_all_columns, select_features)

__version__ = "0.1.0"

__all__ = ["FORMATS", "MAGIC", "MatrixFormatError", "load_matrix", "load_matrix_device", "load_matrix_pinned",
           "load_vector", "save_matrix", "REFITS", "FeatureSelectConfig", "FeatureSelectionReport", "SelectionExhaustedError", "score_all_columns",
           "select_features",
           "DIVERGENCE_FACTOR", "DRIFT_TOL", "ORDERINGS", "BatchSolveReport", "BlockConfig", "DeviceBatch",
           "DeviceMatrix", "DivergenceError", "SolveConfig", "SolveReport", "block_deltas", "colnorms",
           "coordinate_update", "residual_norm", "solve_bak", "solve_bak_batched", "solve_bakp", "to_device_batch",
           "to_device_matrix"]
