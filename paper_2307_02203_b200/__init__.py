"""B200-native neural dependence fields: the reference-to-all-vertices NDF query
and its ground-truth estimators (Pearson, KSG-MI) on hand-written sm_100a kernels.

Drop-in for the hot path of the reference ``ndf`` package: same public names
and signatures for the query (``NdfModel.forward``, ``reconstruct_field``) and
the estimators (``pearson*``, ``ksg_mi``, ``ground_truth_field``); the compute
runs in ``libndf_b200.so`` (C-ABI, include/ndf_b200.h).  There is no CPU
fallback: without the library or a B200 the compute calls raise DeviceError.
"""

from .ensemble import (DeviceEnsemble, EnsembleField, GridDomain, load_ensemble,
                       load_ensemble_device, sample_at,
                       sample_many, save_ensemble)
from .errors import (ConfigError, CorruptFileError, DataError, DegenerateSampleError,
                     DeviceError, FormatError, ModelCorruptError, NdfError, NotFoundError,
                     ParameterError, ShapeError, TrainingError, UnknownVariableError)
from .measures import (CorrelationMeasure, FieldGrid, digamma, gaussian_mi_analytic,
                       grid_positions, ground_truth_field, ground_truth_field_device, ksg_mi,
                       ksg_rows, load_field_grid, pair_estimators_device, pearson,
                       pearson_against, pearson_rowwise, save_field_grid)
from .model import DeviceModel, ModelSpec, NdfModel, as_model, load_model, save_model
from .service import (ROLE_MU, ROLE_NU, ComparisonResult, FieldResponse, benchmark,
                      compare_to_ground_truth, difference_field, psnr,
                      difference_response, forward, matrix_reconstruct, reconstruct_field,
                      reconstruct_field_device, reconstruct_multi_device, reconstruct_response)
from .training import sample_pairs_with_targets, targets, targets_device

__version__ = "0.1.0"

__all__ = [
    "ConfigError", "CorrelationMeasure", "CorruptFileError", "DataError", "DegenerateSampleError",
    "DeviceEnsemble", "DeviceError", "DeviceModel", "EnsembleField", "FieldGrid", "FormatError",
    "GridDomain", "ModelCorruptError", "ModelSpec", "NdfError", "NdfModel", "NotFoundError",
    "ParameterError", "ROLE_MU", "ROLE_NU", "ShapeError", "TrainingError", "UnknownVariableError",
    "as_model", "benchmark", "difference_field", "forward", "digamma", "gaussian_mi_analytic", "grid_positions",
    "ground_truth_field", "ground_truth_field_device", "ksg_mi", "ksg_rows", "load_ensemble",
    "load_ensemble_device",
    "load_field_grid", "load_model", "matrix_reconstruct", "pair_estimators_device", "pearson",
    "pearson_against", "pearson_rowwise", "reconstruct_field", "reconstruct_field_device",
    "reconstruct_multi_device", "sample_at", "FieldResponse", "reconstruct_response",
    "difference_response",
    "sample_many", "save_ensemble", "save_field_grid", "save_model",
    "sample_pairs_with_targets", "targets", "targets_device",
    "ComparisonResult", "compare_to_ground_truth", "psnr",
]
