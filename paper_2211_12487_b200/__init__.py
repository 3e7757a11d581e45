"""B200-native TT-ICE / TT-ICE* per-increment update (arXiv 2211.12487).

Hot path: hand-written sm_100a CUDA (DMMA f64 tiles, shared-memory Jacobi
eigen-solve) behind the C ABI in include/ttg.h; this package is the Python
host mirror of the reference's ingest/update/reconstruct API.
"""
from .errors import (ConfigError, DimensionError, Error, FormatError, IndexError_, NumericError,  # noqa: F401
                     ResourceError, StateError)
from .ttstream import (Context, DeviceIncrement, HeuristicConfig, IncrementErrors, IncrementStream,  # noqa: F401
                       TensorTrain, UpdateReport, compression_ratio, default_context, deserialize, list_stream,
                       load_ttc, mean_rre_per_increment, occupancy, per_obs_errors, read_batch,
                       relaxed_tolerance_approx, rpe, rre, save_ttc, serialize, subselect, tt_ice_bootstrap,
                       tt_ice_star_update, tt_ice_update, tt_ice_update_with_tolerances, tt_project,
                       tt_reconstruct, write_batch)
