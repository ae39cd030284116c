"""fdsweep_b200 — B200-native (sm_100a) hot path of arXiv:1511.04355's toolkit.

Python mirror of the reference's solver / fitting / inversion interface
(proj/include/fdsweep/{systems,vecfit,laplace,afs}.hpp), calling the CUDA
library ``libfdsweep_b200.so`` through its C-ABI (include/fdsweep_b200.h).
There is no CPU fallback: importing the package works without a GPU, but
every compute call raises if the library is missing or the device fails.
"""
from .api import (  # noqa: F401
    BemSystem,
    ConvergenceError,
    CudaError,
    Error,
    IoError,
    NumericError,
    RationalModel,
    ValidationError,
    channel_errors,
    eval_model,
    fit_error_evf,
    fsm_invert,
    identify_residues,
    kernel_launches,
    lib,
    library_path,
    rational_invert,
    relocate_poles,
    run_afs,
    select_new_frequency,
    vector_fit,
    zgesv_batch,
)
