"""paper_1510_05237_b200 -- B200-native hot path of enforced-sparse ALS NMF
(Gavin, Gadepally, Kepner, arXiv 1510.05237).

The product is ``libesnmf.so`` (CUDA, sm_100a) behind the C ABI in
``include/esnmf.h``; this package is its ctypes binding.  See DESIGN.md.
"""
from . import checkpoint, comm  # noqa: F401
from .esnmf import (  # noqa: F401
    ESNMF,
    ESNMFError,
    ESNMF_SIDE_U,
    ESNMF_SIDE_V,
    ESNMF_ENFORCE_COLUMN,
    ESNMF_ENFORCE_MATRIX,
    ESNMF_T_SAME,
    ESNMF_T_UNLIMITED,
    SIGNATURES,
    esnmf_create,
    esnmf_destroy,
    esnmf_error,
    esnmf_get_gram,
    esnmf_get_info,
    esnmf_get_ls,
    esnmf_get_U,
    esnmf_get_V,
    esnmf_half_step,
    esnmf_iterate,
    esnmf_options_init,
    esnmf_partition_rows,
    esnmf_phase_times,
    esnmf_profile,
    esnmf_records,
    esnmf_residual,
    esnmf_set_factor,
    esnmf_truncate,
    esnmf_topic_accuracy,
    esnmf_version,
    lib,
)
