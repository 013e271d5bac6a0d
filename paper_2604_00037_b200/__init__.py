"""B200-native (sm_100a) hot path of alternating cross interpolation (ACI), arxiv 2604.00037.

The product is ``libaci.so`` (C-ABI in ``include/aci.h``); this package is its thin ctypes
binding. See DESIGN.md.
"""
from ._binding import (  # noqa: F401
    AciError, TensorTrain, aci_elementwise, aci_elementwise_batch, workspace_query, limits, prrlu, version, load, EXPORTS,
    LIB_PATH,
    TOL_RELATIVE, TOL_ABSOLUTE, ACI_OK, ACI_NOT_CONVERGED,
)
