"""B200-native Compact-Table propagation (arXiv 2507.18413) -- the data-parallel
hot path behind a C ABI (include/ct.h), with a thin Python binding.

    from paper_2507_18413_b200 import Table
"""
from . import ct  # noqa: F401  (C names: ct.ct_create, ct.ct_propagate, ...)
from .ct import (  # noqa: F401
    CT_OK, CT_FAIL, CT_PENDING, CT_EINVAL, CT_ENOMEM, CT_ECUDA, CT_ENCCL, CT_ESTATE,
    CT_POLICY_AUTO, CT_POLICY_DOM, CT_POLICY_DELTA, CTError,
    CT_TABLE_POSITIVE, CT_TABLE_SHORT, CT_TABLE_NEGATIVE, CT_STAR,
)
from .api import Table, State, Batch, Model, HostTable, HostState  # noqa: F401
