"""B200-native ACP-SGD hot path (arXiv 2306.08881, Alg. 2).

The compute path is ``lib/libacp.so`` (sm_100a kernels + NCCL) behind the C
ABI in ``include/acp.h``; this package only marshals arguments. Importing it
loads the library and fails loudly if it has not been built.
"""
from ._lib import (load as _load, AcpError, ACP_NO_EF, ACP_NO_REUSE, ACP_SUM, ACP_POWERSGD,  # noqa: F401
                   ACP_BUCKETED, ACP_CHECK_FINITE, ACP_E_NONFINITE, LIB_PATH, EXPORTED)
from .acp import (AcpContext, nccl_comm_from_group, nccl_comm_destroy, broadcast_unique_id,  # noqa: F401
                  nccl_comm_single, plan_host, DEFAULT_BUCKET_BYTES)

_load()
