"""emm — a B200-native (sm_100a) SGEMM: C <- alpha*op(A)*op(B) + beta*C.

Thin Python binding over the C ABI in ``include/emm.h`` (libemm.so in this
directory).  Argument marshalling only: every step of the product runs in the
library's CUDA kernels.  There is no CPU fallback — if the library is missing
the import of the binding raises.
"""
from .emm import (  # noqa: F401
    EmmError,
    MATH,
    lib,
    launch_count,
    profile_enable,
    profile_read,
    release_cache,
    row_partition,
    sgemm,
    sgemm_ex,
    sgemm_host,
    sgemm_ptr,
    strerror,
    version,
    workspace_bytes,
    Comm,
    broadcast_unique_id,
    get_unique_id,
    multi_panel_cols,
    sgemm_multi,
    local_comms,
)
