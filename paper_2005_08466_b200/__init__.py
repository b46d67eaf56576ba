"""B200-native partitioned NDRange runtime for HaoCL (arxiv 2005.08466).

The reference's OpenCL-like host API (HostContext) over an in-process CUDA
C-ABI (``include/hcl_cabi.h``) with hand-written sm_100a kernels. See
DESIGN.md for the path, the boundary and the kernels.
"""
from ._native import HaoclError  # noqa: F401
from .runtime import (  # noqa: F401
    Handle,
    HandleKind,
    HostContext,
    KernelTask,
    Scheduler,
    SchedulerOptions,
    TimingBreakdown,
    TimingFragment,
    spmv_partition_ranges,
    split_ranges,
)
