"""B200-native (sm_100a) data-consistency operator of MS-LLR MR fingerprinting (arxiv 2310.05647).

The compute path is ``libmrfnufft.so`` (hand-written CUDA for sm_100a behind the C-ABI declared in
``include/mrfnufft.h``).  This package is the thin ctypes binding over it (argument marshalling
only) plus the frame-sharding helper.  There is no CPU fallback: importing ``Plan`` without the
built library raises.
"""
from .sharding import frame_shard  # noqa: F401

__all__ = ["frame_shard", "Plan", "Dictionary", "LLR", "MrfError", "lib", "nccl_comm_create", "nccl_comm_destroy"]


def __getattr__(name):
    if name in ("Plan", "Dictionary", "LLR", "MrfError", "lib", "nccl_comm_create", "nccl_comm_destroy"):
        from . import binding
        return getattr(binding, name)
    raise AttributeError(name)
