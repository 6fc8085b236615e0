"""Frame-axis data parallelism.

The acquisition operator A = F_u C is block-diagonal over time frames (one
undersampled Fourier operator per frame, coil maps shared), so rank g owns a contiguous block of
frames and forward/adjoint/normal need no communication.  Only the CG inner products are global.
"""


def frame_shard(L: int, world: int, rank: int):
    """Contiguous, balanced block of frames for ``rank``: returns (frame_offset, L_local)."""
    if world < 1 or not (0 <= rank < world) or L < 0:
        raise ValueError("bad shard request")
    base, extra = divmod(L, world)
    count = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return offset, count
