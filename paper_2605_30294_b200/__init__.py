"""B200-native RaFI work-item forwarding (arXiv 2605.30294).

The product is the C-ABI library ``librafi.so`` (include/rafi.h,
include/rafi_device.cuh) built from ``csrc/`` for sm_100a; ``rafi`` is its
thin ctypes binding.  Nothing here imports the test oracle.
"""
from .rafi import (Context, RafiError, lib, nccl_comm_destroy, nccl_comm_init, nccl_unique_id,  # noqa: F401
                   plan)
from . import rafi  # noqa: F401

__all__ = ["Context", "RafiError", "lib", "nccl_unique_id", "nccl_comm_init", "nccl_comm_destroy", "plan", "rafi"]
