"""NCCL communicator of the mode-sharded solve, through the library's C ABI (``ss_comm_*``).

The reference keeps every solved mode in one process (``solve_modes`` thread pool,
spectral.py:296-305).  Sharded one process per GPU, the solved modal fields are
gathered to the reconstructing rank with one grouped ncclSend/ncclRecv round
(``ss_comm_gather_modes``): each field lands directly in its global mode slot on the root.

torch.distributed is used only as plumbing: to share the 128-byte NCCL unique id.  The library
opens the NCCL that PyTorch ships (nvidia/nccl wheel) when present, so one NCCL build serves the
process.
"""

from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np

from . import _lib

__all__ = ["ModeComm", "nccl_library_path"]

ID_BYTES = 128


def nccl_library_path():
    """The NCCL shared library PyTorch uses (its nvidia-nccl wheel), or None."""
    try:
        import nvidia.nccl

        for base in list(getattr(nvidia.nccl, "__path__", [])):
            cand = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                return cand
    except Exception:
        pass
    return None


def _prefer_torch_nccl():
    if not os.environ.get("SS_NCCL_LIB"):
        path = nccl_library_path()
        if path:
            os.environ["SS_NCCL_LIB"] = path


class ModeComm:
    """One NCCL communicator over ``world`` ranks (one GPU each)."""

    def __init__(self, rank: int, world: int, device: int, unique_id: bytes):
        if len(unique_id) != ID_BYTES:
            raise ValueError("NCCL unique id must be 128 bytes")
        _prefer_torch_nccl()
        self.rank, self.world, self.device = int(rank), int(world), int(device)
        buf = (C.c_uint8 * ID_BYTES).from_buffer_copy(unique_id)
        h = C.c_void_p()
        _lib.call("ss_comm_create", self.world, self.rank, buf, self.device, C.byref(h))
        self._h = h
        self._finalizer = weakref.finalize(self, _lib.load().ss_comm_destroy, h)

    @staticmethod
    def unique_id() -> bytes:
        _prefer_torch_nccl()
        buf = (C.c_uint8 * ID_BYTES)()
        _lib.call("ss_comm_unique_id", buf)
        return bytes(buf)

    @classmethod
    def from_process_group(cls, device: int, group=None):
        """Create on every rank of the initialised torch.distributed group (id shared by broadcast)."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(rank, world, device, obj[0])

    @classmethod
    def single(cls, device: int):
        """A one-rank communicator (root gathers from itself)."""
        return cls(0, 1, device, cls.unique_id())

    def close(self):
        self._finalizer()

    def gather_modes(self, local, plan, root: int = 0, out=None):
        """Gather per-rank (m_r, N) complex128 fields into the global (sum m_r, N) order of ``plan``.

        ``local`` holds this rank's fields in the order of ``plan[rank]``; on the root the result
        is ``out`` (allocated if None), row ``plan[r][j]`` = field ``j`` of rank ``r``.  Other
        ranks return None.
        """
        torch = _lib.torch_mod()
        if local.dtype != torch.complex128 or local.dim() != 2:
            raise ValueError("local fields must be a 2-D complex128 tensor")
        counts = np.array([len(p) for p in plan], dtype=np.int64)
        if local.shape[0] != counts[self.rank]:
            raise ValueError("local field count does not match plan[rank]")
        dest = np.ascontiguousarray(np.concatenate([np.asarray(p, dtype=np.int64) for p in plan]))
        n = int(local.shape[1])
        local = local.contiguous()
        if self.rank == root and out is None:
            out = torch.empty((int(counts.sum()), n), dtype=torch.complex128, device=local.device)
        _lib.call("ss_comm_gather_modes", self._h, _lib.dptr(local) if local.numel() else None,
                  int(counts[self.rank]), n, n, _lib.dptr(out) if self.rank == root else None,
                  _lib.ptr(counts, C.c_int64), _lib.ptr(dest, C.c_int64), int(root),
                  _lib.stream_ptr(local.device))
        return out if self.rank == root else None

    def reduce_sum(self, values, root: int = 0):
        """Sum a float64 device tensor over ranks into ``root``'s copy (in place; ncclReduce)."""
        if values.dtype.is_complex or values.element_size() != 8:
            raise ValueError("reduce_sum takes a float64 tensor")
        values = values.contiguous()
        _lib.call("ss_comm_reduce_sum", self._h, _lib.dptr(values), values.numel(), int(root),
                  _lib.stream_ptr(values.device))
        return values

    def allreduce_max(self, values):
        """Elementwise max over ranks of a float64 device tensor (in place)."""
        _lib.call("ss_comm_allreduce_max", self._h, _lib.dptr(values), values.numel(), _lib.stream_ptr(values.device))
        return values
