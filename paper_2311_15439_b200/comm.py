"""Communicator of the batch-sharded training step (sxen_comm_* in include/sxen_cuda.h).

The reference merges its worker threads' accumulators in worker order before the optimizer steps
(src/trainer.cpp:101-128); across GPUs the workers are ranks and the merge is a SUM all-reduce.  Two transports:
``Comm.nccl`` (one process per GPU; the id travels over any side channel -- ``Comm.from_torch`` uses the process group a
torchrun launch already has) and ``Comm.local`` (all ranks in this process, one host thread each; the library's own
peer-memory kernel, ranks may share a device)."""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence

from . import _abi
from .errors import raise_for


class CommError(RuntimeError):
    """SXEN_NCCL_ERROR: the exchange between ranks failed (no reference analogue)."""


def _check(lib, st: int) -> None:
    if st == _abi.NCCL_ERROR:
        raise CommError(lib.sxen_last_error().decode())
    raise_for(lib, st)


class Comm:
    def __init__(self, handle: C.c_void_p):
        from . import lib
        self._lib = lib
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.sxen_comm_destroy(self._h)
            self._h = None

    @staticmethod
    def unique_id() -> bytes:
        """ncclGetUniqueId: rank 0 draws it and hands the 128 bytes to the other ranks."""
        from . import lib
        buf = C.create_string_buffer(128)
        _check(lib, lib.sxen_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, unique_id: bytes, world: int, rank: int, device: int) -> "Comm":
        from . import lib
        if len(unique_id) != 128:
            raise ValueError("comm: an ncclUniqueId is 128 bytes")
        h = C.c_void_p()
        _check(lib, lib.sxen_comm_create(C.create_string_buffer(unique_id, 128), world, rank, device, C.byref(h)))
        return cls(h)

    @classmethod
    def from_torch(cls, device: int, group=None) -> "Comm":
        """One NCCL communicator per rank of an initialised torch.distributed group (any backend carries the id)."""
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        box = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        return cls.nccl(box[0], world, rank, device)

    @classmethod
    def local(cls, devices: Sequence[int]) -> List["Comm"]:
        """All ranks in this process (drive each from its own thread); devices[r] is rank r's device."""
        from . import lib
        n = len(devices)
        arr = (C.c_int32 * n)(*devices)
        out = (C.c_void_p * n)()
        _check(lib, lib.sxen_comm_create_local(n, arr, out))
        return [cls(C.c_void_p(out[i])) for i in range(n)]

    def abort(self) -> None:
        """Marks the group broken so peers leave their collectives with CommError instead of waiting for a failed rank."""
        _check(self._lib, self._lib.sxen_comm_abort(self._h))

    def info(self):
        w, r, d, k = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _check(self._lib, self._lib.sxen_comm_info(self._h, C.byref(w), C.byref(r), C.byref(d), C.byref(k)))
        return {"world": w.value, "rank": r.value, "device": d.value, "kind": "nccl" if k.value == 0 else "local"}

    @property
    def world(self) -> int:
        return self.info()["world"]

    @property
    def rank(self) -> int:
        return self.info()["rank"]

    def allreduce(self, tensor, stream=None) -> None:
        """In-place SUM over the ranks of a contiguous float32 / float64 CUDA tensor, ordered on ``stream``."""
        import torch
        from .encoding import _stream_ptr
        if not tensor.is_cuda or not tensor.is_contiguous():
            raise ValueError("all-reduce: a contiguous CUDA tensor is required")
        typ = {torch.float32: _abi.COORD_F32, torch.float64: _abi.COORD_F64}.get(tensor.dtype)
        if typ is None:
            raise ValueError("all-reduce: float32 or float64 only")
        _check(self._lib, self._lib.sxen_comm_allreduce(self._h, C.c_void_p(tensor.data_ptr()), tensor.numel(), typ,
                                                        _stream_ptr(stream, tensor.device)))
