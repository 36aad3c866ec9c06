"""Collective callbacks for multi-rank handles (``esnmf_comm`` in include/esnmf.h).

* ``nccl_comm`` -- the library's OWN NCCL communicator (esnmf_nccl_comm_create):
  ncclAllGather / ncclAllReduce issued by the library on its stream, no host
  callback, so sharded iterations are captured into CUDA graphs.  The default
  for one process per GPU (bench.py --gpus N).

The library calls ``allgather(ctx, send, recv, bytes_per_rank, stream)`` and
``allreduce_sum_f64(ctx, buf, count, stream)`` with DEVICE pointers, stream
ordered on ``stream``.  Two implementations, both plumbing only:

* ``TorchDistComm`` -- one process per GPU, torch.distributed (NCCL over
  NVLink on B200 boxes); the collective is enqueued on the library's stream.
* ``LoopbackGroup`` -- P logical ranks as P handles in P threads on ONE device
  (tests): the threads meet at a host barrier and copy device buffers; no
  kernel ever waits on another rank.
"""
from __future__ import annotations

import ctypes
import threading

from .esnmf import ALLGATHER_FN, ALLREDUCE_FN, esnmf_comm


class _DevBuf:
    """Zero-copy torch view of raw device memory (``__cuda_array_interface__``)."""

    def __init__(self, ptr: int, nbytes: int, typestr: str = "|u1", itemsize: int = 1):
        self.__cuda_array_interface__ = {"shape": (nbytes // itemsize,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def dev_tensor(ptr: int, nbytes: int, dtype="u8"):
    import torch

    ts, sz = {"u8": ("|u1", 1), "f64": ("<f8", 8)}[dtype]
    return torch.as_tensor(_DevBuf(ptr, nbytes, ts, sz), device="cuda")


def _make_struct(ag, ar):
    c = esnmf_comm()
    c.ctx = None
    c.allgather = ALLGATHER_FN(ag)
    c.allreduce_sum_f64 = ALLREDUCE_FN(ar)
    return c


class TorchDistComm:
    """torch.distributed collectives on the library's stream."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.struct = _make_struct(self._allgather, self._allreduce)

    def _allgather(self, ctx, send, recv, nbytes, stream):
        import torch

        try:
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                s = dev_tensor(send, nbytes)
                r = dev_tensor(recv, nbytes * self.world)
                self.dist.all_gather_into_tensor(r, s, group=self.group)
            return 0
        except Exception as e:  # pragma: no cover - reported through ESNMF_ECOMM
            print("esnmf allgather failed:", e)
            return 1

    def _allreduce(self, ctx, buf, count, stream):
        import torch

        try:
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                b = dev_tensor(ctypes.cast(buf, ctypes.c_void_p).value, 8 * count, "f64")
                self.dist.all_reduce(b, group=self.group)
            return 0
        except Exception as e:  # pragma: no cover
            print("esnmf allreduce failed:", e)
            return 1


def nccl_comm(device: int, group=None):
    """The library's own NCCL communicator over a torch.distributed group: rank 0
    draws the NCCL unique id (esnmf_nccl_unique_id), the group broadcasts it
    (any backend: gloo on CPU, NCCL on GPUs), every rank creates the communicator
    collectively.  Returns an ``esnmf.NcclComm`` (``.struct`` for ESNMF(comm=...))."""
    import torch.distributed as dist

    from .esnmf import NcclComm, esnmf_nccl_unique_id

    uid = [esnmf_nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(uid, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return NcclComm(dist.get_world_size(group), dist.get_rank(group), uid[0], device)


def broadcast_nccl_id(group=None) -> bytes:
    """Rank 0's NCCL unique id on every rank of the group (host logic of nccl_comm)."""
    import torch.distributed as dist

    from .esnmf import esnmf_nccl_unique_id

    uid = [esnmf_nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(uid, src=0, group=group)
    return uid[0]


class LoopbackGroup:
    """P logical ranks on one device (P handles driven from P threads)."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.comms = [self._rank_comm(r) for r in range(world)]

    def _rank_comm(self, rank):
        def ag(ctx, send, recv, nbytes, stream):
            import torch

            torch.cuda.ExternalStream(stream).synchronize()
            self.slots[rank] = send
            self.barrier.wait()
            out = dev_tensor(recv, nbytes * self.world)
            for p in range(self.world):
                out[p * nbytes:(p + 1) * nbytes].copy_(dev_tensor(self.slots[p], nbytes))
            torch.cuda.synchronize()
            self.barrier.wait()
            return 0

        def ar(ctx, buf, count, stream):
            import torch

            torch.cuda.ExternalStream(stream).synchronize()
            ptr = ctypes.cast(buf, ctypes.c_void_p).value
            self.slots[rank] = ptr
            self.barrier.wait()
            total = sum(dev_tensor(self.slots[p], 8 * count, "f64").clone() for p in range(self.world))
            torch.cuda.synchronize()
            self.barrier.wait()
            dev_tensor(ptr, 8 * count, "f64").copy_(total)
            torch.cuda.synchronize()
            self.barrier.wait()
            return 0

        return _make_struct(ag, ar)
