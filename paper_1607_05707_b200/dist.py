"""Host transport plugin (irgl_transport, include/irgl/rt.h) over a torch.distributed process
group: one process per GPU without NCCL in the runtime — the round headers and payloads of a
vertex-partitioned graph go through the group's all_gather / all_to_all_single (gloo moves them
between host buffers; the runtime stages them in pinned memory).  torch is plumbing here: the
graph operators and the round protocol are the runtime's (wl_graph_rounds_dist, api.cu).

    pg = torch.distributed.new_group(backend="gloo")
    ctx = Context(transport=TorchTransport(pg, device=local_rank))
"""
from __future__ import annotations

import ctypes as C
import traceback

import torch
import torch.distributed as dist

ALLGATHER = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)
ALLTOALLV = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p,
                        C.POINTER(C.c_int64))


class Transport(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allgather", ALLGATHER), ("alltoallv", ALLTOALLV)]


def _host_bytes(addr: int, n: int) -> torch.Tensor:
    """uint8 tensor viewing n bytes of host memory at addr (an empty tensor for n == 0)."""
    if n == 0:
        return torch.empty(0, dtype=torch.uint8)
    return torch.frombuffer((C.c_uint8 * n).from_address(addr), dtype=torch.uint8)


class TorchTransport:
    """irgl_transport over `group` (default: the world group).  Keep the object alive as long as
    the Context that uses it (the Context holds a reference)."""

    def __init__(self, group=None, device: int = 0):
        self.group = group
        self.device = device
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        R = self.nranks

        def allgather(_user, send, recv, nbytes):
            try:
                src = _host_bytes(send, nbytes).clone()
                outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(R)]
                dist.all_gather(outs, src, group=group)
                for r, t in enumerate(outs):
                    if nbytes:
                        C.memmove(recv + r * nbytes, t.data_ptr(), nbytes)
                return 0
            except Exception:  # errors are values across the C boundary
                traceback.print_exc()
                return 1

        def alltoallv(_user, send, send_bytes, recv, recv_bytes):
            try:
                ss = [int(send_bytes[r]) for r in range(R)]
                rs = [int(recv_bytes[r]) for r in range(R)]
                src = _host_bytes(send, sum(ss)).clone()
                out = torch.empty(sum(rs), dtype=torch.uint8)
                dist.all_to_all_single(out, src, output_split_sizes=rs, input_split_sizes=ss,
                                       group=group)
                if sum(rs):
                    C.memmove(recv, out.data_ptr(), sum(rs))
                return 0
            except Exception:
                traceback.print_exc()
                return 1

        self._cb = (ALLGATHER(allgather), ALLTOALLV(alltoallv))  # keep the thunks alive
        self.struct = Transport(None, self._cb[0], self._cb[1])
