"""Cross-rank exchanges of the v-MFA iteration over torch.distributed
(SURVEY §8(e)); the caller owns the process group (NCCL over NVLink on the
GPU box, gloo in the CPU tests).

Per main iteration (include/vmfa_b200.h phase API):
  phase_estep_local -> cooc exchange -> phase_estep_finish -> phase_stats_local
  -> allreduce(STATS) -> phase_update -> phase_free_energy_local
  -> allreduce(SCALARS)

The co-occurrence exchange is either the dense C x C table (all-reduce of
exact int64 sums) or, for large C, the sparse owner-routed lists: every rank
sends the (c, c~) entries of component c to the rank owning c (block
ownership [rC/p, (r+1)C/p)), the owner reduces and selects g_c, and the
selected rows are combined by an int32 all-reduce (each row is non-zero on
its owner only). Both reproduce the single-rank g bit for bit: the sums are
exact integers.
"""
from __future__ import annotations

import numpy as np

XCHG_COOC, XCHG_STATS, XCHG_SCALARS, XCHG_G = 0, 1, 2, 3
_TYPESTR = {0: "<i8", 1: "<f8", 2: "<i4"}


class _DevArray:
    """A device pointer as a torch-consumable CUDA array."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = dict(shape=(n,), typestr=typestr, data=(ptr, False), version=3)


def device_view(ptr: int, n: int, typestr: str):
    import torch
    if n == 0:
        return torch.empty(0, dtype={"<i8": torch.int64, "<f8": torch.float64, "<i4": torch.int32}[typestr],
                           device="cuda")
    return torch.as_tensor(_DevArray(ptr, n, typestr), device="cuda")


def _host_staged(group=None) -> bool:
    """gloo reduces host memory: device tensors are staged through the host."""
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def all_reduce(t, group=None):
    import torch.distributed as dist
    if t.is_cuda and _host_staged(group):
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, group=group)


def owner_ranges(C: int, world: int):
    """Block ownership of components: rank r owns [floor(rC/p), floor((r+1)C/p))."""
    return [(r * C // world, (r + 1) * C // world) for r in range(world)]


def route_lists(arrays, counts, group=None):
    """All-to-all of parallel 1-D tensors: the first counts[0] entries of every
    array go to rank 0, the next counts[1] to rank 1, ... Returns the received
    arrays (concatenated in source-rank order) and the received counts."""
    import torch
    import torch.distributed as dist
    dev = arrays[0].device
    if dev.type == "cuda" and _host_staged(group):
        out, rc = route_lists([a.cpu() for a in arrays], counts, group)
        return [o.to(dev) for o in out], rc
    send = torch.as_tensor(np.asarray(counts, np.int64), device=dev)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    rc = [int(v) for v in recv.cpu()]
    sc = [int(v) for v in np.asarray(counts)]
    out = []
    for a in arrays:
        o = torch.empty(sum(rc), dtype=a.dtype, device=dev)
        dist.all_to_all_single(o, a.contiguous(), output_split_sizes=rc, input_split_sizes=sc, group=group)
        out.append(o)
    return out, rc


def _on_ctx_stream(sess):
    """Collectives on the context's own stream: the phase calls enqueue their
    kernels there, so an all-reduce issued on it is ordered after the
    producer and before the consumer without a host synchronisation (NCCL
    orders its work on torch's current stream)."""
    import torch
    return torch.cuda.stream(torch.cuda.ExternalStream(sess.stream()))


def allreduce_buffer(sess, which: int, group=None):
    """Sum an exchange buffer across ranks. Stream contract: the reduction is
    enqueued on the context's stream (NCCL) and the call returns once it is
    complete, so the next phase call may read the buffer."""
    import torch
    ptr, n, dt = sess.exchange_buffer(which)
    t = device_view(ptr, n, _TYPESTR[dt])
    with _on_ctx_stream(sess):
        all_reduce(t, group)
    torch.cuda.ExternalStream(sess.stream()).synchronize()


def cooc_exchange(sess, rank: int, world: int, group=None):
    """The co-occurrence exchange between phase_estep_local and
    phase_estep_finish: dense all-reduce, or the sparse owner-routed lists."""
    import torch
    if not sess.cooc_sparse():
        allreduce_buffer(sess, XCHG_COOC, group)
        return
    (pk, pc, ph, pl), counts = sess.cooc_local_list(world)
    n = int(counts.sum())
    # keys are u32 (c << b | c~ < 2^32): moved as int32 bit patterns
    arrays = [device_view(pk, n, "<i4"), device_view(pc, n, "<i8"), device_view(ph, n, "<i8"),
              device_view(pl, n, "<i8")]
    got, rc = route_lists(arrays, counts, group)
    torch.cuda.synchronize()
    sess.cooc_select([int(t.data_ptr()) if t.numel() else 0 for t in got], sum(rc), rank, world)
    allreduce_buffer(sess, XCHG_G, group)
