"""ZeRO-3 data parallelism around the update phase.

One process per GPU.  Rank r owns ``shard(P, N, SG)[r]`` (core.py:139-170):
its fp32 optimizer state, its grads and its slice of the working copy.  The
update phase itself is rank-local — no collective on the
data path.  Around it:

* before: **reduce-scatter** of the bf16 grads — fused into the phase
  (``PeerGrads``: K1 sums every rank's grads of the shard over NVLink as it
  streams the state), or bucketed per subgroup index j (bucket j = every
  rank's subgroup j; an NCCL all-to-all hands each rank its pieces, summed
  locally in rank order) — both with the same rounding, so the two modes
  train to the same bits;
* after: **all-gather** of the bf16 working copy, bucketed the same way.
  ``gather_params_overlapped`` makes a comm stream wait on the *engine event*
  of the action that finalises subgroup j's working copy (its GPU_UPDATE, or
  its H2D_PARAMS16 for a host subgroup) and launches bucket j's all-gather
  right away, so gathers overlap the rest of the phase.

Full-model buffers use the model's flat (rank-major) layout padded to
``N * ceil(P/N)``; the last rank's missing tail is zero padding so every
collective has equal counts.  NCCL over NVLink/NVSwitch is the product
backend; the same code runs on gloo (CPU tests; 16-bit tensors exchanged as
raw bits).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .state import Subgroup, shard


@dataclass(frozen=True)
class ShardLayout:
    """Where every rank's subgroups live in the padded full-model buffer."""

    total_params: int
    world: int
    subgroup_size: int
    per_rank: int  # ceil(P / N): every rank's padded share
    ranks: tuple[tuple[Subgroup, ...], ...]

    @classmethod
    def build(cls, total_params: int, world: int, subgroup_size: int) -> "ShardLayout":
        parts = shard(total_params, world, subgroup_size)
        return cls(total_params, world, subgroup_size, math.ceil(total_params / world),
                   tuple(tuple(p) for p in parts))

    @property
    def padded_total(self) -> int:
        return self.per_rank * self.world

    @property
    def num_buckets(self) -> int:
        """Bucket count: subgroups of the fullest rank (rank 0)."""
        return len(self.ranks[0])

    def bucket_span(self, j: int) -> tuple[int, int]:
        """(start, size) of bucket j inside one rank's padded share; the size
        is rank 0's subgroup j (padding covers shorter ranks)."""
        sg = self.ranks[0][j]
        return sg.start, sg.size

    def global_offset(self, rank: int, local_start: int) -> int:
        return rank * self.per_rank + local_start

    def rank_of_bucket_piece(self, rank: int, j: int) -> tuple[int, int]:
        """(valid elements, padding) of rank's piece of bucket j."""
        start, size = self.bucket_span(j)
        mine = sum(g.size for g in self.ranks[rank])
        valid = max(0, min(size, mine - start))
        return valid, size - valid


class BucketedCollectives:
    """Bucketed reduce-scatter / all-gather over a torch process group."""

    def __init__(self, layout: ShardLayout, group=None) -> None:
        import torch.distributed as dist

        self.layout = layout
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.world != layout.world:
            raise ValueError(f"layout is for {layout.world} ranks, group has {self.world}")
        self.backend = dist.get_backend(group)

    def _views(self, full, j):
        start, size = self.layout.bucket_span(j)
        return [full[self.layout.global_offset(r, start): self.layout.global_offset(r, start) + size]
                for r in range(self.world)]

    def reduce_scatter_bucket(self, full_grads, out, j: int, scale: float = 1.0) -> None:
        """Bucket j of the grad reduce-scatter: ``out`` (this rank's piece of
        bucket j) = the rank-order sum of every rank's grads for it, with the
        declared rounding of ``oracle.reduce_scatter`` / ``dos_gsrc`` (fp32
        adds in rank order, one rounding to the grad dtype, then the scale
        rounded once more) — bit-identical to the reduce-scatter fused into
        the phase (``PeerGrads``).

        The collective only moves bytes: an all-to-all hands each rank every
        rank's 16-bit piece of its shard (the same (N-1)/N traffic as a ring
        reduce-scatter, over NVLink under NCCL), and the sum runs on this
        rank in rank order (``dos_reduce_scatter_cuda``).  A reduction inside
        NCCL would add in its own order and round in 16 bits at every hop."""
        import torch
        import torch.distributed as dist

        views = self._views(full_grads, j)
        size = views[0].numel()
        if out.numel() != size:
            raise ValueError(f"bucket {j} piece has {size} elements, out has {out.numel()}")
        if out.element_size() != 2:
            raise TypeError("the grads must be half precision")
        recv = torch.empty(self.world * size, dtype=out.dtype, device=out.device)
        parts = list(recv.split(size))
        if self.backend == "nccl":
            dist.all_to_all(parts, [v.contiguous() for v in views], group=self.group)
        else:  # gloo: 16-bit floats unsupported and CUDA tensors staged: exchange the raw bits on the host
            send = torch.cat([v.contiguous().view(torch.uint8).cpu() for v in views])
            got = torch.empty_like(send)
            dist.all_to_all_single(got, send, group=self.group)
            recv.view(torch.uint8).copy_(got)
        reduce_in_rank_order(parts, out, scale)

    def all_gather_bucket(self, full_params, mine, j: int):
        """Every rank's piece of bucket j into the full-model buffer."""
        import torch
        import torch.distributed as dist

        views = self._views(full_params, j)
        if self.backend == "nccl":
            return dist.all_gather(views, mine, group=self.group, async_op=True)
        # gloo: gather exactly-widened fp32 copies (16-bit floats unsupported)
        src = mine.contiguous()
        if src.element_size() == 2 and src.is_floating_point():
            wide = [torch.empty(v.numel(), dtype=torch.float32, device=v.device) for v in views]
            dist.all_gather(wide, src.float(), group=self.group)
            for v, w in zip(views, wide):
                v.copy_(w.to(v.dtype))
        else:
            dist.all_gather(views, src, group=self.group)
        return None

    def reduce_scatter_all(self, full_grads, shard_grads, scale: float | None = None) -> None:
        """All buckets; ``shard_grads`` is this rank's padded share (per_rank).
        ``scale`` (e.g. 1/N to average) is applied inside the reduction, with
        the fused path's rounding."""
        for j in range(self.layout.num_buckets):
            start, size = self.layout.bucket_span(j)
            self.reduce_scatter_bucket(full_grads, shard_grads[start:start + size], j,
                                       1.0 if scale is None else float(scale))

    def all_gather_all(self, full_params, shard_params):
        works = []
        for j in range(self.layout.num_buckets):
            start, size = self.layout.bucket_span(j)
            works.append(self.all_gather_bucket(full_params, shard_params[start:start + size], j))
        for w in works:
            if w is not None:
                w.wait()


def reduce_in_rank_order(parts, out, scale: float = 1.0) -> None:
    """``out`` = lowp(sum of ``parts`` in list order, fp32 RN adds), then
    lowp(f32(that) * f32(scale)) if scale != 1 — ``oracle.reduce_scatter``'s
    rule.  CUDA tensors: one ``dos_reduce_scatter_cuda`` launch on the
    current stream (up to DOS_MAX_PEERS + 1 sources per launch); host tensors
    (gloo CPU tests): the same arithmetic in torch."""
    import ctypes as C

    import torch

    from . import _native as N

    if out.is_cuda and len(parts) <= N.DOS_MAX_PEERS + 1:
        dt = N.DOS_BF16 if out.dtype == torch.bfloat16 else N.DOS_F16
        srcs = (C.c_void_p * len(parts))(*[p.data_ptr() for p in parts])
        N.check(N.lib().dos_reduce_scatter_cuda(out.data_ptr(), srcs, len(parts), dt, float(scale), out.numel(),
                                                torch.cuda.current_stream(out.device).cuda_stream))
        return
    acc = parts[0].float()
    for p in parts[1:]:
        acc = acc + p.float()  # fp32 RN, rank order
    r = acc.to(out.dtype)  # RNE
    if scale != 1.0:
        r = (r.float() * torch.tensor(scale, dtype=torch.float32, device=r.device)).to(out.dtype)
    out.copy_(r)


def _ipc_bases(buf, group=None) -> dict[int, int]:
    """Exchange CUDA IPC handles of ``buf`` (a device tensor) with every rank
    of ``group`` and map theirs: rank -> base address of that rank's ``buf``
    in this process (this rank maps to its own pointer)."""
    import ctypes as C

    import torch.distributed as dist

    from . import _native as N

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    handle = C.create_string_buffer(64)
    off = C.c_uint64()
    N.check(N.lib().dos_ipc_export(buf.data_ptr(), handle, C.byref(off)))
    everyone = [None] * world
    dist.all_gather_object(everyone, (rank, handle.raw, off.value), group=group)
    bases = {rank: buf.data_ptr()}
    for r, h, o in everyone:
        if r == rank:
            continue
        ptr = C.c_void_p()
        N.check(N.lib().dos_ipc_import(h, o, C.byref(ptr)))
        bases[r] = ptr.value
    return bases


@dataclass(frozen=True)
class GradSources:
    """The fused reduce-scatter's inputs for one rank (include/dos.h
    ``dos_state_desc.src_g``): ``ptrs[r]`` is where this rank's shard starts
    in rank r's full-model grad buffer, in rank order (``ptrs[self_rank]`` is
    the local one); ``scale`` is applied after the sum (1/N to average)."""

    ptrs: tuple[int, ...]
    self_rank: int
    scale: float = 1.0


class PeerGrads:
    """Every rank's full-model grad buffer mapped into this process (CUDA IPC,
    one node): the sources of the reduce-scatter fused into the update phase.

    Replaces the bucketed NCCL reduce-scatter before the phase: K1 reads the
    shard's grads of every rank over NVLink and sums them in rank order while
    it streams the fp32 state, and each host subgroup's grads are reduced on
    the device right before their D2H flush.  The caller synchronises the
    ranks before the phase (every backward done) and after it (no rank
    overwrites grads a peer is still reading).
    """

    def __init__(self, full_grads, layout: ShardLayout, group=None) -> None:
        import torch.distributed as dist

        from . import _native as N

        if full_grads.element_size() != 2:
            raise TypeError("the full-model grad buffer must be half precision")
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        if self.world > N.DOS_MAX_PEERS + 1:
            raise ValueError(f"fused reduce-scatter supports up to {N.DOS_MAX_PEERS + 1} ranks")
        bases = _ipc_bases(full_grads, group)
        shard_bytes = 2 * self.rank * layout.per_rank
        self.ptrs = tuple(bases[r] + shard_bytes for r in range(self.world))
        self.group = group

    def sources(self, scale: float = 1.0) -> GradSources:
        return GradSources(self.ptrs, self.rank, float(scale))


class PeerTargets:
    """The fused all-gather's destinations: every peer's full-model buffer,
    mapped into this process with CUDA IPC (one node, NVLink/NVSwitch P2P).

    ``targets`` lists, for each other rank, the address where *this* rank's
    shard begins inside that rank's full-model buffer; passed as
    ``execute_plan(..., peers=targets)``, K1 stores every updated working-copy
    element there in the same pass (and the copy engine forwards host
    subgroups after their H2D_PARAMS16), so no separate all-gather runs.
    Callers synchronise the ranks (a barrier) after the phase before
    reading the gathered buffer.
    """

    def __init__(self, full_params, layout: ShardLayout, group=None) -> None:
        import torch.distributed as dist

        from . import _native as N

        if full_params.element_size() != 2:
            raise TypeError("the full-model buffer must be half precision")
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if world - 1 > N.DOS_MAX_PEERS:
            raise ValueError(f"fused all-gather supports up to {N.DOS_MAX_PEERS + 1} ranks")
        self.bases = {r: b for r, b in _ipc_bases(full_params, group).items() if r != rank}
        shard_bytes = 2 * rank * layout.per_rank
        self.targets = [self.bases[r] + shard_bytes for r in sorted(self.bases)]
        self.group = group

    def barrier(self) -> None:
        import torch.distributed as dist

        dist.barrier(group=self.group)


def gather_params_overlapped(coll: BucketedCollectives, plan, working_copy, full_params, comm_stream=None):
    """``execute_plan(..., on_submitted=...)`` hook: all-gather each bucket as
    soon as this rank's subgroup j has its final working copy.

    ``working_copy`` is this rank's device working copy (``residency.model16``),
    ``full_params`` the padded full-model buffer.  Returns a callable taking the
    B200Target; after it runs, every bucket's all-gather is queued on NCCL
    behind the engine event of the action that finalised that subgroup, so the
    gathers overlap the rest of the phase.
    """
    import torch

    fin = finalising_actions(plan)
    lay = coll.layout
    rank = coll.rank

    def hook(target) -> list:
        stream = comm_stream or torch.cuda.Stream(device=working_copy.device)
        works = []
        with torch.cuda.stream(stream):
            for j in range(lay.num_buckets):
                start, size = lay.bucket_span(j)
                valid, pad = lay.rank_of_bucket_piece(rank, j)
                if valid:
                    target.stream_wait(fin[j], stream)
                if pad:
                    piece = torch.zeros(size, dtype=working_copy.dtype, device=working_copy.device)
                    if valid:
                        piece[:valid].copy_(working_copy[start:start + valid])
                else:
                    piece = working_copy[start:start + size]
                works.append(coll.all_gather_bucket(full_params, piece, j))
        hook.works = works
        hook.stream = stream
        return works

    return hook


def finalising_actions(plan) -> dict[int, int]:
    """Subgroup -> id of the device action after which its working copy is final.

    Fast subgroups: their GPU_UPDATE (K1 stores the working copy).  Host
    subgroups: their H2D_PARAMS16.  Every one is a device-lane action, so
    the engine holds a CUDA event for it.
    """
    from .plan import ActionKind, Device

    out: dict[int, int] = {}
    for a in plan.actions:
        if a.kind is ActionKind.GPU_UPDATE:
            out[a.subgroup] = a.id
        elif a.kind is ActionKind.H2D_PARAMS16 and plan.devices[a.subgroup] is Device.CPU:
            out[a.subgroup] = a.id
    return out


# ---------------------------------------------------------------- host cores per rank


def plan_core_binding(allowed, gpu_nodes, node_cpus, local_rank: int) -> list[int]:
    """The host cores rank ``local_rank`` should run H1 on, when every local
    rank's process starts with the same affinity mask (torchrun).

    ``gpu_nodes[r]``: NUMA node of local rank r's GPU (-1 unknown);
    ``node_cpus[node]``: that node's CPUs.  Ranks whose GPUs sit on the same
    node split that node's allowed CPUs into equal contiguous slices (the
    paper pins each rank's CPU optimizer work to its socket, §8(e)); without
    NUMA information the allowed CPUs are split evenly across all ranks.  A
    single rank keeps its GPU's node (all allowed CPUs when that is unknown)."""
    allowed = sorted(set(allowed))
    world = len(gpu_nodes)
    if world <= 1:
        node = gpu_nodes[0] if world else -1
        mine = [c for c in allowed if c in set(node_cpus.get(node, ()))] if node >= 0 else []
        return mine or allowed
    node = gpu_nodes[local_rank]
    pool = [c for c in allowed if c in set(node_cpus.get(node, ()))] if node >= 0 else []
    peers = [r for r in range(world) if gpu_nodes[r] == node] if pool else list(range(world))
    if not pool:
        pool = allowed
    k, i = len(peers), peers.index(local_rank)
    if len(pool) < k:  # fewer cores than ranks: share round-robin
        return [pool[i % len(pool)]]
    per = len(pool) // k
    return pool[i * per:(i + 1) * per]


def _parse_cpulist(text: str) -> list[int]:
    out: list[int] = []
    for part in text.strip().split(","):
        if not part:
            continue
        a, _, b = part.partition("-")
        out.extend(range(int(a), int(b or a) + 1))
    return out


def gpu_numa_node(device_index: int) -> int:
    """NUMA node of a GPU from sysfs (-1 when unknown)."""
    import torch

    try:
        p = torch.cuda.get_device_properties(device_index)
        bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as fh:
            return int(fh.read().strip())
    except Exception:
        return -1


def bind_host_cores(local_rank: int, local_world: int) -> list[int]:
    """Restrict this process (and libdos's H1 team) to its share of the host
    cores: the CPUs of its GPU's NUMA node, split among the local ranks on
    that node.  Returns the CPUs chosen."""
    import os

    import torch

    from . import _native as N

    nodes = ([gpu_numa_node(i) for i in range(local_world)] if torch.cuda.device_count() >= local_world
             else [-1] * local_world)
    node_cpus: dict[int, list[int]] = {}
    for nd in set(nodes):
        if nd >= 0:
            try:
                with open(f"/sys/devices/system/node/node{nd}/cpulist") as fh:
                    node_cpus[nd] = _parse_cpulist(fh.read())
            except OSError:
                pass
    cpus = plan_core_binding(os.sched_getaffinity(0), nodes, node_cpus, local_rank)
    os.sched_setaffinity(0, cpus)
    N.lib().dos_set_host_threads(len(cpus))  # rebuilds the team inside the new mask
    return cpus
