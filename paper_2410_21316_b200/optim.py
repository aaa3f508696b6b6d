"""A torch-optimizer-style ``step()`` over the B200 update phase.

``DeepOptimizerStates(params, ...)`` flattens a model's half-precision CUDA
parameters into one padded full-model buffer and re-points every parameter
(``.data``) and its ``.grad`` at views of it, so

* backward accumulates straight into the flat grad buffer (no copy);
* this rank's chunk of the flat param buffer *is* the residency's working
  copy: the phase's K1 / H2D_PARAMS16 stores update the model in place.

One process per GPU.  With ``process_group`` of N ranks the state is
ZeRO-3 sharded (``shard(P, N, SG)``, core.py:139-170): each rank keeps the
fp32 master params, Adam m and v of its own chunk in its pinned host pool,
and ``step()`` runs

1. the reduce-scatter of the bf16 grads into this rank's chunk (summed;
   ``average_grads`` divides by N) — by default fused into the phase: K1
   reads every rank's grads of the shard over NVLink (CUDA IPC,
   ``distributed.PeerGrads``) and sums them in rank order while it streams
   the fp32 state, and each host subgroup's grads are reduced on the device
   right before their D2H flush; with ``fused_reduce=False`` a bucketed NCCL
   reduce-scatter runs before the phase,
2. inside the phase, the D2H flush of the grads the host lane will read
   (§8(f) row 1; ``execute_plan(flush_grads=True)``),
3. the update phase (``execute_plan``) with the all-gather fused in: K1
   stores every updated working-copy element into each peer's full-model
   buffer over NVLink (CUDA IPC, ``distributed.PeerTargets``) and the copy
   engine forwards host subgroups after their H2D_PARAMS16, then one
   barrier; with ``fused_gather=False`` each bucket's NCCL all-gather is
   instead chained onto the engine event that finalises its subgroup
   (``distributed.gather_params_overlapped``),
4. a per-iteration re-fit: explore-then-exploit over strides by measured
   span (``policy.StrideTuner``), identical on every rank.
"""

from __future__ import annotations

import numpy as np

from . import policy
from .distributed import BucketedCollectives, PeerGrads, PeerTargets, ShardLayout, gather_params_overlapped
from .executor import AdamHyper, execute_plan
from .plan import Device, build_plan
from .state import ShardedOptimizer, lowp_downscale


class DeepOptimizerStates:
    def __init__(self, params, lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8, weight_decay: float = 0.0,
                 *, subgroup_size: int = 100_000_000, profile=None, stride="auto", static_ratio=0.0,
                 master_params=None, process_group=None, average_grads: bool = False, explore: int = 3,
                 fused_gather: bool = True, fused_reduce: bool = True, hbm_budget_bytes: int | None = None) -> None:
        """``static_ratio``: the TwinFlow fraction of subgroups whose fp32
        state is homed in HBM, or "auto" for as many as fit in
        ``hbm_budget_bytes`` (default: the HBM free now minus a 4 GB headroom —
        pass an explicit budget to leave room for activations)."""
        import torch
        import torch.distributed as dist

        self.params = [p for p in params if p.requires_grad]
        if not self.params:
            raise ValueError("no trainable parameters")
        dt = self.params[0].dtype
        if dt not in (torch.bfloat16, torch.float16) or any(p.dtype != dt or not p.is_cuda for p in self.params):
            raise TypeError("parameters must all be CUDA bfloat16 or all CUDA float16")
        self.lowp = "bf16" if dt == torch.bfloat16 else "fp16"
        self.hyper = AdamHyper(lr=lr, beta1=betas[0], beta2=betas[1], eps=eps, weight_decay=weight_decay)
        self.group = process_group
        self.world = dist.get_world_size(process_group) if process_group is not None else 1
        self.rank = dist.get_rank(process_group) if process_group is not None else 0
        self.average_grads = average_grads
        dev = self.params[0].device
        total = sum(p.numel() for p in self.params)
        sg = min(int(subgroup_size), -(-total // self.world))
        self.layout = lay = ShardLayout.build(total, self.world, sg)
        self.offset = self.rank * lay.per_rank
        mine = sum(g.size for g in lay.ranks[self.rank])

        # full-model flat buffers (padded), params and grads re-pointed into them
        self.flat = torch.zeros(lay.padded_total, dtype=dt, device=dev)
        self.flat_grad = torch.zeros(lay.padded_total, dtype=dt, device=dev)
        off = 0
        with torch.no_grad():
            for p in self.params:
                n = p.numel()
                self.flat[off:off + n].copy_(p.detach().reshape(-1))
                p.data = self.flat[off:off + n].view(p.shape)
                p.grad = self.flat_grad[off:off + n].view(p.shape)
                off += n

        sizes = [g.size for g in lay.ranks[self.rank]]
        # "auto" may resolve to every subgroup resident on purpose: plan without the all-static warning
        self._plan = policy._quiet_plan if static_ratio == "auto" else (
            lambda n, k, r: build_plan(n, k, static_ratio=r))
        if static_ratio == "auto":
            # capacity-aware: as many subgroups homed in HBM as fit beside two
            # windows (the grads and working copy already live in the flat buffers)
            budget = torch.cuda.mem_get_info(dev)[0] if hbm_budget_bytes is None else int(hbm_budget_bytes) + (4 << 30)
            r = policy.capacity_static_ratio(sizes, budget, lowp_bytes_per_param=0)
            static_ratio = -self._max_over_ranks(-r) if self.world > 1 else r  # same plan shape everywhere
        static = self._plan(len(sizes), 1, static_ratio).static_set
        # sparse pinned pool: host memory only for the host-homed subgroups
        opt = ShardedOptimizer.allocate(mine, sg, lowp=self.lowp,
                                        host_homed=[i for i in range(len(sizes)) if i not in static])
        chunk = self.flat[self.offset:self.offset + mine]
        m32 = None
        if master_params is not None:
            flat_m = torch.cat([m.detach().reshape(-1).float().cpu() for m in master_params])
            if flat_m.numel() != total:
                raise ValueError("master_params must match params element for element")
            m32 = flat_m[self.offset:self.offset + mine].contiguous()
            del flat_m
            with torch.no_grad():  # working copy = RNE of the masters
                chunk.copy_(torch.from_numpy(lowp_downscale(m32.numpy(), self.lowp).view(np.int16)).view(dt))

        def masters(a: int, b: int):
            """fp32 masters of [a, b) of this rank's chunk, widened one range at
            a time (never the whole shard at once: it is not in the HBM budget)."""
            return chunk[a:b].float() if m32 is None else m32[a:b]

        w16 = chunk.view(torch.int16)
        for a, b in opt.host_runs("state"):
            for lo in range(a, b, sg):
                hi = min(b, lo + sg)
                torch.from_numpy(opt._p[lo:hi]).copy_(masters(lo, hi))
            opt._m[a:b] = 0
            opt._v[a:b] = 0
        for a, b in opt.host_runs("lowp"):
            torch.from_numpy(opt._w[a:b].view(np.int16)).copy_(w16[a:b])
            opt._g[a:b] = 0
        self.opt = opt
        self.res = opt.to_device(dev, grads=self.flat_grad[self.offset:self.offset + mine], model16=chunk)
        self.res.set_static(static)  # residents start zeroed (m, v) ...
        for i in sorted(static):
            g = opt.subgroups[i]
            self.res.static_views(i)[0].copy_(masters(g.start, g.stop))  # ... with their masters in HBM
        del m32
        self.coll = BucketedCollectives(lay, process_group) if self.world > 1 else None
        if master_params is not None and self.coll is not None:
            self._publish_chunk()  # every rank's copy of the model now holds every rank's new chunk
        # fused all-gather: K1 writes the working copy straight into every
        # peer's full-model buffer (IPC-mapped); else bucketed overlapped gathers
        self.peers = PeerTargets(self.flat, lay, process_group) if (self.world > 1 and fused_gather) else None
        # fused reduce-scatter: every rank's grad buffer IPC-mapped, reduced inside the phase
        self.peer_grads = PeerGrads(self.flat_grad, lay, process_group) if (self.world > 1 and fused_reduce) else None

        if profile is None:
            from .catalog import get_profile

            profile = get_profile("b200-node")
        self.profile = profile
        self.static_ratio = static_ratio
        self.sizes = sizes
        self.tuner = None
        if stride == "auto":
            # measured host rates (profile_b200.measure_profile earlier in this process) let the
            # fluid host-DRAM model order the exploration
            from . import profile_b200

            self.tuner = policy.StrideTuner(profile, self.sizes, range(1, 7), static_ratio, explore=explore,
                                            rates=profile_b200.host_rates())
            if self.world > 1:  # the same exploration order on every rank
                box = [self.tuner.queue]
                dist.broadcast_object_list(box, src=0, group=process_group)
                self.tuner.queue = list(box[0])
            stride = self.tuner.next_stride()
        self.plan = self._plan(len(self.sizes), stride, static_ratio)
        self.last = None

    @property
    def step_count(self) -> int:
        return self.opt.step

    def zero_grad(self, set_to_none: bool = False) -> None:
        if set_to_none:
            raise ValueError("grads are views of the flat HBM buffer; use zero_grad(set_to_none=False)")
        self.flat_grad.zero_()

    def _publish_chunk(self) -> None:
        """All-gather this rank's chunk of the working copy into every rank's
        full-model buffer (after it was rewritten outside a phase: init from
        masters, load_state_dict), then synchronise."""
        import torch

        lay = self.layout
        self.coll.all_gather_all(self.flat, self.flat[self.offset:self.offset + lay.per_rank])
        torch.cuda.current_stream(self.res.device).synchronize()
        self._barrier()

    def _check_grads_alias_flat(self) -> None:
        """Grads only reach the optimizer through the flat buffer: a ``.grad``
        replaced by something else (``zero_grad(set_to_none=True)`` on the
        model, a user assignment) would be silently ignored — refuse it."""
        lo = self.flat_grad.data_ptr()
        hi = lo + self.flat_grad.numel() * self.flat_grad.element_size()
        for i, p in enumerate(self.params):
            g = p.grad
            if g is None or not (lo <= g.data_ptr() < hi):
                raise RuntimeError(
                    f"parameter {i}: .grad no longer aliases the optimizer's flat grad buffer "
                    f"({'None' if g is None else 'a different tensor'}); clear grads with "
                    f"DeepOptimizerStates.zero_grad() or model.zero_grad(set_to_none=False)")

    def _reduce_grads(self) -> None:
        lay = self.layout
        own = self.flat_grad[self.offset:self.offset + lay.per_rank]
        self.coll.reduce_scatter_all(self.flat_grad, own, scale=1.0 / self.world if self.average_grads else None)

    def _flush_host_grads(self) -> None:
        """D2H of the grads the host lane will read (CPU subgroups only)."""
        import torch

        g = self.res.grads.view(torch.int16)
        host = torch.from_numpy(self.opt._g.view(np.int16))
        for i, sg in enumerate(self.opt.subgroups):
            if self.plan.devices[i] is Device.CPU:
                host[sg.start:sg.stop].copy_(g[sg.start:sg.stop], non_blocking=True)
        torch.cuda.current_stream(self.res.device).synchronize()

    def _barrier(self) -> None:
        import torch.distributed as dist

        dist.barrier(group=self.group)

    def _max_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64)
        if dist.get_backend(self.group) == "nccl":
            t = t.to(self.params[0].device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def step(self):
        import torch

        self._check_grads_alias_flat()
        torch.cuda.current_stream(self.res.device).synchronize()  # backward done
        gsrc = None
        if self.peer_grads is not None:
            self._barrier()  # every rank's grads are complete before any rank reads them
            gsrc = self.peer_grads.sources(1.0 / self.world if self.average_grads else 1.0)
        elif self.coll is not None:
            self._reduce_grads()
            torch.cuda.current_stream(self.res.device).synchronize()
        hook = None
        if self.coll is not None and self.peers is None:
            hook = gather_params_overlapped(self.coll, self.plan, self.res.model16, self.flat)
        # the host lane's grads are flushed D2H inside the phase (flush_grads)
        self.last = execute_plan(self.opt, self.plan, self.profile, self.hyper, on_submitted=hook,
                                 peers=self.peers.targets if self.peers is not None else None, flush_grads=True,
                                 grad_sources=gsrc)
        if hook is not None:
            for w in hook.works:
                if w is not None:
                    w.wait()
            torch.cuda.current_stream(self.res.device).wait_stream(hook.stream)
        if self.peers is not None or self.peer_grads is not None:
            # every rank's peer stores have landed and no rank still reads a
            # peer's grads (each finished its phase) before anyone moves on
            self._barrier()
        if self.tuner is not None and self.last.measured is not None:
            self.tuner.record(self.plan.stride, int(self._max_over_ranks(self.last.measured.span_ns)))
            nxt = self.tuner.next_stride()
            if nxt != self.plan.stride:
                self.plan = self._plan(len(self.sizes), nxt, self.static_ratio)
        return self.last

    def master_params(self) -> np.ndarray:
        """This rank's fp32 master params (a copy assembled from each
        subgroup's home tier; a sparse pool is not materialised)."""
        return self.res.export_state("_p")

    def state_dict(self) -> dict:
        """This rank's fp32 state, each subgroup read from its home tier (a
        sparse pool is not materialised on the host)."""
        res = self.res
        return {"step": self.opt.step, "rank": self.rank, "world": self.world, "offset": self.offset,
                "params32": res.export_state("_p"), "momentum32": res.export_state("_m"),
                "variance32": res.export_state("_v"), "hyper": self.hyper}

    def load_state_dict(self, sd: dict) -> None:
        import torch

        if (sd.get("rank", 0), sd.get("world", 1)) != (self.rank, self.world):
            raise ValueError("state dict belongs to another rank / world size")
        res, opt = self.res, self.opt
        for name, key in (("_p", "params32"), ("_m", "momentum32"), ("_v", "variance32")):
            res.import_state(name, sd[key])
        opt.step = int(sd["step"])
        # the working copy (this rank's chunk of the model) = RNE of the masters
        w = lowp_downscale(np.ascontiguousarray(sd["params32"], dtype=np.float32), self.lowp)
        with torch.no_grad():
            res.model16.view(torch.int16).copy_(torch.from_numpy(w.view(np.int16)))
        for a, b in opt.host_runs("lowp"):
            opt._w[a:b] = w[a:b]
        res.host_stale.discard("_w")
        if self.coll is not None:
            self._publish_chunk()  # peers' copies of this chunk were stale until the next step's gather
