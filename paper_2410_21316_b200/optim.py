"""A torch-optimizer-style ``step()`` over the B200 update phase.

``DeepOptimizerStates(params, ...)`` flattens a model's half-precision CUDA
parameters into one shard and re-points every parameter (``.data``) and its
``.grad`` at views of the residency's flat HBM buffers, so

* backward accumulates straight into the flat grad buffer (no copy);
* the update phase's working-copy stores (K1 for fast subgroups,
  H2D_PARAMS16 for host subgroups) *are* the model's parameters: no
  all-params copy after the step.

fp32 master params (exact widening of the initial half-precision params,
or caller-provided), Adam m and v live in the pinned host pool.  Each
``step()``: flush the grads of host-scheduled subgroups D2H (the §8(f) row-1
gradient path), run ``execute_plan`` on the current plan, then re-fit the
machine profile from the measured timeline and re-choose the stride
(the per-iteration split of the north star).
"""

from __future__ import annotations

import numpy as np

from . import policy
from .executor import AdamHyper, execute_plan
from .plan import Device, build_plan
from .state import ShardedOptimizer


class DeepOptimizerStates:
    def __init__(self, params, lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8, weight_decay: float = 0.0,
                 *, subgroup_size: int = 100_000_000, profile=None, stride="auto", static_ratio: float = 0.0,
                 master_params=None, replan: bool = True) -> None:
        import torch

        self.params = [p for p in params if p.requires_grad]
        if not self.params:
            raise ValueError("no trainable parameters")
        dt = self.params[0].dtype
        if dt not in (torch.bfloat16, torch.float16) or any(p.dtype != dt or not p.is_cuda for p in self.params):
            raise TypeError("parameters must all be CUDA bfloat16 or all CUDA float16")
        self.lowp = "bf16" if dt == torch.bfloat16 else "fp16"
        self.hyper = AdamHyper(lr=lr, beta1=betas[0], beta2=betas[1], eps=eps, weight_decay=weight_decay)
        total = sum(p.numel() for p in self.params)
        sg = min(int(subgroup_size), total)
        opt = ShardedOptimizer.allocate(total, sg, lowp=self.lowp)
        dev = self.params[0].device
        off = 0
        with torch.no_grad():
            for p in self.params:
                n = p.numel()
                src = p.detach().reshape(-1)
                if master_params is None:
                    torch.from_numpy(opt._p[off:off + n]).copy_(src.float())  # exact widening
                opt._w[off:off + n] = src.view(torch.int16).cpu().numpy().view(opt._w.dtype)
                off += n
            if master_params is not None:
                flat = torch.cat([m.detach().reshape(-1).float().cpu() for m in master_params])
                if flat.numel() != total:
                    raise ValueError("master_params must match params element for element")
                opt._p[:] = flat.numpy()
        opt._m[:] = 0
        opt._v[:] = 0
        opt._g[:] = 0
        self.opt = opt
        self.res = opt.to_device(dev)
        # re-point params and grads at the flat HBM buffers
        off = 0
        for p in self.params:
            n = p.numel()
            p.data = self.res.model16[off:off + n].view(p.shape)
            p.grad = self.res.grads[off:off + n].view(p.shape)
            off += n
        if profile is None:
            from .catalog import get_profile

            profile = get_profile("b200-node")
        self.profile = profile
        self.static_ratio = static_ratio
        self.replan = replan and stride == "auto"
        sizes = [g.size for g in opt.subgroups]
        if stride == "auto":
            stride, _ = policy.choose_stride(profile, sizes, range(1, 7), static_ratio)
        self.plan = build_plan(len(sizes), stride, static_ratio=static_ratio)
        self.last = None

    @property
    def step_count(self) -> int:
        return self.opt.step

    def zero_grad(self, set_to_none: bool = False) -> None:
        if set_to_none:
            raise ValueError("grads are views of the flat HBM buffer; use zero_grad(set_to_none=False)")
        self.res.grads.zero_()

    def _flush_host_grads(self) -> None:
        """D2H of the grads the host lane will read (CPU subgroups only)."""
        import torch

        g = self.res.grads.view(torch.int16)
        host = torch.from_numpy(self.opt._g.view(np.int16))
        for i, sg in enumerate(self.opt.subgroups):
            if self.plan.devices[i] is Device.CPU:
                host[sg.start:sg.stop].copy_(g[sg.start:sg.stop], non_blocking=True)
        torch.cuda.current_stream(self.res.device).synchronize()

    def step(self):
        import torch

        torch.cuda.current_stream(self.res.device).synchronize()  # backward done
        self._flush_host_grads()
        self.last = execute_plan(self.opt, self.plan, self.profile, self.hyper)
        if self.replan and self.last.measured is not None:
            sizes = [g.size for g in self.opt.subgroups]
            self.profile = policy.refit_profile(self.profile, self.last.measured, sizes)
            stride, _ = policy.choose_stride(self.profile, sizes, range(1, 7), self.static_ratio)
            if stride != self.plan.stride:
                self.plan = build_plan(len(sizes), stride, static_ratio=self.static_ratio)
        return self.last

    def master_params(self) -> np.ndarray:
        """fp32 master params (host image, synchronised)."""
        return self.opt.params32

    def state_dict(self) -> dict:
        return {"step": self.opt.step, "params32": self.opt.params32.copy(), "momentum32": self.opt.momentum32.copy(),
                "variance32": self.opt.variance32.copy(), "hyper": self.hyper, "stride": self.plan.stride}

    def load_state_dict(self, sd: dict) -> None:
        self.res.sync_all_host()
        self.opt._p[:] = sd["params32"]
        self.opt._m[:] = sd["momentum32"]
        self.opt._v[:] = sd["variance32"]
        self.opt.step = int(sd["step"])
        from .state import lowp_downscale

        self.opt._w[:] = lowp_downscale(self.opt._p, self.lowp)
        self.res.push_host()
