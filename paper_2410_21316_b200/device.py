"""B200 residency of a shard and the ``B200Target`` plugin.

Memory layout of one rank on the B200 (HBM) and its host (pinned pool):

  host (pinned, registered)          HBM
  -------------------------          ---
  params32/momentum32/variance32     grads        lowp[P]   (resident: backward/RS writes it)
    fp32[P] — home tier of every     model16      lowp[P]   (authoritative working copy)
    dynamic and CPU subgroup         static p/m/v fp32, one allocation per static resident
  grads16   lowp[P] — host image     slots[num_slots] x {m, v, p} fp32[SG_max]
    used by CPU subgroups              (the in-flight windows; engine-owned)
  model16   lowp[P] — staging for
    CPU-downscaled params (H2D_PARAMS16 source) and the lazy host image

A sparse host pool (``ShardedOptimizer.allocate(host_homed=...)``) commits
host memory only for subgroups homed on the host; a static resident's home is
then its HBM allocation alone, and its host range is committed only if it
leaves the static set (or the caller reads the full host arrays).

``B200Target`` is the third implementation of the reference's UpdateTarget
protocol (pkg/src/optistate/scheduler.py:388-399), after SimTarget and
ExecutorTarget: durations/bytes come from the profile (so ``run_update``'s
virtual timeline is the prediction and equals ``simulate_update_phase``),
and ``apply`` hands each action to the native engine (dos_exec_submit),
which enqueues it on the B200's copy/compute streams or the host lane and
returns at once.  ``finish`` waits for the phase and returns the *measured*
timeline.
"""

from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _native as N
from .plan import KIND_CODE, LANE_CODE, ActionKind, Lane, ScheduledAction, UpdatePlan
from .state import SUBGROUP_STATE_BYTES_PER_PARAM, ShardedOptimizer, SystemProfile, bias_corrections
from .timing import SimTarget


def _torch():
    import torch

    return torch


class DeviceResidency:
    """What of one ShardedOptimizer lives in HBM, and host/device coherence."""

    def __init__(self, opt: ShardedOptimizer, device=None, grads=None, model16=None) -> None:
        """``grads``/``model16`` may be caller-owned CUDA views (e.g. this
        rank's chunk of a full-model buffer, so the phase writes the model's
        parameters in place); otherwise they are allocated here.  Their
        current contents are replaced by the host images (in a sparse pool:
        where the host range is committed)."""
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device visible: the B200 update phase needs a GPU (no CPU fallback)")
        N.lib()  # fail loudly now if the native library is missing
        self.opt = opt
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.tdtype = torch.float16 if opt.lowp == "fp16" else torch.bfloat16
        P = opt.total_params
        nsg = len(opt.subgroups)
        for name, t in (("grads", grads), ("model16", model16)):
            if t is not None and (t.dtype != self.tdtype or t.numel() != P or not t.is_contiguous()
                                  or t.device != self.device):
                raise ValueError(f"{name} must be a contiguous {self.tdtype} tensor of {P} elements on {self.device}")
        with torch.cuda.device(self.device):
            self.grads = grads if grads is not None else torch.empty(P, dtype=self.tdtype, device=self.device)
            self.model16 = model16 if model16 is not None else torch.empty(P, dtype=self.tdtype, device=self.device)
        self.sg_start = np.array([g.start for g in opt.subgroups], dtype=np.int64)
        self.sg_size = np.array([g.size for g in opt.subgroups], dtype=np.int64)
        self.static_set: frozenset[int] = frozenset()
        self.static_off = np.full(nsg, -1, dtype=np.int64)  # >= 0: HBM-resident (engine marker)
        self.static_sg: dict[int, tuple] = {}  # subgroup -> (p, m, v) fp32 HBM tensors
        self._static_ptrs = (C.c_void_p * max(1, 3 * nsg))()
        self.host_stale: set[str] = set()  # host images behind the device
        self._engines: dict[tuple, "Engine"] = {}
        self.push_host()

    # ---- coherence
    def _h2d(self, dst, src: np.ndarray) -> None:
        torch = _torch()
        dst.view(torch.int16 if dst.element_size() == 2 else torch.int32).copy_(
            torch.from_numpy(src.view(np.int16 if src.itemsize == 2 else np.int32)), non_blocking=False)

    def _d2h(self, dst: np.ndarray, src) -> None:
        torch = _torch()
        torch.from_numpy(dst.view(np.int16 if dst.itemsize == 2 else np.int32)).copy_(
            src.view(torch.int16 if src.element_size() == 2 else torch.int32), non_blocking=False)

    def _h2d_lowp(self, dst, src: np.ndarray) -> None:
        """Upload a half-precision host array.  In a sparse pool only the
        committed ranges have a host image; elsewhere the device copy is the
        only one and is left as it is (it is pulled to the host if the range
        is ever committed, ``on_host_commit``)."""
        for a, b in self.opt.host_runs("lowp"):
            self._h2d(dst[a:b], src[a:b])

    def _d2h_lowp(self, dst: np.ndarray, src) -> None:
        for a, b in self.opt.host_runs("lowp"):
            self._d2h(dst[a:b], src[a:b])

    def push_host(self) -> None:
        """Host arrays became authoritative (init, a host-side update): re-upload."""
        opt = self.opt
        self._h2d_lowp(self.grads, opt._g)
        self._h2d_lowp(self.model16, opt._w)
        for sg in self.static_set:
            self._upload_static(sg)
        self.host_stale.clear()

    def sync_host(self, name: str) -> None:
        if name not in self.host_stale:
            return
        self.host_stale.discard(name)
        opt = self.opt
        if name == "_w":
            self._d2h_lowp(opt._w, self.model16)
            return
        if name == "_g":
            self._d2h_lowp(opt._g, self.grads)
            return
        k = ("_p", "_m", "_v").index(name)
        dst = getattr(opt, name)
        opt.ensure_host(self.static_set, "state")
        for sg in self.static_set:
            a, n = int(self.sg_start[sg]), int(self.sg_size[sg])
            self._d2h(dst[a:a + n], self.static_sg[sg][k])

    def on_host_commit(self, subgroups, group: str) -> None:
        """A sparse pool just committed these subgroups' host ranges (they
        read as zeros): copy in what the device holds for them — the grads
        and working copy ("lowp"), or a static resident's fp32 state."""
        opt = self.opt
        for sg in subgroups:
            a, n = int(self.sg_start[sg]), int(self.sg_size[sg])
            if group == "lowp":
                self._d2h(opt._g[a:a + n], self.grads[a:a + n])
                self._d2h(opt._w[a:a + n], self.model16[a:a + n])
            elif sg in self.static_sg:
                for k, name in enumerate(("_p", "_m", "_v")):
                    self._d2h(getattr(opt, name)[a:a + n], self.static_sg[sg][k])

    def sync_all_host(self) -> None:
        """Make every host image current (a host-side pass over the whole
        shard follows).  In a sparse pool every range is committed first:
        an uncommitted static resident's range is filled from its HBM home."""
        n = len(self.opt.subgroups)
        self.opt.ensure_host(range(n), "state")
        self.opt.ensure_host(range(n), "lowp")
        for name in ("_w", "_g", "_p", "_m", "_v"):
            self.sync_host(name)

    def host_modified(self) -> None:
        """Call after writing host arrays directly (e.g. a host-only update)."""
        self.sync_all_host()
        self.push_host()

    def load_grads(self, grads) -> None:
        """New step gradients: a CUDA tensor (flushed to the host image for
        CPU subgroups) or a host array of the lowp kind (uploaded)."""
        torch = _torch()
        opt = self.opt
        if isinstance(grads, torch.Tensor):
            if grads.numel() != opt.total_params:
                raise ValueError("grads must hold total_params elements")
            src = grads.reshape(-1).to(device=self.device, dtype=self.tdtype)
            self.grads.copy_(src)
            self._d2h_lowp(opt._g, self.grads)
            return
        arr = np.asarray(grads)
        if arr.dtype != opt._g.dtype or arr.shape != opt._g.shape:
            raise TypeError(f"grads must be {opt._g.dtype}{opt._g.shape}")
        opt.grads16[:] = arr  # (a full host write: commits every range of a sparse pool)
        self._h2d(self.grads, opt._g)

    def _upload_static(self, sg: int) -> None:
        """Host image -> the subgroup's HBM home (zeros where a sparse pool
        never committed the range: that is what the host image holds)."""
        a, n = int(self.sg_start[sg]), int(self.sg_size[sg])
        for k, name in enumerate(("_p", "_m", "_v")):
            dst = self.static_sg[sg][k]
            if self.opt.host_committed(sg, "state"):
                self._h2d(dst, getattr(self.opt, name)[a:a + n])
            else:
                dst.zero_()

    # ---- whole-shard export / import without materialising a sparse pool
    def export_state(self, name: str) -> np.ndarray:
        """A fresh (pageable) copy of ``params32``/``momentum32``/``variance32``
        ("_p"/"_m"/"_v") assembled from each subgroup's home tier — the host
        pool for host-homed subgroups, HBM for static residents — without
        committing any host range (a checkpoint of a shard larger than the
        host pool stays possible)."""
        k = ("_p", "_m", "_v").index(name)
        opt = self.opt
        src = getattr(opt, name)
        out = np.empty(opt.total_params, dtype=np.float32)
        for sg in opt.subgroups:
            if sg.index in self.static_set:
                out[sg.slice] = self.static_sg[sg.index][k].cpu().numpy()
            else:
                out[sg.slice] = src[sg.slice]
        return out

    def import_state(self, name: str, values: np.ndarray) -> None:
        """Inverse of ``export_state``: each subgroup's slice goes to its home."""
        torch = _torch()
        k = ("_p", "_m", "_v").index(name)
        opt = self.opt
        values = np.ascontiguousarray(values, dtype=np.float32).reshape(-1)
        if values.size != opt.total_params:
            raise ValueError(f"{name} must hold {opt.total_params} elements")
        opt.ensure_host([g.index for g in opt.subgroups if g.index not in self.static_set], "state")
        dst = getattr(opt, name)
        for sg in opt.subgroups:
            if sg.index in self.static_set:
                self.static_sg[sg.index][k].copy_(torch.from_numpy(values[sg.slice]))
            else:
                dst[sg.slice] = values[sg.slice]
        if self.static_set:  # residents' host images (where committed) are now behind HBM
            self.host_stale.add(name)

    def static_views(self, sg: int) -> tuple:
        """(p, m, v) fp32 HBM tensors of static subgroup ``sg`` (its home
        while resident: write them to initialise a device-homed subgroup)."""
        if sg not in self.static_sg:
            raise ValueError(f"subgroup {sg} is not HBM-resident")
        return self.static_sg[sg]

    def set_static(self, static_set: frozenset[int]) -> None:
        """Make exactly ``static_set`` HBM-resident (TwinFlow-style statics).

        Each resident owns its own HBM allocation, so the set changes one
        subgroup at a time: leaving subgroups are written back to (and, in a
        sparse pool, committed on) the host and freed before joining ones are
        allocated and uploaded; staying ones do not move."""
        static_set = frozenset(static_set)
        if static_set == self.static_set:
            return
        torch = _torch()
        opt = self.opt
        leaving = sorted(self.static_set - static_set)
        joining = sorted(static_set - self.static_set)
        if leaving:
            # ranges committed just now are filled from HBM by on_host_commit;
            # the others get their (possibly newer) HBM state written home here
            had_home = [sg for sg in leaving if opt.host_committed(sg, "state")]
            opt.ensure_host(leaving, "state")
            for sg in had_home:
                a, n = int(self.sg_start[sg]), int(self.sg_size[sg])
                for k, name in enumerate(("_p", "_m", "_v")):
                    self._d2h(getattr(opt, name)[a:a + n], self.static_sg[sg][k])
            for sg in leaving:
                del self.static_sg[sg]
                self.static_off[sg] = -1
                for k in range(3):
                    self._static_ptrs[3 * sg + k] = None
        with torch.cuda.device(self.device):
            for sg in joining:
                n = int(self.sg_size[sg])
                self.static_sg[sg] = tuple(torch.empty(n, dtype=torch.float32, device=self.device) for _ in range(3))
                self._upload_static(sg)
                self.static_off[sg] = 0
                for k in range(3):
                    self._static_ptrs[3 * sg + k] = self.static_sg[sg][k].data_ptr()
        self.static_set = static_set

    def after_phase(self, host_io: bool = False, flush_grads: bool = False) -> None:
        if not host_io:  # with host_io the engine mirrored the working copy to the host
            self.host_stale.add("_w")
        if flush_grads:  # the device grads are the step's (reduced) grads; the host image may
            self.host_stale.add("_g")  # not hold them (the grad ring bypasses it)
        if self.static_set:
            self.host_stale.update(("_p", "_m", "_v"))

    # ---- engine cache
    def engine(self, num_slots: int, slot_elems: int, host_threads: int = 0, fuse: bool = True) -> "Engine":
        key = (num_slots, slot_elems, host_threads, fuse)
        eng = self._engines.get(key)
        if eng is None:
            # one engine per residency: drop others (frees their HBM slots)
            for e in self._engines.values():
                e.close()
            self._engines.clear()
            eng = Engine(self.device.index, num_slots, slot_elems, host_threads, fuse)
            self._engines[key] = eng
        return eng

    def state_desc(self, host_io: bool = False, peers=None, flush_grads: bool = False,
                   grad_sources=None, host_io_ahead: int = 0,
                   host_updates: int = -1) -> tuple[N.dos_state_desc, list]:
        """``peers``: addresses (ints) where this shard starts in each peer's
        full-model buffer — the fused all-gather targets (include/dos.h).
        ``grad_sources``: a ``distributed.GradSources`` (fused reduce-scatter)."""
        opt = self.opt
        peers = list(peers or ())
        if len(peers) > N.DOS_MAX_PEERS:
            raise ValueError(f"at most {N.DOS_MAX_PEERS} peers")
        peer_arr = (C.c_void_p * max(1, len(peers)))(*peers)
        srcs = list(grad_sources.ptrs) if grad_sources is not None else []
        if len(srcs) > N.DOS_MAX_PEERS + 1:
            raise ValueError(f"at most {N.DOS_MAX_PEERS + 1} grad sources")
        src_arr = (C.c_void_p * max(1, len(srcs)))(*srcs)
        keep = [self.sg_start, self.sg_size, self.static_off, peer_arr, src_arr, self._static_ptrs]
        p64 = C.POINTER(C.c_int64)
        d = N.dos_state_desc(
            num_subgroups=len(opt.subgroups),
            sg_start=self.sg_start.ctypes.data_as(p64),
            sg_size=self.sg_size.ctypes.data_as(p64),
            static_offset=self.static_off.ctypes.data_as(p64),
            lowp_dtype=opt.lowp_code,
            host_p=N.ptr(opt._p), host_m=N.ptr(opt._m), host_v=N.ptr(opt._v),
            host_g=N.ptr(opt._g), host_lowp=N.ptr(opt._w),
            dev_g=self.grads.data_ptr(), dev_lowp=self.model16.data_ptr(),
            dev_static_p=None, dev_static_m=None, dev_static_v=None,
            dev_static_sg=C.cast(self._static_ptrs, C.POINTER(C.c_void_p)),
            host_io_ahead=host_io_ahead,
            host_updates=host_updates,
            host_io=1 if host_io else 0,
            npeers=len(peers),
            peer_lowp=C.cast(peer_arr, C.POINTER(C.c_void_p)),
            flush_grads=1 if flush_grads else 0,
            nsrc_g=len(srcs),
            self_rank=grad_sources.self_rank if grad_sources is not None else 0,
            src_g=C.cast(src_arr, C.POINTER(C.c_void_p)),
            grad_scale=grad_sources.scale if grad_sources is not None else 1.0,
        )
        return d, keep


class Engine:
    """Owner of one native engine (streams, HBM slots, host-lane worker)."""

    def __init__(self, device: int, num_slots: int, slot_elems: int, host_threads: int = 0, fuse: bool = True):
        cfg = N.dos_exec_config(device=device, num_slots=num_slots, slot_elems=slot_elems,
                                host_threads=host_threads, fuse_downscale=1 if fuse else 0)
        h = C.c_void_p()
        N.check(N.lib().dos_exec_create(C.byref(cfg), C.byref(h)))
        self.handle = h
        self.num_slots = num_slots
        self.slot_elems = slot_elems

    def close(self) -> None:
        if self.handle:
            N.lib().dos_exec_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _PlanDescs:
    """The plan's actions as C structs, built once per plan object."""

    def __init__(self, plan: UpdatePlan) -> None:
        n = len(plan.actions)
        self.descs = (N.dos_action_desc * n)()
        self._keep = []
        p32 = C.POINTER(C.c_int32)
        for a in plan.actions:
            d = self.descs[a.id]
            d.id = a.id
            d.kind = KIND_CODE[ActionKind(a.kind.value)]  # by value: reference plans work too
            d.subgroup = a.subgroup
            d.lane = LANE_CODE[Lane(a.lane.value)]
            d.is_static = 1 if (a.subgroup >= 0 and a.subgroup in plan.static_set) else 0
            deps = np.array(a.deps, dtype=np.int32)
            batch = np.array(a.batch, dtype=np.int32)
            self._keep += [deps, batch]
            d.num_deps = len(a.deps)
            d.deps = deps.ctypes.data_as(p32)
            d.batch_len = len(a.batch)
            d.batch = batch.ctypes.data_as(p32)


_DESC_CACHE: dict[int, tuple[UpdatePlan, _PlanDescs]] = {}


def plan_descs(plan: UpdatePlan) -> _PlanDescs:
    hit = _DESC_CACHE.get(id(plan))
    if hit is not None and hit[0] is plan:
        return hit[1]
    if len(_DESC_CACHE) > 16:
        _DESC_CACHE.clear()
    pd = _PlanDescs(plan)
    _DESC_CACHE[id(plan)] = (plan, pd)
    return pd


def slots_for(profile: SystemProfile, plan: UpdatePlan, sizes: Sequence[int]) -> tuple[int, int]:
    """(physical windows, elements per window piece) for this plan."""
    dyn = [sizes[i] for i in plan.dynamic_fast]
    if not dyn:
        return 1, 0
    biggest = max(dyn)
    cap = profile.fast_capacity_bytes
    windows = 2 if cap is None else min(2, cap // (SUBGROUP_STATE_BYTES_PER_PARAM * biggest))
    if windows < 1:
        raise N.InfeasibleConfigError(
            f"fast tier capacity {cap} B cannot hold one in-flight subgroup window of "
            f"{SUBGROUP_STATE_BYTES_PER_PARAM * biggest} B")
    return windows, biggest


class B200Target(SimTarget):
    """UpdateTarget that executes the plan on a B200 and its host.

    Predicted durations/bytes are SimTarget's (from ``profile``); ``apply``
    submits the action to the native engine without waiting.  Call
    ``finish()`` after ``run_update`` to wait and get measured events.
    """

    def __init__(self, profile: SystemProfile, plan: UpdatePlan, optimizer: ShardedOptimizer, hyper,
                 step: int, *, host_threads: int = 0, fuse_downscale: bool = True,
                 host_io: bool = False, peers=None, flush_grads: bool = False, grad_sources=None) -> None:
        if host_io and flush_grads:
            raise ValueError("host_io reads the grads from the host image; flush_grads copies them there")
        if grad_sources is not None and not flush_grads:
            raise ValueError("the fused reduce-scatter (grad_sources) runs with flush_grads=True")
        sizes = tuple(g.size for g in optimizer.subgroups)
        super().__init__(profile, plan, sizes)
        self.opt = optimizer
        self.hyper = hyper
        self.step = step
        self.residency = optimizer.to_device()
        self.residency.set_static(plan.static_set)
        # a sparse pool commits what this plan reads or writes on the host
        # (no-ops for a dense pool or ranges already committed)
        nsg = len(sizes)
        optimizer.ensure_host([i for i in range(nsg) if i not in plan.static_set], "state")
        optimizer.ensure_host(range(nsg) if host_io else
                              [i for i in range(nsg) if plan.devices[i].value == "cpu"], "lowp")
        self.num_slots, slot_elems = slots_for(profile, plan, sizes)
        self.engine = self.residency.engine(self.num_slots, slot_elems, host_threads, fuse_downscale)
        self._descs = plan_descs(plan)
        self.host_io = host_io
        self.peers = list(peers or ())
        self.flush_grads = flush_grads
        self.grad_sources = grad_sources
        self._begun = False
        self._submitted = 0

    def _begin(self) -> None:
        # with host buffers, residents that lead the fast lane get their grads
        # just ahead of it; residents that trail it get them all at phase start
        first_fast = next((a.subgroup for a in self.plan.actions if a.kind.value == "gpu_update"), None)
        ahead = 2 if (self.host_io and first_fast is not None and first_fast in self.plan.static_set) else 0
        host_updates = sum(1 for a in self.plan.actions if a.kind.value == "cpu_update")
        desc, keep = self.residency.state_desc(self.host_io, self.peers, self.flush_grads, self.grad_sources, ahead,
                                               host_updates)
        self._keep = (desc, keep)
        h = self.hyper
        bc1, bc2 = bias_corrections(h.beta1, h.beta2, self.step)
        sc = N.scalars(h.lr, h.beta1, h.beta2, h.eps, bc1, bc2, getattr(h, "weight_decay", 0.0))
        self._sc = sc
        N.check(N.lib().dos_exec_begin(self.engine.handle, C.byref(desc), C.byref(sc), len(self.plan.actions)))
        self._begun = True

    def apply(self, action, start_ns: int, end_ns: int) -> None:
        if not self._begun:
            self._begin()
        rc = N.lib().dos_exec_submit(self.engine.handle, C.byref(self._descs.descs[action.id]))
        self._submitted += 1
        if rc != N.DOS_OK:
            msg = N.lib().dos_last_error().decode(errors="replace")
            self.finish(raise_errors=False)  # drain what was enqueued before failing
            exc = {N.DOS_ESTATE: AssertionError, N.DOS_EINFEASIBLE: N.InfeasibleConfigError,
                   N.DOS_EINVAL: ValueError, N.DOS_ETYPE: TypeError}.get(rc, RuntimeError)
            raise exc(f"submit of action {action.id}: {msg}")

    def stream_wait(self, action_id: int, stream) -> None:
        """Make a torch/CUDA ``stream`` wait for submitted device action ``action_id``."""
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        N.check(N.lib().dos_exec_stream_wait(self.engine.handle, int(action_id), handle))

    def finish(self, raise_errors: bool = True) -> tuple[ScheduledAction, ...]:
        """Wait for the phase; measured events in emission order."""
        if not self._begun:
            return ()
        n = self._submitted
        s = np.zeros(max(n, 1), dtype=np.int64)
        e = np.zeros(max(n, 1), dtype=np.int64)
        p64 = C.POINTER(C.c_int64)
        rc = N.lib().dos_exec_finish(self.engine.handle, s.ctypes.data_as(p64), e.ctypes.data_as(p64), n)
        self._begun = False
        if rc != N.DOS_OK:
            if raise_errors:
                N.check(rc)
            return ()
        acts = self.plan.actions
        return tuple(ScheduledAction(action=acts[i], start_ns=int(s[i]), end_ns=int(e[i]),
                                     bytes=self.bytes_of(acts[i])) for i in range(n))


def load_shard(params32, momentum32, variance32, grads16, model16, subgroup_size: int, *, lowp: str = "bf16",
               static_set=frozenset(), device=None) -> ShardedOptimizer:
    """A B200-attached shard built from whole-shard arrays, each subgroup
    written straight to its home: the static residents' fp32 state into their
    HBM allocations (no host memory for it: sparse pinned pool), everyone
    else's into the pinned pool; grads and working copy to HBM (and to the
    host images of host-homed subgroups).

    ``params32``/``momentum32``/``variance32``: float32 arrays (numpy or CPU
    torch); ``grads16``/``model16``: the half-precision kind's bits (numpy
    float16 for fp16, uint16 bf16 bits for bf16)."""
    torch = _torch()
    p, m, v = (np.ascontiguousarray(np.asarray(x, dtype=np.float32)).reshape(-1)
               for x in (params32, momentum32, variance32))
    want16 = np.dtype(np.float16) if lowp == "fp16" else np.dtype(np.uint16)
    g, w = (np.ascontiguousarray(np.asarray(x)).reshape(-1) for x in (grads16, model16))
    total = p.size
    for name, a, dt in (("momentum32", m, np.float32), ("variance32", v, np.float32), ("grads16", g, want16),
                        ("model16", w, want16)):
        if a.size != total:
            raise ValueError(f"{name} must hold {total} elements")
        if a.dtype != dt:
            raise TypeError(f"{name} must be {np.dtype(dt)}, got {a.dtype}")
    static_set = frozenset(int(i) for i in static_set)
    nsg = -(-total // int(subgroup_size))
    if any(i < 0 or i >= nsg for i in static_set):
        raise ValueError(f"static subgroups must be in [0, {nsg})")
    opt = ShardedOptimizer.allocate(total, subgroup_size, lowp=lowp, host_homed=[i for i in range(nsg)
                                                                                  if i not in static_set])
    for a, b in opt.host_runs("state"):
        opt._p[a:b], opt._m[a:b], opt._v[a:b] = p[a:b], m[a:b], v[a:b]
    for a, b in opt.host_runs("lowp"):
        opt._g[a:b], opt._w[a:b] = g[a:b], w[a:b]
    res = opt.to_device(device)
    res.set_static(static_set)
    i16 = lambda x: torch.from_numpy(x.view(np.int16))
    for i in sorted(static_set):
        sl = opt.subgroups[i].slice
        for t, src in zip(res.static_views(i), (p, m, v)):
            t.copy_(torch.from_numpy(src[sl]))
        res.grads.view(torch.int16)[sl].copy_(i16(g[sl]))
        res.model16.view(torch.int16)[sl].copy_(i16(w[sl]))
    return opt
