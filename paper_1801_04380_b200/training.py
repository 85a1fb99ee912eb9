"""Real training on a B200: execute the planner's schedule with the CUDA executor.

``Executor`` owns one ``sn_exec`` (libsnexec.so): the device arena sized to the
planner's pool capacity, the parameter/gradient blocks, the copy streams and
the captured CUDA graph of one iteration.  ``run_training`` is the new public
entry point next to the reference's ``run_simulation``: it plans with the same
``SimConfig`` and then runs real iterations, returning the ``SimReport`` plus
measured throughput.

Layer semantics the reference leaves open are fixed here and
in ``oracle/numerics.py`` identically:
  * POOL  ``mode=max`` (default; padding never wins) or ``mode=avg`` (divisor k*k)
  * LRN   ``size=5 alpha=1e-4 beta=0.75 k=2.0`` (AlexNet), y = x / (k + alpha/size * sum x^2)^beta
  * DROPOUT ``rate=0.5``; mask = hash(seed, layer, iteration, index) (no stored mask)
  * BN    batch statistics, eps 1e-5, momentum 0.1 (running stats updated once per iteration)
  * SOFTMAX (terminal) + cross-entropy, mean over the batch
  * ACT   ReLU; JOIN = elementwise sum; FC flattens NHWC (h, w, c) order
Tensors are fp32 NHWC; CONV/FC contract on tcgen05 in tf32 with fp32 accumulation
(``precision="tf32"``, the default) or, with ``precision="fp32"``, as 3xTF32
split operands (hi.hi + hi.lo + lo.hi, fp32-level products) in the generic
gather kernel -- the fp32-faithful mode the numeric parity tests pin at 1e-4.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

from . import _cabi, _native
from .errors import DeviceError, KIND_TO_EXC, MemschedError
from .netgraph import LayerKind, NetworkDef
from .simulator import SimConfig, SimReport, plan_handle, report_from_handle

__all__ = ["LayerNumerics", "layer_numerics", "Executor", "TrainingReport", "run_training",
           "init_parameters", "param_layout"]


class NumericsC(C.Structure):
    _fields_ = [("pool_mode", C.c_int32), ("lrn_size", C.c_int32), ("lrn_alpha", C.c_float),
                ("lrn_beta", C.c_float), ("lrn_k", C.c_float), ("dropout_rate", C.c_float),
                ("bn_eps", C.c_float), ("bn_momentum", C.c_float)]


class ExecOptionsC(C.Structure):
    _fields_ = [("device", C.c_int32), ("elide_backups", C.c_int32), ("use_graph", C.c_int32),
                ("num_classes", C.c_int32), ("seed", C.c_uint64), ("lr", C.c_float),
                ("grad_scale", C.c_float), ("precision", C.c_int32), ("stash", C.c_int32),
                ("stash_device", C.c_int32), ("autotune", C.c_int32), ("dp_comm", C.c_void_p),
                ("dp_world", C.c_int32), ("dp_rank", C.c_int32), ("dp_bucket_bytes", C.c_int64)]


PRECISIONS = {"tf32": 0, "fp32": 1}


class ExecMemC(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "arena_bytes", "params_grads_bytes", "layer_state_bytes", "input_bytes", "wgrad_scratch_bytes",
        "other_scratch_bytes", "host_stash_bytes", "device_stash_bytes", "peer_stash_bytes", "device_total_bytes",
        "wgrad_partials_outside_pool_bytes",
        "planned_arena_high_water")]


class CatalogC(C.Structure):
    _fields_ = [("layer", C.c_int32), ("op", C.c_int32), ("halo", C.c_int32), ("pairs", C.c_int32),
                ("bn", C.c_int32), ("subpix", C.c_int32), ("us", C.c_float), ("chosen", C.c_int32)]


class TimingC(C.Structure):
    _fields_ = [("step_ms", C.c_float), ("h2d_ms", C.c_float), ("d2h_ms", C.c_float),
                ("kernels", C.c_int64), ("d2h_bytes", C.c_int64), ("h2d_bytes", C.c_int64),
                ("arena_high_water", C.c_int64)]


@dataclass(frozen=True)
class LayerNumerics:
    pool_mode: int = 0
    lrn_size: int = 5
    lrn_alpha: float = 1e-4
    lrn_beta: float = 0.75
    lrn_k: float = 2.0
    dropout_rate: float = 0.5
    bn_eps: float = 1e-5
    bn_momentum: float = 0.1


def _num(params: dict, key: str, default):
    v = params.get(key, default)
    return v if isinstance(v, (int, float)) and not isinstance(v, bool) else default


def layer_numerics(net: NetworkDef) -> list[LayerNumerics]:
    out = []
    for lay in net.layers:
        p = lay.params
        mode = p.get("mode", "max")
        if mode not in ("max", "avg"):
            raise MemschedError(f"layer {lay.name!r}: POOL mode must be max or avg, got {mode!r}")
        out.append(LayerNumerics(
            pool_mode=1 if mode == "avg" else 0,
            lrn_size=int(_num(p, "size", 5)), lrn_alpha=float(_num(p, "alpha", 1e-4)),
            lrn_beta=float(_num(p, "beta", 0.75)), lrn_k=float(_num(p, "k", 2.0)) if lay.kind is LayerKind.LRN else 2.0,
            dropout_rate=float(_num(p, "rate", 0.5)),
            bn_eps=float(_num(p, "eps", 1e-5)), bn_momentum=float(_num(p, "momentum", 0.1))))
    return out


def param_layout(net: NetworkDef, shapes: dict[int, tuple[int, ...]]) -> dict[int, dict]:
    """Canonical (unpadded) parameter tensors per layer.

    CONV: w [K][R][S][C] (KRSC), b [K]; FC: w [O][I] over the NHWC-flattened
    input, b [O]; BN: gamma [C], beta [C].
    """
    out: dict[int, dict] = {}
    for lay in net.layers:
        if lay.kind is LayerKind.CONV:
            cin = shapes[lay.prev[0]][0]
            k = lay.params["k"]
            out[lay.id] = {"w": (shapes[lay.id][0], k, k, cin), "b": (shapes[lay.id][0],)}
        elif lay.kind is LayerKind.FC:
            fan_in = math.prod(shapes[lay.prev[0]])
            out[lay.id] = {"w": (shapes[lay.id][0], fan_in), "b": (shapes[lay.id][0],)}
        elif lay.kind is LayerKind.BN:
            out[lay.id] = {"w": (shapes[lay.id][0],), "b": (shapes[lay.id][0],)}
    return out


def init_parameters(net: NetworkDef, seed: int = 2, head_scale: float = 1.0) -> dict[int, dict]:
    """He-uniform CONV/FC weights (bound sqrt(6/fan_in)), small uniform biases,
    BN gamma = 1 / beta = 0; torch CPU generator, layer order.  ``head_scale``
    multiplies the classifier (the FC feeding the terminal SOFTMAX): small
    values keep the initial softmax away from saturation, which keeps
    gradient comparisons well conditioned."""
    import torch
    from .costmodel import propagate_shapes
    shapes = propagate_shapes(net)
    g = torch.Generator().manual_seed(seed)
    head = {p for l in net.layers if l.kind is LayerKind.SOFTMAX for p in l.prev}
    params: dict[int, dict] = {}
    for lid, spec in param_layout(net, shapes).items():
        kind = net.layers[lid].kind
        if kind is LayerKind.BN:
            params[lid] = {"w": torch.ones(spec["w"]), "b": torch.zeros(spec["b"])}
            continue
        fan_in = math.prod(spec["w"][1:])
        bound = math.sqrt(6.0 / fan_in)
        w = (torch.rand(spec["w"], generator=g) * 2 - 1) * bound
        b = (torch.rand(spec["b"], generator=g) * 2 - 1) / math.sqrt(fan_in)
        if lid in head:
            w, b = w * head_scale, b * head_scale
        params[lid] = {"w": w, "b": b}
    return params


def _xlib():
    L = _native.executor()
    if not getattr(L, "_sn_configured", False):
        P = C.POINTER
        L.sn_exec_last_error.restype = C.c_char_p
        L.sn_exec_last_error_kind.restype = C.c_int
        L.sn_exec_create.argtypes = [C.c_void_p, C.c_void_p, P(NumericsC), P(ExecOptionsC), P(C.c_void_p)]
        L.sn_exec_destroy.argtypes = [C.c_void_p]
        L.sn_exec_destroy.restype = None
        L.sn_exec_params.argtypes = [C.c_void_p, P(C.c_void_p), P(C.c_void_p), P(C.c_int64)]
        L.sn_exec_param_slice.argtypes = [C.c_void_p, C.c_int32] + [P(C.c_int64)] * 4
        L.sn_exec_inputs.argtypes = [C.c_void_p, P(C.c_void_p), P(C.c_void_p), P(C.c_int64)]
        L.sn_exec_step.argtypes = [C.c_void_p, C.c_int32, P(C.c_float), P(TimingC)]
        L.sn_exec_step_host.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, P(C.c_float), P(TimingC)]
        L.sn_exec_step_host_pipelined.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                  C.c_int32, P(C.c_float), P(TimingC)]
        L.sn_exec_train_host.argtypes = [C.c_void_p, C.c_int32, P(C.c_void_p), P(C.c_void_p), C.c_int32,
                                         P(C.c_float), P(TimingC)]
        L.sn_exec_read_tensor.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int64]
        L.sn_exec_apply_update.argtypes = [C.c_void_p, C.c_float, C.c_float]
        L.sn_exec_workspace_use.argtypes = [C.c_void_p, P(C.c_int32), P(C.c_int32)]
        L.sn_exec_transfer_stats.argtypes = [C.c_void_p, P(C.c_int64), P(C.c_double), P(C.c_int64),
                                             P(C.c_double), P(C.c_double)]
        L.sn_exec_profile.argtypes = [C.c_void_p, P(C.c_float), P(C.c_int32), P(C.c_int32), C.c_size_t,
                                      P(C.c_size_t)]
        L.sn_exec_census.argtypes = [C.c_void_p, P(C.c_int32), C.c_size_t, C.c_char_p, C.c_size_t,
                                     P(C.c_size_t)]
        L.sn_exec_memory.argtypes = [C.c_void_p, P(ExecMemC)]
        L.sn_exec_arena_fill.argtypes = [C.c_void_p]
        L.sn_exec_arena_scan.argtypes = [C.c_void_p, P(C.c_int64), P(C.c_int64)]
        L.sn_exec_catalog.argtypes = [C.c_void_p, P(CatalogC), C.c_size_t, P(C.c_size_t)]
        L.sn_exec_kernel_times.argtypes = [C.c_void_p, C.c_int32, P(C.c_float), P(C.c_int32), C.c_size_t,
                                           P(C.c_size_t)]
        L.sn_exec_stream.argtypes = [C.c_void_p]
        L.sn_exec_stream.restype = C.c_void_p
        L._sn_configured = True
    return L


def _raise_exec(L) -> None:
    kind = L.sn_exec_last_error_kind()
    msg = L.sn_exec_last_error().decode("utf-8", "replace")
    raise KIND_TO_EXC.get(kind, DeviceError)(msg)


class Executor:
    """One training replica on one B200, executing the planner's tape."""

    def __init__(self, net: NetworkDef, config: SimConfig, device: int = 0, *, seed: int = 2,
                 dropout_seed: int = 1234, lr: float = 0.01, grad_scale: float = 1.0,
                 elide_backups: bool = True, use_graph: bool = True, params: dict | None = None,
                 precision: str = "tf32", dp=None, dp_bucket_bytes: int = 0, stash: str = "host",
                 stash_device: int | None = None, autotune: bool = False) -> None:
        import torch
        if not torch.cuda.is_available():
            raise DeviceError("run_training needs a CUDA device (B200); there is no CPU fallback")
        self.net = net
        self.config = config
        self.plan = plan_handle(net, config)   # raises the reference's errors
        self.report: SimReport = report_from_handle(net, config, self.plan)
        self.L = _xlib()
        nums = (NumericsC * len(net.layers))(*[
            NumericsC(n.pool_mode, n.lrn_size, n.lrn_alpha, n.lrn_beta, n.lrn_k, n.dropout_rate,
                      n.bn_eps, n.bn_momentum) for n in layer_numerics(net)])
        if precision not in PRECISIONS:
            raise MemschedError(f"precision must be one of {sorted(PRECISIONS)}, got {precision!r}")
        self.precision = precision
        # data-parallel replica (dp.DPContext): NCCL communicator for the bucketed
        # gradient all-reduce; each rank draws its own dropout masks, and the
        # update applies lr * sum_ranks(grad) / world unless grad_scale is given
        self.dp = dp if (dp is not None and dp.world > 1) or (dp is not None and dp.force_comm) else None
        comm = None
        if self.dp is not None:
            from .dp import rank_seed
            comm = self.dp.comm(device)
            dropout_seed = rank_seed(dropout_seed, self.dp)
            if grad_scale == 1.0:
                grad_scale = 1.0 / self.dp.world
        # Unified Tensor Pool backing store of copied-out tensors: pinned host
        # memory ("host", PCIe) or HBM of a device ("device": stash_device, an
        # NVLink peer, or this GPU itself as a loopback)
        if stash not in ("host", "device"):
            raise MemschedError(f"stash must be 'host' or 'device', got {stash!r}")
        opts = ExecOptionsC(device, int(elide_backups), int(use_graph), 0, dropout_seed, lr, grad_scale,
                            PRECISIONS[precision], int(stash == "device"),
                            device if stash_device is None else stash_device, int(autotune), comm,
                            self.dp.world if self.dp else 1, self.dp.rank if self.dp else 0, dp_bucket_bytes)
        self.ptr = C.c_void_p()
        torch.cuda.set_device(device)
        torch.cuda.synchronize()
        if self.L.sn_exec_create(self.plan.ptr, None, nums, C.byref(opts), C.byref(self.ptr)) != 0:
            _raise_exec(self.L)
        self.device = device
        self.batch = config.cost.batch
        p, g, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        self.L.sn_exec_params(self.ptr, C.byref(p), C.byref(g), C.byref(n))
        self.params_ptr, self.grads_ptr, self.n_params = p.value, g.value, n.value
        im, lab, nimg = C.c_void_p(), C.c_void_p(), C.c_int64()
        self.L.sn_exec_inputs(self.ptr, C.byref(im), C.byref(lab), C.byref(nimg))
        self.images_ptr, self.labels_ptr, self.image_floats = im.value, lab.value, nimg.value
        from .costmodel import propagate_shapes
        self.shapes = propagate_shapes(net)
        self.data_id = net.data_id
        # the executor takes NHWC images with the net's own channel count and
        # lays them out for the stem itself (channel / spatial padding on device)
        self.c_real = self.shapes[self.data_id][0]
        self.set_parameters(params if params is not None else init_parameters(net, seed))

    # ---- parameters ---------------------------------------------------------
    def _slice(self, lid: int) -> tuple[int, int, int, int]:
        wo, wn, bo, bn = (C.c_int64() for _ in range(4))
        self.L.sn_exec_param_slice(self.ptr, lid, C.byref(wo), C.byref(wn), C.byref(bo), C.byref(bn))
        return wo.value, wn.value, bo.value, bn.value

    def _flat(self, which: str):
        import torch
        base = self.params_ptr if which == "params" else self.grads_ptr
        return _device_view(base, self.n_params, self.device)

    def set_parameters(self, params: dict[int, dict]) -> None:
        import torch
        flat = self._flat("params")
        for lid, t in params.items():
            wo, wn, bo, bn = self._slice(lid)
            w = t["w"]
            if self.net.layers[lid].kind is LayerKind.CONV and w.shape[3] != self._conv_cin(lid):
                pad = self._conv_cin(lid) - w.shape[3]
                w = torch.nn.functional.pad(w, (0, pad))
            flat[wo:wo + wn].copy_(w.reshape(-1).to(flat.device))
            flat[bo:bo + bn].copy_(t["b"].reshape(-1).to(flat.device))
        torch.cuda.synchronize(self.device)

    def _conv_cin(self, lid: int) -> int:
        wo, wn, _, _ = self._slice(lid)
        k = self.net.layers[lid].params["k"]
        return wn // (self.shapes[lid][0] * k * k)

    def get(self, which: str = "grads") -> dict[int, dict]:
        """Canonical (unpadded) copies of parameters or gradients, on CPU."""
        import torch
        torch.cuda.synchronize(self.device)
        flat = self._flat(which).cpu()
        out = {}
        for lid, spec in param_layout(self.net, self.shapes).items():
            wo, wn, bo, bn = self._slice(lid)
            w = flat[wo:wo + wn]
            if self.net.layers[lid].kind is LayerKind.CONV:
                K, R, S, Cr = spec["w"]
                w = w.reshape(K, R, S, wn // (K * R * S))[..., :Cr]
            out[lid] = {"w": w.reshape(spec["w"]).clone(), "b": flat[bo:bo + bn].clone()}
        return out

    # ---- inputs / steps -----------------------------------------------------
    def set_inputs(self, images, labels) -> None:
        """images: (B, C, H, W) or NHWC (B, H, W, C) float32 tensor; labels (B,)."""
        import torch
        img = images
        if img.dim() == 4 and img.shape[1] == self.c_real and img.shape[-1] != self.c_real:
            img = img.permute(0, 2, 3, 1)
        img = img.float().contiguous()
        dst = _device_view(self.images_ptr, self.image_floats, self.device)
        dst.copy_(img.reshape(-1).to(dst.device))
        lab = _device_view(self.labels_ptr, self.batch, self.device, torch.int32)
        lab.copy_(labels.to(torch.int32).reshape(-1).to(lab.device))
        torch.cuda.synchronize(self.device)

    def step(self, update: bool = True) -> tuple[float, TimingC]:
        loss = C.c_float()
        t = TimingC()
        if self.L.sn_exec_step(self.ptr, int(update), C.byref(loss), C.byref(t)) != 0:
            _raise_exec(self.L)
        return loss.value, t

    def step_host(self, images_host, labels_host, update: bool = True) -> tuple[float, TimingC]:
        """End to end: host (pinned) buffers in, loss out, copies timed."""
        loss = C.c_float()
        t = TimingC()
        if self.L.sn_exec_step_host(self.ptr, images_host.data_ptr(), labels_host.data_ptr(), int(update),
                                    C.byref(loss), C.byref(t)) != 0:
            _raise_exec(self.L)
        return loss.value, t

    def step_host_pipelined(self, images_host, labels_host, next_images_host=None, next_labels_host=None,
                            update: bool = True) -> tuple[float, TimingC]:
        """One end-to-end step on pinned host buffers that also stages the next
        batch's host->device copy behind this step's compute."""
        loss = C.c_float()
        t = TimingC()
        rc = self.L.sn_exec_step_host_pipelined(
            self.ptr, images_host.data_ptr(), labels_host.data_ptr(),
            None if next_images_host is None else next_images_host.data_ptr(),
            None if next_labels_host is None else next_labels_host.data_ptr(), int(update),
            C.byref(loss), C.byref(t))
        if rc != 0:
            _raise_exec(self.L)
        return loss.value, t

    def train_host(self, batches, update: bool = True) -> list[tuple[float, TimingC]]:
        """End to end over a sequence of pinned host (images NHWC, labels int32)
        batches in one native call (sn_exec_train_host): batch i+1 is copied to
        the device while step i computes (the data layer's one-batch prefetch)
        and step i's loss is read back while step i+1 runs.  Returns
        [(loss, timing)] per step; the timing (device ms per step, mean over
        the call) is shared."""
        batches = list(batches)
        n = len(batches)
        if n == 0:
            return []
        imgs = (C.c_void_p * n)(*[b[0].data_ptr() for b in batches])
        labs = (C.c_void_p * n)(*[b[1].data_ptr() for b in batches])
        losses = (C.c_float * n)()
        t = TimingC()
        if self.L.sn_exec_train_host(self.ptr, n, imgs, labs, int(update), losses, C.byref(t)) != 0:
            _raise_exec(self.L)
        return [(losses[i], t) for i in range(n)]

    def workspace_use(self) -> tuple[int, int]:
        """(CONV weight gradients with their split-K partials in the planned conv
        workspace, ones that needed scratch outside the pool)."""
        a, b = C.c_int32(), C.c_int32()
        if self.L.sn_exec_workspace_use(self.ptr, C.byref(a), C.byref(b)) != 0:
            _raise_exec(self.L)
        return a.value, b.value

    def transfer_stats(self) -> dict:
        """PCIe evidence of the last iteration: bytes, copy-engine ms and GB/s per
        direction, and the ms the compute stream was blocked on fetches."""
        db, hb = C.c_int64(), C.c_int64()
        dm, hm, xm = C.c_double(), C.c_double(), C.c_double()
        if self.L.sn_exec_transfer_stats(self.ptr, C.byref(db), C.byref(dm), C.byref(hb), C.byref(hm),
                                         C.byref(xm)) != 0:
            _raise_exec(self.L)
        gbs = lambda b, m: round(b / (m * 1e6), 2) if m > 0 else None  # noqa: E731
        return {"d2h_bytes": db.value, "d2h_ms": round(dm.value, 4), "d2h_GBps": gbs(db.value, dm.value),
                "h2d_bytes": hb.value, "h2d_ms": round(hm.value, 4), "h2d_GBps": gbs(hb.value, hm.value),
                "exposed_ms": round(xm.value, 4)}

    def read_activation(self, lid: int):
        """Layer output still resident at the end of the iteration, as (B, C, H, W)
        or (B, F); only meaningful when liveness is off (nothing is freed)."""
        import torch
        shape = self.shapes[lid]
        n = self.batch * math.prod(shape)
        out = torch.empty(n, device=f"cuda:{self.device}")
        if self.L.sn_exec_read_tensor(self.ptr, 0, lid, out.data_ptr(), n) != 0:
            _raise_exec(self.L)
        torch.cuda.synchronize(self.device)
        if len(shape) == 3:
            c, h, w = shape
            return out.reshape(self.batch, h, w, c).permute(0, 3, 1, 2).cpu()
        return out.reshape(self.batch, -1).cpu()

    def profile(self):
        """Per-action device ms of one eager iteration: [(ms, layer, type)]."""
        n = C.c_size_t()
        self.L.sn_exec_profile(self.ptr, None, None, None, 0, C.byref(n))
        ms = (C.c_float * max(1, n.value))()
        lay = (C.c_int32 * max(1, n.value))()
        typ = (C.c_int32 * max(1, n.value))()
        if self.L.sn_exec_profile(self.ptr, ms, lay, typ, n.value, C.byref(n)) != 0:
            _raise_exec(self.L)
        return [(ms[i], lay[i], typ[i]) for i in range(n.value)]

    def memory(self) -> dict:
        """Bytes the executor allocated, by purpose (sn_exec_memory)."""
        m = ExecMemC()
        if self.L.sn_exec_memory(self.ptr, C.byref(m)) != 0:
            _raise_exec(self.L)
        return {n: getattr(m, n) for n, _ in ExecMemC._fields_}

    def measure_arena(self) -> dict:
        """Measured arena use of one iteration: the arena is filled with a
        sentinel, one step runs (no update), and the 1 KiB blocks any kernel or
        copy wrote are counted on the device (the union of every placement in
        the iteration; gradient buffers are placed from the top of the pool,
        as the reference's BlockPool(high=True) does, so the highest written
        block is the arena's end whenever a gradient buffer was allocated)."""
        if self.L.sn_exec_arena_fill(self.ptr) != 0:
            _raise_exec(self.L)
        self.step(update=False)
        hw, touched = C.c_int64(), C.c_int64()
        if self.L.sn_exec_arena_scan(self.ptr, C.byref(hw), C.byref(touched)) != 0:
            _raise_exec(self.L)
        return {"measured_arena_written_bytes": touched.value, "measured_arena_highest_written_byte": hw.value}

    def catalog(self) -> list[dict]:
        """The measured CONV kernel-variant catalog (``autotune=True``): every
        variant timed per layer shape and op, and which one the layers of that
        shape run (empty without autotune)."""
        n = C.c_size_t()
        self.L.sn_exec_catalog(self.ptr, None, 0, C.byref(n))
        buf = (CatalogC * max(1, n.value))()
        if self.L.sn_exec_catalog(self.ptr, buf, n.value, C.byref(n)) != 0:
            _raise_exec(self.L)
        ops = ("fwd", "dgrad", "wgrad")
        return [{"layer": self.net.layers[e.layer].name, "op": ops[e.op],
                 "variant": {"halo": e.halo, "pairs": e.pairs, "bn": e.bn, "subpix": e.subpix},
                 "us": round(e.us, 2), "chosen": bool(e.chosen)} for e in buf[:n.value]]

    def kernel_times(self, reps: int = 3) -> list[tuple[int, float]]:
        """(action index, microseconds) of every kernel of one serial iteration
        in issue order: the iteration replayed node by node with a CUDA event
        pair around each kernel, median of ``reps`` replays."""
        n = C.c_size_t()
        if self.L.sn_exec_kernel_times(self.ptr, reps, None, None, 0, C.byref(n)) != 0:
            _raise_exec(self.L)
        us = (C.c_float * max(1, n.value))()
        act = (C.c_int32 * max(1, n.value))()
        if self.L.sn_exec_kernel_times(self.ptr, reps, us, act, n.value, C.byref(n)) != 0:
            _raise_exec(self.L)
        return [(act[i], us[i]) for i in range(n.value)]

    def census(self) -> list[list[str]]:
        """Per tape action (the same list ``profile`` times), the mangled names
        of the kernels it launches, from one captured serial iteration."""
        n = C.c_size_t()
        self.L.sn_exec_census(self.ptr, None, 0, None, 0, C.byref(n))
        counts = (C.c_int32 * max(1, n.value))()
        cap = 1 << 22
        buf = C.create_string_buffer(cap)
        if self.L.sn_exec_census(self.ptr, counts, n.value, buf, cap, C.byref(n)) != 0:
            _raise_exec(self.L)
        per = buf.value.decode("utf-8", "replace").split("\x1e")[:n.value]
        out = [[k for k in p.split("\n") if k] for p in per]
        assert [len(o) for o in out] == list(counts[:n.value]), "census name list truncated"
        return out

    def apply_update(self, lr: float, grad_scale: float = 1.0) -> None:
        if self.L.sn_exec_apply_update(self.ptr, lr, grad_scale) != 0:
            _raise_exec(self.L)

    def grads_tensor(self):
        return self._flat("grads")

    def close(self) -> None:
        if getattr(self, "ptr", None) is not None and self.ptr.value:
            self.L.sn_exec_destroy(self.ptr)
            self.ptr = None

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass


def _device_view(ptr: int, n: int, device: int, dtype=None):
    """A non-owning torch view of executor memory (no caching-allocator use)."""
    import torch
    dtype = dtype or torch.float32
    esize = torch.empty((), dtype=dtype).element_size()

    class _Holder:
        __cuda_array_interface__ = {
            "shape": (n,), "typestr": {4: "<f4"}[esize] if dtype == torch.float32 else "<i4",
            "data": (ptr, False), "version": 3, "strides": None}

    return torch.as_tensor(_Holder(), device=f"cuda:{device}")


@dataclass(frozen=True)
class TrainingReport:
    schedule: SimReport
    images_per_s: float
    ms_per_step: float
    losses: tuple[float, ...]
    kernels_per_step: int
    d2h_bytes_per_step: int
    h2d_bytes_per_step: int
    extras: dict = field(default_factory=dict)


def run_training(net: NetworkDef, config: SimConfig, iters: int = 10, warmup: int = 3, device: int = 0,
                 seed: int = 0, **exec_kw) -> TrainingReport:
    """Plan with ``config`` (exactly as ``run_simulation``) and train for real."""
    import torch
    ex = Executor(net, config, device=device, **exec_kw)
    from .costmodel import propagate_shapes
    c, h, w = propagate_shapes(net)[net.data_id]
    g = torch.Generator().manual_seed(seed)
    images = torch.randn(config.cost.batch, c, h, w, generator=g)
    labels = torch.randint(0, max(1, math.prod(propagate_shapes(net)[net.terminal_id])),
                           (config.cost.batch,), generator=torch.Generator().manual_seed(seed + 1))
    ex.set_inputs(images, labels)
    for _ in range(warmup):
        ex.step()
    losses, times = [], []
    t = None
    for _ in range(iters):
        loss, t = ex.step()
        losses.append(loss)
        times.append(t.step_ms)
    ms = sum(times) / max(1, len(times))
    extras = {"memory": ex.memory(), "arena": ex.measure_arena()}
    rep = TrainingReport(schedule=ex.report, images_per_s=config.cost.batch / (ms / 1e3) if ms else 0.0,
                         ms_per_step=ms, losses=tuple(losses), kernels_per_step=t.kernels if t else 0,
                         d2h_bytes_per_step=t.d2h_bytes if t else 0, h2d_bytes_per_step=t.h2d_bytes if t else 0,
                         extras=extras)
    ex.close()
    return rep
