"""ctypes mirror of include/superneurons.h and NetworkDef marshaling."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _native
from .errors import KIND_TO_EXC, MemschedError
from .netgraph import LayerKind, NetworkDef

KIND_CODE = {k: i for i, k in enumerate([
    LayerKind.DATA, LayerKind.CONV, LayerKind.POOL, LayerKind.ACT, LayerKind.LRN, LayerKind.BN,
    LayerKind.FC, LayerKind.DROPOUT, LayerKind.SOFTMAX, LayerKind.JOIN])}
PARAM_KEYS = ("c", "h", "w", "out", "k", "s", "p")
RC_CODE = {None: 0, "speed": 1, "memory": 2, "cost-aware": 3}
RC_NAME = {1: "speed", 2: "memory"}
ALGO_NAMES = ("implicit-gemm", "gemm-workspace", "fft")
INT64_MAX = (1 << 63) - 1


class NetDesc(C.Structure):
    _fields_ = [
        ("name", C.c_char_p), ("n_layers", C.c_int32), ("kinds", C.POINTER(C.c_int32)),
        ("names", C.POINTER(C.c_char_p)), ("name_reprs", C.POINTER(C.c_char_p)),
        ("prev_off", C.POINTER(C.c_int32)), ("prev_idx", C.POINTER(C.c_int32)),
        ("next_off", C.POINTER(C.c_int32)), ("next_idx", C.POINTER(C.c_int32)),
        ("param_state", C.POINTER(C.c_int8)), ("param_int", C.POINTER(C.c_int64)),
        ("param_repr", C.POINTER(C.c_char_p)),
    ]


class SimConfigC(C.Structure):
    _fields_ = [
        ("pool_bytes", C.c_int64), ("liveness", C.c_int32), ("offload", C.c_int32),
        ("cache", C.c_int32), ("recompute", C.c_int32), ("convselect", C.c_int32),
        ("batch", C.c_int64), ("dtype_bytes", C.c_int64), ("time_per_elem", C.c_double),
        ("heavy_time_per_elem", C.c_double), ("backward_time_factor", C.c_double),
        ("bandwidth_bytes_per_s", C.c_double),
    ]


class ReportC(C.Structure):
    _fields_ = [
        ("num_layers", C.c_int32), ("num_steps", C.c_int32), ("peak_bytes", C.c_int64),
        ("peak_step", C.c_int32), ("peak_layer", C.c_int32), ("peak_live_count", C.c_int64),
        ("peak_working_bytes", C.c_int64), ("peak_stash_bytes", C.c_int64),
        ("min_pool_bytes", C.c_int64), ("baseline_peak_bytes", C.c_int64),
        ("liveness_peak_bytes", C.c_int64), ("compute_s", C.c_double), ("stall_s", C.c_double),
        ("stall_prefetch_s", C.c_double), ("stall_demand_s", C.c_double),
        ("stall_backup_s", C.c_double), ("transfer_busy_s", C.c_double), ("total_s", C.c_double),
        ("scheduled_transfer_bytes", C.c_int64), ("scheduled_transfer_count", C.c_int64),
        ("demand_transfer_bytes", C.c_int64), ("demand_transfer_count", C.c_int64),
        ("cache_hits", C.c_int64), ("evictions", C.c_int64), ("extra_forward_steps", C.c_int64),
        ("planned_extra_forward_steps", C.c_int64), ("pool_high_water_bytes", C.c_int64),
        ("n_rows", C.c_int32), ("n_selections", C.c_int32), ("n_modes", C.c_int32),
    ]


class RowC(C.Structure):
    _fields_ = [
        ("index", C.c_double), ("layer", C.c_int32), ("phase", C.c_int32),
        ("resident_bytes", C.c_int64), ("live_count", C.c_int64), ("pool_used_bytes", C.c_int64),
        ("compute_s", C.c_double), ("stall_s", C.c_double), ("transfer_bytes", C.c_int64),
    ]


class SelectionC(C.Structure):
    _fields_ = [
        ("step", C.c_double), ("layer", C.c_int32), ("phase", C.c_int32), ("algo", C.c_int32),
        ("pad_", C.c_int32), ("workspace_bytes", C.c_int64), ("free_bytes", C.c_int64),
    ]


class EventC(C.Structure):
    _fields_ = [
        ("op", C.c_char), ("pad_", C.c_char * 3), ("a", C.c_int32), ("b", C.c_int32),
        ("e", C.c_int32), ("c", C.c_int64), ("d", C.c_int64),
    ]


class LayerCostC(C.Structure):
    _fields_ = [
        ("ndim", C.c_int32), ("pad_", C.c_int32), ("shape", C.c_int64 * 3),
        ("out_elems", C.c_int64), ("out_bytes", C.c_int64), ("device_bytes", C.c_int64),
        ("grad_bytes", C.c_int64), ("param_bytes", C.c_int64), ("fwd_time", C.c_double),
        ("bwd_time", C.c_double),
    ]


_configured = False


def lib() -> C.CDLL:
    global _configured
    L = _native.planner()
    if not _configured:
        P = C.POINTER
        sz = P(C.c_size_t)
        L.sn_version.restype = C.c_char_p
        L.sn_last_error.restype = C.c_char_p
        L.sn_last_error_kind.restype = C.c_int
        L.sn_plan_create.argtypes = [P(NetDesc), P(SimConfigC), P(C.c_void_p)]
        L.sn_analyze.argtypes = [P(NetDesc), P(SimConfigC), P(C.c_void_p)]
        L.sn_build_costs.argtypes = [P(NetDesc), P(SimConfigC), P(C.c_void_p)]
        L.sn_plan_destroy.argtypes = [C.c_void_p]
        L.sn_plan_destroy.restype = None
        L.sn_plan_report.argtypes = [C.c_void_p, P(ReportC)]
        L.sn_plan_rows.argtypes = [C.c_void_p, P(RowC), C.c_size_t, sz]
        L.sn_plan_selections.argtypes = [C.c_void_p, P(SelectionC), C.c_size_t, sz]
        L.sn_plan_modes.argtypes = [C.c_void_p, P(C.c_int32), C.c_size_t, sz]
        L.sn_plan_tape.argtypes = [C.c_void_p, P(P(EventC)), sz]
        L.sn_plan_costs.argtypes = [C.c_void_p, P(LayerCostC), C.c_size_t, sz]
        L.sn_plan_order.argtypes = [C.c_void_p, P(C.c_int32), C.c_size_t, sz]
        L.sn_plan_demands.argtypes = [C.c_void_p, P(C.c_int64), C.c_size_t, sz]
        L.sn_debug_pyset.argtypes = [P(C.c_int64), C.c_size_t, P(C.c_int64), C.c_size_t,
                                     P(C.c_int64), C.c_size_t, P(C.c_int64), C.c_size_t, sz]
        _configured = True
    return L


def raise_last(L: C.CDLL) -> None:
    kind = L.sn_last_error_kind()
    msg = L.sn_last_error().decode("utf-8", "replace")
    exc = KIND_TO_EXC.get(kind, MemschedError)
    raise exc(msg)


@dataclass
class MarshaledNet:
    """Keeps the ctypes buffers alive for as long as the descriptor is used."""

    desc: NetDesc
    keep: list


def marshal_net(net: NetworkDef) -> MarshaledNet:
    n = len(net.layers)
    keep: list = []

    def arr(ctype, values):
        a = (ctype * max(1, len(values)))(*values)
        keep.append(a)
        return a

    kinds = arr(C.c_int32, [KIND_CODE[l.kind] for l in net.layers])
    names = arr(C.c_char_p, [l.name.encode() for l in net.layers])
    reprs = arr(C.c_char_p, [repr(l.name).encode() for l in net.layers])
    prev_off, prev_idx, next_off, next_idx = [0], [], [0], []
    for l in net.layers:
        prev_idx.extend(l.prev)
        prev_off.append(len(prev_idx))
        next_idx.extend(l.next)
        next_off.append(len(next_idx))
    state, ints, preprs = [], [], []
    for l in net.layers:
        for key in PARAM_KEYS:
            if key not in l.params:
                state.append(0), ints.append(0), preprs.append(None)
                continue
            v = l.params[key]
            if isinstance(v, int) and not isinstance(v, bool):
                if abs(v) > INT64_MAX:
                    raise MemschedError(
                        f"layer {l.name!r} parameter {key!r} exceeds the 64-bit planner range")
                state.append(1), ints.append(v), preprs.append(None)
            else:
                state.append(2), ints.append(0), preprs.append(repr(v).encode())
    name_b = net.name.encode()
    keep.append(name_b)
    desc = NetDesc(name_b, n, kinds, names, reprs, arr(C.c_int32, prev_off),
                   arr(C.c_int32, prev_idx), arr(C.c_int32, next_off), arr(C.c_int32, next_idx),
                   arr(C.c_int8, state), arr(C.c_int64, ints), arr(C.c_char_p, preprs))
    return MarshaledNet(desc, keep)


def sim_config(pool_bytes: int, features, cost) -> SimConfigC:
    f = features.normalized()
    for name, v in (("pool_bytes", pool_bytes), ("batch", cost.batch), ("dtype_bytes", cost.dtype_bytes)):
        if abs(int(v)) > INT64_MAX:
            raise MemschedError(f"{name} exceeds the 64-bit planner range")
    return SimConfigC(int(pool_bytes), int(f.liveness), int(f.offload), int(f.cache),
                      RC_CODE[f.recompute], int(f.convselect), int(cost.batch), int(cost.dtype_bytes),
                      float(cost.time_per_elem), float(cost.heavy_time_per_elem),
                      float(cost.backward_time_factor), float(cost.bandwidth_bytes_per_s))


class PlanHandle:
    """Owns an ``sn_plan*``; fetches arrays lazily."""

    def __init__(self, net: NetworkDef, cfg: SimConfigC, mode: str = "run") -> None:
        self.L = lib()
        self.net = net
        self.m = marshal_net(net)
        self.ptr = C.c_void_p()
        fn = {"run": self.L.sn_plan_create, "analyze": self.L.sn_analyze,
              "costs": self.L.sn_build_costs}[mode]
        if fn(C.byref(self.m.desc), C.byref(cfg), C.byref(self.ptr)) != 0:
            raise_last(self.L)

    def __del__(self) -> None:
        ptr = getattr(self, "ptr", None)
        if ptr is not None and ptr.value:
            self.L.sn_plan_destroy(ptr)
            self.ptr = None

    def _array(self, fn, ctype):
        n = C.c_size_t()
        if fn(self.ptr, None, 0, C.byref(n)) != 0:
            raise_last(self.L)
        buf = (ctype * max(1, n.value))()
        if fn(self.ptr, buf, n.value, C.byref(n)) != 0:
            raise_last(self.L)
        return buf[: n.value]

    def report(self) -> ReportC:
        r = ReportC()
        if self.L.sn_plan_report(self.ptr, C.byref(r)) != 0:
            raise_last(self.L)
        return r

    def rows(self):
        return self._array(self.L.sn_plan_rows, RowC)

    def selections(self):
        return self._array(self.L.sn_plan_selections, SelectionC)

    def modes(self):
        return self._array(self.L.sn_plan_modes, C.c_int32)

    def costs(self):
        return self._array(self.L.sn_plan_costs, LayerCostC)

    def order(self):
        return list(self._array(self.L.sn_plan_order, C.c_int32))

    def demands(self):
        return list(self._array(self.L.sn_plan_demands, C.c_int64))

    def tape(self) -> list[EventC]:
        ptr = C.POINTER(EventC)()
        n = C.c_size_t()
        if self.L.sn_plan_tape(self.ptr, C.byref(ptr), C.byref(n)) != 0:
            raise_last(self.L)
        return [ptr[i] for i in range(n.value)]

    def tape_as_lists(self) -> list[list]:
        """The tape in the golden-vector vocabulary of tests/golden/make_golden.py."""
        kinds = ("act", "grad", "ws")
        out: list[list] = []
        for e in self.tape():
            op = e.op.decode()
            if op == "A":
                out.append(["A", kinds[e.a], e.b, e.c, e.d, e.e])
            elif op == "F":
                out.append(["F", kinds[e.a], e.b])
            elif op in "CB":
                out.append([op, e.b, "" if e.e < 0 else ALGO_NAMES[e.e], int(e.d)])
            else:
                out.append([op, e.b])
        return out
