"""Reconfigure path: shard layouts, transfer plans and the
device executor, over the C-ABI in include/coadapt_reshard.h.

Names follow SPEC.md's reshard module: ``layout_for``,
``plan_transfers``, ``estimate_reconfig_latency``, the plan CSV; execution
is ``TransferPlan.execute`` — a device pull of every destination region from
the source packs (local HBM or NVLink peers mapped with ``device.ipc_open``)
in place of SPEC's ``execute_in_memory``.

A rank's training state is one *pack* per state plane (bf16 parameters, each
fp32 optimizer state): its shards back to back in (layer, tensor) order,
row-major, each starting on a 64-element boundary (``Shard.pack_offset``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

from . import _lib as L
from ._lib import check, lib

SRC, DST = 0, 1
ROLE_ALL, ROLE_PULL, ROLE_PUSH = 0, 1, 2
POLICIES = {"canonical": 0, "spread": 1}


@dataclass(frozen=True)
class TensorDecl:
    name: str
    shape: tuple
    tp_axis: int = -1  # -1: replicated on every TP rank


@dataclass(frozen=True)
class ModelSpec:
    """SPEC.md:419-423."""
    layers: int
    per_layer: tuple
    optimizer_state_multiplier: int = 2
    param_bytes: int = 2
    state_bytes: int = 4

    def key(self, layer: int, tensor: int) -> str:
        return f"layer{layer}.{self.per_layer[tensor].name}"

    @property
    def bytes_per_element(self) -> int:
        return self.param_bytes + self.optimizer_state_multiplier * self.state_bytes


@dataclass(frozen=True)
class Shard:
    """ShardDescriptor."""
    layer: int
    tensor: int
    owner: int
    canonical: bool
    global_shape: tuple
    global_offset: tuple
    local_shape: tuple
    pack_offset: int


@dataclass(frozen=True)
class Move:
    src_rank: int
    dst_rank: int
    layer: int
    tensor: int
    offset: tuple
    extent: tuple
    bytes: int
    local: bool


def _dtp(s) -> tuple:
    if isinstance(s, str):  # "d2t1p4" or "2,1,4" (strategy.hpp:44-45)
        import re
        m = re.fullmatch(r"d(\d+)t(\d+)p(\d+)|(\d+),(\d+),(\d+)", s.strip())
        if not m:
            raise L.ValidationError(f"bad strategy label {s!r}")
        g = [x for x in m.groups() if x is not None]
        return int(g[0]), int(g[1]), int(g[2])
    d, t, p = s
    return int(d), int(t), int(p)


class TransferPlan:
    """layout_for(src) + layout_for(dst) + plan_transfers."""

    def __init__(self, model: ModelSpec, src, dst, policy: str = "canonical"):
        self.model = model
        self.src_dtp, self.dst_dtp = _dtp(src), _dtp(dst)
        if policy not in POLICIES:
            raise L.ValidationError(f"unknown source policy {policy!r}")
        n = len(model.per_layer)
        decls = (L.TensorDeclC * max(1, n))()
        self._names = [ts.name.encode() for ts in model.per_layer]
        for i, ts in enumerate(model.per_layer):
            if not 1 <= len(ts.shape) <= L.MAXD:
                raise L.ValidationError(f"{ts.name}: tensors have 1..{L.MAXD} axes")
            decls[i].name = self._names[i]
            decls[i].ndim = len(ts.shape)
            decls[i].tp_axis = int(ts.tp_axis)
            for k, e in enumerate(ts.shape):
                decls[i].shape[k] = int(e)
        m = L.ReshardModelC(int(model.layers), n, C.cast(decls, C.POINTER(L.TensorDeclC)),
                            int(model.optimizer_state_multiplier), int(model.param_bytes),
                            int(model.state_bytes), 0)
        h = C.c_void_p()
        check(lib().coadapt_reshard_plan_create(C.byref(m), (C.c_int32 * 3)(*self.src_dtp),
                                                (C.c_int32 * 3)(*self.dst_dtp), POLICIES[policy],
                                                C.byref(h)))
        self.handle = h
        info = L.ReshardInfoC()
        check(lib().coadapt_reshard_plan_info(h, C.byref(info)))
        self.info = info

    def close(self) -> None:
        if getattr(self, "handle", None):
            lib().coadapt_reshard_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass

    # ---------------------------------------------------------------- plan
    @property
    def total_bytes(self) -> int:
        return int(self.info.total_bytes)

    @property
    def max_bytes_per_rank(self) -> int:
        return int(self.info.max_bytes_per_rank)

    @property
    def local_bytes(self) -> int:
        return int(self.info.local_bytes)

    def moves(self) -> list:
        n = C.c_size_t(0)
        check(lib().coadapt_reshard_moves(self.handle, None, C.byref(n)))
        buf = (L.MoveC * max(1, n.value))()
        check(lib().coadapt_reshard_moves(self.handle, buf, C.byref(n)))
        out = []
        for m in buf[:n.value]:
            k = m.ndim
            out.append(Move(m.src_rank, m.dst_rank, m.layer, m.tensor, tuple(m.offset[:k]),
                            tuple(m.extent[:k]), int(m.bytes), bool(m.local)))
        return out

    def shards(self, side: int = DST) -> list:
        n = C.c_size_t(0)
        check(lib().coadapt_reshard_shards(self.handle, side, None, C.byref(n)))
        buf = (L.ShardC * max(1, n.value))()
        check(lib().coadapt_reshard_shards(self.handle, side, buf, C.byref(n)))
        return [Shard(s.layer, s.tensor, s.owner, bool(s.canonical), tuple(s.global_shape[:s.ndim]),
                      tuple(s.global_offset[:s.ndim]), tuple(s.local_shape[:s.ndim]), int(s.pack_offset))
                for s in buf[:n.value]]

    def pack_numel(self, side: int, rank: int) -> int:
        v = C.c_uint64()
        check(lib().coadapt_reshard_pack_numel(self.handle, side, int(rank), C.byref(v)))
        return int(v.value)

    def csv(self) -> str:
        need = C.c_size_t(0)
        check(lib().coadapt_reshard_plan_csv(self.handle, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value + 1)
        check(lib().coadapt_reshard_plan_csv(self.handle, buf, need.value + 1, C.byref(need)))
        return buf.value.decode()

    def latency(self, bandwidth_bytes_per_s: float = 1.0e9, fixed_overhead_s: float = 20.0) -> float:
        out = C.c_double()
        check(lib().coadapt_reshard_latency(self.handle, float(bandwidth_bytes_per_s),
                                            float(fixed_overhead_s), C.byref(out)))
        return out.value

    # ------------------------------------------------------------- execute
    def execute(self, src_packs: Sequence, dst_packs: Sequence, dst_rank: Optional[int] = None,
                src_rank: Optional[int] = None, elem_bytes: Optional[int] = None,
                device: Optional[int] = None, stream=None) -> None:
        """Copy the plan's regions for one state plane.  Default: every move
        (all packs visible here).  ``dst_rank=r``: pull the moves into r
        (this GPU reads local + peer sources); ``src_rank=r``: push the moves
        out of r (this GPU writes local + peer destinations).  Packs are
        CUDA tensors or raw device addresses (ints, e.g. IPC-mapped peers);
        None where unused."""
        from .device import _ptr, _stream
        if dst_rank is not None and src_rank is not None:
            raise L.ValidationError("pass dst_rank (pull) or src_rank (push), not both")
        role, rank = ((ROLE_PULL, dst_rank) if dst_rank is not None and dst_rank >= 0 else
                      (ROLE_PUSH, src_rank) if src_rank is not None else (ROLE_ALL, -1))
        ns, nd = len(src_packs), len(dst_packs)
        sp = (C.c_void_p * max(1, ns))(*[None if x is None else _ptr(x) for x in src_packs])
        dp = (C.c_void_p * max(1, nd))(*[None if x is None else _ptr(x) for x in dst_packs])
        if elem_bytes is None or device is None:
            t = next((x for x in list(dst_packs) + list(src_packs) if hasattr(x, "element_size")), None)
            if t is None:
                raise L.ValidationError("pass elem_bytes and device with raw pointers")
            elem_bytes = t.element_size() if elem_bytes is None else elem_bytes
            device = t.device.index if device is None else device
        check(lib().coadapt_reshard_execute(self.handle, role, int(rank), sp, ns, dp, nd,
                                            int(elem_bytes), int(device), _stream(stream)))


def plan_transfers(model: ModelSpec, src, dst, policy: str = "canonical") -> TransferPlan:
    return TransferPlan(model, src, dst, policy)


def layout_for(model: ModelSpec, strategy) -> list:
    """ShardLayout of one strategy as a list of Shards."""
    return TransferPlan(model, strategy, strategy).shards(SRC)


def estimate_reconfig_latency(plan: TransferPlan, bandwidth_bytes_per_s: float = 1.0e9,
                              fixed_overhead_s: float = 20.0) -> float:
    return plan.latency(bandwidth_bytes_per_s, fixed_overhead_s)
