"""Model shapes and (d,t,p) gradient-shard layouts.

A ModelSpec lists the parameter tensors of a transformer with the axis tensor
parallelism splits (or None when the tensor is replicated on every TP rank).
``rank_layout`` applies the spec's layout rules (contiguous PP
stages, equal contiguous TP chunks, DP replication) Megatron-style and
returns the rank's flattened gradient bucket as

* ``segments``  — (offset, numel, weight) for BucketPlan: weight 0 marks a
  copy another rank already counts (replicated tensor on tp_rank != 0, the
  tied-embedding copy on the last PP stage), so the global squared norm sums
  every logical parameter exactly once (north_star dedup);
* ``gen``       — generator segments mapping each bucket element to its
  logical parameter index, so synthetic gradients are layout-independent.

The four shapes are the BASELINE.json configs: GPT-2-small
(125M; vocab padded to 50304 as Megatron does), Llama-3.2-3B, Llama-2-7B
and Qwen2.5-32B.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

# synthetic value distribution: G_i = +-2^-10, exact in bf16
G0 = 2.0 ** -10
IH_STD = math.sqrt((4294967296.0 - 1.0) / 3.0)  # Irwin-Hall(4, 16-bit) std


def noise_unit_for(phi_true: float, micro_batch: int, g0: float = G0) -> float:
    """fp32 noise unit giving Var(zeta) = phi_true * g0^2 / B_m."""
    import numpy as np
    return float(np.float32(g0 * math.sqrt(phi_true / micro_batch) / IH_STD))


@dataclass(frozen=True)
class TensorSpec:
    name: str
    shape: tuple
    split_axis: Optional[int]  # TP split axis, None = replicated
    stage: str = "layer"       # "embed" | "layer" | "final" | "head"
    tied_to: Optional[str] = None  # head tied to the embedding


@dataclass
class ModelSpec:
    name: str
    layers: int
    per_layer: list
    embed: list
    final: list
    head: list = field(default_factory=list)
    tied: bool = False

    def tensors_in_order(self):
        """(TensorSpec, layer or None) over the whole model, logical order."""
        for t in self.embed:
            yield t, None
        for li in range(self.layers):
            for t in self.per_layer:
                yield t, li
        for t in self.final:
            yield t, None
        if not self.tied:
            for t in self.head:
                yield t, None

    def numel(self) -> int:
        return sum(math.prod(t.shape) for t, _ in self.tensors_in_order())


def _llama(name, vocab, h, layers, ffn, heads, kv_heads, tied, qkv_bias=False):
    hd = h // heads
    qkv_rows = h + 2 * kv_heads * hd
    per = [TensorSpec("input_norm", (h,), None),
           TensorSpec("qkv", (qkv_rows, h), 0)]
    if qkv_bias:
        per.append(TensorSpec("qkv_bias", (qkv_rows,), 0))
    per += [TensorSpec("o_proj", (h, h), 1),
            TensorSpec("post_norm", (h,), None),
            TensorSpec("gate_up", (2 * ffn, h), 0),
            TensorSpec("down", (h, ffn), 1)]
    embed = [TensorSpec("embed", (vocab, h), 0, "embed")]
    final = [TensorSpec("final_norm", (h,), None, "final")]
    head = [TensorSpec("lm_head", (vocab, h), 0, "head")]
    return ModelSpec(name, layers, per, embed, final, head, tied)


def gpt2_small() -> ModelSpec:
    h, ffn, vocab, pos = 768, 3072, 50304, 1024
    per = [TensorSpec("ln1_w", (h,), None), TensorSpec("ln1_b", (h,), None),
           TensorSpec("qkv_w", (3 * h, h), 0), TensorSpec("qkv_b", (3 * h,), 0),
           TensorSpec("proj_w", (h, h), 1), TensorSpec("proj_b", (h,), None),
           TensorSpec("ln2_w", (h,), None), TensorSpec("ln2_b", (h,), None),
           TensorSpec("fc_w", (ffn, h), 0), TensorSpec("fc_b", (ffn,), 0),
           TensorSpec("fc2_w", (h, ffn), 1), TensorSpec("fc2_b", (h,), None)]
    embed = [TensorSpec("wte", (vocab, h), 0, "embed"), TensorSpec("wpe", (pos, h), None, "embed")]
    final = [TensorSpec("lnf_w", (h,), None, "final"), TensorSpec("lnf_b", (h,), None, "final")]
    head = [TensorSpec("lm_head", (vocab, h), 0, "head")]
    return ModelSpec("gpt2-125m", 12, per, embed, final, head, tied=True)


def llama32_3b() -> ModelSpec:
    return _llama("llama3.2-3b", 128256, 3072, 28, 8192, 24, 8, tied=True)


def llama2_7b() -> ModelSpec:
    return _llama("llama2-7b", 32000, 4096, 32, 11008, 32, 32, tied=False)


def qwen25_32b() -> ModelSpec:
    return _llama("qwen2.5-32b", 152064, 5120, 64, 27648, 40, 8, tied=False, qkv_bias=True)


def tiny_model(layers=4, h=64, ffn=128, vocab=96, tied=False) -> ModelSpec:
    """Small Llama-like spec for tests (every dim divisible by t in {1,2,4})."""
    return _llama(f"tiny-l{layers}", vocab, h, layers, ffn, 4, 2, tied=tied, qkv_bias=True)


MODELS = {"125m": gpt2_small, "3b": llama32_3b, "7b": llama2_7b, "32b": qwen25_32b}


@dataclass
class RankLayout:
    rank: int
    coords: tuple           # (i_d, i_t, i_p)
    numel: int              # bucket elements
    segments: list          # [(offset, numel, weight)]
    gen: list               # [(local_off, numel, global_base, row_len, row_stride)]
    names: list             # tensor label per segment

    @property
    def counted(self) -> int:
        return sum(n for _, n, w in self.segments if w != 0.0)


def rank_coords(rank: int, d: int, t: int, p: int) -> tuple:
    """Megatron order: tp fastest, then dp, then pp."""
    i_t = rank % t
    i_d = (rank // t) % d
    i_p = rank // (t * d)
    return i_d, i_t, i_p


def rank_layout(spec: ModelSpec, d: int, t: int, p: int, rank: int) -> RankLayout:
    if spec.layers % p:
        raise ValueError(f"{spec.name}: {spec.layers} layers not divisible by p={p}")
    i_d, i_t, i_p = rank_coords(rank, d, t, p)
    lo, hi = i_p * spec.layers // p, (i_p + 1) * spec.layers // p
    # logical base offset of every (tensor, layer) in the unsharded model
    base, cursor = {}, 0
    for ts, li in spec.tensors_in_order():
        base[(ts.name, li)] = cursor
        cursor += math.prod(ts.shape)
    local = []
    if i_p == 0:
        local += [(ts, None, 1.0) for ts in spec.embed]
    for li in range(lo, hi):
        local += [(ts, li, 1.0) for ts in spec.per_layer]
    if i_p == p - 1:
        local += [(ts, None, 1.0) for ts in spec.final]
        if spec.tied:
            # the head is the embedding: on a separate last stage it is a
            # copy whose gradient Megatron all-reduces with stage 0 -> w = 0
            local += [(ts, None, 0.0 if p > 1 else None) for ts in spec.embed[:1]]
        else:
            local += [(ts, None, 1.0) for ts in spec.head]
    segs, gens, names, off = [], [], [], 0
    for ts, li, w in local:
        if w is None:
            continue  # p == 1 and tied: the head is the embedding already here
        b = base[(ts.name, li)]
        shape = ts.shape
        full = math.prod(shape)
        if ts.split_axis is None:
            n = full
            gens.append((off, n, b, n, n))
            weight = w if i_t == 0 else 0.0
        else:
            ax = ts.split_axis
            if shape[ax] % t:
                raise ValueError(f"{ts.name}{shape}: axis {ax} not divisible by t={t}")
            n = full // t
            if ax == 0:
                rows = shape[0] // t
                inner = full // shape[0]
                gens.append((off, n, b + i_t * rows * inner, n, n))
            else:
                cols = shape[1] // t
                gens.append((off, n, b + i_t * cols, cols, shape[1]))
            weight = w
        segs.append((off, n, weight))
        names.append(f"{ts.name}" + (f".{li}" if li is not None else ""))
        off += n
    return RankLayout(rank, (i_d, i_t, i_p), off, segs, gens, names)


def world_layouts(spec: ModelSpec, d: int, t: int, p: int) -> list:
    return [rank_layout(spec, d, t, p, r) for r in range(d * t * p)]


def algorithmic_bytes(spec: ModelSpec, d: int, t: int, p: int, M: int, esize: int, fused: bool) -> int:
    """Bytes one GNS step must read: every rank's counted shard
    once per micro-batch, plus one read of the synchronised mean gradient
    (each DP replica its 1/d slice) when d > 1; 0 extra when fused (d == 1)."""
    lay = world_layouts(spec, d, t, p)
    micro = sum(l.counted for l in lay) * M * esize
    # mean read: each model-parallel shard read once per box (d slices)
    mean = 0 if (fused and d == 1) else sum(l.counted for l in lay if l.coords[0] == 0) * esize
    return micro + mean


# ---------------------------------------------------------------- native twin

_STAGE = {"embed": 0, "layer": 1, "final": 2, "head": 3}


def to_native(spec: ModelSpec):
    """The spec as a coadapt_grad_model (coadapt_segments.h); returns the
    struct and the ctypes objects it points into (keep both alive)."""
    import ctypes as C
    from . import _lib as L
    ts = [t for t in spec.embed] + [t for t in spec.per_layer] + [t for t in spec.final]
    if not spec.tied:
        ts += [t for t in spec.head]
    arr = (L.GradTensorC * max(1, len(ts)))()
    names = []
    for i, t in enumerate(ts):
        nm = C.c_char_p(t.name.encode())
        names.append(nm)
        arr[i].name = nm.value
        arr[i].stage = _STAGE[t.stage]
        arr[i].ndim = len(t.shape)
        arr[i].tp_axis = -1 if t.split_axis is None else int(t.split_axis)
        for a, n in enumerate(t.shape):
            arr[i].shape[a] = int(n)
    nm = spec.name.encode()
    m = L.GradModelC(nm, spec.layers, 1 if spec.tied else 0, arr, len(ts))
    return m, (arr, names, nm)


def native_rank_layout(spec: ModelSpec, d: int, t: int, p: int, rank: int) -> RankLayout:
    """rank_layout() computed by the library's C++ generator
    (coadapt::gns_segments through coadapt_gns_segments)."""
    import ctypes as C
    from . import _lib as L
    m, keep = to_native(spec)
    cnt, numel, coords = C.c_size_t(0), C.c_uint64(0), (C.c_int32 * 3)()
    L.check(L.lib().coadapt_gns_segments(C.byref(m), d, t, p, rank, None, None, 0, C.byref(cnt),
                                         C.byref(numel), coords))
    n = cnt.value
    segs, gens = (L.SegmentC * max(1, n))(), (L.GenSegmentC * max(1, n))()
    L.check(L.lib().coadapt_gns_segments(C.byref(m), d, t, p, rank, segs, gens, n, C.byref(cnt),
                                         C.byref(numel), coords))
    del keep
    return RankLayout(rank, (coords[0], coords[1], coords[2]), numel.value,
                      [(s.offset, s.numel, s.weight) for s in segs[:n]],
                      [(g.local_off, g.numel, g.global_base, g.row_len, g.row_stride) for g in gens[:n]],
                      [])
