"""CPU oracle for the reshard module — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's reference leg may import
this.  It restates SPEC.md's reshard module in plain
Python/numpy so the product (coadapt::reshard planner + the device executor
in csrc/reshard.cu) can be checked against it:

* layout_for        SPEC.md:445-453 (contiguous PP stages, equal TP split,
                    DP replication) + the choices documented in
                    include/coadapt/reshard.hpp (Megatron rank order,
                    TP-replicated tensors, 64-element pack alignment);
* plan_transfers    SPEC.md:455-463 (per-axis interval intersection against
                    the canonical source copies; pieces already on the
                    destination rank are local);
* execute_in_memory SPEC.md:465-473 (moves applied in any order, memory
                    accounting of source-resident + staged + target-resident
                    bytes);
* estimate_reconfig_latency SPEC.md:475-483; plan CSV SPEC.md:501.

Parity pinning: the reference ships no code or vectors for this module
(SPEC only), so the oracle is pinned on SPEC.md's worked examples
(tests/test_reshard.py::test_spec_examples_*) and on the direct
global-tensor check SPEC.md:472 names (every destination element equals the
global tensor at that index).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

PACK_ALIGN = 64


@dataclass
class Tensor:
    name: str
    shape: tuple
    tp_axis: int = -1


@dataclass
class Model:
    layers: int
    per_layer: list
    optimizer_state_multiplier: int = 2
    param_bytes: int = 2
    state_bytes: int = 4

    @property
    def bytes_per_element(self) -> int:
        return self.param_bytes + self.optimizer_state_multiplier * self.state_bytes

    def key(self, layer: int, tensor: int) -> str:
        return f"layer{layer}.{self.per_layer[tensor].name}"


@dataclass
class Shard:
    layer: int
    tensor: int
    owner: int
    canonical: bool
    global_shape: tuple
    global_offset: tuple
    local_shape: tuple
    pack_offset: int

    @property
    def numel(self) -> int:
        return math.prod(self.local_shape)


@dataclass
class Layout:
    dtp: tuple
    shards: list
    replica_groups: list
    pack_numel: list = field(default_factory=list)


@dataclass
class Move:
    src_rank: int
    dst_rank: int
    layer: int
    tensor: int
    offset: tuple
    extent: tuple
    bytes: int
    local: bool
    src_shard: int
    dst_shard: int


def coords(rank: int, dtp: tuple) -> tuple:
    """(i_d, i_t, i_p), tp fastest then dp then pp."""
    d, t, p = dtp
    return (rank // t) % d, rank % t, rank // (t * d)


def layout_for(model: Model, dtp: tuple) -> Layout:
    d, t, p = dtp
    if min(dtp) < 1:
        raise ValueError("degrees must be >= 1")
    if model.layers % p:
        raise ValueError("layers not divisible by p")
    for ts in model.per_layer:
        if ts.tp_axis >= 0 and ts.shape[ts.tp_axis] % t:
            raise ValueError(f"{ts.name}: axis not divisible by t")
    n = d * t * p
    shards, groups, packs = [], [[] for _ in range(d)], []
    per_stage = model.layers // p
    for r in range(n):
        i_d, i_t, i_p = coords(r, dtp)
        groups[i_d].append(r)
        cur = 0
        for layer in range(i_p * per_stage, (i_p + 1) * per_stage):
            for ti, ts in enumerate(model.per_layer):
                off = [0] * len(ts.shape)
                loc = list(ts.shape)
                if ts.tp_axis >= 0:
                    loc[ts.tp_axis] = ts.shape[ts.tp_axis] // t
                    off[ts.tp_axis] = i_t * loc[ts.tp_axis]
                canonical = i_d == 0 and (ts.tp_axis >= 0 or i_t == 0)
                sh = Shard(layer, ti, r, canonical, tuple(ts.shape), tuple(off), tuple(loc), cur)
                cur += -(-sh.numel // PACK_ALIGN) * PACK_ALIGN
                shards.append(sh)
        packs.append(cur)
    return Layout(tuple(dtp), shards, groups, packs)


def _intersect(a: Shard, b: Shard):
    off, ext = [], []
    for i in range(len(a.global_shape)):
        lo = max(a.global_offset[i], b.global_offset[i])
        hi = min(a.global_offset[i] + a.local_shape[i], b.global_offset[i] + b.local_shape[i])
        if hi <= lo:
            return None
        off.append(lo)
        ext.append(hi - lo)
    return tuple(off), tuple(ext)


def _contains(s: Shard, off, ext) -> bool:
    return all(s.global_offset[i] <= off[i] and off[i] + ext[i] <= s.global_offset[i] + s.local_shape[i]
               for i in range(len(off)))


def plan_transfers(model: Model, src: Layout, dst: Layout, policy: str = "canonical"):
    """-> (moves, total_wire_bytes, max_wire_bytes_received_by_one_rank, local_bytes)"""
    sd_, st_, _ = src.dtp
    moves, total, local_b = [], 0, 0
    recv = [0] * math.prod(dst.dtp)
    bpe = model.bytes_per_element
    for di, D in enumerate(dst.shards):
        replica = coords(D.owner, dst.dtp)[0] % sd_ if policy == "spread" else 0
        covered = 0
        for si, S in enumerate(src.shards):
            if (S.layer, S.tensor) != (D.layer, D.tensor):
                continue
            i_d, i_t, _ = coords(S.owner, src.dtp)
            if i_d != replica or not (model.per_layer[S.tensor].tp_axis >= 0 or i_t == 0):
                continue
            box = _intersect(D, S)
            if box is None:
                continue
            off, ext = box
            pick = si
            for li, Lsh in enumerate(src.shards):
                if (Lsh.owner == D.owner and (Lsh.layer, Lsh.tensor) == (D.layer, D.tensor)
                        and _contains(Lsh, off, ext)):
                    pick = li
                    break
            n = math.prod(ext)
            src_rank = src.shards[pick].owner
            loc = src_rank == D.owner
            mv = Move(src_rank, D.owner, D.layer, D.tensor, off, ext, n * bpe, loc, pick, di)
            moves.append(mv)
            covered += n
            if loc:
                local_b += mv.bytes
            else:
                total += mv.bytes
                recv[D.owner] += mv.bytes
        if covered != D.numel:
            raise AssertionError(f"shard {model.key(D.layer, D.tensor)} on {D.owner} not covered")
    return moves, total, max(recv) if recv else 0, local_b


def estimate_reconfig_latency(total_wire_bytes: int, bandwidth: float, overhead: float) -> float:
    if not bandwidth > 0:
        raise ValueError("bandwidth must be > 0")
    return overhead + total_wire_bytes / bandwidth


def plan_csv(model: Model, moves) -> str:
    rows = ["key,src_rank,dst_rank,offsets,extents,bytes,local"]
    for m in moves:
        rows.append(f"{model.key(m.layer, m.tensor)},{m.src_rank},{m.dst_rank},"
                    f"{';'.join(map(str, m.offset))},{';'.join(map(str, m.extent))},{m.bytes},"
                    f"{1 if m.local else 0}")
    return "\n".join(rows) + "\n"


# ---------------------------------------------------------------- state


def global_state(model: Model, seed: int, dtype=np.float32) -> dict:
    """Deterministic global tensors, key -> array of the declared shape.
    Values are distinct small integers (exact in bf16 up to 256; the GPU
    tests compare raw bit patterns, so any payload works)."""
    rng = np.random.default_rng(seed)
    out = {}
    for layer in range(model.layers):
        for ti, ts in enumerate(model.per_layer):
            out[(layer, ti)] = rng.integers(0, 2 ** 15, size=ts.shape, dtype=np.int64).astype(dtype)
    return out


def _box(sh: Shard, off=None, ext=None):
    off = sh.global_offset if off is None else off
    ext = sh.local_shape if ext is None else ext
    return tuple(slice(o, o + e) for o, e in zip(off, ext))


def pack_from_global(layout: Layout, rank: int, state: dict, dtype) -> np.ndarray:
    """A rank's pack (SPEC's "state" restricted to its shards), padding 0."""
    buf = np.zeros(layout.pack_numel[rank], dtype=dtype)
    for sh in layout.shards:
        if sh.owner == rank:
            buf[sh.pack_offset:sh.pack_offset + sh.numel] = state[(sh.layer, sh.tensor)][_box(sh)].ravel()
    return buf


def execute_in_memory(model: Model, src: Layout, dst: Layout, moves, src_packs: list, dtype,
                      staging_bytes: int = 0, order=None):
    """apply moves (in `order` if given) from the source
    packs into fresh destination packs.  Returns (dst_packs, peak_bytes)
    where peak_bytes follows the SPEC accounting per rank: source-resident +
    staged + target-resident, freeing a source shard once its last move has
    been applied."""
    es = np.dtype(dtype).itemsize
    dst_packs = [np.zeros(n, dtype=dtype) for n in dst.pack_numel]
    idx = list(range(len(moves))) if order is None else list(order)
    remaining = {}
    for m in moves:
        remaining[m.src_shard] = remaining.get(m.src_shard, 0) + 1
    resident = [0] * max(len(src.pack_numel), len(dst.pack_numel))
    for sh in src.shards:
        resident[sh.owner] += sh.numel * es
    target_done = [0] * len(dst.pack_numel)
    peak = max(resident)
    for i in idx:
        m = moves[i]
        S, D = src.shards[m.src_shard], dst.shards[m.dst_shard]
        sbox = tuple(slice(o - g, o - g + e) for o, g, e in zip(m.offset, S.global_offset, m.extent))
        dbox = tuple(slice(o - g, o - g + e) for o, g, e in zip(m.offset, D.global_offset, m.extent))
        sview = src_packs[S.owner][S.pack_offset:S.pack_offset + S.numel].reshape(S.local_shape)
        dview = dst_packs[D.owner][D.pack_offset:D.pack_offset + D.numel].reshape(D.local_shape)
        dview[dbox] = sview[sbox]
        n = math.prod(m.extent) * es
        target_done[D.owner] += n
        staged = 0 if m.local else min(n, staging_bytes) if staging_bytes else n
        peak = max(peak, resident[D.owner] + target_done[D.owner] + staged)
        remaining[m.src_shard] -= 1
        if remaining[m.src_shard] == 0:
            resident[S.owner] -= S.numel * es
    return dst_packs, peak
