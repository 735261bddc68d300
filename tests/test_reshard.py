"""Reshard planning — CPU tests.

The product planner (coadapt::reshard via include/coadapt_reshard.h) is
checked against SPEC.md's worked examples and, on randomized model specs and
strategy pairs, move-for-move against the oracle restatement
(oracle/reshard_oracle.py).  The oracle itself is pinned on the same SPEC
examples and on the direct global-tensor check (content conservation and
A->B->A round trips, any move order).  Device execution is tests/
test_gpu_reshard.py.
"""
import itertools
import math
import random

import numpy as np
import pytest

from oracle import reshard_oracle as O
from paper_2604_26687_b200 import _lib as L
from paper_2604_26687_b200 import reshard as R


def to_oracle(m: R.ModelSpec) -> O.Model:
    return O.Model(m.layers, [O.Tensor(t.name, tuple(t.shape), t.tp_axis) for t in m.per_layer],
                   m.optimizer_state_multiplier, m.param_bytes, m.state_bytes)


def strategies(n: int, layers: int):
    return [(d, t, p) for d in range(1, n + 1) for t in range(1, n + 1) for p in range(1, n + 1)
            if d * t * p == n and layers % p == 0]


def random_model(rng: random.Random, t_max: int = 8) -> R.ModelSpec:
    tensors = []
    for i in range(rng.randint(1, 4)):
        nd = rng.choice([1, 1, 2, 2, 2, 3])
        shape = [rng.choice([1, 3, 8, 16, 24, 40, 64]) for _ in range(nd)]
        ax = rng.randint(-1, nd - 1)
        if ax >= 0:
            shape[ax] = t_max * rng.randint(1, 8)
        tensors.append(R.TensorDecl(f"t{i}", tuple(shape), ax))
    return R.ModelSpec(rng.choice([2, 4, 8]), tuple(tensors), rng.randint(0, 2))


def as_tuple(m):
    return (m.src_rank, m.dst_rank, m.layer, m.tensor, tuple(m.offset), tuple(m.extent), m.bytes,
            bool(m.local))


# ------------------------------------------------------------ SPEC examples

TOY = R.ModelSpec(2, (R.TensorDecl("w", (8,), 0),))


def test_spec_examples_layout():
    """SPEC.md:451-453."""
    sh = R.layout_for(TOY, (1, 2, 1))
    assert [(s.layer, s.owner, s.global_offset, s.local_shape) for s in sh] == [
        (0, 0, (0,), (4,)), (1, 0, (0,), (4,)), (0, 1, (4,), (4,)), (1, 1, (4,), (4,))]
    sh = R.layout_for(TOY, (1, 1, 2))
    assert [(s.layer, s.owner, s.local_shape) for s in sh] == [(0, 0, (8,)), (1, 1, (8,))]
    sh = R.layout_for(TOY, (2, 1, 1))  # d=2 replicates; replica 0 canonical
    assert [(s.owner, s.canonical) for s in sh] == [(0, True), (0, True), (1, False), (1, False)]
    o = O.layout_for(to_oracle(TOY), (2, 1, 1))
    assert o.replica_groups == [[0], [1]]


def test_spec_examples_plan():
    """SPEC.md:459-462."""
    one = R.ModelSpec(1, (R.TensorDecl("w", (8,), 0),))
    p = R.plan_transfers(one, (1, 2, 1), (1, 4, 1))
    mv = p.moves()
    assert len(mv) == 4
    src = {s.owner: s for s in R.layout_for(one, (1, 2, 1))}
    for m in mv:  # each fully contained in one source shard
        s = src[m.src_rank]
        assert s.global_offset[0] <= m.offset[0] and m.offset[0] + m.extent[0] <= s.global_offset[0] + 4
    p = R.plan_transfers(one, (1, 4, 1), (1, 2, 1))
    per_dst = {}
    for m in p.moves():
        per_dst.setdefault(m.dst_rank, []).append(m)
    assert sorted(len(v) for v in per_dst.values()) == [2, 2]
    for a in [(1, 2, 1), (2, 2, 1), (1, 1, 2), (2, 1, 1)]:
        m2 = R.ModelSpec(2, (R.TensorDecl("w", (8, 4), 0), R.TensorDecl("n", (4,), -1)))
        p = R.plan_transfers(m2, a, a)
        assert p.total_bytes == 0 and all(m.local for m in p.moves())


def test_oracle_spec_examples():
    one = O.Model(1, [O.Tensor("w", (8,), 0)])
    mv, tot, _, _ = O.plan_transfers(one, O.layout_for(one, (1, 2, 1)), O.layout_for(one, (1, 4, 1)))
    assert len(mv) == 4 and [m.offset[0] for m in mv] == [0, 2, 4, 6]
    mv, _, _, _ = O.plan_transfers(one, O.layout_for(one, (1, 4, 1)), O.layout_for(one, (1, 2, 1)))
    assert [m.dst_rank for m in mv] == [0, 0, 1, 1]
    lay = O.layout_for(one, (2, 2, 1))
    mv, tot, _, _ = O.plan_transfers(one, lay, lay)
    assert tot == 0 and all(m.local for m in mv)


# --------------------------------------------------- product vs oracle


@pytest.mark.parametrize("seed", range(6))
def test_plan_matches_oracle_random(seed):
    rng = random.Random(seed)
    for _ in range(40):
        m = random_model(rng)
        n = rng.choice([1, 2, 4, 8])
        ss = strategies(n, m.layers)
        a = rng.choice(ss)
        b = rng.choice(strategies(rng.choice([1, 2, 4, 8]), m.layers))
        policy = rng.choice(["canonical", "spread"])
        p = R.plan_transfers(m, a, b, policy)
        om = to_oracle(m)
        la, lb = O.layout_for(om, a), O.layout_for(om, b)
        mv, tot, mx, loc = O.plan_transfers(om, la, lb, policy)
        assert [as_tuple(x) for x in p.moves()] == [as_tuple(x) for x in mv]
        assert (p.total_bytes, p.max_bytes_per_rank, p.local_bytes) == (tot, mx, loc)
        assert [p.pack_numel(R.SRC, r) for r in range(math.prod(a))] == la.pack_numel
        assert [(s.owner, s.pack_offset, s.global_offset, s.local_shape, s.canonical)
                for s in p.shards(R.DST)] == [(s.owner, s.pack_offset, s.global_offset, s.local_shape,
                                               s.canonical) for s in lb.shards]
        assert p.csv() == O.plan_csv(om, mv)


def test_tiling_and_plan_completeness():
    """canonical shards tile each tensor; every destination
    element is written exactly once."""
    rng = random.Random(11)
    for _ in range(60):
        m = to_oracle(random_model(rng))
        a = rng.choice(strategies(8, m.layers))
        b = rng.choice(strategies(4, m.layers))
        la, lb = O.layout_for(m, a), O.layout_for(m, b)
        for lay in (la, lb):
            for rep in range(lay.dtp[0]):
                for layer in range(m.layers):
                    for ti, ts in enumerate(m.per_layer):
                        paint = np.zeros(ts.shape, np.int32)
                        for s in lay.shards:
                            if (s.layer, s.tensor) != (layer, ti):
                                continue
                            i_d, i_t, _ = O.coords(s.owner, lay.dtp)
                            if i_d == rep and (ts.tp_axis >= 0 or i_t == 0):
                                paint[O._box(s)] += 1
                        assert (paint == 1).all()
        mv, _, _, _ = O.plan_transfers(m, la, lb)
        hits = {di: np.zeros(s.local_shape, np.int32) for di, s in enumerate(lb.shards)}
        for x in mv:
            D = lb.shards[x.dst_shard]
            hits[x.dst_shard][tuple(slice(o - g, o - g + e) for o, g, e in
                                    zip(x.offset, D.global_offset, x.extent))] += 1
        assert all((h == 1).all() for h in hits.values())


@pytest.mark.parametrize("dtype", [np.float32, np.uint16])
def test_oracle_conservation_round_trip_any_order(dtype):
    """A->B gives the global tensors' regions; A->B->A is
    the identity; moves apply in any order."""
    rng = random.Random(5)
    for trial in range(40):
        m = to_oracle(random_model(rng))
        a = rng.choice(strategies(rng.choice([2, 4, 8]), m.layers))
        b = rng.choice(strategies(rng.choice([1, 2, 4, 8]), m.layers))
        la, lb = O.layout_for(m, a), O.layout_for(m, b)
        st = O.global_state(m, trial, dtype)
        src = [O.pack_from_global(la, r, st, dtype) for r in range(len(la.pack_numel))]
        mv, _, _, _ = O.plan_transfers(m, la, lb)
        order = list(range(len(mv)))
        rng.shuffle(order)
        out, peak = O.execute_in_memory(m, la, lb, mv, src, dtype, order=order)
        for r in range(len(lb.pack_numel)):
            assert np.array_equal(out[r], O.pack_from_global(lb, r, st, dtype))
        es = np.dtype(dtype).itemsize
        # a pull holds both layouts plus the piece in flight (the SPEC's
        # max(src, dst) + staging bound needs a staged schedule; see DESIGN)
        stage = max((math.prod(x.extent) for x in mv), default=0) * es
        assert peak <= (max(la.pack_numel) + max(lb.pack_numel)) * es + stage
        back, _, _, _ = O.plan_transfers(m, lb, la)
        again, _ = O.execute_in_memory(m, lb, la, back, out, dtype)
        for r in range(len(la.pack_numel)):
            assert np.array_equal(again[r], src[r])


def test_spread_policy_same_bytes_more_sources():
    m = R.ModelSpec(4, (R.TensorDecl("w", (64, 32), 0), R.TensorDecl("n", (32,), -1)))
    c = R.plan_transfers(m, (2, 1, 1), (4, 1, 1), "canonical")
    s = R.plan_transfers(m, (2, 1, 1), (4, 1, 1), "spread")
    assert c.total_bytes == s.total_bytes > 0
    assert {x.src_rank for x in c.moves() if not x.local} == {0}
    assert {x.src_rank for x in s.moves() if not x.local} == {0, 1}


# ------------------------------------------------------------- latency, csv


def llama3b_like() -> R.ModelSpec:
    T = R.TensorDecl
    return R.ModelSpec(28, (T("q", (3072, 3072), 0), T("k", (1024, 3072), 0), T("v", (1024, 3072), 0),
                            T("o", (3072, 3072), 1), T("gate", (8192, 3072), 0),
                            T("up", (8192, 3072), 0), T("down", (3072, 8192), 1),
                            T("norm1", (3072,)), T("norm2", (3072,))))


def test_latency_model():
    """SPEC.md:475-483."""
    m = llama3b_like()
    same = R.plan_transfers(m, (2, 2, 2), (2, 2, 2))
    assert same.total_bytes == 0 and same.latency(1e9, 20.0) == 20.0
    p = R.plan_transfers(m, (1, 2, 4), (1, 4, 2))
    t1 = p.latency(1e9, 20.0) - 20.0
    t2 = p.latency(2e9, 20.0) - 20.0
    assert t2 == pytest.approx(t1 / 2, rel=1e-15)
    assert p.latency(1e9, 20.0) == O.estimate_reconfig_latency(p.total_bytes, 1e9, 20.0)
    # defaults put 3B-scale transitions in the paper's 30-56 s band
    for a, b in [((1, 2, 4), (1, 4, 2)), ((2, 2, 2), (1, 4, 2)), ((1, 8, 1), (1, 4, 2)),
                 ((2, 1, 4), (2, 2, 2))]:
        assert 30.0 <= R.estimate_reconfig_latency(R.plan_transfers(m, a, b)) <= 60.0
    # monotone in wire bytes
    plans = [R.plan_transfers(m, (2, 2, 2), b) for b in strategies(8, 28)]
    for x, y in itertools.combinations(plans, 2):
        if x.total_bytes <= y.total_bytes:
            assert x.latency() <= y.latency()
    with pytest.raises(L.ValidationError):
        p.latency(0.0, 1.0)


def test_csv_header_and_rows():
    p = R.plan_transfers(R.ModelSpec(1, (R.TensorDecl("w", (4, 8), 1),)), (1, 1, 1), (1, 2, 1))
    lines = p.csv().splitlines()
    assert lines[0] == "key,src_rank,dst_rank,offsets,extents,bytes,local"
    assert lines[1:] == ["layer0.w,0,0,0;0,4;4,160,1", "layer0.w,0,1,0;4,4;4,160,0"]


def test_validation():
    with pytest.raises(L.ValidationError):
        R.plan_transfers(R.ModelSpec(3, (R.TensorDecl("w", (8,), 0),)), (1, 1, 2), (1, 1, 1))
    with pytest.raises(L.ValidationError):
        R.plan_transfers(R.ModelSpec(2, (R.TensorDecl("w", (6,), 0),)), (1, 4, 1), (1, 1, 1))
    with pytest.raises(L.ValidationError):
        R.plan_transfers(R.ModelSpec(2, (R.TensorDecl("w", (6,), 3),)), (1, 1, 1), (1, 1, 1))
    with pytest.raises(L.ValidationError):
        R.plan_transfers(R.ModelSpec(2, (R.TensorDecl("w", (0,), -1),)), (1, 1, 1), (1, 1, 1))
    with pytest.raises(L.ValidationError):
        R.plan_transfers(TOY, (0, 1, 1), (1, 1, 1))
    with pytest.raises(L.ValidationError):
        R.plan_transfers(TOY, "d2x", (1, 1, 1))
