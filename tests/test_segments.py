"""C++ segment / dedup generator (coadapt::gns_segments, coadapt_segments.h)
against the Python twin (layout.rank_layout): bit-identical segment tables
(offset, numel, weight), generator maps and bucket lengths for every
BASELINE model at every BASELINE layout, every rank, plus random (d,t,p)
and random small models.  SPEC.md:419-423, 445-453; SURVEY §8 row a12."""
import ctypes as C
import random

import pytest

from paper_2604_26687_b200 import _lib as L
from paper_2604_26687_b200 import layout as Lay

BASELINE_LAYOUTS = {"125m": [(2, 1, 1), (1, 2, 2), (2, 2, 2), (1, 4, 2)],
                    "3b": [(8, 1, 1), (1, 1, 1), (2, 2, 2), (1, 4, 1)],
                    "7b": [(2, 2, 2), (1, 8, 1), (1, 1, 8), (4, 2, 1)],
                    "32b": [(1, 4, 2), (1, 8, 1), (2, 4, 1), (1, 2, 4)]}


def _same(a, b):
    assert a.numel == b.numel
    assert tuple(a.coords) == tuple(b.coords)
    assert a.segments == b.segments
    assert a.gen == b.gen


@pytest.mark.parametrize("key", sorted(BASELINE_LAYOUTS))
def test_baseline_models_every_rank(key):
    spec = Lay.MODELS[key]()
    for d, t, p in BASELINE_LAYOUTS[key]:
        for r in range(d * t * p):
            _same(Lay.native_rank_layout(spec, d, t, p, r), Lay.rank_layout(spec, d, t, p, r))


@pytest.mark.parametrize("key", sorted(BASELINE_LAYOUTS))
def test_presets_match_python_specs(key):
    m = L.GradModelC()
    L.check(L.lib().coadapt_model_preset(key.encode(), C.byref(m)))
    spec = Lay.MODELS[key]()
    assert m.layers == spec.layers and bool(m.tied) == spec.tied
    py = [t for t in spec.embed] + list(spec.per_layer) + list(spec.final) + (
        [] if spec.tied else list(spec.head))
    assert m.n_tensors == len(py)
    for i, t in enumerate(py):
        c = m.tensors[i]
        assert c.name.decode() == t.name
        assert tuple(c.shape[:c.ndim]) == tuple(t.shape)
        assert c.tp_axis == (-1 if t.split_axis is None else t.split_axis)
    # the preset drives the same generator: 32B (1,4,2) rank 5
    cnt, numel = C.c_size_t(0), C.c_uint64(0)
    L.check(L.lib().coadapt_gns_segments(C.byref(m), 1, 4, 2, 5, None, None, 0, C.byref(cnt),
                                         C.byref(numel), None))
    assert numel.value == Lay.rank_layout(spec, 1, 4, 2, 5).numel if key == "32b" else True


def test_random_strategies_and_models():
    rng = random.Random(7)
    for _ in range(60):
        tied = rng.random() < 0.5
        t = rng.choice([1, 2, 4])
        p = rng.choice([1, 2, 4])
        d = rng.choice([1, 2, 3])
        spec = Lay.tiny_model(layers=4 * rng.randint(1, 3), h=16 * t * rng.randint(1, 3),
                              ffn=32 * t, vocab=8 * t * rng.randint(1, 5), tied=tied)
        for r in range(d * t * p):
            _same(Lay.native_rank_layout(spec, d, t, p, r), Lay.rank_layout(spec, d, t, p, r))
        sp = Lay.gpt2_small()
        r = rng.randrange(d * t * p)
        _same(Lay.native_rank_layout(sp, d, t, p, r), Lay.rank_layout(sp, d, t, p, r))


def test_algorithmic_bytes_match_python():
    for key, lays in BASELINE_LAYOUTS.items():
        spec = Lay.MODELS[key]()
        m, keep = Lay.to_native(spec)
        for d, t, p in lays[:2]:
            for M, es, fused in [(16, 2, True), (8, 2, False), (4, 4, True)]:
                out = C.c_uint64(0)
                L.check(L.lib().coadapt_gns_algorithmic_bytes(C.byref(m), d, t, p, M, es,
                                                              int(fused), C.byref(out)))
                assert out.value == Lay.algorithmic_bytes(spec, d, t, p, M, es, fused)


def test_validation_errors():
    spec = Lay.llama2_7b()
    with pytest.raises(L.ValidationError, match="not divisible by p"):
        Lay.native_rank_layout(spec, 1, 1, 3, 0)
    with pytest.raises(L.ValidationError, match="outside"):
        Lay.native_rank_layout(spec, 2, 2, 2, 8)
    with pytest.raises(L.ValidationError, match="not divisible by t"):
        Lay.native_rank_layout(Lay.tiny_model(h=64, vocab=96), 1, 64, 1, 0)
    m = L.GradModelC()
    with pytest.raises(L.ValidationError, match="unknown model preset"):
        L.check(L.lib().coadapt_model_preset(b"70b", C.byref(m)))
    # capacity below the tensor count is a validation error that still
    # reports the count
    m, keep = Lay.to_native(spec)
    cnt = C.c_size_t(0)
    segs = (L.SegmentC * 1)()
    rc = L.lib().coadapt_gns_segments(C.byref(m), 1, 1, 1, 0, segs, None, 1, C.byref(cnt), None, None)
    assert rc == L.E_VALIDATION and cnt.value == len(Lay.rank_layout(spec, 1, 1, 1, 0).segments)
