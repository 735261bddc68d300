"""Finalize in the same pass (north_star item 2; Alg. 1):
coadapt_gns_fused_sqnorm_finalize / coadapt_gns_mean_sqnorm_finalize run
finalize_step + update_ema + gns in the last CTA of the step's last
reduction.  Every result must be bit-identical to the separate
reduction -> finalize launches, on the TMA path, on the LDG fallback
(unaligned views: the tail then runs as its own launch), for an all-weight-0
plan (no chunks at all), under CUDA-graph capture, and over several steps so
the EMA state is exercised."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _env():
    from paper_2604_26687_b200 import _lib as L
    from paper_2604_26687_b200 import device as D
    from paper_2604_26687_b200 import layout as Lay
    torch.cuda.set_device(0)
    return L, D, Lay


def _same(a, b):
    ra, rb = a.result(), b.result()
    assert np.array_equal(a.partials(), b.partials())
    assert ra.state.as_tuple() == rb.state.as_tuple()
    assert (ra.stats.signal, ra.stats.noise, ra.stats.noise_raw, ra.stats.mean_grad_sq) == \
        (rb.stats.signal, rb.stats.noise, rb.stats.noise_raw, rb.stats.mean_grad_sq)
    assert np.array_equal(np.array([ra.phi, ra.b_simple]), np.array([rb.phi, rb.b_simple]),
                          equal_nan=True)  # phi is NaN while unavailable
    assert (ra.phi_available, ra.status) == (rb.phi_available, rb.status)
    return ra


@pytest.mark.parametrize("offset", [0, 1])  # 1: unaligned views -> LDG + separate tail
def test_fused_with_finalize_equals_separate(offset):
    L, D, Lay = _env()
    spec = Lay.tiny_model(layers=4, h=256, ffn=512, vocab=1000)
    lays = Lay.world_layouts(spec, 1, 2, 2)  # 4 virtual ranks -> 4 launches per step
    M = 6
    cap = max(l.numel for l in lays) + 8
    raw = [torch.empty(cap, dtype=torch.bfloat16, device="cuda") for _ in range(M)]
    plans = [D.BucketPlan(l.segments, l.numel, L.BF16, 0) for l in lays]
    a, b = D.GnsDevice(1, M, 2 * M, 0), D.GnsDevice(1, M, 2 * M, 0)
    unit = Lay.noise_unit_for(256.0, 2)
    for step in range(3):
        a.begin_step()
        b.begin_step()
        for r, (lay, plan) in enumerate(zip(lays, plans)):
            views = [x[offset:offset + lay.numel] for x in raw]
            for m in range(M):
                D.synth_fill(views[m], lay.gen, 90 + step, m, Lay.G0, unit)
            a.fused_sqnorm(plan, views)
            if r + 1 < len(lays):
                b.fused_sqnorm(plan, views)
            else:
                b.fused_sqnorm_finalize(plan, views, 2 * M * 2048)
        a.finalize(2 * M * 2048)
        r = _same(a, b)
    assert r.state.tokens_seen == 3 * 2 * M * 2048 and r.phi_available


def test_mean_slice_with_finalize_equals_separate_d2():
    L, D, Lay = _env()
    spec = Lay.tiny_model(layers=4, h=256, ffn=512, vocab=1000)
    d, M = 2, 3
    lays = Lay.world_layouts(spec, d, 2, 1)
    cap = max(l.numel for l in lays)
    bufs = [torch.empty(cap, dtype=torch.bfloat16, device="cuda") for _ in range(M)]
    mean = torch.empty(cap, dtype=torch.bfloat16, device="cuda")
    unit = Lay.noise_unit_for(64.0, 1)
    a, b = D.GnsDevice(d, M, d * M, 0), D.GnsDevice(d, M, d * M, 0)
    a.begin_step()
    b.begin_step()
    for r, lay in enumerate(lays):
        i_d = lay.coords[0]
        plan = D.BucketPlan(lay.segments, lay.numel, L.BF16, 0)
        sl = D.BucketPlan(lay.segments, lay.numel, L.BF16, 0, slice_index=i_d, slice_count=d)
        views = [x[:lay.numel] for x in bufs]
        for m in range(M):
            D.synth_fill(views[m], lay.gen, 7, i_d * M + m, Lay.G0, unit)
        D.synth_mean_fill(mean[:lay.numel], lay.gen, 7, 0, d * M, Lay.G0, unit)
        for g in (a, b):
            g.micro_sqnorm_batched(plan, views, [i_d] * M, list(range(M)))
        a.mean_sqnorm(sl, mean[:lay.numel])
        if r + 1 < len(lays):
            b.mean_sqnorm(sl, mean[:lay.numel])
        else:
            b.mean_sqnorm_finalize(sl, mean[:lay.numel], d * M * 2048)
        torch.cuda.synchronize()
    a.finalize(d * M * 2048)
    _same(a, b)


def test_all_weight_zero_plan_still_finalizes():
    L, D, Lay = _env()
    n, M = 4096, 2
    plan = D.BucketPlan([(0, n, 0.0)], n, L.BF16, 0)  # nothing counted: no chunks
    bufs = [torch.ones(n, dtype=torch.bfloat16, device="cuda") for _ in range(M)]
    a, b = D.GnsDevice(1, M, M, 0), D.GnsDevice(1, M, M, 0)
    for g in (a, b):
        g.begin_step()
    a.fused_sqnorm(plan, bufs)
    a.finalize(M * 2048)
    b.fused_sqnorm_finalize(plan, bufs, M * 2048)
    r = _same(a, b)
    assert r.stats.signal == 0.0 and r.stats.noise == 0.0


def test_inpass_finalize_under_graph_capture():
    L, D, Lay = _env()
    spec = Lay.tiny_model(layers=4, h=256, ffn=512, vocab=1000)
    lay = Lay.rank_layout(spec, 1, 2, 2, 3)
    M = 4
    bufs = [torch.empty(lay.numel, dtype=torch.bfloat16, device="cuda") for _ in range(M)]
    plan = D.BucketPlan(lay.segments, lay.numel, L.BF16, 0)
    graphed, eager = D.GnsDevice(1, M, M, 0), D.GnsDevice(1, M, M, 0)
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        graphed.begin_step(s)
        graphed.fused_sqnorm_finalize(plan, bufs, M * 2048, s)
    unit = Lay.noise_unit_for(256.0, 1)
    for step in range(3):
        with torch.cuda.stream(s):
            for m in range(M):
                D.synth_fill(bufs[m], lay.gen, 300 + step, m, Lay.G0, unit, s)
            graph.replay()
        graphed.result()
        eager.begin_step(s)
        eager.fused_sqnorm(plan, bufs, s)
        eager.finalize(M * 2048, s)
        _same(graphed, eager)


def test_inpass_finalize_rejects_nccl_without_mailboxes():
    L, D, Lay = _env()
    g = D.GnsDevice(1, 2, 2, 0)
    # a gns attached to a one-rank communicator is fine (local finalize) ...
    g.attach_nccl(1, 0, D.nccl_unique_id())
    n = 1024
    plan = D.BucketPlan([(0, n, 1.0)], n, L.BF16, 0)
    bufs = [torch.ones(n, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    g.begin_step()
    g.fused_sqnorm_finalize(plan, bufs, 2 * 2048)
    assert g.result().status == 0
    with pytest.raises(L.ValidationError):
        g.fused_sqnorm_finalize(plan, bufs, -1)
