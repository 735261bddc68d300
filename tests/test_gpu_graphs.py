"""The whole device step is CUDA-graph capturable: begin_step,
the fused pass (TMA kernel), the (no-op on one GPU) all-reduce, finalize and
the pinned D2H of the result are recorded once and replayed; results equal
the eager step bit for bit, and the EMA advances once per replay."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_capture_and_replay_gns_step():
    from paper_2604_26687_b200 import _lib as L
    from paper_2604_26687_b200 import device as D
    from paper_2604_26687_b200 import layout as Lay
    torch.cuda.set_device(0)
    spec = Lay.tiny_model(layers=4, h=256, ffn=512, vocab=1000)
    lay = Lay.rank_layout(spec, 1, 2, 2, 1)
    M = 4
    bufs = []
    for m in range(M):
        b = torch.empty(lay.numel, dtype=torch.bfloat16, device="cuda")
        D.synth_fill(b, lay.gen, 3, m, Lay.G0, Lay.noise_unit_for(256.0, 1))
        bufs.append(b)
    plan = D.BucketPlan(lay.segments, lay.numel, L.BF16, 0)
    eager = D.GnsDevice(1, M, M, 0)
    graphed = D.GnsDevice(1, M, M, 0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        # warm-up outside capture: builds the plan's chunk table, opts the
        # kernel into large shared memory
        graphed.begin_step(s)
        graphed.fused_sqnorm(plan, bufs, s)
        graphed.finalize(M * 2048, s)
    s.synchronize()
    from paper_2604_26687_b200._lib import GnsState
    graphed.set_state(GnsState.default())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        graphed.begin_step(s)
        graphed.fused_sqnorm(plan, bufs, s)
        graphed.allreduce(s)
        graphed.finalize(M * 2048, s)
    for step in range(3):
        graph.replay()
        rg = graphed.result()
        eager.begin_step()
        eager.fused_sqnorm(plan, bufs)
        eager.finalize(M * 2048)
        re = eager.result()
        assert np.array_equal(graphed.partials(), eager.partials())
        assert rg.state.as_tuple() == re.state.as_tuple()
        assert (rg.phi, rg.b_simple) == (re.phi, re.b_simple)
    assert rg.state.tokens_seen == 3 * M * 2048


def test_capture_without_warmup_every_launch_shape():
    """plans build every device table at creation, so a d > 1
    step (batched K1 on the TMA ring, the K2 mean slice) and a d = 1 fused
    step can be captured with no eager call before; replays equal eager."""
    from paper_2604_26687_b200 import _lib as L
    from paper_2604_26687_b200 import device as D
    from paper_2604_26687_b200 import layout as Lay
    torch.cuda.set_device(0)
    spec = Lay.tiny_model(layers=4, h=256, ffn=512, vocab=1000)
    lay = Lay.rank_layout(spec, 2, 2, 1, 1)
    unit = Lay.noise_unit_for(256.0, 1)
    for d, M in ((2, 3), (1, 5)):
        bufs = [torch.empty(lay.numel, dtype=torch.bfloat16, device="cuda") for _ in range(M)]
        mean = torch.empty(lay.numel, dtype=torch.bfloat16, device="cuda")
        plan = D.BucketPlan(lay.segments, lay.numel, L.BF16, 0)
        sl = D.BucketPlan(lay.segments, lay.numel, L.BF16, 0, slice_index=d - 1, slice_count=d)
        graphed, eager = D.GnsDevice(d, M, d * M, 0), D.GnsDevice(d, M, d * M, 0)
        s = torch.cuda.Stream()

        def body(g, stream):
            g.begin_step(stream)
            if d == 1:
                g.fused_sqnorm(plan, bufs, stream)
            else:
                for i_d in range(d):
                    g.micro_sqnorm_batched(plan, bufs, [i_d] * M, list(range(M)), stream)
                g.mean_sqnorm(sl, mean, stream)
            g.allreduce(stream)
            g.finalize(d * M * 2048, stream)

        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            body(graphed, s)
        for step in range(3):
            with torch.cuda.stream(s):
                for m in range(M):
                    D.synth_fill(bufs[m], lay.gen, 40 + step, m, Lay.G0, unit, s)
                D.synth_mean_fill(mean, lay.gen, 40 + step, 0, M, Lay.G0, unit, s)
                graph.replay()
            rg = graphed.result()
            body(eager, s)
            re = eager.result()
            assert np.array_equal(graphed.partials(), eager.partials())
            assert rg.state.as_tuple() == re.state.as_tuple()
