"""GnsManager: the GNS manager in a real PyTorch
forward-backward loop.  Parameters' .grad are views into one bf16 bucket;
after each micro-batch the B200 accumulate kernel folds the bucket into the
fp32 main_grad with s_m fused in.  Checked against plain torch: main_grad
bit-identical to Megatron's ``main_grad.add_(grad)`` in micro-batch order,
s_m and ‖ḡ‖² to fp64 torch sums, the finalized step to the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402


def _model(seed):
    torch.manual_seed(seed)
    return torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.GELU(),
                               torch.nn.Linear(512, 256)).cuda().to(torch.bfloat16)


def _data(M, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    xs = [torch.randn(8, 256, device="cuda", generator=g).to(torch.bfloat16) for _ in range(M)]
    ys = [torch.randn(8, 256, device="cuda", generator=g).to(torch.bfloat16) for _ in range(M)]
    return xs, ys


def _reference(model, xs, ys):
    params = [p for p in model.parameters()]
    grads = []
    for x, y in zip(xs, ys):
        loss = torch.nn.functional.mse_loss(model(x).float(), y.float())
        grads.append(torch.autograd.grad(loss, params))
    main = [torch.zeros_like(p, dtype=torch.float32) for p in params]
    for gm in grads:
        for a, g in zip(main, gm):
            a.add_(g)
    s = [sum(float((g.double() ** 2).sum()) for g in gm) for gm in grads]
    return grads, main, s


@pytest.mark.parametrize("hooks", [False, True])
def test_manager_d1_matches_torch(hooks):
    from paper_2604_26687_b200.trainer import GnsManager
    M = 4
    model = _model(0)
    xs, ys = _data(M, 1)
    _, main_ref, s_ref = _reference(model, xs, ys)
    mgr = GnsManager(model.parameters(), micro_count=M, global_batch=M * 8)
    if hooks:
        mgr.install_hooks()
    mgr.begin_step()
    for x, y in zip(xs, ys):
        torch.nn.functional.mse_loss(model(x).float(), y.float()).backward()
        if not hooks:
            mgr.after_backward()
    r = mgr.finish_step(tokens=M * 8 * 2048)
    # main_grad bit-identical to torch's fp32 accumulation in micro order
    for p, (o, n), a in zip(mgr.params, mgr._slots, main_ref):
        assert torch.equal(mgr.main_grad[o:o + n].view_as(a), a)
        assert not p.grad.any()  # bucket cleared for the next micro-batch
    parts = mgr.gns.partials()
    assert np.allclose(parts[:-1], s_ref, rtol=1e-12, atol=0)
    g2_ref = sum(float((a.double() ** 2).sum()) for a in main_ref) / M ** 2
    assert abs(parts[-1] - g2_ref) <= 1e-12 * g2_ref
    st = O.finalize_step(parts[:-1], parts[-1], M * 8)
    assert (r.stats.signal, r.stats.noise) == (st.signal, st.noise)
    # a second step through the same views works (views survived)
    mgr.begin_step()
    for x, y in zip(xs, ys):
        torch.nn.functional.mse_loss(model(x).float(), y.float()).backward()
        if not hooks:
            mgr.after_backward()
    mgr.finish_step(tokens=M * 8 * 2048)
    assert np.array_equal(mgr.gns.partials(), parts)
    mgr.remove_hooks()


def test_manager_d2_slots_sum_to_reference():
    """d = 2 emulated on one GPU: two managers (DP ranks), DP-summed
    main_grad handed to finish_step; their slot vectors sum to the job's."""
    from paper_2604_26687_b200.trainer import GnsManager
    M, d = 2, 2
    models = [_model(0), _model(0)]  # replicas: same weights
    data = [_data(M, 10 + r) for r in range(d)]
    refs = [_reference(models[r], *data[r]) for r in range(d)]
    mgrs = [GnsManager(models[r].parameters(), micro_count=M, global_batch=d * M * 8,
                       dp_size=d, dp_rank=r) for r in range(d)]
    for r in range(d):
        mgrs[r].begin_step()
        for x, y in zip(*data[r]):
            torch.nn.functional.mse_loss(models[r](x).float(), y.float()).backward()
            mgrs[r].after_backward()
    synced = mgrs[0].main_grad + mgrs[1].main_grad  # the DP all-reduce (sum)
    for r in range(d):
        mgrs[r].gns.allreduce()  # no communicator: local slots only
    tot = np.zeros(d * M + 1)
    for r in range(d):
        mgrs[r].finish_step(tokens=d * M * 8 * 2048, synced_main_grad=synced)
        tot += mgrs[r].gns.partials()
    s_ref = refs[0][2] + refs[1][2]
    assert np.allclose(tot[:-1], s_ref, rtol=1e-12, atol=0)
    g2_ref = float((synced.double() ** 2).sum()) / (d * M) ** 2
    assert abs(tot[-1] - g2_ref) <= 1e-12 * g2_ref


def test_manager_d2_nvlink_allreduce_form():
    """d = 2 emulated on one GPU through the all-reduce form: each manager
    all-reduces its slice of both replicas' main_grad in place (local
    pointers stand in for the CUDA-IPC peers); afterwards both main_grads
    equal the DP mean bit for bit and the slots sum to the job's values."""
    from paper_2604_26687_b200.trainer import GnsManager
    M, d = 2, 2
    models = [_model(0), _model(0)]
    data = [_data(M, 20 + r) for r in range(d)]
    refs = [_reference(models[r], *data[r]) for r in range(d)]
    mgrs = [GnsManager(models[r].parameters(), micro_count=M, global_batch=d * M * 8,
                       dp_size=d, dp_rank=r) for r in range(d)]
    for r in range(d):
        mgrs[r].begin_step()
        for x, y in zip(*data[r]):
            torch.nn.functional.mse_loss(models[r](x).float(), y.float()).backward()
            mgrs[r].after_backward()
    mean_ref = (mgrs[0].main_grad + mgrs[1].main_grad) * 0.5  # fp32, replica order
    reps = [mgrs[0].main_grad, mgrs[1].main_grad]
    tot = np.zeros(d * M + 1)
    for r in range(d):
        mgrs[r].finish_step(tokens=d * M * 8 * 2048, replicas=reps)
        tot += mgrs[r].gns.partials()
    torch.cuda.synchronize()
    assert torch.equal(mgrs[0].main_grad, mean_ref) and torch.equal(mgrs[1].main_grad, mean_ref)
    s_ref = refs[0][2] + refs[1][2]
    assert np.allclose(tot[:-1], s_ref, rtol=1e-12, atol=0)
    g2_ref = float((mean_ref.double() ** 2).sum()) / M ** 2
    assert abs(tot[-1] - g2_ref) <= 1e-12 * g2_ref


def test_finish_step_without_host_sync():
    """finish_step(wait=False) enqueues the step and returns at once; the
    result is not ready while the stream is still busy (a sleep kernel queued
    ahead of it), poll() never blocks, and once the stream drains the result
    equals the blocking form's, bit for bit, over several steps."""
    from paper_2604_26687_b200.trainer import GnsManager
    M = 4
    xs, ys = _data(M, 5)
    mods = [_model(3), _model(3)]
    mgrs = [GnsManager(m.parameters(), micro_count=M, global_batch=M * 8) for m in mods]
    for step in range(3):
        for k, (model, mgr) in enumerate(zip(mods, mgrs)):
            mgr.begin_step()
            for x, y in zip(xs, ys):
                torch.nn.functional.mse_loss(model(x).float(), y.float()).backward()
                mgr.after_backward()
            if k == 0:
                blocking = mgr.finish_step(tokens=M * 8 * 2048)
            else:
                torch.cuda._sleep(200_000_000)  # ~0.1 s of GPU time queued ahead
                assert mgr.finish_step(tokens=M * 8 * 2048, wait=False) is None
                assert not mgr.gns.result_ready() and mgr.poll() is None
                torch.cuda.synchronize()
                assert mgr.gns.result_ready()
                polled = mgr.poll()
                assert polled is not None
                r = mgr.result()
                for a in (polled, r):
                    assert a.state.as_tuple() == blocking.state.as_tuple()
                    assert (a.stats.signal, a.stats.noise, a.b_simple) == \
                        (blocking.stats.signal, blocking.stats.noise, blocking.b_simple)
            # the optimizer step would go here; keep both models identical
    for mgr in mgrs:
        mgr.gns.close()


def test_result_ready_before_any_finalize_is_an_error():
    from paper_2604_26687_b200 import _lib as L
    from paper_2604_26687_b200 import device as D
    g = D.GnsDevice(1, 2, 2, 0)
    with pytest.raises(L.ValidationError):
        g.result_ready()
    g.close()
