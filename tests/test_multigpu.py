"""N > 1 path.

* CPU (gloo, world_size 2): the host-side logic — block mapping of the job's
  d*t*p ranks onto processes, slot algebra, unique-id broadcast — with the
  all-reduce of the N+1 partial scalars done by torch.distributed over gloo
  and the partials computed by the oracle; the result must equal the
  single-process computation.
* GPU (>= 2 devices): tests/mp_gns_worker.py under torch.distributed.run —
  the library's own NCCL all-reduce of the slots against a one-GPU run.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _job_partials(lays, ranks, M, d, seed, unit):
    """oracle: slot vector (d*M s values + gbar^2) contributed by `ranks`"""
    out = np.zeros(d * M + 1)
    for vr in ranks:
        lay = lays[vr]
        i_d = lay.coords[0]
        for m in range(M):
            buf = O.synth_fill(lay.numel, O.BF16, lay.gen, seed, i_d * M + m, 2 ** -10, unit)
            out[i_d * M + m] += O.sqnorm(buf, O.BF16, lay.segments)
        mean = O.synth_mean_fill(lay.numel, O.BF16, lay.gen, seed, 0, d * M, 2 ** -10, unit)
        # this DP replica's slice of its shard (same cut as coadapt_plan_create_slice)
        n = lay.numel
        lo = (n * i_d // d) & ~63
        hi = n if i_d + 1 == d else (n * (i_d + 1) // d) & ~63
        segs = []
        for o, k, w in lay.segments:
            b, e = max(o, lo), min(o + k, hi)
            if b < e:
                segs.append((b, e - b, w))
        out[-1] += O.sqnorm(mean, O.BF16, segs)
    return out


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    import torch
    from paper_2604_26687_b200 import dist as Dist
    from paper_2604_26687_b200 import layout as Lay
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = Lay.tiny_model(layers=4, h=32, ffn=64, vocab=64, tied=True)
    d, t, p, M = 2, 2, 2, 2
    lays = Lay.world_layouts(spec, d, t, p)
    unit = Lay.noise_unit_for(256.0, 1)
    mine = Dist.block_map(d * t * p, world, rank)
    part = torch.from_numpy(_job_partials(lays, mine, M, d, 5, unit))
    dist.all_reduce(part)  # stands in for the library's NCCL all-reduce
    uid = Dist.share_unique_id(dist, lambda: b"unique-id-from-rank-0".ljust(128, b"\0"), rank)
    if rank == 0:
        full = _job_partials(lays, list(range(d * t * p)), M, d, 5, unit)
        q.put((part.numpy().tolist(), full.tolist(), uid[:21]))
    dist.barrier()
    dist.destroy_process_group()


def test_block_map():
    from paper_2604_26687_b200 import dist as Dist
    assert Dist.block_map(8, 2, 1) == [4, 5, 6, 7]
    assert sorted(sum((Dist.block_map(8, 4, r) for r in range(4)), [])) == list(range(8))
    with pytest.raises(ValueError):
        Dist.block_map(8, 3, 0)


def test_gloo_two_process_allreduce_matches_single_process():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    part, full, uid = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert np.allclose(part, full, rtol=1e-13, atol=0)
    assert uid == b"unique-id-from-rank-0"
    # and the finalize on those slots matches the oracle's single-process step
    st = O.finalize_step(part[:-1], part[-1], len(part) - 1)
    st_ref = O.finalize_step(full[:-1], full[-1], len(full) - 1)
    assert st.signal == pytest.approx(st_ref.signal, rel=1e-12)


@pytest.mark.gpu
def test_nccl_two_gpus_matches_one_gpu():
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (gpurun --gpus 2)")
    world = 4 if n >= 4 else 2
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 400),
           os.path.join(HERE, "mp_gns_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    rep = json.loads(lines[-1])
    print(json.dumps(rep))
    # NCCL's communicator init lines (NCCL_DEBUG=INFO) prove the rank count
    print("\n".join(l for l in r.stdout.splitlines() + r.stderr.splitlines()
                    if "comm" in l and "nRanks" in l))
    assert rep["ok"], rep


@pytest.mark.gpu
def test_fused_reduce_scatter_norm_over_nvlink():
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (gpurun --gpus 2)")
    world = 4 if n >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29900 + os.getpid() % 90),
           os.path.join(HERE, "mp_rs_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    rep = json.loads(lines[-1])
    assert rep["ok"], rep


@pytest.mark.gpu
def test_reshard_pull_over_nvlink():
    """§8 f4: every rank pulls its new shards from the peers' packs (CUDA
    IPC) — all strategy pairs of the world size, bit-exact vs the oracle,
    plus a TP -> PP round trip at 0.5 GB per rank with the pull bandwidth."""
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (gpurun --gpus 2)")
    world = 4 if n >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29400 + os.getpid() % 90),
           os.path.join(HERE, "mp_reshard_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    rep = json.loads(lines[-1])
    print(json.dumps(rep))
    assert rep["ok"], rep


@pytest.mark.gpu
def test_single_process_drives_all_gpus():
    """One host thread, one GnsDevice per GPU: communicators from
    ncclCommInitAll, the slot all-reduce as one NCCL group; every GPU's
    result equals the one-GPU computation of the same world."""
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (gpurun --gpus 2)")
    from paper_2604_26687_b200 import _lib as L
    from paper_2604_26687_b200 import device as D
    from paper_2604_26687_b200 import dist as Dist
    from paper_2604_26687_b200 import layout as Lay
    spec = Lay.tiny_model(layers=4, h=256, ffn=512, vocab=1000)
    d, t, p, M = 2, 2, 2, 2
    lays = Lay.world_layouts(spec, d, t, p)
    unit = Lay.noise_unit_for(256.0, 1)

    def reduce_on(dev, g, ranks, stream):
        with torch.cuda.device(dev):
            for vr in ranks:
                lay = lays[vr]
                i_d = lay.coords[0]
                plan = D.BucketPlan(lay.segments, lay.numel, L.BF16, dev)
                b = torch.empty(lay.numel, dtype=torch.bfloat16, device=f"cuda:{dev}")
                for m in range(M):
                    D.synth_fill(b, lay.gen, 11, i_d * M + m, Lay.G0, unit, stream)
                    g.micro_sqnorm(plan, b, i_d, m, stream)
                D.synth_mean_fill(b, lay.gen, 11, 0, d * M, Lay.G0, unit, stream)
                sl = D.BucketPlan(lay.segments, lay.numel, L.BF16, dev, slice_index=i_d, slice_count=d)
                g.mean_sqnorm(sl, b, stream)
                torch.cuda.synchronize(dev)

    one = D.GnsDevice(d, M, d * M, 0)
    s0 = torch.cuda.Stream(device=0)
    one.begin_step(s0)
    reduce_on(0, one, range(len(lays)), s0)
    one.finalize(d * M * 2048, s0)
    ref = one.result()
    gs = [D.GnsDevice(d, M, d * M, dev) for dev in range(n)]
    D.attach_nccl_all(gs)
    streams = [torch.cuda.Stream(device=dev) for dev in range(n)]
    for dev in range(n):
        gs[dev].begin_step(streams[dev])
        reduce_on(dev, gs[dev], Dist.block_map(len(lays), n, dev), streams[dev])
    D.allreduce_group(gs, streams)
    for dev in range(n):
        gs[dev].finalize(d * M * 2048, streams[dev])
    for dev in range(n):
        r = gs[dev].result()
        assert abs(r.b_simple - ref.b_simple) <= 1e-12 * abs(ref.b_simple)
        assert np.allclose(gs[dev].partials(), one.partials(), rtol=1e-13, atol=0)


@pytest.mark.gpu
def test_nvls_switch_reduced_allreduce():
    """f2, NVLS form: fp32 buckets in multicast-bound memory all-reduced by
    the NVSwitch (multimem.ld_reduce / multimem.st); bit-exact on 2 GPUs,
    within the d-term fp32 sum bound on 4; bf16 refused."""
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (gpurun --gpus 2)")
    world = 4 if n >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + os.getpid() % 90),
           os.path.join(HERE, "mp_nvls_worker.py")]
    # the multicast handle must travel by SCM_RIGHTS (no pidfd_getfd fallback)
    env = dict(os.environ, COADAPT_NVLS_SHARE="socket")
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    rep = json.loads(lines[-1])
    assert rep["ok"], rep


@pytest.mark.gpu
def test_trainer_main_grad_in_nvls_memory():
    """f1 + f2: GnsManager with nvls_dist — main_grad all-reduced by the
    NVSwitch inside finish_step; main_grad, s_m, gbar^2 and phi vs torch."""
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (gpurun --gpus 2)")
    world = 4 if n >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29800 + os.getpid() % 90),
           os.path.join(HERE, "mp_trainer_nvls_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    rep = json.loads(lines[-1])
    assert rep["ok"], rep


@pytest.mark.gpu
def test_eight_rank_exchange_on_fewer_gpus():
    """The 8-peer mailbox exchange (the 8 x B200 case gpurun cannot provide)
    with 8 processes on the box's 2 or 4 GPUs: in-pass and standalone forms
    equal the one-GPU job for 4 steps, phi bit-identical on all 8 ranks."""
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (gpurun --gpus 2)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr", "127.0.0.1", "--master-port", str(29300 + os.getpid() % 90),
           os.path.join(HERE, "mp_p2p8_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    rep = json.loads(lines[-1])
    print(json.dumps(rep))
    assert rep["ok"], rep
