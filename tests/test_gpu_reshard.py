"""Device execution of reshard plans — GPU parity.

All ranks of both layouts live on cuda:0 as separate packs (virtual ranks;
the multi-GPU NVLink version is tests/mp_reshard_worker.py).  The executor
(coadapt_reshard_execute) must reproduce, bit for bit, the packs the oracle
builds straight from the global tensors (oracle/reshard_oracle.py,
SPEC.md:472's direct global-tensor check), for every element size, any
pointer alignment, whole-plan and per-destination execution; at a 3B-scale
size the A->B->A round trip must be the identity.
"""
import math
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import reshard_oracle as O  # noqa: E402
from paper_2604_26687_b200 import _lib as L  # noqa: E402
from paper_2604_26687_b200 import reshard as R  # noqa: E402

from test_reshard import llama3b_like, random_model, strategies, to_oracle  # noqa: E402

NP = {1: np.uint8, 2: np.int16, 4: np.float32, 8: np.float64}


def upload(a: np.ndarray, misalign: int = 0):
    """device copy of `a`; misalign > 0 places it `misalign` elements into a
    larger allocation so the pack pointer is not 16-byte aligned"""
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    if not misalign:
        return t, t
    big = torch.zeros(a.size + misalign, dtype=t.dtype, device="cuda")
    big[misalign:] = t
    return big[misalign:], big


@pytest.mark.parametrize("es", [1, 2, 4, 8])
@pytest.mark.parametrize("misalign", [0, 1])
def test_execute_matches_oracle(es, misalign):
    rng = random.Random(100 * es + misalign)
    dt = NP[es]
    for trial in range(12):
        m = random_model(rng)
        a = rng.choice(strategies(rng.choice([1, 2, 4, 8]), m.layers))
        b = rng.choice(strategies(rng.choice([1, 2, 4, 8]), m.layers))
        policy = rng.choice(["canonical", "spread"])
        om = to_oracle(m)
        la, lb = O.layout_for(om, a), O.layout_for(om, b)
        st = O.global_state(om, trial, dt)
        src = [upload(O.pack_from_global(la, r, st, dt), misalign)[0] for r in range(len(la.pack_numel))]
        want = [O.pack_from_global(lb, r, st, dt) for r in range(len(lb.pack_numel))]
        p = R.plan_transfers(m, a, b, policy)
        dst = [upload(np.zeros(n, dt), misalign)[0] for n in lb.pack_numel]
        p.execute(src, dst)
        torch.cuda.synchronize()
        for r in range(len(dst)):
            assert np.array_equal(dst[r].cpu().numpy(), want[r]), (a, b, r)
        # one destination at a time (the one-process-per-GPU form)
        dst2 = [upload(np.zeros(n, dt), misalign)[0] for n in lb.pack_numel]
        for r in range(len(dst2)):
            p.execute(src, dst2, dst_rank=r)
        torch.cuda.synchronize()
        for r in range(len(dst2)):
            assert torch.equal(dst2[r], dst[r])
        # one source at a time (push)
        dst3 = [upload(np.zeros(n, dt), misalign)[0] for n in lb.pack_numel]
        for r in range(len(src)):
            p.execute(src, dst3, src_rank=r)
        torch.cuda.synchronize()
        for r in range(len(dst3)):
            assert torch.equal(dst3[r], dst[r])


def test_execute_validation():
    m = R.ModelSpec(2, (R.TensorDecl("w", (64, 32), 0),))
    p = R.plan_transfers(m, (1, 2, 1), (1, 1, 2))
    src = [torch.zeros(p.pack_numel(R.SRC, r), dtype=torch.int16, device="cuda") for r in range(2)]
    dst = [torch.zeros(p.pack_numel(R.DST, r), dtype=torch.int16, device="cuda") for r in range(2)]
    with pytest.raises(L.ValidationError):
        p.execute(src, [dst[0], None])  # dst pack of rank 1 missing
    with pytest.raises(L.ValidationError):
        p.execute([src[0], None], dst)  # source of rank 1 missing
    with pytest.raises(L.ValidationError):
        p.execute(src, [src[0], dst[1]])  # destination aliases a source
    with pytest.raises(L.ValidationError):
        p.execute(src, dst, elem_bytes=3)
    with pytest.raises(L.ValidationError):
        p.execute(src[:1], dst)
    # a destination rank only needs the sources its moves read
    need = {x.src_rank for x in p.moves() if x.dst_rank == 1}
    p.execute([s if r in need else None for r, s in enumerate(src)], [None, dst[1]], dst_rank=1)


def _pad_mask(p, side, rank, n):
    keep = torch.zeros(n, dtype=torch.bool, device="cuda")
    for s in p.shards(side):
        if s.owner == rank:
            keep[s.pack_offset:s.pack_offset + math.prod(s.local_shape)] = True
    return keep


def test_round_trip_3b_scale_virtual_ranks():
    """llama-3.2-3B-shaped layers, d1t2p4 -> d1t4p2 -> d1t2p4 on one GPU:
    2 x 5.4 GB of bf16 packs; the round trip must be the identity."""
    m = llama3b_like()
    fwd = R.plan_transfers(m, (1, 2, 4), (1, 4, 2))
    back = R.plan_transfers(m, (1, 4, 2), (1, 2, 4))
    g = torch.Generator(device="cuda").manual_seed(7)
    A = []
    for r in range(8):
        n = fwd.pack_numel(R.SRC, r)
        x = torch.randint(-32768, 32767, (n,), dtype=torch.int16, device="cuda", generator=g)
        x[~_pad_mask(fwd, R.SRC, r, n)] = 0
        A.append(x)
    B = [torch.zeros(fwd.pack_numel(R.DST, r), dtype=torch.int16, device="cuda") for r in range(8)]
    fwd.execute(A, B)
    A2 = [torch.zeros_like(x) for x in A]
    back.execute(B, A2)
    torch.cuda.synchronize()
    for r in range(8):
        assert torch.equal(A2[r], A[r]), r
    # spot-check B against the global tensors for one key: layer 5 "down"
    # (tp axis 1) is rebuilt from the A packs by the torch reference below
    ti = 6
    lay_a, lay_b = fwd.shards(R.SRC), fwd.shards(R.DST)
    full = torch.empty(m.per_layer[ti].shape, dtype=torch.int16, device="cuda")
    for s in lay_a:
        if (s.layer, s.tensor) == (5, ti) and s.canonical:
            sl = tuple(slice(o, o + e) for o, e in zip(s.global_offset, s.local_shape))
            full[sl] = A[s.owner][s.pack_offset:s.pack_offset + math.prod(s.local_shape)].view(s.local_shape)
    for s in lay_b:
        if (s.layer, s.tensor) == (5, ti):
            sl = tuple(slice(o, o + e) for o, e in zip(s.global_offset, s.local_shape))
            got = B[s.owner][s.pack_offset:s.pack_offset + math.prod(s.local_shape)].view(s.local_shape)
            assert torch.equal(got, full[sl])
