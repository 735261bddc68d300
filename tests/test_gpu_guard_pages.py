"""Out-of-bounds detection without compute-sanitizer (closed on this pool:
profiles/r02_sanitizer.txt): every bucket handed to the kernels sits in
virtual memory whose neighbouring 2 MiB granules are reserved but NOT mapped
(cuMemAddressReserve + cuMemCreate/cuMemMap of the middle only), with the
bucket's first byte at the start of the mapping or its last byte at the end.
A single byte read or written outside the bucket faults the context
(CUDA_ERROR_ILLEGAL_ADDRESS) and fails the test.  Covered: K1f (TMA ring,
M = 1, 2, 7, 16, shapes with both consumer groups), its LDG fallback for
unaligned views, the batched K1 ring, K2 DP slices, the in-pass finalize, the
trainer form KA (which also WRITES main_grad, guarded the same way), every
result bit-identical to the same launch on ordinary torch buffers."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


class Guarded:
    """`nbytes` of device memory placed flush against unmapped granules."""

    def __init__(self, nbytes: int, at_end: bool, device: int = 0):
        from cuda.bindings import driver as drv
        self.drv = drv
        prop = drv.CUmemAllocationProp()
        prop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = device
        err, gran = drv.cuMemGetAllocationGranularity(
            prop, drv.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM)
        assert err == drv.CUresult.CUDA_SUCCESS
        size = (nbytes + gran - 1) // gran * gran
        err, self.va = drv.cuMemAddressReserve(size + 2 * gran, gran, 0, 0)
        assert err == drv.CUresult.CUDA_SUCCESS
        err, self.handle = drv.cuMemCreate(size, prop, 0)
        assert err == drv.CUresult.CUDA_SUCCESS
        self.mid = int(self.va) + gran
        assert drv.cuMemMap(self.mid, size, 0, self.handle, 0)[0] == drv.CUresult.CUDA_SUCCESS
        acc = drv.CUmemAccessDesc()
        acc.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = device
        acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        assert drv.cuMemSetAccess(self.mid, size, [acc], 1)[0] == drv.CUresult.CUDA_SUCCESS
        self.size, self.gran = size, gran
        self.ptr = self.mid + (size - nbytes if at_end else 0)
        self.nbytes = nbytes

    def copy_to(self, t: torch.Tensor):
        torch.cuda.synchronize()
        assert self.drv.cuMemcpyDtoD(t.data_ptr(), self.ptr, self.nbytes)[0] == \
            self.drv.CUresult.CUDA_SUCCESS

    def copy_from(self, t: torch.Tensor):
        torch.cuda.synchronize()
        assert self.drv.cuMemcpyDtoD(self.ptr, t.data_ptr(), self.nbytes)[0] == \
            self.drv.CUresult.CUDA_SUCCESS

    def close(self):
        torch.cuda.synchronize()
        d = self.drv
        d.cuMemUnmap(self.mid, self.size)
        d.cuMemRelease(self.handle)
        d.cuMemAddressFree(self.va, self.size + 2 * self.gran)


def _env():
    from paper_2604_26687_b200 import _lib as L
    from paper_2604_26687_b200 import device as D
    from paper_2604_26687_b200 import layout as Lay
    torch.cuda.set_device(0)
    return L, D, Lay


def _fill(D, L, ptr, numel, gen, seed, sample, unit):
    arr, n = D._gen_array(gen)
    L.check(L.lib().coadapt_synth_fill(C.c_void_p(ptr), L.BF16, arr, n, seed, sample,
                                       C.c_float(2.0 ** -10), C.c_float(unit),
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)))


def _check(ok_parts, ref_parts):
    assert np.array_equal(ok_parts, ref_parts), (ok_parts, ref_parts)


@pytest.mark.parametrize("at_end", [True, False])
@pytest.mark.parametrize("M", [1, 2, 7, 16])
def test_fused_and_batched_stay_inside_guarded_buckets(M, at_end):
    L, D, Lay = _env()
    spec = Lay.tiny_model(layers=8, h=512, ffn=1024, vocab=4096)
    lay = Lay.rank_layout(spec, 1, 2, 2, 1)  # weight-0 holes inside the bucket
    n = lay.numel - lay.numel % 8  # 16-byte multiple: TMA path at both ends
    segs = [(o, min(k, n - o), w) for o, k, w in lay.segments if o < n]
    gen = [(0, n, 0, n, n)]
    unit = Lay.noise_unit_for(256.0, 1)
    guards = [Guarded(n * 2, at_end) for _ in range(M)]
    plain = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(M)]
    for m, g in enumerate(guards):
        _fill(D, L, g.ptr, n, gen, 11, m, unit)
        g.copy_to(plain[m])
    plan = D.BucketPlan(segs, n, L.BF16, 0)
    try:
        for use in ("fused", "batched", "inpass"):
            if use != "batched" and M < 2:
                continue
            # (N = d*M must be >= 2: M = 1 runs as d = 2)
            a = D.GnsDevice(1, M, M, 0) if M > 1 else D.GnsDevice(2, M, 2, 0)
            b = D.GnsDevice(1, M, M, 0) if M > 1 else D.GnsDevice(2, M, 2, 0)
            a.begin_step()
            b.begin_step()
            if use == "fused":
                a.fused_sqnorm(plan, [g.ptr for g in guards])
                b.fused_sqnorm(plan, plain)
            elif use == "inpass":
                a.fused_sqnorm_finalize(plan, [g.ptr for g in guards], M * 2048)
                b.fused_sqnorm_finalize(plan, plain, M * 2048)
                assert a.result().b_simple == b.result().b_simple
            else:
                a.micro_sqnorm_batched(plan, [g.ptr for g in guards], [0] * M, list(range(M)))
                b.micro_sqnorm_batched(plan, plain, [0] * M, list(range(M)))
            torch.cuda.synchronize()
            _check(a.partials(), b.partials())
            a.close()
            b.close()
    finally:
        for g in guards:
            g.close()


@pytest.mark.parametrize("at_end", [True, False])
def test_ldg_fallback_slices_and_trainer_form_stay_inside(at_end):
    L, D, Lay = _env()
    n = 3 * 1792 * 148 + 37  # odd: the views below are only 2-byte aligned
    segs = [(0, 1000, 1.0), (1000, 5000, 0.0), (6000, n - 6000, 1.0)]
    gen = [(0, n, 0, n, n)]
    unit = Lay.noise_unit_for(64.0, 1)
    M = 4
    guards = [Guarded(n * 2, at_end) for _ in range(M)]
    # the plain reference buckets get the same address mod 16 (so the same
    # TMA-or-LDG path and edge split as the guarded ones)
    k = (guards[0].ptr % 16) // 2
    plain = [torch.empty(n + 8, dtype=torch.bfloat16, device="cuda")[k:k + n] for _ in range(M)]
    nk8 = n - n % 8
    mg = Guarded(nk8 * 4, at_end)  # fp32 main_grad, written by KA
    extra = []
    try:
        for m, g in enumerate(guards):
            _fill(D, L, g.ptr, n, gen, 3, m, unit)
            g.copy_to(plain[m])
        plan = D.BucketPlan(segs, n, L.BF16, 0)
        # at_end: n is odd, so the bucket addresses are only 2-byte aligned
        # and K1f / K1 take their LDG forms; at the start they take the TMA ring
        a, b = D.GnsDevice(1, M, M, 0), D.GnsDevice(1, M, M, 0)
        for g in (a, b):
            g.begin_step()
        a.fused_sqnorm(plan, [g.ptr for g in guards])
        b.fused_sqnorm(plan, plain)
        torch.cuda.synchronize()
        _check(a.partials(), b.partials())
        # K2: every DP slice of the guarded "mean"
        for d in (2, 3):
            a2, b2 = D.GnsDevice(d, 1, d, 0), D.GnsDevice(d, 1, d, 0)
            for g in (a2, b2):
                g.begin_step()
            for i in range(d):
                sl = D.BucketPlan(segs, n, L.BF16, 0, slice_index=i, slice_count=d)
                a2.mean_sqnorm(sl, guards[0].ptr)
                b2.mean_sqnorm(sl, plain[0])
                torch.cuda.synchronize()
                sl.close()
            _check(a2.partials(), b2.partials())
        # KA (needs 16-byte aligned buffers): a whole-vector length so the
        # guarded grads and main_grad still end flush against unmapped memory
        nk = n - n % 8
        kg = [Guarded(nk * 2, at_end) for _ in range(M)]
        extra.extend(kg)
        for m in range(M):
            kg[m].copy_from(plain[m][:nk].contiguous())
        kplan = D.BucketPlan([(o, min(q, nk - o), w) for o, q, w in segs if o < nk], nk, L.BF16, 0)
        main_plain = torch.zeros(nk, dtype=torch.float32, device="cuda")
        plain_k = [p[:nk].clone() for p in plain]  # aligned copies
        ka, kb = D.GnsDevice(1, M, M, 0), D.GnsDevice(1, M, M, 0)
        for g in (ka, kb):
            g.begin_step()
        for m in range(M):
            L.check(L.lib().coadapt_gns_accumulate(ka.handle, kplan.handle, C.c_void_p(mg.ptr),
                                                   C.c_void_p(kg[m].ptr), 0, m,
                                                   (1 if m == 0 else 0) | (2 if m == M - 1 else 0),
                                                   C.c_double(1.0 / (M * M)),
                                                   C.c_void_p(torch.cuda.current_stream().cuda_stream)))
            kb.accumulate(kplan, main_plain, plain_k[m], 0, m, first=m == 0, last_mean=m == M - 1)
        torch.cuda.synchronize()
        _check(ka.partials(), kb.partials())
        back = torch.empty(nk, dtype=torch.float32, device="cuda")
        mg.copy_to(back)
        assert torch.equal(back, main_plain)
    finally:
        for g in guards + [mg] + extra:
            g.close()
