"""Kernel micro-benchmark: K1 (single-bucket sqnorm), K1f (fused) and the
read-only probe on large resident buffers, CUDA-event timed, L2 >> bytes.

    python tools/kbench.py [--gb 8] [--reps 10] [--fused-m 16]
Prints one JSON line.  (Development tool; bench.py is the contract.)
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_26687_b200 import _lib as L  # noqa: E402
from paper_2604_26687_b200 import device as D  # noqa: E402


SUSTAIN = [0.0]


def timed(fn, reps, stream):
    fn()
    torch.cuda.synchronize()
    if SUSTAIN[0] > 0:
        # run for SUSTAIN seconds; time only the second half (steady state)
        import time
        t0 = time.time()
        while time.time() - t0 < SUSTAIN[0] / 2:
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
        n = 0
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        t1 = time.time()
        while time.time() - t1 < SUSTAIN[0] / 2:
            for _ in range(5):
                fn()
            n += 5
            torch.cuda.synchronize()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n / 1e3
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=8.0)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--fused-m", type=int, default=16)
    ap.add_argument("--fused-gb", type=float, default=16.0)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--kernels", default="k1,probe,k1f,accum",
                    help="comma list of k1, probe, k1f, accum")
    ap.add_argument("--phi", type=float, default=256.0,
                    help="synthetic noise scale of the data (power depends on the bits)")
    ap.add_argument("--sustain", type=float, default=0.0,
                    help="seconds of back-to-back launches per kernel (power-cap steady state)")
    args = ap.parse_args()
    SUSTAIN[0] = args.sustain
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    dt = {"bf16": L.BF16, "fp32": L.FP32, "fp16": L.FP16}[args.dtype]
    tdt = D.DTYPE_TO_TORCH[dt]
    es = D.ESIZE[dt]
    n = int(args.gb * 1e9 / es)
    x = torch.empty(n, dtype=tdt, device="cuda")
    from paper_2604_26687_b200 import layout as Lay
    unit = Lay.noise_unit_for(args.phi, 1)
    D.synth_fill(x, [(0, n, 0, n, n)], 1, 0, 2.0 ** -10, unit)
    plan = D.BucketPlan([(0, n, 1.0)], n, dt, 0)
    g = D.GnsDevice(1, args.fused_m, args.fused_m, 0)
    out = {"variant": os.environ.get("COADAPT_BF16_VARIANT", "default"), "dtype": args.dtype}
    ks = set(args.kernels.split(","))
    out["tma_shape"] = os.environ.get("COADAPT_TMA_SHAPE", "default")
    with torch.cuda.stream(s):
        if "k1" in ks:
            sec = timed(lambda: g.micro_sqnorm(plan, x, 0, 0, s), args.reps, s)
            out["k1_gbs"] = round(n * es / sec / 1e9, 1)
        sink = torch.zeros(1, dtype=torch.float64, device="cuda")
        if "probe" in ks:
            sec = timed(lambda: D.read_probe(x, sink, s), args.reps, s)
            out["probe_gbs"] = round(n * es / sec / 1e9, 1)
        del x
        torch.cuda.empty_cache()
        M = args.fused_m
        nb = int(args.fused_gb * 1e9 / es / M)
        bufs = [torch.empty(nb, dtype=tdt, device="cuda") for _ in range(M)]
        for m, b in enumerate(bufs):
            D.synth_fill(b, [(0, nb, 0, nb, nb)], 1, m, 2.0 ** -10, unit)
        fplan = D.BucketPlan([(0, nb, 1.0)], nb, dt, 0)
        if "k1f" in ks:
            sec = timed(lambda: g.fused_sqnorm(fplan, bufs, s), args.reps, s)
            out["k1f_gbs"] = round(nb * M * es / sec / 1e9, 1)
            out["k1f_bytes"] = nb * M * es
        if "accum" not in ks:
            print(json.dumps(out), flush=True)
            return
        # trainer form: fp32 main_grad += grad with s_m fused, vs torch's add_
        na = nb
        main = torch.zeros(na, dtype=torch.float32, device="cuda")
        aplan = D.BucketPlan([(0, na, 1.0)], na, dt, 0)
        acc_bytes = na * (es + 8)  # read grad, read + write main_grad
        sec = timed(lambda: g.accumulate(aplan, main, bufs[1], 0, 1, stream=s), args.reps, s)
        out["accum_fused_gbs"] = round(acc_bytes / sec / 1e9, 1)
        out["accum_fused_ms"] = round(sec * 1e3, 3)
        sec_t = timed(lambda: main.add_(bufs[1]), args.reps, s)
        out["accum_torch_ms"] = round(sec_t * 1e3, 3)
        out["accum_torch_gbs"] = round(acc_bytes / sec_t / 1e9, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
