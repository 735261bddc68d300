"""bench.py — GNS estimate throughput on B200 (BASELINE.json metric).

One "step" is one full online-GNS optimizer step of the configured job over
synthetic gradients of the named model shape: every (rank, micro-batch)
squared norm + the mean-gradient norm (fused for d = 1), the NCCL scalar
all-reduce, the device finalize/EMA/phi kernel, the phi read-back and the
CPU goodput decision over the candidate table (config C5 = the "full goodput
step").  The d*t*p ranks of the job are block-mapped onto the N GPUs
(strong scaling: total work fixed).  value = algorithmic bytes of the whole
job per step / step time (max over ranks, CUDA events).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c2|c3|c1]
    python bench.py --impl reference ...   # CPU reference arm (oracle port)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GNS estimate gradient GB/s and % HBM roofline at 1/2/4/8 B200 vs CPU ref"
UNIT = "GB/s"

# BASELINE.json configs; M for C3 is the survey's proposal.
CONFIGS = {
    "c1": dict(shape="125m", d=2, t=1, p=1, M=4, Bm=2, dtype="fp32", seed=0xC0905 + 0),
    "c2": dict(shape="3b", d=8, t=1, p=1, M=8, Bm=2, dtype="bf16", seed=0xC0905 + 1),
    "c3": dict(shape="7b", d=2, t=2, p=2, M=8, Bm=2, dtype="bf16", seed=0xC0905 + 2),
    "c4": dict(shape="32b", d=1, t=4, p=2, M=16, Bm=1, dtype="bf16", seed=0xC0905 + 3),
}
PHI_TRUE = 256.0
SEQ_LEN = 2048


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--x1", choices=["nccl", "p2p"], default="p2p",
                    help="N > 1 slot all-reduce: fused with finalize over NVLink mailboxes "
                         "(default), or NCCL all-reduce + finalize")
    ap.add_argument("--finalize", choices=["inpass", "separate"], default="inpass",
                    help="finalize (and the N > 1 slot exchange) in the last reduction's "
                         "last CTA (default), or as its own launch(es) after it")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-elems", type=int, default=128 << 20, help="sample elements per micro-bucket")
    return ap.parse_args()


def workload_name(c):
    return f"gns-step {c['shape']} {c['dtype']} (d,t,p)=({c['d']},{c['t']},{c['p']}) M={c['M']}"


def candidate_costs(n_gpus_job: int):
    """Synthetic throughput table over every (d,t,p) of the
    job's GPU count, with saturating curves that cross (Fig. 2)."""
    out = []
    for d in range(1, n_gpus_job + 1):
        if n_gpus_job % d:
            continue
        for t in range(1, n_gpus_job // d + 1):
            if (n_gpus_job // d) % t:
                continue
            p = n_gpus_job // (d * t)
            out.append((d, t, p, 1000.0 * d ** 0.5 * (1.0 + 0.2 * t), 8.0 * d * d + 4.0 * p))
    return out


def read_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(path))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def traffic_for(config_key):
    """dram bytes per launch of the dominant kernel, from the committed ncu
    summary (profiles/traffic.json), or None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return t.get(config_key)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        # nvidia-smi takes ~0.1-0.5 s to start: wait for its first sample so a
        # short timed region is still covered (and drop that warm-up sample)
        t0 = time.time()
        while not self.rows and time.time() - t0 < 5.0:
            time.sleep(0.01)
        self.skip = len(self.rows)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        rows = self.rows[getattr(self, "skip", 0):]
        if not rows:  # region shorter than the sampling period: one query now
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits", "-i", str(self.index)],
                                     capture_output=True, text=True, timeout=10).stdout
                rows = [[x.strip() for x in line.split(",")] for line in out.splitlines() if line]
            except Exception:
                rows = []
        self.rows = rows
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for nm, v in zip(names, r[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- distributed plumbing

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def init_dist(ws, backend):
    import torch.distributed as dist
    if ws > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group(backend)
    return dist


# ---------------------------------------------------------------- CPU oracle timing

def cpu_oracle_rate(host_bufs, dtype_code, segs, seconds, nthreads):
    """Time the oracle's fused fp64 pass (oracle/oracle.c) over host buffers
    until `seconds` elapse; returns (GB/s, bytes per pass, passes)."""
    from oracle import oracle as O
    nbytes = sum(b.nbytes for b in host_bufs)
    passes, t0 = 0, time.perf_counter()
    while True:
        O.fused_sqnorms(host_bufs, dtype_code, segs, nthreads)
        passes += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return nbytes * passes / el / 1e9, nbytes, passes, el


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- reference arm

def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0  # the reference arm is rank 0 only
    import numpy as np
    from oracle import oracle as O
    from paper_2604_26687_b200 import layout as Lay
    c = CONFIGS[args.config]
    spec = Lay.MODELS[c["shape"]]()
    lay = Lay.rank_layout(spec, c["d"], c["t"], c["p"], 0)
    dt = O.FP32 if c["dtype"] == "fp32" else O.BF16
    es = 4 if dt == O.FP32 else 2
    M = c["M"]
    E = min(lay.numel, 32 << 20)  # bounded sample per micro-bucket
    gen = [(0, E, 0, E, E)]
    segs = [(o, min(n, E - o), w) for o, n, w in lay.segments if o < E]
    unit = Lay.noise_unit_for(PHI_TRUE, c["Bm"])
    bufs = [O.synth_fill(E, dt, gen, c["seed"], m, Lay.G0, unit) for m in range(M)]
    nth = host_threads()
    costs = candidate_costs(c["d"] * c["t"] * c["p"])
    ents = O.feasible_candidates(O.synth_profile(costs, [16, 32, 64, 128, 256, 512, 1024, 2048],
                                                 [1, 2, 4, 8], True, 0.0, 0.0, 1e300))
    st = O.State.default()

    def step():
        s, ss = O.fused_sqnorms(bufs, dt, segs, nth)
        stats = O.finalize_step(s, ss / (M * M), M * c["Bm"])
        O.update_ema(st, stats, M * c["Bm"] * SEQ_LEN)
        phi = O.gns(st)
        O.decide(ents, phi, ents[0], 1000.0, 900.0, reconfig_cost=40.0)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    nbytes = M * sum(n for _, n, w in segs if w) * es
    v = nbytes * args.steps / el / 1e9
    sample = (f"{M} micro-buckets x first {E} elements of rank 0's {c['shape']} shard "
              f"({nbytes / 1e9:.3f} GB per step), oracle fused fp64 pass + finalize/EMA/decide")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": c["dtype"], "data": "synthetic",
            "config": {"workload": workload_name(c), "sample": sample},
            "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": nth, "kind": "port",
                             "sample": sample},
            "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm

def run_ours(args):
    import numpy as np
    import torch

    from paper_2604_26687_b200 import _lib as L
    from paper_2604_26687_b200 import device as D
    from paper_2604_26687_b200 import gns as G
    from paper_2604_26687_b200 import layout as Lay

    ws, rank, local = dist_env()
    if ws > 1:
        # keep NCCL's communicator init lines (one per rank, "nRanks N") in
        # the log so the rank count of the run is checkable
        if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
    dist = init_dist(ws, "nccl")
    torch.cuda.set_device(local)
    dev = local
    c = CONFIGS[args.config]
    d, t, p, M = c["d"], c["t"], c["p"], c["M"]
    R = d * t * p
    if R % ws:
        raise SystemExit(f"{R} ranks of the job do not block-map onto {ws} GPUs")
    spec = Lay.MODELS[c["shape"]]()
    lays = Lay.world_layouts(spec, d, t, p)
    mine = lays[rank * R // ws:(rank + 1) * R // ws]
    dt = L.FP32 if c["dtype"] == "fp32" else L.BF16
    tdt = torch.float32 if dt == L.FP32 else torch.bfloat16
    es = 4 if dt == L.FP32 else 2
    fused = d == 1
    unit = Lay.noise_unit_for(PHI_TRUE, c["Bm"])
    B_g = d * M * c["Bm"]
    stream = torch.cuda.Stream(device=dev)

    # -- resident synthetic buffers: one pool of M micro-buckets sized for the
    #    largest local rank; virtual ranks sharing a GPU share the pool (the
    #    bytes each reduction streams from HBM are the job's exact bytes).
    numel = max(l.numel for l in mine)
    first = mine[0]
    pool = []
    with torch.cuda.stream(stream):
        for m in range(M):
            b = torch.zeros(numel, dtype=tdt, device="cuda")
            D.synth_fill(b, first.gen, c["seed"], first.coords[0] * M + m, Lay.G0, unit)
            pool.append(b)
        mean = None
        if not fused:
            mean = torch.zeros(numel, dtype=tdt, device="cuda")
            D.synth_mean_fill(mean, first.gen, c["seed"], 0, d * M, Lay.G0, unit)
    stream.synchronize()
    plans = [D.BucketPlan(l.segments, numel, dt, dev) for l in mine]
    slices = [D.BucketPlan(l.segments, numel, dt, dev, slice_index=l.coords[0], slice_count=d)
              for l in mine] if not fused else []
    g = D.GnsDevice(d, M, B_g, dev)
    if ws > 1:
        uid = D.nccl_unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        g.attach_nccl(ws, rank, obj[0])
        if args.x1 == "p2p":
            from paper_2604_26687_b200 import dist as Dist
            p2p_bases = Dist.attach_p2p(g, dist, ws, rank)

    costs = candidate_costs(R)
    # marshalled once: the per-step decide is then one C call (~6 us, not ~80)
    cands = G.CandidateTable(G.synth_candidates(costs, [16, 32, 64, 128, 256, 512, 1024, 2048],
                                                [1, 2, 4, 8], True))
    current = next(x for x in cands if (x.d, x.t, x.p) == (d, t, p)) if any(
        (x.d, x.t, x.p) == (d, t, p) for x in cands) else cands[0]

    # algorithmic bytes: every rank's counted shard x M, plus the
    # mean-gradient slices when d > 1
    job_bytes = Lay.algorithmic_bytes(spec, d, t, p, M, es, fused)
    local_bytes = sum(l.counted for l in mine) * M * es
    if not fused:
        local_bytes += sum(pl.active_elements for pl in slices) * es
    # one launch per virtual rank covers its M micro-buckets (fused pass, or
    # the batched K1 over the M buckets)
    launch_bytes = [pl.active_elements * es * M for pl in plans]

    ev_pairs, tail_pairs, decide_s = [], [], []
    mean_pairs, step_marks = [], []  # K2 launches; (step start, last launch end) per step

    # in-pass: the step's last reduction launch finalizes in its last CTA
    # (after the NVLink slot exchange when N > 1) — north_star item 2
    inpass = args.finalize == "inpass" and (ws == 1 or args.x1 == "p2p")
    tokens = B_g * SEQ_LEN

    def step(timed):
        if timed:
            s0 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
        g.begin_step(stream)
        for i, pl in enumerate(plans):
            last = inpass and i + 1 == len(plans)
            if timed:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            if fused:
                if last:
                    g.fused_sqnorm_finalize(pl, pool, tokens, stream)
                else:
                    g.fused_sqnorm(pl, pool, stream)
            else:
                g.micro_sqnorm_batched(pl, pool, [mine[i].coords[0]] * M, list(range(M)), stream)
            if timed:
                e1.record(stream)
                # the launch that also waits for the peers' slots (N > 1) is
                # kept out of the kernel roofline
                ev_pairs.append((e0, e1, launch_bytes[i], not (last and fused and ws > 1)))
            if not fused:
                if timed:
                    m0 = torch.cuda.Event(enable_timing=True)
                    m1 = torch.cuda.Event(enable_timing=True)
                    m0.record(stream)
                if last:
                    g.mean_sqnorm_finalize(slices[i], mean, tokens, stream)
                else:
                    g.mean_sqnorm(slices[i], mean, stream)
                if timed:
                    m1.record(stream)
                    mean_pairs.append((m0, m1))
        if timed:
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            f0.record(stream)
        if not inpass:
            if args.x1 == "p2p" and ws > 1:
                g.allreduce_finalize_p2p(tokens, stream)
            else:
                g.allreduce(stream)
                g.finalize(tokens, stream)
        if timed:
            f1.record(stream)
            tail_pairs.append((f0, f1))
            step_marks.append((s0, f1))
        r = g.result()  # phi -> host (waits for this step)
        h0 = time.perf_counter()
        G.decide(cands, r.phi if r.phi_available else None, current, 1000.0, 900.0, reconfig_cost=40.0)
        if timed:
            decide_s.append(time.perf_counter() - h0)
        return r

    for _ in range(args.warmup):
        step(False)
    # read-only streaming peak on this box (same load path, no math)
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    probe_bytes = pool[0].numel() * pool[0].element_size()
    with torch.cuda.stream(stream):
        D.read_probe(pool[0], sink, stream)
        pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pe0.record(stream)
        for k in range(3):
            D.read_probe(pool[k % M], sink, stream)
        pe1.record(stream)
    stream.synchronize()
    ro_peak = 3 * probe_bytes / (pe0.elapsed_time(pe1) / 1e3) / 1e9

    clocks = ClockSampler(dev)
    if os.environ.get("COADAPT_BENCH_NO_CLOCKS") == "1":  # diagnosis only: no sampler
        clocks.start = lambda: None
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = D.kernel_launches()
    clocks.start()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for _ in range(args.steps):
        r = step(True)
    t_end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = D.kernel_launches() - launches0
    if ws > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end) / args.steps
    if ws > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = job_bytes / (ms / 1e3) / 1e9

    # C5 "full goodput step" latency split: the reductions,
    # the all-reduce + finalize tail on the device, the host decide()
    red_ms = sum(a.elapsed_time(b) for a, b, _, _ in ev_pairs) / args.steps
    tail_ms = sum(a.elapsed_time(b) for a, b in tail_pairs) / max(1, len(tail_pairs))
    mean_ms = sum(a.elapsed_time(b) for a, b in mean_pairs) / args.steps
    # the stream's idle time between steps (phi D2H, host wake-up, decide,
    # the next step's first launch): last launch end -> next step start
    idle = [step_marks[k][1].elapsed_time(step_marks[k + 1][0]) for k in range(len(step_marks) - 1)]
    idle_ms = sum(idle) / len(idle) if idle else 0.0
    red_all = [red_ms]
    if ws > 1:  # per-GPU reduction time: the max-over-ranks step waits for the slowest
        rt = torch.tensor([red_ms], dtype=torch.float64, device="cuda")
        gat = [torch.zeros_like(rt) for _ in range(ws)]
        dist.all_gather(gat, rt)
        red_all = [float(x.item()) for x in gat]
        ct = torch.tensor([float((clk or {}).get("sm_mhz") or 0.0)], dtype=torch.float64, device="cuda")
        cg = [torch.zeros_like(ct) for _ in range(ws)]
        dist.all_gather(cg, ct)
        if clk is not None:
            clk["sm_mhz_per_gpu"] = [float(x.item()) for x in cg]
    # the tail on its own: all ranks aligned by a barrier + sync first, so
    # the number is the exchange + finalize latency without the wait for the
    # slowest GPU's reductions (that wait is rank_skew_ms)
    synced = []
    for _ in range(20 if ws > 1 else 5):
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        if args.x1 == "p2p" and ws > 1:
            g.allreduce_finalize_p2p(B_g * SEQ_LEN, stream)
        else:
            g.allreduce(stream)
            g.finalize(B_g * SEQ_LEN, stream)
        a1.record(stream)
        torch.cuda.synchronize()
        synced.append(a0.elapsed_time(a1))
    synced_ms = statistics.median(synced)
    if ws > 1:
        tt = torch.tensor([synced_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        synced_ms = float(tt.item())
    goodput_step = {"step_ms": round(ms, 4), "reductions_ms": round(red_ms, 4),
                    "reductions_ms_per_gpu": [round(x, 4) for x in red_all],
                    "mean_slices_ms": round(mean_ms, 4) if not fused else None,
                    "between_steps_idle_ms": round(idle_ms, 4),
                    "between_steps_idle_ms_each": [round(x, 3) for x in idle],
                    "rank_skew_ms": round(max(red_all) - min(red_all), 4),
                    "allreduce_finalize_ms": round(tail_ms, 4),
                    "allreduce_finalize_ms_synced": round(synced_ms, 4),
                    "x1": (("p2p: slot exchange + finalize in one kernel over NVLink"
                            if args.x1 == "p2p" else "nccl all-reduce + finalize kernel")
                           if ws > 1 else "local (one GPU)"),
                    "finalize": ("in-pass: in the last CTA of the step's last reduction launch"
                                 + (" after the NVLink slot exchange" if ws > 1 else "")
                                 + "; allreduce_finalize_ms measures only the host-side gap "
                                   "after it, allreduce_finalize_ms_synced the standalone "
                                   "exchange + finalize kernel" if inpass else "separate launches"),
                    "decide_ms": round(1e3 * sum(decide_s) / max(1, len(decide_s)), 4),
                    "candidates": len(cands)}

    # dominant-kernel roofline (per-launch CUDA events on the launching stream)
    kept = [e for e in ev_pairs if e[3]] or ev_pairs
    durs = [a.elapsed_time(b) / 1e3 for a, b, _, _ in kept]
    byts = [x for _, _, x, _ in kept]
    achieved = sum(byts) / sum(durs) / 1e9
    peak, peak_kind = read_peak()
    kname = "fused_tma_kernel (K1f)" if fused else "fused_tma_kernel<MEAN=false> (K1 on the TMA ring)"
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic_for(args.config),
            "kernel": kname, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}, copy)",
            "read_only_peak_gbs_this_box": round(ro_peak, 1),
            "frac_of_read_only_peak": round(achieved / ro_peak, 4),
            "frac_of_nominal_8000": round(achieved / 8000.0, 4),
            "avg_launch_ms": round(1e3 * sum(durs) / len(durs), 4),
            "bytes_per_launch": int(sum(byts) / len(byts))}

    # -- e2e: the same step through the host-pointer entry point (pinned host
    #    buckets, H2D inside the timed region), bounded sample per bucket
    e2e = None
    if not args.no_e2e:
        E = min(args.e2e_elems, numel)
        # pinned host sample of every rank on this box: at most a quarter of
        # the host RAM and 16 GiB in total (8 ranks x 16 buckets x 268 MB
        # would pin 34 GB); the metric is a rate, so a smaller sample per
        # rank changes nothing but the step length
        try:
            import psutil
            cap = min(16 << 30, psutil.virtual_memory().total // 4)
            per_elem = (M + (0 if fused else 1)) * es * ws
            E = min(E, max(1 << 22, cap // per_elem // 64 * 64))
        except ImportError:
            pass
        segs_e = [(o, min(n, E - o), w) for o, n, w in mine[0].segments if o < E]
        plan_e = D.BucketPlan(segs_e, E, dt, dev)
        host = [pool[m][:E].cpu().pin_memory() for m in range(M)]
        if not fused:  # d > 1: this rank's DP slice of the synchronised mean
            d_job = c["d"]
            slice_e = D.BucketPlan(segs_e, E, dt, dev, slice_index=0, slice_count=d_job)
            host_mean = mean[:E].cpu().pin_memory()
        ge = D.GnsDevice(1, M, B_g, dev)
        if ws > 1:
            uid = D.nccl_unique_id() if rank == 0 else bytes(128)
            obj = [uid]
            dist.broadcast_object_list(obj, src=0)
            ge.attach_nccl(ws, rank, obj[0])

        def estep():
            ge.begin_step(stream)
            if fused:
                ge.fused_sqnorm_host(plan_e, host, stream)
            else:
                for m in range(M):
                    ge.micro_sqnorm_host(plan_e, host[m], 0, m, stream)
                ge.mean_sqnorm_host(slice_e, host_mean, stream)
            ge.allreduce(stream)
            ge.finalize(B_g * SEQ_LEN, stream)
            rr = ge.result()
            G.decide(cands, rr.phi if rr.phi_available else None, current, 1000.0, 900.0,
                     reconfig_cost=40.0)

        estep()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            estep()
        b.record(stream)
        torch.cuda.synchronize()
        ems = a.elapsed_time(b) / args.e2e_steps
        if ws > 1:
            tt = torch.tensor([ems], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        ebytes = (plan_e.active_bytes * M + (0 if fused else slice_e.active_bytes)) * ws
        h2d = E * es * M
        if not fused:
            lo_e, hi_e = D.dp_slice(E, d_job, 0)
            h2d += (hi_e - lo_e) * es
        entry = ("coadapt_gns_fused_sqnorm_host (H2D overlapped with the fused reduction)"
                 if fused else "coadapt_gns_micro_sqnorm_host x M + coadapt_gns_mean_sqnorm_host "
                               "of DP slice 0 (H2D overlapped with K1)")
        # the e2e roofline: plain pinned H2D copy rate of this GPU's link,
        # measured with the same buffers (all ranks copying at once)
        hb0 = host[0]
        dbuf = torch.empty_like(hb0, device="cuda")
        with torch.cuda.stream(stream):
            dbuf.copy_(hb0, non_blocking=True)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if ws > 1:
                stream.synchronize()
                dist.barrier()
            c0.record(stream)
            for _ in range(4):
                dbuf.copy_(hb0, non_blocking=True)
            c1.record(stream)
        stream.synchronize()
        h2d_gbs = 4 * hb0.numel() * hb0.element_size() / (c0.elapsed_time(c1) / 1e3) / 1e9
        del dbuf
        if ws > 1:
            tt = torch.tensor([h2d_gbs], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt)  # aggregate over the GPUs
            h2d_gbs = float(tt.item())
        e2e_value = ebytes / (ems / 1e3) / 1e9
        e2e = {"value": round(e2e_value, 3), "unit": UNIT,
               "h2d_peak_gbs": round(h2d_gbs, 1),
               # bytes actually copied per second (all GPUs) / the link rate
               "frac_of_h2d_peak": round(h2d * ws / (ems / 1e3) / 1e9 / h2d_gbs, 4),
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(
                   __import__("ctypes").sizeof(L.GnsResult)),
               "sample": f"first {E} elements of each of the {M} micro-buckets per GPU, "
                         f"pinned host memory -> {entry} -> allreduce -> finalize -> phi D2H "
                         "-> decide"}
        ge.close()
        del host

    # -- CPU baseline (rank 0, N = 1): the oracle on this box's host cores
    cpu = None
    if not args.no_cpu and rank == 0 and ws == 1:
        from oracle import oracle as O
        E = min(numel, 32 << 20)
        hb = [(pool[m][:E].cpu().view(torch.int16).numpy().view(np.uint16) if dt == L.BF16
               else pool[m][:E].cpu().numpy()) for m in range(M)]
        segs_c = [(o, min(n, E - o), w) for o, n, w in mine[0].segments if o < E]
        nth = host_threads()
        rate, nb, passes, el = cpu_oracle_rate(hb, dt, segs_c, args.cpu_seconds, nth)
        # SURVEY 8(d) variant (i): the reference's sequential model, 1 thread,
        # on a quarter of the sample
        hb1 = [b[:E // 4] for b in hb]
        segs_1 = [(o, min(n, E // 4 - o), w) for o, n, w in segs_c if o < E // 4]
        r1, nb1, p1, el1 = cpu_oracle_rate(hb1, dt, segs_1, max(2.0, args.cpu_seconds / 4), 1)
        cpu = {"value": round(rate, 3), "unit": UNIT, "cores": nth, "kind": "port",
               "sample": f"oracle fused fp64 pass over the first {E} elements of the {M} "
                         f"micro-buckets ({nb / 1e9:.2f} GB), {passes} passes in {el:.1f} s",
               "single_thread": {"value": round(r1, 3), "unit": UNIT, "cores": 1,
                                 "sample": f"same pass over the first {E // 4} elements, "
                                           f"{p1} passes in {el1:.1f} s"},
               "cpu": cpu_model()}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": c["dtype"], "data": "synthetic",
                "config": {"workload": workload_name(c), "shape": c["shape"],
                           "job_ranks": R, "ranks_per_gpu": R // ws, "micro_batches": M,
                           "global_batch": B_g, "bytes_per_step": job_bytes,
                           "local_bytes_per_step_rank0": local_bytes,
                           "l2": "inputs >> 126 MB L2 (each bucket streams GBs); no flush needed",
                           "x1": args.x1 if ws > 1 else "local",
                           "pool": ("virtual ranks on one GPU share one resident set of M buckets"
                                    if R // ws > 1 else "one resident set of M buckets per rank")},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "goodput_step": goodput_step,
                "clocks": clk,
                "result": {"phi": r.phi if r.phi_available else None, "b_simple": r.b_simple,
                           "signal": r.stats.signal, "noise": r.stats.noise,
                           "gradient": ("replicated: the virtual ranks on a GPU reduce the same "
                                        "resident buckets, so phi is that of a job whose ranks hold "
                                        "identical shards (the bytes streamed are the job's); the "
                                        "job's own phi is checked against the oracle in "
                                        "tests/test_gpu_fullsize_oracle.py"
                                        if R // ws > 1 else "each rank its own shard")}}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
