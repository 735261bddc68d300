"""Concurrent pinned H2D rate of every GPU of the box, with and without
binding each rank's process (and so its pinned host pages, first-touched by
that process) to the CPUs NVML reports as local to its GPU.  torchrun, one
rank per GPU; rank 0 prints one JSON line.  Probe for bench.py's e2e leg at
N > 1 (profiles/r02_h2d_numa.txt)."""
import json
import os
import sys

import torch
import torch.distributed as dist


def gpu_cpus(index: int):
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(index)
    words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
    cpus = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
    node = None
    try:
        node = pynvml.nvmlDeviceGetNumaNodeId(h)
    except Exception:
        pass
    return cpus, node


def rate(local: int, ws: int, n: int, reps: int = 6) -> float:
    h = torch.empty(n, dtype=torch.uint8)
    h.fill_(1)  # first touch by this process (its current CPU set)
    h = h.pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    return reps * n / (a.elapsed_time(b) / 1e3) / 1e9


def main():
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    cpus, node = gpu_cpus(local)
    if os.environ.get("BIND") == "1" and cpus:
        os.sched_setaffinity(0, cpus)
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    r = rate(local, ws, 2 << 30)
    t = torch.tensor([r], dtype=torch.float64, device="cuda")
    allr = [torch.zeros_like(t) for _ in range(ws)]
    dist.all_gather(allr, t)
    info = [None] * ws
    dist.all_gather_object(info, {"gpu": local, "numa": node, "cpus": f"{cpus[0]}-{cpus[-1]}" if cpus else None,
                                  "n_cpus": len(cpus)})
    if rank == 0:
        per = [round(float(x.item()), 1) for x in allr]
        print(json.dumps({"world": ws, "bind": os.environ.get("BIND") == "1", "per_gpu_gbs": per,
                          "sum_gbs": round(sum(per), 1), "topology": info}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
