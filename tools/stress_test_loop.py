"""Run one GPU parity test function repeatedly in one process (flake hunt)."""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import test_gpu_parity as T  # noqa: E402
from paper_2604_26687_b200 import _lib as L  # noqa: E402
from paper_2604_26687_b200 import device as D  # noqa: E402

torch.cuda.set_device(0)
name = sys.argv[1]
reps = int(sys.argv[2])
fails = 0
for r in range(reps):
    for M in (3, 4):
        try:
            getattr(T, name)(D, L, M)
        except AssertionError as e:
            fails += 1
            print("FAIL rep", r, "M", M, str(e)[:300], flush=True)
print("fails", fails, "of", 2 * reps, flush=True)
