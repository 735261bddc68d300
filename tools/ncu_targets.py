"""One launch of each auxiliary kernel, for a single-GPU `ncu --set full`
capture (profiles/r01b_ncu_aux_*.csv):
  KA accumulate_kernel  (trainer form: 1 Gi bf16 grads into fp32 main_grad, s_m fused)
  KR rs_kernel          (reduce-scatter + gbar^2, d = 2 replicas both local)
  KX reshard_copy_kernel (TP (1,2,1) -> PP (1,1,2) of 4 x 8192^2 bf16, virtual ranks)
Each is launched once after a warm-up launch (ncu: -k regex:... -s 1 -c 1)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26687_b200 import _lib as L  # noqa: E402
from paper_2604_26687_b200 import device as D  # noqa: E402
from paper_2604_26687_b200 import reshard as R  # noqa: E402


def main():
    torch.cuda.set_device(0)
    n = 1 << 30
    g = D.GnsDevice(2, 2, 4, 0)
    plan = D.BucketPlan([(0, n, 1.0)], n, L.BF16, 0)
    grad = torch.randn(n, device="cuda").to(torch.bfloat16)
    main_grad = torch.zeros(n, dtype=torch.float32, device="cuda")
    for _ in range(2):  # KA
        g.begin_step()
        g.accumulate(plan, main_grad, grad, 0, 0, first=True)
    rep = [grad, torch.randn(n, device="cuda").to(torch.bfloat16)]
    lo, hi = D.dp_slice(n, 2, 0)
    out = torch.empty(hi - lo, dtype=torch.bfloat16, device="cuda")
    for _ in range(2):  # KR
        g.begin_step()
        g.reduce_scatter_sqnorm(plan, rep, 0, out, 0.5)
    T = R.TensorDecl
    m = R.ModelSpec(2, (T("w", (8192, 8192), 0), T("o", (8192, 8192), 1)))
    p = R.plan_transfers(m, (1, 2, 1), (1, 1, 2))
    src = [torch.randint(-100, 100, (p.pack_numel(R.SRC, r),), dtype=torch.int16, device="cuda")
           for r in range(2)]
    dst = [torch.zeros(p.pack_numel(R.DST, r), dtype=torch.int16, device="cuda") for r in range(2)]
    for _ in range(2):  # KX
        p.execute(src, dst)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
