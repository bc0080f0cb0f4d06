"""Small Q(f,f) launches for compute-sanitizer (racecheck / synccheck / memcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_q.py --op hs_n12 --cells 8

Runs the folded Q(f,f) kernel, the bilinear Q(f2,f3) kernel and one RK4 step
on a few cells of one operator, then checks the result against the oracle so a
sanitizer-perturbed schedule that changes the numbers is also caught.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import q_oracle  # noqa: E402
from paper_2605_28475_b200 import engine, inputs  # noqa: E402
from paper_2605_28475_b200.operator import load_cache  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--op", default="hs_n4")
ap.add_argument("--cells", type=int, default=8)
ap.add_argument("--no-check", action="store_true")
a = ap.parse_args()

op = load_cache(os.path.join(ROOT, "operators", a.op + ".bfct"))
cfg = op.cfg
cells = inputs.perturbed_maxwellians(cfg.n_k, cfg.l_max, a.cells, seed=3)
f = torch.from_numpy(cells).cuda()
f3 = torch.from_numpy(inputs.perturbed_maxwellians(cfg.n_k, cfg.l_max, a.cells, seed=4)).cuda()
plan = engine.plan_for(op)
print("plan", plan.info, flush=True)
q = engine.evaluate_batch(plan, f)
q12 = engine.evaluate_batch(plan, f, f3)
y = f.clone()
work = torch.empty((3,) + tuple(f.shape), dtype=torch.float64, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
plan.rk4_step_device(y.data_ptr(), work.data_ptr(), a.cells, 0.01, flag.data_ptr(),
                     torch.cuda.current_stream().cuda_stream)
mom = torch.empty((a.cells, 5), dtype=torch.float64, device="cuda")
plan.moments_device(q.data_ptr(), mom.data_ptr(), a.cells, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
if not a.no_check:
    oop = q_oracle.OracleOperator.from_operator(op)
    ws = q_oracle.angular_workspace(oop)
    qh, q12h = q.cpu().numpy(), q12.cpu().numpy()
    f3h = f3.cpu().numpy()
    for i in (0, a.cells - 1):
        e1 = q_oracle.rel_err(qh[i], q_oracle.q_angular_first(oop, cells[i], workspace=ws))
        e2 = q_oracle.rel_err(q12h[i], q_oracle.q_angular_first(oop, cells[i], f3h[i], workspace=ws))
        print(f"cell {i}: rel err Q(f,f) {e1:.2e}  Q(f2,f3) {e2:.2e}")
        assert e1 <= 1e-12 and e2 <= 1e-12
    assert int(flag.item()) == 0
    assert float(mom.abs().max()) == 0.0
print("sanitize_q ok", a.op, a.cells, os.environ.get("BFQ_KERNEL", "2"))
