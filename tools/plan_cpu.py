"""Host-only plan statistics for an N=L=n operator with the REAL Gaunt table and a
synthetic slot-symmetric R (no GPU needed): prints the plan's packing report.
Usage: BFQ_PLAN_STATS=2 python tools/plan_cpu.py 16"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2605_28475_b200 import engine, rbuild  # noqa: E402
from paper_2605_28475_b200.operator import FactorizedOperator, RTensor, SpectralConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = SpectralConfig(n, n, 1.0)
g = rbuild.build_gaunt_coo(cfg.l_max)
nk, nt = cfg.n_k, g.channels.n_t
rng = np.random.default_rng(1)
r = rng.standard_normal((nk, nk, nk, nt))
sw = np.array([g.channels.tau(l1, l3, l2) - 1 for (l1, l2, l3) in g.channels.triplets])
r = 0.5 * (r + r.transpose(0, 2, 1, 3)[..., sw])  # R[k,a,b,tau] = R[k,b,a,tau']
op = FactorizedOperator(RTensor(np.ascontiguousarray(r), g.channels, 1.0), g, cfg)
print(engine.host_plan_info(op))
