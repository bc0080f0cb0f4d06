import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np, torch
from project_funcs import FUNCS
from paper_2605_28475_b200 import project as gp
from paper_2605_28475_b200.operator import SpectralConfig
from oracle.project_oracle import ProjectionOracle

def rel(a, b): return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
l_max, order = int(sys.argv[1]), int(sys.argv[2])
cfg = SpectralConfig(3, l_max, 1.0)
pts = gp.project_points(cfg, order)
names = sorted(FUNCS)
base = FUNCS[names[0]](pts)
rng = np.random.default_rng(0)
pf = gp.Projector(cfg, order)
os.environ["BFQ_PROJ_NOFOLD"] = "1"
pu = gp.Projector(cfg, order)
print("kernels", pf.kernel, pu.kernel, "grid", pf.n_v, pf.n_t, pf.n_p)
orc = ProjectionOracle(cfg.k_max, cfg.l_max, gp.projection_grid(cfg.l_max, order))
cases = {"f0": base, "rev": base[::-1].copy(), "rand": rng.standard_normal(base.size)}
nv, nt, npp = pf.n_v, pf.n_t, pf.n_p
for v in (0, nv // 2, nv - 1):
    for t in (0, 17, nt - 1):
        x = np.zeros((nv, nt, npp)); x[v, t] = rng.standard_normal(npp); cases[f"v{v}t{t}"] = x.reshape(-1)
for name, h in cases.items():
    s = torch.from_numpy(h[None].copy()).cuda()
    a = pf.project(s).cpu().numpy()[0]; b = pu.project(s).cpu().numpy()[0]; r = orc.project(h)
    print(f"{name:10s} fold-vs-oracle {rel(a, r):.2e}  nofold-vs-oracle {rel(b, r):.2e}  fold-vs-nofold {rel(a, b):.2e}")
