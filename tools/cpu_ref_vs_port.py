"""Build container only (needs /root/reference): time the reference's own
evaluate(op, c, "angular_first") against the oracle port (the bench's CPU arm
on the GPU box) on the same cells, one thread each, to show the port is a
faithful stand-in for the reference's CPU speed.  Writes one JSON line per
operator."""
import json
import os
import sys
import time

import numpy as np
from threadpoolctl import threadpool_limits

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from boltzfact import basis, cache, contraction  # noqa: E402

from oracle import q_oracle  # noqa: E402
from paper_2605_28475_b200 import inputs  # noqa: E402
from paper_2605_28475_b200.operator import load_cache  # noqa: E402

for name, n in (("hs_n8", 8), ("hs_n12", 3)):
    path = os.path.join(ROOT, "operators", name + ".bfct")
    ref_op = cache.load_cache(path)
    our = q_oracle.OracleOperator.from_operator(load_cache(path))
    ws = q_oracle.angular_workspace(our)
    cfg = ref_op.cfg
    cells = inputs.perturbed_maxwellians(cfg.k_max + 1, cfg.l_max, n, seed=3)
    with threadpool_limits(limits=1):
        contraction.evaluate(ref_op, basis.CoefficientField(cells[0].copy(), cfg))  # warm caches
        q_oracle.q_angular_first(our, cells[0], workspace=ws)
        t0 = time.perf_counter()
        ref = [contraction.evaluate(ref_op, basis.CoefficientField(c.copy(), cfg)).values for c in cells]
        t_ref = (time.perf_counter() - t0) / n
        t0 = time.perf_counter()
        port = [q_oracle.q_angular_first(our, c, workspace=ws) for c in cells]
        t_port = (time.perf_counter() - t0) / n
    err = max(q_oracle.rel_err(p, r) for p, r in zip(port, ref))
    print(json.dumps({"operator": name, "cells": n, "threads": 1, "reference_s_per_cell": t_ref,
                      "port_s_per_cell": t_port, "port_over_reference_time": t_port / t_ref,
                      "max_rel_diff": err}), flush=True)
