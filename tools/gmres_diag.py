"""configs[4] GMRES diagnostics (run on the GPU box from the repo root):

    python tools/gmres_diag.py --precond 0 --max-iter 1000 --out gpurun_out/diag.json

One solve of the metamaterial-cell mixed BVP with the residual history of bem_gmres_history
(Arnoldi estimate per iteration, true |b - A x| / |b| at every restart), plus a linearity
probe of the operator through bem_apply: eps = |A(x + y) - A x - A y| / |A(x + y)| for the
solution x and a random y of the same norm (the rounding noise that no Krylov method can
get under), and the amplification |A x| ... |x| / |b| that turns it into a residual floor.
Environment switches of the library (EBEM_BEM_PRECISE_M2L, ...) are passed through."""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precond", type=int, default=0)
    ap.add_argument("--restart", type=int, default=50)
    ap.add_argument("--max-iter", type=int, default=1000)
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--nc", type=int, default=160)
    ap.add_argument("--level", type=int, default=5)
    ap.add_argument("--voids", type=int, default=64)
    ap.add_argument("--max-pts", type=int, default=1536)
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--probe", type=int, default=1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    import paper_1612_04082_b200 as eb
    from workloads import geometry as geo
    d = geo.metamaterial_cell(nc=a.nc, level=a.level, nvoids=a.voids)
    verts = torch.from_numpy(d["verts"]).cuda()
    bc = torch.from_numpy(d["bc_type"]).cuda()
    val = torch.from_numpy(d["bc_val"]).cuda()
    op = eb.bem_create(verts, nq=16, max_pts=a.max_pts, p=a.p, K=d["K"], G=d["G"])
    x = torch.zeros((d["verts"].shape[0], 3), device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, it, res = eb.bem_gmres_solve(op, bc, val, x, restart=a.restart, max_iter=a.max_iter, tol=a.tol,
                                    precond=a.precond, check=False)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    est, true = eb.bem_gmres_history(op)
    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("EBEM_")}, "precond": a.precond,
           "restart": a.restart, "max_iter": a.max_iter, "tol": a.tol, "npanels": int(d["verts"].shape[0]),
           "iterations": it, "rel_residual": res, "solve_s": sec, "true_at_restarts": true.tolist(),
           # per cycle: the lowest Arnoldi estimate reached inside it
           "cycle_min_estimate": [float(est[k:k + a.restart].min()) for k in range(0, len(est), a.restart)],
           "estimate_every_10": est[::10].tolist()}
    if a.probe:
        b = eb.bem_rhs(op, bc, val)
        torch.manual_seed(0)
        y = torch.randn_like(x)
        y *= x.norm() / y.norm()
        Ax, Ay, Axy = (eb.bem_apply(op, bc, v) for v in (x, y, x + y))
        r = (-b.double()) - Ax.double()          # bem_rhs returns -b with the sign of Eq. num2's right side
        r2 = b.double() - Ax.double()
        out["probe"] = {
            "eps_linearity": float(((Axy.double() - Ax.double() - Ay.double()).norm() / Axy.double().norm()).item()),
            "norm_b": float(b.double().norm().item()), "norm_x": float(x.double().norm().item()),
            "norm_Ax": float(Ax.double().norm().item()), "norm_Ay": float(Ay.double().norm().item()),
            "resid_bem_apply_minus": float((r.norm() / b.double().norm()).item()),
            "resid_bem_apply_plus": float((r2.norm() / b.double().norm()).item())}
    s = json.dumps(out)
    print(s, flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    main()
