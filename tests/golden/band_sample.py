"""One perturbed reference solve for the iteration band of an ill-conditioned
full-size case (make_fullsize.py band_iterations, one sample per process so
the band can be widened in parallel).  Prints one JSON line.

python tests/golden/band_sample.py <case> <level|color> <op|factor> <seed> [maxit]
python tests/golden/band_sample.py --merge <full_*.npz> <plan> <result files...>
(C3 colour: seeds 11-13, op and factor, widened the fixture's band)
Test infrastructure; run in the build container only."""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

import numpy as np  # noqa: E402

from make_fullsize import CASES, bs, ref_matrix  # noqa: E402


def main(case, plan, kind, seed, maxit=200, tol=1e-8):
    a, rhs = ref_matrix(CASES[case]())
    p = bs.level_schedule(a.pattern) if plan == "level" else bs.graph_color(a.pattern)
    f = bs.decompose(a, p)
    rng = np.random.default_rng(seed)
    op = bs.MatrixOperator(a)
    if kind == "op":
        base = op.apply_array
        op.apply_array = lambda v: (lambda y: y * (1.0 + 1e-15 * rng.standard_normal(y.shape)))(base(v))
    else:
        for ph in (f._forward, f._backward):
            ph.blocks[:] *= 1.0 + 1e-14 * rng.standard_normal(ph.blocks.shape)
        f._diag_bwd[:] *= 1.0 + 1e-14 * rng.standard_normal(f._diag_bwd.shape)
    _, rep = bs.bicgstab(op, f, rhs, stop=bs.StoppingCriteria(tol, maxit))
    print(json.dumps({"case": case, "plan": plan, "kind": kind, "seed": seed,
                      "iterations": rep.iterations, "converged": bool(rep.converged)}), flush=True)


def merge(npz_name, plan, files):
    """Widen <plan>_band of tests/golden/<npz_name> with band_sample.py
    results (JSON lines in files)."""
    p = HERE / npz_name
    with np.load(p) as z:
        d = {k: z[k] for k in z.files}
    its = [float(v) for v in d[f"{plan}_band"]]
    extra = 0
    for fn in files:
        for ln in open(fn):
            if ln.startswith("{"):
                its.append(float(json.loads(ln)["iterations"]))
                extra += 1
    d[f"{plan}_band"] = np.array([min(its), max(its)])
    # the fixture's band came from 1 + 2 x 3 solves (make_fullsize.py --band 3)
    d[f"{plan}_band_samples"] = np.array(int(d.get(f"{plan}_band_samples", 7)) + extra)
    np.savez_compressed(p, **d)
    print(npz_name, plan, d[f"{plan}_band"])


if __name__ == "__main__":
    a = sys.argv[1:]
    if a[0] == "--merge":      # --merge <npz> <plan> <json files...>
        merge(a[1], a[2], a[3:])
    else:
        main(a[0], a[1], a[2], int(a[3]), int(a[4]) if len(a) > 4 else 200)
