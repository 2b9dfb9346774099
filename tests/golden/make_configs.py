"""Golden fixtures for the BASELINE configs the reference generator cannot
express (C2 masked / NORNE-like, C3 heterogeneous), computed by the
UNMODIFIED reference package on systems built by this repo's seeded
harness generators (paper_2309_11488_b200/synthetic.py, pure numpy).

Run in the build container only (the reference is absent on the GPU box):
    python tests/golden/make_configs.py [--full]
Small systems get the full pipeline (plans, factors, apply, solves); the
full-size C2 system (47,605 cells) gets a compact digest: plan arrays,
iteration counts, norms and x.  ``--full`` also runs the full-size C3
system (350,336 cells) through the reference (minutes) and stores its
report plus a perturbation band (factors scaled by 1 + 1e-14 N(0,1)).
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import blocksolve as bs  # noqa: E402
from make_golden import system_case  # noqa: E402

from paper_2309_11488_b200 import synthetic as S  # noqa: E402

C2 = dict(nx=46, ny=112, nz=22, seed=2309)
C3 = dict(nx=92, ny=224, nz=17, sigma_k=1.0, diagonal_boost=1e-2)
C3_TOL = 1e-8


def ref_matrix(bundle):
    a = bundle.a
    p = bs.SparsityPattern(a.num_block_rows, a.pattern.row_pointers, a.pattern.column_indices)
    return bs.BlockMatrix(p, a.block_size, a.values.copy()), bs.BlockVector(bundle.rhs.data.copy(),
                                                                           a.block_size)


def small_cases():
    m = S.generate_masked(14, 16, 8, seed=11)
    a, rhs = ref_matrix(m)
    system_case("masked_14x16x8", a, rhs, strategies=("level", "color"))
    h = S.generate_heterogeneous(10, 12, 6, sigma_k=1.5, diagonal_boost=1e-3, seed=3)
    a, rhs = ref_matrix(h)
    system_case("hetero_10x12x6", a, rhs, strategies=("level", "color"))


def digest(name, bundle, tol, plans=("level", "color"), band=0):
    a, rhs = ref_matrix(bundle)
    out = {"n": np.array(a.num_block_rows), "nnzb": np.array(a.pattern.num_blocks)}
    meta = {}
    for s in plans:
        t0 = time.time()
        plan = bs.level_schedule(a.pattern) if s == "level" else bs.graph_color(a.pattern)
        out[f"{s}_row_group"] = plan.row_group.astype(np.int32)
        f = bs.decompose(a, plan)
        out[f"{s}_invd_norm"] = np.array(np.linalg.norm(f.inverted_diagonals))
        out[f"{s}_lu_norm"] = np.array(np.linalg.norm(f.combined.values))
        x, rep = bs.bicgstab(bs.MatrixOperator(a), f, rhs, stop=bs.StoppingCriteria(tol, 200))
        out[f"{s}_report"] = np.array([rep.converged, rep.iterations, rep.initial_norm,
                                       rep.final_norm])
        if x.data.size <= 300_000:
            out[f"{s}_x"] = x.data
        else:   # large systems: a fixed random sample of the solution + its norm
            idx = np.random.default_rng(7).choice(x.data.size, 4096, replace=False)
            out["x_idx"] = idx
            out[f"{s}_x_sample"] = x.data[idx]
            out[f"{s}_x_norm"] = np.array(np.linalg.norm(x.data))
        its = [rep.iterations]
        rng = np.random.default_rng(1234)
        # the reference's own spread under rounding-level perturbations: an
        # operator whose results carry 1e-15 relative noise (what a different
        # summation order does) ...
        for _ in range(band):
            op = bs.MatrixOperator(a)
            base = op.apply_array

            def noisy(v, base=base):
                y = base(v)
                return y * (1.0 + 1e-15 * rng.standard_normal(y.shape))
            op.apply_array = noisy
            _, r2 = bs.bicgstab(op, f, rhs, stop=bs.StoppingCriteria(tol, 200))
            its.append(r2.iterations)
        # ... and factors scaled by 1 + 1e-14 N(0,1)
        for _ in range(band):   # the reference's own iteration spread under factor noise
            for ph in (f._forward, f._backward):   # what the apply reads
                ph.blocks[:] *= 1.0 + 1e-14 * rng.standard_normal(ph.blocks.shape)
            f._diag_bwd[:] *= 1.0 + 1e-14 * rng.standard_normal(f._diag_bwd.shape)
            _, r2 = bs.bicgstab(bs.MatrixOperator(a), f, rhs, stop=bs.StoppingCriteria(tol, 200))
            its.append(r2.iterations)
        out[f"{s}_band"] = np.array([min(its), max(its)])
        meta[s] = {"iterations": rep.iterations, "band": [min(its), max(its)],
                   "seconds": round(time.time() - t0, 1)}
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, json.dumps(meta))


def c4_digest():
    """C4 (100^3, reference generator): the reference's own iteration counts
    and solution samples for both plans (its per-row loops take minutes)."""
    from blocksolve.io import GeneratorSpec, generate
    g = generate(GeneratorSpec(100, 100, 100, seed=0))
    out, meta = {}, {}
    idx = np.random.default_rng(7).choice(g.rhs.data.size, 4096, replace=False)
    out["x_idx"] = idx
    for s in ("level", "color"):
        t0 = time.time()
        plan = bs.level_schedule(g.a.pattern) if s == "level" else bs.graph_color(g.a.pattern)
        f = bs.decompose(g.a, plan)
        x, rep = bs.bicgstab(bs.MatrixOperator(g.a), f, g.rhs, stop=bs.StoppingCriteria(1e-8, 200))
        out[f"{s}_report"] = np.array([rep.converged, rep.iterations, rep.initial_norm,
                                       rep.final_norm])
        out[f"{s}_x_sample"] = x.data[idx]
        out[f"{s}_x_norm"] = np.array(np.linalg.norm(x.data))
        out[f"{s}_groups"] = np.array(plan.group_count)
        meta[s] = {"iterations": rep.iterations, "seconds": round(time.time() - t0, 1)}
    np.savez_compressed(HERE / "c4_digest.npz", **out)
    print("c4_digest", json.dumps(meta))


def main():
    if "--c4" in sys.argv:
        return c4_digest()
    if "--c3-only" not in sys.argv:
        small_cases()
        digest("c2_masked_digest", S.generate_masked(**C2), 1e-8)
    if "--full" in sys.argv or "--c3-only" in sys.argv:
        digest("c3_hetero_digest", S.generate_heterogeneous(**C3), C3_TOL, plans=("level",),
               band=3)


if __name__ == "__main__":
    main()
