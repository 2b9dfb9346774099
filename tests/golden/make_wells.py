"""Golden fixtures for wells from the
UNMODIFIED reference: generator wells, separate well application
(WellAugmentedOperator), coupled folding (fold_into_matrix) and
solve_with_fallback in both well modes.

Run in the build container only:  python tests/golden/make_wells.py
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent

import numpy as np  # noqa: E402

import blocksolve as bs  # noqa: E402
from blocksolve.io import GeneratorSpec, generate  # noqa: E402
from blocksolve.krylov import WellAugmentedOperator  # noqa: E402
from blocksolve.wells import WellMode, fold_into_matrix  # noqa: E402

CASES = {
    "wells_std_8x7x5": dict(nx=8, ny=7, nz=5, well_count=3, well_kind="standard", seed=4),
    "wells_ms_8x7x5": dict(nx=8, ny=7, nz=5, well_count=2, well_kind="multisegment", seed=5),
    "wells_std_b2_6x6x4": dict(nx=6, ny=6, nz=4, block_size=2, well_count=2,
                               well_kind="standard", well_depth=4, seed=6),
}


def main():
    rng = np.random.default_rng(99)
    for name, kw in CASES.items():
        g = generate(GeneratorSpec(**kw))
        a, rhs, wells = g.a, g.rhs, g.wells
        out = {"rp": a.pattern.row_pointers, "ci": a.pattern.column_indices, "vals": a.values,
               "rhs": rhs.data, "b": np.array(a.block_size)}
        for k, w in enumerate(wells.standard):
            out[f"std{k}_cells"] = w.perforated_cells
            out[f"std{k}_b"] = w.b_blocks
            out[f"std{k}_c"] = w.c_blocks
            out[f"std{k}_dinv"] = w.d_inverse
        for k, w in enumerate(wells.multisegment):
            out[f"ms{k}_cells"] = w.b_cells
            out[f"ms{k}_b"] = w.b_blocks
            out[f"ms{k}_c"] = w.c_blocks
            out[f"ms{k}_d"] = w.d_dense
        x = rng.uniform(-1, 1, size=rhs.data.size)
        out["x"] = x
        out["op_x"] = WellAugmentedOperator(a, wells).apply_array(x)
        f = fold_into_matrix(a, wells)
        out["fold_rp"], out["fold_ci"], out["fold_vals"] = (f.pattern.row_pointers,
                                                            f.pattern.column_indices, f.values)
        for mode in (WellMode.SEPARATE, WellMode.COUPLED):
            for backend in (bs.Backend.LEVEL_SCHEDULED, bs.Backend.GRAPH_COLORED):
                cfg = bs.SolverConfig(backend=backend, well_mode=mode,
                                      stop=bs.StoppingCriteria(1e-8, 200))
                xs, rep = bs.solve_with_fallback(cfg, a, rhs, wells)
                tag = f"{mode.value}_{backend.value}"
                out[f"{tag}_x"] = xs.data
                out[f"{tag}_report"] = np.array([rep.converged, rep.iterations,
                                                 rep.initial_norm, rep.final_norm,
                                                 rep.fallback_used])
        np.savez_compressed(OUT / f"{name}.npz", **out)
        print(name, {k: v for k, v in out.items() if k.endswith("_report")})


if __name__ == "__main__":
    main()
