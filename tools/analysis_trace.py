"""Timeline of the sync-free level / colour kernels on C4: each row's
publication time against its level (the DAG depth the wavefront follows)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402

a = P.generate(P.GeneratorSpec(100, 100, 100, seed=0)).a
pat = D.DevPattern.upload(a.pattern)
n = pat.n
lev = P.level_schedule(a.pattern).row_group
g = torch.empty(n, dtype=torch.int32, device="cuda")
tr = torch.zeros(n, dtype=torch.int64, device="cuda")
for kind, name in ((0, "level"), (1, "color")):
    for _ in range(2):
        D.lib().b2s_analysis_trace(kind, n, pat.rp.data_ptr(), pat.ci.data_ptr(), g.data_ptr(),
                                   tr.data_ptr(), D.stream())
    t = tr.cpu().numpy()
    t = (t - t.min()) / 1e3
    L = lev.max() + 1
    done = np.full(L, -1.0)
    first = np.full(L, 1e18)
    np.maximum.at(done, lev, t)
    np.minimum.at(first, lev, t)
    print(json.dumps({"kernel": name, "total_us": float(t.max()),
                      "level_done_us": [round(float(done[q]), 1) for q in range(0, L, 20)],
                      "level_first_us": [round(float(first[q]), 1) for q in range(0, L, 20)],
                      "rows_done_at_us": {str(q): int((t <= q).sum()) for q in (100, 200, 400, 800, 1200)}}))
