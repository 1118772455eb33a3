"""Dev tool (GPU box): first difference between the tiled batched refactorization and the oracle on a
committed fixture."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2306_14337_b200 as rlu
from paper_2306_14337_b200.batch import BatchedFactors
from tests.fixtures import golden_fixture

name = sys.argv[1] if len(sys.argv) > 1 else "kkt_small"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 3
fx = golden_fixture(name)
vals = np.stack([fx.values[k % len(fx.values)] for k in range(B)])
f = BatchedFactors(fx.sym, B)
print("info", {k: v for k, v in f.info.items() if k in ("tiled", "tile_rows", "blocks", "blocked_rows", "tile_smem_bytes", "tile_grid")})
failed = f.refactorize(vals, raise_on_zero_pivot=False)
print("failed rows", failed)
ro, dp = fx.sym.row_offsets, fx.sym.diag_pos
for s in range(B):
    ref, _ = fx.oracle.factorize(vals[s])
    got = f.values(s)
    bad = np.nonzero(~((got == ref) | (np.isnan(got) & np.isnan(ref))))[0]
    if bad.size == 0:
        print("scenario", s, "bitwise equal")
        continue
    rows = np.searchsorted(ro, bad, side="right") - 1
    print("scenario", s, "differing entries", bad.size, "rows", np.unique(rows)[:20], "first entry", bad[0], "row", rows[0],
          "offset in row", bad[0] - ro[rows[0]], "row len", ro[rows[0] + 1] - ro[rows[0]], "nl", dp[rows[0]] - ro[rows[0]],
          "got", got[bad[0]], "ref", ref[bad[0]])
f.close()
