"""Phase timestamps of the fused softmax-loss kernel (CTA 0), on a library
built with -DMPC3_LOSS_TRACE (tools/dbg/build_variant.sh losstrace
-DMPC3_LOSS_TRACE; run through tools/dbg/run_variants.sh)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import rss as R  # noqa: E402
from paper_2104_10949_b200 import _capi  # noqa: E402
from paper_2104_10949_b200.engine import TrioSession  # noqa: E402

rows, d = 128, 10
rng = np.random.default_rng(0)
z = R.share(R.fx_encode(rng.uniform(-6, 6, (rows, d))), rng)
y = R.share(R.fx_encode(np.eye(d)[rng.integers(0, d, rows)]), rng)
s = TrioSession(1)
zs, ys = s.from_components(z), s.from_components(y)
phases = [None, "table set-up", "max_tree", "x = z - max", "exp chain", "row sum", "reciprocal",
          "mul + truncate - y"]
acc = np.zeros(16)
for it in range(6):
    s.softmax_loss(zs, ys)
    torch.cuda.synchronize()
    t = (C.c_ulonglong * 16)()
    assert _capi.lib().mpc3_dbg_loss_trace(t) == 0
    if it >= 1:
        acc += np.array(t[:], dtype=np.float64) - t[0]
acc /= 5
for k in range(1, 8):
    print(f"{phases[k]:20s} {(acc[k] - acc[k - 1]) / 1e3:7.2f} us")
print(f"{'total (CTA 0)':20s} {acc[7] / 1e3:7.2f} us")
if 0 < acc[8] < acc[2]:  # the per-level fill path only (the up-front fill skips these marks)
  print("max_tree level 0:", ", ".join(f"{nm} {(acc[b] - acc[a]) / 1e3:.2f} us" for nm, a, b in
                                   (("streams + head constants", 1, 8), ("keystream fill", 8, 9), ("circuit", 9, 10),
                                    ("odd column", 10, 11))))
