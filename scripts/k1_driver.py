"""K1 (build_weight_table) on the c3 weights for ncu: the single-pass
(deferred) build and the two-pass build, three of each, L2 flushed before
every build.  Usage: python scripts/k1_driver.py [cfg]"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2604_01356_b200 as drs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = torch.from_numpy(bench.make_weights(cfg)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for deferred in (True, False):
    for r in range(3):
        flush.fill_(r)
        drs.build_weight_table(w, check=False, deferred=deferred)
torch.cuda.synchronize()
print("k1 driver done")
