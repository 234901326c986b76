"""Debug: one forward at the given item size / local ranks (THREADS scatter)."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2605_30294_b200 import rafi  # noqa: E402

B, L, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ctx = rafi.Context(B, n * L, local_ranks=L, device=0)
for l in range(L):
    ctx.drv_emit_synthetic(synth.PATTERNS["uniform"], 17, 0, n, local=l)
print("G", ctx.forward())
