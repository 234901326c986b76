"""Map which (B, L, scatter, tile) cases fail: each case in its own process."""
import subprocess
import sys

cases = []
for B in (20, 24, 40, 44, 52, 100):
    for L in (1, 2, 4):
        for sc in (1,):
            for T in (0, 512, 1024):
                cases.append((B, L, sc, T))
code = r'''
import sys; sys.path.insert(0, ".")
import synth
from paper_2605_30294_b200 import rafi
B, L, sc, T = map(int, sys.argv[1:5])
n = 20001
ctx = rafi.Context(B, n * L, local_ranks=L, device=0)
ctx.set_option(rafi.OPT_SCATTER, sc)
if T: ctx.set_option(rafi.OPT_TILE, T)
for l in range(L):
    ctx.drv_emit_synthetic(synth.PATTERNS["uniform"], 17, 0, n, local=l)
print(ctx.forward(), ctx.get_option(rafi.OPT_TILE))
'''
for c in cases:
    r = subprocess.run([sys.executable, "-c", code] + [str(x) for x in c], capture_output=True, text=True)
    out = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr.strip().splitlines()[-1][-80:]
    print(c, "ok" if r.returncode == 0 else "FAIL", out, flush=True)
