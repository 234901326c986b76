"""Binning at R logical ranks on one GPU (measurement helper, not product).

    python scripts/prof_binning.py [--L 8] [--n 16777216] [--B 48] [--tiles 256,512,...]
        [--scatter auto|threads|bulk] [--steps 5] [--warmup 2]

For each tile size: forwards the whole L-rank world (FUSED into local queues)
with RAFI_OPT_TIMING and prints one JSON line per tile with the histogram,
scan and scatter times and their HBM GB/s (algorithmic 2B+8 bytes per item).
Used for tile sweeps and as the target program of ncu captures.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
from paper_2605_30294_b200 import rafi  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--L", type=int, default=8)
    p.add_argument("--n", type=int, default=16 * 1024 * 1024)
    p.add_argument("--B", type=int, default=48)
    p.add_argument("--tiles", default="0")
    p.add_argument("--scatter", default="auto", choices=["auto", "threads", "bulk"])
    p.add_argument("--pattern", default="uniform")
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=2)
    a = p.parse_args()
    import torch
    torch.cuda.set_device(0)
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6457.1
    s = torch.cuda.Stream()
    ctx = rafi.Context(a.B, a.n + a.n // 8, stream=s, local_ranks=a.L)
    if a.scatter != "auto":
        ctx.set_option(rafi.OPT_SCATTER, {"threads": rafi.SCATTER_THREADS, "bulk": rafi.SCATTER_BULK}[a.scatter])
    for tile in [int(t) for t in a.tiles.split(",")]:
        try:
            ctx.set_option(rafi.OPT_TILE, tile)
        except rafi.RafiError as e:
            print(json.dumps({"tile": tile, "error": str(e)}))
            continue
        for k in range(a.warmup + a.steps):
            if k == a.warmup:
                ctx.set_option(rafi.OPT_TIMING, 1)
            for l in range(a.L):
                ctx.drv_emit_synthetic(synth.PATTERNS[a.pattern], synth.CONFIG_SEEDS[2], k, a.n, local=l)
            ctx.forward()
        st = ctx.stats()
        K = st["acc_forwards"]
        ph = {q: st["acc_ms_" + q] / K for q in ("hist", "scan", "count_exchange", "scatter")}
        items = a.L * a.n
        tot = sum(ph.values())
        print(json.dumps({"tile": ctx.get_option(rafi.OPT_TILE), "L": a.L, "n": a.n, "B": a.B,
                          "scatter": {1: "threads", 2: "bulk"}[ctx.get_option(rafi.OPT_SCATTER)], "ms": ph,
                          "binning_gbs": items * (2 * a.B + 8) / (tot / 1e3) / 1e9,
                          "binning_frac": items * (2 * a.B + 8) / (tot / 1e3) / 1e9 / peak,
                          "scatter_frac": items * (2 * a.B + 4) / (ph["scatter"] / 1e3) / 1e9 / peak,
                          "hist_frac": items * 4 / (ph["hist"] / 1e3) / 1e9 / peak}), flush=True)
        ctx.set_option(rafi.OPT_TIMING, 0)
    ctx.close()


if __name__ == "__main__":
    main()
