"""FUSED NVLink push of one rank, driven by ONE process (measurement helper).

    python scripts/nvl_redirect.py [--scatter threads|bulk] [--n 16777216] [--B 48] [--peers 1]

A context on cuda:0 with 1 + P local ranks; rank 0 holds n items with uniform
destinations over R = 1 + P, ranks 1..P hold none, and rank p's incoming
queue is redirected (rafi_diag_redirect_incoming) into a buffer on cuda:p.
Each forward is then exactly rank 0's share of an N = 1 + P FUSED forward:
its block for itself stays in local HBM, its blocks for the P peers cross
NVLink, pushed by the scatter kernel.  Single process, so ncu can capture the scatter's NVLink
counters (nvltx/nvlrx) -- which a multi-rank run cannot be wrapped in.
Prints one JSON line: scatter ms, remote bytes, GB/s.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2605_30294_b200 import rafi  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--scatter", default="threads", choices=["threads", "bulk"])
    p.add_argument("--n", type=int, default=16 * 1024 * 1024)
    p.add_argument("--B", type=int, default=48)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=2)
    p.add_argument("--peers", type=int, default=1)
    a = p.parse_args()
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    cap = a.n + a.n // 8
    P = a.peers
    ctx = rafi.Context(a.B, cap, stream=s, local_ranks=1 + P)
    ctx.set_option(rafi.OPT_SCATTER, {"threads": rafi.SCATTER_THREADS, "bulk": rafi.SCATTER_BULK}[a.scatter])
    remote = [torch.empty(cap * a.B + 256, dtype=torch.uint8, device="cuda:%d" % p) for p in range(1, P + 1)]
    for p in range(1, P + 1):
        ctx.diag_redirect_incoming(p, remote[p - 1])
    items = torch.from_numpy(synth.make_items(0, 0, a.n, max(a.B, 16))[:, :a.B].copy()).cuda()
    dests = torch.from_numpy(synth.make_dests("uniform", synth.CONFIG_SEEDS[2], 0, 0, a.n, 1 + P)).cuda()
    for k in range(a.warmup + a.steps):
        if k == a.warmup:
            ctx.set_option(rafi.OPT_TIMING, 1)
        ctx.emit_bulk(items, dests, a.n, local=0)
        G = ctx.forward()
        assert G == a.n, G
    st = ctx.stats()
    K = st["acc_forwards"]
    ms = st["acc_ms_scatter"] / K
    to_peers = int(ctx.matrix()[0, 1:].sum())
    rb = to_peers * a.B
    print(json.dumps({"scatter": a.scatter, "tile": ctx.get_option(rafi.OPT_TILE), "n": a.n, "B": a.B, "peers": P,
                      "items_to_peers": to_peers, "remote_bytes": rb, "scatter_ms": ms,
                      "remote_gbs": rb / (ms / 1e3) / 1e9,
                      "local_bytes": (a.n - to_peers) * a.B,
                      "what": "rank 0 of an N=%d FUSED forward, one process; remote_gbs = bytes pushed to "
                              "cuda:1..%d / scatter kernel time" % (1 + P, P)}), flush=True)
    for p in range(1, P + 1):
        ctx.diag_redirect_incoming(p, None)
    ctx.close()


if __name__ == "__main__":
    main()
