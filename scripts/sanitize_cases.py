"""Small forwarding cases for compute-sanitizer runs (memcheck / racecheck /
synccheck, one tool per call):

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py

Covers every kernel family: bulk emit (16/4/1-byte units), device emit
(drivers), histogram (register and generic counters), scan + plan, FUSED and
PEER scatter (staged and unstaged items), copy, wrap-up, async forward.
Each case is checked against the oracle so a silent corruption also fails.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from helpers import make_inputs, p1_forward  # noqa: E402
from paper_2605_30294_b200 import rafi  # noqa: E402


def case(B, L, n, pattern, exchange):
    inputs = make_inputs(L, n, B, pattern, 99 + B, invalid_frac=0.01)
    with rafi.Context(B, max(n * L, 1), local_ranks=L) as ctx:
        ctx.set_option(rafi.OPT_EXCHANGE, exchange)
        for l, (it, ds) in enumerate(inputs):
            ctx.emit_bulk(torch.from_numpy(it).cuda(), torch.from_numpy(ds).cuda(), len(ds), local=l)
        p1_forward(ctx, L, B)
    print("ok B=%d L=%d n=%d %s exch=%d" % (B, L, n, pattern, exchange), flush=True)


def main():
    torch.cuda.set_device(0)
    for exch in (rafi.EXCHANGE_FUSED, rafi.EXCHANGE_PEER):
        case(48, 4, 3001, "uniform", exch)      # 16-B units, register histogram
        case(44, 3, 2999, "skewed", exch)       # 4-B units
        case(3, 2, 2500, "uniform", exch)       # byte units
        case(520, 2, 700, "uniform", exch)      # unstaged items, warp-per-item
        case(16, 40, 300, "uniform", exch)      # generic histogram (R > 32)
    # device-side emit + async forward with device G
    s = torch.cuda.Stream()
    G = torch.zeros(1, dtype=torch.int64, device="cuda")
    with rafi.Context(32, 8000, local_ranks=2, stream=s) as ctx:
        for l in range(2):
            ctx.drv_emit_synthetic(synth.PATTERNS["uniform"], 1, 0, 3000, local=l)
        ctx.forward_async(G)
        s.synchronize()
        assert int(G.item()) == 6000
        ctx.sync_host()
    print("sanitize cases ok", flush=True)


if __name__ == "__main__":
    main()
