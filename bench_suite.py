"""bench_suite.py -- the other BASELINE.json configs and the paper-style sweeps.

    python bench_suite.py <workload> [--gpus N]      (N > 1: under torch.distributed.run)

workloads:
  cfg1    2 ranks, 4096 x 32-B items/rank, uniform random walk, 3 rounds + termination
  cfg3    2x2x2-brick ray marcher, 4M rays/rank, rounds until all rays exit
  cfg4    2x2x2-macrocell RK4 advection, 1M seeds/rank (8M total), 64 rounds
  cfg5    N-body-style uniform all-to-all, 32M items/rank, item size sweep 16..128 B
  sweep   items per rank 2^10..2^24 at 44 B (Fig. "bandwidth" analogue)

The 8-rank configs run as 8 ranks on the available GPUs: 8/N logical ranks per
GPU (local_ranks), exchanged by the FUSED path over local HBM and NVLink.
Prints one JSON line per measurement on rank 0.  Times are device times
(CUDA events on the context stream), max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def setup(args):
    import torch
    import torch.distributed as dist
    from paper_2605_30294_b200 import rafi
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        obj = [rafi.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = rafi.nccl_comm_init(world, rank, obj[0], local)
    return torch, dist, rafi, world, rank, local, dev, comm


class Env:
    def __init__(self, args):
        (self.torch, self.dist, self.rafi, self.world, self.rank, self.local, self.dev,
         self.comm) = setup(args)
        self.stream = self.torch.cuda.current_stream()
        self.scatter = {"auto": 0, "threads": 1, "bulk": 2}[getattr(args, "scatter", "auto")]
        self.tile = getattr(args, "tile", 0)
        self.control = {"auto": 0, "nccl": 1, "peer": 2}[getattr(args, "control", "auto")]

    def configure(self, ctx):
        """Apply the --scatter choice (RAFI_OPT_SCATTER) to a new context."""
        if self.scatter:
            ctx.set_option(self.rafi.OPT_SCATTER, self.scatter)
        if self.tile:
            ctx.set_option(self.rafi.OPT_TILE, self.tile)
        if self.control:
            ctx.set_option(self.rafi.OPT_CONTROL, self.control)
        return ctx

    def ctx(self, B, cap, L=1):
        return self.configure(self.rafi.Context(B, cap, comm=self.comm, stream=self.stream, local_ranks=L,
                                                device=self.local))

    def sync(self):
        self.torch.cuda.synchronize()
        if self.world > 1:
            self.dist.barrier(device_ids=[self.local])
        self.torch.cuda.synchronize()

    def max(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def timed(self, fn):
        """Device time of fn() (ms), barrier-bracketed, max over ranks."""
        e0 = self.torch.cuda.Event(enable_timing=True)
        e1 = self.torch.cuda.Event(enable_timing=True)
        self.sync()
        e0.record(self.stream)
        out = fn()
        e1.record(self.stream)
        self.sync()
        return self.max(e0.elapsed_time(e1)), out

    def emit(self, line):
        if self.rank == 0:
            line.setdefault("n_gpus", self.world)
            print(json.dumps(line), flush=True)

    def close(self, ctx=None):
        if ctx is not None:
            ctx.close()


def grid_dims(R):
    return {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}.get(R, (R, 1, 1))


# ----------------------------------------------------------------------------- cfg1

def run_cfg1(env, args):
    import synth
    R, n, B = 2, 4096, 32
    if env.world > R:
        return
    L = R // env.world
    seed = synth.CONFIG_SEEDS[1]
    ctx = env.ctx(B, 2 * n * L if L > 1 else 2 * n, L)

    def one_run():
        Gs = []
        for l in range(L):
            ctx.drv_emit_synthetic(synth.PATTERNS["uniform"], seed, 0, n, local=l)
        for k in range(1, 6):          # seed forward, 3 walk rounds, terminating forward
            Gs.append(ctx.forward())
            ctx.drv_random_walk(seed, k, 3)
        return Gs

    for _ in range(3):
        one_run()
    reps = 20
    ms, Gs = env.timed(lambda: [one_run() for _ in range(reps)][-1])
    assert Gs == [R * n] * 4 + [0], Gs
    per_run = ms / reps
    env.emit({"workload": "cfg1: 2 ranks x 4096 x 32-B items, seed + 3 random-walk rounds + terminating forward",
              "metric": "ms per forwarding round (latency-bound)", "ms_per_run": per_run,
              "ms_per_round": per_run / 5, "items_per_s": 4 * R * n / (per_run / 1e3),
              "local_ranks": L, "G": Gs})
    ctx.close()


def run_latency(env, args):
    """Per-round latency of a small random-walk round (cfg1 shape): the
    blocking rafi_forward loop vs CUDA-graph replays of [walk step +
    rafi_forward_async] with device-side G (NEXT-3)."""
    import synth
    R, n, B = 2, args.items or 4096, 32
    if env.world > R:
        return
    L = R // env.world
    torch = env.torch
    seed = synth.CONFIG_SEEDS[1]
    side = torch.cuda.Stream(device=env.dev)
    ctx = env.configure(env.rafi.Context(B, 2 * n, comm=env.comm, stream=side, local_ranks=L, device=env.local))
    G_dev = torch.zeros(1, dtype=torch.int64, device=env.dev)
    for l in range(L):
        ctx.drv_emit_synthetic(synth.PATTERNS["uniform"], seed, 0, n, local=l)
    ctx.forward()
    K = 200
    for k in range(5):
        ctx.drv_random_walk(seed, 1, 10**9)
        ctx.forward()
    env.stream = side
    ms_sync, _ = env.timed(lambda: [(ctx.drv_random_walk(seed, 1, 10**9), ctx.forward()) for _ in range(K)])
    ctx.capture_begin()
    ctx.drv_random_walk(seed, 1, 10**9)
    ctx.forward_async(G_dev)
    ex = ctx.capture_end()
    for _ in range(5):
        ctx.graph_launch(ex)
    ms_graph, _ = env.timed(lambda: [ctx.graph_launch(ex) for _ in range(K)])
    side.synchronize()
    assert int(G_dev.item()) == R * n
    ctx.sync_host()
    env.rafi.Context.graph_destroy(ex)
    env.emit({"workload": "latency: %d ranks x %d x %d-B items, random-walk round (app step + forward)" % (R, n, B),
              "metric": "us per round", "sync_forward_us": 1e3 * ms_sync / K, "graph_async_us": 1e3 * ms_graph / K,
              "local_ranks": L})
    ctx.close()


def run_nbody(env, args):
    """NEXT-2: the three-context N-body exchange pattern at
    R=8: migrate 40-B particles, broadcast 24-B root nodes, 4-B refinement
    requests, 24-B subtree responses -- four forwards per step."""
    R = 8
    L = R // env.world
    n = args.items or 1024 * 1024
    torch = env.torch
    P = env.ctx(40, 2 * n, L)
    V = env.ctx(24, 64 * R, L)
    Q = env.ctx(4, 4 * R, L)
    stats = torch.zeros((L, 42), dtype=torch.int64, device=env.dev)
    for l in range(L):
        P.drv_nbody_seed(n, 0x5EED0005, local=l)
    P.forward()
    G = [0, 0, 0, 0]

    def step():
        P.drv_nbody_migrate(1.0 / 64)
        G[0] = P.forward()
        P.drv_nbody_stats(stats)
        V.drv_nbody_root(stats)
        G[1] = V.forward()
        V.drv_nbody_refine(Q, stats, 0.25)
        G[2] = Q.forward()
        Q.drv_nbody_respond(V, stats)
        G[3] = V.forward()

    for _ in range(3):
        step()
    K = 10
    ms, _ = env.timed(lambda: [step() for _ in range(K)])
    env.emit({"workload": "nbody: 3 contexts (40/24/4-B items), R=8, %d particles/rank, 4 forwards per step" % n,
              "metric": "ms per N-body exchange step", "ms_per_step": ms / K,
              "particles_per_s": R * n * K / (ms / 1e3), "G_last_step": list(G), "local_ranks": L})
    P.close(); V.close(); Q.close()


def run_streamlines(env, args):
    """NEXT-4: streamlines on a sampled ABC-flow field (129^3 vertices), R=8
    macrocell blocks with one-vertex halos, 1M seeds/rank, 64 RK4 steps."""
    import numpy as np
    R = 8
    L = R // env.world
    n = args.items or 1024 * 1024
    torch = env.torch
    nv = 129
    c = np.linspace(0.0, 1.0, nv)
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    tp = 2 * np.pi
    field = np.ascontiguousarray(np.stack((np.sin(tp * z) + 0.43 * np.cos(tp * y), 0.7 * np.sin(tp * x) + np.cos(tp * z),
                                           0.43 * np.sin(tp * y) + 0.7 * np.cos(tp * x)), axis=-1), dtype=np.float32)
    h = 0.4 * (1.0 / (nv - 1)) / (2 * float(np.abs(field).max()))
    rng = np.random.default_rng(0x5EED0004 + env.rank)
    ctx = env.ctx(16, 2 * n + 4096, L)
    f = env.rafi.StreamField(ctx, field, grid_dims(R))
    rpos = torch.zeros((R * n, 3), dtype=torch.float32, device=env.dev)
    rst = torch.zeros((R * n,), dtype=torch.int32, device=env.dev)

    def run():
        for l in range(L):
            f.seed(rng.random((n, 3)).astype(np.float32), (env.rank * L + l) * n, local=l)
        total, k = 0, 0
        while True:
            G = ctx.forward()
            total += G
            if G == 0:
                return total, k
            k += 1
            f.step(k, h, 1e-7, 64, rpos, rst)

    run()
    ms, (total, rounds) = env.timed(run)
    env.emit({"workload": "streamlines: ABC flow on a 129^3 lattice, R=8 blocks + halo, %d seeds/rank, 64 RK4 steps"
                          % n, "metric": "forwarded work items/sec (app + forward, all rounds)",
              "value": total / (ms / 1e3), "unit": "items/s", "rounds": rounds, "forwarded_items": total,
              "ms_total": ms, "halo_misses": f.halo_misses(), "local_ranks": L})
    f.close()
    ctx.close()


# ----------------------------------------------------------------------------- cfg3 / cfg4

def run_cfg3(env, args):
    R = 8
    L = R // env.world
    n = args.items or 4 * 1024 * 1024
    B, g = 48, grid_dims(R)
    p_thr, max_b, max_s, seed = int(0.01 * 2**32), 4, 256, 0x5EED0003
    torch = env.torch
    ctx = env.ctx(B, 2 * n, L)
    res = torch.full((R * n,), -1.0, dtype=torch.float32, device=env.dev)

    def run():
        for l in range(L):
            ctx.drv_march_seed(n, seed, g, local=l)
        total, rounds = 0, 0
        while True:
            G = ctx.forward()
            total += G
            if G == 0:
                return total, rounds
            rounds += 1
            ctx.drv_march_step(rounds, seed, p_thr, max_b, max_s, g, res)

    run()  # warm-up
    ctx.set_option(env.rafi.OPT_TIMING, 1)
    ms, (total, rounds) = env.timed(run)
    env.emit({"workload": "cfg3: 2x2x2-brick ray marcher, %d x 48-B rays/rank, p_scatter=0.01, until G=0" % n,
              "metric": "forwarded work items/sec (app + forward, all rounds)", "value": total / (ms / 1e3),
              "unit": "items/s", "rounds": rounds, "forwarded_items": total, "ms_total": ms, "local_ranks": L})
    ctx.close()


def run_cfg4(env, args):
    R = 8
    L = R // env.world
    n = args.items or 1024 * 1024
    g = grid_dims(R)
    omega, eps, h, max_rounds, seed = 2 * math.pi / 64, 1.0 / 128, 1.0, 64, 0x5EED0004
    ctx = env.ctx(16, 2 * n, L)

    def run():
        for l in range(L):
            ctx.drv_advect_seed(n, seed, g, local=l)
        total, rounds = 0, 0
        while True:
            G = ctx.forward()
            total += G
            if G == 0:
                return total, rounds
            rounds += 1
            ctx.drv_advect_step(rounds, max_rounds, omega, eps, h, g)

    run()
    ms, (total, rounds) = env.timed(run)
    env.emit({"workload": "cfg4: 2x2x2-macrocell RK4 advection, %d x 16-B seeds/rank (%d total), 64 rounds"
                          % (n, n * R),
              "metric": "forwarded work items/sec (app + forward, all rounds)", "value": total / (ms / 1e3),
              "unit": "items/s", "rounds": rounds, "forwarded_items": total, "ms_total": ms,
              "ms_per_round": ms / max(rounds, 1), "local_ranks": L})
    ctx.close()


# ----------------------------------------------------------------------------- cfg5 / sweep

def fwd_rate(env, B, n, steps=5, warmup=2, pattern="uniform", graph=False, ranks=0):
    """emit_bulk + forward of n items/rank, R = ranks (default: world, one
    rank per GPU; otherwise R / world logical ranks per GPU, sharing one item
    payload per GPU, each with its own destinations).
    With graph=True the step is also captured as a CUDA graph of
    [emit_bulk + rafi_forward_async] and replayed (device-side G, no host
    synchronisation per step): the per-step latency without host overhead."""
    import synth
    torch = env.torch
    N = env.world
    R = ranks or N
    L = R // N
    # payload bytes only matter for throughput here (parity is tested elsewhere): device RNG
    gen = torch.Generator(device=env.dev)
    gen.manual_seed(synth.CONFIG_SEEDS[5] + env.rank)
    items = torch.randint(0, 256, (n, B), dtype=torch.uint8, device=env.dev, generator=gen)
    dests = [torch.from_numpy(synth.make_dests(pattern, synth.CONFIG_SEEDS[5], env.rank * L + l, 0, n, R)).to(env.dev)
             for l in range(L)]
    side = torch.cuda.Stream(device=env.dev)
    ctx = env.configure(env.rafi.Context(B, n + n // 8 + 4096, comm=env.comm, stream=side, device=env.local,
                                         local_ranks=L))
    saved, env.stream = env.stream, side

    def emit_all():
        for l in range(L):
            ctx.emit_bulk(items, dests[l], n, local=l)

    for _ in range(warmup):
        emit_all()
        ctx.forward()

    def loop():
        for _ in range(steps):
            emit_all()
            ctx.forward()

    ms, _ = env.timed(loop)  # un-instrumented: blocking forwards replay their cached graph
    ctx.set_option(env.rafi.OPT_TIMING, 1)
    ms_instr, _ = env.timed(loop)  # instrumented pass: CUDA events between launches, for scatter_ms
    st = ctx.stats()
    scat = st["acc_ms_scatter"] / max(st["acc_forwards"], 1)
    Cm = ctx.matrix()  # bytes this GPU pushes to other GPUs per forward
    mine = slice(env.rank * L, env.rank * L + L)
    remote = (int(Cm[mine, :].sum()) - int(Cm[mine, mine].sum())) * B
    out = {"items_per_rank": n, "item_bytes": B, "ranks": R, "local_ranks": L, "ms_per_step": ms / steps,
           "instrumented_ms_per_step": ms_instr / steps,
           "value": R * n * steps / (ms / 1e3), "unit": "items/s",
           "scatter": {1: "threads", 2: "bulk"}[ctx.get_option(env.rafi.OPT_SCATTER)],
           "tile": ctx.get_option(env.rafi.OPT_TILE), "scatter_ms": scat,
           "scatter_hbm_gbs": L * n * (2 * B + 4) / (scat / 1e3) / 1e9,
           "binning_ms": (st["acc_ms_hist"] + st["acc_ms_scan"] + st["acc_ms_scatter"]) / max(st["acc_forwards"], 1),
           "nvlink_gbs_per_gpu": (remote / (scat / 1e3) / 1e9) if N > 1 else None}
    out["binning_hbm_frac"] = L * n * (2 * B + 8) / (out["binning_ms"] / 1e3) / 1e9 / 6457.1
    if graph:
        ctx.set_option(env.rafi.OPT_TIMING, 0)
        G_dev = torch.zeros(1, dtype=torch.int64, device=env.dev)
        ctx.capture_begin()
        emit_all()
        ctx.forward_async(G_dev)
        ex = ctx.capture_end()
        for _ in range(3):
            ctx.graph_launch(ex)
        K = 50
        msg, _ = env.timed(lambda: [ctx.graph_launch(ex) for _ in range(K)])
        side.synchronize()
        assert int(G_dev.item()) == R * n
        ctx.sync_host()
        env.rafi.Context.graph_destroy(ex)
        out["graph_ms_per_step"] = msg / K
        out["graph_value"] = R * n * K / (msg / 1e3)
    env.stream = saved
    ctx.close()
    del items, dests
    torch.cuda.empty_cache()
    return out


def run_cfg5(env, args):
    n = args.items or 32 * 1024 * 1024
    sizes = [int(x) for x in args.sizes.split(",")] if args.sizes else [16, 24, 32, 40, 44, 48, 64, 96, 128]
    for B in sizes:
        try:
            r = fwd_rate(env, B, n, ranks=args.ranks)
        except env.rafi.RafiError as e:  # e.g. a --tile that does not fit this item size
            env.emit({"item_bytes": B, "skipped": str(e)})
            continue
        r["workload"] = "cfg5: uniform all-to-all over R=%d, %d items/rank, %d-B items, %d logical rank(s) per GPU" % (
            r["ranks"], n, B, r["local_ranks"])
        env.emit(r)


def run_sweep(env, args):
    for e in range(10, 25, 2):
        r = fwd_rate(env, 44, 1 << e, steps=10 if e < 20 else 5, graph=True)
        r["workload"] = "sweep: 2^%d x 44-B items/rank, uniform over R=%d" % (e, env.world)
        env.emit(r)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("workload", choices=["cfg1", "cfg3", "cfg4", "cfg5", "sweep", "latency", "nbody", "streamlines"])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--items", type=int, default=0)
    p.add_argument("--scatter", default="auto", choices=["auto", "threads", "bulk"])
    p.add_argument("--tile", type=int, default=0, help="RAFI_OPT_TILE (0 = automatic)")
    p.add_argument("--control", default="auto", choices=["auto", "nccl", "peer"])
    p.add_argument("--sizes", default="", help="cfg5: comma-separated item sizes (default: the full sweep)")
    p.add_argument("--ranks", type=int, default=8, help="cfg5: ranks R (configs[4]: 8), R / N logical ranks per GPU")
    args = p.parse_args()
    env = Env(args)
    {"cfg1": run_cfg1, "cfg3": run_cfg3, "cfg4": run_cfg4, "cfg5": run_cfg5, "sweep": run_sweep,
     "latency": run_latency, "nbody": run_nbody, "streamlines": run_streamlines}[args.workload](
        env, args)
    if env.comm:
        env.rafi.nccl_comm_destroy(env.comm)
    if env.world > 1:
        env.dist.destroy_process_group()


if __name__ == "__main__":
    main()
