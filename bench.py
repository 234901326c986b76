"""bench.py -- forwarded work items/s of the RaFI hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl rafi|reference]
    (N > 1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N)

One STEP = one pass of the whole hot path over one batch per rank:
  a1 emit (rafi_emit_bulk of every rank's resident batch), then rafi_forward:
  a2 histogram, a3 scan, a4 stable scatter, a5 count exchange, a6 payload
  exchange, a7 wrap-up, a8 termination count.
Workload: BASELINE.json configs[1] itself -- 8 ranks, 16,777,216 synthetic
48-byte items per rank (the FWDRay shape), uniformly random
destinations over the 8 ranks, one forward.  On N GPUs each GPU hosts 8/N of
the ranks as logical ranks of one context (N=1: the whole 8-rank world on
one B200; N=8: one rank per GPU), so the total work is fixed (strong
scaling).  Inputs are resident in HBM before the timed region (805 MB of
items per rank > 126 MB L2, so no L2 reuse between steps).  value = items
all ranks forwarded / max-over-ranks device time.  e2e = the same metric
through the C ABI with HOST buffers: each step copies the batches in from
pinned memory (inside rafi_emit_bulk) and reads the incoming queues back to
pinned memory.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

DEF_N = 16 * 1024 * 1024
DEF_B = 48
DEF_R = 8  # configs[1]: 8 ranks
METRIC = "forwarded work items/sec"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="rafi", choices=["rafi", "reference"])
    p.add_argument("--items", type=int, default=DEF_N, help="items per rank per step")
    p.add_argument("--ranks", type=int, default=DEF_R, help="ranks R of the world (split evenly over the GPUs)")
    p.add_argument("--item-bytes", type=int, default=DEF_B)
    p.add_argument("--pattern", default="uniform")
    p.add_argument("--exchange", default="auto", choices=["auto", "nccl", "peer", "fused"])
    p.add_argument("--control", default="auto", choices=["auto", "nccl", "peer"])
    p.add_argument("--scatter", default="auto", choices=["auto", "threads", "bulk"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="skip the supplementary graph-replay measurement")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extras", action="store_true", help="skip the device_emit block")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the oracle cpu_baseline sample")
    return p.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def nvlink_ceilings(N):
    """NVLink ceilings measured on this pool by tools/p2p_bw (profiles/nvlink_ceilings.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "nvlink_ceilings.json")) as f:
            return json.load(f).get(str(N))
    except Exception:
        return None


def workload_config(args, N):
    R = args.ranks
    return {
        "workload": "configs[1]%s: %d ranks x %d x %d-B items/rank, %s dest over the %d ranks, 1 forward/step"
                    % ("" if (R, args.items, args.item_bytes, args.pattern) == (DEF_R, DEF_N, DEF_B, "uniform")
                       else " (modified)", R, args.items, args.item_bytes, args.pattern, R),
        "items_per_rank": args.items, "item_bytes": args.item_bytes, "ranks": R, "pattern": args.pattern,
        "ranks_per_gpu": R // N,
        "l2": "inputs larger than L2 (%.0f MiB per rank resident)" % (args.items * (args.item_bytes + 4) / 2**20),
        "step": "emit_bulk of every rank + forward (hist, scan, scatter, count exchange, payload exchange, wrap-up)",
        "parallelism": "%d GPU%s x %d logical rank%s" % (N, "s" if N > 1 else "", R // N, "s" if R // N > 1 else ""),
    }


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region.

    Started before the warm-up: nvidia-smi's start-up (NVML init) takes the
    driver's locks for ~0.1-0.3 s, and when it overlapped the ~15-ms timed
    region it stalled every rank's CUDA calls (N=4: 1.41 vs 1.32 ms per step).
    Samples are taken every 100 ms and kept when they fall within 150 ms of
    the timed region (the nearest one if none does)."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.window = None

    def mark(self, t0, t1):
        """Wall-clock bounds (time.perf_counter) of the timed region."""
        self.window = (t0, t1)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t_end = time.perf_counter() + 5.0  # the first sample = nvidia-smi is past its start-up
            while not self.lines and time.perf_counter() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.window and lines:
            t0, t1 = self.window
            near = [(t, ln) for t, ln in lines if t0 - 0.15 <= t <= t1 + 0.15]
            lines = near or [min(lines, key=lambda x: abs(x[0] - t0))]
        for _, ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


# ----------------------------------------------------------------------------- oracle (CPU)

def host_facts():
    """nproc and CPU model of the host the oracle runs on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


class pinned_to_core0:
    """Pin the calling thread to core 0 (taskset -c 0) while the single-threaded oracle runs."""

    def __enter__(self):
        self.old = None
        try:
            self.old = os.sched_getaffinity(0)
            os.sched_setaffinity(0, {min(self.old)})
            self.core = min(self.old)
        except Exception:
            self.core = None
        return self

    def __exit__(self, *a):
        if self.old:
            os.sched_setaffinity(0, self.old)


def oracle_step_rate(R, n, B, pattern, seconds, max_reps=50):
    """The oracle as it stands (single-threaded C): one step = sequential
    emit of every rank's batch + forward, on a bounded sample of the
    workload.  Returns (items/s, reps, sample description)."""
    import oracle
    import synth
    batches = []
    for s in range(R):
        it = synth.make_items(s, 0, n, max(B, 16))[:, :B].copy()
        ds = synth.make_dests(pattern, synth.CONFIG_SEEDS[2], s, 0, n, R)
        batches.append((it, ds))
    cap = n + n // 8 + 4096
    w = oracle.World(R, cap, B)
    times = []
    with pinned_to_core0():
        t_end = time.perf_counter() + seconds
        while len(times) < max_reps and (time.perf_counter() < t_end or len(times) < 2):
            t0 = time.perf_counter()
            for s, (it, ds) in enumerate(batches):
                w.emit_many(s, it, ds)
            G = w.forward()
            times.append(time.perf_counter() - t0)
            assert G == R * n, G
    w.close()
    med = statistics.median(times)
    return R * n / med, len(times), "R=%d x %d items x %d B (%s), emit+forward per step, median of %d" % (
        R, n, B, pattern, len(times))


def cpu_sample_size(args, R):
    # ~1-2 s per oracle step on one core: 2M items per step in total
    return max(1024, min(args.items, (2 * 1024 * 1024) // R))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    N, R = args.gpus, args.ranks
    n = cpu_sample_size(args, R)
    import oracle
    import synth
    batches = []
    for s in range(R):
        it = synth.make_items(s, 0, n, max(args.item_bytes, 16))[:, :args.item_bytes].copy()
        ds = synth.make_dests(args.pattern, synth.CONFIG_SEEDS[2], s, 0, n, R)
        batches.append((it, ds))
    w = oracle.World(R, n + n // 8 + 4096, args.item_bytes)

    def step():
        for s, (it, ds) in enumerate(batches):
            w.emit_many(s, it, ds)
        assert w.forward() == R * n

    with pinned_to_core0():
        for _ in range(args.warmup):
            step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        dt = time.perf_counter() - t0
    v = R * n * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "items/s", "n_gpus": N, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (synth/ SplitMix64 recipe)",
        "config": workload_config(args, N),
        "cpu_baseline": dict({"value": v, "unit": "items/s", "cores": 1, "kind": "oracle",
                              "sample": "R=%d x %d items x %d B per step (bounded sample of the workload), "
                                        "sequential emit + plain forward, single-threaded C oracle pinned to "
                                        "one core (sched_setaffinity, as taskset -c 0)" % (R, n, args.item_bytes)},
                             **host_facts()),
        "e2e": {"value": v, "unit": "items/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- NVLink counters

def stored_nvlink_counters(scatter, B, n, N):
    """NVLink byte counters of the FUSED scatter from the stored single-process
    ncu capture (profiles/r02_nvlink_counters.json; scripts/nvl_redirect.py).
    Not read live: NVML does not expose the NVLink byte counters on these boxes
    (nvidia-smi nvlink -gt d: N/A), and querying NVML next to the timed region
    stalled the first steps by ~10 ms."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_nvlink_counters.json")) as f:
            tab = json.load(f)
    except Exception:
        return {"available": False, "why": "profiles/r02_nvlink_counters.json missing"}
    key = "scatter_%s/B%d/n%d/R2" % (scatter, B, n)
    if key not in tab:
        return {"available": False, "why": "no stored capture for %s" % key}
    return dict(tab[key], available=True, source="STORED, not measured in this run: " + tab["_capture"] +
                "; rank 0 of an N=2 FUSED forward driven by one process (N=%d here)" % N)


# ----------------------------------------------------------------------------- supplementary blocks

def bench_device_emit(rafi, torch, stream, items_d, dests_d, args, hbm_peak):
    """The app-facing emit (rafi::Queue<T>::emitOutgoing, warp-aggregated
    atomics, vector stores) re-emitting the resident batch: algorithmic bytes
    2(B+4) per item (read item + dest, write item + dest)."""
    n, B = args.items, args.item_bytes
    ctx = rafi.Context(B, n, stream=stream)
    out = {}
    try:
        for batch in (8, 1):
            evs = []
            for k in range(args.warmup + args.steps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                ctx.drv_emit_items(items_d, dests_d, n, batch=batch)
                b.record(stream)
                if k >= args.warmup:
                    evs.append((a, b))
                assert ctx.forward() == n  # empties the queue (untimed)
            stream.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in evs) / len(evs)
            byts = n * 2 * (B + 4)
            gbs = byts / (ms / 1e3) / 1e9
            out["batch%d" % batch] = {"ms": ms, "achieved_gbs": gbs, "frac": gbs / hbm_peak,
                                      "items_per_s": n / (ms / 1e3)}
        best = out["batch8"]
        return dict(best, items=n, algorithmic_bytes=n * 2 * (B + 4), single=out["batch1"],
                    what="rafi_drv_emit_items, the app-facing device emit: threads load items (16-B vectors) "
                         "and emit through rafi::Queue<T> (16-B vector stores); top level = batched "
                         "emitOutgoing<8> (one warp atomicAdd per 256 items), 'single' = one emitOutgoing per "
                         "item (one warp atomicAdd per 32 items: bounded by the emit counter's per-address L2 "
                         "atomic rate); CUDA events around each launch")
    finally:
        ctx.close()


# ----------------------------------------------------------------------------- GPU arm

def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import synth
    from paper_2605_30294_b200 import rafi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    N = world
    if world != args.gpus:
        print("warning: --gpus %d but WORLD_SIZE %d; using %d" % (args.gpus, world, world), file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        obj = [rafi.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = rafi.nccl_comm_init(world, rank, obj[0], local)

    B, n, R = args.item_bytes, args.items, args.ranks
    if R % N:
        raise SystemExit("--ranks %d must be a multiple of the GPU count %d" % (R, N))
    L = R // N  # logical ranks per GPU (global ranks rank*L .. rank*L+L-1)
    # the context's own (non-default) stream: everything below is ordered on
    # it, and it can be captured into a CUDA graph
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.synchronize()
    cap = n + n // 8 + 4096
    ctx = rafi.Context(B, cap, comm=comm, stream=stream, device=local, local_ranks=L)
    if args.exchange != "auto":
        ctx.set_option(rafi.OPT_EXCHANGE, {"nccl": rafi.EXCHANGE_NCCL, "peer": rafi.EXCHANGE_PEER,
                                           "fused": rafi.EXCHANGE_FUSED}[args.exchange])
    exchange = {1: "nccl", 2: "peer", 3: "fused"}[ctx.get_option(rafi.OPT_EXCHANGE)]
    if args.scatter != "auto":
        ctx.set_option(rafi.OPT_SCATTER, {"threads": rafi.SCATTER_THREADS, "bulk": rafi.SCATTER_BULK}[args.scatter])
    scatter = {1: "threads", 2: "bulk"}[ctx.get_option(rafi.OPT_SCATTER)]
    ctx_tile = ctx.get_option(rafi.OPT_TILE)
    if args.control != "auto":
        ctx.set_option(rafi.OPT_CONTROL, {"nccl": rafi.CONTROL_NCCL, "peer": rafi.CONTROL_PEER}[args.control])
    control = {1: "nccl", 2: "peer", 3: "host"}[ctx.get_option(rafi.OPT_CONTROL)] if N > 1 else None

    # resident inputs (generated on the host by the shared generator, uploaded
    # once).  The item payload is generated once per GPU and shared by its
    # logical ranks (16M x 48 B takes seconds to generate on the host); every
    # rank has its own destinations.
    items_h = synth.make_items(rank * L, 0, n, max(B, 16))[:, :B].copy()
    dests_h = [synth.make_dests(args.pattern, synth.CONFIG_SEEDS[2], rank * L + l, 0, n, R) for l in range(L)]
    items_d = torch.from_numpy(items_h).to(dev)
    dests_d = [torch.from_numpy(d).to(dev) for d in dests_h]

    def emit_all(items, dests):
        for l in range(L):
            ctx.emit_bulk(items, dests[l], n, local=l)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---- warm-up (the clock sampler starts first: its start-up must not overlap the timed region)
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        emit_all(items_d, dests_d)
        G = ctx.forward()
    assert G == R * n, (G, R * n)

    # ---- timed region (device-timed: CUDA events on the context stream,
    # barrier + synchronize on both sides, max over ranks).  The library runs
    # un-instrumented here (RAFI_OPT_TIMING is off by default): every blocking
    # forward replays the CUDA graph the warm-up steps captured.
    assert ctx.get_option(rafi.OPT_TIMING) == 0
    l0 = ctx.stats()["kernel_launches"]
    barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    f_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    w0 = time.perf_counter()
    t_start.record(stream)
    for k in range(args.steps):
        emit_all(items_d, dests_d)
        f_ev[k][0].record(stream)     # forward only (a2-a8): events around each rafi_forward
        G = ctx.forward()
        f_ev[k][1].record(stream)
    t_end.record(stream)
    barrier()
    clocks.mark(w0, time.perf_counter())
    clk = clocks.stop()
    ms_fwd = max_over_ranks(sum(a.elapsed_time(b) for a, b in f_ev))
    st = ctx.stats()
    launches = st["kernel_launches"] - l0
    # bytes this GPU pushes to OTHER GPUs per step (its ranks' rows of the
    # count matrix, columns of ranks hosted elsewhere), same plan every step
    Cm = ctx.matrix()
    mine = slice(rank * L, rank * L + L)
    remote = (int(Cm[mine, :].sum()) - int(Cm[mine, mine].sum())) * B * args.steps
    ms_total = t_start.elapsed_time(t_end)
    ms_max = max_over_ranks(ms_total)
    K = args.steps

    # ---- instrumented pass: the same K steps with RAFI_OPT_TIMING, i.e. CUDA
    # events recorded on the context stream between the kernel launches of
    # every emit and forward (launched one by one, not from the graph); the
    # per-kernel durations of the rooflines come from here
    ctx.set_option(rafi.OPT_TIMING, 1)
    barrier()
    i_start = torch.cuda.Event(enable_timing=True)
    i_end = torch.cuda.Event(enable_timing=True)
    i_start.record(stream)
    for k in range(args.steps):
        emit_all(items_d, dests_d)
        ctx.forward()
    i_end.record(stream)
    barrier()
    st = ctx.stats()
    ms_instr = max_over_ranks(i_start.elapsed_time(i_end)) / K
    assert st["acc_forwards"] == K and st["acc_emits"] == K * L, (st["acc_forwards"], st["acc_emits"])
    value = R * n * K / (ms_max / 1e3)
    ms_step = ms_max / K
    forward_only = {"value": R * n * K / (ms_fwd / 1e3), "unit": "items/s", "ms_per_forward": ms_fwd / K,
                    "what": "rafi_forward alone (hist, scan, count exchange, scatter/payload exchange, wrap-up, "
                            "termination count), emission excluded: the paper's sort-and-send (PAPER:449); CUDA "
                            "events around each forward inside the timed region, max over ranks"}
    ph = {k: st["acc_ms_" + k] / K for k in ("emit", "hist", "scan", "scatter", "count_exchange",
                                            "payload_exchange", "wrapup")}  # per step (emit: all L launches)
    per_launch = dict(ph, emit=ph["emit"] / L)

    # ---- rooflines: algorithmic bytes per launch / average launch duration
    hbm_peak, peak_src = load_peaks()
    nin = sum(ctx.num_incoming(l) for l in range(L))
    alg = {  # bytes per launch; DESIGN.md "Rooflines" (one emit launch per rank; hist/scatter cover all L)
        "emit": n * 2 * (B + 4),
        "hist": L * n * 4,
        "scatter": L * n * (B + 4 + B),
        "payload_exchange": nin * 2 * B if (N == 1 and exchange != "fused") else None,
    }
    kern = {}
    for k, byts in alg.items():
        if byts is None or per_launch[k] <= 0:
            continue
        gbs = byts / (per_launch[k] / 1e3) / 1e9
        kern[k] = {"ms": per_launch[k], "bytes": byts, "achieved_gbs": gbs, "frac": gbs / hbm_peak,
                   "launches_per_step": L if k == "emit" else 1}
    dom = max(kern, key=lambda k: kern[k]["ms"])
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        key = "%s/B%d/n%d/R%d/N%d" % (dom, B, n, R, N)
        traffic = tr.get(key)
        if traffic is not None:
            traffic_src = "STORED, not measured in this run: dram__bytes_read.sum + dram__bytes_write.sum of " \
                          "one ncu --set full capture, %s" % tr.get("_capture", tr.get("_about", "")[:160])
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": dom, "achieved": kern[dom]["achieved_gbs"], "peak": hbm_peak,
                "unit": "GB/s", "frac": kern[dom]["frac"], "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": peak_src, "algorithmic_bytes_per_launch": kern[dom]["bytes"]}
    exch = None
    xfer_ms = ph["scatter"] if exchange == "fused" else ph["payload_exchange"]
    if N > 1 and xfer_ms > 0:
        # remote payload bytes this GPU sends per step / time of the phase that moves them
        # (FUSED: the scatter pushes over NVLink; staged: the copy kernel / NCCL send-recv)
        gbs = (remote / K) / (xfer_ms / 1e3) / 1e9
        ceil = nvlink_ceilings(N)
        exch = {"gbs_per_gpu": gbs, "frac_of_900": gbs / 900.0, "frac_of_770_measured_p2p": gbs / 770.0,
                "transport": exchange, "remote_bytes_per_step": remote / K, "kernel_ms": xfer_ms,
                "ceilings_gbs": ceil, "nvlink_counters": stored_nvlink_counters(scatter, B, n, N) if exchange == "fused" else None}
        if exchange == "fused" and xfer_ms >= max(v["ms"] for v in kern.values()):
            # the step's dominant phase moves bytes over NVLink: that is its roofline
            # (peak: the profiling guide's measured 770 GB/s peer copy per direction)
            roofline = {"bound": "nvlink", "kernel": "scatter",
                        "achieved": gbs, "peak": 770.0, "unit": "GB/s", "frac": gbs / 770.0,
                        "traffic": None, "peak_source": "B200_PROFILING.md: measured peer copy 770 GB/s per "
                        "direction (nominal 900); this box's ceilings from tools/p2p_bw in ceilings_gbs",
                        "algorithmic_bytes_per_launch": remote / K}

    # ---- end to end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        ctx.set_option(rafi.OPT_TIMING, 0)
        items_p = torch.from_numpy(items_h).pin_memory()
        dests_p = [torch.from_numpy(d).pin_memory() for d in dests_h]
        # two pinned result buffers per rank: step k's read-back (copy-out
        # stream) overlaps step k+1's host-to-device copy (copy-in stream) over
        # full-duplex PCIe
        outs = [[torch.empty((cap, B), dtype=torch.uint8).pin_memory() for _ in range(2)] for _ in range(L)]
        # as many steps as the device-resident measurement: the pipeline's
        # one-time fill (first upload) and drain (last read-back) are inside
        # the timed region and amortise over K steps
        Ke = max(3, K)
        for k in range(2):
            emit_all(items_p, dests_p)
            ctx.forward()
            for l in range(L):
                ctx.read_incoming_async(outs[l][k % 2][: ctx.num_incoming(l)], local=l)
        ctx.read_wait()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        d2h = 0
        e0.record(stream)
        for k in range(Ke):
            emit_all(items_p, dests_p)                      # H2D inside the calls (host pointers)
            ctx.forward()
            for l in range(L):
                m = ctx.num_incoming(l)
                ctx.read_incoming_async(outs[l][k % 2][:m], local=l)  # D2H of the result
                d2h += m * B
        ctx.read_wait()                                    # every result is in host memory
        e1.record(stream)
        barrier()
        ms_e = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": R * n * Ke / (ms_e / 1e3), "unit": "items/s", "h2d_bytes_per_step": L * n * (B + 4),
               "d2h_bytes_per_step": int(d2h / Ke), "steps": Ke}

    # ---- the same step as an application-side CUDA graph (NEXT-3): [emit_bulk +
    # rafi_forward_async] captured once and replayed K times, G stays on the
    # device (no host synchronisation per step); supplementary, not the headline
    graph = None
    if not args.no_graph and exchange == "fused":  # rafi_forward_async is FUSED-only
        ctx.set_option(rafi.OPT_TIMING, 0)
        G_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        ctx.capture_begin()
        emit_all(items_d, dests_d)
        ctx.forward_async(G_dev)
        ex = ctx.capture_end()
        for _ in range(args.warmup):
            ctx.graph_launch(ex)
        barrier()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(K):
            ctx.graph_launch(ex)
        g1.record(stream)
        barrier()
        ms_g = max_over_ranks(g0.elapsed_time(g1))
        assert int(G_dev.item()) == R * n
        ctx.sync_host()
        rafi.Context.graph_destroy(ex)
        graph = {"value": R * n * K / (ms_g / 1e3), "unit": "items/s", "ms_per_step": ms_g / K,
                 "what": "[emit_bulk + rafi_forward_async] captured as one CUDA graph, replayed K times"}

    # ---- binning at N=1: the whole R-rank world's histogram + scan + scatter
    # (the instrumented phases of the headline steps), against (2B+8) bytes per item
    binning = None
    if N == 1:
        bms = ph["hist"] + ph["scan"] + ph["count_exchange"] + ph["scatter"]
        byts = R * n * (2 * B + 8)
        binning = {"workload": "the headline world: %d ranks x %d x %d-B items on one GPU, FUSED into local queues"
                               % (R, n, B), "ranks": R, "items": R * n, "ms": bms,
                   "ms_phases": {k: ph[k] for k in ("hist", "scan", "count_exchange", "scatter")},
                   "algorithmic_bytes": byts, "achieved_gbs": byts / (bms / 1e3) / 1e9,
                   "frac": byts / (bms / 1e3) / 1e9 / hbm_peak, "frac_of_8tbs": byts / (bms / 1e3) / 1e9 / 8000.0,
                   "scatter_frac": kern["scatter"]["frac"], "peak": hbm_peak, "tile": ctx_tile,
                   "what": "histogram + scan(+plan) + stable scatter of one forward; bytes = (2B+8) per item: "
                           "hist reads 4, scatter reads B+4 and writes B; from the instrumented pass"}

    # ---- supplementary single-GPU block: the device-side emit
    device_emit = None
    if N == 1 and not args.no_extras:
        ctx.close()
        ctx = None
        torch.cuda.empty_cache()
        device_emit = bench_device_emit(rafi, torch, stream, items_d, torch.zeros(n, dtype=torch.int32, device=dev),
                                        args, hbm_peak)

    # ---- cpu baseline: the oracle on the host, rank 0 at N=1 only
    cpu = None
    if N == 1 and rank == 0 and not args.no_cpu_baseline:
        ns = cpu_sample_size(args, R)
        v, reps, desc = oracle_step_rate(R, ns, B, args.pattern, args.cpu_seconds)
        cpu = dict({"value": v, "unit": "items/s", "cores": 1, "kind": "oracle",
                    "sample": desc + " (single-threaded C oracle on the GPU box host, pinned to one core "
                                     "with sched_setaffinity as taskset -c 0)"}, **host_facts())

    line = {
        "metric": METRIC, "value": value, "unit": "items/s", "n_gpus": N, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (synth/ SplitMix64 recipe; resident in HBM)", "config": workload_config(args, N),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "clocks": clk, "phases_ms": ph, "phases_source": "instrumented pass of the same K steps (CUDA events "
        "between launches); its ms_per_step: %.4f" % ms_instr, "kernels": kern, "exchange": exch, "exchange_transport": exchange,
        "graph_replay": graph, "scatter_write": scatter, "tile": ctx_tile, "control": control, "per_gpu_items_per_s": value / N,
        "forward_only": forward_only, "binning": binning, "device_emit": device_emit,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ctx is not None:
        ctx.close()
    if comm:
        rafi.nccl_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
