"""N>1 step-time diagnostic (measurement helper, not product).

    torchrun --nproc-per-node 2 scripts/diag_n2.py

For several (control, forward-graph) settings: K blocking steps of
[emit_bulk + forward] with host timestamps around each call and CUDA events
around each step, printed per rank, to find where a blocking step's time goes.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from paper_2605_30294_b200 import rafi  # noqa: E402


def main():
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    obj = [rafi.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = rafi.nccl_comm_init(world, rank, obj[0], local)
    n, B, K = 16 * 1024 * 1024, 48, 10
    items = torch.from_numpy(synth.make_items(rank, 0, n, B)[:, :B].copy()).to(dev)
    dests = torch.from_numpy(synth.make_dests("uniform", synth.CONFIG_SEEDS[2], rank, 0, n, world)).to(dev)
    stream = torch.cuda.Stream(device=dev)
    ctx = rafi.Context(B, n + n // 8 + 4096, comm=comm, stream=stream, device=local)
    for control, graph in ((rafi.CONTROL_PEER, 1), (rafi.CONTROL_PEER, 0), (rafi.CONTROL_NCCL, 1), (rafi.CONTROL_NCCL, 0)):
        ctx.set_option(rafi.OPT_CONTROL, control)
        ctx.set_option(rafi.OPT_FORWARD_GRAPH, graph)
        for _ in range(3):
            ctx.emit_bulk(items, dests, n)
            ctx.forward()
        torch.cuda.synchronize()
        dist.barrier(device_ids=[local])
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        host = []
        for k in range(K):
            t0 = time.perf_counter()
            ev[k][0].record(stream)
            ctx.emit_bulk(items, dests, n)
            t1 = time.perf_counter()
            ctx.forward()
            t2 = time.perf_counter()
            ev[k][1].record(stream)
            host.append((round((t1 - t0) * 1e3, 3), round((t2 - t1) * 1e3, 3)))
        torch.cuda.synchronize()
        dev_ms = [round(a.elapsed_time(b), 3) for a, b in ev]
        print(json.dumps({"rank": rank, "control": control, "graph": graph, "dev_ms": dev_ms, "host_ms": host}),
              flush=True)
        dist.barrier(device_ids=[local])
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
