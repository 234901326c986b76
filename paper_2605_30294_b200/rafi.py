"""ctypes binding of librafi (include/rafi.h) -- argument marshalling only.

Every step of the forwarding path runs in librafi's CUDA kernels; this module
only converts Python/torch/numpy arguments to plain pointers and sizes.  There
is no fallback: if librafi.so is missing or fails to load, importing this
module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RAFI_LIB_PATH selects a tuning variant built by `build.py --variants` (benchmarks only)
LIB_PATH = os.environ.get("RAFI_LIB_PATH") or os.path.join(_HERE, "librafi.so")

OK = 0
ERR_INVALID_ARG = -1
ERR_CUDA = -2
ERR_NCCL = -3
ERR_NOMEM = -4
ERR_RECV_OVERFLOW = -5
ERR_STATE = -6
ERR_UNSUPPORTED = -7
ERR_TIMEOUT = -8
ERR_BOOTSTRAP = -9

OPT_EXCHANGE = 1
OPT_TIMING = 2
OPT_TILE = 3
OPT_SELF_DIRECT = 4
OPT_SCATTER = 5
OPT_CONTROL = 7
OPT_FORWARD_GRAPH = 8
OPT_PEER_TIMEOUT_MS = 9
CONTROL_AUTO, CONTROL_NCCL, CONTROL_PEER, CONTROL_HOST = 0, 1, 2, 3
SCATTER_AUTO, SCATTER_THREADS, SCATTER_BULK = 0, 1, 2
EXCHANGE_AUTO, EXCHANGE_NCCL, EXCHANGE_PEER, EXCHANGE_FUSED = 0, 1, 2, 3


class DeviceView(C.Structure):
    _fields_ = [
        ("in_", C.c_void_p), ("num_in", C.c_uint64), ("num_in_dev", C.c_void_p),
        ("out", C.c_void_p), ("dest", C.c_void_p), ("ctr", C.c_void_p), ("invalid", C.c_void_p),
        ("capacity", C.c_uint64), ("item_bytes", C.c_uint32), ("num_ranks", C.c_int32),
        ("my_rank", C.c_int32), ("reserved", C.c_int32),
    ]


class CreateParams(C.Structure):
    _fields_ = [
        ("item_bytes", C.c_size_t), ("capacity", C.c_size_t), ("nccl_comm", C.c_void_p),
        ("stream", C.c_void_p), ("local_ranks", C.c_int), ("device", C.c_int),
    ]


# int (*rafi_allgather_fn)(void* user, const void* send, void* recv, size_t bytes)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)


class Bootstrap(C.Structure):
    _fields_ = [("nprocs", C.c_int), ("proc", C.c_int), ("allgather", ALLGATHER_FN), ("user", C.c_void_p)]


def torch_allgather(group=None):
    """A rafi_allgather_fn over a torch.distributed CPU (gloo) group: plumbing
    for rafi_create_boot (the host transport the paper uses MPI for)."""
    import torch
    import torch.distributed as dist

    def fn(user, send, recv, nbytes):
        try:
            world = dist.get_world_size(group)
            src = torch.zeros(max(nbytes, 1), dtype=torch.uint8)
            if nbytes:
                C.memmove(src.data_ptr(), send, nbytes)
            outs = [torch.empty_like(src) for _ in range(world)]
            dist.all_gather(outs, src, group=group)
            for p, o in enumerate(outs):
                if nbytes:
                    C.memmove(recv + p * nbytes, o.data_ptr(), nbytes)
            return 0
        except Exception:  # noqa: BLE001  (reported to the library as a failed collective)
            return 1

    return fn


class Stats(C.Structure):
    _fields_ = [
        ("round", C.c_uint64), ("n_out", C.c_uint64), ("dropped", C.c_uint64), ("invalid", C.c_uint64),
        ("num_in", C.c_uint64), ("bytes_sent_remote", C.c_uint64), ("bytes_recv_remote", C.c_uint64),
        ("G", C.c_int64), ("num_ranks", C.c_int32), ("my_rank", C.c_int32),
        ("ms_hist", C.c_float), ("ms_scan", C.c_float), ("ms_scatter", C.c_float),
        ("ms_count_exchange", C.c_float), ("ms_payload_exchange", C.c_float), ("ms_wrapup", C.c_float),
        ("ms_total", C.c_float), ("ms_reserved", C.c_float),
        ("kernel_launches", C.c_uint64), ("forward_launches", C.c_uint64),
        ("acc_ms_emit", C.c_double), ("acc_ms_hist", C.c_double), ("acc_ms_scan", C.c_double),
        ("acc_ms_scatter", C.c_double), ("acc_ms_count_exchange", C.c_double),
        ("acc_ms_payload_exchange", C.c_double), ("acc_ms_wrapup", C.c_double), ("acc_ms_total", C.c_double),
        ("acc_forwards", C.c_uint64), ("acc_emits", C.c_uint64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "ms_reserved"}


# (restype, argtypes) of every exported symbol; tests check this list against include/rafi.h
SIGNATURES = {
    "rafi_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_size_t, C.c_size_t, C.c_void_p, C.c_void_p]),
    "rafi_create_ex": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(CreateParams)]),
    "rafi_create_boot": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(CreateParams), C.POINTER(Bootstrap)]),
    "rafi_selftest_peer_control": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_longlong,
                                             C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "rafi_drv_emit_items": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int]),
    "rafi_diag_redirect_incoming": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "rafi_resize": (C.c_int, [C.c_void_p, C.c_size_t]),
    "rafi_destroy": (None, [C.c_void_p]),
    "rafi_get_device_view": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(DeviceView)]),
    "rafi_num_incoming": (C.c_uint64, [C.c_void_p, C.c_int]),
    "rafi_emit_bulk": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64]),
    "rafi_forward": (C.c_int64, [C.c_void_p]),
    "rafi_num_ranks": (C.c_int, [C.c_void_p]),
    "rafi_local_ranks": (C.c_int, [C.c_void_p]),
    "rafi_rank_of": (C.c_int, [C.c_void_p, C.c_int]),
    "rafi_capacity": (C.c_uint64, [C.c_void_p]),
    "rafi_item_bytes": (C.c_uint64, [C.c_void_p]),
    "rafi_read_incoming": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_uint64]),
    "rafi_read_outgoing": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_uint64)]),
    "rafi_read_binned": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64]),
    "rafi_read_incoming_async": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_uint64]),
    "rafi_read_wait": (C.c_int, [C.c_void_p]),
    "rafi_get_matrix": (C.c_int, [C.c_void_p, C.c_void_p]),
    "rafi_get_stats": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(Stats)]),
    "rafi_set_option": (C.c_int, [C.c_void_p, C.c_int, C.c_longlong]),
    "rafi_get_option": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_longlong)]),
    "rafi_status_str": (C.c_char_p, [C.c_int]),
    "rafi_last_error": (C.c_char_p, []),
    "rafi_abi_version": (C.c_int, []),
    "rafi_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "rafi_nccl_comm_init": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_void_p, C.c_int]),
    "rafi_nccl_comm_destroy": (C.c_int, [C.c_void_p]),
    "rafi_drv_emit_synthetic": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint32, C.c_uint64,
                                          C.c_uint64, C.c_int, C.c_uint64]),
    "rafi_drv_random_walk": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32]),
    "rafi_drv_advect_seed": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int]),
    "rafi_drv_advect_step": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_float, C.c_float, C.c_float,
                                       C.c_int, C.c_int, C.c_int]),
    "rafi_drv_march_seed": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int]),
    "rafi_drv_march_step": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                      C.c_int, C.c_int, C.c_int, C.c_void_p]),
    "rafi_drv_nbody_seed": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64]),
    "rafi_drv_nbody_migrate": (C.c_int, [C.c_void_p, C.c_float]),
    "rafi_drv_nbody_stats": (C.c_int, [C.c_void_p, C.c_void_p]),
    "rafi_drv_nbody_root": (C.c_int, [C.c_void_p, C.c_void_p]),
    "rafi_drv_nbody_refine": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_float]),
    "rafi_drv_nbody_respond": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "rafi_drv_stream_create": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.POINTER(C.c_void_p)]),
    "rafi_drv_stream_seed": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_uint32]),
    "rafi_drv_stream_step": (C.c_int, [C.c_void_p, C.c_uint32, C.c_float, C.c_float, C.c_uint32, C.c_void_p,
                                       C.c_void_p]),
    "rafi_drv_stream_destroy": (C.c_int, [C.c_void_p]),
    "rafi_drv_stream_halo_misses": (C.c_int, [C.c_void_p, C.POINTER(C.c_int)]),
    "rafi_forward_async": (C.c_int, [C.c_void_p, C.c_void_p]),
    "rafi_sync_host": (C.c_int, [C.c_void_p]),
    "rafi_capture_begin": (C.c_int, [C.c_void_p]),
    "rafi_capture_end": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "rafi_graph_launch": (C.c_int, [C.c_void_p, C.c_void_p]),
    "rafi_graph_destroy": (C.c_int, [C.c_void_p]),
    "rafi_plan": (C.c_int, [C.c_int, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                            C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_int)]),
}

_lib = None


def lib():
    """Load librafi.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("librafi.so not built: run `python -m paper_2605_30294_b200.build` (%s)" % LIB_PATH)
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class RafiError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = lib().rafi_last_error().decode(errors="replace")
        super().__init__("%s: %s (%s)" % (where, lib().rafi_status_str(status).decode(), msg))


def _check(rc, where):
    if rc != OK:
        raise RafiError(rc, where)
    return rc


def _ptr(x):
    """Plain address of a torch tensor / numpy array / int (no copies)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data
    raise TypeError("unsupported buffer type %r" % type(x))


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream  # torch.cuda.Stream


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().rafi_nccl_unique_id(buf), "rafi_nccl_unique_id")
    return buf.raw


def nccl_comm_init(nranks: int, rank: int, uid: bytes, device: int = -1) -> int:
    comm = C.c_void_p()
    buf = C.create_string_buffer(bytes(uid), 128)
    _check(lib().rafi_nccl_comm_init(C.byref(comm), nranks, rank, buf, device), "rafi_nccl_comm_init")
    return comm.value


def nccl_comm_destroy(comm: int):
    _check(lib().rafi_nccl_comm_destroy(comm), "rafi_nccl_comm_destroy")


def selftest_peer_control(P: int, L: int, rounds: int, absent: int = -1, timeout_ms: int = 0, device: int = -1):
    """rafi_selftest_peer_control: returns (bad matrix entries, processes that timed out)."""
    bad, tout = C.c_uint64(), C.c_uint64()
    _check(lib().rafi_selftest_peer_control(device, P, L, rounds, absent, timeout_ms, C.byref(bad), C.byref(tout)),
           "rafi_selftest_peer_control")
    return bad.value, tout.value


def plan(C_matrix: np.ndarray, capacity: int, d: int):
    """Host-side plan for destination d from the R x R count matrix (rafi_plan)."""
    Cm = np.ascontiguousarray(C_matrix, dtype=np.uint64)
    R = Cm.shape[0]
    rc_, ro, so = (np.zeros(R, np.uint64) for _ in range(3))
    tot, G, ovf = C.c_uint64(), C.c_uint64(), C.c_int()
    _check(lib().rafi_plan(R, Cm.ctypes.data, capacity, d, rc_.ctypes.data, ro.ctypes.data, so.ctypes.data,
                           C.byref(tot), C.byref(G), C.byref(ovf)), "rafi_plan")
    return {"recv_count": rc_, "recv_off": ro, "src_off": so, "total": tot.value, "G": G.value,
            "overflow": bool(ovf.value)}


class StreamField:
    """Streamline proxy state (include/rafi_drivers.h, NEXT-4): per-rank field
    blocks with a one-vertex halo on the device."""

    def __init__(self, ctx: "Context", field: np.ndarray, grid):
        field = np.ascontiguousarray(field, dtype=np.float32)
        nz, ny, nx, three = field.shape
        assert three == 3
        h = C.c_void_p()
        _check(lib().rafi_drv_stream_create(ctx.handle, field.ctypes.data, nx, ny, nz, *grid, C.byref(h)),
               "rafi_drv_stream_create")
        self._h = h.value

    def seed(self, seeds: np.ndarray, id0: int, local: int = 0):
        seeds = np.ascontiguousarray(seeds, dtype=np.float32)
        _check(lib().rafi_drv_stream_seed(self._h, local, seeds.ctypes.data, seeds.shape[0], id0), "rafi_drv_stream_seed")

    def step(self, rnd, h, eps, max_steps, result_pos, result_steps):
        _check(lib().rafi_drv_stream_step(self._h, rnd, h, eps, max_steps, _ptr(result_pos), _ptr(result_steps)),
               "rafi_drv_stream_step")

    def halo_misses(self) -> int:
        v = C.c_int()
        _check(lib().rafi_drv_stream_halo_misses(self._h, C.byref(v)), "rafi_drv_stream_halo_misses")
        return v.value

    def close(self):
        if getattr(self, "_h", None):
            lib().rafi_drv_stream_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """One RaFI host context (HostContext<T>)."""

    def __init__(self, item_bytes: int, capacity: int, comm: int | None = None, stream=None,
                 local_ranks: int = 1, device: int = -1, bootstrap=None):
        """bootstrap: (nprocs, proc, allgather) for rafi_create_boot, where
        allgather is a Python callable (user, send, recv, nbytes) -> int such as
        torch_allgather(); None = rafi_create_ex (NCCL communicator only)."""
        p = CreateParams(item_bytes, capacity, comm, _stream_ptr(stream), local_ranks, device)
        h = C.c_void_p()
        if bootstrap is None:
            _check(lib().rafi_create_ex(C.byref(h), C.byref(p)), "rafi_create_ex")
        else:
            nprocs, proc, fn = bootstrap
            self._allgather = ALLGATHER_FN(fn)  # kept alive as long as the context
            b = Bootstrap(nprocs, proc, self._allgather, None)
            _check(lib().rafi_create_boot(C.byref(h), C.byref(p), C.byref(b)), "rafi_create_boot")
        self._h = h.value
        self.item_bytes = int(item_bytes)
        self.local_ranks = int(local_ranks)

    # -- lifecycle --------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().rafi_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def resize(self, capacity: int):
        _check(lib().rafi_resize(self._h, capacity), "rafi_resize")

    # -- properties ---------------------------------------------------------------
    @property
    def num_ranks(self):
        return lib().rafi_num_ranks(self._h)

    @property
    def capacity(self):
        return int(lib().rafi_capacity(self._h))

    def rank_of(self, local=0):
        return lib().rafi_rank_of(self._h, local)

    def set_option(self, key, value):
        _check(lib().rafi_set_option(self._h, key, int(value)), "rafi_set_option")

    def get_option(self, key):
        v = C.c_longlong()
        _check(lib().rafi_get_option(self._h, key, C.byref(v)), "rafi_get_option")
        return v.value

    def device_view(self, local=0) -> DeviceView:
        v = DeviceView()
        _check(lib().rafi_get_device_view(self._h, local, C.byref(v)), "rafi_get_device_view")
        return v

    # -- hot path ----------------------------------------------------------------
    def emit_bulk(self, items, dests, n: int | None = None, local: int = 0):
        if n is None:
            n = len(dests)
        _check(lib().rafi_emit_bulk(self._h, local, _ptr(items), _ptr(dests), int(n)), "rafi_emit_bulk")

    def diag_redirect_incoming(self, grank: int, queue=None):
        """rafi_diag_redirect_incoming: FUSED pushes for global rank `grank` go
        to `queue` (a device tensor, possibly on another GPU) until restored
        with queue=None.  Measurement only (see include/rafi.h)."""
        _check(lib().rafi_diag_redirect_incoming(self._h, grank, None if queue is None else _ptr(queue)),
               "rafi_diag_redirect_incoming")

    def forward(self) -> int:
        G = lib().rafi_forward(self._h)
        if G < 0:
            raise RafiError(int(G), "rafi_forward")
        return int(G)

    # N-body exchange pattern (three contexts; include/rafi_drivers.h)
    def drv_nbody_seed(self, n: int, seed: int, local: int = 0):
        _check(lib().rafi_drv_nbody_seed(self._h, local, n, seed), "rafi_drv_nbody_seed")

    def drv_nbody_migrate(self, dt: float):
        _check(lib().rafi_drv_nbody_migrate(self._h, dt), "rafi_drv_nbody_migrate")

    def drv_nbody_stats(self, stats_dev):
        _check(lib().rafi_drv_nbody_stats(self._h, _ptr(stats_dev)), "rafi_drv_nbody_stats")

    def drv_nbody_root(self, stats_dev):
        _check(lib().rafi_drv_nbody_root(self._h, _ptr(stats_dev)), "rafi_drv_nbody_root")

    def drv_nbody_refine(self, qctx: "Context", stats_dev, theta2: float):
        _check(lib().rafi_drv_nbody_refine(self._h, qctx._h, _ptr(stats_dev), theta2), "rafi_drv_nbody_refine")

    def drv_nbody_respond(self, vctx: "Context", stats_dev):
        _check(lib().rafi_drv_nbody_respond(self._h, vctx._h, _ptr(stats_dev)), "rafi_drv_nbody_respond")

    def forward_async(self, G_dev):
        """NEXT-3: enqueue a FUSED forward with no host sync; G lands in G_dev (device u64)."""
        _check(lib().rafi_forward_async(self._h, _ptr(G_dev)), "rafi_forward_async")

    def sync_host(self):
        _check(lib().rafi_sync_host(self._h), "rafi_sync_host")

    def capture_begin(self):
        _check(lib().rafi_capture_begin(self._h), "rafi_capture_begin")

    def capture_end(self) -> int:
        e = C.c_void_p()
        _check(lib().rafi_capture_end(self._h, C.byref(e)), "rafi_capture_end")
        return e.value

    def graph_launch(self, exec_handle: int):
        _check(lib().rafi_graph_launch(self._h, exec_handle), "rafi_graph_launch")

    @staticmethod
    def graph_destroy(exec_handle: int):
        _check(lib().rafi_graph_destroy(exec_handle), "rafi_graph_destroy")

    def forward_rc(self) -> int:
        """rafi_forward's raw return (G >= 0 or a negative status)."""
        return int(lib().rafi_forward(self._h))

    # -- proxy drivers (include/rafi_drivers.h) -----------------------------------
    def drv_emit_synthetic(self, pattern: int, seed: int, rnd: int, n: int, seq0: int = 0, target: int = 0,
                           invalid_threshold: int = 0, local: int = 0):
        _check(lib().rafi_drv_emit_synthetic(self._h, local, pattern, seed, rnd, n, seq0, target, invalid_threshold),
               "rafi_drv_emit_synthetic")

    def drv_emit_items(self, items, dests, n: int | None = None, local: int = 0, batch: int = 1):
        """Device re-emit of a resident batch through rafi::Queue<T>::emitOutgoing
        (batch = 1) or the batched emitOutgoing<8> (batch = 8)."""
        if n is None:
            n = len(dests)
        _check(lib().rafi_drv_emit_items(self._h, local, _ptr(items), _ptr(dests), int(n), int(batch)),
               "rafi_drv_emit_items")

    def drv_random_walk(self, seed: int, rnd: int, last_round: int):
        _check(lib().rafi_drv_random_walk(self._h, seed, rnd, last_round), "rafi_drv_random_walk")

    def drv_advect_seed(self, n: int, seed: int, grid, local: int = 0):
        _check(lib().rafi_drv_advect_seed(self._h, local, n, seed, *grid), "rafi_drv_advect_seed")

    def drv_advect_step(self, rnd: int, max_rounds: int, omega: float, eps: float, h: float, grid):
        _check(lib().rafi_drv_advect_step(self._h, rnd, max_rounds, omega, eps, h, *grid), "rafi_drv_advect_step")

    def drv_march_seed(self, n: int, seed: int, grid, local: int = 0):
        _check(lib().rafi_drv_march_seed(self._h, local, n, seed, *grid), "rafi_drv_march_seed")

    def drv_march_step(self, rnd: int, seed: int, p_thr: int, max_bounces: int, max_steps: int, grid, result):
        _check(lib().rafi_drv_march_step(self._h, rnd, seed, p_thr, max_bounces, max_steps, *grid, _ptr(result)),
               "rafi_drv_march_step")

    # -- introspection --------------------------------------------------------------
    def num_incoming(self, local=0) -> int:
        return int(lib().rafi_num_incoming(self._h, local))

    def read_incoming(self, local=0, first=0, count=None, out=None) -> np.ndarray:
        n = self.num_incoming(local)
        if count is None:
            count = n - first
        if out is None:
            out = np.empty((count, self.item_bytes), np.uint8)
        _check(lib().rafi_read_incoming(self._h, local, _ptr(out), first, count), "rafi_read_incoming")
        return out

    def read_incoming_async(self, out, local=0, first=0, count=None):
        """Enqueue the read-back of the incoming queue into `out` (pinned host or device)."""
        if count is None:
            count = self.num_incoming(local) - first
        _check(lib().rafi_read_incoming_async(self._h, local, _ptr(out), first, count), "rafi_read_incoming_async")
        return out

    def read_wait(self):
        _check(lib().rafi_read_wait(self._h), "rafi_read_wait")

    def read_outgoing(self, local=0, with_items=True):
        ctr, inv = C.c_uint64(), C.c_uint64()
        _check(lib().rafi_read_outgoing(self._h, local, None, None, C.byref(ctr), C.byref(inv)), "rafi_read_outgoing")
        n = min(ctr.value, self.capacity)
        items = np.empty((n, self.item_bytes), np.uint8)
        dests = np.empty(n, np.int32)
        _check(lib().rafi_read_outgoing(self._h, local, _ptr(items) if with_items else None, _ptr(dests),
                                        C.byref(ctr), C.byref(inv)), "rafi_read_outgoing")
        return items, dests, ctr.value, inv.value

    def read_binned(self, local=0, count=None) -> np.ndarray:
        if count is None:
            count = self.stats(local)["n_out"]
        out = np.empty((count, self.item_bytes), np.uint8)
        _check(lib().rafi_read_binned(self._h, local, _ptr(out), count), "rafi_read_binned")
        return out

    def matrix(self) -> np.ndarray:
        R = self.num_ranks
        m = np.zeros((R, R), np.uint64)
        _check(lib().rafi_get_matrix(self._h, m.ctypes.data), "rafi_get_matrix")
        return m

    def stats(self, local=0) -> dict:
        s = Stats()
        _check(lib().rafi_get_stats(self._h, local, C.byref(s)), "rafi_get_stats")
        return s.as_dict()
