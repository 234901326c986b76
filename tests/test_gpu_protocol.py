"""The peer-control protocol (RAFI_CONTROL_PEER) on one GPU.

Across GPUs, the count exchange (a5) and the completion barrier of
a FUSED forward run inside kernels: each process pushes its count rows into
every peer's CUDA-IPC mailbox, fences once, raises a flag, and spins with
ld.acquire.sys until every peer's flag is up (kernels.cu, ctl_counts_block /
ctl_barrier_block).  Processes on one GPU cannot run that protocol (nothing
co-schedules their kernels), so rafi_selftest_peer_control runs the SAME
device functions with P co-resident blocks of one cooperative launch, each
block playing one process with its own mailbox and its own copy of the
matrix, over several rounds (the per-round epochs), and with one process
missing (the timeout path must give up without trapping).
"""
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_2605_30294_b200 import rafi  # noqa: E402


@pytest.mark.parametrize("P,L", [(2, 1), (3, 2), (4, 1), (8, 1), (8, 4), (16, 2), (64, 1), (128, 2)])
def test_peer_protocol_rounds(P, L):
    bad, timed_out = rafi.selftest_peer_control(P, L, rounds=6, timeout_ms=20000)
    assert bad == 0 and timed_out == 0


@pytest.mark.parametrize("P,absent", [(2, 1), (4, 0), (8, 5)])
def test_peer_protocol_missing_process_times_out(P, absent):
    """A process that never arrives: every other one gives up after the
    timeout and flags it (RAFI_OPT_PEER_TIMEOUT_MS) instead of trapping; the
    CUDA context stays usable afterwards."""
    bad, timed_out = rafi.selftest_peer_control(P, 1, rounds=3, absent=absent, timeout_ms=200)
    assert bad == 0 and timed_out == P - 1
    x = torch.arange(1000, device="cuda")      # the context is healthy
    assert int(x.sum().item()) == 499500
    bad, timed_out = rafi.selftest_peer_control(P, 1, rounds=2, timeout_ms=20000)
    assert bad == 0 and timed_out == 0


def test_peer_protocol_rejects_unbounded_wait_on_missing_process():
    with pytest.raises(rafi.RafiError):
        rafi.selftest_peer_control(4, 1, rounds=1, absent=2, timeout_ms=0)


def test_peer_timeout_option_roundtrip():
    with rafi.Context(16, 100) as ctx:
        assert ctx.get_option(rafi.OPT_PEER_TIMEOUT_MS) == 20000
        ctx.set_option(rafi.OPT_PEER_TIMEOUT_MS, 0)
        assert ctx.get_option(rafi.OPT_PEER_TIMEOUT_MS) == 0
        with pytest.raises(rafi.RafiError):
            ctx.set_option(rafi.OPT_PEER_TIMEOUT_MS, -1)
