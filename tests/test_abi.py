"""The C-ABI library loads and exports every symbol include/rafi.h declares;
host-side planning (rafi_plan) agrees with the oracle.  CPU only."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import synth
from paper_2605_30294_b200 import rafi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    names = set()
    for h in ("rafi.h", "rafi_drivers.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        names |= set(re.findall(r"\b(rafi_[a-z0-9_]+)\s*\(", txt))
    return sorted(names)


@pytest.fixture(scope="module")
def L():
    from paper_2605_30294_b200 import build
    build.build()
    return rafi.lib()


def test_every_declared_symbol_is_exported(L):
    names = header_functions()
    assert len(names) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", rafi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (rafi_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    # the binding declares exactly the header's functions
    assert sorted(rafi.SIGNATURES) == names


def test_library_is_sm100a_and_links_one_nccl(L):
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", rafi.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "sm_100a" in sass
    deps = subprocess.run(["ldd", rafi.LIB_PATH], capture_output=True, text=True).stdout
    assert "libnccl.so.2" in deps and "libcudart" not in deps   # cudart static, NCCL = torch's


def test_status_strings_and_version(L):
    assert L.rafi_abi_version() == 2
    assert L.rafi_status_str(0) == b"RAFI_OK"
    assert L.rafi_status_str(rafi.ERR_RECV_OVERFLOW) == b"RAFI_ERR_RECV_OVERFLOW"


def test_create_rejects_bad_args_without_gpu(L):
    h = ctypes.c_void_p()
    assert L.rafi_create(ctypes.byref(h), 0, 16, None, None) == rafi.ERR_INVALID_ARG
    assert L.rafi_create(ctypes.byref(h), 16, 1 << 32, None, None) == rafi.ERR_INVALID_ARG


def test_struct_layouts_match_header(L, tmp_path):
    """ctypes mirrors of the header's structs match what a C compiler lays out."""
    structs = {"rafi_device_view": rafi.DeviceView, "rafi_create_params": rafi.CreateParams,
               "rafi_stats": rafi.Stats}
    rename = {"in_": "in"}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "rafi.h"', "int main(void){"]
    for cname, py in structs.items():
        lines.append('printf("%%s %%zu\\n", "%s", sizeof(%s));' % (cname, cname))
        for f, _ in py._fields_:
            lines.append('printf("%%s.%%s %%zu\\n", "%s", "%s", offsetof(%s, %s));' % (cname, f, cname, rename.get(f, f)))
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = dict(l.rsplit(" ", 1) for l in subprocess.check_output([str(exe)]).decode().split("\n") if l)
    for cname, py in structs.items():
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got["%s.%s" % (cname, f)]) == getattr(py, f).offset, (cname, f)


@pytest.mark.parametrize("trial", range(25))
def test_plan_matches_oracle(L, trial):
    rng = np.random.default_rng(trial)
    R = int(rng.integers(1, 9))
    B = 16
    n = int(rng.integers(0, 60))
    w = oracle.World(R, n * R + 1, B)
    for s in range(R):
        it = synth.make_items(s, 0, n, B)
        ds = synth.make_dests(str(rng.choice(["uniform", "skewed", "ring"])), trial, s, 0, n, R)
        for i in range(n):
            w.emit(s, it[i].tobytes(), int(ds[i]))
    G = w.forward()
    Cm = w.C()
    for d in range(R):
        p = rafi.plan(Cm, w.cap, d)
        assert list(p["recv_off"]) == list(w.recv_off()[d])
        assert list(p["src_off"]) == list(w.send_off()[:, d])
        assert list(p["recv_count"]) == list(Cm[:, d])
        assert p["total"] == w.num_incoming(d)
        assert p["G"] == G and not p["overflow"]


def test_plan_overflow_is_global(L):
    Cm = np.array([[0, 3], [0, 2]], np.uint64)   # rank 1 would receive 5 > 4
    for d in range(2):
        assert rafi.plan(Cm, 4, d)["overflow"]     # every rank decides alike (Z3)
    assert not rafi.plan(Cm, 5, 0)["overflow"]


def test_binding_constants_match_header():
    """Every status code and option value the Python binding names equals the
    #define in include/rafi.h (the binding is marshalling only)."""
    txt = open(os.path.join(ROOT, "include", "rafi.h")).read()
    defs = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define RAFI_([A-Z0-9_]+)\s+\(?(-?\d+)\)?", txt)}
    defs.update({m.group(1): int(m.group(2)) for m in re.finditer(r"\bRAFI_([A-Z0-9_]+)\s*=\s*(-?\d+)", txt)})
    names = [n for n in dir(rafi) if re.fullmatch(r"(ERR_[A-Z_]+|OPT_[A-Z_]+|EXCHANGE_[A-Z]+|SCATTER_[A-Z]+|"
                                                 r"CONTROL_[A-Z]+|OK)", n)]
    assert len(names) >= 25
    for n in names:
        assert n in defs, "RAFI_%s missing from rafi.h" % n
        assert getattr(rafi, n) == defs[n], n
    for prefix in ("OPT_", "EXCHANGE_", "SCATTER_", "CONTROL_"):
        for d in defs:
            if d.startswith(prefix):
                assert hasattr(rafi, d), "binding lacks %s" % d
