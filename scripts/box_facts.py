"""Host and NVLink facts of a GPU box (measurement helper, not product).

    python scripts/box_facts.py > gpurun_out/facts.json

Records nproc, CPU model, RAM, GPU count and whether NVML exposes the NVLink
data-throughput counters (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX) used to
confirm that exchange bytes crossed NVLink.
"""
import json
import os
import subprocess


def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=60).stdout.strip()
    except Exception as e:  # noqa: BLE001
        return "error: %s" % e


facts = {
    "nproc": os.cpu_count(),
    "affinity": len(os.sched_getaffinity(0)),
    "cpu_model": sh("lscpu | grep 'Model name' | head -1 | cut -d: -f2").strip(),
    "numa": sh("lscpu | grep -i 'NUMA node(s)'"),
    "mem": sh("free -g | head -2"),
    "gpus": sh("nvidia-smi --query-gpu=index,name,memory.total --format=csv,noheader"),
    "topo": sh("nvidia-smi topo -m | head -12"),
}
try:
    import pynvml as N
    N.nvmlInit()
    h = N.nvmlDeviceGetHandleByIndex(0)
    out = {}
    for name in ("NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES",
                 "NVML_FI_DEV_NVLINK_COUNT_XMIT_PACKETS", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX",
                 "NVML_FI_DEV_NVLINK_LINK_COUNT"):
        fid = getattr(N, name)
        res = []
        for scope in (0xFFFFFFFF, 0, 1, 17):
            try:
                v = N.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
                res.append({"scope": scope, "ret": int(v.nvmlReturn), "type": int(v.valueType),
                            "ull": int(v.value.ullVal)})
            except Exception as e:  # noqa: BLE001
                res.append({"scope": scope, "err": str(e)})
        out[name] = res
    facts["nvml_nvlink"] = out
except Exception as e:  # noqa: BLE001
    facts["nvml_nvlink"] = "error: %s" % e
print(json.dumps(facts, indent=1))
