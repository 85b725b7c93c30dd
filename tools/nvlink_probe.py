#!/usr/bin/env python
"""Which NVLink byte counters does this driver expose?  Copies a known number
of bytes from GPU 0 to GPU 1 (peer copy over NVLink) and reads, before and
after: the NVML field values NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_{TX,RX} per link
and with the all-links scope, and `nvidia-smi nvlink -gt d`.  Prints one JSON
line per method with the counted bytes next to the copied bytes, so
tools/nvlink_phases.py can use the method that counts.  Needs 2 GPUs.
"""

import json
import re
import subprocess

import torch


def smi_bytes(i):
    try:
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(i)], capture_output=True, text=True,
                             timeout=20).stdout
    except Exception as ex:  # pragma: no cover
        return None, repr(ex)
    tx = rx = 0
    for ln in out.splitlines():
        m = re.search(r"Link \d+: Data Tx: (\d+) KiB", ln)
        if m:
            tx += int(m.group(1))
        m = re.search(r"Link \d+: Data Rx: (\d+) KiB", ln)
        if m:
            rx += int(m.group(1))
    return (tx * 1024, rx * 1024), out[:400]


def nvml_fields(h, nv, scope_all):
    f = [nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX]
    req = [(x, 0xFFFFFFFF) for x in f] if scope_all else [(x, l) for x in f for l in range(18)]
    vals = nv.nvmlDeviceGetFieldValues(h, req)
    tx = rx = 0
    rets = set()
    for (fid, _), v in zip(req, vals):
        rets.add(int(v.nvmlReturn))
        if v.nvmlReturn != 0:
            continue
        if fid == f[0]:
            tx += int(v.value.ullVal)
        else:
            rx += int(v.value.ullVal)
    return (tx * 1024, rx * 1024), sorted(rets)


def main():
    import pynvml as nv
    nv.nvmlInit()
    hs = [nv.nvmlDeviceGetHandleByIndex(i) for i in range(2)]
    nbytes = 4 << 30
    a = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0").fill_(1)
    b = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    torch.cuda.synchronize()
    before = {"smi": [smi_bytes(i)[0] for i in range(2)],
              "nvml_links": [nvml_fields(h, nv, False)[0] for h in hs],
              "nvml_all": [nvml_fields(h, nv, True)[0] for h in hs]}
    for _ in range(4):
        b.copy_(a)
    torch.cuda.synchronize()
    after = {"smi": [smi_bytes(i)[0] for i in range(2)],
             "nvml_links": [nvml_fields(h, nv, False)[0] for h in hs],
             "nvml_all": [nvml_fields(h, nv, True)[0] for h in hs]}
    print(json.dumps({"copied_bytes": 4 * nbytes, "smi_sample": smi_bytes(0)[1],
                      "nvml_returns": [nvml_fields(hs[0], nv, False)[1], nvml_fields(hs[0], nv, True)[1]]}))
    for m in before:
        d = []
        for i in range(2):
            if before[m][i] is None or after[m][i] is None:
                d.append(None)
            else:
                d.append([after[m][i][0] - before[m][i][0], after[m][i][1] - before[m][i][1]])
        print(json.dumps({"method": m, "gpu0_tx_rx": d[0], "gpu1_tx_rx": d[1]}))


if __name__ == "__main__":
    main()
