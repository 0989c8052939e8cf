"""Quick per-box check: device-to-device copy bandwidth (GB/s), SM/memory
clocks, and config B's frame time — to tell box-to-box variance from
regressions."""
import json
import subprocess
import sys

import torch

n = 1 << 30                      # 2 GiB per buffer (int16)
a = torch.empty(n, dtype=torch.int16, device="cuda")
b = torch.empty_like(a)
a.fill_(1)
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    b.copy_(a)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
smi = subprocess.run(["nvidia-smi", "--query-gpu=name,serial,clocks.sm,clocks.mem,clocks.max.mem,"
                      "power.limit,ecc.mode.current", "--format=csv,noheader"],
                     capture_output=True, text=True).stdout.strip()
print(json.dumps({"copy_GBps": 2 * 2 * n / ms / 1e6, "smi": smi}))
