"""Sustained HBM copy bandwidth and clocks under load (is HBM throttled under the power cap?).
Runs b.copy_(a) over 2 x 4 GiB back to back for ~8 s, timing every 10 copies with CUDA events,
while nvidia-smi samples SM / memory clocks and power."""
import subprocess
import time

import torch

n = 1 << 30                                           # 1 Gi fp32 = 4 GiB
a = torch.empty(n, device="cuda", dtype=torch.float32).uniform_()
b = torch.empty_like(a)
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.active",
                        "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, text=True)
time.sleep(1.5)
res = []
t_end = time.time() + 8
while time.time() < t_end:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        b.copy_(a)
    e1.record()
    e1.synchronize()
    res.append(10 * 2 * 4 * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
smi.terminate()
lines = smi.communicate()[0].strip().splitlines()
print("copy GB/s per 10-copy batch:", [round(x) for x in res])
print("nvidia-smi samples (sm MHz, mem MHz, W, reasons):")
for l in lines[::4]:
    print("  ", l)
