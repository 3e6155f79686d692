"""Measure the dense INT8 tensor ceiling on this B200 with the library GEMM torch._int_mm
(cuBLASLt IMMA), 8192^3, same method as MEASURED_PEAKS.json's bf16 figure: best of 10
(burst) and back-to-back for ~4 s (sustained).  Writes a JSON line to stdout."""
import json
import time

import torch

N = 8192
a = torch.randint(-128, 127, (N, N), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (N, N), dtype=torch.int8, device="cuda").t().contiguous().t()
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); torch._int_mm(a, b); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 1e3)
iters = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.time()
e0.record()
while time.time() - t0 < 4.0:
    for _ in range(20):
        torch._int_mm(a, b)
    iters += 20
    torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
sus = e0.elapsed_time(e1) / 1e3 / iters
ops = 2.0 * N ** 3
print(json.dumps({"int8_tops": round(ops / best / 1e12, 1), "int8_tops_sustained": round(ops / sus / 1e12, 1),
                  "how": "torch._int_mm int8 8192^3 (2*N^3 ops): best of 10 (burst), back to back 4 s (sustained)"}))
