"""Measured INT8 tensor-core peak on this B200 (cuBLASLt through torch._int_mm,
8192^3, best of 20 after warm-up) -> MEASURED_INT8.json. The roofline of the
Ozaki Gram kernel is quoted against it."""
import json
import os
import sys

import torch

n = 8192
a = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda")
for _ in range(5):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
tops = 2.0 * n ** 3 / (best / 1e3) / 1e12
out = {"int8_tops": round(tops, 1), "gpu_name": torch.cuda.get_device_name(0),
       "how": f"torch._int_mm (cuBLASLt) int8 {n}^3, int32 accumulate, best of 20 (CUDA events)",
       "nominal_int8_dense_tops": 4500.0}
print(json.dumps(out))
path = sys.argv[1] if len(sys.argv) > 1 else "MEASURED_INT8.json"
with open(path, "w") as f:
    json.dump(out, f, indent=1)
