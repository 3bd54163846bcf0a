"""Measure the dense TF32 tensor peak (torch.matmul fp32 with TF32 enabled,
8192^3, CUDA events) the way MEASURED_PEAKS.json measures bf16; the 3xTF32
FP32-grade ceiling is this peak / 3.  Writes gpurun_out/tf32_peak.json."""
import json
import os
import time

import torch

torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
best = 0.0
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    a @ b
    e.record()
    e.synchronize()
    best = max(best, 2 * n**3 / (s.elapsed_time(e) * 1e-3) / 1e12)
# sustained: back to back for ~4 s
t0 = time.time()
cnt = 0
s = torch.cuda.Event(enable_timing=True)
e = torch.cuda.Event(enable_timing=True)
s.record()
while time.time() - t0 < 4.0:
    a @ b
    cnt += 1
e.record()
e.synchronize()
sus = 2 * n**3 * cnt / (s.elapsed_time(e) * 1e-3) / 1e12
# fp32 SIMT (TF32 off) for reference
torch.backends.cuda.matmul.allow_tf32 = False
a @ b
torch.cuda.synchronize()
s.record()
for _ in range(3):
    a @ b
e.record()
e.synchronize()
fp32 = 3 * 2 * n**3 / (s.elapsed_time(e) * 1e-3) / 1e12
out = {"tf32_tflops": round(best, 1), "tf32_tflops_sustained": round(sus, 1), "fp32_simt_tflops": round(fp32, 1),
       "gpu": torch.cuda.get_device_name(), "how": "torch.matmul fp32 8192^3, allow_tf32 (burst best of 10, "
       "sustained 4 s); fp32 with TF32 off for the SIMT figure", "when": time.strftime("%Y-%m-%dT%H:%M:%SZ",
                                                                                          time.gmtime())}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/tf32_peak.json", "w"), indent=1)
print(json.dumps(out))
