#!/bin/bash
# One-shot box probe: host CPU, FP64 peaks (DMMA/DFMA loops + cuBLAS DGEMM via torch).
set -x
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
./tools/probe_fp64
python - <<'PY'
import torch, time
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device='cuda'); b = torch.randn(n, n, dtype=torch.float64, device='cuda')
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"cublas dgemm {n}^3: {2*n**3/best/1e9:.2f} TFLOP/s ({best:.2f} ms)")
x = torch.empty(1 << 30, dtype=torch.float64, device='cuda'); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print(f"copy 8 GiB: {2*8*(1<<30)/best/1e6:.1f} GB/s")
PY
