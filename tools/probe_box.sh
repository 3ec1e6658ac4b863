#!/bin/bash
# One-off probe of the GPU box: host RAM, cores, NUMA, PCIe, H2D bandwidth.
mkdir -p gpurun_out
{
nvidia-smi; nvidia-smi topo -m; free -g; nproc; lscpu | head -30; ulimit -a;
cat /sys/fs/cgroup/memory.max 2>/dev/null; cat /proc/meminfo | head -5
nvidia-smi -q | grep -iA3 "PCIe Generation\|Link Width" | head -20
python - <<'PY'
import torch, time
x = torch.empty(256<<20, dtype=torch.uint8, pin_memory=True)
y = torch.empty(256<<20, dtype=torch.uint8, device='cuda')
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
best=1e9
for _ in range(10):
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); y.copy_(x, non_blocking=True); e.record(); e.synchronize()
    best=min(best, s.elapsed_time(e))
print("H2D GB/s", (256<<20)/best/1e6)
best=1e9
for _ in range(10):
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); x.copy_(y, non_blocking=True); e.record(); e.synchronize()
    best=min(best, s.elapsed_time(e))
print("D2H GB/s", (256<<20)/best/1e6)
print(torch.cuda.get_device_properties(0))
PY
} > gpurun_out/probe.txt 2>&1
cat gpurun_out/probe.txt | head -150
