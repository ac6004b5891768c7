#!/bin/bash
# Box probe: host topology, memory limits, PCIe link state.
set -x
nproc; lscpu | head -30
free -g; df -h /dev/shm /tmp; ulimit -l; ulimit -a
grep -i huge /proc/meminfo; cat /sys/kernel/mm/transparent_hugepage/enabled
which numactl lspci nsys; numactl -H 2>/dev/null
ls /sys/devices/system/node/
nvidia-smi; nvidia-smi topo -m
nvidia-smi -q | grep -iE -A2 'PCIe Generation|Link Width|Bus Id|Max Link|Current' | head -80
cat /proc/cmdline
dmesg 2>/dev/null | grep -i iommu | head
ls /sys/class/iommu 2>/dev/null
python - <<'PY'
import torch, time
print(torch.cuda.get_device_properties(0))
p = torch.cuda.get_device_properties(0)
print("sms", p.multi_processor_count)
for mb in (64, 256, 1024):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    print(f"H2D {mb} MiB: {10*n/ (s.elapsed_time(e)*1e-3)/1e9:.2f} GB/s")
    s.record()
    for _ in range(10): h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    print(f"D2H {mb} MiB: {10*n/ (s.elapsed_time(e)*1e-3)/1e9:.2f} GB/s")
PY
