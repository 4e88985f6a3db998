# NUMA layout of the GPU box and pinned-memory H2D bandwidth per CPU node
nvidia-smi topo -m 2>&1 | head -8
lscpu | grep -i "numa\|socket\|^CPU(s)" 
BDF=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-F' 'a-f' | sed 's/^0000//;s/^/0000/')
echo "gpu bdf $BDF"; ls /sys/bus/pci/devices/ | grep -i "${BDF#0000:}" ; for d in /sys/bus/pci/devices/*; do if [ "$(cat $d/vendor 2>/dev/null)" = "0x10de" ] && [ "$(cat $d/class)" = "0x030200" ]; then echo "$d numa=$(cat $d/numa_node) cpus=$(cat $d/local_cpulist)"; fi; done
for node in /sys/devices/system/node/node*; do echo "$node cpus=$(cat $node/cpulist)"; done
cat > /tmp/h2d.py <<'PY'
import os, sys, torch, time, json
n = 1 << 29
h = torch.empty(n, dtype=torch.float32, pin_memory=True); h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
best = 0
for _ in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    best = max(best, n * 4 / (time.perf_counter() - t) / 1e9)
print(json.dumps({"cpus": sys.argv[1], "h2d_GBps": round(best, 1)}))
PY
for node in /sys/devices/system/node/node*; do c=$(cat $node/cpulist); taskset -c $c python /tmp/h2d.py "$c"; done
python /tmp/h2d.py any
