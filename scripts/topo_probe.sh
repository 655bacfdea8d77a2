#!/bin/bash
# Box topology for the host-path (e2e) design: CPU/NUMA layout, the GPU's
# PCIe link and NUMA node, and host memory.
set +e
lscpu | egrep "Model name|Socket|NUMA|^CPU\(s\)|Thread|Core"
echo "affinity: $(python -c 'import os; print(len(os.sched_getaffinity(0)), sorted(os.sched_getaffinity(0))[:4], "...")')"
free -g | head -2
nvidia-smi topo -m 2>/dev/null | head -20
for d in /sys/bus/pci/devices/*; do
  if [ "$(cat $d/vendor 2>/dev/null)" = "0x10de" ] && [ "$(cat $d/class 2>/dev/null | cut -c1-6)" = "0x0302" ]; then
    echo "$d numa_node=$(cat $d/numa_node) local_cpulist=$(cat $d/local_cpulist) link=$(cat $d/current_link_speed 2>/dev/null) x$(cat $d/current_link_width 2>/dev/null)"
  fi
done
nvidia-smi --query-gpu=index,pci.bus_id,pcie.link.gen.current,pcie.link.width.current --format=csv
