#!/bin/bash
# Host facts of the GPU box (cores, NUMA, RAM, topology) -> gpurun_out/box_info.txt
mkdir -p gpurun_out
{
  echo "== lscpu"; lscpu
  echo "== numa nodes"; for n in /sys/devices/system/node/node*; do echo "$n: $(cat $n/cpulist)"; done
  echo "== gpu numa"; cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c
  echo "== affinity"; python -c 'import os; print(sorted(os.sched_getaffinity(0)))'
  echo "== free"; free -g
  echo "== topo"; nvidia-smi topo -m
  echo "== numba"; python -c 'import numba; print(numba.__version__)' 2>&1
  echo "== thp"; cat /sys/kernel/mm/transparent_hugepage/enabled
} > gpurun_out/box_info.txt 2>&1
