mkdir -p gpurun_out
{ nvidia-smi topo -m; nproc; lscpu | grep -iE "numa|socket|model name"; cat /sys/bus/pci/devices/$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | tr 'A-F' 'a-f' | sed 's/^0000//;s/^/0000/' | cut -c1-12)/local_cpulist; nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader; ls /sys/devices/system/node/ | head; python -c "import os; print(sorted(os.sched_getaffinity(0)))"; } > gpurun_out/numa.txt 2>&1
echo done
