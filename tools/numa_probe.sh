nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader
BDF=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-Z' 'a-z' | sed 's/^0000//; s/^\(....\):/\1:/')
ls /sys/bus/pci/devices/ | grep -i "$(echo $BDF | cut -c5-)" | head -3
for d in /sys/bus/pci/devices/*; do if [ -f $d/numa_node ] && [ "$(cat $d/vendor)" = "0x10de" ] && [ "$(cat $d/class | cut -c1-6)" = "0x0302" ]; then echo "$d numa=$(cat $d/numa_node) cpus=$(cat $d/local_cpulist)"; fi; done
nproc; cat /sys/devices/system/node/online; for n in /sys/devices/system/node/node*; do echo "$n $(cat $n/cpulist)"; done
python -c "import os; print('affinity', sorted(os.sched_getaffinity(0))[:8], len(os.sched_getaffinity(0)))"
which numactl taskset
