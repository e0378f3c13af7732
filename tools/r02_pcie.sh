#!/bin/bash
# PCIe counters of the a6 copy kernels (ncu), VERDICT r1 weak #8
TAG=${TAG:-r02_vX}
mkdir -p gpurun_out
ncu --query-metrics 2>/dev/null | grep -i -E "pcie" > gpurun_out/${TAG}_pcie_metrics.txt
M=$(grep -o -E "^pcie__[A-Za-z0-9_]+" gpurun_out/${TAG}_pcie_metrics.txt | sort -u | sed 's/$/.sum/' | paste -sd, -)
echo "metrics: $M"
timeout 900 ncu --metrics ${M}${M:+,}gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:k_copy_pages -s 40 -c 12 --csv --log-file gpurun_out/${TAG}_pcie.csv python tools/xfer_probe.py > gpurun_out/${TAG}_pcie_run.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/${TAG}_pcie_run.log; head -c 3000 gpurun_out/${TAG}_pcie.csv
