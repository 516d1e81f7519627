#!/bin/bash
# ncu --set full (+source) of the named kernels during one cfg 3 update_D.  Usage: TAG regex1 [regex2 ...]
TAG=$1; shift
mkdir -p gpurun_out
python tools/time_update.py > gpurun_out/${TAG}_time.log 2>&1
AMGF_SETUP_TIMING=1 python tools/time_update.py > gpurun_out/${TAG}_time_ph.log 2>&1
ncu --nvtx --nvtx-include "upd/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_upd_launches.csv python tools/profile_update.py > /dev/null 2>&1
python tools/launches.py gpurun_out/${TAG}_upd_launches.csv > gpurun_out/${TAG}_upd_launches.txt
i=0
for K in "$@"; do
  i=$((i+1))
  ncu --nvtx --nvtx-include "upd/" --set full --import-source on --clock-control none -k regex:"$K" -c 1 \
      -o gpurun_out/${TAG}_k$i python tools/profile_update.py > /dev/null 2>&1
  ncu -i gpurun_out/${TAG}_k$i.ncu-rep --page details --csv > gpurun_out/${TAG}_k${i}_details.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_k$i.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/${TAG}_k${i}_source.csv 2>/dev/null
done
grep "update_D ms" gpurun_out/${TAG}_time_ph.log | tail -2
