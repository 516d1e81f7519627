#!/bin/bash
# A/B of update_D timing across library variants: tools/ab_upd.sh TAG kernel_regex variant...
TAG=$1; K=$2; shift 2
for V in "" "$@"; do
  L=${V:+libamgf_$V.so}
  AMGF_LIB=$L AMGF_SETUP_TIMING=1 python tools/time_update.py > gpurun_out/${TAG}_${V:-base}.log 2>&1
  AMGF_LIB=$L ncu --nvtx --nvtx-include "upd/" --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" --csv \
      python tools/profile_update.py 2>/dev/null | grep -v "^==" | awk -F'","' '{print $5, $NF}' >> gpurun_out/${TAG}_${V:-base}.log
  echo "${V:-base}: $(grep 'update_D ms' gpurun_out/${TAG}_${V:-base}.log | tail -1)"; grep -v "update_D\|step\|alone" gpurun_out/${TAG}_${V:-base}.log | tail -3
done
