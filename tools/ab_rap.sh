#!/bin/bash
TAG=$1
bash tools/upd_prof.sh $TAG
for V in r64 r80n4; do
  AMGF_LIB=libamgf_$V.so AMGF_SETUP_TIMING=1 python tools/time_update.py > gpurun_out/${TAG}_$V.log 2>&1
  AMGF_LIB=libamgf_$V.so ncu --nvtx --nvtx-include "upd/" --metrics gpu__time_duration.sum --clock-control none -k regex:k_gal_rap2 --csv python tools/profile_update.py 2>/dev/null | grep k_gal_rap2 | tail -1 >> gpurun_out/${TAG}_$V.log
done
