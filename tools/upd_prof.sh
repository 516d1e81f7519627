#!/bin/bash
# One gpurun call: GPU tests, update_D timing (overlapped and serial), update_D launch list.  Usage: TAG
TAG=${1:-u}
bash tools/chk.sh $TAG "ncu --nvtx --nvtx-include 'upd/' --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_upd_launches.csv python tools/profile_update.py > /dev/null 2>&1; python tools/launches.py gpurun_out/${TAG}_upd_launches.csv > gpurun_out/${TAG}_upd_launches.txt; AMGF_SERIAL_SETUP=1 AMGF_SETUP_TIMING=1 python tools/time_update.py > gpurun_out/${TAG}_serial.log 2>&1"
grep "update_D ms" gpurun_out/${TAG}_time_ph.log | tail -1; grep "update_D ms" gpurun_out/${TAG}_serial.log | tail -1
