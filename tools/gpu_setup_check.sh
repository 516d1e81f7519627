#!/bin/bash
# parity subset for the setup kernels + update_D timing and launch list (cfg 3)
TAG=${1:-setup}
python -m pytest tests -m gpu -x -q -k "setup_parity or factor or golden or update_D or cfg2 or import or edge or superset" > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
AMGF_SETUP_TIMING=1 python tools/time_update.py > gpurun_out/${TAG}_time.log 2>&1
ncu --nvtx --nvtx-include "upd/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/profile_update.py > gpurun_out/${TAG}_ncu.log 2>&1
python tools/launches.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches.txt
tail -3 gpurun_out/${TAG}_tests.log; tail -4 gpurun_out/${TAG}_time.log
