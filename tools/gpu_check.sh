#!/bin/bash
# One gpurun call: parity subset, timing A/B, ncu launch list of one apply (cfg 3).  Usage: tools/gpu_check.sh TAG [pytest -k expr]
TAG=${1:-chk}; K=${2:-"cfg3 or parity_cfg2 or golden"}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
python tools/time_apply.py 3 > gpurun_out/${TAG}_time.jsonl 2>&1
AMGF_NO_SLICE_BALANCE=1 python tools/time_apply.py 3 >> gpurun_out/${TAG}_time.jsonl 2>&1
ncu --nvtx --nvtx-include "apply/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_apply_launches.csv python tools/profile_apply.py 3 > gpurun_out/${TAG}_ncu.log 2>&1
python tools/launches.py gpurun_out/${TAG}_apply_launches.csv > gpurun_out/${TAG}_apply_launches.txt 2>&1
tail -3 gpurun_out/${TAG}_tests.log; cat gpurun_out/${TAG}_time.jsonl | cut -c1-300
