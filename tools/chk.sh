#!/bin/bash
# One gpurun call: full GPU test suite + numeric re-setup timing (+ optional extra command).  Usage: TAG [extra]
TAG=${1:-chk}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
python tools/time_update.py > gpurun_out/${TAG}_time.log 2>&1
AMGF_SETUP_TIMING=1 python tools/time_update.py > gpurun_out/${TAG}_time_ph.log 2>&1
if [ -n "$2" ]; then eval "$2"; fi
tail -3 gpurun_out/${TAG}_tests.log; tail -4 gpurun_out/${TAG}_time.log
