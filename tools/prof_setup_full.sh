#!/bin/bash
# ncu --set full of the numeric re-setup's top kernels (cfg 3, one update_D) + the launch list.  Usage: TAG
TAG=${1:-su}
mkdir -p gpurun_out
python tools/time_update.py > gpurun_out/${TAG}_time.log 2>&1
ncu --nvtx --nvtx-include "upd/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_upd_launches.csv python tools/profile_update.py > /dev/null 2>&1
python tools/launches.py gpurun_out/${TAG}_upd_launches.csv > gpurun_out/${TAG}_upd_launches.txt
for K in "k_spgemm_dense" "k_P_values" "k_band_chol" "k_nd_gemm" "k_spgemm_vals_warp"; do
  ncu --nvtx --nvtx-include "upd/" --set full --import-source on --clock-control none -k regex:"$K" -c 2 \
      -o gpurun_out/${TAG}_$K python tools/profile_update.py > /dev/null 2>&1
  ncu -i gpurun_out/${TAG}_$K.ncu-rep --page raw --csv > gpurun_out/${TAG}_${K}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_$K.ncu-rep --page details --csv > gpurun_out/${TAG}_${K}_details.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_$K.ncu-rep --page source --csv > gpurun_out/${TAG}_${K}_source.csv 2>/dev/null
done
tail -3 gpurun_out/${TAG}_time.log; tail -1 gpurun_out/${TAG}_upd_launches.txt
