#!/bin/bash
# Round-end measurement set (one gpurun call): default bench line, reference arm, apply / PCG-iteration launch lists
# (ncu, serialised), ncu --set full of the fine SpMV and the level-1 SpMV, update_D launch list.
TAG=${1:-r02}
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
ncu --nvtx --nvtx-include "apply/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_apply_launches.csv python tools/profile_apply.py 3 > /dev/null 2>&1
python tools/launches.py gpurun_out/${TAG}_apply_launches.csv > gpurun_out/${TAG}_apply_launches.txt
AMGF_HOST_LOOP=1 ncu --nvtx --nvtx-include "pcg/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_pcg_launches.csv python tools/profile_pcg_iter.py > /dev/null 2>&1
python tools/launches.py gpurun_out/${TAG}_pcg_launches.csv > gpurun_out/${TAG}_pcg_launches.txt
ncu --nvtx --nvtx-include "upd/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_upd_launches.csv python tools/profile_update.py > /dev/null 2>&1
python tools/launches.py gpurun_out/${TAG}_upd_launches.csv > gpurun_out/${TAG}_upd_launches.txt
ncu --nvtx --nvtx-include "apply/" --set full --clock-control none -k regex:"k_sell" -c 6 -o gpurun_out/${TAG}_sell_full \
    python tools/profile_apply.py 3 > /dev/null 2>&1
ncu -i gpurun_out/${TAG}_sell_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_sell_full_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_sell_full.ncu-rep
tail -c 300 gpurun_out/${TAG}_bench.json; tail -1 gpurun_out/${TAG}_apply_launches.txt
